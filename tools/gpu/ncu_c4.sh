#!/bin/sh
# C4 (64 x 512^2, 200 it): plain run, launch list, ncu --set full of the loop
# kernels and the dense pass (one GPU).  Usage: sh tools/gpu/ncu_c4.sh TAG [bench args]
TAG=${1:-c4}; shift
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline $*"
mkdir -p gpurun_out
timeout 300 $B > gpurun_out/${TAG}_plain.json 2>&1; echo plain rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo launches rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_cluster|k_grid|k_dense_fast|k_sample" -s 3 -c 3 -o gpurun_out/${TAG}_full $B > gpurun_out/${TAG}_ncu_full.log 2>&1; echo full rc=$?
