#!/bin/sh
# Round profile set (one GPU): bench lines for every workload, the reference
# arm, launch lists and ncu --set full captures of the dominant kernels.
# Usage: sh tools/gpu/profile_all.sh TAG   (outputs in gpurun_out/TAG_*)
T=${1:-r02}
mkdir -p gpurun_out
B="python bench.py"
$B > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err; echo c4 rc=$?
$B --precision f64 --no-cpu-baseline > gpurun_out/${T}_bench_c4_f64.json 2>&1; echo c4f64 rc=$?
for w in c1 c2 c3; do $B --workload $w --no-cpu-baseline > gpurun_out/${T}_bench_$w.json 2>&1; echo $w rc=$?; done
$B --workload c5 --steps 3 > gpurun_out/${T}_bench_c5.json 2>&1; echo c5 rc=$?
$B --workload pixel > gpurun_out/${T}_bench_pixel.json 2>&1; echo pixel rc=$?
$B --impl reference > gpurun_out/${T}_bench_ref.json 2>&1; echo ref rc=$?
Q="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c4_launches.csv $B $Q > /dev/null 2>&1; echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_cluster_push|k_dense_fast" -s 3 -c 3 -o gpurun_out/${T}_c4_full $B $Q > gpurun_out/${T}_c4_ncu.log 2>&1; echo c4 ncu rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_grid_flags" -s 1 -c 1 -o gpurun_out/${T}_c3_full $B --workload c3 $Q > gpurun_out/${T}_c3_ncu.log 2>&1; echo c3 ncu rc=$?
ncu --set full --clock-control none -k regex:"k_grid_flags" -s 1 -c 1 -o gpurun_out/${T}_c5_full $B --workload c5 $Q > gpurun_out/${T}_c5_ncu.log 2>&1; echo c5 ncu rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_pixel_step" -s 5 -c 1 -o gpurun_out/${T}_pixel_full $B --workload pixel $Q > gpurun_out/${T}_pixel_ncu.log 2>&1; echo pixel ncu rc=$?
