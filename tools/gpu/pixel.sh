#!/bin/sh
# Pixel engine: GPU pixel tests, bench line, ncu --set full of k_pixel_step
# (one GPU).  Usage: sh tools/gpu/pixel.sh TAG
T=${1:-pix}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_pixel.py -m gpu -x -q -s -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/${T}_tests.log
python bench.py --workload pixel --no-cpu-baseline > gpurun_out/${T}_bench.json 2>&1; echo bench rc=$?
python -c "import json; d=json.loads(open('gpurun_out/${T}_bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['kernel_ms'], d['roofline']['frac'])"
ncu --set full --clock-control none --import-source on -k regex:"k_pixel_step" -s 5 -c 1 -o gpurun_out/${T}_full python bench.py --workload pixel --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_ncu.log 2>&1; echo ncu rc=$?
