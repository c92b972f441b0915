#!/bin/sh
# fast-path parity subset + C4 bench (one GPU)
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -s -p no:cacheprovider -k "not c5_matches" > gpurun_out/quick_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/quick_tests.log
python bench.py --no-e2e --no-cpu-baseline > gpurun_out/quick_c4.json 2>&1; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/quick_c4.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['kernel_ms'])"
