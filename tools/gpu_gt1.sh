python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -s -p no:cacheprovider --durations=15 > gpurun_out/gt1.log 2>&1
echo rc=$?
