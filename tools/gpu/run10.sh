timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu.log | grep -E "FAILED|passed|failed|Error"
MESHREG_B200_DEBUG=1 timeout 600 python tools/e2e_breakdown.py 64 2>&1 | grep -v candidate | tail -7
