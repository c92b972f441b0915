mkdir -p gpurun_out
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "coverage" > gpurun_out/san.log 2>&1; echo rc=$?
head -60 gpurun_out/san.log
