#!/bin/sh
# The GPU test suite with per-test durations and the achieved parity errors
# (-s prints them) into gpurun_out/gpu_tests.log.
python -m pytest tests -m gpu -x -q -s -p no:cacheprovider --durations=25 > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
