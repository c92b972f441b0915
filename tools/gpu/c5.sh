timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -k c5 -x 2>&1 | tail -15
