timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "paths_agree or path_selection" 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "c3" 2>&1 | tail -3
MESHREG_B200_DEBUG=1 timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "grid|^\{" | tail -3 | cut -c1-600
