timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "grid or path_selection" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -x -k "c3 or c5" 2>&1 | tail -2
MESHREG_B200_DEBUG=1 timeout 300 python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -E "grid|^\{" | tail -2 | cut -c1-160
MESHREG_B200_GRID_SYNC=barrier timeout 300 python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-160
