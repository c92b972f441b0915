timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
timeout 1500 python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-200
MESHREG_B200_GRID_SYNC=barrier timeout 1500 python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-200
