timeout 900 python bench.py --impl reference --steps 1 --warmup 0 2>&1 | tail -1
timeout 600 python bench.py --workload c1 --steps 3 --warmup 3 2>&1 | tail -1 | cut -c1-200
