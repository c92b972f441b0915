timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x 2>&1 | tail -2
timeout 300 python tools/push_profile.py 64 c4 2>&1 | tail -8
for w in c4 c2 c1; do timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-140; done
