timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "paths_agree or golden or batch or pipelined" 2>&1 | tail -3
for w in c4 c2 c1; do MESHREG_B200_DEBUG=1 timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -E "exchange|^\{" | tail -2 | cut -c1-160; done
for w in c4 c2; do MESHREG_B200_EXCHANGE=pull timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-160; done
