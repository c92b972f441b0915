timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x 2>&1 | tail -2
timeout 300 python tools/phase_profile.py 1 c2 2>&1 | tail -14
for w in c4 c2 c1 c3; do timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['ms_per_step'], d['path'])"; done
