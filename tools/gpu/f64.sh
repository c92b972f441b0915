for w in c4 c2; do timeout 600 python bench.py --workload $w --precision f64 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$w f64', d['value'], d['ms_per_step'], d['path'])"; done
