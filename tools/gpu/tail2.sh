timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -1
MESHREG_B200_DEBUG=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "tail|^\{" | tail -2 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'], d['gpu_launches'])
    else: print(l.strip())"
