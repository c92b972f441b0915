for w in c2 c4; do
MESHREG_B200_DEBUG=1 timeout 300 python bench.py --workload $w --steps 2 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -3 | python -c "
import sys, json
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print(d['config']['workload'], d['value'], d['ms_per_step'], d['path'], d['kernel_ms'], d['gpu_launches'], d['roofline'])
    else: print(l)
"
done
