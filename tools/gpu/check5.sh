timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -1
for w in c2 c1; do timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_$w.log; python -c "
import json; d=json.loads(open('gpurun_out/bench_$w.log').read()); print('$w', d['value'], d['ms_per_step'], d['path'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['ms_per_step'])"; done
