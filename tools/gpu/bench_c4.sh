timeout 900 python bench.py > gpurun_out/bench_c4.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_c4.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['clocks'])"
