timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c4.log 2>&1; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_c4.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['clocks'])"
