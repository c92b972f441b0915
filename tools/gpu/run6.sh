timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log | grep -E "FAILED|passed|failed|Error"
timeout 300 python tools/phase_profile.py 8 c4
for w in c1 c2 c4; do
timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; echo $w rc=$?
tail -1 gpurun_out/bench_$w.log | python -c "
import sys, json
d=json.loads(sys.stdin.readline()); print(d['config']['workload'][:40], d['value'], d['ms_per_step'], d['kernel_ms'])"
done
