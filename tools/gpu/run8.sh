timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu.log | grep -E "FAILED|passed|failed|Error"
for w in c1 c2 c4; do
MESHREG_B200_DEBUG=1 timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; echo $w rc=$?
grep "meshreg_b200: cluster" gpurun_out/bench_$w.log | head -3
grep "candidate" gpurun_out/bench_$w.log | head -20
tail -1 gpurun_out/bench_$w.log | python -c "
import sys, json
d=json.loads(sys.stdin.readline()); print(d['config']['workload'][:40], d['value'], d['ms_per_step'], d['kernel_ms'])"
done
