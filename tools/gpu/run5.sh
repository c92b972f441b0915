mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_gpu.log | grep -E "FAILED|passed|failed|Error" | head -20
for w in c1 c2 c4; do
MESHREG_B200_DEBUG=1 timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; echo $w rc=$?
grep meshreg_b200 gpurun_out/bench_$w.log | head -3
tail -1 gpurun_out/bench_$w.log | python -c "
import sys, json
d=json.loads(sys.stdin.readline()); print(d['config']['workload'][:60], d['value'], d['ms_per_step'], d['path'], d['kernel_ms'], d['roofline']['frac'])"
done
B="python bench.py --workload c4 --pairs 8 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cluster -s 1 -c 1 -o gpurun_out/prof_cluster3 $B > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
