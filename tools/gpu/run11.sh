for w in c3; do
timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; echo $w rc=$?
tail -1 gpurun_out/bench_$w.log | python -c "
import sys, json
d=json.loads(sys.stdin.readline()); print(d['config']['workload'][:50], d['value'], d['ms_per_step'], d['path'], d['kernel_ms'])"
done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_full.log
