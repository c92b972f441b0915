MESHREG_B200_DEBUG=1 timeout 1500 python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo rc=$?
grep -E "grid|generic path|^\{" gpurun_out/bench_c5.log | cut -c1-700 | tail -4
