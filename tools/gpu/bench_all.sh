timeout 900 python bench.py > gpurun_out/bench_c4.log 2>&1; echo c4 rc=$?
for w in c1 c2 c3; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; echo $w rc=$?; done
