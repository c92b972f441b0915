mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_c4.log
timeout 600 python bench.py --steps 5 --warmup 3 --precision f64 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_f64.log 2>&1; echo bench64 rc=$?
tail -1 gpurun_out/bench_c4_f64.log
B="python bench.py --pairs 16 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sample -s 10 -c 2 -o gpurun_out/prof_sample $B > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
