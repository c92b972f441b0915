timeout 900 python -m pytest tests/test_gpu_pixel.py -q -p no:cacheprovider > gpurun_out/pytest_pixel.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_pixel.log
timeout 600 python bench.py --workload pixel --steps 3 --warmup 3 > gpurun_out/bench_pixel.log 2>&1; echo bench rc=$?
tail -3 gpurun_out/bench_pixel.log
timeout 600 python bench.py --workload pixel --precision f64 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-400
timeout 900 python bench.py --impl reference --workload pixel --steps 1 --warmup 0 2>&1 | tail -1
B="python bench.py --workload pixel --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_pixel.csv $B > gpurun_out/ncu_launch_pixel.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pixel_iter" -s 5 -c 1 -o gpurun_out/prof_pixel $B > gpurun_out/ncu_full_pixel.log 2>&1; echo ncu2 rc=$?
