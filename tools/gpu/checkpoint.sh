# round checkpoint: smoke, GPU tests, benches, ncu evidence for profiles/
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c4.log 2>&1; echo bench rc=$?
for w in c1 c2 c3; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; echo $w rc=$?; done
timeout 900 python bench.py --workload pixel --steps 3 --warmup 3 > gpurun_out/bench_pixel.log 2>&1; echo pixel rc=$?
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $B > gpurun_out/ncu_launch_c4.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cluster_register|k_dense_fast|k_pad_planar4" -s 3 -c 3 -o gpurun_out/prof_c4 $B > gpurun_out/ncu_full_c4.log 2>&1; echo ncu2 rc=$?
B3="python bench.py --workload c3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_grid_register" -s 2 -c 1 -o gpurun_out/prof_c3 $B3 > gpurun_out/ncu_c3.log 2>&1; echo ncu3 rc=$?
