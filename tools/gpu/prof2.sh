timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -1
B2="python bench.py --workload c2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B2 > gpurun_out/c2_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cluster_push" -s 2 -c 1 -o gpurun_out/prof_c2_push $B2 > gpurun_out/ncu_c2.log 2>&1; echo ncu_c2 rc=$?
B3="python bench.py --workload c3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B3 > gpurun_out/c3_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_grid_flags" -s 2 -c 1 -o gpurun_out/prof_c3_flags $B3 > gpurun_out/ncu_c3.log 2>&1; echo ncu_c3 rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $B3 > /dev/null 2>&1; echo ncu_l rc=$?
