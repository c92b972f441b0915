B="python bench.py --workload c2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/c2_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cluster_register" -s 2 -c 1 -o gpurun_out/prof_c2 $B > gpurun_out/ncu_c2.log 2>&1; echo ncu rc=$?
B3="python bench.py --workload c3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B3 > gpurun_out/c3_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_grid_register" -s 2 -c 1 -o gpurun_out/prof_c3 $B3 > gpurun_out/ncu_c3.log 2>&1; echo ncu rc=$?
