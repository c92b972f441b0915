B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cluster_register|k_dense_fast|k_pad_planar4" -s 3 -c 3 -o gpurun_out/prof_c4 $B > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
