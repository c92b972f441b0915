# C4 with the tail split: launch list + ncu --set full of the main cluster kernel,
# the tail's push kernel and the dense pass
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/plain.log 2>&1; echo plain rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4d.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cluster_register|k_cluster_push|k_dense_fast" -s 3 -c 3 -o gpurun_out/prof_c4d $B > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
