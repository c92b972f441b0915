# host mesh build (mrb_mesh_build_many) + GPU suite + default bench
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu.log
nproc
timeout 600 python bench.py > gpurun_out/bench_c4.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_c4.log | python -c "
import sys,json; d=json.loads(sys.stdin.read()); e=d['e2e']; print(d['value'], d['ms_per_step'], e['value'], e['ms_per_step'], e['mesh_setup_ms_per_step'], e['value_with_mesh_setup'])"
