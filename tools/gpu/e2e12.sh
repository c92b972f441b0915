# GPU suite + e2e device timeline + default bench
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu.log
MESHREG_B200_DEBUG=2 timeout 600 python tools/e2e_many.py 64 0 > gpurun_out/e2e_dbg.log 2>&1; tail -34 gpurun_out/e2e_dbg.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_c4.log | python -c "
import sys,json; d=json.loads(sys.stdin.read()); e=d['e2e']; print(d['value'], d['ms_per_step'], e['value'], e['ms_per_step'], e['mesh_setup_ms_per_step'], e['value_with_mesh_setup'])"
