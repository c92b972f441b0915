"""Time mrb_register_many end to end (debug aid)."""
import ctypes as C, os, sys, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
from paper_1411_2141_b200 import _lib
P = int(sys.argv[1]) if len(sys.argv) > 1 else 64
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 0
deferred = len(sys.argv) > 3 and sys.argv[3] == "dev"  # device mesh setup, timed
report_only = len(sys.argv) > 4 and sys.argv[4] == "report"  # no dense outputs
lib = _lib.load(); ctx = _lib.context(0)
spec, _ = bench.workload_spec("c4")
pairs = [bench.load_pair("c4", s) for s in range(P)]
pairs = [(p[0], p[1], np.ascontiguousarray(p[2]), np.ascontiguousarray(p[3], np.int64)) + tuple(p[4:])
         for p in pairs]
W = H = spec.size
cfg = _lib.mrb_config(0.005, 0.8, 0.0, spec.iterations, 1, _lib.PREC_F32, 0)
re_h = torch.from_numpy(np.stack([p[0] for p in pairs])).pin_memory()
te_h = torch.from_numpy(np.stack([p[1] for p in pairs])).pin_memory()
n_tot = sum(len(p[2]) for p in pairs)
u_h = torch.empty((n_tot, 2), dtype=torch.float64).pin_memory()
dense = [torch.empty((P, H, W), dtype=torch.float32).pin_memory() for _ in range(3)]
for rep in range(3):
    t0 = time.perf_counter()
    hs = bench.mesh_handles(lib, [(p[2], p[3]) for p in pairs], deferred=deferred)
    t_mesh = time.perf_counter() - t0
    arr = (C.c_void_p * P)(*hs)
    rc = lib.mrb_register_many(ctx, P, arr, W, H, _lib.F32, re_h.data_ptr(), te_h.data_ptr(), C.byref(cfg), chunk, _lib.F32,
                               u_h.data_ptr(), *((None,) * 3 if report_only else (d.data_ptr() for d in dense)), None, None, None, None, None, None, 0)
    print(f"rep {rep}: rc {rc} {1e3*(time.perf_counter()-t0):.1f} ms (mesh handles {1e3*t_mesh:.1f} ms)"
          + (f" ({lib.mrb_last_error(ctx).decode()})" if rc else ""), flush=True)
    for h in hs: lib.mrb_mesh_destroy(h)
