import ctypes as C, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_1411_2141_b200 import _lib
lib = _lib.load(); ctx = _lib.context(0)
spec, _ = bench.workload_spec(sys.argv[1])
pairs = [bench.load_pair(sys.argv[1], 0)]
W = H = spec.size
cfg = _lib.mrb_config(0.005, 0.8, 0.0, spec.iterations, 1, _lib.PREC_F32, 0)
re_h = torch.from_numpy(np.stack([p[0] for p in pairs])).pin_memory()
te_h = torch.from_numpy(np.stack([p[1] for p in pairs])).pin_memory()
n_tot = sum(len(p[2]) for p in pairs)
u_h = torch.empty((n_tot, 2), dtype=torch.float64).pin_memory()
mesh_in = [(np.ascontiguousarray(p[2]), np.ascontiguousarray(p[3], np.int64)) for p in pairs]
for rep in range(3):
    t0 = time.perf_counter()
    hs = bench.mesh_handles(lib, mesh_in, deferred=True)
    tm = time.perf_counter() - t0
    arr = (C.c_void_p * 1)(*hs)
    rc = lib.mrb_register_many(ctx, 1, arr, W, H, _lib.F32, re_h.data_ptr(), te_h.data_ptr(), C.byref(cfg), 0, _lib.F32,
                               u_h.data_ptr(), None, None, None, None, None, None, None, None, None, 0)
    print(f"rep {rep}: rc {rc} {1e3*(time.perf_counter()-t0):.1f} ms (handles {1e3*tm:.1f})", flush=True)
    for h in hs: lib.mrb_mesh_destroy(h)
