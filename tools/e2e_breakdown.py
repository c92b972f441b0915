"""Stage timing of one end-to-end batch registration through the C ABI (debug aid)."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1411_2141_b200 import _lib  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 64
lib = _lib.load()
ctx = _lib.context(0)
spec, _ = bench.workload_spec("c4")
pairs = [bench.load_pair("c4", s) for s in range(P)]
W = H = spec.size
cfg = _lib.mrb_config(0.005, 0.8, 0.0, spec.iterations, 1, _lib.PREC_F32, 0)
re_h = torch.from_numpy(np.stack([p[0] for p in pairs])).pin_memory()
te_h = torch.from_numpy(np.stack([p[1] for p in pairs])).pin_memory()
n_tot = sum(len(p[2]) for p in pairs)
u_h = torch.empty((n_tot, 2), dtype=torch.float64).pin_memory()
dense = [torch.empty((P, H, W), dtype=torch.float32).pin_memory() for _ in range(3)]
for rep in range(3):
    t = [time.perf_counter()]
    hs = bench.mesh_handles(lib, [(p[2], p[3]) for p in pairs])
    t.append(time.perf_counter())
    arr = (C.c_void_p * P)(*hs)
    b = C.c_void_p()
    assert lib.mrb_batch_create(ctx, P, arr, W, H, _lib.F32, C.byref(cfg), C.byref(b)) == 0
    lib.mrb_ctx_synchronize(ctx)
    t.append(time.perf_counter())
    lib.mrb_batch_set_images(b, re_h.data_ptr(), te_h.data_ptr(), 0)
    lib.mrb_ctx_synchronize(ctx)
    t.append(time.perf_counter())
    lib.mrb_batch_run(b)
    lib.mrb_ctx_synchronize(ctx)
    t.append(time.perf_counter())
    lib.mrb_batch_get_results(b, _lib.F32, u_h.data_ptr(), *(d.data_ptr() for d in dense))
    lib.mrb_batch_sync(b)
    t.append(time.perf_counter())
    lib.mrb_batch_destroy(b)
    for h in hs:
        lib.mrb_mesh_destroy(h)
    lib.mrb_ctx_synchronize(ctx)
    t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"rep {rep}: host mesh build {d[0]:.1f} | batch_create {d[1]:.1f} | set_images {d[2]:.1f} | "
          f"run {d[3]:.1f} | get_results+sync {d[4]:.1f} | destroy {d[5]:.1f} ms")
print("host cores", len(os.sched_getaffinity(0)))
