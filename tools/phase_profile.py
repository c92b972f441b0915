"""Phase timing of the cluster kernel from clock64() stamps (debug aid).

usage: MESHREG_B200_PROFILE_PHASES=1 python tools/phase_profile.py [pairs] [workload]
(needs a library built with MRB_NVCC_FLAGS=-DMRB_PHASE_PROFILE)
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["MESHREG_B200_PROFILE_PHASES"] = "1"
import bench  # noqa: E402
from paper_1411_2141_b200 import _lib  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
wl = sys.argv[2] if len(sys.argv) > 2 else "c4"
lib = _lib.load()
ctx = _lib.context(0)
spec, _ = bench.workload_spec(wl)
pairs = [bench.load_pair(wl, s) for s in range(P)]
W = H = spec.size
cfg = _lib.mrb_config(0.005, 0.8, 0.0, spec.iterations, 1, _lib.PREC_F32, 0)
hs = bench.mesh_handles(lib, [(p[2], p[3]) for p in pairs])
arr = (C.c_void_p * P)(*hs)
b = C.c_void_p()
assert lib.mrb_batch_create(ctx, P, arr, W, H, _lib.F32, C.byref(cfg), C.byref(b)) == 0
re = np.ascontiguousarray(np.stack([p[0] for p in pairs]))
te = np.ascontiguousarray(np.stack([p[1] for p in pairs]))
lib.mrb_batch_set_images(b, re.ctypes.data, te.ctypes.data, 0)
for _ in range(2):
    lib.mrb_batch_run(b)
    lib.mrb_batch_sync(b)
cs = lib.mrb_batch_path(b)
n = P * cs * 8 * 16
buf = np.zeros(n, np.int64)
assert lib.mrb_batch_phase_profile(b, buf.ctypes.data, n) == 0
buf = buf.reshape(P * cs, 8, 16)
names = ["A sample", "cbar#1", "halo+ctl", "sync", "B grad", "sync_or", "(C start)", "cbar#2",
         "halo u0", "sync", "C smooth"]
slots = [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11]
d = np.diff(buf[:, 2:8, :12].astype(np.float64), axis=2)  # iterations 2..7
print(f"cluster size {cs}, {P} pairs; mean cycles per phase (iterations 2-7, all CTAs):")
tot = 0
for i, nm in enumerate(names):
    v = d[:, :, i]
    tot += v.mean()
    print(f"  {nm:10s} mean {v.mean():8.0f}  max {v.max():8.0f}")
it = np.diff(buf[:, 2:8, 0].astype(np.float64), axis=1)
print(f"  per-iteration {it.mean():.0f} cycles (sum of phases {tot:.0f})")
