"""H2D copy rate of a 16 MB pinned buffer while the C4 loop kernel runs
(context for the e2e pipeline's topology copies) vs on an idle GPU."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1411_2141_b200 import _lib  # noqa: E402

lib = _lib.load()
ctx = _lib.context(0)
spec, _ = bench.workload_spec("c4")
pairs = [bench.load_pair("c4", s) for s in range(64)]
cfg = _lib.mrb_config(0.005, 0.8, 0.0, 200, 1, _lib.PREC_F32, 0)
hs = bench.mesh_handles(lib, [(p[2], p[3]) for p in pairs])
arr = (C.c_void_p * 64)(*hs)
b = C.c_void_p()
assert lib.mrb_batch_create(ctx, 64, arr, 512, 512, _lib.F32, C.byref(cfg), C.byref(b)) == 0
re = torch.from_numpy(np.stack([p[0] for p in pairs])).cuda()
te = torch.from_numpy(np.stack([p[1] for p in pairs])).cuda()
torch.cuda.synchronize()
lib.mrb_batch_set_images(b, re.data_ptr(), te.data_ptr(), 1)
lib.mrb_batch_run(b)
lib.mrb_batch_sync(b)
for mb in (16, 64):
    h = torch.empty(mb << 18, dtype=torch.float32).pin_memory()
    d = torch.empty(mb << 18, dtype=torch.float32, device="cuda")
    side = torch.cuda.Stream()
    for load in (False, True):
        torch.cuda.synchronize()
        if load:
            lib.mrb_batch_run(b)  # ~6 ms on the library's stream
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(side):
            e0.record(side)
            for _ in range(4):
                d.copy_(h, non_blocking=True)
            e1.record(side)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"{mb} MB x4 H2D {'during the C4 run' if load else 'idle GPU'}: "
              f"{4 * mb / 1024 / (ms / 1e3):.1f} GB/s", flush=True)
# the same copies right after the host wrote the pinned buffer (cache-hot,
# as the topology staging buffer is after write_topo)
for mb in (16,):
    h = torch.empty(mb << 18, dtype=torch.float32).pin_memory()
    d = torch.empty(mb << 18, dtype=torch.float32, device="cuda")
    hn = h.numpy()
    for rep in range(3):
        torch.cuda.synchronize()
        hn[:] = float(rep)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        print(f"{mb} MB H2D right after a host write: {mb / 1024 / (e0.elapsed_time(e1) / 1e3):.1f} GB/s",
              flush=True)
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        print(f"{mb} MB H2D again: {mb / 1024 / (e0.elapsed_time(e1) / 1e3):.1f} GB/s", flush=True)
