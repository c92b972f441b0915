"""Debug aid: run one fast-path batch and print each CTA's progress markers
(host-mapped, readable while the kernel runs)."""
import ctypes as C
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ["MESHREG_B200_PROFILE_PHASES"] = "mapped"
from paper_1411_2141_b200 import _lib  # noqa: E402
import paper_1411_2141_b200 as mrb  # noqa: E402
from conftest import golden  # noqa: E402

g = golden(sys.argv[1])
lib = _lib.load()
ctx = _lib.context()
mesh = mrb.TriMesh(g["V"], g["T_in"])
H, W = g["re"].shape
cfg = _lib.mrb_config(0.001, 0.8, 0.0, int(os.environ.get("IT", "1")), int(os.environ.get("PASSES", "1")), _lib.PREC_F32, 0)
arr = (C.c_void_p * 1)(mesh._h)
b = C.c_void_p()
assert lib.mrb_batch_create(ctx, 1, arr, W, H, _lib.F32, C.byref(cfg), C.byref(b)) == 0
re = np.ascontiguousarray(g["re"].astype(np.float32))
te = np.ascontiguousarray(g["te"].astype(np.float32))
lib.mrb_batch_set_images(b, re.ctypes.data, te.ctypes.data, 0)
cs = lib.mrb_batch_path(b)
done = []
th = threading.Thread(target=lambda: done.append(lib.mrb_batch_run(b) or lib.mrb_batch_sync(b)),
                      daemon=True)
th.start()
time.sleep(3)
buf = np.zeros(cs * 128, np.int64)
lib.mrb_batch_phase_profile(b, buf.ctypes.data, buf.size)
buf = buf.reshape(cs, 128)[:, :6]
print("finished" if done else "HUNG", "cs", cs)
for r in range(cs):
    print(r, buf[r].tolist())
os._exit(0)
