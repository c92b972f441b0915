"""Run one pixel-engine configuration (subprocess-isolated debugging aid):
python tools/pix_dbg.py prec W H iterations passes lam"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_2141_b200.baseline import PixelBatch  # noqa: E402

prec, W, H, it, passes, lam = sys.argv[1], *map(int, sys.argv[2:6]), float(sys.argv[6])
rng = np.random.default_rng(0)
re = np.ascontiguousarray(rng.uniform(0, 255, (1, H, W)).astype(np.float32))
te = np.ascontiguousarray(rng.uniform(0, 255, (1, H, W)).astype(np.float32))
b = PixelBatch(1, W, H, 0.001, lam, it, passes, precision=prec)
b.set_images(re, te)
b.run()
print(prec, W, H, it, passes, lam, "->", b.sync()[0])
