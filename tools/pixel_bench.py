"""Timing of the pixel-grid engine on BASELINE-sized 512x512 pairs:
python tools/pixel_bench.py [pairs] [precision] [iterations] [runs]."""
import sys
import time

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))

from paper_1411_2141_b200.baseline import PixelBatch
from paper_1411_2141_b200.synthetic import CONFIGS, make_pair

P = int(sys.argv[1]) if len(sys.argv) > 1 else 64
prec = sys.argv[2] if len(sys.argv) > 2 else "f32"
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 100
runs = int(sys.argv[4]) if len(sys.argv) > 4 else 2
pairs = [make_pair(CONFIGS["c2"], s) for s in range(P)]
re = np.ascontiguousarray(np.stack([p[0] for p in pairs]).astype(np.float32))
te = np.ascontiguousarray(np.stack([p[1] for p in pairs]).astype(np.float32))
b = PixelBatch(P, 512, 512, iterations=iters, precision=prec)
b.set_images(re, te)
for _ in range(runs):
    b.run()
    b.sync()
it, tot = b.kernel_times()
npx = P * 512 * 512
print(f"P={P} {prec} iters={iters}: fused iteration kernel {it * 1e3:.1f} us, run {tot:.2f} ms, "
      f"{npx / (it * 1e-3) / 1e9:.2f} Gpx/s per iteration")
b.close()
