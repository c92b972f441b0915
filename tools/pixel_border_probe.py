"""Pixel engine: iteration-kernel time for the same pixel count at three image sizes
(the share of border / ragged tiles falls with the size): python tools/pixel_border_probe.py"""
import sys, os
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_1411_2141_b200.baseline import PixelBatch
from paper_1411_2141_b200.synthetic import CONFIGS, make_pair
def run(P, cfg, size):
    pairs = [make_pair(CONFIGS[cfg], s) for s in range(P)]
    re = np.ascontiguousarray(np.stack([p[0] for p in pairs]).astype(np.float32))
    te = np.ascontiguousarray(np.stack([p[1] for p in pairs]).astype(np.float32))
    b = PixelBatch(P, size, size, iterations=100, precision="f32")
    b.set_images(re, te)
    for _ in range(3):
        b.run(); b.sync()
    it, tot = b.kernel_times()
    print(f"P={P} {size}^2: iteration kernel {it*1e3:.1f} us, {P*size*size/(it*1e-3)/1e9:.2f} Gpx/s", flush=True)
    b.close()
run(64, "c2", 512)
run(16, "c3", 1024)
run(1, "c5", 4096)
