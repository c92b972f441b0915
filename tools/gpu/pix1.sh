# pixel engine: parity tests + a first timing of the fused iteration kernel
timeout 900 python -m pytest tests/test_gpu_pixel.py -q -p no:cacheprovider -x > gpurun_out/pytest_pixel.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_pixel.log
timeout 300 python - <<'PY' 2>&1 | tail -20
import numpy as np, time
from paper_1411_2141_b200.baseline import PixelBatch
from paper_1411_2141_b200.synthetic import CONFIGS, make_pair
for P, prec in ((64, "f32"), (8, "f32"), (1, "f32"), (8, "f64")):
    re = np.stack([make_pair(CONFIGS["c2"], s)[0] for s in range(P)]).astype(np.float32)
    te = np.stack([make_pair(CONFIGS["c2"], s)[1] for s in range(P)]).astype(np.float32)
    b = PixelBatch(P, 512, 512, iterations=100, precision=prec)
    b.set_images(re, te)
    b.run(); b.sync(); b.run(); b.sync()
    it, tot = b.kernel_times()
    t0 = time.perf_counter(); b.run(); r = b.sync(); t1 = time.perf_counter()
    npx = P * 512 * 512
    print(f"P={P} {prec}: iter kernel {it*1e3:.1f} us, run(timed) {tot:.2f} ms, graph run wall {1e3*(t1-t0):.2f} ms,"
          f" {npx*100/(it*1e-3)/1e9:.1f} Gpx-iter/s, {16*npx/(it*1e-3)/1e9:.0f} GB/s(u r+w)", type(r[0]).__name__)
    b.close()
PY
