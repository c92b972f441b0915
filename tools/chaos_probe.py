"""C3 x255: fp64 and fp32 paths against the fp64 oracle by iteration count."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import meshreg_oracle as O  # noqa: E402
import paper_1411_2141_b200 as mrb  # noqa: E402
from f32_emulation import register32  # noqa: E402
from paper_1411_2141_b200.synthetic import CONFIGS, make_pair  # noqa: E402


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-30))


spec = CONFIGS["c3"]
re32, te32 = make_pair(spec, 0, scale=255.0)
m = np.load(os.path.join(ROOT, "data", "meshes", "c3_s0_x255.npz"))
V, T = m["V"], m["T"].astype(np.int64)
om = O.Mesh(V, T)
re = mrb.ImageGrid(1024, 1024, re32.astype(np.float64))
te = mrb.ImageGrid(1024, 1024, te32.astype(np.float64))
mesh = mrb.TriMesh(V, T)
for it in (5, 10, 20, 50, 100, 200):
    u_ref, info = O.register(re32, te32, om, max_iterations=it, energy_tolerance=0.0)
    line = f"it={it:4d} max|u|={np.abs(u_ref).max():6.2f} E={info['energy_trace'][-1]:.6e}"
    if it <= 20:
        ue, _ = register32(re32.astype(np.float64), te32.astype(np.float64), om, max_iterations=it)
        line += f" emu32 {rel(ue, u_ref):.2e}"
    for prec in ("f64", "f32"):
        u, rep, (ux, uy, wp) = mrb.register(re, te, mesh, mrb.SolverConfig(
            max_iterations=it, energy_tolerance=0.0), precision=prec, return_dense=True)
        line += (f" | {prec}: u {rel(u, u_ref):.2e} w {rel(wp, info['warped']):.2e} "
                 f"trace {rel(rep.energy_trace, info['energy_trace']):.1e}")
    print(line, flush=True)
