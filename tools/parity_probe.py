"""Print the achieved fp32 error of every fast path against the fp64 oracle and
the fp32 emulation (tests/f32_emulation.py), by iteration count."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import meshreg_oracle as O  # noqa: E402
import paper_1411_2141_b200 as mrb  # noqa: E402
from f32_emulation import register32  # noqa: E402


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-30))


def probe(name, re32, te32, V, T, iters_list, paths):
    h, w = re32.shape
    om = O.Mesh(V, T)
    re = mrb.ImageGrid(w, h, re32.astype(np.float64))
    te = mrb.ImageGrid(w, h, te32.astype(np.float64))
    mesh = mrb.TriMesh(V, T)
    for it in iters_list:
        u_ref, info = O.register(re32, te32, om, max_iterations=it, energy_tolerance=0.0)
        u_emu, _ = register32(re32.astype(np.float64), te32.astype(np.float64), om, max_iterations=it)
        line = f"{name} it={it:4d} max|u|={np.abs(u_ref).max():7.3f} emu={rel(u_emu, u_ref):.2e}"
        for path in paths:
            os.environ.pop("MESHREG_B200_PATH", None)
            os.environ.pop("MESHREG_B200_EXCHANGE", None)
            if path in ("grid", "generic", "cluster"):
                os.environ["MESHREG_B200_PATH"] = path
            elif path in ("push", "pull"):
                os.environ["MESHREG_B200_PATH"] = "cluster"
                os.environ["MESHREG_B200_EXCHANGE"] = path
            u, rep, (ux, uy, wp) = mrb.register(re, te, mesh, mrb.SolverConfig(
                max_iterations=it, energy_tolerance=0.0), precision="f32", return_dense=True)
            line += (f" | {path}: u {rel(u, u_ref):.2e} vsemu {rel(u, u_emu):.2e}"
                     f" w {rel(wp, info['warped']):.2e} msd {abs(rep.msd_after / info['msd_after'] - 1):.1e}")
        print(line, flush=True)


if __name__ == "__main__":
    g = np.load(os.path.join(ROOT, "tests", "golden", "c1_x255.npz"))
    probe("c1_x255", g["re"], g["te"], g["V"], g["T_in"], [1, 2, 5, 10, 20, 50, 100],
          ["", "generic", "grid", "push", "pull"])
    if len(sys.argv) > 1:
        from paper_1411_2141_b200.synthetic import CONFIGS, make_pair
        m = np.load(os.path.join(ROOT, "data", "meshes", "c2_s0_x255.npz"))
        re, te = make_pair(CONFIGS["c2"], 0, scale=255.0)
        probe("c2_x255", re, te, m["V"], m["T"].astype(np.int64), [10, 50, 200],
              ["", "generic", "cluster"])
