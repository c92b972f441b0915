"""Time the mesher (generate_mesh) per BASELINE configuration, with a
per-stage breakdown.  GPU box: python tools/mesher_bench.py c1 c2 c3 c5

Prints one JSON line per configuration: node / triangle counts, total
seconds and the stages (GPU front end: Canny + magnitudes; native: samplers,
Delaunay, smoothing, flips).  The reference mesher's times for the same
meshes are in data/meshes/*.npz (mesher_seconds, measured in the build
container by tools/make_meshes.py).
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1411_2141_b200 as mrb  # noqa: E402
import importlib  # noqa: E402
D = importlib.import_module("paper_1411_2141_b200.delaunay")
from paper_1411_2141_b200 import meshgen as G  # noqa: E402
from paper_1411_2141_b200.synthetic import CONFIGS, make_pair  # noqa: E402


def stages(img, budget, cfg):
    t = {}
    w, h = img.width, img.height
    c0 = time.perf_counter()
    corners = np.array([[0.0, 0.0], [w - 1.0, 0.0], [0.0, h - 1.0], [w - 1.0, h - 1.0]])
    n_canny = int(round(budget.target_nodes * budget.canny_fraction))
    pc = G.canny_sample(img, cfg, n_canny)
    t["canny_sample"] = time.perf_counter() - c0
    c0 = time.perf_counter()
    n_half = int(round(budget.target_nodes * budget.halftone_fraction)) + (n_canny - len(pc))
    ph = G.halftone_sample(img, n_half, cfg.min_node_spacing, seed=cfg.seed)
    t["halftone_sample"] = time.perf_counter() - c0
    c0 = time.perf_counter()
    partial = D.dedupe_points(np.vstack([corners, pc, ph]))
    nu = budget.target_nodes - len(partial)
    pts = D.dedupe_points(np.vstack([partial, G.uniform_sample(w, h, nu)])) if nu >= 4 else partial
    t["uniform_dedupe"] = time.perf_counter() - c0
    c0 = time.perf_counter()
    tris = D._delaunay_tris(pts)
    t["delaunay"] = time.perf_counter() - c0
    c0 = time.perf_counter()
    G._smooth_tris(tris, img, cfg)
    t["smooth"] = time.perf_counter() - c0
    c0 = time.perf_counter()
    tris.flip(cfg.flip_passes)
    t["flip"] = time.perf_counter() - c0
    return tris.arrays(), t


def main(names):
    for name in names:
        spec = CONFIGS[name]
        _, te = make_pair(spec, 0)
        img = mrb.ImageGrid(spec.size, spec.size, te.astype(np.float64))
        budget, cfg = G.NodeBudget(spec.target_nodes), G.MeshGenConfig(seed=0)
        G.generate_mesh(mrb.ImageGrid(64, 64, te[:64, :64].astype(np.float64)),
                        G.NodeBudget(100), cfg)  # warm-up (context, module load)
        t0 = time.perf_counter()
        m = G.generate_mesh(img, budget, cfg)
        total = time.perf_counter() - t0
        (V, T), st = stages(img, budget, cfg)
        assert np.array_equal(V, m.vertices) and np.array_equal(T, m.triangles)
        rec = {"config": name, "image": spec.size, "nodes": int(len(V)), "triangles": int(len(T)),
               "generate_mesh_s": round(total, 4),
               "stages_s": {k: round(v, 4) for k, v in st.items()}}
        path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "data", "meshes", f"{name}_s0.npz")
        if os.path.exists(path):
            ref = np.load(path)
            same = bool(np.array_equal(ref["V"], V) and np.array_equal(ref["T"].astype(np.int64), T))
            if "mesher_seconds" in ref.files:  # written by the reference mesher
                rec["reference_mesher_s"] = float(ref["mesher_seconds"])
                rec["bit_identical_to_reference"] = same
            else:  # cached output of this package's mesher (bench.py)
                rec["identical_to_cached_package_mesh"] = same
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3"])
