"""Golden vectors for the content-adaptive mesher, produced by running the
REFERENCE mesher itself (pkg/src/meshreg/meshgen.py, delaunay.py).

Run in the build container only (imports /root/reference/pkg/src/meshreg):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_mesher_golden.py

Writes tests/golden/mesher.npz.  Inputs mirror the reference's own mesher
tests (test_meshgen.py, test_delaunay.py: random_smooth_image, step_image,
constant_image, the square / grid / random point sets, the constructed flip
violation, the perturbed-mesh flip audit) plus a x255 BASELINE-style pair;
outputs are the reference's results for every stage: gradient magnitudes,
Canny masks, sampler points, Floyd-Steinberg dots, uniform layouts,
de-duplication, Delaunay, flips, CVT/ODT smoothing, generate_mesh and
quality_stats.
"""
import importlib
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import meshreg as mr  # noqa: E402
from scipy import ndimage  # noqa: E402

G = importlib.import_module("meshreg.meshgen")
D = importlib.import_module("meshreg.delaunay")
from paper_1411_2141_b200.synthetic import PairSpec, make_pair  # noqa: E402


def smooth_image(w, h, seed, amplitude=60.0):
    """The reference conftest.random_smooth_image."""
    rng = np.random.default_rng(seed)
    data = ndimage.gaussian_filter(rng.standard_normal((h, w)), 2.0, mode="nearest")
    lo, hi = data.min(), data.max()
    return 120.0 + amplitude * (data - lo) / max(hi - lo, 1e-12) - amplitude / 2


def step_image(w, h, edge_col):
    data = np.full((h, w), 0.0)
    data[:, edge_col:] = 255.0
    return data


def main():
    out = {}
    # ---- images and the image-space stages -------------------------------
    spec = PairSpec("g", 64, 8, 0, 2.0, 400, 40)
    _, te255 = make_pair(spec, seed=3, scale=255.0)
    images = {
        "smooth48x40s9": smooth_image(48, 40, 9),
        "smooth64s8": smooth_image(64, 64, 8),
        "smooth96s10": smooth_image(96, 96, 10),
        "step32x24": step_image(32, 24, 10),
        "step64": step_image(64, 64, 20),
        "const64": np.full((64, 64), 50.0),
        "gen64x255": te255.astype(np.float64),
    }
    cfg = mr.MeshGenConfig()
    for name, data in images.items():
        h, w = data.shape
        img = mr.ImageGrid(w, h, data)
        out[f"img_{name}"] = data
        for s in (1.0, 1.4, 1.5):
            out[f"mag{s}_{name}"] = G._gradient_magnitude(data, s)
        out[f"canny_{name}"] = G._canny_edges(data, 1.4, 8.0, 24.0)
        out[f"cannypts_{name}"] = G.canny_sample(img, cfg, 50)
        out[f"cannypts5_{name}"] = G.canny_sample(img, mr.MeshGenConfig(min_node_spacing=5.0), 100)
        out[f"half_{name}"] = G.halftone_sample(img, 60, 3.0, seed=3)
        out[f"half4_{name}"] = G.halftone_sample(img, 40, 4.0, seed=9)
        for target, seed in ((90, 1), (150, 3)):
            m = G.generate_mesh(img, mr.NodeBudget(target_nodes=target), mr.MeshGenConfig(seed=seed))
            out[f"genV_{name}_{target}"] = m.vertices
            out[f"genT_{name}_{target}"] = m.triangles
        frozen = G.generate_mesh(img, mr.NodeBudget(target_nodes=100),
                                 mr.MeshGenConfig(seed=0, cvt_iterations=0, odt_iterations=0))
        out[f"frozenV_{name}"] = frozen.vertices
        out[f"frozenT_{name}"] = frozen.triangles
        sm = G.smooth_mesh(frozen, img, mr.MeshGenConfig(cvt_iterations=4, odt_iterations=3))
        out[f"smoothV_{name}"] = sm.vertices
        out[f"smoothT_{name}"] = sm.triangles
        q = G.quality_stats(m)
        out[f"quality_{name}"] = np.array([q["n_nodes"], q["n_triangles"], q["n_edges"],
                                           q["min_area"], q["min_angle"],
                                           q["delaunay_violations"]], dtype=np.float64)
    out["image_names"] = np.array(list(images))
    # ---- Floyd-Steinberg --------------------------------------------------
    rng = np.random.default_rng(4)
    dens = [np.full((40, 50), 0.12), np.full((40, 50), 0.35), rng.uniform(0, 0.6, (33, 47))]
    for k, dmap in enumerate(dens):
        for s in (0, 1):
            out[f"fs_in{k}"] = dmap
            out[f"fs_out{k}_{s}"] = G._floyd_steinberg(dmap, serpentine_start=s)
    # ---- uniform layouts --------------------------------------------------
    for (w, h, b) in ((100, 80, 4), (100, 100, 9), (100, 80, 5), (200, 150, 16), (200, 150, 25),
                      (200, 150, 40), (200, 150, 100), (200, 150, 500), (512, 512, 2399),
                      (64, 64, 96)):
        out[f"uniform_{w}_{h}_{b}"] = G.uniform_sample(w, h, b)
    # ---- point sets: dedupe, delaunay, flips ------------------------------
    pts = {
        "three": np.array([(0, 0), (2, 0), (0, 3)], float),
        "square": np.array([(0, 0), (1, 0), (0, 1), (1, 1)], float),
        "rand20": np.random.default_rng(7).uniform(0, 100, (20, 2)),
        "grid5x4": np.column_stack([a.ravel() for a in np.meshgrid(np.arange(5.0), np.arange(4.0))]),
        "rand120": np.random.default_rng(19).uniform(-50, 50, (120, 2)),
        "dups": np.array([(0, 0), (1, 0), (0, 1), (1e-12, 1e-12), (1, 0)], float),
        "rand40": np.random.default_rng(3).uniform(0, 10, (40, 2)),
        "rand40rev": np.random.default_rng(3).uniform(0, 10, (40, 2))[::-1].copy(),
        "grid30": np.column_stack([a.ravel() for a in np.meshgrid(np.arange(30.0), np.arange(30.0))]),
        "intpts": np.random.default_rng(5).integers(0, 60, (700, 2)).astype(float),
    }
    for name, P in pts.items():
        out[f"pts_{name}"] = P
        out[f"dedupe_{name}"] = D.dedupe_points(P)
        m = D.delaunay(P)
        out[f"delV_{name}"] = m.vertices
        out[f"delT_{name}"] = m.triangles
    out["point_names"] = np.array(list(pts))
    out["dedupe_tol_in"] = np.array([[0, 0], [0, 5e-10], [0, 2], [1, 1]], float)
    out["dedupe_tol_out"] = D.dedupe_points(out["dedupe_tol_in"])
    # constructed violation (test_delaunay.py:137-148)
    V = np.array([(0.0, 0.0), (4.0, 0.0), (2.0, 2.6), (2.0, -0.4)])
    T = np.array([(0, 1, 2), (1, 0, 3)])
    fixed = D.flip_edges(mr.build_adjacency(V, T), passes=8)
    out.update(flipc_V=V, flipc_T=T, flipc_outT=fixed.triangles)
    # perturbed meshes (test_delaunay.py:150-175)
    rng = np.random.default_rng(23)
    for trial in range(5):
        base = D.delaunay(rng.uniform(0, 40, (25, 2)))
        V = base.vertices.copy()
        T = base.triangles
        for i in np.nonzero(~base.boundary)[0]:
            proposal = V[i] + rng.uniform(-1.5, 1.5, 2)
            old = V[i].copy()
            V[i] = proposal
            a, b, c = V[T[:, 0]], V[T[:, 1]], V[T[:, 2]]
            ar = (b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (c[:, 0] - a[:, 0]) * (b[:, 1] - a[:, 1])
            if ar.min() < 1e-6:
                V[i] = old
        mesh = mr.build_adjacency(V, T)
        fixed = D.flip_edges(mesh, passes=50)
        out[f"flipp{trial}_V"] = V
        out[f"flipp{trial}_T"] = T
        out[f"flipp{trial}_outT"] = fixed.triangles
        out[f"flipp{trial}_viol"] = np.array([D.delaunay_violations(mesh.vertices, mesh.triangles),
                                              D.delaunay_violations(fixed.vertices, fixed.triangles)])
    path = os.path.join(HERE, "mesher.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB, {len(out)} arrays)")


if __name__ == "__main__":
    main()
