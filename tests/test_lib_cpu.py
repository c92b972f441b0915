"""The C-ABI library loads and exports every symbol include/*.h declares; the
host-side mesh setup (no GPU needed) is bit-exact with the reference."""
import ctypes
import glob
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden
import paper_1411_2141_b200 as mrb
from paper_1411_2141_b200 import _lib


def declared_symbols():
    names = set()
    for hdr in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(hdr).read()
        names |= set(re.findall(r"\b(mrb_[a-z0-9_]+)\s*\(", text))
    return sorted(names)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.EXPORTED)
    assert b"sm_100a" in _lib.load().mrb_version()


@pytest.mark.parametrize("name", ["gen64", "gen64_x255", "gen64_p0", "gen96_tol", "plateau64",
                                  "accept_c3", "identical48", "c1"])
def test_native_mesh_setup_bit_exact(name):
    g = golden(name)
    mesh = mrb.TriMesh(g["V"], g["T_in"])
    assert np.array_equal(mesh.triangles, g["T"])
    if "ring_idx" in g.files:
        assert np.array_equal(np.concatenate(mesh.rings), g["ring_idx"])
        assert np.array_equal(np.concatenate(mesh.incident), g["inc_idx"])
        assert np.array_equal(mesh.edges, g["edges"])
        assert np.array_equal(mesh.valence, g["valence"])
        assert np.array_equal(mesh.boundary, g["boundary"])
    if "L_indptr" in g.files:
        L = mrb.build_laplacian(mesh)
        geom = mesh.geometry
        for key, A in (("L", L), ("gx", geom.grad_x_op), ("gy", geom.grad_y_op),
                       ("avg", geom.vertex_average_op)):
            assert np.array_equal(A.indptr, g[key + "_indptr"]), key
            assert np.array_equal(A.indices, g[key + "_indices"]), key
            assert np.array_equal(A.data, g[key + "_data"]), key
    if "areas" in g.files:
        geom = mesh.geometry
        assert np.array_equal(geom.areas, g["areas"])
        assert np.array_equal(geom.coeffs, g["coeffs"])
        assert np.array_equal(geom.vertex_areas, g["vertex_areas"])


def test_build_many_matches_single_builds():
    """mrb_mesh_build_many (host worker pool) gives the same meshes as one
    mrb_mesh_build each, and reports the lowest-index invalid mesh."""
    gs = [golden(n) for n in ("gen64", "c1", "plateau64", "accept_c3", "gen64_x255")]
    many = mrb.TriMesh.build_many([(g["V"], g["T_in"]) for g in gs] * 3)
    assert len(many) == 15
    for k, mesh in enumerate(many):
        g = gs[k % len(gs)]
        one = mrb.TriMesh(g["V"], g["T_in"])
        assert np.array_equal(mesh.triangles, one.triangles)
        assert np.array_equal(mesh.edges, one.edges)
        assert np.array_equal(np.concatenate(mesh.rings), np.concatenate(one.rings))
        for a, b in ((mrb.build_laplacian(mesh), mrb.build_laplacian(one)),
                     (mesh.geometry.vertex_average_op, one.geometry.vertex_average_op),
                     (mesh.geometry.grad_x_op, one.geometry.grad_x_op)):
            assert np.array_equal(a.indices, b.indices) and np.array_equal(a.data, b.data)
    assert mrb.TriMesh.build_many([]) == []
    bad = [(gs[0]["V"], gs[0]["T_in"]), ([(0, 0), (1, 0), (2, 0)], [(0, 1, 2)]),
           ([(0, 0), (1, 0), (0, 1)], [(0, 1, 3)])]
    with pytest.raises(ValueError) as e:
        mrb.TriMesh.build_many(bad)
    assert str(e.value) == "degenerate triangle 0 (area 0)"


def test_mesh_validation_messages_match_reference():
    # texts of mesh.py:61-123
    with pytest.raises(ValueError, match=r"vertices must be \(n, 2\)"):
        mrb.TriMesh(np.zeros((3, 3)), [(0, 1, 2)])
    with pytest.raises(ValueError, match="with m >= 1"):
        mrb.TriMesh(np.zeros((3, 2)), np.zeros((0, 3)))
    with pytest.raises(ValueError, match="vertex coordinates must be finite"):
        mrb.TriMesh([(0, 0), (1, np.nan), (0, 1)], [(0, 1, 2)])
    with pytest.raises(ValueError, match="triangle index out of range"):
        mrb.TriMesh([(0, 0), (1, 0), (0, 1)], [(0, 1, 3)])
    with pytest.raises(ValueError, match="repeated vertex"):
        mrb.TriMesh([(0, 0), (1, 0), (0, 1)], [(0, 1, 1)])
    with pytest.raises(ValueError) as e:
        mrb.TriMesh([(0, 0), (1, 0), (2, 0)], [(0, 1, 2)])
    assert str(e.value) == "degenerate triangle 0 (area 0)"
    with pytest.raises(ValueError, match="non-manifold"):
        mrb.TriMesh([(0, 0), (1, 0), (0, 1), (0, -1), (0.3, 0.7)],
                    [(0, 1, 2), (0, 1, 3), (0, 1, 4)])


def test_orientation_and_known_answers():
    # square split on the diagonal, one triangle clockwise (mesh.py:79-82)
    m = mrb.TriMesh([(0.0, 0.0), (1.0, 0.0), (1.0, 1.0), (0.0, 1.0)], [(0, 2, 1), (0, 2, 3)])
    assert m.triangles.tolist() == [[0, 1, 2], [0, 2, 3]]
    # single triangle: L = [[0,.5,.5],[.5,0,.5],[.5,.5,0]] (test_mesh_ops.py:201-204)
    t = mrb.TriMesh([(0, 0), (1, 0), (0, 1)], [(0, 1, 2)])
    assert np.array_equal(mrb.build_laplacian(t).toarray(),
                          np.array([[0, .5, .5], [.5, 0, .5], [.5, .5, 0]]))
    assert m.boundary.all()


def test_solver_config_validation():
    with pytest.raises(ValueError):
        mrb.SolverConfig(tau=0.0)
    with pytest.raises(ValueError):
        mrb.SolverConfig(lam=1.0)
    with pytest.raises(ValueError):
        mrb.SolverConfig(max_iterations=0)
    with pytest.raises(ValueError):
        mrb.SolverConfig(smoothing_passes=-1)
    cfg = mrb.SolverConfig()
    assert (cfg.tau, cfg.lam, cfg.max_iterations, cfg.smoothing_passes) == (0.005, 0.8, 100, 1)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    img = mrb.ImageGrid(4, 4, np.arange(16.0))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        img.sample(1.5, 1.5)


def test_locate_and_scalar_mesh_helpers():
    """PointLocator/locate (densefield.py:62-127) through the native host
    locator, and the scalar helpers triangle_gradient / vertex_gradient /
    umbrella (mesh.py:216-251) — host-side, no GPU."""
    import paper_1411_2141_b200 as mrb
    g = golden("gen64")
    mesh = mrb.TriMesh(g["V"], g["T_in"])
    loc = mrb.PointLocator(mesh)
    h, w = g["re"].shape
    for q in (0, 17, 64 * 31 + 5, h * w - 1):  # pixel-map golden: tri + weights
        x, y = q % w, q // w
        t, wts = mrb.locate(loc, (x, y))
        assert t == int(g["tri_of"].reshape(-1)[q])
        if "pm_weights" in g.files:
            assert np.array_equal(wts, g["pm_weights"].reshape(-1, 3)[q])
    with pytest.raises(mrb.MeshCoverageError, match=r"point \(-5\.0, 3\.5\) not covered"):
        mrb.locate(loc, (-5.0, 3.5))
    import meshreg_oracle as O
    m = O.Mesh(g["V"], g["T_in"])
    geom = mrb.TriangleGeometry(mesh)
    f = np.sin(g["V"][:, 0] / 7.0) + g["V"][:, 1] / 13.0
    gt = mrb.triangle_gradient(geom, 5, f)
    assert gt == tuple(float(v) for v in f[m.T[5]] @ m.coeffs[5])  # oracle geometry
    gv = mrb.vertex_gradient(mesh, geom, f, 3)
    a = geom.areas[mesh.incident[3]]
    gr = np.einsum("tc,tcd->td", f[geom.triangles[mesh.incident[3]]], geom.coeffs[mesh.incident[3]])
    assert gv == tuple(float(v) for v in (a[:, None] * gr).sum(axis=0) / a.sum())
    u = np.stack([f, 2 * f], axis=1)
    assert np.array_equal(mrb.umbrella(mesh, u, 3), u[mesh.rings[3]].mean(axis=0) - u[3])
    assert mrb.umbrella(mesh, f, 3) == float(f[mesh.rings[3]].mean() - f[3])
