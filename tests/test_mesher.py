"""Content-adaptive mesher against the reference's
own outputs (tests/golden/mesher.npz, made by make_mesher_golden.py from the
reference meshgen.py / delaunay.py), bit for bit.

CPU tests cover the host-native stages (Delaunay, flips, de-duplication,
uniform layout, Floyd-Steinberg, halftone thinning, CVT/ODT smoothing fed the
reference's gradient magnitude) through the C ABI; `gpu` tests cover the GPU
front end (gradient magnitude, Canny, samplers), the whole generate_mesh
pipeline and the GPU Delaunay audit, and at full size the BASELINE C1-C3
meshes the reference mesher produced (data/meshes).
"""
import ctypes as C
import importlib
import os

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
from paper_1411_2141_b200 import _lib
D = importlib.import_module("paper_1411_2141_b200.delaunay")
from paper_1411_2141_b200 import meshgen as G
from paper_1411_2141_b200.image import ImageGrid
from paper_1411_2141_b200.mesh import TriMesh

GM = np.load(os.path.join(GOLDEN, "mesher.npz"), allow_pickle=False)
IMAGES = [str(n) for n in GM["image_names"]]
POINTS = [str(n) for n in GM["point_names"]]


def arrays(tris):
    return tris.arrays()


# ---------------------------------------------------------------------------
# host-native stages (no GPU)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", POINTS)
def test_delaunay_bit_exact(name):
    """dedupe_points + Bowyer-Watson + flip_edges(100) (delaunay.py:30-178):
    vertices and triangle ids identical to the reference's."""
    P = GM[f"pts_{name}"]
    assert np.array_equal(D.dedupe_points(P), GM[f"dedupe_{name}"])
    V, T = D._delaunay_tris(P).arrays()
    assert np.array_equal(V, GM[f"delV_{name}"])
    assert np.array_equal(T, GM[f"delT_{name}"])


def test_delaunay_order_independent_and_tie_break():
    """test_delaunay.py:58-68,116-127: the lexicographic diagonal of a
    cocircular square; the same set in another order gives the same mesh."""
    a = D._delaunay_tris(GM["pts_rand40"]).arrays()
    b = D._delaunay_tris(GM["pts_rand40rev"]).arrays()
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    V, T = D._delaunay_tris(GM["pts_square"]).arrays()
    idx = {tuple(v): i for i, v in enumerate(V.tolist())}
    edges = {tuple(sorted((int(t[k]), int(t[(k + 1) % 3])))) for t in T for k in range(3)}
    assert tuple(sorted((idx[(0.0, 0.0)], idx[(1.0, 1.0)]))) in edges
    assert tuple(sorted((idx[(1.0, 0.0)], idx[(0.0, 1.0)]))) not in edges


def test_dedupe_tolerance_and_errors():
    assert np.array_equal(D.dedupe_points(GM["dedupe_tol_in"]), GM["dedupe_tol_out"])
    with pytest.raises(ValueError, match="finite"):
        D.dedupe_points([[0.0, np.nan]])
    with pytest.raises(ValueError, match="at least 3"):
        D._delaunay_tris([(0, 0), (1, 1)])
    with pytest.raises(ValueError, match="collinear"):
        D._delaunay_tris([(0, 0), (1, 1), (2, 2), (3, 3)])
    with pytest.raises(ValueError, match="at least 3"):
        D._delaunay_tris([(0, 0), (0, 0), (1, 1)])


def _flip(V, T, passes):
    h = C.c_void_p()
    err = C.create_string_buffer(256)
    V = np.ascontiguousarray(V, np.float64)
    T = np.ascontiguousarray(T, np.int64)
    assert _lib.load().mrb_tris_create(len(V), _lib.ptr(V), len(T), _lib.ptr(T), C.byref(h),
                                       err, 256) == 0, err.value
    t = D._Tris(h.value)
    changed = t.flip(passes)
    return changed, t.arrays()[1]


def test_flip_constructed_violation():
    """test_delaunay.py:137-148: the non-Delaunay diagonal is replaced."""
    changed, T = _flip(GM["flipc_V"], GM["flipc_T"], 8)
    assert changed > 0
    assert np.array_equal(T, GM["flipc_outT"])


@pytest.mark.parametrize("trial", range(5))
def test_flip_perturbed_meshes(trial):
    """test_delaunay.py:150-175: flip_edges(passes=50) of perturbed meshes,
    same triangles as the reference."""
    _, T = _flip(GM[f"flipp{trial}_V"], GM[f"flipp{trial}_T"], 50)
    assert np.array_equal(T, GM[f"flipp{trial}_outT"])


def test_flip_fixed_point_returns_same_mesh():
    V, T = D._delaunay_tris(GM["pts_rand20"]).arrays()
    changed, T2 = _flip(V, T, 8)
    assert changed == 0 and np.array_equal(T, T2)


def test_uniform_layouts_bit_exact():
    for key in GM.files:
        if key.startswith("uniform_"):
            _, w, h, b = key.split("_")
            assert np.array_equal(G.uniform_sample(int(w), int(h), int(b)), GM[key]), key
    with pytest.raises(ValueError, match=">= 4"):
        G.uniform_sample(10, 10, 3)


def test_floyd_steinberg_bit_exact():
    for k in range(3):
        for s in (0, 1):
            assert np.array_equal(G._floyd_steinberg(GM[f"fs_in{k}"], s), GM[f"fs_out{k}_{s}"])


@pytest.mark.parametrize("name", IMAGES)
def test_halftone_host_stage_bit_exact(name):
    """Pairwise mass, Floyd-Steinberg, seeded permutation and thinning fed
    the reference's gradient magnitude (meshgen.py:188-216)."""
    mag = GM[f"mag1.0_{name}"]
    for key, budget, spacing, seed in (("half", 60, 3.0, 3), ("half4", 40, 4.0, 9)):
        got = G._halftone_from_mag(mag, budget, spacing, seed)
        want = GM[f"{key}_{name}"]
        assert got.shape == want.reshape(-1, 2).shape and np.array_equal(got, want.reshape(-1, 2))


@pytest.mark.parametrize("name", IMAGES)
def test_smooth_mesh_host_stage_bit_exact(name):
    """CVT (4) + ODT (3) relaxation of the frozen-pipeline mesh with the
    reference's sigma-1.5 gradient magnitude (meshgen.py:269-327)."""
    V, T = GM[f"frozenV_{name}"], GM[f"frozenT_{name}"]
    h = C.c_void_p()
    err = C.create_string_buffer(256)
    lib = _lib.load()
    assert lib.mrb_tris_create(len(V), _lib.ptr(np.ascontiguousarray(V)), len(T),
                               _lib.ptr(np.ascontiguousarray(T)), C.byref(h), err, 256) == 0
    t = D._Tris(h.value)
    mag = np.ascontiguousarray(GM[f"mag1.5_{name}"])
    rows, cols = mag.shape
    assert lib.mrb_smooth_mesh(t.h, cols, rows, _lib.ptr(mag), 4, 3, err, 256) == 0, err.value
    V2, T2 = t.arrays()
    assert np.array_equal(V2, GM[f"smoothV_{name}"])
    assert np.array_equal(T2, GM[f"smoothT_{name}"])


def test_config_validation_messages():
    with pytest.raises(ValueError, match="sum"):
        G.NodeBudget(target_nodes=10, canny_fraction=0.5, halftone_fraction=0.5,
                     uniform_fraction=0.5)
    with pytest.raises(ValueError, match="target_nodes"):
        G.NodeBudget(target_nodes=3)
    with pytest.raises(ValueError, match="canny_low"):
        G.MeshGenConfig(canny_low=30.0, canny_high=10.0)
    with pytest.raises(ValueError, match="spacing"):
        G.MeshGenConfig(min_node_spacing=0.5)
    with pytest.raises(ValueError, match="counts"):
        G.MeshGenConfig(cvt_iterations=-1)


# ---------------------------------------------------------------------------
# GPU front end and the whole pipeline
# ---------------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("name", IMAGES)
def test_gradient_magnitude_and_canny_bit_exact(name):
    """Gaussian (scipy order), np.gradient, glibc hypot, sector thinning and
    hysteresis on the GPU equal the reference's arrays exactly."""
    data = GM[f"img_{name}"]
    for s in (1.0, 1.4, 1.5):
        assert np.array_equal(G.gradient_magnitude(data, s), GM[f"mag{s}_{name}"]), s
    assert np.array_equal(G.canny_edges(data, 1.4, 8.0, 24.0), GM[f"canny_{name}"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", IMAGES)
def test_samplers_bit_exact(name):
    data = GM[f"img_{name}"]
    img = ImageGrid(data.shape[1], data.shape[0], data)
    got = G.canny_sample(img, G.MeshGenConfig(), 50)
    assert np.array_equal(got, GM[f"cannypts_{name}"].reshape(-1, 2))
    got = G.canny_sample(img, G.MeshGenConfig(min_node_spacing=5.0), 100)
    assert np.array_equal(got, GM[f"cannypts5_{name}"].reshape(-1, 2))
    assert np.array_equal(G.halftone_sample(img, 60, 3.0, seed=3), GM[f"half_{name}"].reshape(-1, 2))
    assert len(G.canny_sample(img, G.MeshGenConfig(), 0)) == 0
    assert len(G.halftone_sample(img, 0, 3.0)) == 0


@pytest.mark.gpu
@pytest.mark.parametrize("name", IMAGES)
def test_generate_mesh_bit_exact(name):
    """The whole pipeline (meshgen.py:365-396) at two budgets / seeds, the
    frozen (no relaxation) variant, smooth_mesh and quality_stats."""
    data = GM[f"img_{name}"]
    img = ImageGrid(data.shape[1], data.shape[0], data)
    for target, seed in ((90, 1), (150, 3)):
        m = G.generate_mesh(img, G.NodeBudget(target_nodes=target), G.MeshGenConfig(seed=seed))
        assert np.array_equal(m.vertices, GM[f"genV_{name}_{target}"]), target
        assert np.array_equal(m.triangles, GM[f"genT_{name}_{target}"]), target
    frozen = G.generate_mesh(img, G.NodeBudget(target_nodes=100),
                             G.MeshGenConfig(seed=0, cvt_iterations=0, odt_iterations=0))
    assert np.array_equal(frozen.vertices, GM[f"frozenV_{name}"])
    assert np.array_equal(frozen.triangles, GM[f"frozenT_{name}"])
    sm = G.smooth_mesh(frozen, img, G.MeshGenConfig(cvt_iterations=4, odt_iterations=3))
    assert np.array_equal(sm.vertices, GM[f"smoothV_{name}"])
    q = G.quality_stats(m)
    want = GM[f"quality_{name}"]
    got = [q["n_nodes"], q["n_triangles"], q["n_edges"], q["min_area"], q["min_angle"],
           q["delaunay_violations"]]
    assert got[:3] == [int(x) for x in want[:3]] and got[5] == int(want[5])
    assert got[3] == want[3]
    assert abs(got[4] - want[4]) <= 1e-9 * max(abs(want[4]), 1.0)
    assert m.n_vertices - m.n_edges + m.n_triangles == 1  # Euler (test_meshgen.py:234-237)


@pytest.mark.gpu
def test_delaunay_violations_counts():
    for trial in range(5):
        V, T = GM[f"flipp{trial}_V"], GM[f"flipp{trial}_T"]
        mesh = TriMesh(V, T)
        assert D.delaunay_violations(mesh.vertices, mesh.triangles) == GM[f"flipp{trial}_viol"][0]
        fixed = D.flip_edges(mesh, passes=50)
        assert D.delaunay_violations(fixed.vertices, fixed.triangles) == GM[f"flipp{trial}_viol"][1]


@pytest.mark.gpu
@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["c1", "c2", "c3"])
def test_generate_mesh_full_size_matches_reference_mesher(cfg):
    """BASELINE configs 1-3: the mesh generate_mesh builds from the template
    equals, bit for bit, the one the reference mesher wrote (data/meshes,
    tools/make_meshes.py; ~3k, 12k and 50k nodes).  The seed-0 meshes are
    committed as tests/golden/refmesh_<cfg>_s0.npz (written by
    tools/make_meshes.py with the reference package in the build container)."""
    from paper_1411_2141_b200.synthetic import CONFIGS, make_pair
    path = os.path.join(ROOT, "tests", "golden", f"refmesh_{cfg}_s0.npz")
    if not os.path.exists(path):
        path = os.path.join(ROOT, "data", "meshes", f"{cfg}_s0.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} absent")
    ref = np.load(path)
    spec = CONFIGS[cfg]
    _, te = make_pair(spec, 0)
    img = ImageGrid(spec.size, spec.size, te.astype(np.float64))
    m = G.generate_mesh(img, G.NodeBudget(spec.target_nodes), G.MeshGenConfig(seed=0))
    assert np.array_equal(m.vertices, ref["V"])
    assert np.array_equal(m.triangles, ref["T"].astype(np.int64))
