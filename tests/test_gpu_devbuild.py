"""Device-side mesh setup (meshbuild.cuh) against the host build.

mrb_mesh_device_check builds a deferred mesh and one cluster topology on the
GPU and compares every array the fast path reads with the host build
(mesh_host.cpp build_mesh, plan_topo + write_topo): device-order vertices,
triangles, node order, fp32 self terms and 1/valence, the one-ring CSR, the
fp64 fused operator and the topology bytes must be identical.  Registration
through deferred handles must equal registration through TriMesh bit for bit.
"""
import numpy as np
import pytest

import paper_1411_2141_b200 as mrb
from conftest import GOLDEN_CASES, golden

pytestmark = pytest.mark.gpu

# cluster shapes and whole-GPU grid shapes (148 CTAs, up to 8 nodes per thread)
SHAPES = [(1, 1), (2, 2), (4, 1), (9, 2), (16, 1), (16, 2), (148, 1), (148, 4)]


def perturbed_grid(k, seed):
    from bench import fallback_mesh
    V, T = fallback_mesh(511, k * k)
    rng = np.random.default_rng(seed)
    V = V + rng.uniform(-0.3, 0.3, V.shape)
    T = T.copy()
    T[1::2] = T[1::2][:, [0, 2, 1]]  # clockwise input triangles
    return V, T


def cases():
    out = []
    for name in GOLDEN_CASES:
        g = golden(name)
        out.append((name, g["V"], g["T_in"].astype(np.int64)))
    # 1.6k, 12k, 24k nodes (one 8-CTA cluster per mesh) and 44k nodes (the
    # grid-wide build kernels of large meshes)
    for k, seed in ((40, 0), (110, 1), (156, 2), (210, 3)):
        V, T = perturbed_grid(k, seed)
        out.append((f"grid{k}", V, T))
    return out


@pytest.mark.parametrize("name,V,T", cases(), ids=[c[0] for c in cases()])
def test_device_build_bit_identical_to_host(name, V, T):
    for cs, npt in SHAPES:
        if len(V) > cs * 768 * npt:
            continue
        d = mrb.DeferredMesh.create_many([(V, T)])[0]
        mism = d.device_check(cs, npt)
        assert not mism.any(), (name, cs, npt, mism.tolist())


def test_mesher_meshes_device_build():
    """Content-adaptive meshes of the package mesher (the bench's C4 meshes,
    bit-identical to the reference mesher's) in the C4 shapes."""
    from paper_1411_2141_b200.synthetic import CONFIGS, make_pair
    spec = CONFIGS["c2"]
    for seed in (0, 1):
        _, te = make_pair(spec, seed)
        m = mrb.generate_mesh(mrb.ImageGrid(spec.size, spec.size, te.astype(np.float64)),
                              mrb.NodeBudget(spec.target_nodes), mrb.MeshGenConfig(seed=0))
        for cs, npt in ((9, 2), (16, 1)):
            d = mrb.DeferredMesh.create_many([(m.vertices, m.triangles)])[0]
            mism = d.device_check(cs, npt)
            assert not mism.any(), (seed, cs, npt, mism.tolist())


@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_register_batch_deferred_equals_trimesh(precision):
    """The golden pairs through DeferredMesh handles (device setup; fp64: the
    fp64 self terms and double2 cluster topologies too) and through TriMesh
    (host setup): identical fields, reports and dense outputs."""
    names = ["gen64", "plateau64", "gen64_x255", "gen96_tol", "c1", "gen64", "accept_c3"]
    res, tes, VT = [], [], []
    for n in names:
        g = golden(n)
        h, w = g["re"].shape
        res.append(g["re"])
        tes.append(g["te"])
        VT.append((g["V"], g["T_in"]))
    cfg = mrb.SolverConfig(tau=0.002, max_iterations=60, energy_tolerance=0.0)
    for size in sorted({r.shape for r in res}):
        idx = [k for k, r in enumerate(res) if r.shape == size]
        H, W = size
        rr = [mrb.ImageGrid(W, H, res[k]) for k in idx]
        tt = [mrb.ImageGrid(W, H, tes[k]) for k in idx]
        host = mrb.register_batch(rr, tt, [mrb.TriMesh(*VT[k]) for k in idx], cfg,
                                  precision=precision, return_dense=True)
        dev = mrb.register_batch(rr, tt, mrb.DeferredMesh.create_many([VT[k] for k in idx]),
                                 cfg, precision=precision, return_dense=True)
        for a, b in zip(host, dev):
            assert type(a) is type(b)
            if isinstance(a, Exception):
                assert str(a) == str(b)
                continue
            assert np.array_equal(a[0], b[0])
            assert a[1].energy_trace == b[1].energy_trace
            assert a[1].msd_after == b[1].msd_after and a[1].msd_before == b[1].msd_before
            assert all(np.array_equal(x, y) for x, y in zip(a[2], b[2]))


def test_register_batch_deferred_invalid_meshes():
    """Connectivity checks run on the device: a non-manifold mesh and a mesh
    with a lone vertex raise the reference's messages (mesh.py:99-122)."""
    g = golden("gen64")
    h, w = g["re"].shape
    re, te = mrb.ImageGrid(w, h, g["re"]), mrb.ImageGrid(w, h, g["te"])
    V, T = g["V"], g["T_in"].astype(np.int64)
    cfg = mrb.SolverConfig(max_iterations=10)
    # a fourth triangle on the edge of triangle 0
    a, b = int(T[0, 0]), int(T[0, 1])
    V2 = np.vstack([V, [[(V[a, 0] + V[b, 0]) / 2 + 0.37, (V[a, 1] + V[b, 1]) / 2 + 0.21]],
                    [[(V[a, 0] + V[b, 0]) / 2 - 0.29, (V[a, 1] + V[b, 1]) / 2 - 0.33]]])
    T2 = np.vstack([T, [[a, b, len(V)]], [[a, b, len(V) + 1]]])
    with pytest.raises(ValueError) as want:
        mrb.TriMesh(V2, T2)
    out = mrb.register_batch([re, re], [te, te],
                             mrb.DeferredMesh.create_many([(V, T), (V2, T2)]), cfg,
                             precision="f32")
    assert isinstance(out[1], ValueError) and str(out[1]) == str(want.value)
    V3 = np.vstack([V, [[5.0, 5.0]]])
    with pytest.raises(ValueError) as want3:
        mrb.TriMesh(V3, T)
    out = mrb.register_batch([re], [te], mrb.DeferredMesh.create_many([(V3, T)]), cfg,
                             precision="f32")
    assert isinstance(out[0], ValueError) and str(out[0]) == str(want3.value)


def test_register_batch_deferred_coverage_error():
    """A deferred mesh that leaves pixels uncovered: its pair raises
    MeshCoverageError with the reference's message (densefield.py:176-182),
    the other pairs of the batch register normally (the early rasters of the
    device setup carry the coverage check)."""
    g = golden("gen64")
    h, w = g["re"].shape
    re, te = mrb.ImageGrid(w, h, g["re"]), mrb.ImageGrid(w, h, g["te"])
    V, T = g["V"], g["T_in"].astype(np.int64)
    # a mesh of the upper half only
    keep = V[T].max(axis=1)[:, 1] <= (h - 1) / 2
    used = np.unique(T[keep])
    remap = -np.ones(len(V), np.int64)
    remap[used] = np.arange(len(used))
    Vh, Th = V[used], remap[T[keep]]
    cfg = mrb.SolverConfig(max_iterations=10)
    with pytest.raises(mrb.MeshCoverageError) as want:
        mrb.register(re, te, mrb.TriMesh(Vh, Th), cfg, precision="f32")
    out = mrb.register_batch([re, re, re], [te, te, te],
                             mrb.DeferredMesh.create_many([(V, T), (Vh, Th), (V, T)]), cfg,
                             precision="f32")
    assert isinstance(out[1], mrb.MeshCoverageError) and str(out[1]) == str(want.value)
    u0, rep0 = mrb.register(re, te, mrb.TriMesh(V, T), cfg, precision="f32")
    for k in (0, 2):
        assert np.array_equal(out[k][0], u0)
