"""Full-size BASELINE configurations on the GPU against the CPU oracle run
live (the oracle finishes C2 in ~5 s and C3 in ~20 s), plus size-independent
properties at full size.  Meshes come from the reference-mesher cache
(data/meshes, produced by tools/make_meshes.py); without it the package
mesher builds the same meshes.

Tolerances (BASELINE.json north_star): u / dense field / warped image within
1e-4 relative (fp32), MSD within 1e-5 relative.
"""
import os

import numpy as np
import pytest

import meshreg_oracle as O
import paper_1411_2141_b200 as mrb
from conftest import ROOT
from paper_1411_2141_b200.synthetic import CONFIGS, make_pair

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def load(cfg, seed=0, x255=False):
    path = os.path.join(ROOT, "data", "meshes", f"{cfg}_s{seed}{'_x255' if x255 else ''}.npz")
    committed = os.path.join(ROOT, "tests", "golden", f"refmesh_{cfg}_s{seed}.npz")
    if not x255 and os.path.exists(committed):  # reference-mesher output, committed
        path = committed
    spec = CONFIGS[cfg]
    re, te = make_pair(spec, seed, scale=255.0 if x255 else 1.0)
    if not os.path.exists(path):
        # no reference-mesher cache (fresh checkout): the package mesher makes
        # the same mesh (bit-identical, tests/test_mesher.py)
        m = mrb.generate_mesh(mrb.ImageGrid(spec.size, spec.size, te.astype(np.float64)),
                              mrb.NodeBudget(spec.target_nodes), mrb.MeshGenConfig(seed=0))
        return spec, re, te, m.vertices.copy(), m.triangles.copy()
    m = np.load(path)
    return spec, re, te, m["V"], m["T"].astype(np.int64)


def relinf(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-30))


TOL_U = 1e-4     # u, dense field, warped image: relative to the reference's max
TOL_MSD = 1e-5   # msd_before / msd_after: relative


def check_against_oracle(tag, rep, u, dense, u_ref, info):
    """Assert the north_star tolerances and print the achieved errors."""
    ux, uy, warped = dense
    err = dict(u=relinf(u, u_ref), ux=relinf(ux, info["ux"]), uy=relinf(uy, info["uy"]),
               warped=relinf(warped, info["warped"]),
               trace=relinf(rep.energy_trace, info["energy_trace"]),
               msd_after=abs(rep.msd_after / info["msd_after"] - 1),
               msd_before=abs(rep.msd_before / info["msd_before"] - 1))
    print(f"\n{tag}: " + " ".join(f"{k} {v:.2e}" for k, v in err.items()))
    assert rep.iterations_run == info["iterations_run"]
    assert err["trace"] < 1e-5, err
    for k in ("u", "ux", "uy", "warped"):
        assert err[k] < TOL_U, (k, err)
    assert err["msd_after"] < TOL_MSD and err["msd_before"] < 1e-12, err
    return err


@pytest.mark.parametrize("cfg,x255,path", [("c2", False, ""), ("c2", True, ""), ("c3", False, ""),
                                           ("c2", False, "cluster"), ("c2", True, "cluster"),
                                           ("c1", True, "")])
def test_full_size_matches_oracle(cfg, x255, path, monkeypatch):
    """Default path (a single C2/C3 pair runs on the whole-GPU grid kernel)
    and the cluster kernel forced, against the live oracle, at the configs'
    full iteration counts, at [0,1] and x255 (large motion: up to 84 px at
    C2); the north_star tolerances, no loosening."""
    if path:
        monkeypatch.setenv("MESHREG_B200_PATH", path)
    else:
        monkeypatch.delenv("MESHREG_B200_PATH", raising=False)
    spec, re32, te32, V, T = load(cfg, 0, x255)
    iters = spec.iterations
    u_ref, info = O.register(re32, te32, O.Mesh(V, T), tau=0.005, lam=0.8,
                             max_iterations=iters, smoothing_passes=1, energy_tolerance=0.0)
    S = spec.size
    re = mrb.ImageGrid(S, S, re32.astype(np.float64))
    te = mrb.ImageGrid(S, S, te32.astype(np.float64))
    mesh = mrb.TriMesh(V, T)
    cfg_ = mrb.SolverConfig(max_iterations=iters, energy_tolerance=0.0)
    u, rep, dense = mrb.register(re, te, mesh, cfg_, precision="f32", return_dense=True)
    check_against_oracle(f"{cfg}{'x255' if x255 else ''} {path or 'default'} {iters} it",
                         rep, u, dense, u_ref, info)


@pytest.mark.parametrize("precision,iters,tol_u,tol_w", [("f64", 20, 1e-9, 1e-9),
                                                         ("f32", 5, 1e-4, 1e-4)])
def test_c3_x255_chaotic_prefix(precision, iters, tol_u, tol_w, monkeypatch):
    """C3 x255 (1024^2 with 30 sharp-edged rectangles at [0,255]) is chaotic
    in the reference itself: its energy rises after ~iteration 10 (6.44e5 ->
    1.01e6 at 200) and perturbations grow ~1e4x per 10 iterations.  Even our
    fp64 path, which differs from the reference only in summation order
    (~1e-16), departs by 1.9e-3 at 50 iterations; a plain numpy fp32
    emulation departs by 1.3e-2 at 20 (profiles/r02_c3x255_chaos.log).  So
    the case is checked over the prefix where a result is determined by the
    inputs rather than by rounding: fp64 to 1e-9 over 20 iterations, fp32 to
    the north_star 1e-4 over 5."""
    monkeypatch.delenv("MESHREG_B200_PATH", raising=False)
    spec, re32, te32, V, T = load("c3", 0, True)
    u_ref, info = O.register(re32, te32, O.Mesh(V, T), tau=0.005, lam=0.8, max_iterations=iters,
                             smoothing_passes=1, energy_tolerance=0.0)
    S = spec.size
    re = mrb.ImageGrid(S, S, re32.astype(np.float64))
    te = mrb.ImageGrid(S, S, te32.astype(np.float64))
    u, rep, (ux, uy, warped) = mrb.register(re, te, mrb.TriMesh(V, T), mrb.SolverConfig(
        max_iterations=iters, energy_tolerance=0.0), precision=precision, return_dense=True)
    eu, ew = relinf(u, u_ref), relinf(warped, info["warped"])
    print(f"\nc3x255 {precision} {iters} it: u {eu:.2e} warped {ew:.2e}")
    assert rep.iterations_run == iters
    assert eu < tol_u and ew < tol_w
    assert relinf(ux, info["ux"]) < tol_u and relinf(uy, info["uy"]) < tol_u
    assert abs(rep.msd_after / info["msd_after"] - 1) < (1e-10 if precision == "f64" else 1e-5)


@pytest.mark.parametrize("x255", [False, True])
def test_fp64_cluster_loop_matches_oracle(x255, monkeypatch):
    """precision="f64" (the reference's width, the API default): a C2 pair
    on the persistent fp64 cluster kernel (k_cluster64, 16 CTAs x 768 nodes)
    against the live oracle at 1e-9, and the same run through the generic
    three-kernel loop (MESHREG_B200_PATH=generic) agrees with it."""
    monkeypatch.delenv("MESHREG_B200_PATH", raising=False)
    spec, re32, te32, V, T = load("c2", 0, x255)
    iters = 200 if not x255 else 40
    u_ref, info = O.register(re32, te32, O.Mesh(V, T), tau=0.005, lam=0.8, max_iterations=iters,
                             smoothing_passes=1, energy_tolerance=0.0)
    S = spec.size
    re = mrb.ImageGrid(S, S, re32.astype(np.float64))
    te = mrb.ImageGrid(S, S, te32.astype(np.float64))
    cfg = mrb.SolverConfig(max_iterations=iters, energy_tolerance=0.0)
    u, rep, (ux, uy, warped) = mrb.register(re, te, mrb.TriMesh(V, T), cfg, precision="f64",
                                            return_dense=True)
    eu, ew = relinf(u, u_ref), relinf(warped, info["warped"])
    print(f"\nc2{'x255' if x255 else ''} f64 cluster {iters} it: u {eu:.2e} warped {ew:.2e}")
    assert rep.iterations_run == iters
    assert eu < 1e-9 and ew < 1e-9
    assert relinf(ux, info["ux"]) < 1e-9 and relinf(uy, info["uy"]) < 1e-9
    assert relinf(rep.energy_trace, info["energy_trace"]) < 1e-10
    assert abs(rep.msd_after / info["msd_after"] - 1) < 1e-10
    # the pull exchange (cluster barriers) gives bit-identical fields and
    # energies to the default push exchange; the generic loop agrees to 1e-9
    monkeypatch.setenv("MESHREG_B200_EXCHANGE", "pull")
    u3, rep3 = mrb.register(re, te, mrb.TriMesh(V, T), cfg, precision="f64")
    assert np.array_equal(u3, u) and rep3.energy_trace == rep.energy_trace
    monkeypatch.delenv("MESHREG_B200_EXCHANGE")
    monkeypatch.setenv("MESHREG_B200_PATH", "generic")
    u2, rep2 = mrb.register(re, te, mrb.TriMesh(V, T), cfg, precision="f64")
    assert relinf(u2, u) < 1e-9


def test_c5_matches_oracle(monkeypatch):
    """BASELINE config 5 as specified: the 4096^2 pair (300 blobs + 100
    rectangles, 24 px peak warp), its ~500k-node content-adaptive mesh from the
    package mesher (bit-identical to the reference mesher's algorithm), all
    300 iterations with energy_tolerance 0, on the default whole-GPU grid
    kernel, against the live oracle (vectorised pixel map, same map)."""
    monkeypatch.delenv("MESHREG_B200_PATH", raising=False)
    spec, re32, te32, V, T = load("c5", 0)
    iters = spec.iterations
    om = O.Mesh(V, T)
    assert om.n >= 490000
    u_ref, info = O.register(re32, te32, om, tau=0.005, lam=0.8, max_iterations=iters,
                             smoothing_passes=1, energy_tolerance=0.0, vec_pixel_map=True)
    S = spec.size
    re = mrb.ImageGrid(S, S, re32.astype(np.float64))
    te = mrb.ImageGrid(S, S, te32.astype(np.float64))
    u, rep, dense = mrb.register(re, te, mrb.TriMesh(V, T),
                                 mrb.SolverConfig(max_iterations=iters, energy_tolerance=0.0),
                                 precision="f32", return_dense=True)
    check_against_oracle(f"c5 {iters} it", rep, u, dense, u_ref, info)


def test_full_size_properties():
    spec, re32, te32, V, T = load("c2", 0)
    S = spec.size
    re = mrb.ImageGrid(S, S, re32.astype(np.float64))
    te = mrb.ImageGrid(S, S, te32.astype(np.float64))
    mesh = mrb.TriMesh(V, T)
    cfg = mrb.SolverConfig(max_iterations=200, energy_tolerance=0.0)
    # determinism: fixed-order reductions, no float atomics in value paths
    a = mrb.register(re, te, mesh, cfg, precision="f32", return_dense=True)
    b = mrb.register(re, te, mesh, cfg, precision="f32", return_dense=True)
    assert np.array_equal(a[0], b[0]) and a[1].energy_trace == b[1].energy_trace
    assert all(np.array_equal(x, y) for x, y in zip(a[2], b[2]))
    # identical images: zero residual, zero motion, tolerance exit at 6
    u, rep = mrb.register(te, te, mesh, mrb.SolverConfig(max_iterations=200), precision="f32")
    assert np.abs(u).max() == 0.0 and rep.iterations_run == 6
    assert rep.msd_before == 0.0 and rep.msd_after == 0.0
    # batch of full-size pairs == single registrations (fast path, 2 nodes/thread)
    spec1, re1, te1, V1, T1 = load("c2", 1)
    mesh1 = mrb.TriMesh(V1, T1)
    imgs = [(re, te, mesh), (mrb.ImageGrid(S, S, re1.astype(np.float64)),
                             mrb.ImageGrid(S, S, te1.astype(np.float64)), mesh1)] * 2
    out = mrb.register_batch([x[0] for x in imgs], [x[1] for x in imgs], [x[2] for x in imgs],
                             cfg, precision="f32")
    assert np.array_equal(out[0][0], out[2][0]) and np.array_equal(out[1][0], out[3][0])
    assert relinf(out[0][0], a[0]) < 1e-5  # different cluster shape, same tolerance class


def test_c4_batch_pairs_match_oracle():
    """BASELINE config 4 as the bench runs it: all 64 pairs (seeds 0..63) in
    one register_batch call (throughput shape + latency-shape tail wave);
    8 pairs spread over the batch, including the tail, against the oracle."""
    pairs = [load("c2", s) for s in range(64)]
    S = pairs[0][0].size
    cfg = mrb.SolverConfig(max_iterations=200, energy_tolerance=0.0)
    res = [mrb.ImageGrid(S, S, p[1].astype(np.float64)) for p in pairs]
    tes = [mrb.ImageGrid(S, S, p[2].astype(np.float64)) for p in pairs]
    meshes = [mrb.TriMesh(p[3], p[4]) for p in pairs]
    out = mrb.register_batch(res, tes, meshes, cfg, precision="f32", return_dense=True)
    for k in (0, 9, 18, 27, 36, 45, 60, 63):
        p = pairs[k]
        u_ref, info = O.register(p[1], p[2], O.Mesh(p[3], p[4]), tau=0.005, lam=0.8,
                                 max_iterations=200, smoothing_passes=1, energy_tolerance=0.0)
        u, rep, dense = out[k]
        check_against_oracle(f"c4 pair {k}", rep, u, dense, u_ref, info)


def _c5_scale_inputs():
    """4096x4096 smooth pair with a sub-pixel-to-few-pixel motion and a
    structured ~500k-node mesh (the C5 node count; the reference mesher needs
    ~10 h at that size)."""
    from bench import fallback_mesh
    S = 4096
    y, x = np.mgrid[0:S, 0:S].astype(np.float64)
    base = lambda xx, yy: (0.5 + 0.25 * np.sin(xx / 53.0) * np.cos(yy / 71.0)
                           + 0.2 * np.exp(-((xx - 1500.0) ** 2 + (yy - 2600.0) ** 2) / 2e5))
    re = base(x, y).astype(np.float32)
    te = base(x - 1.7 + 0.5 * np.sin(y / 400.0), y + 1.1).astype(np.float32)
    V, T = fallback_mesh(S, 500000)
    return S, re, te, V, T


def test_c5_scale_grid_kernel_matches_generic_path(monkeypatch):
    """At C5 scale (500k nodes, 8 nodes per thread on the whole-GPU grid) the
    persistent grid kernel and the generic three-kernel loop agree to the fp32
    tolerance class; the run is deterministic."""
    S, re32, te32, V, T = _c5_scale_inputs()
    re = mrb.ImageGrid(S, S, re32.astype(np.float64))
    te = mrb.ImageGrid(S, S, te32.astype(np.float64))
    mesh = mrb.TriMesh(V, T)
    assert mesh.n_vertices >= 490000
    cfg = mrb.SolverConfig(max_iterations=20, energy_tolerance=0.0)
    monkeypatch.delenv("MESHREG_B200_PATH", raising=False)
    a = mrb.register(re, te, mesh, cfg, precision="f32", return_dense=True)
    b = mrb.register(re, te, mesh, cfg, precision="f32", return_dense=True)
    monkeypatch.setenv("MESHREG_B200_PATH", "generic")
    g = mrb.register(re, te, mesh, cfg, precision="f32", return_dense=True)
    assert np.array_equal(a[0], b[0]) and a[1].energy_trace == b[1].energy_trace
    assert a[1].iterations_run == g[1].iterations_run == 20
    assert relinf(a[1].energy_trace, g[1].energy_trace) < 1e-5
    assert relinf(a[0], g[0]) < 1e-4
    assert relinf(a[2][2], g[2][2]) < 1e-4  # warped image
    assert abs(a[1].msd_after / g[1].msd_after - 1) < 1e-5
    assert a[1].msd_after < a[1].msd_before


@pytest.mark.parametrize("path,exchange", [("grid", ""), ("cluster", "push"), ("cluster", "pull")])
def test_repeatability_under_timing_variation(path, exchange, monkeypatch):
    """The asynchronous exchanges (epoch-tagged grid words, st.async push,
    DSMEM pull) must give bit-identical results run after run and across
    batch sizes (different timing, co-running clusters)."""
    monkeypatch.setenv("MESHREG_B200_PATH", path)
    if exchange:
        monkeypatch.setenv("MESHREG_B200_EXCHANGE", exchange)
    spec, re32, te32, V, T = load("c2", 0, True)  # x255: real motion, cell crossings
    S = spec.size
    re = mrb.ImageGrid(S, S, re32.astype(np.float64))
    te = mrb.ImageGrid(S, S, te32.astype(np.float64))
    mesh = mrb.TriMesh(V, T)
    cfg = mrb.SolverConfig(tau=0.001, max_iterations=60, energy_tolerance=0.0)
    first = mrb.register(re, te, mesh, cfg, precision="f32", return_dense=True)
    for _ in range(6):
        again = mrb.register(re, te, mesh, cfg, precision="f32", return_dense=True)
        assert np.array_equal(again[0], first[0])
        assert again[1].energy_trace == first[1].energy_trace
        assert np.array_equal(again[2][2], first[2][2])
    if path == "cluster":  # the same pair inside a batch of 5 co-running clusters
        out = mrb.register_batch([re] * 5, [te] * 5, [mrb.TriMesh(V, T) for _ in range(5)], cfg,
                                 precision="f32")
        for u, rep in out:
            assert np.array_equal(u, out[0][0]) and rep.energy_trace == out[0][1].energy_trace


def test_c4_tail_wave_in_latency_shape(monkeypatch):
    """64 C4 pairs: the last partial wave runs in the latency shape (a second
    launch).  Per-node arithmetic does not depend on the cluster shape, so the
    fields are bit-identical to the single-shape run; energies agree to the
    rounding of the (shape-dependent) fixed-order reduction."""
    pairs = [load("c2", s) for s in range(64)]
    S = pairs[0][0].size
    res = [mrb.ImageGrid(S, S, p[1].astype(np.float64)) for p in pairs]
    tes = [mrb.ImageGrid(S, S, p[2].astype(np.float64)) for p in pairs]
    cfg = mrb.SolverConfig(max_iterations=50, energy_tolerance=0.0)
    monkeypatch.setenv("MESHREG_B200_NO_GROUPS", "1")
    tail = mrb.register_batch(res, tes, [mrb.TriMesh(p[3], p[4]) for p in pairs], cfg,
                              precision="f32")
    monkeypatch.setenv("MESHREG_B200_NO_TAIL", "1")
    plain = mrb.register_batch(res, tes, [mrb.TriMesh(p[3], p[4]) for p in pairs], cfg,
                               precision="f32")
    for (u1, r1), (u2, r2) in zip(tail, plain):
        assert np.array_equal(u1, u2)
        assert relinf(r1.energy_trace, r2.energy_trace) < 1e-12
