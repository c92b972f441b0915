"""GPU parity: the sm_100a path (through the C ABI) against the reference's
golden vectors and the CPU oracle.

Tolerances (BASELINE.json north_star): displacement field and warped image
within 1e-4 relative (fp32), MSD within 1e-5 relative, connectivity / CSR /
pixel map bit-exact.  The fp64 path is held to 1e-9.
"""
import numpy as np
import pytest

import meshreg_oracle as O
import paper_1411_2141_b200 as mrb
from conftest import GOLDEN_CASES, golden

pytestmark = pytest.mark.gpu

TOL = {"f32": dict(u=1e-4, dense=1e-4, msd=1e-5, trace=1e-5),
       "f64": dict(u=1e-9, dense=1e-9, msd=1e-10, trace=1e-10)}


def relinf(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def images(g):
    h, w = g["re"].shape
    return mrb.ImageGrid(w, h, g["re"]), mrb.ImageGrid(w, h, g["te"])


def cfg_of(g):
    tau, lam, iters, passes, tol = g["cfg"]
    return mrb.SolverConfig(tau=float(tau), lam=float(lam), max_iterations=int(iters),
                            smoothing_passes=int(passes), energy_tolerance=float(tol))


def check_register(g, precision, name):
    re, te = images(g)
    mesh = mrb.TriMesh(g["V"], g["T_in"])
    cfg = cfg_of(g)
    u, rep, (ux, uy, warped) = mrb.register(re, te, mesh, cfg, precision=precision,
                                            return_dense=True)
    tol = TOL[precision]  # the same tolerances for every case, large motion included
    err = dict(trace=relinf(rep.energy_trace, g["trace"]))
    if np.abs(g["u"]).max() > 0:
        err["u"] = relinf(u, g["u"])
    if "ux" in g.files:
        if np.abs(g["ux"]).max() > 0:
            err["ux"], err["uy"] = relinf(ux, g["ux"]), relinf(uy, g["uy"])
        err["warped"] = relinf(warped, g["warped"])
        ref = float(g["msd_after"])
        err["msd_after"] = abs(rep.msd_after - ref) / max(ref, 1e-300)
    print(f"\n{name} {precision}: " + " ".join(f"{k} {v:.2e}" for k, v in err.items()))
    assert rep.iterations_run == int(g["iterations_run"])
    assert err["trace"] <= tol["trace"], (name, err)
    if "u" in err:
        assert err["u"] <= tol["u"], (name, err)
    else:
        assert np.abs(u).max() < 1e-12
    assert abs(rep.msd_before - float(g["msd_before"])) <= tol["msd"] * max(float(g["msd_before"]), 1e-300)
    for k in ("ux", "uy", "warped"):
        if k in err:
            assert err[k] <= tol["dense"], (name, err)
    if "msd_after" in err:
        assert err["msd_after"] <= tol["msd"], (name, err)


@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_register_matches_reference_golden(name, precision):
    check_register(golden(name), precision, name)


@pytest.mark.parametrize("name", ["gen64", "gen64_x255", "accept_c3", "c1"])
def test_pixel_map_bit_exact(name):
    g = golden(name)
    mesh = mrb.TriMesh(g["V"], g["T_in"])
    h, w = g["re"].shape
    tri_of, wts = mrb.pixel_map(mesh, w, h)
    assert np.array_equal(tri_of, g["tri_of"])
    if "pm_weights" in g.files:
        assert np.array_equal(wts, g["pm_weights"])


@pytest.mark.parametrize("name", ["gen64", "gen64_x255"])
def test_single_operations(name):
    g = golden(name)
    re, te = images(g)
    mesh = mrb.TriMesh(g["V"], g["T_in"])
    u, grad = g["unit_u"], g["unit_grad"]
    assert relinf(mrb.warp_sample(te, mesh.vertices, u), g["unit_warp_sample"]) < 1e-14
    assert abs(mrb.energy(re, te, mesh, u) / float(g["unit_energy"]) - 1) < 1e-12
    assert relinf(mrb.energy_gradient(re, te, mesh, u), g["unit_energy_gradient"]) < 1e-10
    f = te.sample(mesh.vertices[:, 0], mesh.vertices[:, 1])
    assert relinf(mrb.vertex_gradient_all(mesh, mesh.geometry, f), g["unit_vgrad"]) < 1e-10
    L = mrb.build_laplacian(mesh)
    assert np.array_equal(mrb.smooth_displacement(L, u, 0.8, 2), g["unit_smooth2"])
    h, w = g["re"].shape
    out = mrb.step(u, grad, mrb.SolverConfig(), L, mesh.vertices, (w, h))
    assert np.array_equal(out, g["unit_step"])
    assert abs(mrb.msd(te, re) / float(g["unit_msd"]) - 1) < 1e-13


def test_divergence_guard_message():
    g = golden("diverge64")
    re, te = images(g)
    mesh = mrb.TriMesh(g["V"], g["T_in"])
    with pytest.raises(mrb.DivergenceError) as exc:
        mrb.register(re, te, mesh, mrb.SolverConfig(tau=0.1), precision="f64")
    # same text; the four energies agree to fp64 round-off amplified by a
    # divergent (chaotic) run, so they are compared numerically
    import re as _re
    num = r"\[([^\]]*)\]"
    got, want = str(exc.value), str(g["error"])
    assert _re.sub(num, "[]", got) == _re.sub(num, "[]", want)
    a = np.array([float(x) for x in _re.search(num, got).group(1).split(",")])
    b = np.array([float(x) for x in _re.search(num, want).group(1).split(",")])
    assert np.abs(a / b - 1).max() < 1e-6
    # fp32 follows a different trajectory once the run is chaotic (tau=0.1);
    # the guard itself is exercised on the fp32 path by the rises KAT below.


def test_msd_after_equals_dense_warp_msd():
    # test_registration.py:334-346
    g = golden("plateau64")
    re, te = images(g)
    mesh = mrb.TriMesh(g["V"], g["T_in"])
    u, rep = mrb.register(re, te, mesh, mrb.SolverConfig(max_iterations=30), precision="f64")
    dense = mrb.densify(mesh, u, 64, 64)
    assert rep.msd_after == mrb.msd(mrb.warp_image(te, dense), re)
    assert len(rep.energy_trace) == rep.iterations_run


def test_identical_images_exit_early():
    g = golden("identical48")
    re, te = images(g)
    mesh = mrb.TriMesh(g["V"], g["T_in"])
    for precision in ("f32", "f64"):
        u, rep = mrb.register(re, te, mesh, precision=precision)
        assert np.abs(u).max() == 0.0
        assert rep.msd_before == 0.0 and rep.msd_after == 0.0
        assert rep.iterations_run == 6 and all(e == 0.0 for e in rep.energy_trace)


def test_size_mismatch():
    a = mrb.ImageGrid(16, 16, np.zeros(256))
    b = mrb.ImageGrid(16, 17, np.zeros(272))
    mesh = mrb.TriMesh([(0, 0), (15, 0), (0, 15), (15, 15)], [(0, 1, 2), (1, 3, 2)])
    with pytest.raises(ValueError, match="sizes differ"):
        mrb.register(b, a, mesh)


def test_warp_zero_field_identity_and_ramp():
    rng = np.random.default_rng(3)
    img = mrb.ImageGrid(20, 15, rng.uniform(50, 200, 300))
    out = mrb.warp_image(img, mrb.DenseField(np.zeros((15, 20)), np.zeros((15, 20))))
    assert np.array_equal(out.data, img.data)
    gx, gy = np.meshgrid(np.arange(16.0), np.arange(12.0))
    ramp = mrb.ImageGrid(16, 12, gx)
    out = mrb.warp_image(ramp, mrb.DenseField(np.ones((12, 16)), np.zeros((12, 16))))
    assert np.abs(out.data - np.minimum(gx + 1.0, 15.0)).max() < 1e-9


def test_sampling_known_answers():
    # exact at pixel centres, constant and ramp reproduction incl. borders
    rng = np.random.default_rng(0)
    data = rng.uniform(0, 255, (9, 11))
    img = mrb.ImageGrid(11, 9, data)
    ys, xs = np.mgrid[0:9, 0:11]
    assert np.array_equal(img.sample(xs.astype(float), ys.astype(float)), data)
    gx, gy = np.meshgrid(np.arange(11.0), np.arange(9.0))
    ramp = mrb.ImageGrid(11, 9, 3.0 + 2.0 * gx - 0.5 * gy)
    x = rng.uniform(-1, 11, 500)
    y = rng.uniform(-1, 9, 500)
    want = 3.0 + 2.0 * np.clip(x, 0, 10) - 0.5 * np.clip(y, 0, 8)
    assert np.abs(ramp.sample(x, y) - want).max() < 1e-10
    const = mrb.ImageGrid(5, 4, np.full(20, 7.25))
    assert np.abs(const.sample(x, y) - 7.25).max() < 1e-12
    assert isinstance(img.sample(1.5, 2.5), float)


def test_energy_known_answers():
    te = mrb.ImageGrid(8, 8, np.full(64, 3.0))
    re = mrb.ImageGrid(8, 8, np.full(64, 1.0))
    mesh = mrb.TriMesh([(0, 0), (7, 0), (0, 7), (7, 7), (3.5, 3.5)],
                       [(0, 1, 4), (1, 3, 4), (3, 2, 4), (2, 0, 4)])
    assert mrb.energy(re, te, mesh, np.zeros((5, 2))) == pytest.approx(2.0 * 5)
    g = mrb.energy_gradient(re, te, mesh, np.zeros((5, 2)))
    assert np.abs(g).max() < 1e-12


def test_step_known_answers():
    angles = np.linspace(0.0, 2.0 * np.pi, 7)[:-1]
    V = np.vstack([[0.0, 0.0], np.column_stack([np.cos(angles), np.sin(angles)])])
    hexm = mrb.TriMesh(V, [(0, 1 + i, 1 + (i + 1) % 6) for i in range(6)])
    L = mrb.build_laplacian(hexm)
    grad = np.zeros((7, 2))
    grad[0] = (100.0, 0.0)
    out = mrb.step(np.zeros((7, 2)), grad, mrb.SolverConfig(tau=0.005, smoothing_passes=0), L)
    assert out[0, 0] == pytest.approx(-0.5, abs=1e-15)
    assert np.abs(out[1:]).max() == 0.0
    # hexagon centre smoothing (test_mesh_ops.py:232-238)
    u = np.zeros((7, 2))
    u[1:, 0] = 1.0
    sm = mrb.smooth_displacement(L, u, 0.8, 1)
    assert sm[0, 0] == pytest.approx(0.8)
    # any column count, like the reference's L @ u: (n,), (n, 1), (n, 3) give
    # the columns of the (n, 2) result
    cols3 = np.column_stack([u[:, 0], 2.0 * u[:, 0], u[:, 1] + 0.25])
    sm3 = mrb.smooth_displacement(L, cols3, 0.8, 2)
    assert sm3.shape == (7, 3)
    for k in range(3):
        one = mrb.smooth_displacement(L, cols3[:, k], 0.8, 2)
        assert one.shape == (7,) and np.array_equal(one, sm3[:, k])
        assert np.array_equal(mrb.smooth_displacement(L, cols3[:, k:k + 1], 0.8, 2)[:, 0], one)
    assert np.array_equal(sm3[:, 0], mrb.smooth_displacement(L, u, 0.8, 2)[:, 0])
    bad = np.zeros((7, 2))
    bad[2, 1] = np.nan
    with pytest.raises(mrb.DivergenceError):
        mrb.step(np.zeros((7, 2)), bad, mrb.SolverConfig(), L)
    moved = mrb.TriMesh(V + 5.0, hexm.triangles)
    out = mrb.step(np.zeros((7, 2)), np.full((7, 2), -1e6), mrb.SolverConfig(smoothing_passes=0),
                   mrb.build_laplacian(moved), vertices=moved.vertices, domain=(11, 11))
    assert (moved.vertices + out).max() <= 10.0 + 1e-9


def test_coverage_error():
    tri = mrb.TriMesh([(0, 0), (4, 0), (0, 4)], [(0, 1, 2)])
    with pytest.raises(mrb.MeshCoverageError):
        mrb.densify(tri, np.zeros((3, 2)), 5, 5)


@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_batch_equals_single(precision):
    names = ["gen64", "gen64_x255", "plateau64"]
    gs = [golden(n) for n in names]
    # equal sizes only: gen64 / gen64_x255 / plateau64 are all 64x64
    res, tes, meshes = [], [], []
    for g in gs:
        r, t = images(g)
        res.append(r)
        tes.append(t)
        meshes.append(mrb.TriMesh(g["V"], g["T_in"]))
    cfg = mrb.SolverConfig(tau=0.001, max_iterations=25, energy_tolerance=0.0)
    batch = mrb.register_batch(res, tes, meshes, cfg, precision=precision)
    for (u, rep), r, t, m in zip(batch, res, tes, meshes):
        u1, rep1 = mrb.register(r, t, m, cfg, precision=precision)
        assert np.array_equal(u, u1)
        assert rep.energy_trace == rep1.energy_trace
        assert rep.msd_after == rep1.msd_after


def test_oracle_agrees_on_fresh_seeds():
    # seeded generator pairs the golden files do not contain, fp32 path vs oracle
    from paper_1411_2141_b200.synthetic import PairSpec, make_pair
    g = golden("gen64")
    for seed in (11, 12):
        spec = PairSpec("t", 64, 8, 0, 2.0, 150, 30)
        re32, te32 = make_pair(spec, seed, scale=25.0)
        om = O.Mesh(g["V"], g["T_in"])
        u_ref, info = O.register(re32, te32, om, tau=0.001, max_iterations=30,
                                 energy_tolerance=0.0)
        re = mrb.ImageGrid(64, 64, re32.astype(np.float64))
        te = mrb.ImageGrid(64, 64, te32.astype(np.float64))
        mesh = mrb.TriMesh(g["V"], g["T_in"])
        u, rep, (ux, uy, wp) = mrb.register(re, te, mesh, mrb.SolverConfig(
            tau=0.001, max_iterations=30, energy_tolerance=0.0), precision="f32",
            return_dense=True)
        assert relinf(u, u_ref) < 1e-4
        assert relinf(wp, info["warped"]) < 1e-4
        assert abs(rep.msd_after / info["msd_after"] - 1) < 1e-5


def test_rises_guard_fp32_and_message_format():
    # gen64_x255 with the default tau diverges steadily in the reference
    # (energy +4% per step), on both precisions (solver.py:178-184)
    g = golden("gen64_x255")
    re, te = images(g)
    mesh = mrb.TriMesh(g["V"], g["T_in"])
    for precision in ("f32", "f64"):
        with pytest.raises(mrb.DivergenceError) as exc:
            mrb.register(re, te, mesh, mrb.SolverConfig(tau=0.005), precision=precision)
        msg = str(exc.value)
        assert msg.startswith("energy increased for 10 consecutive iterations (last values [") \
            or msg in ("energy became non-finite; reduce tau",
                       "non-finite gradient; reduce the step size tau"), msg


@pytest.mark.parametrize("path", ["cluster", "push", "pull", "grid", "generic"])
@pytest.mark.parametrize("name", ["gen64", "gen64_x255", "gen64_p0", "gen64_p2", "c1", "accept_c3"])
def test_fp32_paths_agree_with_reference(name, path, monkeypatch):
    """The persistent cluster kernel (default exchange, and push / pull halo
    exchange forced), the whole-GPU grid kernel (forced here on small meshes;
    chosen by size for C3/C5) and the generic three-kernel loop all meet the
    fp32 tolerances."""
    monkeypatch.delenv("MESHREG_B200_EXCHANGE", raising=False)
    if path in ("generic", "grid"):
        monkeypatch.setenv("MESHREG_B200_PATH", path)
    else:
        monkeypatch.delenv("MESHREG_B200_PATH", raising=False)
        if path in ("push", "pull"):  # cluster kernel with a forced halo exchange
            monkeypatch.setenv("MESHREG_B200_EXCHANGE", path)
    check_register(golden(name), "f32", name)


def test_path_selection(monkeypatch):
    """mrb_batch_path: cluster size > 0, minus the grid CTA count < 0, 0 generic."""
    import ctypes as C
    from paper_1411_2141_b200 import _lib
    g = golden("gen64")
    lib = _lib.load()
    ctx = _lib.context()
    mesh = mrb.TriMesh(g["V"], g["T_in"])
    cfg = _lib.mrb_config(0.005, 0.8, 0.0, 10, 1, _lib.PREC_F32, 0)
    seen = {}
    for path in ("", "grid", "generic"):
        if path:
            monkeypatch.setenv("MESHREG_B200_PATH", path)
        else:
            monkeypatch.delenv("MESHREG_B200_PATH", raising=False)
        arr = (C.c_void_p * 1)(mesh._h)
        b = C.c_void_p()
        assert lib.mrb_batch_create(ctx, 1, arr, 64, 64, _lib.F32, C.byref(cfg), C.byref(b)) == 0
        seen[path] = lib.mrb_batch_path(b)
        lib.mrb_batch_destroy(b)
    assert seen[""] > 0 and seen["grid"] < 0 and seen["generic"] == 0


@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_pipelined_batch_chunks_and_per_pair_errors(precision):
    """mrb_register_many with one pair per chunk (both pipeline streams,
    several chunks in flight) equals single registrations; a diverging pair
    yields its DivergenceError without affecting the others."""
    names = ["gen64", "plateau64", "gen64_x255", "gen64", "plateau64"]
    res, tes, meshes = [], [], []
    for n in names:
        g = golden(n)
        r, t = images(g)
        res.append(r)
        tes.append(t)
        meshes.append(mrb.TriMesh(g["V"], g["T_in"]))
    cfg = mrb.SolverConfig(tau=0.005, max_iterations=40, energy_tolerance=0.0)
    out = mrb.register_batch(res, tes, meshes, cfg, precision=precision, return_dense=True,
                             chunk_pairs=1)
    assert isinstance(out[2], mrb.DivergenceError)  # gen64_x255 diverges at tau=0.005
    assert "consecutive iterations" in str(out[2])
    for k in (0, 1, 3, 4):
        u, rep, (ux, uy, warped) = out[k]
        u1, rep1, (ux1, uy1, w1) = mrb.register(res[k], tes[k], meshes[k], cfg,
                                                precision=precision, return_dense=True)
        assert np.array_equal(u, u1)
        assert rep.energy_trace == rep1.energy_trace
        assert rep.msd_after == rep1.msd_after and rep.msd_before == rep1.msd_before
        assert np.array_equal(warped, w1) and np.array_equal(ux, ux1)
    # identical inputs give identical results (determinism across chunks/streams)
    assert np.array_equal(out[0][0], out[3][0]) and np.array_equal(out[1][0], out[4][0])


def test_register_batch_wave_groups_deferred_topologies(monkeypatch):
    """More pairs than one wave of clusters: mrb_register_many launches per
    wave group, uploads each group's topologies just ahead of its launch and
    copies results back per group.  Bit-identical to one launch of the same
    batch, and to the oracle within the fp32 tolerance."""
    names = ["gen64", "gen64_x255", "plateau64"]
    gs = [golden(n) for n in names]
    P = 300  # small meshes: one wave holds ~150 clusters
    res, tes, meshes, which = [], [], [], []
    for i in range(P):
        g = gs[i % 3]
        r, t = images(g)
        res.append(r)
        tes.append(t)
        meshes.append(mrb.TriMesh(g["V"], g["T_in"]))  # distinct mesh objects
        which.append(i % 3)
    cfg = mrb.SolverConfig(tau=0.001, max_iterations=20, energy_tolerance=0.0)
    out = mrb.register_batch(res, tes, meshes, cfg, precision="f32", return_dense=True)
    monkeypatch.setenv("MESHREG_B200_NO_GROUPS", "1")
    meshes2 = [mrb.TriMesh(gs[k]["V"], gs[k]["T_in"]) for k in which]
    ref = mrb.register_batch(res, tes, meshes2, cfg, precision="f32", return_dense=True)
    for i, (o, r) in enumerate(zip(out, ref)):
        assert np.array_equal(o[0], r[0]), i
        assert o[1].energy_trace == r[1].energy_trace
        assert all(np.array_equal(a, b) for a, b in zip(o[2], r[2]))
    for k in range(3):  # and the oracle
        g = gs[k]
        u_ref, info = O.register(g["re"], g["te"], O.Mesh(g["V"], g["T_in"]), tau=0.001, lam=0.8,
                                 max_iterations=20, smoothing_passes=1, energy_tolerance=0.0)
        assert np.abs(out[k][0] - u_ref).max() <= 1e-4 * max(np.abs(u_ref).max(), 1e-30)


def test_register_batch_reports_call_level_failures():
    """A failure that stops mrb_register_many before any pair ran (here: one
    mesh does not cover the image, found while the batch's pixel maps are
    built) never reads as success: the uncovered pair gets the reference's
    MeshCoverageError, the others their results; an invalid configuration
    makes every pair carry the ValueError."""
    g = golden("gen64")
    re, te = images(g)
    good = mrb.TriMesh(g["V"], g["T_in"])
    small = mrb.TriMesh([(0, 0), (40, 0), (0, 40), (40, 40)], [(0, 1, 2), (1, 3, 2)])
    cfg = mrb.SolverConfig(tau=0.001, max_iterations=10, energy_tolerance=0.0)
    for precision in ("f32", "f64"):
        out = mrb.register_batch([re, re], [te, te], [good, small], cfg, precision=precision)
        assert isinstance(out[1], mrb.MeshCoverageError), out[1]
        u1, rep1 = mrb.register(re, te, good, cfg, precision=precision)
        assert np.array_equal(out[0][0], u1) and out[0][1].energy_trace == rep1.energy_trace
    import ctypes as C
    from paper_1411_2141_b200 import _lib
    lib = _lib.load()
    bad = _lib.mrb_config(-1.0, 0.8, 0.0, 10, 1, _lib.PREC_F32, 0)  # tau <= 0
    arr = (C.c_void_p * 2)(good._h, good._h)
    P, n = 2, good.n_vertices
    img = np.ascontiguousarray(np.stack([g["re"], g["re"]]).astype(np.float32))
    u = np.zeros((P * n, 2))
    codes = np.zeros(P, np.int32)  # zeros == OK: the library must overwrite them
    msgs = C.create_string_buffer(P * 256)
    rc = lib.mrb_register_many(_lib.context(), P, arr, 64, 64, _lib.F32, _lib.ptr(img),
                               _lib.ptr(img), C.byref(bad), 0, _lib.F64, _lib.ptr(u), None, None,
                               None, None, None, None, None, _lib.ptr(codes), msgs, 256)
    assert rc == _lib.E_VALUE
    assert list(codes) == [_lib.E_VALUE, _lib.E_VALUE]
    assert b"tau" in msgs.raw[:256]
