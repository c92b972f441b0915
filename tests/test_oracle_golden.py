"""Pin the CPU oracle (oracle/meshreg_oracle.py) against golden vectors that
the reference itself produced (tests/golden/make_golden.py)."""
import numpy as np
import pytest

import meshreg_oracle as O
from conftest import golden


def test_oracle_register_bit_exact(golden_case):
    name, g = golden_case
    m = O.Mesh(g["V"], g["T_in"])
    assert np.array_equal(m.T, g["T"])
    tau, lam, iters, passes, tol = g["cfg"]
    u, info = O.register(g["re"], g["te"], m, tau=tau, lam=lam, max_iterations=int(iters),
                         smoothing_passes=int(passes), energy_tolerance=tol)
    assert info["iterations_run"] == int(g["iterations_run"])
    assert np.array_equal(np.array(info["energy_trace"]), g["trace"])
    assert np.array_equal(u, g["u"])
    assert info["msd_before"] == float(g["msd_before"])
    if "ux" in g.files:
        assert np.array_equal(info["ux"], g["ux"])
        assert np.array_equal(info["uy"], g["uy"])
        assert np.array_equal(info["warped"], g["warped"])
        assert info["msd_after"] == float(g["msd_after"])


def test_oracle_connectivity_and_csr_bit_exact(golden_case):
    name, g = golden_case
    m = O.Mesh(g["V"], g["T_in"])
    if "ring_idx" in g.files:
        assert np.array_equal(m.ring_ptr, g["ring_ptr"]) and np.array_equal(m.ring_idx, g["ring_idx"])
        assert np.array_equal(m.inc_ptr, g["inc_ptr"]) and np.array_equal(m.inc_idx, g["inc_idx"])
        assert np.array_equal(m.edges, g["edges"])
        assert np.array_equal(m.valence, g["valence"])
        assert np.array_equal(m.boundary, g["boundary"])
    for key, mine in (("L", m.lap), ("gx", m.gx), ("gy", m.gy), ("avg", m.avg)):
        if key + "_indptr" in g.files:
            for a, b in zip(mine, (g[key + "_indptr"], g[key + "_indices"], g[key + "_data"])):
                assert np.array_equal(a, b), key
    if "areas" in g.files:
        assert np.array_equal(m.areas, g["areas"])
        assert np.array_equal(m.coeffs, g["coeffs"])
        assert np.array_equal(m.vertex_areas, g["vertex_areas"])


@pytest.mark.parametrize("name", ["gen64", "gen64_x255", "accept_c3", "c1"])
def test_oracle_pixel_map_bit_exact(name):
    g = golden(name)
    m = O.Mesh(g["V"], g["T_in"])
    h, w = g["re"].shape
    tri, wts = O.pixel_map(m, w, h)
    assert np.array_equal(tri, g["tri_of"])
    if "pm_weights" in g.files:
        assert np.array_equal(wts, g["pm_weights"])
    # the vectorised map used at C5 size is the same map, bit for bit
    tri2, wts2 = O.pixel_map_vec(m, w, h, chunk=97)
    assert np.array_equal(tri2, tri) and np.array_equal(wts2, wts)


def test_oracle_warp_image_row_blocks():
    # the row-blocked warp equals one whole-image sample call
    g = golden("c1_x255")
    te = g["te"].astype(np.float64)
    h, w = te.shape
    rng = np.random.default_rng(5)
    ux, uy = rng.normal(0, 3, (2, h, w))
    gx, gy = np.meshgrid(np.arange(w, dtype=np.float64), np.arange(h, dtype=np.float64))
    assert np.array_equal(O.warp_image(te, ux, uy), O.sample(te, gx + ux, gy + uy))


@pytest.mark.parametrize("name", ["c1_x255", "c1", "gen64_x255"])
def test_fp32_emulation_meets_north_star_tolerance(name):
    """fp32 arithmetic itself (tests/f32_emulation.py: what the fast path
    computes) stays inside the north_star tolerance of the fp64 reference on
    the large-motion goldens, so the GPU tests can hold the fast path to 1e-4."""
    from f32_emulation import register32
    g = golden(name)
    tau, lam, it, p, tol = g["cfg"]
    u, trace = register32(g["re"].astype(np.float64), g["te"].astype(np.float64),
                          O.Mesh(g["V"], g["T_in"]), float(tau), float(lam), int(it), int(p))
    err = np.abs(u - g["u"]).max() / np.abs(g["u"]).max()
    print(f"{name}: fp32 emulation u relinf {err:.2e}")
    assert err < 1e-5
    n = len(trace)
    assert np.abs(np.array(trace) - g["trace"][:n]).max() / np.abs(g["trace"]).max() < 1e-5


@pytest.mark.parametrize("name", ["gen64", "gen64_x255"])
def test_oracle_single_operations(name):
    g = golden(name)
    m = O.Mesh(g["V"], g["T_in"])
    u, grad = g["unit_u"], g["unit_grad"]
    assert np.array_equal(O.warp_sample(g["te"], m.V, u), g["unit_warp_sample"])
    assert O.energy(g["re"], g["te"], m, u) == float(g["unit_energy"])
    assert np.array_equal(O.energy_gradient(g["re"], g["te"], m, u), g["unit_energy_gradient"])
    f = O.sample(g["te"], m.V[:, 0], m.V[:, 1])
    assert np.array_equal(O.vertex_gradient_all(m, f), g["unit_vgrad"])
    assert np.array_equal(O.smooth_displacement(m, u, 0.8, 2), g["unit_smooth2"])
    h, w = g["re"].shape
    assert np.array_equal(O.step(m, u, grad, 0.005, 0.8, 1, m.V, (w, h)), g["unit_step"])
    assert O.msd(g["te"], g["re"]) == float(g["unit_msd"])


def test_oracle_divergence_message():
    g = golden("diverge64")
    m = O.Mesh(g["V"], g["T_in"])
    with pytest.raises(O.OracleDivergence) as exc:
        O.register(g["re"], g["te"], m, tau=0.1)
    assert str(exc.value) == str(g["error"])


# ---- pixel-grid engine (baseline.py) ----------------
PIXEL_CASES = ["pixel64", "pixel96_p1", "pixel48_lam0"]


@pytest.mark.parametrize("name", PIXEL_CASES)
def test_oracle_register_pixelwise_bit_exact(name):
    g = golden(name)
    tau, lam, iters, passes = g["cfg"]
    ux, uy, info = O.register_pixelwise(g["re"], g["te"], tau=tau, lam=lam,
                                        iterations=int(iters), smoothing_passes=int(passes))
    assert info["iterations_run"] == int(g["iterations_run"])
    assert np.array_equal(np.array(info["energy_trace"]), g["trace"])
    assert np.array_equal(ux, g["ux"]) and np.array_equal(uy, g["uy"])
    assert np.array_equal(info["warped"], g["warped"])
    assert info["msd_before"] == float(g["msd_before"])
    assert info["msd_after"] == float(g["msd_after"])


def test_oracle_pixel_units_bit_exact():
    g = golden("pixel_units")
    gx, gy = O.sample_gradient(g["img"], g["pts"][:, 0], g["pts"][:, 1])
    assert np.array_equal(gx, g["gx"]) and np.array_equal(gy, g["gy"])
    assert np.array_equal(O.grid_umbrella_smooth(g["plane"], 0.6), g["smooth"])


def test_oracle_pixel_divergence_message():
    g = golden("pixel_diverge48")
    with pytest.raises(O.OracleDivergence) as e:
        O.register_pixelwise(g["re"], g["te"], tau=0.2)
    assert str(e.value) == str(g["error"])


def test_oracle_pixel_validation():
    z = np.zeros((8, 8))
    for kw, msg in ((dict(tau=0.0), "tau must be positive"), (dict(lam=1.0), "lambda must be in [0, 1)"),
                    (dict(iterations=0), "iterations must be >= 1")):
        with pytest.raises(ValueError, match=msg.replace("[", r"\[").replace(")", r"\)")):
            O.register_pixelwise(z, z, **kw)
    with pytest.raises(ValueError, match="image sizes differ"):
        O.register_pixelwise(z, np.zeros((8, 9)))
