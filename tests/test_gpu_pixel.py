"""GPU parity of the pixel-grid engine (reference baseline.py; SURVEY.md §8(f)
row 1) against the reference's golden vectors and the CPU oracle.

Tolerances (BASELINE.json north_star): fp64 state within 1e-10 relative of
the reference (the only differences are the fixed-order fp64 energy sum and
fused multiply-adds inside the 16-tap dot products); fp32 state within 1e-4
relative for fields and warped image, 1e-5 for energies / MSD.  The smoothing
pass alone is bit-exact (exact-rounding fp64 ops in numpy's order).
"""
import numpy as np
import pytest

import meshreg_oracle as O
import paper_1411_2141_b200 as mrb
from conftest import golden
from paper_1411_2141_b200 import _lib
from paper_1411_2141_b200.baseline import PixelBatch

pytestmark = pytest.mark.gpu


def relinf(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def grid(a):
    a = np.asarray(a, np.float64)
    return mrb.ImageGrid(a.shape[1], a.shape[0], a)


def run_golden(name, precision):
    g = golden(name)
    tau, lam, iters, passes = g["cfg"]
    field, rep = mrb.register_pixelwise(grid(g["re"]), grid(g["te"]), tau=tau, lam=lam,
                                        iterations=int(iters), smoothing_passes=int(passes),
                                        precision=precision)
    return g, field, rep


@pytest.mark.parametrize("name", ["pixel64", "pixel96_p1", "pixel48_lam0"])
def test_pixelwise_golden_f64(name):
    g, field, rep = run_golden(name, "f64")
    assert rep.iterations_run == int(g["iterations_run"])
    assert relinf(rep.energy_trace, g["trace"]) < 1e-12
    assert relinf(field.ux, g["ux"]) < 1e-10 and relinf(field.uy, g["uy"]) < 1e-10
    assert rep.msd_before == pytest.approx(float(g["msd_before"]), rel=1e-14)
    assert rep.msd_after == pytest.approx(float(g["msd_after"]), rel=1e-10)
    assert isinstance(field, mrb.PixelField)
    assert rep.config["max_iterations"] == int(g["cfg"][2])
    assert rep.config["smoothing_passes"] == int(g["cfg"][3])


@pytest.mark.parametrize("name", ["pixel64", "pixel96_p1", "pixel48_lam0"])
def test_pixelwise_golden_f32(name):
    g, field, rep = run_golden(name, "f32")
    assert rep.iterations_run == int(g["iterations_run"])
    assert relinf(rep.energy_trace, g["trace"]) < 1e-5
    assert relinf(field.ux, g["ux"]) < 1e-4 and relinf(field.uy, g["uy"]) < 1e-4
    assert rep.msd_after == pytest.approx(float(g["msd_after"]), rel=1e-5)


def test_pixel_batch_warped_matches_golden():
    g = golden("pixel64")
    tau, lam, iters, passes = g["cfg"]
    re = np.ascontiguousarray(g["re"][None])  # not exact in fp32: pass fp64 images
    te = np.ascontiguousarray(g["te"][None])
    for prec in ("f64", "f32"):
        b = PixelBatch(1, 64, 64, tau, lam, int(iters), int(passes), precision=prec,
                       img_dtype=_lib.F64)
        b.set_images(np.ascontiguousarray(re), np.ascontiguousarray(te))
        for _ in range(2):  # second run replays the captured CUDA graph
            b.run()
            ux, uy, warped = (np.empty((1, 64, 64)) for _ in range(3))
            b.get_results(ux, uy, warped)
            rep = b.sync()[0]
            tol = 1e-10 if prec == "f64" else 1e-4
            assert relinf(warped[0], g["warped"]) < tol
            assert relinf(ux[0], g["ux"]) < tol
            assert relinf(rep.energy_trace, g["trace"]) < (1e-12 if prec == "f64" else 1e-5)
        # pad, trace, warp, msd + one k_pixel_step per iteration + the final smoothing
        assert b.launches_per_run() == 4 + int(iters) + 1
        b.close()


def test_sample_gradient_and_grid_smooth_units():
    g = golden("pixel_units")
    img = grid(g["img"])
    gx, gy = img.sample_gradient(g["pts"][:, 0], g["pts"][:, 1])
    assert np.abs(gx - g["gx"]).max() <= 1e-12 * max(1.0, np.abs(g["gx"]).max())
    assert np.abs(gy - g["gy"]).max() <= 1e-12 * max(1.0, np.abs(g["gy"]).max())
    sx, sy = img.sample_gradient(3.25, 4.5)  # scalar in, scalar out
    ox, oy = O.sample_gradient(g["img"], 3.25, 4.5)
    assert isinstance(sx, float) and sx == pytest.approx(ox[0], rel=1e-13)
    assert sy == pytest.approx(oy[0], rel=1e-13)
    assert np.array_equal(mrb.grid_umbrella_smooth(g["plane"], 0.6), g["smooth"])
    # a constant plane is a fixed point everywhere (baseline.py:30-31)
    c = np.full((9, 5), 2.5)
    assert np.array_equal(mrb.grid_umbrella_smooth(c, 0.8), c)


def test_pixel_divergence_message():
    g = golden("pixel_diverge48")
    for prec in ("f64", "f32"):
        with pytest.raises(mrb.DivergenceError) as e:
            mrb.register_pixelwise(grid(g["re"]), grid(g["te"]), tau=0.2, precision=prec)
        assert str(e.value) == str(g["error"])


def test_pixel_validation_messages():
    z = grid(np.zeros((8, 8)))
    with pytest.raises(ValueError, match="tau must be positive, got 0.0"):
        mrb.register_pixelwise(z, z, tau=0.0)
    with pytest.raises(ValueError, match=r"lambda must be in \[0, 1\), got 1.0"):
        mrb.register_pixelwise(z, z, lam=1.0)
    with pytest.raises(ValueError, match="iterations must be >= 1"):
        mrb.register_pixelwise(z, z, iterations=0)
    with pytest.raises(ValueError, match="image sizes differ"):
        mrb.register_pixelwise(z, grid(np.zeros((8, 9))))


@pytest.mark.parametrize("w,h,passes,lam", [(70, 45, 3, 0.8), (37, 90, 6, 0.5), (2, 2, 3, 0.8),
                                            (130, 33, 9, 0.7), (50, 50, -1, 0.8)])
def test_pixelwise_ragged_sizes_and_many_passes(w, h, passes, lam):
    """Tiles that do not divide the image, more passes than one fused launch
    holds (kPixMaxR = 4 -> extra smoothing-only launches), negative passes
    (range() is empty) — against the live oracle."""
    rng = np.random.default_rng(w * 1000 + h)
    yy, xx = np.mgrid[0:h, 0:w]
    re = 128 + 40 * np.sin(xx / 5.0) * np.cos(yy / 7.0) + rng.normal(0, 1, (h, w))
    te = 128 + 40 * np.sin((xx - 1.3) / 5.0) * np.cos((yy + 0.7) / 7.0) + rng.normal(0, 1, (h, w))
    ux_o, uy_o, info = O.register_pixelwise(re, te, tau=0.002, lam=lam, iterations=25,
                                            smoothing_passes=passes)
    field, rep = mrb.register_pixelwise(grid(re), grid(te), tau=0.002, lam=lam, iterations=25,
                                        smoothing_passes=passes, precision="f64")
    assert relinf(rep.energy_trace, info["energy_trace"]) < 1e-12
    assert relinf(field.ux, ux_o) < 1e-10 and relinf(field.uy, uy_o) < 1e-10
    assert rep.msd_after == pytest.approx(info["msd_after"], rel=1e-10)


def test_pixelwise_batch_matches_single_and_identical_pair():
    g1, g2 = golden("pixel64"), golden("pixel96_p1")
    ims = [(grid(g1["re"]), grid(g1["te"])), (grid(g1["te"]), grid(g1["te"]))]
    out = mrb.register_pixelwise_batch([a for a, _ in ims], [b for _, b in ims], iterations=30,
                                       precision="f64")
    single = mrb.register_pixelwise(ims[0][0], ims[0][1], iterations=30, precision="f64")
    assert np.array_equal(out[0][0].ux, single[0].ux)
    assert out[0][1].energy_trace == single[1].energy_trace
    # identical images: zero residual -> zero field, zero energy
    assert np.abs(out[1][0].ux).max() == 0.0 and out[1][1].msd_after == 0.0
    assert all(e == 0.0 for e in out[1][1].energy_trace)
    with pytest.raises(ValueError, match="share one image size"):
        mrb.register_pixelwise_batch([ims[0][0], grid(g2["re"])], [ims[0][1], grid(g2["te"])])


def test_pixel_report_msd_is_the_shared_metric():
    """report.msd_after equals msd(warp_image(template, field), reference)
    EXACTLY at the reference's width (reference test_baseline.py:56-64): the
    engine's final warp and MSD round like the public warp_image / msd."""
    from paper_1411_2141_b200 import synthetic as S
    ref = S.smooth_texture(48, 40, seed=9, low=100, high=156)
    _, te = S.warped_pair(ref, S.plateau_shift_field(48, 40, shift=(1.0, -0.5)))
    out, report = mrb.register_pixelwise(ref, te, iterations=25, precision="f64")
    assert report.msd_after == mrb.msd(mrb.warp_image(te, out), ref)
    assert report.msd_before == mrb.msd(te, ref)


@pytest.mark.slow
def test_pixelwise_full_size_512_vs_oracle():
    """A BASELINE-sized 512x512 pair (config 2 image size), 100 iterations,
    3 passes, against the live oracle; plus determinism."""
    from paper_1411_2141_b200.synthetic import CONFIGS, make_pair
    re32, te32 = make_pair(CONFIGS["c2"], 0)
    re, te = re32.astype(np.float64), te32.astype(np.float64)
    ux_o, uy_o, info = O.register_pixelwise(re, te, iterations=100)
    for prec, tol in (("f64", 1e-10), ("f32", 1e-4)):
        field, rep = mrb.register_pixelwise(grid(re), grid(te), iterations=100, precision=prec)
        assert relinf(field.ux, ux_o) < tol and relinf(field.uy, uy_o) < tol
        assert relinf(rep.energy_trace, info["energy_trace"]) < tol / 10
        assert rep.msd_after == pytest.approx(info["msd_after"], rel=tol / 10)
    again = mrb.register_pixelwise(grid(re), grid(te), iterations=100, precision="f32")
    assert np.array_equal(again[0].ux, field.ux) and again[1].energy_trace == rep.energy_trace
