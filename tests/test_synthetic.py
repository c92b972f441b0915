"""The reference package's synthetic generators (reference synthetic.py),
mirrored in paper_1411_2141_b200.synthetic, against vectors the reference
itself produced (tests/golden/make_synthetic_golden.py)."""
import os

import numpy as np
import pytest

from paper_1411_2141_b200 import synthetic as S

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "synthetic_ref.npz"))


def test_textures_and_fields_bit_identical():
    assert np.array_equal(S.smooth_texture(40, 28, seed=3).data, G["texture"])
    assert np.array_equal(S.smooth_texture(24, 24, seed=5, sigma=2.0, low=100, high=156).data,
                          G["texture_args"])
    b = S.gaussian_bump_field(32, 20, (10.5, 12.0), 5.0, (1.0, -2.0))
    assert np.array_equal(b.ux, G["bump_ux"]) and np.array_equal(b.uy, G["bump_uy"])
    r = S.random_bump_field(40, 28, seed=2, n_bumps=3, max_amplitude=2.5, sigma_range=(6.0, 11.0))
    assert np.array_equal(r.ux, G["rand_ux"]) and np.array_equal(r.uy, G["rand_uy"])
    assert abs(float(np.max(np.hypot(r.ux, r.uy))) - 2.5) < 1e-12
    p = S.plateau_shift_field(40, 28, shift=(2.0, -1.0))
    assert np.array_equal(p.ux, G["plateau_ux"]) and np.array_equal(p.uy, G["plateau_uy"])
    assert np.array_equal(S.brain_phantom(48, seed=1).data, G["phantom"])


def test_flat_texture_and_stack_errors():
    flat = S.smooth_texture(1, 1, seed=0)  # one pixel: no range to stretch
    assert np.all(flat.data == 0.5 * (78.0 + 182.0))
    with pytest.raises(ValueError, match="count must be >= 1"):
        S.slice_stack(8, 8, 0)


@pytest.mark.gpu
def test_warped_pair_and_slice_stack_match_reference():
    r = S.random_bump_field(40, 28, seed=2, n_bumps=3, max_amplitude=2.5, sigma_range=(6.0, 11.0))
    ref, te = S.warped_pair(S.smooth_texture(40, 28, seed=3), r)
    assert np.abs(te.data - G["warped_te"]).max() <= 1e-12 * np.abs(G["warped_te"]).max()
    st = S.slice_stack(40, 28, 3, seed=4, max_shift=1.5)
    got = np.stack([s.data for s in st])
    assert np.abs(got - G["stack"]).max() <= 1e-12 * np.abs(G["stack"]).max()
