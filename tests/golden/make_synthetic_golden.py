"""Golden vectors of the reference's synthetic generators (reference
synthetic.py), made by importing the reference in the build container:
    python tests/golden/make_synthetic_golden.py
writes tests/golden/synthetic_ref.npz (small sizes; the GPU box has no copy
of the reference)."""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import meshreg.synthetic as S  # noqa: E402

out = {}
out["texture"] = S.smooth_texture(40, 28, seed=3).data
out["texture_args"] = S.smooth_texture(24, 24, seed=5, sigma=2.0, low=100, high=156).data
b = S.gaussian_bump_field(32, 20, (10.5, 12.0), 5.0, (1.0, -2.0))
out["bump_ux"], out["bump_uy"] = b.ux, b.uy
r = S.random_bump_field(40, 28, seed=2, n_bumps=3, max_amplitude=2.5, sigma_range=(6.0, 11.0))
out["rand_ux"], out["rand_uy"] = r.ux, r.uy
p = S.plateau_shift_field(40, 28, shift=(2.0, -1.0))
out["plateau_ux"], out["plateau_uy"] = p.ux, p.uy
out["phantom"] = S.brain_phantom(48, seed=1).data
ref, te = S.warped_pair(S.smooth_texture(40, 28, seed=3), r)
out["warped_te"] = te.data
st = S.slice_stack(40, 28, 3, seed=4, max_shift=1.5)
out["stack"] = np.stack([s.data for s in st])
np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "synthetic_ref.npz"),
                    **out)
print({k: v.shape for k, v in out.items()})
