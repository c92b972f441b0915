"""Seeded synthetic image pairs for the BASELINE.json configurations.

This is input generation, not the registration path: it produces the fp32
reference/template pairs that BOTH the B200 path and the CPU reference are fed
("Synthetic inputs").  The paper's brain-CT data is not
available (reference PAPER.md:182,204), so these seeded pairs stand in for it
with the shapes and value distributions BASELINE.json's `configs` give.

Draw order (one ``np.random.default_rng(seed)`` per pair):
  1. per blob: cx, cy ~ U(0,S); sigma ~ U(8,30); a ~ U(0.2,1); add a*exp(-r^2/2sigma^2)
  2. per rectangle: x0, y0 ~ integers(0,S); w, h ~ integers(S//32, S//4);
     paint img[y0:y0+h, x0:x0+w] = U(0.3, 0.9)
  3. add normal(0, 0.01) per pixel; clip to [0, 1]
  4. per RBF (8): cx, cy ~ U(0,S); ax, ay ~ U(-1,1); sigma = 40 px; rescale so
     max |u| == peak
  5. Re = fp32(img); Te = fp32(backward Catmull-Rom warp of Re by the field),
     the same warp the reference uses to build its own synthetic pairs
     (reference synthetic.py:88-91 -> densefield.py:190-199).

The warp below is a plain numpy statement of that interpolant so that the
generator runs anywhere (the GPU box has no copy of the reference).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["PairSpec", "CONFIGS", "make_pair", "catmull_rom_warp", "scaled_pair",
           # the reference package's own generators (reference synthetic.py:17-24)
           "smooth_texture", "gaussian_bump_field", "random_bump_field",
           "plateau_shift_field", "warped_pair", "slice_stack", "brain_phantom"]


@dataclass(frozen=True)
class PairSpec:
    name: str
    size: int
    n_blobs: int
    n_rects: int
    peak: float
    target_nodes: int
    iterations: int


# BASELINE.json "configs" (alpha has no reference parameter: SURVEY.md §0.1)
CONFIGS = {
    "c1": PairSpec("c1", 256, 20, 0, 4.0, 3000, 100),
    "c2": PairSpec("c2", 512, 40, 0, 8.0, 12000, 200),
    "c3": PairSpec("c3", 1024, 80, 30, 12.0, 50000, 200),
    "c4": PairSpec("c4", 512, 40, 0, 8.0, 12000, 200),  # 64 pairs, seeds 0..63
    "c5": PairSpec("c5", 4096, 300, 100, 24.0, 500000, 300),
}


def _extend_axis(a, axis):
    a = np.moveaxis(a, axis, 0)
    n = a.shape[0]
    if n >= 3:
        lo = 3.0 * a[0] - 3.0 * a[1] + a[2]
        hi = 3.0 * a[-1] - 3.0 * a[-2] + a[-3]
    elif n == 2:
        lo = 2.0 * a[0] - a[1]
        hi = 2.0 * a[-1] - a[-2]
    else:
        lo = hi = a[0]
    out = np.concatenate([lo[None], a, hi[None]], axis=0)
    return np.moveaxis(out, 0, axis)


def _cr(t):
    t2 = t * t
    t3 = t2 * t
    return (
        0.5 * (-t3 + 2.0 * t2 - t),
        0.5 * (3.0 * t3 - 5.0 * t2 + 2.0),
        0.5 * (-3.0 * t3 + 4.0 * t2 + t),
        0.5 * (t3 - t2),
    )


def catmull_rom_warp(img, ux, uy):
    """out(p) = img(p + u(p)), Catmull-Rom, clamped, quadratic border ring."""
    img = np.asarray(img, dtype=np.float64)
    h, w = img.shape
    ext = _extend_axis(_extend_axis(img, 1), 0)
    gx, gy = np.meshgrid(np.arange(w, dtype=np.float64), np.arange(h, dtype=np.float64))
    x = np.clip(gx + ux, 0.0, w - 1.0)
    y = np.clip(gy + uy, 0.0, h - 1.0)
    x0 = np.minimum(np.floor(x), max(w - 2, 0)).astype(np.int64)
    y0 = np.minimum(np.floor(y), max(h - 2, 0)).astype(np.int64)
    wx = _cr(x - x0)
    wy = _cr(y - y0)
    out = np.zeros_like(x)
    for j in range(4):
        row = np.zeros_like(x)
        for i in range(4):
            row += wx[i] * ext[y0 + j, x0 + i]
        out += wy[j] * row
    return out


def make_pair(spec: PairSpec, seed: int, scale: float = 1.0):
    """Return (re, te) as float32 (H, W) arrays for one seeded pair.

    ``scale`` multiplies the clipped [0,1] image before the warp (the x255
    large-motion parity cases of SURVEY.md §8(c) use scale=255).
    """
    S = spec.size
    rng = np.random.default_rng(seed)
    gx, gy = np.meshgrid(np.arange(S, dtype=np.float64), np.arange(S, dtype=np.float64))
    img = np.zeros((S, S))
    for _ in range(spec.n_blobs):
        cx = rng.uniform(0, S)
        cy = rng.uniform(0, S)
        sig = rng.uniform(8.0, 30.0)
        a = rng.uniform(0.2, 1.0)
        img += a * np.exp(-((gx - cx) ** 2 + (gy - cy) ** 2) / (2.0 * sig * sig))
    for _ in range(spec.n_rects):
        x0 = int(rng.integers(0, S))
        y0 = int(rng.integers(0, S))
        rw = int(rng.integers(S // 32, S // 4))
        rh = int(rng.integers(S // 32, S // 4))
        img[y0:y0 + rh, x0:x0 + rw] = rng.uniform(0.3, 0.9)
    img += rng.normal(0.0, 0.01, size=(S, S))
    img = np.clip(img, 0.0, 1.0) * scale
    ux = np.zeros((S, S))
    uy = np.zeros((S, S))
    for _ in range(8):
        cx = rng.uniform(0, S)
        cy = rng.uniform(0, S)
        ax = rng.uniform(-1.0, 1.0)
        ay = rng.uniform(-1.0, 1.0)
        bump = np.exp(-((gx - cx) ** 2 + (gy - cy) ** 2) / (2.0 * 40.0 * 40.0))
        ux += ax * bump
        uy += ay * bump
    peak = float(np.max(np.hypot(ux, uy)))
    if peak > 1e-12:
        ux *= spec.peak / peak
        uy *= spec.peak / peak
    re = img.astype(np.float32)
    te = catmull_rom_warp(re.astype(np.float64), ux, uy).astype(np.float32)
    return re, te


def scaled_pair(spec: PairSpec, seed: int):
    """The x255 large-motion variant of a config pair."""
    return make_pair(spec, seed, scale=255.0)


# --------------------------------------------------------------------------
# The reference package's synthetic module (reference synthetic.py:27-135):
# textures, bump fields, slice stacks and the brain phantom its tests and its
# bench harness draw their inputs from.  Same seeds, draw order and formulas,
# so a caller of `meshreg.synthetic` gets the same arrays here; the warps run
# through this package's warp_image (the GPU path).

def _pixel_coordinates(width, height):
    """(x, y) coordinate planes of a width x height grid, float64."""
    xs = np.arange(width, dtype=np.float64)
    ys = np.arange(height, dtype=np.float64)
    return np.meshgrid(xs, ys)


def _gaussian_filter(a, sigma, **kw):
    from scipy import ndimage
    return ndimage.gaussian_filter(a, sigma, **kw)


def smooth_texture(width, height, seed=0, sigma=3.0, low=78.0, high=182.0):
    """Gaussian-filtered white noise stretched linearly onto [low, high]
    (a flat result maps to the mid value); reference synthetic.py:27-42."""
    from .image import ImageGrid
    field = _gaussian_filter(np.random.default_rng(seed).standard_normal((height, width)),
                             sigma, mode="nearest")
    fmin, fmax = float(field.min()), float(field.max())
    if fmax - fmin < 1e-12:
        return ImageGrid(width, height, np.full((height, width), 0.5 * (low + high)))
    return ImageGrid(width, height, low + (field - fmin) * ((high - low) / (fmax - fmin)))


def gaussian_bump_field(width, height, center, sigma, amplitude):
    """amplitude * exp(-|p - center|^2 / (2 sigma^2)) per component
    (reference synthetic.py:45-51)."""
    from .densefield import DenseField
    x, y = _pixel_coordinates(width, height)
    g = np.exp(-((x - center[0]) ** 2 + (y - center[1]) ** 2) / (2.0 * sigma * sigma))
    return DenseField(amplitude[0] * g, amplitude[1] * g)


def random_bump_field(width, height, seed=0, n_bumps=3, max_amplitude=4.0,
                      sigma_range=(30.0, 55.0)):
    """n_bumps random Gaussian bumps summed, then scaled to a peak magnitude
    of max_amplitude pixels (reference synthetic.py:54-74; draws per bump:
    cx, cy, sigma, then the amplitude pair)."""
    from .densefield import DenseField
    rng = np.random.default_rng(seed)
    total_x = np.zeros((height, width))
    total_y = np.zeros((height, width))
    for _ in range(n_bumps):
        cx = rng.uniform(0.25 * width, 0.75 * width)
        cy = rng.uniform(0.25 * height, 0.75 * height)
        s = rng.uniform(*sigma_range)
        amp = rng.uniform(-1.0, 1.0, size=2)
        one = gaussian_bump_field(width, height, (cx, cy), s, (amp[0], amp[1]))
        total_x += one.ux
        total_y += one.uy
    top = float(np.max(np.hypot(total_x, total_y)))
    if top > 1e-12:
        total_x *= max_amplitude / top
        total_y *= max_amplitude / top
    return DenseField(total_x, total_y)


def plateau_shift_field(width, height, shift=(2.0, 0.0), frac=0.42, power=8):
    """A translation by `shift` that a super-Gaussian window exp(-r^power)
    fades out toward the border (reference synthetic.py:77-85)."""
    from .densefield import DenseField
    x, y = _pixel_coordinates(width, height)
    rho = np.hypot((x - (width - 1) / 2.0) / (frac * width),
                   (y - (height - 1) / 2.0) / (frac * height))
    window = np.exp(-(rho ** power))
    return DenseField(shift[0] * window, shift[1] * window)


def warped_pair(reference, field):
    """(Re, Te) with Te(p) = Re(p + u(p)) (reference synthetic.py:88-91)."""
    from .densefield import warp_image
    return reference, warp_image(reference, field)


def slice_stack(width, height, count, seed=0, max_shift=2.0):
    """`count` slices: a texture, then each slice the previous one warped by
    a fresh two-bump field of peak max_shift (reference synthetic.py:94-108)."""
    from .densefield import warp_image
    if count < 1:
        raise ValueError("count must be >= 1")
    rng = np.random.default_rng(seed)
    stack = [smooth_texture(width, height, seed=seed)]
    while len(stack) < count:
        field = random_bump_field(width, height, seed=int(rng.integers(2**31)), n_bumps=2,
                                  max_amplitude=max_shift)
        stack.append(warp_image(stack[-1], field))
    return stack


def brain_phantom(size=512, seed=0):
    """Elliptic head: bright shell, textured interior, two dark lobes, a
    final 1.2-px blur (reference synthetic.py:111-135)."""
    from .image import ImageGrid
    rng = np.random.default_rng(seed)
    x, y = _pixel_coordinates(size, size)
    mid = (size - 1) / 2.0
    rho = np.hypot((x - mid) / (0.42 * size), (y - mid) / (0.34 * size))
    img = np.where(rho < 1.0, 70.0, 0.0)
    img[(rho >= 0.88) & (rho < 1.0)] = 235.0
    noise = _gaussian_filter(rng.standard_normal((size, size)), 6.0)
    noise = 60.0 * (noise - noise.min()) / max(noise.max() - noise.min(), 1e-12)
    inside = rho < 0.88
    img[inside] = 90.0 + noise[inside]
    for ox in (-0.16, 0.16):
        ex = (x - mid - ox * size) / (0.05 * size)
        ey = (y - mid + 0.05 * size) / (0.16 * size)
        img[ex * ex + ey * ey < 1.0] = 25.0
    return ImageGrid(size, size, _gaussian_filter(img, 1.2))
