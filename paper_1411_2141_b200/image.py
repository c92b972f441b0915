"""Image container and MSD (mirror of reference pkg/src/meshreg/image.py).

`ImageGrid` keeps the reference's container semantics (image.py:25-131):
row-major float64 (H, W), read-only, finite-checked.  Sampling and `msd` run
on the GPU through libmeshreg_b200 (no CPU fallback).  File I/O
(load_image/save_image) is not on the registration path and is out of scope.
"""

from __future__ import annotations

import numpy as np

from . import _lib

__all__ = ["ImageGrid", "msd"]


class ImageGrid:
    """Immutable 2-D intensity field, x = column, y = row (image.py:25-55)."""

    __slots__ = ("width", "height", "data")

    def __init__(self, width, height, data):
        width = int(width)
        height = int(height)
        if width < 1 or height < 1:
            raise ValueError(f"image dimensions must be positive, got {width}x{height}")
        arr = np.asarray(data, dtype=np.float64)
        if arr.size != width * height:
            raise ValueError(
                f"data has {arr.size} values, expected {width * height} for {width}x{height}")
        if not np.all(np.isfinite(arr)):
            raise ValueError("image intensities must be finite")
        arr = arr.reshape(height, width).copy()
        arr.setflags(write=False)
        self.width = width
        self.height = height
        self.data = arr

    @property
    def shape(self):
        return (self.height, self.width)

    def sample(self, x, y):
        """Catmull-Rom bicubic value at continuous coordinates (image.py:73-84),
        computed by the sm_100a sampling kernel in fp64."""
        x = np.asarray(x, dtype=np.float64)
        y = np.asarray(y, dtype=np.float64)
        scalar = x.ndim == 0 and y.ndim == 0
        xb, yb = np.broadcast_arrays(x, y)
        pts = np.ascontiguousarray(np.stack([xb.ravel(), yb.ravel()], axis=1))
        out = sample_points(self, pts)
        return float(out[0]) if scalar else out.reshape(xb.shape)

    def sample_gradient(self, x, y):
        """Analytic (d/dx, d/dy) of the bicubic interpolant (image.py:86-103),
        one-sided at clamped out-of-domain points; fp64 on the GPU."""
        x = np.asarray(x, dtype=np.float64)
        y = np.asarray(y, dtype=np.float64)
        scalar = x.ndim == 0 and y.ndim == 0
        xb, yb = np.broadcast_arrays(x, y)
        pts = np.ascontiguousarray(np.stack([xb.ravel(), yb.ravel()], axis=1))
        lib = _lib.load()
        ctx = _lib.context()
        data, dt = _lib.image_payload(self.data)
        gx = np.empty(pts.shape[0])
        gy = np.empty(pts.shape[0])
        rc = lib.mrb_sample_gradient(ctx, self.width, self.height, dt, _lib.ptr(data),
                                     pts.shape[0], _lib.ptr(pts), _lib.ptr(gx), _lib.ptr(gy))
        _lib.check(rc, ctx, (ValueError, RuntimeError, RuntimeError))
        if scalar:
            return float(gx[0]), float(gy[0])
        return gx.reshape(xb.shape), gy.reshape(xb.shape)

    def __eq__(self, other):
        if not isinstance(other, ImageGrid):
            return NotImplemented
        return self.shape == other.shape and np.array_equal(self.data, other.data)

    def __repr__(self):
        return f"ImageGrid({self.width}x{self.height})"


def sample_points(img, pts, u=None):
    """Sample `img` (any object with width/height/data) at pts (+ u), fp64."""
    lib = _lib.load()
    ctx = _lib.context()
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    n = pts.shape[0]
    u = np.zeros_like(pts) if u is None else np.ascontiguousarray(u, dtype=np.float64)
    data, dt = _lib.image_payload(img.data)
    out = np.empty(n, dtype=np.float64)
    rc = lib.mrb_warp_sample(ctx, img.width, img.height, dt, _lib.ptr(data), n, _lib.ptr(pts),
                             _lib.ptr(u), _lib.ptr(out))
    _lib.check(rc, ctx, (ValueError, RuntimeError, RuntimeError))
    return out


def msd(a, b):
    """Mean squared intensity difference (image.py:181-186), fp64 on device."""
    if a.shape != b.shape:
        raise ValueError(f"dimension mismatch: {a.shape} vs {b.shape}")
    lib = _lib.load()
    ctx = _lib.context()
    da = np.ascontiguousarray(a.data, dtype=np.float64)
    db = np.ascontiguousarray(b.data, dtype=np.float64)
    out = np.zeros(1)
    rc = lib.mrb_msd(ctx, da.size, _lib.ptr(da), _lib.ptr(db), _lib.ptr(out))
    _lib.check(rc, ctx, (ValueError, RuntimeError, RuntimeError))
    return float(out[0])
