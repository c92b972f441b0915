"""Image container and MSD (mirror of reference pkg/src/meshreg/image.py).

`ImageGrid` keeps the reference's container semantics (image.py:25-131):
row-major float64 (H, W), read-only, finite-checked.  Sampling and `msd` run
on the GPU through libmeshreg_b200 (no CPU fallback).  load_image /
save_image read and write the reference's file formats (image.py:190-296:
PGM P2/P5 up to 16 bit, PNG through Pillow, rescaled to [0, 255]); they feed
the command-line front end (cli.py).
"""

from __future__ import annotations

import os
import re

import numpy as np

from . import _lib

__all__ = ["ImageGrid", "msd", "load_image", "save_image", "FileFormatError"]


class FileFormatError(ValueError):
    """Malformed or unsupported image / field / mesh file (image.py:21-22)."""


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


# ---- file formats (image.py:190-296) ----------------------------------------
_PNG_SIGNATURE = b"\x89PNG\r\n\x1a\n"
_LUMA = (0.299, 0.587, 0.114)  # Rec. 601, as the reference converts colour PNGs


def load_image(path):
    """PGM (P2 text / P5 binary, maxval <= 65535) or PNG -> ImageGrid with
    intensities rescaled so that full scale is 255.0 (image.py:197-209)."""
    with open(path, "rb") as fh:
        head = fh.read(8)
    if head[:2] in (b"P2", b"P5"):
        return _read_pgm(path)
    if head == _PNG_SIGNATURE:
        return _read_png(path)
    raise FileFormatError(f"unsupported image format: {path!r}")


def save_image(img, path):
    """8-bit binary PGM or grayscale PNG by extension; values rounded half to
    even and clamped to [0, 255] (image.py:212-228)."""
    pix = np.clip(np.rint(img.data), 0, 255).astype(np.uint8)
    ext = os.path.splitext(str(path))[1].lower()
    if ext == ".pgm":
        with open(path, "wb") as fh:
            fh.write(b"P5\n%d %d\n255\n" % (img.width, img.height))
            fh.write(pix.tobytes())
    elif ext == ".png":
        from PIL import Image as _PIL

        _PIL.fromarray(pix, mode="L").save(path, format="PNG")
    else:
        raise ValueError(f"unsupported output extension: {ext!r} (use .pgm or .png)")


def _pgm_header(blob):
    """Width, height and maxval tokens after the magic (comments allowed
    between tokens), and the offset of the pixel data: one whitespace byte
    after the last token (image.py:258-276)."""
    tokens = []
    pos = 2
    number = re.compile(rb"[0-9]+")
    while len(tokens) < 3 and pos < len(blob):
        c = blob[pos:pos + 1]
        if c == b"#":
            end = blob.find(b"\n", pos)
            pos = len(blob) if end < 0 else end + 1
        elif c.isspace():
            pos += 1
        else:
            m = number.match(blob, pos)
            if m is None:
                raise FileFormatError("malformed PGM header")
            tokens.append(int(m.group(0)))
            pos = m.end()
    return tokens, pos + 1


def _read_pgm(path):
    with open(path, "rb") as fh:
        blob = fh.read()
    tokens, body = _pgm_header(blob)
    if len(tokens) < 3:
        raise FileFormatError(f"truncated PGM header in {path!r}")
    width, height, maxval = tokens
    if width < 1 or height < 1:
        raise FileFormatError(f"zero-dimension PGM image in {path!r}")
    if not 0 < maxval <= 65535:
        raise FileFormatError(f"PGM maxval {maxval} out of range in {path!r}")
    count = width * height
    if blob[:2] == b"P2":
        vals = np.array(blob[body:].split()[:count], dtype=np.float64)
    else:
        dt = np.dtype(">u2" if maxval > 255 else "u1")
        vals = np.frombuffer(blob[body:body + count * dt.itemsize], dtype=dt).astype(np.float64)
    if vals.size != count:
        raise FileFormatError(f"PGM pixel data truncated in {path!r}")
    return ImageGrid(width, height, vals * (255.0 / maxval))


def _read_png(path):
    from PIL import Image as _PIL

    with _PIL.open(path) as im:
        im.load()
        if im.width < 1 or im.height < 1:
            raise FileFormatError(f"zero-dimension PNG image in {path!r}")
        mode = im.mode
        if mode == "L":
            arr = np.asarray(im, dtype=np.float64)
        elif mode == "LA":
            arr = np.asarray(im.convert("L"), dtype=np.float64)
        elif mode in ("I", "I;16", "I;16B", "I;16L"):
            arr = np.asarray(im, dtype=np.float64) * (255.0 / 65535.0)
        elif mode in ("RGB", "RGBA", "P"):
            rgb = np.asarray(im.convert("RGB"), dtype=np.float64)
            arr = _LUMA[0] * rgb[..., 0] + _LUMA[1] * rgb[..., 1] + _LUMA[2] * rgb[..., 2]
        else:
            raise FileFormatError(f"unsupported PNG mode {mode!r} in {path!r}")
    return ImageGrid(arr.shape[1], arr.shape[0], arr)
