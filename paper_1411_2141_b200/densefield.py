"""Dense fields (mirror of reference pkg/src/meshreg/densefield.py).

densify and warp_image run on the GPU: the pixel->triangle map is rasterised
once per (mesh, W, H) with fp64 predicates in numpy's operation order
(lowest-index tie-break, densefield.py:148-174) and a host fallback for
pixels the raster leaves unassigned (PointLocator/locate, 62-127).  The MRDF
and CSV file formats are not on the registration path (out of scope).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .image import ImageGrid
from .mesh import as_mesh

__all__ = ["DenseField", "MeshCoverageError", "densify", "warp_image", "pixel_map"]


class DenseField:
    """Per-pixel displacement planes ux/uy (densefield.py:33-55)."""

    __slots__ = ("width", "height", "ux", "uy")

    def __init__(self, ux, uy):
        ux = np.asarray(ux, dtype=np.float64)
        uy = np.asarray(uy, dtype=np.float64)
        if ux.ndim != 2 or ux.shape != uy.shape:
            raise ValueError(f"displacement planes must match, got {ux.shape} vs {uy.shape}")
        if not (np.all(np.isfinite(ux)) and np.all(np.isfinite(uy))):
            raise ValueError("displacement planes must be finite")
        self.height, self.width = ux.shape
        self.ux = ux
        self.uy = uy

    @property
    def shape(self):
        return (self.height, self.width)

    @classmethod
    def zero(cls, width, height):
        return cls(np.zeros((height, width)), np.zeros((height, width)))


class MeshCoverageError(RuntimeError):
    """An in-domain point was not covered by any mesh triangle."""


def _errs():
    from .solver import DivergenceError
    return (ValueError, DivergenceError, MeshCoverageError)


def _default_size(mesh, width, height):
    V = mesh.vertices
    if width is None:
        width = int(round(V[:, 0].max())) + 1
    if height is None:
        height = int(round(V[:, 1].max())) + 1
    return int(width), int(height)


def densify(mesh, u, width=None, height=None):
    """Barycentric interpolation of node displacements to pixels
    (densefield.py:130-187)."""
    mesh = as_mesh(mesh)
    u = np.ascontiguousarray(u, dtype=np.float64)
    if u.shape != (mesh.n_vertices, 2):
        raise ValueError(f"displacement shape {u.shape} != ({mesh.n_vertices}, 2)")
    width, height = _default_size(mesh, width, height)
    ux = np.empty((height, width))
    uy = np.empty((height, width))
    lib = _lib.load()
    ctx = _lib.context()
    rc = lib.mrb_densify(ctx, mesh._h, width, height, _lib.ptr(u), _lib.ptr(ux), _lib.ptr(uy))
    _lib.check(rc, ctx, _errs())
    return DenseField(ux, uy)


def warp_image(template, field):
    """Backward warp out(p) = Te(p + u(p)) (densefield.py:190-199)."""
    if (field.height, field.width) != template.shape:
        raise ValueError(f"field {field.shape} does not match image {template.shape}")
    data, dt = _lib.image_payload(template.data)
    ux = np.ascontiguousarray(field.ux, dtype=np.float64)
    uy = np.ascontiguousarray(field.uy, dtype=np.float64)
    out = np.empty((field.height, field.width))
    lib = _lib.load()
    ctx = _lib.context()
    rc = lib.mrb_warp_image(ctx, field.width, field.height, dt, _lib.ptr(data), _lib.ptr(ux),
                            _lib.ptr(uy), _lib.ptr(out))
    _lib.check(rc, ctx, _errs())
    return ImageGrid(field.width, field.height, out)


def pixel_map(mesh, width, height):
    """(tri_of (H, W) int64, weights (H, W, 3)) — the map densify uses
    (densefield.py:148-182), exported for bit-exact parity checks."""
    mesh = as_mesh(mesh)
    tri_of = np.empty((height, width), np.int64)
    w = np.empty((height, width, 3))
    lib = _lib.load()
    ctx = _lib.context()
    rc = lib.mrb_pixel_map(ctx, mesh._h, int(width), int(height), _lib.ptr(tri_of), _lib.ptr(w))
    _lib.check(rc, ctx, _errs())
    return tri_of, w
