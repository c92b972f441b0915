"""Delaunay triangulation and edge flipping (mirror of reference
pkg/src/meshreg/delaunay.py).

Same names, arguments, results and exceptions as the reference, computed by
libmeshreg_b200 (no CPU fallback):

* ``delaunay`` / ``flip_edges`` / ``dedupe_points`` run in native C++
  (csrc/mesher_host.cpp).  Bowyer-Watson locates each point by walking the
  triangulation and grows its cavity through triangle adjacency instead of
  scanning every triangle ever created (delaunay.py:151-160, O(n^2)); the
  triangle ids, the cavity-edge order of the reference's Python set and every
  floating-point expression are reproduced, so the triangulation is
  bit-identical to the reference's.
* ``delaunay_violations`` (the mesh audit) is a GPU kernel.
* ``circumcircles`` is the reference's small elementwise helper, kept in
  numpy on the host.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .mesh import TriMesh

__all__ = ["delaunay", "flip_edges", "dedupe_points", "delaunay_violations", "circumcircles"]

# Cocircularity slack, in pixels of circumcircle depth (delaunay.py:27).
TIE_EPS = 1e-9
_ERR = 512


def dedupe_points(points, tol=1e-9):
    """Lexicographically sorted points with near-duplicates (within tol)
    removed (delaunay.py:30-51)."""
    P = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, 2))
    out = np.empty_like(P)
    cnt = C.c_int64()
    err = C.create_string_buffer(_ERR)
    rc = _lib.load().mrb_dedupe_points(P.shape[0], _lib.ptr(P), float(tol), _lib.ptr(out),
                                       C.byref(cnt), err, _ERR)
    if rc != _lib.OK:
        raise ValueError(err.value.decode())
    return out[: cnt.value].copy()


def circumcircles(V, T):
    """Circumcenters and squared radii of triangles as (cx, cy, r2) arrays
    (delaunay.py:54-72)."""
    V = np.asarray(V, dtype=np.float64)
    T = np.asarray(T, dtype=np.int64)
    a = V[T[:, 0]]
    b = V[T[:, 1]]
    c = V[T[:, 2]]
    ab = b - a
    ac = c - a
    d = 2.0 * (ab[:, 0] * ac[:, 1] - ab[:, 1] * ac[:, 0])
    with np.errstate(divide="ignore", invalid="ignore"):
        ab2 = (ab * ab).sum(axis=1)
        ac2 = (ac * ac).sum(axis=1)
        ux = (ac[:, 1] * ab2 - ab[:, 1] * ac2) / d
        uy = (ab[:, 0] * ac2 - ac[:, 0] * ab2) / d
    bad = ~np.isfinite(ux) | ~np.isfinite(uy)
    ux[bad] = 0.0
    uy[bad] = 0.0
    r2 = ux * ux + uy * uy
    r2[bad] = np.inf
    return a[:, 0] + ux, a[:, 1] + uy, r2


class _Tris:
    """Owner of a native mrb_tris handle (a triangulation between mesher
    stages)."""

    def __init__(self, handle):
        self.h = handle

    @classmethod
    def from_mesh(cls, mesh):
        V = np.ascontiguousarray(mesh.vertices, dtype=np.float64)
        T = np.ascontiguousarray(mesh.triangles, dtype=np.int64)
        h = C.c_void_p()
        err = C.create_string_buffer(_ERR)
        rc = _lib.load().mrb_tris_create(V.shape[0], _lib.ptr(V), T.shape[0], _lib.ptr(T),
                                         C.byref(h), err, _ERR)
        if rc != _lib.OK:
            raise ValueError(err.value.decode())
        return cls(h.value)

    def arrays(self):
        lib = _lib.load()
        n, m = C.c_int64(), C.c_int64()
        lib.mrb_tris_counts(self.h, C.byref(n), C.byref(m))
        V = np.empty((n.value, 2), np.float64)
        T = np.empty((m.value, 3), np.int64)
        lib.mrb_tris_export(self.h, _lib.ptr(V), _lib.ptr(T))
        return V, T

    def to_mesh(self):
        V, T = self.arrays()
        return TriMesh(V, T)

    def flip(self, passes):
        changed = C.c_int32()
        err = C.create_string_buffer(_ERR)
        rc = _lib.load().mrb_flip_edges(self.h, int(passes), C.byref(changed), err, _ERR)
        if rc != _lib.OK:
            raise ValueError(err.value.decode())
        return changed.value

    def __del__(self):
        if self.h and _lib._lib is not None:
            _lib._lib.mrb_tris_destroy(self.h)
            self.h = None


def _delaunay_tris(points):
    P = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, 2))
    h = C.c_void_p()
    err = C.create_string_buffer(_ERR)
    rc = _lib.load().mrb_delaunay(P.shape[0], _lib.ptr(P), C.byref(h), err, _ERR)
    if rc == _lib.E_VALUE:
        raise ValueError(err.value.decode())
    if rc != _lib.OK:
        raise RuntimeError(err.value.decode())
    return _Tris(h.value)


def delaunay(points):
    """Delaunay triangulation of a 2-D point set as a :class:`TriMesh`
    (delaunay.py:75-91).  Near-duplicates (within 1e-9) are removed first;
    ValueError for fewer than three distinct points or an all-collinear set."""
    return _delaunay_tris(points).to_mesh()


def flip_edges(mesh, passes=16):
    """Flip interior edges until every one passes the local Delaunay test,
    at most ``passes`` sweeps (delaunay.py:181-199).  Returns ``mesh`` itself
    when nothing flipped, else a new TriMesh."""
    t = _Tris.from_mesh(mesh)
    if t.flip(passes) == 0:
        return mesh
    return t.to_mesh()


def delaunay_violations(V, T, margin=1e-9):
    """Count (triangle, vertex) pairs where a vertex sits deeper than
    ``margin`` inside a circumcircle (delaunay.py:290-309), on the GPU."""
    V = np.ascontiguousarray(np.asarray(V, dtype=np.float64).reshape(-1, 2))
    T = np.ascontiguousarray(np.asarray(T, dtype=np.int64).reshape(-1, 3))
    ctx = _lib.context()
    cnt = C.c_int64()
    rc = _lib.load().mrb_delaunay_violations(ctx, V.shape[0], _lib.ptr(V), T.shape[0],
                                             _lib.ptr(T), float(margin), C.byref(cnt))
    _lib.check(rc, ctx, (ValueError, RuntimeError, RuntimeError))
    return int(cnt.value)
