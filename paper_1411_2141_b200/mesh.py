"""Mesh connectivity and operators (mirror of reference pkg/src/meshreg/mesh.py).

`TriMesh` validates, orients and builds connectivity, CSR operators and
geometry in native code (mrb_mesh_build), bit-exact with the reference
(TriMesh.__init__ mesh.py:58-123, TriangleGeometry 173-213, build_laplacian
254-265).  The operators are returned as scipy CSR arrays exactly like the
reference's, and the per-iteration operators run on the GPU.
"""

from __future__ import annotations

import ctypes as C
import weakref

import numpy as np
from scipy import sparse

from . import _lib

__all__ = [
    "TriMesh",
    "DeferredMesh",
    "TriangleGeometry",
    "build_adjacency",
    "vertex_gradient_all",
    "triangle_gradient",
    "vertex_gradient",
    "umbrella",
    "build_laplacian",
    "smooth_displacement",
]

DEGENERATE_AREA = 1e-9


def _mesh_arrays(vertices, triangles):
    V = np.ascontiguousarray(np.asarray(vertices, dtype=np.float64))
    T = np.ascontiguousarray(np.asarray(triangles, dtype=np.int64))
    if V.ndim != 2 or V.shape[1] != 2:
        raise ValueError(f"vertices must be (n, 2), got {V.shape}")
    if T.ndim != 2 or T.shape[1] != 3 or T.shape[0] < 1:
        raise ValueError(f"triangles must be (m, 3) with m >= 1, got {T.shape}")
    return V, T


class TriMesh:
    """Static 2-D triangulation with one-ring connectivity (mesh.py:31-145)."""

    def __init__(self, vertices, triangles):
        V, T = _mesh_arrays(vertices, triangles)
        lib = _lib.load()
        h = C.c_void_p()
        err = C.create_string_buffer(512)
        rc = lib.mrb_mesh_build(V.shape[0], _lib.ptr(V), T.shape[0], _lib.ptr(T), C.byref(h),
                                err, 512)
        if rc != _lib.OK:
            raise ValueError(err.value.decode())
        self._adopt(h.value, V)

    @classmethod
    def build_many(cls, meshes):
        """[(vertices, triangles), ...] -> [TriMesh], built in parallel on the
        library's host worker pool (mrb_mesh_build_many).  Raises the
        ValueError the first invalid mesh (lowest index) would raise alone."""
        arrs = [_mesh_arrays(V, T) for V, T in meshes]
        k = len(arrs)
        if k == 0:
            return []
        lib = _lib.load()
        n = np.array([V.shape[0] for V, _ in arrs], np.int64)
        m = np.array([T.shape[0] for _, T in arrs], np.int64)
        Vp = (C.c_void_p * k)(*(V.ctypes.data for V, _ in arrs))
        Tp = (C.c_void_p * k)(*(T.ctypes.data for _, T in arrs))
        out = (C.c_void_p * k)()
        bad = C.c_int32(-1)
        err = C.create_string_buffer(512)
        rc = lib.mrb_mesh_build_many(k, _lib.ptr(n), Vp, _lib.ptr(m), Tp, out, C.byref(bad),
                                     err, 512)
        if rc != _lib.OK:
            raise ValueError(err.value.decode())
        meshes = []
        for (V, _), h in zip(arrs, out):
            obj = cls.__new__(cls)
            obj._adopt(h, V)
            meshes.append(obj)
        return meshes

    def _adopt(self, handle, V):
        lib = _lib.load()
        self._h = handle
        self._fin = weakref.finalize(self, lib.mrb_mesh_destroy, self._h)
        counts = np.zeros(6, dtype=np.int64)
        lib.mrb_mesh_counts(self._h, _lib.ptr(counts))
        n, m, ne = (int(c) for c in counts[:3])
        self._counts = counts
        tri = np.empty((m, 3), np.int64)
        edges = np.empty((ne, 2), np.int64)
        valence = np.empty(n, np.int64)
        boundary = np.empty(n, np.uint8)
        ring_ptr = np.empty(n + 1, np.int64)
        ring_idx = np.empty(2 * ne, np.int64)
        inc_ptr = np.empty(n + 1, np.int64)
        inc_idx = np.empty(3 * m, np.int64)
        lib.mrb_mesh_export_connectivity(
            self._h, *(_lib.ptr(a) for a in (tri, edges, valence, boundary, ring_ptr, ring_idx,
                                             inc_ptr, inc_idx)))
        self.vertices = V
        self.triangles = tri
        self.vertices.setflags(write=False)
        self.triangles.setflags(write=False)
        self.edges = edges
        self.valence = valence
        self.boundary = boundary.astype(bool)
        self._ring = (ring_ptr, ring_idx)
        self._inc = (inc_ptr, inc_idx)
        self._rings = self._incident = None
        self._geometry = None

    @property
    def rings(self):
        """Sorted one-ring neighbour ids per vertex (mesh.py:107-113), split lazily."""
        if self._rings is None:
            self._rings = np.split(self._ring[1], self._ring[0][1:-1])
        return self._rings

    @property
    def incident(self):
        """Ascending incident triangle ids per vertex (mesh.py:114-117), split lazily."""
        if self._incident is None:
            self._incident = np.split(self._inc[1], self._inc[0][1:-1])
        return self._incident

    @property
    def n_vertices(self):
        return self.vertices.shape[0]

    @property
    def n_triangles(self):
        return self.triangles.shape[0]

    @property
    def n_edges(self):
        return self.edges.shape[0]

    @property
    def geometry(self):
        if self._geometry is None:
            self._geometry = TriangleGeometry(self)
        return self._geometry

    def _csr(self, which, shape):
        nnz = int(self._counts[{_lib.CSR_LAPLACIAN: 3, _lib.CSR_GRAD_X: 4, _lib.CSR_GRAD_Y: 4,
                                _lib.CSR_VERTEX_AVG: 5}[which]])
        indptr = np.empty(shape[0] + 1, np.int64)
        indices = np.empty(nnz, np.int64)
        data = np.empty(nnz, np.float64)
        _lib.load().mrb_mesh_export_csr(self._h, which, _lib.ptr(indptr), _lib.ptr(indices),
                                        _lib.ptr(data))
        return indptr, indices, data

    def __repr__(self):
        return f"TriMesh({self.n_vertices} vertices, {self.n_triangles} triangles)"


_foreign = weakref.WeakKeyDictionary()


class DeferredMesh:
    """A mesh whose per-mesh setup runs on the GPU (no reference counterpart).

    ``DeferredMesh.create_many([(V, T), ...])`` (mrb_mesh_create_many) runs
    only the checks of TriMesh.__init__ that need no connectivity (mesh.py:61-
    86: finite coordinates, index range, repeated indices, degenerate area,
    with the reference's messages) and the CCW reorientation.  The first
    ``register_batch`` that runs the meshes on the fp32 cluster path builds
    their connectivity, geometry, fused operator and fast-path topology on the
    GPU, bit-identical to TriMesh's host build; every other use builds on the
    host first, and a mesh the reference would reject (non-manifold edge,
    valence < 2) raises the reference's ValueError there."""

    def __init__(self):
        raise TypeError("use DeferredMesh.create_many")

    @classmethod
    def create_many(cls, meshes):
        arrs = [_mesh_arrays(V, T) for V, T in meshes]
        k = len(arrs)
        if k == 0:
            return []
        lib = _lib.load()
        n = np.array([V.shape[0] for V, _ in arrs], np.int64)
        m = np.array([T.shape[0] for _, T in arrs], np.int64)
        Vp = (C.c_void_p * k)(*(V.ctypes.data for V, _ in arrs))
        Tp = (C.c_void_p * k)(*(T.ctypes.data for _, T in arrs))
        out = (C.c_void_p * k)()
        bad = C.c_int32(-1)
        err = C.create_string_buffer(512)
        rc = lib.mrb_mesh_create_many(k, _lib.ptr(n), Vp, _lib.ptr(m), Tp, out, C.byref(bad),
                                      err, 512)
        if rc != _lib.OK:
            raise ValueError(err.value.decode())
        res = []
        for (V, T), h in zip(arrs, out):
            obj = cls.__new__(cls)
            obj._h = h
            obj._fin = weakref.finalize(obj, lib.mrb_mesh_destroy, h)
            obj.vertices = V
            obj.vertices.setflags(write=False)
            obj._n, obj._m = V.shape[0], T.shape[0]
            res.append(obj)
        return res

    @property
    def n_vertices(self):
        return self._n

    @property
    def n_triangles(self):
        return self._m

    def device_check(self, cluster_size, nodes_per_thread):
        """Test hook (mrb_mesh_device_check): mismatch counts of the GPU build
        against the host build, all zero when they are bit-identical."""
        out = np.zeros(10, np.int64)
        lib = _lib.load()
        ctx = _lib.context()
        rc = lib.mrb_mesh_device_check(ctx, self._h, int(cluster_size), int(nodes_per_thread),
                                       _lib.ptr(out))
        _lib.check(rc, ctx, (ValueError, RuntimeError, RuntimeError))
        return out

    def __repr__(self):
        return f"DeferredMesh({self._n} vertices, {self._m} triangles)"


def as_mesh(mesh):
    """Accept this package's TriMesh or DeferredMesh, or any object with
    .vertices/.triangles (e.g. a reference meshreg.TriMesh); the native mesh
    is cached."""
    if isinstance(mesh, (TriMesh, DeferredMesh)):
        return mesh
    try:
        got = _foreign.get(mesh)
    except TypeError:
        got = None
    if got is None:
        got = TriMesh(mesh.vertices, mesh.triangles)
        try:
            _foreign[mesh] = got
        except TypeError:
            pass
    return got


def build_adjacency(vertices, triangles):
    return TriMesh(vertices, triangles)


class TriangleGeometry:
    """Areas, Eq. 9 coefficients and CSR operators (mesh.py:162-213)."""

    def __init__(self, mesh):
        mesh = as_mesh(mesh)
        n, m = mesh.n_vertices, mesh.n_triangles
        self.triangles = mesh.triangles
        self.areas = np.empty(m)
        self.coeffs = np.empty((m, 3, 2))
        self.vertex_areas = np.empty(n)
        _lib.load().mrb_mesh_export_geometry(mesh._h, _lib.ptr(self.areas),
                                             _lib.ptr(self.coeffs), _lib.ptr(self.vertex_areas))

        def csr(which, shape):
            p, i, d = mesh._csr(which, shape)
            return sparse.csr_array((d, i, p), shape=shape)

        self.grad_x_op = csr(_lib.CSR_GRAD_X, (m, n))
        self.grad_y_op = csr(_lib.CSR_GRAD_Y, (m, n))
        self.vertex_average_op = csr(_lib.CSR_VERTEX_AVG, (n, m))
        self._mesh = mesh


def build_laplacian(mesh):
    """Row-stochastic one-ring average matrix (mesh.py:254-265)."""
    mesh = as_mesh(mesh)
    n = mesh.n_vertices
    p, i, d = mesh._csr(_lib.CSR_LAPLACIAN, (n, n))
    return sparse.csr_array((d, i, p), shape=(n, n))


def _csr_arrays(L):
    L = sparse.csr_array(L)
    return (np.ascontiguousarray(L.indptr, dtype=np.int64),
            np.ascontiguousarray(L.indices, dtype=np.int64),
            np.ascontiguousarray(L.data, dtype=np.float64))


def smooth_displacement(L, u0, lam, iterations=1):
    """Explicit diffusion u <- (1 - lam) u + lam (L @ u) (mesh.py:268-282),
    on the GPU for any CSR matrix L."""
    if not 0.0 < lam < 1.0:
        raise ValueError(f"smoothing weight must be in (0, 1), got {lam}")
    if iterations < 0:
        raise ValueError("iterations must be >= 0")
    u = np.array(u0, dtype=np.float64, copy=True)
    if iterations == 0:
        return u
    if u.ndim not in (1, 2):
        raise ValueError(f"displacement must be (n,) or (n, k), got {u.shape}")
    # the device kernel smooths (n, 2) fields; any other column count (the
    # reference accepts whatever L @ u does) goes through in column pairs,
    # the columns being independent
    cols = u.reshape(u.shape[0], -1)
    p, i, d = _csr_arrays(L)
    if p.shape[0] != cols.shape[0] + 1:
        raise ValueError(f"dimension mismatch: L is {p.shape[0] - 1} x n, u has "
                         f"{cols.shape[0]} rows")
    lib = _lib.load()
    ctx = _lib.context()
    res = np.empty_like(cols)
    for c0 in range(0, cols.shape[1], 2):
        u2 = np.zeros((cols.shape[0], 2))
        k = min(2, cols.shape[1] - c0)
        u2[:, :k] = cols[:, c0:c0 + k]
        out = np.empty_like(u2)
        rc = lib.mrb_smooth_csr(ctx, u2.shape[0], _lib.ptr(p), _lib.ptr(i), _lib.ptr(d),
                                _lib.ptr(u2), float(lam), int(iterations), _lib.ptr(out))
        _lib.check(rc, ctx, (ValueError, RuntimeError, RuntimeError))
        res[:, c0:c0 + k] = out[:, :k]
    return res.reshape(u.shape)


def triangle_gradient(geom, tri, f):
    """Gradient (gx, gy) of the linear interpolant of ``f`` on one triangle
    (mesh.py:216-221).  A scalar host helper beside the path: the per-vertex
    field on the path is vertex_gradient_all."""
    f = np.asarray(f, dtype=np.float64)
    g = f[geom.triangles[tri]] @ geom.coeffs[tri]
    return float(g[0]), float(g[1])


def vertex_gradient(mesh, geom, f, i):
    """Area-weighted average of the incident-triangle gradients at vertex
    ``i`` (mesh.py:224-233), the reference's operation order."""
    tris = mesh.incident[i]
    if tris.size == 0:
        raise ValueError(f"vertex {i} has no incident triangle")
    f = np.asarray(f, dtype=np.float64)
    areas = geom.areas[tris]
    grads = np.einsum("tc,tcd->td", f[geom.triangles[tris]], geom.coeffs[tris])
    g = (areas[:, None] * grads).sum(axis=0) / areas.sum()
    return float(g[0]), float(g[1])


def umbrella(mesh, u, i):
    """Mean of the one-ring values minus the center value at vertex ``i``
    (mesh.py:244-251), per coordinate for (n,) or (n, d) ``u``."""
    u = np.asarray(u, dtype=np.float64)
    out = u[mesh.rings[i]].mean(axis=0) - u[i]
    return float(out) if np.ndim(out) == 0 else out


def vertex_gradient_all(mesh, geom, f):
    """Per-vertex gradients (n, 2) of a per-vertex scalar (mesh.py:236-241),
    via the fused one-ring operator on the GPU."""
    mesh = as_mesh(mesh)
    f = np.ascontiguousarray(f, dtype=np.float64)
    out = np.empty((mesh.n_vertices, 2))
    lib = _lib.load()
    ctx = _lib.context()
    rc = lib.mrb_vertex_gradient_all(ctx, mesh._h, _lib.ptr(f), _lib.ptr(out))
    _lib.check(rc, ctx, (ValueError, RuntimeError, RuntimeError))
    return out
