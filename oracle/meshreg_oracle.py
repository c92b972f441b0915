"""CPU ORACLE — test infrastructure only, never the product path.

A plain numpy/scipy restatement of the reference `meshreg` registration hot
path (reference root: arxiv/paper_1411_2141, package pkg/src/meshreg).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline legs
may import this module, and only as the checker / the CPU timing arm.  The
B200 package (``paper_1411_2141_b200``) never imports it.

Parity pinning: this restatement is checked against golden vectors produced by
running the reference itself in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``; test
``tests/test_oracle_golden.py``).  The reference ships no golden files of its
own; its known-answer tests are mirrored against the B200
path in ``tests/test_gpu_parity.py`` (sampling, energy, step, warp KATs).

Third-party arithmetic the reference relies on (not vendored there, not pinned:
reference pkg/pyproject.toml:10-14): numpy einsum / fancy indexing / dot and
scipy.sparse CSR mat-vec.  The same libraries are used here, with the same
reduction orders where they matter for exactness (CSR assembly, vertex areas).

Everything is float64 / int64 as in the reference.
"""

from __future__ import annotations

import numpy as np
from scipy import sparse

DEGENERATE_AREA = 1e-9          # mesh.py:28
BARY_EPS = 1e-9                 # densefield.py:31
RISE_THRESHOLD = 1e-4           # solver.py:40


class OracleDivergence(RuntimeError):
    """Mirrors solver.DivergenceError (solver.py:33-34)."""


class OracleCoverage(RuntimeError):
    """Mirrors densefield.MeshCoverageError (densefield.py:58-59)."""


# --------------------------------------------------------------------------
# image sampling (image.py)
# --------------------------------------------------------------------------

def pad_ring(img):
    """One quadratically extrapolated ring, columns first then rows.

    image.py:62-71 (x then y) and _extend image.py:134-148 (3a0-3a1+a2 for
    n>=3, 2a0-a1 for n==2, constant for n==1).
    """
    def one_axis(a, axis):
        a = np.moveaxis(a, axis, 0)
        n = a.shape[0]
        if n >= 3:
            first = 3.0 * a[0] - 3.0 * a[1] + a[2]
            last = 3.0 * a[-1] - 3.0 * a[-2] + a[-3]
        elif n == 2:
            first = 2.0 * a[0] - a[1]
            last = 2.0 * a[-1] - a[-2]
        else:
            first = last = a[0]
        return np.moveaxis(np.concatenate([first[None], a, last[None]]), 0, axis)

    return one_axis(one_axis(np.asarray(img, np.float64), 1), 0)


def cr_weights(t):
    """Catmull-Rom tap weights, image.py:151-164."""
    t2 = t * t
    t3 = t2 * t
    return np.stack([0.5 * (-t3 + 2.0 * t2 - t),
                     0.5 * (3.0 * t3 - 5.0 * t2 + 2.0),
                     0.5 * (-3.0 * t3 + 4.0 * t2 + t),
                     0.5 * (t3 - t2)], axis=-1)


def sample(img, x, y, ext=None):
    """Bicubic Catmull-Rom value at (x, y); image.py:73-84 with _locate
    (105-116: clamp, base cell clipped to size-2) and _gather (118-123)."""
    img = np.asarray(img, np.float64)
    h, w = img.shape
    if ext is None:
        ext = pad_ring(img)
    x = np.atleast_1d(np.asarray(x, np.float64))
    y = np.atleast_1d(np.asarray(y, np.float64))
    x, y = np.broadcast_arrays(x, y)
    xc = np.clip(x, 0.0, w - 1.0)
    yc = np.clip(y, 0.0, h - 1.0)
    cx = np.minimum(np.floor(xc), max(w - 2, 0)).astype(np.int64)
    cy = np.minimum(np.floor(yc), max(h - 2, 0)).astype(np.int64)
    k = np.arange(4)
    taps = ext[cy[..., None, None] + k[:, None], cx[..., None, None] + k[None, :]]
    return np.einsum("...j,...i,...ji->...", cr_weights(yc - cy), cr_weights(xc - cx), taps)


def msd(a, b):
    """image.py:181-186."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape:
        raise ValueError(f"dimension mismatch: {a.shape} vs {b.shape}")
    d = a - b
    return float(np.mean(d * d))


# --------------------------------------------------------------------------
# mesh (mesh.py)
# --------------------------------------------------------------------------

def _area2(V, T):
    """Twice the signed area, mesh.py:153-159 (same operation order)."""
    p, q, r = V[T[:, 0]], V[T[:, 1]], V[T[:, 2]]
    return (q[:, 0] - p[:, 0]) * (r[:, 1] - p[:, 1]) - (r[:, 0] - p[:, 0]) * (q[:, 1] - p[:, 1])


def _csr_from_triplets(rows, cols, vals, shape):
    """Canonical CSR (row-major, columns ascending) of a duplicate-free COO
    triplet set: what scipy's csr_array((data,(row,col))) yields."""
    order = np.lexsort((cols, rows))
    indptr = np.zeros(shape[0] + 1, np.int64)
    np.add.at(indptr, rows + 1, 1)
    return np.cumsum(indptr), cols[order].astype(np.int64), vals[order].astype(np.float64)


class Mesh:
    """Connectivity + geometry of a static triangulation.

    Construction follows TriMesh.__init__ (mesh.py:58-89): validation, CCW
    reorientation by swapping corners 1 and 2, then _build_connectivity
    (mesh.py:91-123) and TriangleGeometry (mesh.py:173-213).
    """

    def __init__(self, vertices, triangles):
        V = np.ascontiguousarray(np.asarray(vertices, np.float64))
        T = np.ascontiguousarray(np.asarray(triangles, np.int64))
        if V.ndim != 2 or V.shape[1] != 2:
            raise ValueError(f"vertices must be (n, 2), got {V.shape}")
        if T.ndim != 2 or T.shape[1] != 3 or T.shape[0] < 1:
            raise ValueError(f"triangles must be (m, 3) with m >= 1, got {T.shape}")
        if not np.all(np.isfinite(V)):
            raise ValueError("vertex coordinates must be finite")
        n = V.shape[0]
        if T.min() < 0 or T.max() >= n:
            raise ValueError("triangle index out of range")
        if np.any((T[:, 0] == T[:, 1]) | (T[:, 1] == T[:, 2]) | (T[:, 0] == T[:, 2])):
            raise ValueError("triangle with repeated vertex index")
        a2 = _area2(V, T)
        if np.any(np.abs(a2) <= 2.0 * DEGENERATE_AREA):
            k = int(np.argmin(np.abs(a2)))
            raise ValueError(f"degenerate triangle {k} (area {abs(a2[k]) / 2.0:g})")
        neg = a2 < 0
        if neg.any():
            T = T.copy()
            T[neg] = T[neg][:, [0, 2, 1]]
        self.V, self.T = V, T
        self.n, self.m = n, T.shape[0]
        self._connectivity()
        self._geometry()

    # mesh.py:91-123
    def _connectivity(self):
        T, n = self.T, self.n
        e = np.sort(np.concatenate([T[:, [0, 1]], T[:, [1, 2]], T[:, [2, 0]]]), axis=1)
        edges, counts = np.unique(e, axis=0, return_counts=True)
        if np.any(counts > 2):
            raise ValueError("non-manifold edge shared by more than two triangles")
        # rings: sorted neighbour ids == sorted union of both edge directions
        src = np.concatenate([edges[:, 0], edges[:, 1]])
        dst = np.concatenate([edges[:, 1], edges[:, 0]])
        order = np.lexsort((dst, src))
        valence = np.bincount(src, minlength=n).astype(np.int64)
        ring_ptr = np.concatenate([[0], np.cumsum(valence)]).astype(np.int64)
        self.ring_ptr, self.ring_idx = ring_ptr, dst[order].astype(np.int64)
        # incident triangles, ascending id
        vt = T.ravel()
        tt = np.repeat(np.arange(self.m), 3)
        order = np.lexsort((tt, vt))
        inc_cnt = np.bincount(vt, minlength=n)
        self.inc_ptr = np.concatenate([[0], np.cumsum(inc_cnt)]).astype(np.int64)
        self.inc_idx = tt[order].astype(np.int64)
        boundary = np.zeros(n, bool)
        b = edges[counts == 1]
        boundary[b[:, 0]] = True
        boundary[b[:, 1]] = True
        self.edges, self.valence, self.boundary = edges, valence, boundary
        if np.any(valence < 2):
            k = int(np.argmin(valence))
            raise ValueError(f"vertex {k} has valence {valence[k]} (< 2)")

    # mesh.py:173-213
    def _geometry(self):
        V, T, n, m = self.V, self.T, self.n, self.m
        a, b, c = V[T[:, 0]], V[T[:, 1]], V[T[:, 2]]
        self.areas = 0.5 * _area2(V, T)
        if np.any(self.areas <= DEGENERATE_AREA):
            raise ValueError("zero-area triangle in geometry")
        e_ab, e_bc, e_ac = b - a, c - b, c - a

        def dot(p, q):
            return p[:, 0] * q[:, 0] + p[:, 1] * q[:, 1]

        # Eq. 9 corner coefficients (mesh.py:193-195), identical op order
        ci = dot(e_ab, e_bc)[:, None] * (c - a) + dot(e_ac, -e_bc)[:, None] * (b - a)
        cj = dot(-e_ab, e_ac)[:, None] * (c - b) + dot(e_bc, -e_ac)[:, None] * (a - b)
        ck = dot(-e_bc, -e_ab)[:, None] * (a - c) + dot(-e_ac, e_ab)[:, None] * (b - c)
        scale = 1.0 / (4.0 * self.areas ** 2)
        self.coeffs = np.stack([ci, cj, ck], axis=1) * scale[:, None, None]
        rows = np.repeat(np.arange(m), 3)
        cols = T.ravel()
        self.gx = _csr_from_triplets(rows, cols, self.coeffs[:, :, 0].ravel(), (m, n))
        self.gy = _csr_from_triplets(rows, cols, self.coeffs[:, :, 1].ravel(), (m, n))
        va = np.zeros(n)
        np.add.at(va, cols, np.repeat(self.areas, 3))   # ascending-triangle order
        self.vertex_areas = va
        wts = np.repeat(self.areas, 3) / va[cols]
        self.avg = _csr_from_triplets(cols, rows, wts, (n, m))
        # Laplacian, mesh.py:254-265
        self.lap = (self.ring_ptr.copy(), self.ring_idx.copy(),
                    np.repeat(1.0 / self.valence, self.valence))
        self._ops = None

    def ops(self):
        if self._ops is None:
            mk = lambda csr, shp: sparse.csr_array((csr[2], csr[1], csr[0]), shape=shp)
            self._ops = (mk(self.gx, (self.m, self.n)), mk(self.gy, (self.m, self.n)),
                         mk(self.avg, (self.n, self.m)), mk(self.lap, (self.n, self.n)))
        return self._ops

    def ring(self, i):
        return self.ring_idx[self.ring_ptr[i]:self.ring_ptr[i + 1]]

    def incident(self, i):
        return self.inc_idx[self.inc_ptr[i]:self.inc_ptr[i + 1]]


def vertex_gradient_all(mesh, f):
    """mesh.py:236-241: avg @ (Gx @ f), avg @ (Gy @ f)."""
    gx, gy, avg, _ = mesh.ops()
    f = np.asarray(f, np.float64)
    return np.stack([avg @ (gx @ f), avg @ (gy @ f)], axis=1)


def smooth_displacement(mesh, u0, lam, passes=1):
    """mesh.py:268-282."""
    if not 0.0 < lam < 1.0:
        raise ValueError(f"smoothing weight must be in (0, 1), got {lam}")
    if passes < 0:
        raise ValueError("iterations must be >= 0")
    L = mesh.ops()[3]
    u = np.array(u0, dtype=np.float64, copy=True)
    for _ in range(passes):
        u = (1.0 - lam) * u + lam * (L @ u)
    return u


# --------------------------------------------------------------------------
# solver (solver.py)
# --------------------------------------------------------------------------

def warp_sample(img, V, u, ext=None):
    """solver.py:91-97."""
    V = np.asarray(V, np.float64)
    u = np.asarray(u, np.float64)
    if u.shape != V.shape:
        raise ValueError(f"displacement shape {u.shape} != vertices {V.shape}")
    return sample(img, V[:, 0] + u[:, 0], V[:, 1] + u[:, 1], ext)


def energy(re, te, mesh, u):
    """solver.py:100-106."""
    r = warp_sample(te, mesh.V, u) - warp_sample(re, mesh.V, u)
    return 0.5 * float(np.dot(r, r))


def energy_gradient(re, te, mesh, u):
    """solver.py:109-121."""
    s_te = warp_sample(te, mesh.V, u)
    s_re = warp_sample(re, mesh.V, u)
    return (s_te - s_re)[:, None] * vertex_gradient_all(mesh, s_te)


def step(mesh, u, grad, tau, lam, passes, V=None, domain=None):
    """solver.py:124-145."""
    grad = np.asarray(grad, np.float64)
    if not np.all(np.isfinite(grad)):
        raise OracleDivergence("non-finite gradient; reduce the step size tau")
    u0 = np.asarray(u, np.float64) - tau * grad
    u1 = smooth_displacement(mesh, u0, lam, passes) if passes > 0 else u0
    if V is not None and domain is not None:
        w, h = domain
        u1 = np.clip(u1, -V, np.array([w - 1.0, h - 1.0]) - V)
    return u1


def register(re, te, mesh, tau=0.005, lam=0.8, max_iterations=100,
             smoothing_passes=1, energy_tolerance=1e-6, want_dense=True, vec_pixel_map=False):
    """The descent loop of solver.py:148-208 followed by densify/warp/MSD.

    Returns (u, info) with info = dict(iterations_run, energy_trace,
    msd_before, msd_after, ux, uy, warped).
    """
    re = np.asarray(re, np.float64)
    te = np.asarray(te, np.float64)
    if re.shape != te.shape:
        raise ValueError(f"image sizes differ: {re.shape} vs {te.shape}")
    h, w = te.shape
    V = mesh.V
    ext_te, ext_re = pad_ring(te), pad_ring(re)
    u = np.zeros((mesh.n, 2))
    trace = []
    rises = 0
    for _ in range(max_iterations):
        s_te = warp_sample(te, V, u, ext_te)
        r = s_te - warp_sample(re, V, u, ext_re)
        e = 0.5 * float(np.dot(r, r))
        if not np.isfinite(e):
            raise OracleDivergence("energy became non-finite; reduce tau")
        if trace and e > trace[-1] * (1.0 + RISE_THRESHOLD) + 1e-12:
            rises += 1
            if rises >= 10:
                raise OracleDivergence(
                    f"energy increased for {rises} consecutive iterations "
                    f"(last values {trace[-3:] + [e]}); reduce tau")
        elif trace and e <= trace[-1]:
            rises = 0
        trace.append(e)
        grad = r[:, None] * vertex_gradient_all(mesh, s_te)
        u = step(mesh, u, grad, tau, lam, smoothing_passes, V, (w, h))
        if len(trace) >= 6:
            base = trace[-6]
            if abs(trace[-1] - base) <= energy_tolerance * max(abs(base), 1e-12):
                break
    info = dict(iterations_run=len(trace), energy_trace=trace, msd_before=msd(te, re))
    if want_dense:
        pmap = pixel_map_vec(mesh, w, h) if vec_pixel_map else None
        ux, uy = densify(mesh, u, w, h, pmap)
        warped = warp_image(te, ux, uy)
        info.update(ux=ux, uy=uy, warped=warped, msd_after=msd(warped, re))
    return u, info


# --------------------------------------------------------------------------
# dense field (densefield.py)
# --------------------------------------------------------------------------

def _bary(V, tri, px, py):
    """densefield.py:99-107, same operation order."""
    a, b, c = V[tri[:, 0]], V[tri[:, 1]], V[tri[:, 2]]
    d = (b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (c[:, 0] - a[:, 0]) * (b[:, 1] - a[:, 1])
    w1 = ((b[:, 0] - px) * (c[:, 1] - py) - (c[:, 0] - px) * (b[:, 1] - py)) / d
    w2 = ((c[:, 0] - px) * (a[:, 1] - py) - (a[:, 0] - px) * (c[:, 1] - py)) / d
    return np.stack([w1, w2, 1.0 - w1 - w2], axis=1)


def _locator(mesh):
    """PointLocator bins, densefield.py:69-95."""
    V, T = mesh.V, mesh.T
    lo, hi = V.min(axis=0), V.max(axis=0)
    span = np.maximum(hi - lo, 1e-9)
    cell = max(2.0, float(np.sqrt(2.0 * span[0] * span[1] / max(T.shape[0], 1))))
    nx = int(np.ceil(span[0] / cell)) + 1
    ny = int(np.ceil(span[1] / cell)) + 1

    def cell_of(x, y):
        bx = int((min(max(x, lo[0]), hi[0]) - lo[0]) / cell)
        by = int((min(max(y, lo[1]), hi[1]) - lo[1]) / cell)
        return min(bx, nx - 1), min(by, ny - 1)

    bins = [[] for _ in range(nx * ny)]
    cmin, cmax = V[T].min(axis=1), V[T].max(axis=1)
    for t in range(T.shape[0]):
        x0, y0 = cell_of(cmin[t, 0], cmin[t, 1])
        x1, y1 = cell_of(cmax[t, 0], cmax[t, 1])
        for by in range(y0, y1 + 1):
            for bx in range(x0, x1 + 1):
                bins[by * nx + bx].append(t)
    return cell_of, nx, [np.array(b, np.int64) for b in bins]


def _locate(mesh, loc, px, py):
    """densefield.py:110-127."""
    cell_of, nx, bins = loc
    bx, by = cell_of(px, py)
    for cand in (bins[by * nx + bx], np.arange(mesh.m)):
        if cand.size == 0:
            continue
        w = _bary(mesh.V, mesh.T[cand], px, py)
        ok = np.nonzero(np.min(w, axis=1) >= -BARY_EPS)[0]
        if ok.size:
            return int(cand[ok[0]]), w[ok[0]]
    raise OracleCoverage(f"point ({px}, {py}) not covered by any triangle")


def pixel_map(mesh, width, height):
    """Pixel -> (triangle, barycentric weights), densefield.py:148-182:
    ascending triangle order, bbox [ceil(min-eps), floor(max+eps)], assign
    only unassigned pixels (lowest index wins), binned-locate fallback."""
    V, T = mesh.V, mesh.T
    tri_of = np.full((height, width), -1, np.int64)
    wts = np.zeros((height, width, 3))
    cmin, cmax = V[T].min(axis=1), V[T].max(axis=1)
    for t in range(mesh.m):
        x0 = max(int(np.ceil(cmin[t, 0] - BARY_EPS)), 0)
        x1 = min(int(np.floor(cmax[t, 0] + BARY_EPS)), width - 1)
        y0 = max(int(np.ceil(cmin[t, 1] - BARY_EPS)), 0)
        y1 = min(int(np.floor(cmax[t, 1] + BARY_EPS)), height - 1)
        if x1 < x0 or y1 < y0:
            continue
        yy, xx = np.mgrid[y0:y1 + 1, x0:x1 + 1]
        yy, xx = yy.ravel(), xx.ravel()
        w = _bary(V, np.repeat(T[t:t + 1], xx.size, axis=0), xx.astype(np.float64),
                  yy.astype(np.float64))
        sel = (np.min(w, axis=1) >= -BARY_EPS) & (tri_of[yy, xx] < 0)
        if sel.any():
            tri_of[yy[sel], xx[sel]] = t
            wts[yy[sel], xx[sel]] = w[sel]
    miss = np.argwhere(tri_of < 0)
    if miss.size:
        loc = _locator(mesh)
        for y, x in miss:
            t, w = _locate(mesh, loc, float(x), float(y))
            tri_of[y, x] = t
            wts[y, x] = w
    return tri_of, wts


def pixel_map_vec(mesh, width, height, chunk=1 << 16):
    """The same pixel map as pixel_map(), vectorised over triangles for
    C5-size meshes (1M triangles; the per-triangle loop takes minutes).

    Triangles are visited in ascending chunks; inside a chunk every
    (triangle, bbox pixel) candidate is tested with the same fp64 _bary
    operations, the lowest containing triangle per pixel is kept, and only
    pixels still unassigned take it — which is the reference's "ascending id,
    assign if unassigned" rule (densefield.py:155-174).  Checked equal to
    pixel_map() on the goldens (tests/test_oracle_golden.py)."""
    V, T = mesh.V, mesh.T
    tri_of = np.full(height * width, -1, np.int64)
    wts = np.zeros((height * width, 3))
    cmin, cmax = V[T].min(axis=1), V[T].max(axis=1)
    x0 = np.maximum(np.ceil(cmin[:, 0] - BARY_EPS).astype(np.int64), 0)
    x1 = np.minimum(np.floor(cmax[:, 0] + BARY_EPS).astype(np.int64), width - 1)
    y0 = np.maximum(np.ceil(cmin[:, 1] - BARY_EPS).astype(np.int64), 0)
    y1 = np.minimum(np.floor(cmax[:, 1] + BARY_EPS).astype(np.int64), height - 1)
    nx = np.maximum(x1 - x0 + 1, 0)
    ny = np.maximum(y1 - y0 + 1, 0)
    for c0 in range(0, mesh.m, chunk):
        tids = np.arange(c0, min(c0 + chunk, mesh.m))
        cnt = nx[tids] * ny[tids]
        tt = np.repeat(tids, cnt)
        if tt.size == 0:
            continue
        k = np.arange(tt.size) - np.repeat(np.cumsum(cnt) - cnt, cnt)
        xx = x0[tt] + k % nx[tt]
        yy = y0[tt] + k // nx[tt]
        w = _bary(V, T[tt], xx.astype(np.float64), yy.astype(np.float64))
        ok = np.min(w, axis=1) >= -BARY_EPS
        tt, w, pix = tt[ok], w[ok], (yy * width + xx)[ok]
        order = np.lexsort((tt, pix))  # per pixel, lowest triangle first
        pix, tt, w = pix[order], tt[order], w[order]
        first = np.ones(pix.size, bool)
        first[1:] = pix[1:] != pix[:-1]
        pix, tt, w = pix[first], tt[first], w[first]
        free = tri_of[pix] < 0
        tri_of[pix[free]] = tt[free]
        wts[pix[free]] = w[free]
    tri_of = tri_of.reshape(height, width)
    wts = wts.reshape(height, width, 3)
    miss = np.argwhere(tri_of < 0)
    if miss.size:
        loc = _locator(mesh)
        for y, x in miss:
            t, w = _locate(mesh, loc, float(x), float(y))
            tri_of[y, x] = t
            wts[y, x] = w
    return tri_of, wts


def densify(mesh, u, width=None, height=None, pmap=None):
    """densefield.py:130-187."""
    u = np.asarray(u, np.float64)
    if u.shape != (mesh.n, 2):
        raise ValueError(f"displacement shape {u.shape} != ({mesh.n}, 2)")
    if width is None:
        width = int(round(mesh.V[:, 0].max())) + 1
    if height is None:
        height = int(round(mesh.V[:, 1].max())) + 1
    tri_of, wts = pmap if pmap is not None else pixel_map(mesh, width, height)
    nodes = mesh.T[tri_of]
    return (wts * u[nodes, 0]).sum(axis=2), (wts * u[nodes, 1]).sum(axis=2)


def warp_image(te, ux, uy):
    """densefield.py:190-199: out(p) = Te(p + u(p))."""
    te = np.asarray(te, np.float64)
    if ux.shape != te.shape:
        raise ValueError(f"field {ux.shape} does not match image {te.shape}")
    h, w = te.shape
    ext = pad_ring(te)
    gx = np.arange(w, dtype=np.float64)
    out = np.empty((h, w))
    step = max(1, (1 << 20) // max(w, 1))  # row blocks: bounded (n,4,4) tap arrays
    for y0 in range(0, h, step):
        y1 = min(h, y0 + step)
        gy = np.arange(y0, y1, dtype=np.float64)[:, None]
        out[y0:y1] = sample(te, gx[None, :] + ux[y0:y1], gy + uy[y0:y1], ext)
    return out


# --------------------------------------------------------------------------
# pixel-grid engine (baseline.py) — SURVEY.md §8(f) row 1
# --------------------------------------------------------------------------

def cr_dweights(t):
    """Derivative Catmull-Rom weights, image.py:167-178."""
    t2 = t * t
    return np.stack([0.5 * (-3.0 * t2 + 4.0 * t - 1.0),
                     0.5 * (9.0 * t2 - 10.0 * t),
                     0.5 * (-9.0 * t2 + 8.0 * t + 1.0),
                     0.5 * (3.0 * t2 - 2.0 * t)], axis=-1)


def sample_gradient(img, x, y, ext=None):
    """Analytic (d/dx, d/dy) of the Catmull-Rom interpolant, image.py:86-103."""
    img = np.asarray(img, np.float64)
    h, w = img.shape
    if ext is None:
        ext = pad_ring(img)
    x = np.atleast_1d(np.asarray(x, np.float64))
    y = np.atleast_1d(np.asarray(y, np.float64))
    x, y = np.broadcast_arrays(x, y)
    xc = np.clip(x, 0.0, w - 1.0)
    yc = np.clip(y, 0.0, h - 1.0)
    cx = np.minimum(np.floor(xc), max(w - 2, 0)).astype(np.int64)
    cy = np.minimum(np.floor(yc), max(h - 2, 0)).astype(np.int64)
    k = np.arange(4)
    taps = ext[cy[..., None, None] + k[:, None], cx[..., None, None] + k[None, :]]
    tx, ty = xc - cx, yc - cy
    wx, wy = cr_weights(tx), cr_weights(ty)
    gx = np.einsum("...j,...i,...ji->...", wy, cr_dweights(tx), taps)
    gy = np.einsum("...j,...i,...ji->...", cr_dweights(ty), wx, taps)
    return gx, gy


def grid_umbrella_smooth(plane, lam):
    """4-neighbour mean blend with edge-aware counts, baseline.py:27-43."""
    total = np.zeros_like(plane)
    count = np.zeros_like(plane)
    total[1:, :] += plane[:-1, :]
    count[1:, :] += 1
    total[:-1, :] += plane[1:, :]
    count[:-1, :] += 1
    total[:, 1:] += plane[:, :-1]
    count[:, 1:] += 1
    total[:, :-1] += plane[:, 1:]
    count[:, :-1] += 1
    return (1.0 - lam) * plane + lam * total / count


def register_pixelwise(re, te, tau=0.005, lam=0.8, iterations=100, smoothing_passes=3):
    """Dense per-pixel engine of baseline.py:46-118.  Returns
    (ux, uy, info) with info = iterations_run, energy_trace, msd_before,
    msd_after, warped."""
    re = np.asarray(re, np.float64)
    te = np.asarray(te, np.float64)
    if re.shape != te.shape:
        raise ValueError(f"image sizes differ: {re.shape} vs {te.shape}")
    if tau <= 0:
        raise ValueError(f"tau must be positive, got {tau}")
    if not 0.0 <= lam < 1.0:
        raise ValueError(f"lambda must be in [0, 1), got {lam}")
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    h, w = re.shape
    gx0, gy0 = np.meshgrid(np.arange(w, dtype=np.float64), np.arange(h, dtype=np.float64))
    ext_te, ext_re = pad_ring(te), pad_ring(re)
    ux = np.zeros((h, w))
    uy = np.zeros((h, w))
    trace = []
    rises = 0
    for _ in range(iterations):
        px, py = gx0 + ux, gy0 + uy
        r = sample(te, px, py, ext_te) - sample(re, px, py, ext_re)
        e = 0.5 * float(np.sum(r * r))
        if not np.isfinite(e):
            raise OracleDivergence("energy became non-finite; reduce tau")
        if trace and e > trace[-1] * (1.0 + RISE_THRESHOLD) + 1e-12:
            rises += 1
            if rises >= 10:
                raise OracleDivergence(
                    f"energy increased for {rises} consecutive iterations; reduce tau")
        elif trace and e <= trace[-1]:
            rises = 0
        trace.append(e)
        dx, dy = sample_gradient(te, px, py, ext_te)
        ux = ux - tau * r * dx
        uy = uy - tau * r * dy
        if lam > 0.0:
            for _ in range(smoothing_passes):
                ux = grid_umbrella_smooth(ux, lam)
                uy = grid_umbrella_smooth(uy, lam)
        np.clip(ux, -gx0, (w - 1.0) - gx0, out=ux)
        np.clip(uy, -gy0, (h - 1.0) - gy0, out=uy)
    warped = warp_image(te, ux, uy)
    info = dict(iterations_run=len(trace), energy_trace=trace, msd_before=msd(te, re),
                msd_after=msd(warped, re), warped=warped)
    return ux, uy, info
