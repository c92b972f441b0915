"""Content-adaptive triangular meshing of an image (mirror of reference
pkg/src/meshreg/meshgen.py).

Same pipeline, names, arguments and results as the reference's
``generate_mesh`` (meshgen.py:365-396), computed by libmeshreg_b200:

* image-space stages on the GPU (csrc/mesher.cuh): the Gaussian filter,
  gradient magnitude and Canny edge detector (Gaussian, np.gradient,
  np.hypot, 4-direction thinning, hysteresis by union-find);
* sequential stages in native C++ (csrc/mesher_host.cpp): spacing-grid
  thinning, Floyd-Steinberg halftoning, the uniform grid, point
  de-duplication, Bowyer-Watson, CVT/ODT relaxation and edge flips.

Every stage reproduces the reference's floating-point operation order, so
``generate_mesh`` returns the reference's mesh bit for bit.  The host
Python here only holds what the reference computes with numpy's own
generators: the Gaussian taps (np.exp, as scipy builds them) and the seeded
``default_rng`` draws of the halftone sampler.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .delaunay import _delaunay_tris, _Tris, dedupe_points, delaunay_violations
from .meshio import load_mesh, load_mesh_json, save_mesh, save_mesh_json
from .mesh import TriMesh

__all__ = [
    "NodeBudget",
    "MeshGenConfig",
    "canny_sample",
    "halftone_sample",
    "uniform_sample",
    "smooth_mesh",
    "generate_mesh",
    "save_mesh",
    "load_mesh",
    "save_mesh_json",
    "load_mesh_json",
    "quality_stats",
    "gradient_magnitude",
    "canny_edges",
]

_ERR = 512


@dataclass(frozen=True)
class NodeBudget:
    """How many mesh nodes to place and how to split them across samplers
    (meshgen.py:41-57)."""

    target_nodes: int
    canny_fraction: float = 0.4
    halftone_fraction: float = 0.4
    uniform_fraction: float = 0.2

    def __post_init__(self):
        total = self.canny_fraction + self.halftone_fraction + self.uniform_fraction
        if abs(total - 1.0) > 1e-9:
            raise ValueError(f"sampler fractions sum to {total}, expected 1")
        if min(self.canny_fraction, self.halftone_fraction, self.uniform_fraction) < 0:
            raise ValueError("sampler fractions must be non-negative")
        if self.target_nodes < 4:
            raise ValueError(f"target_nodes must be >= 4, got {self.target_nodes}")


@dataclass(frozen=True)
class MeshGenConfig:
    """Mesher parameters (meshgen.py:60-77)."""

    canny_low: float = 8.0
    canny_high: float = 24.0
    canny_sigma: float = 1.4
    min_node_spacing: float = 3.0
    cvt_iterations: int = 3
    odt_iterations: int = 2
    flip_passes: int = 16
    seed: int = 0

    def __post_init__(self):
        if not self.canny_low < self.canny_high:
            raise ValueError("canny_low must be below canny_high")
        if self.min_node_spacing < 1.0:
            raise ValueError("min_node_spacing must be >= 1 pixel")
        if min(self.cvt_iterations, self.odt_iterations, self.flip_passes) < 0:
            raise ValueError("iteration counts must be >= 0")


def _gaussian_taps(sigma, truncate=4.0):
    """The 2r+1 taps scipy.ndimage.gaussian_filter correlates with
    (_gaussian_kernel1d with order 0, radius int(truncate*sigma + 0.5))."""
    sd = float(sigma)
    radius = int(truncate * sd + 0.5)
    sigma2 = sigma * sigma
    x = np.arange(-radius, radius + 1)
    phi = np.exp(-0.5 / sigma2 * x ** 2)
    phi = phi / phi.sum()
    return radius, np.ascontiguousarray(phi[::-1], dtype=np.float64)


def _image_array(data):
    arr = np.ascontiguousarray(np.asarray(data, dtype=np.float64))
    if arr.ndim != 2:
        raise ValueError(f"image must be 2-D, got shape {arr.shape}")
    return arr


def gradient_magnitude(data, sigma):
    """hypot(np.gradient(gaussian_filter(data, sigma, mode="nearest")))
    (meshgen.py:99-102), on the GPU."""
    arr = _image_array(data)
    h, w = arr.shape
    r, taps = _gaussian_taps(sigma)
    out = np.empty((h, w), np.float64)
    ctx = _lib.context()
    rc = _lib.load().mrb_gradient_magnitude(ctx, w, h, _lib.ptr(arr), r, _lib.ptr(taps),
                                            _lib.ptr(out))
    _lib.check(rc, ctx, (ValueError, RuntimeError, RuntimeError))
    return out


def canny_edges(data, sigma, low, high):
    """Boolean Canny edge mask (meshgen.py:105-132), on the GPU."""
    arr = _image_array(data)
    h, w = arr.shape
    r, taps = _gaussian_taps(sigma)
    edges = np.empty((h, w), np.uint8)
    ctx = _lib.context()
    rc = _lib.load().mrb_canny_edges(ctx, w, h, _lib.ptr(arr), r, _lib.ptr(taps), float(low),
                                     float(high), _lib.ptr(edges), None)
    _lib.check(rc, ctx, (ValueError, RuntimeError, RuntimeError))
    return edges.astype(bool)


def canny_sample(img, cfg, budget):
    """Up to ``budget`` points on Canny edge pixels, strongest edges first,
    strictly separated by ``cfg.min_node_spacing`` (meshgen.py:135-154)."""
    budget = int(budget)
    if budget <= 0:
        return np.empty((0, 2))
    arr = _image_array(img.data)
    h, w = arr.shape
    r, taps = _gaussian_taps(cfg.canny_sigma)
    out = np.empty((budget, 2), np.float64)
    cnt = C.c_int64()
    ctx = _lib.context()
    rc = _lib.load().mrb_canny_sample(ctx, w, h, _lib.ptr(arr), r, _lib.ptr(taps),
                                      float(cfg.canny_low), float(cfg.canny_high),
                                      float(cfg.min_node_spacing), budget, _lib.ptr(out),
                                      C.byref(cnt))
    _lib.check(rc, ctx, (ValueError, RuntimeError, RuntimeError))
    if cnt.value == 0:
        return np.empty((0, 2))
    return out[: cnt.value].copy()


def _floyd_steinberg(density, serpentine_start=0):
    """Binary dot mask from serpentine Floyd-Steinberg error diffusion of a
    non-negative density map (meshgen.py:157-185), in native code."""
    d = np.ascontiguousarray(np.asarray(density, dtype=np.float64))
    h, w = d.shape
    dots = np.empty((h, w), np.uint8)
    rc = _lib.load().mrb_floyd_steinberg(w, h, _lib.ptr(d), int(serpentine_start), _lib.ptr(dots))
    if rc != _lib.OK:
        raise ValueError("density must be a non-empty 2-D array")
    return dots.astype(bool)


def _thin(xy, order, spacing, budget):
    xy = np.ascontiguousarray(xy, dtype=np.float64)
    order = None if order is None else np.ascontiguousarray(order, dtype=np.int64)
    out = np.empty((max(int(budget), 1), 2), np.float64)
    cnt = C.c_int64()
    rc = _lib.load().mrb_spacing_thin(xy.shape[0], _lib.ptr(xy), _lib.ptr(order), float(spacing),
                                      int(budget), _lib.ptr(out), C.byref(cnt))
    if rc != _lib.OK:
        raise ValueError("spacing thinning failed")
    return out[: cnt.value].copy()


def halftone_sample(img, budget, spacing, seed=0):
    """Texture-following points from Floyd-Steinberg halftoning of the
    gradient-density map, thinned in a seeded random order
    (meshgen.py:188-216).  The gradient magnitude runs on the GPU, the error
    diffusion and thinning in native code; the seeded draws use numpy's
    default_rng exactly as the reference does."""
    budget = int(budget)
    if budget <= 0:
        return np.empty((0, 2))
    return _halftone_from_mag(gradient_magnitude(img.data, 1.0), budget, spacing, seed)


def _halftone_from_mag(mag, budget, spacing, seed):
    """Host half of halftone_sample: pairwise mass, error diffusion, the
    seeded permutation and spacing thinning (meshgen.py:196-216)."""
    mag = np.ascontiguousarray(mag, dtype=np.float64)
    h, w = mag.shape
    rng = np.random.default_rng(seed)
    serpentine = int(rng.integers(2))
    dots = np.empty((h, w), np.uint8)
    total = C.c_double()
    rc = _lib.load().mrb_halftone_dots(w, h, _lib.ptr(mag), int(budget), serpentine,
                                       _lib.ptr(dots), C.byref(total))
    if rc != _lib.OK:
        raise ValueError("halftoning failed")
    if total.value <= 1e-12:
        return np.empty((0, 2))
    ys, xs = np.nonzero(dots)
    if ys.size == 0:
        return np.empty((0, 2))
    order = rng.permutation(ys.size)
    pts = _thin(np.stack([xs, ys], axis=1).astype(np.float64), order, spacing, budget)
    return pts if len(pts) else np.empty((0, 2))


def uniform_sample(width, height, budget):
    """Regular grid of about ``budget`` points including the corners, topped
    up with staggered cell centres (meshgen.py:219-248)."""
    budget = int(budget)
    cap = (math.isqrt(max(budget, 0)) + 2) ** 2 + 8
    out = np.empty((cap, 2), np.float64)
    cnt = C.c_int64()
    err = C.create_string_buffer(_ERR)
    rc = _lib.load().mrb_uniform_sample(int(width), int(height), budget, _lib.ptr(out), cap,
                                        C.byref(cnt), err, _ERR)
    if rc != _lib.OK:
        raise ValueError(err.value.decode())
    return out[: cnt.value].copy()


def _smooth_tris(tris, img, cfg):
    if cfg.cvt_iterations == 0 and cfg.odt_iterations == 0:
        return
    mag = gradient_magnitude(img.data, 1.5)
    h, w = mag.shape
    err = C.create_string_buffer(_ERR)
    rc = _lib.load().mrb_smooth_mesh(tris.h, w, h, _lib.ptr(mag), int(cfg.cvt_iterations),
                                     int(cfg.odt_iterations), err, _ERR)
    if rc != _lib.OK:
        raise ValueError(err.value.decode())


def smooth_mesh(mesh, img, cfg):
    """CVT then ODT relaxation of the node positions toward density-weighted
    one-ring targets; boundary nodes slide along the image edge, corners stay,
    inverting moves are rejected (meshgen.py:269-327)."""
    if cfg.cvt_iterations == 0 and cfg.odt_iterations == 0:
        return mesh
    t = _Tris.from_mesh(mesh)
    _smooth_tris(t, img, cfg)
    return t.to_mesh()


def generate_mesh(img, budget, cfg=None):
    """Full meshing pipeline for an image (meshgen.py:365-396): Canny,
    halftone and uniform samplers against the node budget, de-duplication,
    forced corners, Delaunay, CVT/ODT smoothing and edge flips."""
    cfg = cfg or MeshGenConfig()
    w, h = img.width, img.height
    corners = np.array([[0.0, 0.0], [w - 1.0, 0.0], [0.0, h - 1.0], [w - 1.0, h - 1.0]])
    target = budget.target_nodes

    n_canny = int(round(target * budget.canny_fraction))
    pts_canny = canny_sample(img, cfg, n_canny)
    n_half = int(round(target * budget.halftone_fraction)) + (n_canny - len(pts_canny))
    pts_half = halftone_sample(img, n_half, cfg.min_node_spacing, seed=cfg.seed)

    partial = dedupe_points(np.vstack([corners, pts_canny, pts_half]))
    n_uniform = target - len(partial)
    if n_uniform >= 4:
        pts_uniform = uniform_sample(w, h, n_uniform)
        points = dedupe_points(np.vstack([partial, pts_uniform]))
    else:
        points = partial

    tris = _delaunay_tris(points)
    _smooth_tris(tris, img, cfg)
    tris.flip(cfg.flip_passes)
    return tris.to_mesh()


def quality_stats(mesh, audit_margin=1e-9):
    """Summary quality numbers of the command-line mesh report
    (meshgen.py:455-481); the Delaunay audit runs on the GPU."""
    V = mesh.vertices
    T = mesh.triangles
    a = V[T[:, 0]]
    b = V[T[:, 1]]
    c = V[T[:, 2]]
    areas = 0.5 * ((b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1])
                   - (c[:, 0] - a[:, 0]) * (b[:, 1] - a[:, 1]))
    angles = []
    for p, q, r in ((a, b, c), (b, c, a), (c, a, b)):
        u = q - p
        v = r - p
        cosang = (u * v).sum(axis=1) / (np.linalg.norm(u, axis=1) * np.linalg.norm(v, axis=1))
        angles.append(np.degrees(np.arccos(np.clip(cosang, -1.0, 1.0))))
    return {
        "n_nodes": int(mesh.n_vertices),
        "n_triangles": int(mesh.n_triangles),
        "n_edges": int(mesh.n_edges),
        "min_area": float(areas.min()),
        "min_angle": float(np.min(angles)),
        "delaunay_violations": int(delaunay_violations(V, T, margin=audit_margin)),
    }
