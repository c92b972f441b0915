"""Registration driver (mirror of reference pkg/src/meshreg/solver.py).

`register` runs the whole registration of solver.py:148-208 on the GPU in
one library call: the descent loop with the divergence / tolerance logic
evaluated on the device, then densify, warp and both MSDs.  `register_batch`
is the per-GPU pair queue.  The single-step functions
(warp_sample, energy, energy_gradient, step) are device-backed mirrors of
the reference functions of the same name.

Precision (keyword-only, not a reference parameter):
  "f64" (default) fp64 state and arithmetic; fp32 image storage when the
        inputs are fp32-exact (then the taps are exact).  Agrees with the
        reference to ~1e-12 relative.
  "f32" fp32 state and arithmetic with fp64 energy/MSD reductions — the fast
        mode; agrees to ~1e-6 relative (north_star tolerance 1e-4).
"""

from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import asdict, dataclass, field

import numpy as np

from . import _lib
from .densefield import MeshCoverageError
from .mesh import as_mesh

__all__ = [
    "SolverConfig",
    "RegistrationReport",
    "DivergenceError",
    "warp_sample",
    "energy",
    "energy_gradient",
    "step",
    "register",
    "register_batch",
]

DEFAULT_PRECISION = os.environ.get("MESHREG_B200_PRECISION", "f64")


class DivergenceError(RuntimeError):
    """The descent produced non-finite values or kept increasing the energy."""


RISE_THRESHOLD = 1e-4


def material_rise(previous, current):
    return current > previous * (1.0 + RISE_THRESHOLD) + 1e-12


@dataclass(frozen=True)
class SolverConfig:
    tau: float = 0.005
    lam: float = 0.8
    max_iterations: int = 100
    smoothing_passes: int = 1
    energy_tolerance: float = 1e-6

    def __post_init__(self):
        if self.tau <= 0:
            raise ValueError(f"tau must be positive, got {self.tau}")
        if not 0.0 < self.lam < 1.0:
            raise ValueError(f"lambda must be in (0, 1), got {self.lam}")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be >= 1")
        if self.smoothing_passes < 0:
            raise ValueError("smoothing_passes must be >= 0")
        if self.energy_tolerance < 0:
            raise ValueError("energy_tolerance must be >= 0")

    def to_dict(self):
        return asdict(self)


@dataclass
class RegistrationReport:
    iterations_run: int
    energy_trace: list
    msd_before: float
    msd_after: float
    wall_time: float
    config: dict = field(default_factory=dict)

    def to_dict(self):
        return {
            "iterations_run": self.iterations_run,
            "energy_trace": [float(e) for e in self.energy_trace],
            "msd_before": float(self.msd_before),
            "msd_after": float(self.msd_after),
            "wall_time": float(self.wall_time),
            "config": dict(self.config),
        }


def _errs():
    return (ValueError, DivergenceError, MeshCoverageError)


def _cfg_struct(cfg, precision):
    if precision not in ("f32", "f64"):
        raise ValueError(f"precision must be 'f32' or 'f64', got {precision!r}")
    return _lib.mrb_config(float(cfg.tau), float(cfg.lam), float(cfg.energy_tolerance),
                           int(cfg.max_iterations), int(cfg.smoothing_passes),
                           _lib.PREC_F32 if precision == "f32" else _lib.PREC_F64, 0)


def _pair_payload(reference, template, precision):
    """Both images in one dtype: fp32 when exact (or requested), else fp64."""
    r, dr = _lib.image_payload(reference.data, precision)
    t, dt = _lib.image_payload(template.data, precision)
    if dr != dt:
        r = np.ascontiguousarray(reference.data, dtype=np.float64)
        t = np.ascontiguousarray(template.data, dtype=np.float64)
        dr = _lib.F64
    return r, t, dr


def warp_sample(template, vertices, u):
    """Bicubic template samples at V + u (solver.py:91-97)."""
    from .image import sample_points
    vertices = np.asarray(vertices, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    if u.shape != vertices.shape:
        raise ValueError(f"displacement shape {u.shape} != vertices {vertices.shape}")
    return sample_points(template, vertices, u)


def energy(reference, template, mesh, u):
    """0.5 * sum over nodes of (Te - Re)^2 at V + u (solver.py:100-106)."""
    mesh = as_mesh(mesh)
    u = np.ascontiguousarray(u, dtype=np.float64)
    if u.shape != mesh.vertices.shape:
        raise ValueError(f"displacement shape {u.shape} != vertices {mesh.vertices.shape}")
    r, t, dt = _pair_payload(reference, template, "f64")
    out = np.zeros(1)
    lib = _lib.load()
    ctx = _lib.context()
    rc = lib.mrb_energy(ctx, mesh._h, template.width, template.height, dt, _lib.ptr(r),
                        _lib.ptr(t), _lib.ptr(u), _lib.ptr(out))
    _lib.check(rc, ctx, _errs())
    return float(out[0])


def energy_gradient(reference, template, mesh, u):
    """Residual times the mesh-operator template gradient (solver.py:109-121)."""
    mesh = as_mesh(mesh)
    u = np.ascontiguousarray(u, dtype=np.float64)
    if u.shape != mesh.vertices.shape:
        raise ValueError(f"displacement shape {u.shape} != vertices {mesh.vertices.shape}")
    r, t, dt = _pair_payload(reference, template, "f64")
    out = np.empty((mesh.n_vertices, 2))
    lib = _lib.load()
    ctx = _lib.context()
    rc = lib.mrb_energy_gradient(ctx, mesh._h, template.width, template.height, dt, _lib.ptr(r),
                                 _lib.ptr(t), _lib.ptr(u), _lib.ptr(out))
    _lib.check(rc, ctx, _errs())
    return out


def step(u, grad, cfg, laplacian, vertices=None, domain=None):
    """Descent update, diffusion smoothing, optional domain clamp
    (solver.py:124-145), on the GPU."""
    from scipy import sparse
    grad = np.ascontiguousarray(grad, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    n = u.shape[0]
    L = sparse.csr_array(laplacian)
    p = np.ascontiguousarray(L.indptr, dtype=np.int64)
    i = np.ascontiguousarray(L.indices, dtype=np.int64)
    d = np.ascontiguousarray(L.data, dtype=np.float64)
    clamp = vertices is not None and domain is not None
    V = np.ascontiguousarray(vertices, dtype=np.float64) if clamp else None
    w, h = (int(domain[0]), int(domain[1])) if clamp else (0, 0)
    out = np.empty((n, 2))
    lib = _lib.load()
    ctx = _lib.context()
    rc = lib.mrb_step_csr(ctx, n, _lib.ptr(p), _lib.ptr(i), _lib.ptr(d), _lib.ptr(u),
                          _lib.ptr(grad), float(cfg.tau), float(cfg.lam),
                          int(cfg.smoothing_passes), _lib.ptr(V), w, h, _lib.ptr(out))
    _lib.check(rc, ctx, _errs())
    return out


def register(reference, template, mesh, cfg=None, *, precision=None, return_dense=False):
    """Run the descent loop from u = 0 and the dense final pass
    (solver.py:148-208).  Returns (u (n, 2) float64, RegistrationReport);
    with return_dense=True also (ux, uy, warped) float64 planes."""
    cfg = cfg or SolverConfig()
    precision = precision or DEFAULT_PRECISION
    if reference.shape != template.shape:
        raise ValueError(f"image sizes differ: {reference.shape} vs {template.shape}")
    mesh = as_mesh(mesh)
    r, t, dt = _pair_payload(reference, template, precision)
    W, H = template.width, template.height
    c = _cfg_struct(cfg, precision)
    u = np.empty((mesh.n_vertices, 2))
    trace = np.empty(cfg.max_iterations)
    iters = C.c_int32(0)
    mb, ma = C.c_double(0), C.c_double(0)
    ux = np.empty((H, W))
    uy = np.empty((H, W))
    warped = np.empty((H, W))
    lib = _lib.load()
    ctx = _lib.context()
    t0 = time.perf_counter()
    rc = lib.mrb_register(ctx, mesh._h, W, H, dt, _lib.ptr(r), _lib.ptr(t), C.byref(c),
                          _lib.ptr(u), _lib.ptr(trace), C.byref(iters), C.byref(mb),
                          C.byref(ma), _lib.ptr(ux), _lib.ptr(uy), _lib.ptr(warped))
    wall = time.perf_counter() - t0
    _lib.check(rc, ctx, _errs())
    report = RegistrationReport(
        iterations_run=int(iters.value),
        energy_trace=[float(e) for e in trace[:iters.value]],
        msd_before=float(mb.value),
        msd_after=float(ma.value),
        wall_time=wall,
        config=cfg.to_dict(),
    )
    if return_dense:
        return u, report, (ux, uy, warped)
    return u, report


def register_batch(references, templates, meshes, cfg=None, *, precision=None,
                   return_dense=False, chunk_pairs=0):
    """Register many independent equally-sized pairs (the per-GPU pair queue)
    through the pipelined native entry point mrb_register_many: chunks of
    pairs overlap their host setup, transfers and kernels.  Returns a list
    with, per pair, (u, report) — plus (ux, uy, warped) when return_dense —
    or the exception the reference would have raised for that pair."""
    cfg = cfg or SolverConfig()
    precision = precision or DEFAULT_PRECISION
    P = len(references)
    if not (P == len(templates) == len(meshes)) or P == 0:
        raise ValueError("references, templates and meshes must be equally long and non-empty")
    shape = templates[0].shape
    for a, b in zip(references, templates):
        if a.shape != b.shape:
            raise ValueError(f"image sizes differ: {a.shape} vs {b.shape}")
        if b.shape != shape:
            raise ValueError("all pairs of a batch must share one image size")
    meshes = [as_mesh(m) for m in meshes]
    pays = [_pair_payload(a, b, precision) for a, b in zip(references, templates)]
    dt = _lib.F64 if any(p[2] == _lib.F64 for p in pays) else _lib.F32
    npdt = np.float64 if dt == _lib.F64 else np.float32
    re = np.ascontiguousarray(np.stack([p[0] for p in pays]).astype(npdt))
    te = np.ascontiguousarray(np.stack([p[1] for p in pays]).astype(npdt))
    H, W = shape
    lib = _lib.load()
    ctx = _lib.context()
    c = _cfg_struct(cfg, precision)
    arr = (C.c_void_p * P)(*[m._h for m in meshes])
    n_tot = sum(m.n_vertices for m in meshes)
    u_all = np.empty((n_tot, 2))
    dense = [np.empty((P, H, W)) for _ in range(3)] if return_dense else [None] * 3
    iters = np.zeros(P, np.int32)
    mb = np.zeros(P)
    ma = np.zeros(P)
    trace = np.zeros((P, cfg.max_iterations))
    codes = np.full(P, -1, np.int32)  # -1: never written (cannot read as OK)
    msg_len = 512
    msgs = C.create_string_buffer(P * msg_len)
    rc = lib.mrb_register_many(ctx, P, arr, W, H, dt, _lib.ptr(re), _lib.ptr(te), C.byref(c),
                          int(chunk_pairs), _lib.F64, _lib.ptr(u_all), *(_lib.ptr(d) for d in dense),
                          _lib.ptr(iters), _lib.ptr(mb), _lib.ptr(ma), _lib.ptr(trace),
                          _lib.ptr(codes), msgs, msg_len)
    if rc == _lib.E_COVERAGE and P > 1:
        # a mesh that does not cover the image stops the whole call (the
        # pixel maps are built for the batch at once); the reference raises
        # MeshCoverageError for that pair only, so run the pairs one by one
        out = []
        for a, b, m in zip(references, templates, meshes):
            try:
                out.append(register(a, b, m, cfg, precision=precision, return_dense=return_dense))
            except (ValueError, DivergenceError, MeshCoverageError) as e:
                out.append(e)
        return out
    if rc in (_lib.E_CUDA, _lib.E_INTERNAL) or (codes < 0).any():
        # a device / library failure is not a per-pair outcome: raise it
        _lib.check(rc if rc != _lib.OK else _lib.E_INTERNAL, ctx,
                   (ValueError, DivergenceError, MeshCoverageError))
    out = []
    off = 0
    for p, m in enumerate(meshes):
        u = u_all[off:off + m.n_vertices].copy()
        off += m.n_vertices
        code = int(codes[p])
        if code != _lib.OK:
            text = msgs.raw[p * msg_len:(p + 1) * msg_len].split(b"\0", 1)[0].decode()
            exc = {_lib.E_DIVERGED: DivergenceError, _lib.E_VALUE: ValueError,
                   _lib.E_COVERAGE: MeshCoverageError}.get(code, RuntimeError)
            out.append(exc(text or _lib.last_error(ctx)))
            continue
        k = int(iters[p])
        rep = RegistrationReport(k, [float(e) for e in trace[p, :k]], float(mb[p]), float(ma[p]),
                                 0.0, cfg.to_dict())
        out.append((u, rep, tuple(d[p] for d in dense)) if return_dense else (u, rep))
    return out
