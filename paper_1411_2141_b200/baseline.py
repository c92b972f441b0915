"""Pixel-grid registration engine (mirror of reference pkg/src/meshreg/baseline.py).

One displacement unknown per pixel: residual x analytic-gradient descent,
`smoothing_passes` 4-neighbour umbrella passes, clamp — `iterations` times,
then the dense warp and MSD.  The whole loop runs on the GPU as one fused,
temporally blocked sm_100a kernel per iteration (csrc/pixel.cuh) behind the
C ABI entry points mrb_register_pixelwise / mrb_pixel_batch_*; there is no
CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _lib
from .densefield import DenseField
from .solver import DEFAULT_PRECISION, DivergenceError, RegistrationReport, _pair_payload

__all__ = ["PixelField", "register_pixelwise", "register_pixelwise_batch",
           "grid_umbrella_smooth"]

# baseline.py:22-24: a per-pixel field shares DenseField's layout and checks
PixelField = DenseField


def _errs():
    return (ValueError, DivergenceError, RuntimeError)


def grid_umbrella_smooth(plane, lam):
    """One 4-neighbour blend toward the mean of the existing neighbours
    (baseline.py:27-43), fp64 on the GPU."""
    plane = np.ascontiguousarray(plane, dtype=np.float64)
    if plane.ndim != 2:
        raise ValueError(f"plane must be 2-D, got shape {plane.shape}")
    h, w = plane.shape
    out = np.empty_like(plane)
    lib = _lib.load()
    ctx = _lib.context()
    rc = lib.mrb_grid_umbrella_smooth(ctx, w, h, _lib.ptr(plane), float(lam), _lib.ptr(out))
    _lib.check(rc, ctx, _errs())
    return out


def _pixel_cfg(tau, lam, iterations, smoothing_passes, precision):
    if precision not in ("f32", "f64"):
        raise ValueError(f"precision must be 'f32' or 'f64', got {precision!r}")
    return _lib.mrb_pixel_config(float(tau), float(lam), int(iterations), int(smoothing_passes),
                                 _lib.PREC_F32 if precision == "f32" else _lib.PREC_F64, 0)


def _config_dict(tau, lam, iterations, smoothing_passes):
    return {"tau": tau, "lam": lam, "max_iterations": iterations,
            "smoothing_passes": smoothing_passes}


def register_pixelwise(reference, template, tau=0.005, lam=0.8, iterations=100,
                       smoothing_passes=3, *, precision=None):
    """Dense registration returning (PixelField, RegistrationReport)
    (baseline.py:46-118).  Raises ValueError / DivergenceError with the
    reference's messages."""
    precision = precision or DEFAULT_PRECISION
    if reference.shape != template.shape:
        raise ValueError(f"image sizes differ: {reference.shape} vs {template.shape}")
    c = _pixel_cfg(tau, lam, iterations, smoothing_passes, precision)
    r, t, dt = _pair_payload(reference, template, precision)
    H, W = template.shape
    ux = np.empty((H, W))
    uy = np.empty((H, W))
    trace = np.empty(max(int(iterations), 1))
    iters = C.c_int32(0)
    mb, ma = C.c_double(0), C.c_double(0)
    lib = _lib.load()
    ctx = _lib.context()
    t0 = time.perf_counter()
    rc = lib.mrb_register_pixelwise(ctx, W, H, dt, _lib.ptr(r), _lib.ptr(t), C.byref(c),
                                    _lib.ptr(ux), _lib.ptr(uy), None, _lib.ptr(trace),
                                    C.byref(iters), C.byref(mb), C.byref(ma))
    wall = time.perf_counter() - t0
    _lib.check(rc, ctx, _errs())
    report = RegistrationReport(
        iterations_run=int(iters.value),
        energy_trace=[float(e) for e in trace[:iters.value]],
        msd_before=float(mb.value),
        msd_after=float(ma.value),
        wall_time=wall,
        config=_config_dict(tau, lam, iterations, smoothing_passes),
    )
    return PixelField(ux, uy), report


class PixelBatch:
    """A resident batch of equally sized pairs for the pixel engine
    (mrb_pixel_batch_*): images may be host numpy stacks or device pointers;
    the iteration loop runs as one CUDA graph from the second run on."""

    def __init__(self, n_pairs, width, height, tau=0.005, lam=0.8, iterations=100,
                 smoothing_passes=3, *, precision="f32", img_dtype=_lib.F32):
        self._lib = _lib.load()
        self.ctx = _lib.context()
        self.n_pairs, self.width, self.height = int(n_pairs), int(width), int(height)
        self.iterations = int(iterations)
        self.real = np.float64 if precision == "f64" else np.float32
        c = _pixel_cfg(tau, lam, iterations, smoothing_passes, precision)
        h = C.c_void_p()
        rc = self._lib.mrb_pixel_batch_create(self.ctx, self.n_pairs, self.width, self.height,
                                              img_dtype, C.byref(c), C.byref(h))
        _lib.check(rc, self.ctx, _errs())
        self._h = h.value

    def set_images(self, reference, template, on_device=False):
        ref = reference if on_device else _lib.ptr(reference)
        tmp = template if on_device else _lib.ptr(template)
        _lib.check(self._lib.mrb_pixel_batch_set_images(self._h, ref, tmp, int(on_device)),
                   self.ctx, _errs())

    def run(self):
        _lib.check(self._lib.mrb_pixel_batch_run(self._h), self.ctx, _errs())

    def get_results(self, ux=None, uy=None, warped=None, out_dtype=_lib.F64):
        _lib.check(self._lib.mrb_pixel_batch_get_results(self._h, out_dtype, _lib.ptr(ux),
                                                         _lib.ptr(uy), _lib.ptr(warped)),
                   self.ctx, _errs())

    def sync(self):
        """Wait for the run; returns per pair a RegistrationReport or the
        exception the reference would have raised for it."""
        self._lib.mrb_pixel_batch_sync(self._h)
        out = []
        msg = C.create_string_buffer(512)
        for p in range(self.n_pairs):
            it = C.c_int32(0)
            mb, ma = C.c_double(0), C.c_double(0)
            tr = np.empty(self.iterations)
            rc = self._lib.mrb_pixel_batch_pair_status(self._h, p, C.byref(it), C.byref(mb),
                                                       C.byref(ma), _lib.ptr(tr), msg, 512)
            if rc == _lib.OK:
                out.append(RegistrationReport(int(it.value), [float(e) for e in tr[:it.value]],
                                              float(mb.value), float(ma.value), 0.0, {}))
            elif rc == _lib.E_DIVERGED:
                out.append(DivergenceError(msg.value.decode()))
            else:
                out.append(ValueError(msg.value.decode()))
        return out

    def launches_per_run(self):
        return int(self._lib.mrb_pixel_batch_launches_per_run(self._h))

    def kernel_times(self):
        """(mean ms of the fused iteration kernel, ms of one whole run)."""
        out = np.zeros(2)
        _lib.check(self._lib.mrb_pixel_batch_kernel_times(self._h, _lib.ptr(out)), self.ctx,
                   _errs())
        return float(out[0]), float(out[1])

    def close(self):
        if self._h:
            self._lib.mrb_pixel_batch_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def register_pixelwise_batch(references, templates, tau=0.005, lam=0.8, iterations=100,
                             smoothing_passes=3, *, precision=None):
    """register_pixelwise over many equally sized pairs in one device batch.
    Returns per pair (PixelField, RegistrationReport) or the exception the
    reference would have raised for that pair."""
    precision = precision or DEFAULT_PRECISION
    P = len(references)
    if P == 0 or P != len(templates):
        raise ValueError("references and templates must be equally long and non-empty")
    shape = templates[0].shape
    for a, b in zip(references, templates):
        if a.shape != b.shape:
            raise ValueError(f"image sizes differ: {a.shape} vs {b.shape}")
        if b.shape != shape:
            raise ValueError("all pairs of a batch must share one image size")
    pays = [_pair_payload(a, b, precision) for a, b in zip(references, templates)]
    dt = _lib.F64 if any(p[2] == _lib.F64 for p in pays) else _lib.F32
    npdt = np.float64 if dt == _lib.F64 else np.float32
    re = np.ascontiguousarray(np.stack([p[0] for p in pays]).astype(npdt))
    te = np.ascontiguousarray(np.stack([p[1] for p in pays]).astype(npdt))
    H, W = shape
    b = PixelBatch(P, W, H, tau, lam, iterations, smoothing_passes, precision=precision,
                   img_dtype=dt)
    try:
        b.set_images(re, te)
        b.run()
        ux = np.empty((P, H, W))
        uy = np.empty((P, H, W))
        b.get_results(ux, uy)
        reps = b.sync()
    finally:
        b.close()
    cfg = _config_dict(tau, lam, iterations, smoothing_passes)
    out = []
    for p, rep in enumerate(reps):
        if isinstance(rep, Exception):
            out.append(rep)
        else:
            rep = RegistrationReport(rep.iterations_run, rep.energy_trace, rep.msd_before,
                                     rep.msd_after, rep.wall_time, cfg)
            out.append((PixelField(ux[p], uy[p]), rep))
    return out
