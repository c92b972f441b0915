"""ctypes binding of libmeshreg_b200.so (C ABI: include/meshreg_b200.h).

There is no CPU fallback: if the shared library is missing or no CUDA device
is usable, every compute call raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MESHREG_B200_LIB", os.path.join(_HERE, "libmeshreg_b200.so"))

OK, E_VALUE, E_DIVERGED, E_COVERAGE, E_CUDA, E_INTERNAL = range(6)
F32, F64 = 0, 1
PREC_F32, PREC_F64 = 0, 1
CSR_LAPLACIAN, CSR_GRAD_X, CSR_GRAD_Y, CSR_VERTEX_AVG = range(4)


class mrb_pixel_config(C.Structure):
    _fields_ = [("tau", C.c_double), ("lam", C.c_double), ("iterations", C.c_int32),
                ("smoothing_passes", C.c_int32), ("precision", C.c_int32),
                ("reserved", C.c_int32)]


class mrb_config(C.Structure):
    _fields_ = [("tau", C.c_double), ("lam", C.c_double), ("energy_tolerance", C.c_double),
                ("max_iterations", C.c_int32), ("smoothing_passes", C.c_int32),
                ("precision", C.c_int32), ("reserved", C.c_int32)]


_vp = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)

# name: (restype, argtypes)
_SIGS = {
    "mrb_version": (C.c_char_p, []),
    "mrb_ctx_create": (C.c_int, [_i32, C.POINTER(_vp)]),
    "mrb_ctx_destroy": (C.c_int, [_vp]),
    "mrb_last_error": (C.c_char_p, [_vp]),
    "mrb_ctx_stream": (_vp, [_vp]),
    "mrb_ctx_synchronize": (C.c_int, [_vp]),
    "mrb_mesh_build": (C.c_int, [_i64, _vp, _i64, _vp, C.POINTER(_vp), C.c_char_p, _i32]),
    "mrb_mesh_build_many": (C.c_int, [_i32, _vp, _vp, _vp, _vp, _vp, C.POINTER(_i32), C.c_char_p,
                                      _i32]),
    "mrb_mesh_create_many": (C.c_int, [_i32, _vp, _vp, _vp, _vp, _vp, C.POINTER(_i32), C.c_char_p,
                                       _i32]),
    "mrb_mesh_device_check": (C.c_int, [_vp, _vp, _i32, _i32, _vp]),
    "mrb_mesh_destroy": (C.c_int, [_vp]),
    "mrb_mesh_counts": (C.c_int, [_vp, _vp]),
    "mrb_mesh_export_connectivity": (C.c_int, [_vp] + [_vp] * 8),
    "mrb_mesh_export_csr": (C.c_int, [_vp, _i32, _vp, _vp, _vp]),
    "mrb_mesh_export_geometry": (C.c_int, [_vp, _vp, _vp, _vp]),
    "mrb_pixel_map": (C.c_int, [_vp, _vp, _i32, _i32, _vp, _vp]),
    "mrb_mesh_locate": (C.c_int, [_vp, _i64, _vp, _vp, _vp]),
    "mrb_register": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _vp, _vp, C.POINTER(mrb_config),
                               _vp, _vp, C.POINTER(_i32), _dp, _dp, _vp, _vp, _vp]),
    "mrb_batch_create": (C.c_int, [_vp, _i32, _vp, _i32, _i32, _i32, C.POINTER(mrb_config),
                                   C.POINTER(_vp)]),
    "mrb_batch_destroy": (C.c_int, [_vp]),
    "mrb_batch_set_images": (C.c_int, [_vp, _vp, _vp, _i32]),
    "mrb_batch_run": (C.c_int, [_vp]),
    "mrb_batch_get_results": (C.c_int, [_vp, _i32, _vp, _vp, _vp, _vp]),
    "mrb_batch_sync": (C.c_int, [_vp]),
    "mrb_batch_pair_status": (C.c_int, [_vp, _i32, C.POINTER(_i32), _dp, _dp, _vp, C.c_char_p,
                                        _i32]),
    "mrb_register_many": (C.c_int, [_vp, _i32, _vp, _i32, _i32, _i32, _vp, _vp,
                                    C.POINTER(mrb_config), _i32, _i32, _vp, _vp, _vp, _vp, _vp,
                                    _vp, _vp, _vp, _vp, C.c_char_p, _i32]),
    "mrb_batch_path": (_i32, [_vp]),
    "mrb_batch_loop_kernel": (C.c_char_p, [_vp]),
    "mrb_transfer_bytes": (C.c_int, [_vp, _vp, _i32]),
    "mrb_batch_phase_profile": (C.c_int, [_vp, _vp, _i64]),
    "mrb_batch_launches_per_run": (_i64, [_vp]),
    "mrb_batch_algorithmic_bytes": (C.c_double, [_vp]),
    "mrb_batch_kernel_bytes": (C.c_int, [_vp, _vp]),
    "mrb_batch_kernel_times": (C.c_int, [_vp, _vp]),
    "mrb_warp_sample": (C.c_int, [_vp, _i32, _i32, _i32, _vp, _i64, _vp, _vp, _vp]),
    "mrb_energy": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
    "mrb_energy_gradient": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
    "mrb_vertex_gradient_all": (C.c_int, [_vp, _vp, _vp, _vp]),
    "mrb_smooth_csr": (C.c_int, [_vp, _i64, _vp, _vp, _vp, _vp, C.c_double, _i32, _vp]),
    "mrb_step_csr": (C.c_int, [_vp, _i64, _vp, _vp, _vp, _vp, _vp, C.c_double, C.c_double, _i32,
                               _vp, _i32, _i32, _vp]),
    "mrb_densify": (C.c_int, [_vp, _vp, _i32, _i32, _vp, _vp, _vp]),
    "mrb_warp_image": (C.c_int, [_vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
    "mrb_msd": (C.c_int, [_vp, _i64, _vp, _vp, _vp]),
    # pixel-grid engine (baseline.py)
    "mrb_register_pixelwise": (C.c_int, [_vp, _i32, _i32, _i32, _vp, _vp,
                                         C.POINTER(mrb_pixel_config), _vp, _vp, _vp, _vp,
                                         C.POINTER(_i32), _dp, _dp]),
    "mrb_pixel_batch_create": (C.c_int, [_vp, _i32, _i32, _i32, _i32,
                                         C.POINTER(mrb_pixel_config), C.POINTER(_vp)]),
    "mrb_pixel_batch_destroy": (C.c_int, [_vp]),
    "mrb_pixel_batch_set_images": (C.c_int, [_vp, _vp, _vp, _i32]),
    "mrb_pixel_batch_run": (C.c_int, [_vp]),
    "mrb_pixel_batch_get_results": (C.c_int, [_vp, _i32, _vp, _vp, _vp]),
    "mrb_pixel_batch_sync": (C.c_int, [_vp]),
    "mrb_pixel_batch_pair_status": (C.c_int, [_vp, _i32, C.POINTER(_i32), _dp, _dp, _vp,
                                              C.c_char_p, _i32]),
    "mrb_pixel_batch_launches_per_run": (_i64, [_vp]),
    "mrb_pixel_batch_kernel_times": (C.c_int, [_vp, _vp]),
    "mrb_sample_gradient": (C.c_int, [_vp, _i32, _i32, _i32, _vp, _i64, _vp, _vp, _vp]),
    "mrb_grid_umbrella_smooth": (C.c_int, [_vp, _i32, _i32, _vp, C.c_double, _vp]),
    # content-adaptive mesher (meshgen.py, delaunay.py)
    "mrb_gradient_magnitude": (C.c_int, [_vp, _i32, _i32, _vp, _i32, _vp, _vp]),
    "mrb_canny_edges": (C.c_int, [_vp, _i32, _i32, _vp, _i32, _vp, C.c_double, C.c_double, _vp,
                                  _vp]),
    "mrb_canny_sample": (C.c_int, [_vp, _i32, _i32, _vp, _i32, _vp, C.c_double, C.c_double,
                                   C.c_double, _i64, _vp, _i64p]),
    "mrb_halftone_dots": (C.c_int, [_i32, _i32, _vp, _i64, _i32, _vp, _dp]),
    "mrb_floyd_steinberg": (C.c_int, [_i32, _i32, _vp, _i32, _vp]),
    "mrb_spacing_thin": (C.c_int, [_i64, _vp, _vp, C.c_double, _i64, _vp, _i64p]),
    "mrb_uniform_sample": (C.c_int, [_i32, _i32, _i64, _vp, _i64, _i64p, C.c_char_p, _i32]),
    "mrb_dedupe_points": (C.c_int, [_i64, _vp, C.c_double, _vp, _i64p, C.c_char_p, _i32]),
    "mrb_tris_create": (C.c_int, [_i64, _vp, _i64, _vp, C.POINTER(_vp), C.c_char_p, _i32]),
    "mrb_delaunay": (C.c_int, [_i64, _vp, C.POINTER(_vp), C.c_char_p, _i32]),
    "mrb_flip_edges": (C.c_int, [_vp, _i32, C.POINTER(_i32), C.c_char_p, _i32]),
    "mrb_smooth_mesh": (C.c_int, [_vp, _i32, _i32, _vp, _i32, _i32, C.c_char_p, _i32]),
    "mrb_tris_counts": (C.c_int, [_vp, _i64p, _i64p]),
    "mrb_tris_export": (C.c_int, [_vp, _vp, _vp]),
    "mrb_tris_destroy": (C.c_int, [_vp]),
    "mrb_delaunay_violations": (C.c_int, [_vp, _i64, _vp, _i64, _vp, C.c_double, _i64p]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def load():
    """Load the shared library (raises OSError when it is missing)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise OSError(
                        f"{LIB_PATH} not found: build it with paper_1411_2141_b200/csrc/build.sh "
                        "(or __graft_entry__.build()); there is no CPU fallback")
                lib = C.CDLL(LIB_PATH)
                for name, (res, args) in _SIGS.items():
                    fn = getattr(lib, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = lib
    return _lib


def ptr(a):
    """Raw data pointer of a contiguous numpy array (or None)."""
    if a is None:
        return None
    return a.ctypes.data


_ctx = {}


def context(device=None):
    """Per-process, per-device mrb_ctx (one CUDA stream each)."""
    lib = load()
    if device is None:
        device = int(os.environ.get("MESHREG_B200_DEVICE", "0"))
    c = _ctx.get(device)
    if c is None:
        h = C.c_void_p()
        rc = lib.mrb_ctx_create(device, C.byref(h))
        if rc != OK:
            raise RuntimeError(
                f"meshreg_b200: cannot create a CUDA context on device {device} (code {rc}); "
                "a B200 (sm_100a) GPU is required — there is no CPU fallback")
        c = h.value
        _ctx[device] = c
    return c


def last_error(ctx):
    return load().mrb_last_error(ctx).decode()


def check(rc, ctx, exc_types):
    """Map an MRB_* code to the reference exception type."""
    if rc == OK:
        return
    msg = last_error(ctx) if ctx else ""
    value_error, divergence_error, coverage_error = exc_types
    if rc == E_VALUE:
        raise value_error(msg)
    if rc == E_DIVERGED:
        raise divergence_error(msg)
    if rc == E_COVERAGE:
        raise coverage_error(msg)
    raise RuntimeError(f"meshreg_b200 CUDA failure: {msg or rc}")


def image_payload(data, precision="f64"):
    """(array, dtype code) to hand an image to the library.

    fp32 storage is used when it is exact (or when fp32 arithmetic was
    requested); otherwise the fp64 values are passed unchanged.
    """
    data = np.ascontiguousarray(data, dtype=np.float64)
    as32 = data.astype(np.float32)
    if precision == "f32" or np.array_equal(as32.astype(np.float64), data):
        return as32, F32
    return data, F64
