"""TEST INFRASTRUCTURE — a numpy fp32 emulation of the descent loop.

It states, operation for operation, what the fp32 fast path computes
(fp32 taps / Catmull-Rom weights / residual / fused gradient operator /
smoothing, fp64 positions and energy), on top of the CPU oracle
(oracle/meshreg_oracle.py).  The tests use it to separate the error that
fp32 arithmetic itself carries against the fp64 reference (what the
north_star tolerance has to absorb) from any extra error a kernel adds.
Never imported by the package.
"""
from __future__ import annotations

import numpy as np
from scipy import sparse

import meshreg_oracle as O

f32 = np.float32


def cr_weights32(t):
    """cr_weights<float> (kernels.cuh), image.py:151-164 in fp32."""
    t = t.astype(f32)
    t2 = t * t
    t3 = t2 * t
    h = f32(0.5)
    return np.stack([h * ((-t3 + f32(2) * t2) - t),
                     h * ((f32(3) * t3 - f32(5) * t2) + f32(2)),
                     h * ((f32(-3) * t3 + f32(4) * t2) + t),
                     h * (t3 - t2)], axis=-1)


def sample2_32(ext2, W, H, x, y):
    """(Te, Re) at fp64 positions from the fp32 padded pair (H+2, W+2, 2)."""
    xc = np.clip(x, 0.0, W - 1.0)
    yc = np.clip(y, 0.0, H - 1.0)
    cx = np.minimum(np.floor(xc), W - 2).astype(np.int64)
    cy = np.minimum(np.floor(yc), H - 2).astype(np.int64)
    wx = cr_weights32(xc - cx)
    wy = cr_weights32(yc - cy)
    k = np.arange(4)
    taps = ext2[cy[:, None, None] + k[:, None], cx[:, None, None] + k[None, :]]  # (n,4,4,2)
    acc = np.zeros((x.shape[0], 2), f32)
    for j in range(4):
        row = wx[:, 0, None] * taps[:, j, 0]
        for i in range(1, 4):
            row = wx[:, i, None] * taps[:, j, i] + row
        acc = wy[:, j, None] * row + acc
    return acc[:, 0], acc[:, 1]


class Emu32:
    """Mesh constants of the fp32 path: fused G = avg @ grad in fp64 rounded
    to fp32 (mesh_host.cpp), L = 1/valence in fp32."""

    def __init__(self, mesh: O.Mesh):
        gx, gy, avg, lap = mesh.ops()
        self.Gx = sparse.csr_array(avg @ gx, dtype=np.float64).astype(f32)
        self.Gy = sparse.csr_array(avg @ gy, dtype=np.float64).astype(f32)
        self.L = sparse.csr_array(lap, dtype=np.float64).astype(f32)
        self.V = mesh.V
        self.mesh = mesh


def register32(re, te, mesh, tau=0.005, lam=0.8, max_iterations=100, smoothing_passes=1):
    """fp32 loop; returns (u (fp64 copy of the fp32 state), energy trace)."""
    em = Emu32(mesh)
    h, w = te.shape
    ext2 = np.stack([O.pad_ring(te), O.pad_ring(re)], axis=-1).astype(f32)
    V = em.V
    lo = (-V).astype(f32)
    hi = (np.array([w - 1.0, h - 1.0]) - V).astype(f32)
    u = np.zeros((mesh.n, 2), f32)
    tau32, lam32 = f32(tau), f32(lam)
    om = f32(1) - lam32
    trace = []
    for _ in range(max_iterations):
        s_te, s_re = sample2_32(ext2, w, h, V[:, 0] + u[:, 0].astype(np.float64),
                                V[:, 1] + u[:, 1].astype(np.float64))
        r = s_te - s_re
        trace.append(0.5 * float(np.dot(r.astype(np.float64), r.astype(np.float64))))
        g = np.stack([em.Gx @ s_te, em.Gy @ s_te], axis=1).astype(f32)
        u0 = u - tau32 * (r[:, None] * g)
        for _ in range(smoothing_passes):
            u0 = om * u0 + lam32 * (em.L @ u0).astype(f32)
        u = np.minimum(np.maximum(u0, lo), hi).astype(f32)
    return u.astype(np.float64), trace
