// Pixel-grid engine (reference baseline.py:46-118):
// one displacement per pixel, descent along residual x analytic spline
// gradient of the template (image.py:86-103), `passes` 4-neighbour umbrella
// smoothing passes (baseline.py:27-43), clamp, `iterations` times.
//
// B200 design: one fused kernel per iteration with temporal blocking.  A CTA
// owns a TX x TY tile; it samples Te, Re and dTe/dx, dTe/dy (from the same 16
// taps) for the tile plus a halo of `passes` pixels, applies the descent,
// runs every smoothing pass in shared memory (the valid region shrinks by one
// pixel per pass), clamps and writes its tile of u to the other buffer of a
// double-buffered pair of planes.  HBM traffic per pixel and iteration: read
// u, write u (the image taps hit L1/L2).  The fp64 energy partial of each CTA
// goes to partials[iteration][block]; the trace and the divergence logic are
// evaluated in a fixed order after the loop (the pixel engine has no early
// exit, so the decisions only depend on the trace).
#pragma once

#include "kernels.cuh"

namespace mrb {

constexpr int kPixThreads = 512, kPixMaxR = 4;
// tile per CTA: 64x32 (fp32 state) / 32x32 (fp64 state); the (TX+2R)x(TY+2R)
// ping-pong state tiles stay under the 48 KB static shared-memory limit
template <typename Real> struct PixTile {
  static constexpr int TX = sizeof(Real) == 4 ? 64 : 32, TY = sizeof(Real) == 4 ? 32 : 24;
};

template <typename Real>
struct PixelDev {
  using R2 = typename V2<Real>::type;
  const R2* img;     // padded (H+2)x(W+2) interleaved (Te, Re), ring included
  R2* u[2];          // double-buffered (ux, uy) planes, H x W
  Real* warped;      // H x W
  double* partials;  // [iterations][tiles]
  int W, H, tiles_x, tiles;
};

// padded (Te, Re) image in Real with the ring computed in fp64
template <typename InT, typename Real>
__global__ void k_pixel_pad(const InT* const* __restrict__ re, const InT* const* __restrict__ te,
                            int W, int H, typename V2<Real>::type* __restrict__ out,
                            size_t out_stride) {
  const int Wp = W + 2, Hp = H + 2;
  const InT* r_img = re[blockIdx.y];
  const InT* t_img = te[blockIdx.y];
  auto* dst = out + blockIdx.y * out_stride;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < Wp * Hp; q += gridDim.x * blockDim.x) {
    const int r = q / Wp, c = q - r * Wp;
    typename V2<Real>::type f;
    f.x = Real(ext_tap<InT, double, 1>(t_img, W, H, r, c).v[0]);
    f.y = Real(ext_tap<InT, double, 1>(r_img, W, H, r, c).v[0]);
    dst[q] = f;
  }
}

template <typename Real>
__device__ __forceinline__ void cr_dweights(Real t, Real w[4]) {
  // image.py:167-178
  const Real t2 = mul_rn(t, t);
  const Real h = Real(0.5);
  w[0] = mul_rn(h, sub_rn(add_rn(mul_rn(Real(-3), t2), mul_rn(Real(4), t)), Real(1)));
  w[1] = mul_rn(h, sub_rn(mul_rn(Real(9), t2), mul_rn(Real(10), t)));
  w[2] = mul_rn(h, add_rn(add_rn(mul_rn(Real(-9), t2), mul_rn(Real(8), t)), Real(1)));
  w[3] = mul_rn(h, sub_rn(mul_rn(Real(3), t2), mul_rn(Real(2), t)));
}

// value of Te and Re and the analytic gradient of Te at (x, y), from the
// padded image (no border branch): s = (Te, Re), g = (dTe/dx, dTe/dy)
template <typename Real>
__device__ __forceinline__ void sample_with_gradient(const typename V2<Real>::type* __restrict__ img,
                                                     int W, int H, double x, double y,
                                                     typename V2<Real>::type& s,
                                                     typename V2<Real>::type& g) {
  const double xc = fmin(fmax(x, 0.0), double(W) - 1.0);
  const double yc = fmin(fmax(y, 0.0), double(H) - 1.0);
  const int cx = min(int(xc), W - 2);
  const int cy = min(int(yc), H - 2);
  const Real tx = Real(xc - double(cx)), ty = Real(yc - double(cy));
  Real wx[4], wy[4], dwx[4], dwy[4];
  cr_weights<Real>(tx, wx);
  cr_weights<Real>(ty, wy);
  cr_dweights<Real>(tx, dwx);
  cr_dweights<Real>(ty, dwy);
  const auto* base = img + (size_t(cy) * (W + 2) + cx);
  Real te = 0, re = 0, gx = 0, gy = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    Real rt = 0, rr = 0, rd = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const auto v = __ldg(base + size_t(j) * (W + 2) + i);
      rt = fma(wx[i], v.x, rt);
      rr = fma(wx[i], v.y, rr);
      rd = fma(dwx[i], v.x, rd);
    }
    te = fma(wy[j], rt, te);
    re = fma(wy[j], rr, re);
    gx = fma(wy[j], rd, gx);
    gy = fma(dwy[j], rt, gy);
  }
  s.x = te;
  s.y = re;
  g.x = gx;
  g.y = gy;
}

template <typename Real>
__global__ void __launch_bounds__(kPixThreads)
    k_pixel_iter(const PixelDev<Real>* __restrict__ pairs, int k, int src, Real tau, Real lam,
                 int R, int descend, int clamp) {
  using R2 = typename V2<Real>::type;
  constexpr int kPixTX = PixTile<Real>::TX, kPixTY = PixTile<Real>::TY;
  constexpr int RW = kPixTX + 2 * kPixMaxR, RH = kPixTY + 2 * kPixMaxR;
  __shared__ R2 buf[2][RH * RW];
  __shared__ double sh[2 * kPixThreads / 32];
  const PixelDev<Real>& d = pairs[blockIdx.y];
  const int tile = blockIdx.x;
  const int x0 = (tile % d.tiles_x) * kPixTX, y0 = (tile / d.tiles_x) * kPixTY;
  const R2* __restrict__ uin = d.u[src];
  R2* __restrict__ uout = d.u[src ^ 1];
  const int W = d.W, H = d.H;
  // region cell (ry, rx) <-> pixel (y0 - R + ry, x0 - R + rx)
  const int rw = kPixTX + 2 * R, rh = kPixTY + 2 * R;
  double e2 = 0.0;
  for (int c = threadIdx.x; c < rw * rh; c += kPixThreads) {
    const int ry = c / rw, rx = c - ry * rw;
    const int gy = y0 - R + ry, gx = x0 - R + rx;
    if (gx < 0 || gx >= W || gy < 0 || gy >= H) continue;
    const R2 u = uin[size_t(gy) * W + gx];
    if (!descend) {  // smoothing-only launch (passes beyond kPixMaxR)
      buf[0][ry * RW + rx] = u;
      continue;
    }
    R2 s, g;
    sample_with_gradient<Real>(d.img, W, H, double(gx) + double(u.x), double(gy) + double(u.y),
                               s, g);
    const Real r = sub_rn(s.x, s.y);
    const Real tr = mul_rn(tau, r);  // ux - tau * r * dTe/dx  (baseline.py:94-95)
    R2 o;
    o.x = sub_rn(u.x, mul_rn(tr, g.x));
    o.y = sub_rn(u.y, mul_rn(tr, g.y));
    buf[0][ry * RW + rx] = o;
    if (rx >= R && rx < R + kPixTX && ry >= R && ry < R + kPixTY) e2 += double(r) * double(r);
  }
  __syncthreads();
  int cur = 0;
  for (int p = 0; p < R; ++p) {  // smoothing passes on a shrinking region
    const int m = p + 1;         // margin of still-valid cells
    for (int c = threadIdx.x; c < rw * rh; c += kPixThreads) {
      const int ry = c / rw, rx = c - ry * rw;
      if (rx < m || rx >= rw - m || ry < m || ry >= rh - m) continue;
      const int gy = y0 - R + ry, gx = x0 - R + rx;
      if (gx < 0 || gx >= W || gy < 0 || gy >= H) continue;
      const R2* b = buf[cur];
      // baseline.py:33-43: above, below, left, right; edge-aware counts
      R2 tot;
      tot.x = Real(0);
      tot.y = Real(0);
      Real cnt = Real(0);
      if (gy > 0) {
        const R2 v = b[(ry - 1) * RW + rx];
        tot.x = add_rn(tot.x, v.x);
        tot.y = add_rn(tot.y, v.y);
        cnt = cnt + Real(1);
      }
      if (gy < H - 1) {
        const R2 v = b[(ry + 1) * RW + rx];
        tot.x = add_rn(tot.x, v.x);
        tot.y = add_rn(tot.y, v.y);
        cnt = cnt + Real(1);
      }
      if (gx > 0) {
        const R2 v = b[ry * RW + rx - 1];
        tot.x = add_rn(tot.x, v.x);
        tot.y = add_rn(tot.y, v.y);
        cnt = cnt + Real(1);
      }
      if (gx < W - 1) {
        const R2 v = b[ry * RW + rx + 1];
        tot.x = add_rn(tot.x, v.x);
        tot.y = add_rn(tot.y, v.y);
        cnt = cnt + Real(1);
      }
      const R2 self = b[ry * RW + rx];
      const Real om = sub_rn(Real(1), lam);
      R2 o;  // (1 - lam) * plane + lam * total / count
      o.x = add_rn(mul_rn(om, self.x), div_rn(mul_rn(lam, tot.x), cnt));
      o.y = add_rn(mul_rn(om, self.y), div_rn(mul_rn(lam, tot.y), cnt));
      buf[cur ^ 1][ry * RW + rx] = o;
    }
    __syncthreads();
    cur ^= 1;
  }
  for (int c = threadIdx.x; c < kPixTX * kPixTY; c += kPixThreads) {
    const int ty = c / kPixTX, tx = c - ty * kPixTX;
    const int gy = y0 + ty, gx = x0 + tx;
    if (gx >= W || gy >= H) continue;
    R2 o = buf[cur][(ty + R) * RW + tx + R];
    if (clamp) {  // np.clip(u, -x, (w - 1) - x), baseline.py:100-101
      // (NaN propagates like np.clip; fmin/fmax alone would drop it)
      if (o.x == o.x) o.x = Real(fmin(fmax(double(o.x), -double(gx)), (double(W) - 1.0) - double(gx)));
      if (o.y == o.y) o.y = Real(fmin(fmax(double(o.y), -double(gy)), (double(H) - 1.0) - double(gy)));
    }
    uout[size_t(gy) * W + gx] = o;
  }
  if (!descend) return;
  const double bs = block_sum<kPixThreads>(e2, sh);
  if (threadIdx.x == 0) d.partials[size_t(k) * d.tiles + tile] = bs;
}

// trace[k] = 0.5 * sum of the tile partials of iteration k (fixed order),
// then the divergence logic of baseline.py:81-91 over the trace
template <typename Real>
__global__ void __launch_bounds__(kPixBlock)
    k_pixel_trace(const PixelDev<Real>* __restrict__ pairs, int iterations, double* traces,
                  PairStatus* __restrict__ st) {
  __shared__ double sh[2 * kPixBlock / 32];
  const int p = blockIdx.x;
  const PixelDev<Real>& d = pairs[p];
  double* tr = traces + size_t(p) * iterations;
  for (int k = 0; k < iterations; ++k) {
    double acc = 0.0;
    for (int b = threadIdx.x; b < d.tiles; b += kPixBlock) acc += d.partials[size_t(k) * d.tiles + b];
    const double s = block_sum<kPixBlock>(acc, sh);
    if (threadIdx.x == 0) tr[k] = 0.5 * s;
  }
  if (threadIdx.x != 0) return;
  PairStatus s{};
  s.stop_iter = iterations;
  s.iters = iterations;
  int rises = 0;
  for (int k = 0; k < iterations; ++k) {
    const double e = tr[k];
    if (!isfinite(e)) {
      s.err = ERR_NONFINITE_ENERGY;
      s.err_iter = k;
      break;
    }
    if (k > 0 && e > __dadd_rn(__dmul_rn(tr[k - 1], 1.0 + 1e-4), 1e-12)) {
      if (++rises >= 10) {
        s.err = ERR_RISES;
        s.err_iter = k;
        break;
      }
    } else if (k > 0 && e <= tr[k - 1]) {
      rises = 0;
    }
  }
  s.rises = rises;
  st[p] = s;
}

// warp_image(template, field) + msd(warped, Re) and msd(Te, Re) partials
template <typename Real>
__global__ void __launch_bounds__(kPixBlock)
    k_pixel_warp(const PixelDev<Real>* __restrict__ pairs, int src, PairStatus* st,
                 double2* __restrict__ partials, int blocks_per_pair) {
  __shared__ double sh[2 * kPixBlock / 32];
  const int p = blockIdx.y;
  const PixelDev<Real>& d = pairs[p];
  const int q = blockIdx.x * kPixBlock + threadIdx.x;
  double2 acc = make_double2(0.0, 0.0);
  if (q < d.W * d.H && !st[p].err) {
    const int y = q / d.W, x = q - y * d.W;
    const auto u = d.u[src][q];
    if (!isfinite(u.x) || !isfinite(u.y)) atomicOr(const_cast<int*>(&st[p].dense_nonfinite), 1);
    typename V2<Real>::type s, g;
    sample_with_gradient<Real>(d.img, d.W, d.H, double(x) + double(u.x), double(y) + double(u.y),
                               s, g);
    d.warped[q] = s.x;
    if (!isfinite(s.x)) atomicOr(const_cast<int*>(&st[p].dense_nonfinite), 2);
    const auto own = d.img[size_t(y + 1) * (d.W + 2) + (x + 1)];
    const double d0 = double(own.x) - double(own.y);
    const double d1 = double(s.x) - double(own.y);
    acc.x = d0 * d0;
    acc.y = d1 * d1;
  }
  const double2 bs = block_sum2<kPixBlock>(acc, sh);
  if (threadIdx.x == 0) partials[size_t(p) * blocks_per_pair + blockIdx.x] = bs;
}

__global__ void __launch_bounds__(kPixBlock)
    k_pixel_msd(const double2* __restrict__ partials, int blocks_per_pair, double npx,
                PairStatus* __restrict__ st) {
  __shared__ double sh[2 * kPixBlock / 32];
  const int p = blockIdx.x;
  double2 acc = make_double2(0.0, 0.0);
  for (int b = threadIdx.x; b < blocks_per_pair; b += kPixBlock) {
    const double2 v = partials[size_t(p) * blocks_per_pair + b];
    acc.x += v.x;
    acc.y += v.y;
  }
  const double2 t = block_sum2<kPixBlock>(acc, sh);
  if (threadIdx.x == 0) {
    st[p].msd_before = t.x / npx;
    st[p].msd_after = t.y / npx;
  }
}

// single operations ----------------------------------------------------------
template <typename TapT>
__global__ void k_sample_gradient_points(const TapT* __restrict__ img, int W, int H, int n,
                                         const double* __restrict__ pts, double* __restrict__ gx,
                                         double* __restrict__ gy) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // exact on-the-fly ring (cr_sample's border path) with derivative weights
  const double xc = fmin(fmax(pts[2 * i], 0.0), double(W) - 1.0);
  const double yc = fmin(fmax(pts[2 * i + 1], 0.0), double(H) - 1.0);
  const int cx = min(int(floor(xc)), max(W - 2, 0));
  const int cy = min(int(floor(yc)), max(H - 2, 0));
  double wx[4], wy[4], dwx[4], dwy[4];
  cr_weights<double>(xc - double(cx), wx);
  cr_weights<double>(yc - double(cy), wy);
  cr_dweights<double>(xc - double(cx), dwx);
  cr_dweights<double>(yc - double(cy), dwy);
  double ax = 0, ay = 0;
  for (int j = 0; j < 4; ++j) {
    double rd = 0, rt = 0;
    for (int i2 = 0; i2 < 4; ++i2) {
      const double v = ext_tap<TapT, double, 1>(img, W, H, cy + j, cx + i2).v[0];
      rd = fma(dwx[i2], v, rd);
      rt = fma(wx[i2], v, rt);
    }
    ax = fma(wy[j], rd, ax);
    ay = fma(dwy[j], rt, ay);
  }
  gx[i] = ax;
  gy[i] = ay;
}

__global__ void k_grid_umbrella(const double* __restrict__ in, int W, int H, double lam,
                                double* __restrict__ out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= W * H) return;
  const int y = q / W, x = q - y * W;
  double tot = 0.0, cnt = 0.0;
  if (y > 0) { tot = __dadd_rn(tot, in[q - W]); cnt += 1.0; }
  if (y < H - 1) { tot = __dadd_rn(tot, in[q + W]); cnt += 1.0; }
  if (x > 0) { tot = __dadd_rn(tot, in[q - 1]); cnt += 1.0; }
  if (x < W - 1) { tot = __dadd_rn(tot, in[q + 1]); cnt += 1.0; }
  out[q] = __dadd_rn(__dmul_rn(1.0 - lam, in[q]), __ddiv_rn(__dmul_rn(lam, tot), cnt));
}

}  // namespace mrb
