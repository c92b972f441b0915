// Pixel-grid engine (reference baseline.py:46-118):
// one displacement per pixel, descent along residual x analytic spline
// gradient of the template (image.py:86-103), `passes` 4-neighbour umbrella
// smoothing passes (baseline.py:27-43), clamp, `iterations` times.
//
// B200 design: one fused kernel per iteration, ordered smooth-then-sample.
// A CTA owns a TX x TY tile.  Launch k reads the descended planes of
// iteration k-1 (tile + a halo of `passes` pixels, one TMA box), runs the
// smoothing passes in shared memory (the valid region shrinks by one pixel
// per pass, the last pass fused with the tile phase), clamps, and then
// samples Te, Re and dTe/dx, dTe/dy (from the same 16 taps, a TMA-staged
// image patch) for the tile's OWN pixels only, applies the descent and
// writes the descended planes.  Sampling before smoothing (the reference's
// order inside one iteration) would sample every halo pixel again in each
// neighbouring tile (1.3 samples per pixel at 64x32 with a 3-pixel halo);
// here each pixel is sampled once.  HBM traffic per pixel and iteration:
// read the descended planes, write them, read the (Te, Re) patch.  The fp64
// energy partial of each CTA goes to partials[iteration][block]; the trace
// and the divergence logic are evaluated in a fixed order after the loop
// (the pixel engine has no early exit, so the decisions only depend on the
// trace).
#pragma once

#include <cuda.h>

#include "kernels.cuh"

namespace mrb {

constexpr int kPixThreads = 256, kPixMaxR = 3, kPixMinBlocks = 4;
// tile per CTA: 64x32 (fp32 state) / 32x32 (fp64 state): four / two tile
// cells per thread
template <typename Real> struct PixTile {
  static constexpr int TX = sizeof(Real) == 4 ? 64 : 32, TY = sizeof(Real) == 4 ? 24 : 32;
};

template <typename Real>
struct PixelDev {
  using R2 = typename V2<Real>::type;
  const R2* img;     // padded (H+2) rows x (W+2) of interleaved (Te, Re), ring
                     // included, row pitch `pitch` elements (16-byte multiple)
  const CUtensorMap* tmap;  // TMA descriptor of img (2-D, 8-byte elements)
  R2* u;             // final (ux, uy) plane, H x W
  Real* warped;      // H x W
  double* partials;  // [iterations][tiles]
  int W, H, pitch, tiles_x, tiles;
};

// k_pixel_step's arguments: batch-uniform, passed by value (kernel
// parameter space: no dependent global loads in the prologue); pair p's
// arrays are at fixed strides from the bases
template <typename Real>
struct PixelStepArgs {
  using R2 = typename V2<Real>::type;
  const R2* img;            // padded pair images, img_stride elements apart
  const CUtensorMap* tmap;  // [n] image maps, then [n] plane maps
  R2* w;                    // descended planes: buffer b of pair p at (b n + p) wplane
  R2* u;                    // final planes, H x W each
  double* partials;         // [pair][iteration][tile]
  size_t img_stride, wplane;
  int n, iterations, W, H, pitch, wpitch, tiles_x, tiles;
};

// Shared-memory layout of k_pixel_step for a tile (x0, y0):
//  * patch: the padded (Te, Re) image around the tile, staged by TMA, for
//    the samples: tile + Catmull-Rom footprint (3) + displacement margin
//    kPixD, origin (x0 - kPixD, y0 - kPixD) in padded coordinates (even x: a
//    TMA box starts on a 16-byte boundary of the row);
//  * two state buffers of the tile + the smoothing halo, kPixMaxR rows and
//    kPixHX >= kPixMaxR (even) columns on each side, origin (x0 - kPixHX,
//    y0 - kPixMaxR); the descended planes land in buffer 0 by TMA (zero
//    outside the image).
// One box per tensor map serves every halo R <= kPixMaxR.
constexpr int kPixD = 4, kPixHX = 4;
template <typename Real> struct PixPatch {
  static constexpr int TX = PixTile<Real>::TX, TY = PixTile<Real>::TY;
  static constexpr int PW = (TX + 2 * kPixD + 3 + 1) / 2 * 2, PH = TY + 2 * kPixD + 3;
  static constexpr int BW = TX + 2 * kPixHX, BH = TY + 2 * kPixMaxR;
  static constexpr size_t patch_bytes = size_t(PW) * PH * 2 * sizeof(Real);
  static constexpr size_t buf_bytes = size_t(BW) * BH * 2 * sizeof(Real);
  // the state buffers start 128-byte aligned (TMA shared-memory destination)
  static constexpr size_t buf_off = (patch_bytes + 127) / 128 * 128;
  static constexpr size_t smem_bytes = buf_off + 2 * buf_bytes;
};

__device__ __forceinline__ unsigned pix_smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// padded (Te, Re) image in Real with the ring computed in fp64
template <typename InT, typename Real>
__global__ void k_pixel_pad(const InT* const* __restrict__ re, const InT* const* __restrict__ te,
                            int W, int H, int pitch, typename V2<Real>::type* __restrict__ out,
                            size_t out_stride) {
  const int Wp = W + 2, Hp = H + 2;
  const InT* r_img = re[blockIdx.y];
  const InT* t_img = te[blockIdx.y];
  auto* dst = out + blockIdx.y * out_stride;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < Wp * Hp; q += gridDim.x * blockDim.x) {
    const int r = q / Wp, c = q - r * Wp;
    typename V2<Real>::type f;
    const size_t at = size_t(r) * pitch + c;
    f.x = Real(ext_tap<InT, double, 1>(t_img, W, H, r, c).v[0]);
    f.y = Real(ext_tap<InT, double, 1>(r_img, W, H, r, c).v[0]);
    dst[at] = f;
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

// Clamped cell + fraction of a displaced coordinate q + u (q integer): the
// reference computes xc = clip(q + u, 0, n - 1), c = min(floor(xc), n - 2),
// t = xc - c in fp64 (image.py:105-121).  q + u splits exactly into the
// integer q + floor(u) and the fraction u - floor(u) when u is fp32, so c
// and t come out bit-identical without fp64 arithmetic.  For fp64 state the
// sum q + u rounds, and the reference's t carries that rounding: computed
// the reference's way (report.msd_after == msd(warp_image(te, field), re)
// holds exactly, as in the reference's test_baseline.py).
template <typename Real>
__device__ __forceinline__ void locate_axis(int q, Real u, int n, int& c, Real& t) {
  if constexpr (sizeof(Real) == 8) {
    const double xs = double(q) + u;
    double xc = fmin(fmax(xs, 0.0), double(n) - 1.0);
    if (xs != xs) xc = xs;  // np.clip propagates NaN
    c = min(int(floor(xc)), n - 2);  // xc >= 0 (or NaN -> 0); n = 1 gives c = -1, t = 1 like the reference
    t = xc - double(c);
    return;
  }
  const Real fl = floor(u);
  t = u - fl;  // exact
  c = q + int(fl);
  if (c < 0) {
    c = 0;
    t = Real(0);
  } else if (c >= n - 1) {
    c = n - 2;
    t = Real(1);
  }
}

// packed fp32x2 FMA (FFMA2 on sm_100a): r = a * b + c lane-wise
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long ra, rb, rc, rd;
  memcpy(&ra, &a, 8);
  memcpy(&rb, &b, 8);
  memcpy(&rc, &c, 8);
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
  float2 r;
  memcpy(&r, &rd, 8);
  return r;
}

// (w_i, dw_i) Catmull-Rom weight / derivative pairs by Horner in FFMA2
// (image.py:154-178 expanded: w_i = ((a3 t + a2) t + a1) t + a0,
// dw_i = (b2 t + b1) t + b0)
__device__ __forceinline__ void cr_weight_pairs(float t, float2 wd[4]) {
  const float2 tt = make_float2(t, t);
  const float2 A3[4] = {{-0.5f, 0.f}, {1.5f, 0.f}, {-1.5f, 0.f}, {0.5f, 0.f}};
  const float2 A2[4] = {{1.0f, -1.5f}, {-2.5f, 4.5f}, {2.0f, -4.5f}, {-0.5f, 1.5f}};
  const float2 A1[4] = {{-0.5f, 2.0f}, {0.0f, -5.0f}, {0.5f, 4.0f}, {0.0f, -1.0f}};
  const float2 A0[4] = {{0.0f, -0.5f}, {1.0f, 0.0f}, {0.0f, 0.5f}, {0.0f, 0.0f}};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 h = ffma2(A3[i], tt, A2[i]);
    h = ffma2(h, tt, A1[i]);
    wd[i] = ffma2(h, tt, A0[i]);
  }
}

// value of Te and Re and the analytic gradient of Te at cell (cx, cy) +
// fraction (tx, ty), from the padded image (no border branch):
// s = (Te, Re), g = (dTe/dx, dTe/dy)
template <typename Real, bool SMEM = false>
__device__ __forceinline__ void sample_with_gradient(const typename V2<Real>::type* __restrict__ img,
                                                     int pitch, int cx, int cy, Real tx, Real ty,
                                                     typename V2<Real>::type& s,
                                                     typename V2<Real>::type& g) {
  using R2 = typename V2<Real>::type;
  const R2* base = img + (size_t(cy) * pitch + cx);
  auto tap = [&](int j, int i) -> R2 {
    if constexpr (SMEM)
      return base[j * pitch + i];
    else
      return __ldg(base + size_t(j) * pitch + i);
  };
  if constexpr (std::is_same<Real, float>::value) {
    float2 wdx[4], wdy[4];
    cr_weight_pairs(tx, wdx);
    cr_weight_pairs(ty, wdy);
    float2 acc = make_float2(0.f, 0.f);  // (Te, Re)
    float gx = 0.f, gy = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 row = make_float2(0.f, 0.f);  // (Te, Re) along x
      float rd = 0.f;                      // dTe/dx along x
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 v = tap(j, i);
        row = ffma2(make_float2(wdx[i].x, wdx[i].x), v, row);
        rd = fmaf(wdx[i].y, v.x, rd);
      }
      acc = ffma2(make_float2(wdy[j].x, wdy[j].x), row, acc);
      gx = fmaf(wdy[j].x, rd, gx);
      gy = fmaf(wdy[j].y, row.x, gy);
    }
    s = acc;
    g = make_float2(gx, gy);
  } else {
    Real wx[4], wy[4], dwx[4], dwy[4];
    cr_weights<Real>(tx, wx);
    cr_weights<Real>(ty, wy);
    cr_dweights<Real>(tx, dwx);
    cr_dweights<Real>(ty, dwy);
    Real te = 0, re = 0, gx = 0, gy = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      Real rt = 0, rr = 0, rd = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const auto v = tap(j, i);
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
}

// Pair arithmetic on (x, y) state: packed f32x2 instructions for fp32 state
// (FADD2/FMUL2/FFMA2, tolerance mode), exact-rounding scalar ops for fp64.
__device__ __forceinline__ unsigned long long pk2(float2 a) {
  unsigned long long r;
  memcpy(&r, &a, 8);
  return r;
}
__device__ __forceinline__ float2 upk2(unsigned long long a) {
  float2 r;
  memcpy(&r, &a, 8);
  return r;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)));
  return upk2(d);
}
__device__ __forceinline__ double2 add2(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
// (1 - lam) * self + lq * tot, lq = lam / count (count 4 or 2: an exact
// power-of-two scaling of lam * tot)
__device__ __forceinline__ float2 blend2(float om, float2 self, float lq, float2 tot) {
  unsigned long long d, m;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(m) : "l"(pk2(make_float2(om, om))), "l"(pk2(self)));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pk2(make_float2(lq, lq))), "l"(pk2(tot)), "l"(m));
  return upk2(d);
}
__device__ __forceinline__ double2 blend2(double om, double2 self, double lq, double2 tot) {
  return make_double2(__dadd_rn(__dmul_rn(om, self.x), __dmul_rn(lq, tot.x)),
                      __dadd_rn(__dmul_rn(om, self.y), __dmul_rn(lq, tot.y)));
}

// One grid_umbrella_smooth cell (baseline.py:27-43) of pixel (gx, gy) from
// its value and its neighbour total ((N + S) + W) + E.  INTERIOR: the cell
// and its four neighbours lie inside the image (count = 4).  Otherwise cells
// outside the image hold zero (returned as zero), so a missing neighbour
// adds +0 exactly like the reference's zero-initialised total.
template <typename Real, bool INTERIOR>
__device__ __forceinline__ typename V2<Real>::type smooth_value(
    typename V2<Real>::type self, typename V2<Real>::type tot, int gx, int gy, int W, int H,
    Real om, Real lam) {
  using R2 = typename V2<Real>::type;
  const Real lq4 = lam * Real(0.25);  // exact
  if (INTERIOR) return blend2(om, self, lq4, tot);
  // strictly inside the image (the common case of a border tile): one
  // unsigned compare per axis
  if (unsigned(gx - 1) < unsigned(max(W - 2, 0)) && unsigned(gy - 1) < unsigned(max(H - 2, 0)))
    return blend2(om, self, lq4, tot);
  if (unsigned(gx) >= unsigned(W) || unsigned(gy) >= unsigned(H)) return R2{Real(0), Real(0)};
  const int cnt = (gy > 0) + (gy < H - 1) + (gx > 0) + (gx < W - 1);
  if (cnt == 4) return blend2(om, self, lq4, tot);
  if (cnt == 2) return blend2(om, self, lam * Real(0.5), tot);
  // count 3 (or 0 for a 1-pixel plane: 0 / 0 like numpy)
  R2 v;
  v.x = add_rn(mul_rn(om, self.x), div_rn(mul_rn(lam, tot.x), Real(cnt)));
  v.y = add_rn(mul_rn(om, self.y), div_rn(mul_rn(lam, tot.y), Real(cnt)));
  return v;
}

// the cell at buffer index q (row width BW)
template <typename Real, int BW, bool INTERIOR>
__device__ __forceinline__ typename V2<Real>::type smooth_cell(
    const typename V2<Real>::type* __restrict__ b, int q, int gx, int gy, int W, int H, Real om,
    Real lam) {
  const auto tot = add2(add2(add2(b[q - BW], b[q + BW]), b[q - 1]), b[q + 1]);
  return smooth_value<Real, INTERIOR>(b[q], tot, gx, gy, W, H, om, lam);
}

// fp32 state: the cells at q and q + 1 (q even, so (q, q+1) is one 16-byte
// word): three 128-bit loads (centre, north, south pairs) + two 64-bit loads
// (west of q, east of q+1) instead of ten 64-bit loads; same sums per cell
template <int BW, bool INTERIOR>
__device__ __forceinline__ void smooth_pair(const float2* __restrict__ b, int q, int gx, int gy,
                                            int W, int H, float om, float lam, float2& o0,
                                            float2& o1) {
  const float4 c = *reinterpret_cast<const float4*>(b + q);
  const float4 n = *reinterpret_cast<const float4*>(b + q - BW);
  const float4 s = *reinterpret_cast<const float4*>(b + q + BW);
  const float2 w = b[q - 1], e = b[q + 2];
  const float2 c0 = make_float2(c.x, c.y), c1 = make_float2(c.z, c.w);
  const float2 t0 = add2(add2(add2(make_float2(n.x, n.y), make_float2(s.x, s.y)), w), c1);
  const float2 t1 = add2(add2(add2(make_float2(n.z, n.w), make_float2(s.z, s.w)), c0), e);
  o0 = smooth_value<float, INTERIOR>(c0, t0, gx, gy, W, H, om, lam);
  o1 = smooth_value<float, INTERIOR>(c1, t1, gx + 1, gy, W, H, om, lam);
}

// Smoothing passes M = MM..R-1 of R in shared memory: pass M covers the
// cells at margin M of the tile's R-halo region, (TX + 2(R-M)) x
// (TY + 2(R-M)), reading buffer (M-1)&1 and writing buffer M&1.  Pass R is
// fused into the tile phase of k_pixel_step.  fp32: cells in aligned pairs,
// the region widened to even buffer columns (an extra cell at margin M-1
// overwrites a value no later pass reads).
template <typename Real, int R, int MM, bool INTERIOR>
__device__ __forceinline__ void smooth_passes(
    typename V2<Real>::type (*buf)[PixPatch<Real>::BW * PixPatch<Real>::BH], int x0, int y0,
    int W, int H, Real om, Real lam) {
  if constexpr (MM < R) {
    using PP = PixPatch<Real>;
    constexpr int BW = PP::BW, w = PP::TX + 2 * (R - MM), h = PP::TY + 2 * (R - MM);
    // buffer coordinates of the pass region's first cell
    constexpr int bx0 = kPixHX - R + MM, by0 = kPixMaxR - R + MM;
    const auto* __restrict__ b = buf[(MM - 1) & 1];
    auto* __restrict__ o = buf[MM & 1];
    if constexpr (sizeof(Real) == 4) {
      constexpr int bxe = bx0 & ~1, pw = (bx0 + w - bxe + 1) / 2;  // pairs per row
#pragma unroll 2
      for (int c = threadIdx.x; c < pw * h; c += kPixThreads) {
        const int cy = c / pw, cx = c - cy * pw;  // constant divisor
        const int bx = bxe + 2 * cx, by = by0 + cy;
        float2 o0, o1;
        smooth_pair<BW, INTERIOR>(b, by * BW + bx, x0 + bx - kPixHX, y0 + by - kPixMaxR, W, H,
                                  om, lam, o0, o1);
        *reinterpret_cast<float4*>(o + by * BW + bx) = make_float4(o0.x, o0.y, o1.x, o1.y);
      }
    } else {
#pragma unroll 2
      for (int c = threadIdx.x; c < w * h; c += kPixThreads) {
        const int cy = c / w, cx = c - cy * w;  // constant divisor
        const int bx = bx0 + cx, by = by0 + cy;
        o[by * BW + bx] = smooth_cell<Real, BW, INTERIOR>(b, by * BW + bx, x0 + bx - kPixHX,
                                                         y0 + by - kPixMaxR, W, H, om, lam);
      }
    }
    __syncthreads();
    smooth_passes<Real, R, MM + 1, INTERIOR>(buf, x0, y0, W, H, om, lam);
  }
}

// One launch of the pixel engine for a TX x TY tile (baseline.py:74-101),
// ordered smooth-then-sample so no halo cell is sampled:
//   load:   TMA the previous launch's descended planes (tile + R halo) into
//           shared memory (else the state is zero: iteration 0);
//   R smoothing passes (R-1 in shared memory, the last fused with the tile
//   phase); clamp (after the iteration's last pass);
//   sample: Te, Re and the analytic gradient of Te at the smoothed u of the
//           tile's own pixels (iteration k's energy partial), descent, store
//           the descended planes to w[dst];
//   final:  store u (the registration result) instead.
// Without clamp / sample / final the launch is an extra smoothing launch
// (passes beyond kPixMaxR) that stores to w[dst].
template <typename Real, int R>
__global__ void __launch_bounds__(kPixThreads, kPixMinBlocks)
    k_pixel_step(const PixelStepArgs<Real> a, int k, int src, Real tau, Real lam, int load,
                 int clamp, int sample, int final_out) {
  using R2 = typename V2<Real>::type;
  using PP = PixPatch<Real>;
  constexpr int TX = PP::TX, TY = PP::TY, BW = PP::BW, PW = PP::PW, PH = PP::PH;
  extern __shared__ __align__(128) unsigned char pix_smem[];
  R2* patch = reinterpret_cast<R2*>(pix_smem);
  auto buf = reinterpret_cast<R2(*)[PP::BW * PP::BH]>(pix_smem + PP::buf_off);
  __shared__ double sh[2 * kPixThreads / 32];
  __shared__ __align__(8) unsigned long long mbar;
  // grid (tiles_x, tiles_y, pairs): no division for the tile origin
  const int pair = blockIdx.z, tile = blockIdx.y * a.tiles_x + blockIdx.x;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int W = a.W, H = a.H;
  // patch origin in padded-image coordinates (may be negative: TMA zero-fills)
  const int px0 = x0 - kPixD, py0 = y0 - kPixD;
  constexpr int epr = int(sizeof(R2) / 8);  // 8-byte TMA elements per R2
  const unsigned mb = pix_smem_u32(&mbar);
  if ((load || sample) && threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const unsigned bytes =
        unsigned((sample ? PP::patch_bytes : 0) + (load ? PP::buf_bytes : 0));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes)
                 : "memory");
    if (load)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(pix_smem_u32(buf[0])),
          "l"(reinterpret_cast<unsigned long long>(a.tmap + a.n + pair)), "r"(epr * (x0 - kPixHX)),
          "r"(y0 - kPixMaxR), "r"(src), "r"(mb)
          : "memory");
    if (sample)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3}], [%4];" ::"r"(pix_smem_u32(patch)),
          "l"(reinterpret_cast<unsigned long long>(a.tmap + pair)), "r"(epr * px0), "r"(py0), "r"(mb)
          : "memory");
  }
  __syncthreads();  // mbarrier initialised before anyone waits on it
  if (load || sample)
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(mb)
        : "memory");
  const Real om = sub_rn(Real(1), lam);
  // every smoothed cell and its neighbours inside the image?
  const bool interior = x0 >= R && y0 >= R && x0 + TX + R <= W && y0 + TY + R <= H;
  if constexpr (R > 1) {
    if (load) {
      if (interior)
        smooth_passes<Real, R, 1, true>(buf, x0, y0, W, H, om, lam);
      else
        smooth_passes<Real, R, 1, false>(buf, x0, y0, W, H, om, lam);
    }
  }
  const R2* __restrict__ last = buf[(R - 1) & 1];  // input of the fused pass R
  const int wpitch = a.wpitch;
  // the tile's first pixel in the destination planes: 32-bit offsets from here
  R2* __restrict__ wout =
      a.w + (size_t(src ^ 1) * a.n + pair) * a.wplane + (size_t(y0) * wpitch + x0);
  double e2 = 0.0;
  // clamp + store, or sample + descent + store, for one tile pixel
  auto finish = [&](R2 u, int gx, int gy, Real xlo, Real xhi) {
    if (clamp) {  // np.clip(u, -x, (w - 1) - x), baseline.py:100-101; the
      // bounds are integers, exact in Real (xlo = -x, xhi = w - 1 - x: the
      // thread's column is fixed).  NaN propagates like np.clip.
      if (u.x == u.x) u.x = fmin(fmax(u.x, xlo), xhi);
      if (u.y == u.y) u.y = fmin(fmax(u.y, Real(-gy)), Real(H - 1 - gy));
    }
    if (final_out) {
      a.u[(size_t(pair) * H + gy) * W + gx] = u;
      return;
    }
    if (!sample) {
      wout[(gy - y0) * wpitch + (gx - x0)] = u;
      return;
    }
    int cx, cy;
    Real tx_, ty_;
    locate_axis<Real>(gx, u.x, W, cx, tx_);
    locate_axis<Real>(gy, u.y, H, cy, ty_);
    R2 s, g;
    const int lx = cx - px0, ly = cy - py0;  // footprint inside the patch?
    if (lx >= 0 && lx <= PW - 4 && ly >= 0 && ly <= PH - 4)
      sample_with_gradient<Real, true>(patch, PW, lx, ly, tx_, ty_, s, g);
    else  // displaced beyond kPixD: read the padded image in global memory
      sample_with_gradient<Real>(a.img + pair * a.img_stride, a.pitch, cx, cy, tx_, ty_, s, g);
    const Real r = sub_rn(s.x, s.y);
    const Real tr = mul_rn(tau, r);  // ux - tau * r * dTe/dx  (baseline.py:94-95)
    R2 o;
    o.x = sub_rn(u.x, mul_rn(tr, g.x));
    o.y = sub_rn(u.y, mul_rn(tr, g.y));
    wout[(gy - y0) * wpitch + (gx - x0)] = o;
    e2 = fma(double(r), double(r), e2);
  };
  // one pixel per thread and step: a warp samples 32 consecutive pixels of a
  // row, so each tap load of the warp spans ~32 consecutive patch cells (two
  // shared-memory wavefronts; pairs of pixels per thread would double that)
  // Thread t takes column t % TX of rows t / TX, t / TX + RS, ...: its column,
  // x bounds and buffer column are loop constants.
  static_assert(kPixThreads % TX == 0, "whole tile rows per step");
  constexpr int RS = kPixThreads / TX;
  const int tx = threadIdx.x % TX, gx = x0 + tx;
  if (gx < W) {
    const Real xlo = Real(-gx), xhi = Real(W - 1 - gx);
    const int gy_end = min(y0 + TY, H);
    int q = (threadIdx.x / TX + kPixMaxR) * BW + tx + kPixHX;
#pragma unroll 1
    for (int gy = y0 + threadIdx.x / TX; gy < gy_end; gy += RS, q += RS * BW) {
      R2 u = R2{Real(0), Real(0)};
      if (load) {
        if constexpr (R > 0) {
          u = interior ? smooth_cell<Real, BW, true>(last, q, gx, gy, W, H, om, lam)
                       : smooth_cell<Real, BW, false>(last, q, gx, gy, W, H, om, lam);
        } else {
          u = buf[0][q];
        }
      }
      finish(u, gx, gy, xlo, xhi);
    }
  }
  if (!sample) return;
  const double bs = block_sum<kPixThreads>(e2, sh);
  if (threadIdx.x == 0)
    a.partials[(size_t(pair) * a.iterations + k) * a.tiles + tile] = bs;
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
    const auto u = d.u[q];
    if (!isfinite(u.x) || !isfinite(u.y)) atomicOr(const_cast<int*>(&st[p].dense_nonfinite), 1);
    typename V2<Real>::type s, g;
    int cx, cy;
    Real tx, ty;
    locate_axis<Real>(x, u.x, d.W, cx, tx);
    locate_axis<Real>(y, u.y, d.H, cy, ty);
    sample_with_gradient<Real>(d.img, d.pitch, cx, cy, tx, ty, s, g);
    d.warped[q] = s.x;
    if (!isfinite(s.x)) atomicOr(const_cast<int*>(&st[p].dense_nonfinite), 2);
    const auto own = d.img[size_t(y + 1) * d.pitch + (x + 1)];
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
