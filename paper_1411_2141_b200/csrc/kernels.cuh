// Device code of the B200 registration path (sm_100a).
//
// One registration iteration of the reference (solver.py:171-195) is three
// node-parallel phases separated by the two neighbour exchanges it needs:
//   k_sample : s = Catmull-Rom(Te,Re) at V+u, r = s_te - s_re, fp64 energy
//              partial; the last block of each pair reduces the partials in a
//              fixed order and runs the divergence / tolerance logic
//              (solver.py:174-195) on the device — no host sync per iteration.
//   k_grad   : grad = r * G s_te with G = vertex_average_op ∘ grad_{x,y}_op
//              fused into one one-ring operator (mesh.py:236-241),
//              u0 = u - tau*grad, finite check (solver.py:130-133).
//   k_smooth : u <- (1-lam) u0 + lam L u0 per pass, then the domain clamp
//              (mesh.py:268-282, solver.py:134-144).
// After the loop, k_dense does densify + backward warp + both MSD partials in
// one pass over the pixels (densefield.py:130-199, image.py:181-186).
//
// Precision: TapT is the stored image type (fp32 when the inputs are
// fp32-exact, else fp64), Real the state/arithmetic type.  Positions, the
// pixel map predicates and every reduction are fp64.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace mrb {

constexpr int kNodeBlock = 256;
constexpr int kPixBlock = 256;
// pixel-map sentinel: what cudaMemset(..., 0x7f, ...) leaves in every int
constexpr int kUnassigned = 0x7f7f7f7f;

enum : int {
  ERR_NONE = 0,
  ERR_NONFINITE_ENERGY = 1,  // solver.py:176-177
  ERR_RISES = 2,             // solver.py:178-184
  ERR_NONFINITE_GRAD = 3,    // solver.py:131-132
};

struct PairStatus {
  int stop_iter;  // iterations k < stop_iter run completely
  int err;
  int err_iter;
  int rises;
  int iters;           // len(trace)
  int dense_nonfinite; // ux/uy or warped non-finite (DenseField / ImageGrid checks)
  unsigned ticket;     // last-block counter for the energy reduction
  int pad;
  double msd_before, msd_after;
};

template <typename T> struct V2;
template <> struct V2<float> { using type = float2; };
template <> struct V2<double> { using type = double2; };

// ---- exact-rounding helpers (no FMA contraction), used where the reference's
// ---- numpy operation order is reproduced bit for bit
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

template <typename Real>
__device__ __forceinline__ void cr_weights(Real t, Real w[4]) {
  // image.py:151-164, same operation order
  const Real t2 = mul_rn(t, t);
  const Real t3 = mul_rn(t2, t);
  const Real h = Real(0.5);
  w[0] = mul_rn(h, sub_rn(add_rn(-t3, mul_rn(Real(2), t2)), t));
  w[1] = mul_rn(h, add_rn(sub_rn(mul_rn(Real(3), t3), mul_rn(Real(5), t2)), Real(2)));
  w[2] = mul_rn(h, add_rn(add_rn(mul_rn(Real(-3), t3), mul_rn(Real(4), t2)), t));
  w[3] = mul_rn(h, sub_rn(t3, t2));
}

// C interleaved channels of TapT, row-major H x W.
template <typename TapT, typename Real, int C>
struct Px {
  Real v[C];
};

template <typename TapT, typename Real, int C>
__device__ __forceinline__ Px<TapT, Real, C> load_px(const TapT* __restrict__ img, int W,
                                                     int y, int x) {
  Px<TapT, Real, C> r;
  const int idx = y * W + x;
  if constexpr (C == 2) {
    const typename V2<TapT>::type t =
        __ldg(reinterpret_cast<const typename V2<TapT>::type*>(img) + idx);
    r.v[0] = Real(t.x);
    r.v[1] = Real(t.y);
  } else {
    r.v[0] = Real(__ldg(img + idx));
  }
  return r;
}

// Value of the one-ring-extended image at extended row r, column c
// (image.py:62-71,134-148: extend along x first, then along y).
template <typename TapT, typename Real, int C>
__device__ Px<TapT, Real, C> ext_row(const TapT* img, int W, int y, int c) {
  using P = Px<TapT, Real, C>;
  if (c >= 1 && c <= W) return load_px<TapT, Real, C>(img, W, y, c - 1);
  P out;
  const bool lo = (c == 0);
  if (W >= 3) {
    const P a0 = load_px<TapT, Real, C>(img, W, y, lo ? 0 : W - 1);
    const P a1 = load_px<TapT, Real, C>(img, W, y, lo ? 1 : W - 2);
    const P a2 = load_px<TapT, Real, C>(img, W, y, lo ? 2 : W - 3);
#pragma unroll
    for (int k = 0; k < C; ++k)
      out.v[k] = add_rn(sub_rn(mul_rn(Real(3), a0.v[k]), mul_rn(Real(3), a1.v[k])), a2.v[k]);
  } else if (W == 2) {
    const P a0 = load_px<TapT, Real, C>(img, W, y, lo ? 0 : 1);
    const P a1 = load_px<TapT, Real, C>(img, W, y, lo ? 1 : 0);
#pragma unroll
    for (int k = 0; k < C; ++k) out.v[k] = sub_rn(mul_rn(Real(2), a0.v[k]), a1.v[k]);
  } else {
    out = load_px<TapT, Real, C>(img, W, y, 0);
  }
  return out;
}

template <typename TapT, typename Real, int C>
__device__ Px<TapT, Real, C> ext_tap(const TapT* img, int W, int H, int r, int c) {
  using P = Px<TapT, Real, C>;
  if (r >= 1 && r <= H) return ext_row<TapT, Real, C>(img, W, r - 1, c);
  P out;
  const bool lo = (r == 0);
  if (H >= 3) {
    const P a0 = ext_row<TapT, Real, C>(img, W, lo ? 0 : H - 1, c);
    const P a1 = ext_row<TapT, Real, C>(img, W, lo ? 1 : H - 2, c);
    const P a2 = ext_row<TapT, Real, C>(img, W, lo ? 2 : H - 3, c);
#pragma unroll
    for (int k = 0; k < C; ++k)
      out.v[k] = add_rn(sub_rn(mul_rn(Real(3), a0.v[k]), mul_rn(Real(3), a1.v[k])), a2.v[k]);
  } else if (H == 2) {
    const P a0 = ext_row<TapT, Real, C>(img, W, lo ? 0 : 1, c);
    const P a1 = ext_row<TapT, Real, C>(img, W, lo ? 1 : 0, c);
#pragma unroll
    for (int k = 0; k < C; ++k) out.v[k] = sub_rn(mul_rn(Real(2), a0.v[k]), a1.v[k]);
  } else {
    out = ext_row<TapT, Real, C>(img, W, 0, c);
  }
  return out;
}

// Catmull-Rom sample at continuous (x, y) — ImageGrid.sample, image.py:73-84
// with _locate (105-116): clamp, base cell min(floor, size-2), t = xc - x0.
// Interior cells gather 16 taps straight from the stored image; cells touching
// the border rebuild the extrapolated ring from the stored pixels.
template <typename TapT, typename Real, int C>
__device__ __forceinline__ Px<TapT, Real, C> cr_sample(const TapT* __restrict__ img, int W,
                                                       int H, double x, double y) {
  const double xc = fmin(fmax(x, 0.0), double(W) - 1.0);
  const double yc = fmin(fmax(y, 0.0), double(H) - 1.0);
  const int cx = min(int(floor(xc)), max(W - 2, 0));
  const int cy = min(int(floor(yc)), max(H - 2, 0));
  Real wx[4], wy[4];
  cr_weights<Real>(Real(xc - double(cx)), wx);
  cr_weights<Real>(Real(yc - double(cy)), wy);
  Px<TapT, Real, C> acc;
#pragma unroll
  for (int k = 0; k < C; ++k) acc.v[k] = Real(0);
  if (cx >= 1 && cx <= W - 3 && cy >= 1 && cy <= H - 3) {
    const TapT* base = img + size_t(C) * (size_t(cy - 1) * W + (cx - 1));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      Px<TapT, Real, C> tap[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) tap[i] = load_px<TapT, Real, C>(base, W, j, i);
#pragma unroll
      for (int k = 0; k < C; ++k) {
        Real row = wx[0] * tap[0].v[k];
        row = fma(wx[1], tap[1].v[k], row);
        row = fma(wx[2], tap[2].v[k], row);
        row = fma(wx[3], tap[3].v[k], row);
        acc.v[k] = fma(wy[j], row, acc.v[k]);
      }
    }
  } else {
#pragma unroll 1
    for (int j = 0; j < 4; ++j) {
      Px<TapT, Real, C> tap[4];
      for (int i = 0; i < 4; ++i) tap[i] = ext_tap<TapT, Real, C>(img, W, H, cy + j, cx + i);
#pragma unroll
      for (int k = 0; k < C; ++k) {
        Real row = wx[0] * tap[0].v[k];
        row = fma(wx[1], tap[1].v[k], row);
        row = fma(wx[2], tap[2].v[k], row);
        row = fma(wx[3], tap[3].v[k], row);
        acc.v[k] = fma(wy[j], row, acc.v[k]);
      }
    }
  }
  return acc;
}

// Barycentric weights with numpy's operation order (densefield.py:99-107).
__device__ __forceinline__ void bary_rn(double2 a, double2 b, double2 c, double px, double py,
                                        double w[3]) {
  const double d = __dsub_rn(__dmul_rn(__dsub_rn(b.x, a.x), __dsub_rn(c.y, a.y)),
                             __dmul_rn(__dsub_rn(c.x, a.x), __dsub_rn(b.y, a.y)));
  const double n1 = __dsub_rn(__dmul_rn(__dsub_rn(b.x, px), __dsub_rn(c.y, py)),
                              __dmul_rn(__dsub_rn(c.x, px), __dsub_rn(b.y, py)));
  const double n2 = __dsub_rn(__dmul_rn(__dsub_rn(c.x, px), __dsub_rn(a.y, py)),
                              __dmul_rn(__dsub_rn(a.x, px), __dsub_rn(c.y, py)));
  w[0] = __ddiv_rn(n1, d);
  w[1] = __ddiv_rn(n2, d);
  w[2] = __dsub_rn(__dsub_rn(1.0, w[0]), w[1]);
}

// ---- deterministic block reductions (fixed shuffle tree + ordered warp sum)
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NT / 32; ++k) s += sh[k];
  }
  __syncthreads();
  return s;  // valid in thread 0
}

template <int NT>
__device__ __forceinline__ double2 block_sum2(double2 v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_down_sync(0xffffffffu, v.x, o);
    v.y += __shfl_down_sync(0xffffffffu, v.y, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sh[2 * w] = v.x;
    sh[2 * w + 1] = v.y;
  }
  __syncthreads();
  double2 s = make_double2(0.0, 0.0);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NT / 32; ++k) {
      s.x += sh[2 * k];
      s.y += sh[2 * k + 1];
    }
  }
  __syncthreads();
  return s;
}

// ---- per-pair device descriptor ------------------------------------------
template <typename TapT, typename Real>
struct PairDev {
  using R2 = typename V2<Real>::type;
  // mesh (node-relabelled, read-only)
  const double2* V;
  const int* nb_ptr;
  const int* nb_idx;
  const R2* g_self;
  const R2* g_nb;
  const Real* inv_val;
  const int4* tri;
  const int* tri_of;
  const int* perm;
  // images: interleaved (Te, Re)
  const TapT* img;
  // iteration state
  R2* u;
  Real* ste;
  Real* r;
  R2* ua;
  R2* ub;
  double* trace;
  R2* grad_out;  // optional (energy_gradient / vertex_gradient_all)
  // outputs
  Real* ux;
  Real* uy;
  Real* warped;
  double2* u_out;  // reference vertex order
  int W, H, n;
  int blk_begin, nblk, pix_blk_begin, pix_nblk, pad;
};

// ---- the divergence / tolerance logic of solver.py:176-195 --------------
__device__ __forceinline__ void control_step(PairStatus& s, double* trace, int k, double e,
                                             double tol) {
  if (!isfinite(e)) {  // solver.py:176-177
    s.err = ERR_NONFINITE_ENERGY;
    s.err_iter = k;
    trace[k] = e;
    s.stop_iter = k;
    return;
  }
  if (k > 0) {
    const double prev = trace[k - 1];
    // material_rise: e > prev * (1 + 1e-4) + 1e-12   (solver.py:43-44)
    const double thr = __dadd_rn(__dmul_rn(prev, 1.0 + 1e-4), 1e-12);
    if (e > thr) {
      s.rises += 1;
      if (s.rises >= 10) {  // solver.py:180-184
        s.err = ERR_RISES;
        s.err_iter = k;
        trace[k] = e;
        s.stop_iter = k;
        return;
      }
    } else if (e <= prev) {
      s.rises = 0;
    }
  }
  trace[k] = e;
  s.iters = k + 1;
  if (k + 1 >= 6) {  // solver.py:192-195
    const double base = trace[k - 5];
    const double lhs = fabs(__dsub_rn(e, base));
    const double rhs = __dmul_rn(tol, fmax(fabs(base), 1e-12));
    if (lhs <= rhs) s.stop_iter = k + 1;
  }
}

template <typename TapT, typename Real>
__global__ void __launch_bounds__(kNodeBlock)
    k_sample(const PairDev<TapT, Real>* __restrict__ pairs, PairStatus* __restrict__ st,
             const int* __restrict__ blk_pair, double* __restrict__ partials, int k,
             double tol) {
  __shared__ double sh[2 * kNodeBlock / 32];
  __shared__ bool last;
  const int p = blk_pair[blockIdx.x];
  const PairDev<TapT, Real>& d = pairs[p];
  if (st[p].err || k >= st[p].stop_iter) return;
  const int lb = blockIdx.x - d.blk_begin;
  const int i = lb * kNodeBlock + threadIdx.x;
  double e2 = 0.0;
  if (i < d.n) {
    const double2 v = d.V[i];
    const auto ui = d.u[i];
    const Px<TapT, Real, 2> s =
        cr_sample<TapT, Real, 2>(d.img, d.W, d.H, v.x + double(ui.x), v.y + double(ui.y));
    const Real ri = s.v[0] - s.v[1];
    d.ste[i] = s.v[0];
    d.r[i] = ri;
    e2 = double(ri) * double(ri);
  }
  const double bs = block_sum<kNodeBlock>(e2, sh);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = bs;
    __threadfence();
    const unsigned t = atomicAdd(&st[p].ticket, 1u);
    last = (t == unsigned(d.nblk - 1));
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // fixed-order reduction of this pair's block partials
  double acc = 0.0;
  for (int b = threadIdx.x; b < d.nblk; b += kNodeBlock) acc += __ldcg(partials + d.blk_begin + b);
  const double tot = block_sum<kNodeBlock>(acc, sh);
  if (threadIdx.x == 0) {
    PairStatus s = st[p];
    s.ticket = 0;
    control_step(s, d.trace, k, 0.5 * tot, tol);
    st[p] = s;
  }
}

template <typename Real>
__device__ __forceinline__ typename V2<Real>::type clamp_domain(double ux, double uy, double2 v,
                                                              int W, int H) {
  // np.clip(u1, -V, [W-1, H-1] - V), solver.py:140-144
  const double x = fmin(fmax(ux, -v.x), (double(W) - 1.0) - v.x);
  const double y = fmin(fmax(uy, -v.y), (double(H) - 1.0) - v.y);
  typename V2<Real>::type o;
  o.x = Real(x);
  o.y = Real(y);
  return o;
}

template <typename TapT, typename Real>
__global__ void __launch_bounds__(kNodeBlock)
    k_grad(const PairDev<TapT, Real>* __restrict__ pairs, PairStatus* __restrict__ st,
           const int* __restrict__ blk_pair, int k, Real tau, int passes) {
  const int p = blk_pair[blockIdx.x];
  const PairDev<TapT, Real>& d = pairs[p];
  if (st[p].err || k >= st[p].stop_iter) return;
  const int i = (blockIdx.x - d.blk_begin) * kNodeBlock + threadIdx.x;
  if (i >= d.n) return;
  const Real si = d.ste[i];
  const auto gs = d.g_self[i];
  Real gx = gs.x * si, gy = gs.y * si;
  const int e0 = d.nb_ptr[i], e1 = d.nb_ptr[i + 1];
  for (int e = e0; e < e1; ++e) {
    const auto g = d.g_nb[e];
    const Real sj = d.ste[d.nb_idx[e]];
    gx = fma(g.x, sj, gx);
    gy = fma(g.y, sj, gy);
  }
  const Real ri = d.r[i];
  const Real dx = ri * gx, dy = ri * gy;  // solver.py:189
  if (d.grad_out) {
    typename V2<Real>::type go;
    go.x = dx;
    go.y = dy;
    d.grad_out[i] = go;
    return;
  }
  if (!isfinite(dx) || !isfinite(dy)) {  // solver.py:131-132
    if (atomicCAS(&st[p].err, 0, ERR_NONFINITE_GRAD) == 0) st[p].err_iter = k;
  }
  const auto ui = d.u[i];
  typename V2<Real>::type u0;
  u0.x = ui.x - tau * dx;  // solver.py:133
  u0.y = ui.y - tau * dy;
  if (passes == 0)
    d.u[i] = clamp_domain<Real>(double(u0.x), double(u0.y), d.V[i], d.W, d.H);
  else
    d.ua[i] = u0;
}

template <typename TapT, typename Real>
__global__ void __launch_bounds__(kNodeBlock)
    k_smooth(const PairDev<TapT, Real>* __restrict__ pairs, PairStatus* __restrict__ st,
             const int* __restrict__ blk_pair, int k, Real lam, int pass, int passes) {
  const int p = blk_pair[blockIdx.x];
  const PairDev<TapT, Real>& d = pairs[p];
  if (st[p].err || k >= st[p].stop_iter) return;
  const int i = (blockIdx.x - d.blk_begin) * kNodeBlock + threadIdx.x;
  if (i >= d.n) return;
  const auto* src = (pass & 1) ? d.ub : d.ua;
  const Real iv = d.inv_val[i];
  Real ax = Real(0), ay = Real(0);
  const int e0 = d.nb_ptr[i], e1 = d.nb_ptr[i + 1];
  for (int e = e0; e < e1; ++e) {  // (L @ u)_i, L_ij = 1/valence_i
    const auto uj = src[d.nb_idx[e]];
    ax = fma(iv, uj.x, ax);
    ay = fma(iv, uj.y, ay);
  }
  const auto s = src[i];
  const Real om = Real(1) - lam;
  typename V2<Real>::type o;  // (1 - lam) u + lam (L u), mesh.py:281
  o.x = om * s.x + lam * ax;
  o.y = om * s.y + lam * ay;
  if (pass == passes - 1)
    d.u[i] = clamp_domain<Real>(double(o.x), double(o.y), d.V[i], d.W, d.H);
  else
    ((pass & 1) ? d.ua : d.ub)[i] = o;
}

// densify + warp + MSD partials (densefield.py:130-199, image.py:181-186)
template <typename TapT, typename Real>
__global__ void __launch_bounds__(kPixBlock)
    k_dense(const PairDev<TapT, Real>* __restrict__ pairs, PairStatus* __restrict__ st,
            const int* __restrict__ blk_pair, double2* __restrict__ partials) {
  __shared__ double sh[2 * kPixBlock / 32];
  const int p = blk_pair[blockIdx.x];
  const PairDev<TapT, Real>& d = pairs[p];
  if (st[p].err) return;
  const int q = (blockIdx.x - d.pix_blk_begin) * kPixBlock + threadIdx.x;
  double2 acc = make_double2(0.0, 0.0);
  if (q < d.W * d.H) {
    const int y = q / d.W, x = q - y * d.W;
    const int t = __ldg(d.tri_of + q);
    const int4 tv = __ldg(d.tri + t);
    double w[3];
    bary_rn(d.V[tv.x], d.V[tv.y], d.V[tv.z], double(x), double(y), w);
    const auto ua = d.u[tv.x], ub = d.u[tv.y], uc = d.u[tv.z];
    // (w * u[T]).sum(axis=2): ((w1 ua + w2 ub) + w3 uc), densefield.py:184-187
    const double fx = __dadd_rn(__dadd_rn(__dmul_rn(w[0], double(ua.x)), __dmul_rn(w[1], double(ub.x))),
                                __dmul_rn(w[2], double(uc.x)));
    const double fy = __dadd_rn(__dadd_rn(__dmul_rn(w[0], double(ua.y)), __dmul_rn(w[1], double(ub.y))),
                                __dmul_rn(w[2], double(uc.y)));
    const Real rx = Real(fx), ry = Real(fy);
    d.ux[q] = rx;
    d.uy[q] = ry;
    const Px<TapT, Real, 2> s =
        cr_sample<TapT, Real, 2>(d.img, d.W, d.H, double(x) + double(rx), double(y) + double(ry));
    const Real wv = s.v[0];
    d.warped[q] = wv;
    const auto own = load_px<TapT, double, 2>(d.img, d.W, y, x);  // (Te, Re)
    const double d0 = own.v[0] - own.v[1];
    const double d1 = double(wv) - own.v[1];
    acc.x = d0 * d0;
    acc.y = d1 * d1;
    if (!isfinite(rx) || !isfinite(ry)) atomicOr(&st[p].dense_nonfinite, 1);
    if (!isfinite(wv)) atomicOr(&st[p].dense_nonfinite, 2);
  }
  const double2 bs = block_sum2<kPixBlock>(acc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = bs;
}

template <typename TapT, typename Real>
__global__ void __launch_bounds__(kPixBlock)
    k_msd_final(const PairDev<TapT, Real>* __restrict__ pairs, PairStatus* __restrict__ st,
                const double2* __restrict__ partials) {
  __shared__ double sh[2 * kPixBlock / 32];
  const int p = blockIdx.x;
  const PairDev<TapT, Real>& d = pairs[p];
  double2 acc = make_double2(0.0, 0.0);
  for (int b = threadIdx.x; b < d.pix_nblk; b += kPixBlock) {
    const double2 v = partials[d.pix_blk_begin + b];
    acc.x += v.x;
    acc.y += v.y;
  }
  const double2 tot = block_sum2<kPixBlock>(acc, sh);
  if (threadIdx.x == 0) {
    const double npx = double(d.W) * double(d.H);
    st[p].msd_before = tot.x / npx;
    st[p].msd_after = tot.y / npx;
  }
}

template <typename TapT, typename Real>
__global__ void k_unpermute(const PairDev<TapT, Real>* __restrict__ pairs,
                            const int* __restrict__ blk_pair) {
  const int p = blk_pair[blockIdx.x];
  const PairDev<TapT, Real>& d = pairs[p];
  const int i = (blockIdx.x - d.blk_begin) * kNodeBlock + threadIdx.x;
  if (i >= d.n) return;
  const auto ui = d.u[i];
  d.u_out[d.perm[i]] = make_double2(double(ui.x), double(ui.y));
}

// planar (Re, Te) -> interleaved (Te, Re) taps; also the reset of the state
template <typename InT, typename TapT>
__global__ void k_interleave(const InT* const* __restrict__ re, const InT* const* __restrict__ te,
                             TapT* const* __restrict__ dst, int npx) {
  const int p = blockIdx.y;
  const InT* r = re[p];
  const InT* t = te[p];
  typename V2<TapT>::type* o = reinterpret_cast<typename V2<TapT>::type*>(dst[p]);
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < npx; q += gridDim.x * blockDim.x) {
    typename V2<TapT>::type v;
    v.x = TapT(__ldg(t + q));
    v.y = TapT(__ldg(r + q));
    o[q] = v;
  }
}

__global__ void k_reset_status(PairStatus* st, int n_pairs, int max_iter) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pairs) return;
  PairStatus s{};
  s.stop_iter = max_iter;
  st[p] = s;
}

template <typename Real>
__global__ void k_zero_state(typename V2<Real>::type* u, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    typename V2<Real>::type z;
    z.x = Real(0);
    z.y = Real(0);
    u[i] = z;
  }
}

// ---- pixel -> triangle map (setup), densefield.py:148-174 ---------------
// one warp per triangle; lanes stride over the triangle's pixel bbox and keep
// the lowest triangle id per pixel (atomicMin == ascending-order
// assign-if-unassigned of the reference).
// kRasterLanes threads per triangle: four triangles per warp, so the
// per-triangle setup is shared by a quarter of a warp (a whole warp per
// triangle left most lanes idle: a mesher triangle covers ~20 candidate
// pixels).
constexpr int kRasterLanes = 8;

__device__ __forceinline__ void raster_triangle(const double2* __restrict__ V,
                                                const int4* __restrict__ tri, int t, int lane,
                                                int W, int H, int* __restrict__ tri_of) {
  const int4 tv = tri[t];
  const double2 a = V[tv.x], b = V[tv.y], c = V[tv.z];
  const double mnx = fmin(fmin(a.x, b.x), c.x), mxx = fmax(fmax(a.x, b.x), c.x);
  const double mny = fmin(fmin(a.y, b.y), c.y), mxy = fmax(fmax(a.y, b.y), c.y);
  const long long x0 = max((long long)ceil(__dsub_rn(mnx, 1e-9)), 0LL);
  const long long x1 = min((long long)floor(__dadd_rn(mxx, 1e-9)), (long long)W - 1);
  const long long y0 = max((long long)ceil(__dsub_rn(mny, 1e-9)), 0LL);
  const long long y1 = min((long long)floor(__dadd_rn(mxy, 1e-9)), (long long)H - 1);
  if (x1 < x0 || y1 < y0) return;
  // 32-bit bounding-box arithmetic (a 64-bit division per candidate pixel
  // dominated this kernel)
  const int bw = int(x1 - x0 + 1);
  const int cnt = bw * int(y1 - y0 + 1);
  // Classification by weights from one reciprocal (within a few ulp of the
  // exactly rounded quotients): a pixel clearly inside (all > 1e-7) or
  // clearly outside (one < -1e-7) of the reference's predicate min(w) >=
  // -1e-9 is decided without the two divisions; only the band in between
  // gets the exactly rounded weights (bary_rn, numpy's operation order).
  const double d = __dsub_rn(__dmul_rn(__dsub_rn(b.x, a.x), __dsub_rn(c.y, a.y)),
                             __dmul_rn(__dsub_rn(c.x, a.x), __dsub_rn(b.y, a.y)));
  const double inv = 1.0 / d;
  for (int q = lane; q < cnt; q += kRasterLanes) {
    const int qy = q / bw;
    const int py = int(y0) + qy, px = int(x0) + (q - qy * bw);
    const double fx = double(px), fy = double(py);
    const double n1 = __dsub_rn(__dmul_rn(__dsub_rn(b.x, fx), __dsub_rn(c.y, fy)),
                                __dmul_rn(__dsub_rn(c.x, fx), __dsub_rn(b.y, fy)));
    const double n2 = __dsub_rn(__dmul_rn(__dsub_rn(c.x, fx), __dsub_rn(a.y, fy)),
                                __dmul_rn(__dsub_rn(a.x, fx), __dsub_rn(c.y, fy)));
    const double w1 = n1 * inv, w2 = n2 * inv;
    const double mn = fmin(fmin(w1, w2), (1.0 - w1) - w2);
    bool inside = mn > 1e-7;
    if (!inside && mn >= -1e-7) {  // near an edge: the exact weights decide
      double w[3];
      bary_rn(a, b, c, fx, fy, w);
      inside = fmin(fmin(w[0], w[1]), w[2]) >= -1e-9;
    }
    if (inside) atomicMin(tri_of + size_t(py) * W + px, t);
  }
}

__global__ void k_raster(const double2* __restrict__ V, const int4* __restrict__ tri, int m,
                         int W, int H, int* __restrict__ tri_of) {
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) / kRasterLanes;
  if (t < m) raster_triangle(V, tri, t, threadIdx.x % kRasterLanes, W, H, tri_of);
}

// Many meshes in one launch (blockIdx.y = mesh): setup of a whole batch costs
// three launches instead of three per mesh.  The job table travels in the
// kernel parameters (kRasterJobs x 28 B).
constexpr int kRasterJobs = 128;
struct RasterJobs {
  const double2* V[kRasterJobs];
  const int4* tri[kRasterJobs];
  int* map[kRasterJobs];
  int m[kRasterJobs];
};

__global__ void k_raster_many(const RasterJobs jobs, int W, int H) {
  const int j = blockIdx.y;
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) / kRasterLanes;
  if (t < jobs.m[j])
    raster_triangle(jobs.V[j], jobs.tri[j], t, threadIdx.x % kRasterLanes, W, H, jobs.map[j]);
}

__global__ void k_count_uncovered(const int* __restrict__ tri_of, int npx,
                                  unsigned long long* __restrict__ count) {
  int local = 0;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < npx; q += gridDim.x * blockDim.x)
    local += (tri_of[q] == kUnassigned);
  for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(count, (unsigned long long)local);
}

__global__ void k_count_uncovered_many(const RasterJobs jobs, int npx,
                                       unsigned long long* __restrict__ count) {
  const int* tri_of = jobs.map[blockIdx.y];
  int local = 0;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < npx; q += gridDim.x * blockDim.x)
    local += (tri_of[q] == kUnassigned);
  for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(count + blockIdx.y, (unsigned long long)local);
}

__global__ void k_pixel_weights(const double2* __restrict__ V, const int4* __restrict__ tri,
                                const int* __restrict__ tri_of, int W, int npx,
                                double* __restrict__ w_out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= npx) return;
  const int y = q / W, x = q - y * W;
  const int4 tv = tri[tri_of[q]];
  double w[3];
  bary_rn(V[tv.x], V[tv.y], V[tv.z], double(x), double(y), w);
  w_out[3 * q] = w[0];
  w_out[3 * q + 1] = w[1];
  w_out[3 * q + 2] = w[2];
}

// ---- single-operation kernels (f64, reference vertex order) --------------
template <typename TapT>
__global__ void k_sample_points(const TapT* __restrict__ img, int W, int H, int n,
                                const double* __restrict__ V, const double* __restrict__ u,
                                double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = V[2 * i] + u[2 * i], y = V[2 * i + 1] + u[2 * i + 1];
  out[i] = cr_sample<TapT, double, 1>(img, W, H, x, y).v[0];
}

template <typename TapT>
__global__ void k_warp_image(const TapT* __restrict__ img, int W, int H,
                             const double* __restrict__ ux, const double* __restrict__ uy,
                             double* __restrict__ out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= W * H) return;
  const int y = q / W, x = q - y * W;
  out[q] = cr_sample<TapT, double, 1>(img, W, H, double(x) + ux[q], double(y) + uy[q]).v[0];
}

__global__ void k_densify(const double2* __restrict__ V, const int4* __restrict__ tri,
                          const int* __restrict__ tri_of, const double2* __restrict__ u, int W,
                          int npx, double* __restrict__ ux, double* __restrict__ uy) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= npx) return;
  const int y = q / W, x = q - y * W;
  const int4 tv = tri[tri_of[q]];
  double w[3];
  bary_rn(V[tv.x], V[tv.y], V[tv.z], double(x), double(y), w);
  const double2 a = u[tv.x], b = u[tv.y], c = u[tv.z];
  ux[q] = __dadd_rn(__dadd_rn(__dmul_rn(w[0], a.x), __dmul_rn(w[1], b.x)), __dmul_rn(w[2], c.x));
  uy[q] = __dadd_rn(__dadd_rn(__dmul_rn(w[0], a.y), __dmul_rn(w[1], b.y)), __dmul_rn(w[2], c.y));
}

// generic CSR smoothing / step on reference-order data (mesh.py:268-282)
__global__ void k_csr_smooth(int n, const int64_t* __restrict__ indptr,
                             const int64_t* __restrict__ indices, const double* __restrict__ data,
                             const double2* __restrict__ src, double lam,
                             double2* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double ax = 0.0, ay = 0.0;
  for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
    const double2 v = src[indices[e]];
    ax = __dadd_rn(ax, __dmul_rn(data[e], v.x));
    ay = __dadd_rn(ay, __dmul_rn(data[e], v.y));
  }
  const double om = 1.0 - lam;
  const double2 s = src[i];
  dst[i] = make_double2(__dadd_rn(__dmul_rn(om, s.x), __dmul_rn(lam, ax)),
                        __dadd_rn(__dmul_rn(om, s.y), __dmul_rn(lam, ay)));
}

__global__ void k_descent(int n, const double2* __restrict__ u, const double2* __restrict__ g,
                          double tau, double2* __restrict__ out, int* __restrict__ nonfinite) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 gi = g[i], ui = u[i];
  if (!isfinite(gi.x) || !isfinite(gi.y)) *nonfinite = 1;
  out[i] = make_double2(__dsub_rn(ui.x, __dmul_rn(tau, gi.x)), __dsub_rn(ui.y, __dmul_rn(tau, gi.y)));
}

__global__ void k_clamp(int n, const double2* __restrict__ V, int W, int H, double2* __restrict__ u) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 v = V[i], x = u[i];
  u[i] = make_double2(fmin(fmax(x.x, -v.x), __dsub_rn(double(W) - 1.0, v.x)),
                      fmin(fmax(x.y, -v.y), __dsub_rn(double(H) - 1.0, v.y)));
}

// msd partials with the same block partition / reduction tree as k_dense, so
// msd(warp_image(densify(u)), re) reproduces register's msd_after exactly
__global__ void __launch_bounds__(kPixBlock)
    k_sqdiff_partials(int n, const double* __restrict__ a, const double* __restrict__ b,
                      double* __restrict__ partials) {
  __shared__ double sh[2 * kPixBlock / 32];
  const int q = blockIdx.x * kPixBlock + threadIdx.x;
  double acc = 0.0;
  if (q < n) {
    const double dd = a[q] - b[q];
    acc = dd * dd;
  }
  const double s = block_sum<kPixBlock>(acc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kPixBlock)
    k_sum_final(int nb, const double* __restrict__ partials, double denom,
                double* __restrict__ out) {
  __shared__ double sh[2 * kPixBlock / 32];
  double acc = 0.0;
  for (int b = threadIdx.x; b < nb; b += kPixBlock) acc += partials[b];
  const double s = block_sum<kPixBlock>(acc, sh);
  if (threadIdx.x == 0) *out = s / denom;
}

}  // namespace mrb
