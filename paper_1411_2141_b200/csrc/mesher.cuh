// Content-adaptive mesher (reference meshgen.py / delaunay.py; SURVEY.md
// §8(f) rows 3-4).  Part of the meshreg_b200.cu translation unit (included at
// its end) so it shares the allocator, copy wrappers and error helpers.
//
// Image-space front end on the GPU, bit-exact with the reference's numpy /
// scipy arithmetic:
//   k_gauss_axis<0|1>   scipy.ndimage.gaussian_filter(mode="nearest"): one
//                       correlate1d per axis, axis 0 first, symmetric taps
//                       accumulated x[0]*w0 + (x[-r]+x[r])*w_r + ... + (x[-1]+x[1])*w_1
//                       (scipy's NI_Correlate1D order), no FMA contraction
//   k_grad_mag          np.gradient (central / one-sided differences),
//                       np.hypot as glibc computes it, Canny sector
//   k_nms               4-direction thinning, weak / strong thresholds
//   k_uf_*              hysteresis: ndimage.label(8-connectivity) + "label
//                       holds a strong pixel" as a lock-free union-find
// Sequential stages (Floyd-Steinberg, spacing thinning, Bowyer-Watson, flips,
// CVT/ODT relaxation) are in mesher_host.cpp.
#pragma once

#include "mesher_host.h"

namespace {

constexpr int kMeshBlock = 256;

// glibc hypot (sysdeps/ieee754/dbl-64/e_hypot.c), every operation rounded
// separately so nvcc cannot contract it into FMAs.
__device__ __forceinline__ double d_hypot_kernel(double ax, double ay) {
  double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
  double t1, t2;
  if (h <= __dmul_rn(2.0, ay)) {
    const double delta = __dsub_rn(h, ay);
    t1 = __dmul_rn(ax, __dsub_rn(__dmul_rn(2.0, delta), ax));
    t2 = __dmul_rn(__dsub_rn(delta, __dmul_rn(2.0, __dsub_rn(ax, ay))), delta);
  } else {
    const double delta = __dsub_rn(h, ax);
    t1 = __dmul_rn(__dmul_rn(2.0, delta), __dsub_rn(ax, __dmul_rn(2.0, ay)));
    t2 = __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(4.0, delta), ay), ay), __dmul_rn(delta, delta));
  }
  return __dsub_rn(h, __ddiv_rn(__dadd_rn(t1, t2), __dmul_rn(2.0, h)));
}

__device__ double d_glibc_hypot(double x, double y) {
  if (!isfinite(x) || !isfinite(y)) {
    if (isinf(x) || isinf(y)) return __longlong_as_double(0x7ff0000000000000LL);
    return __dadd_rn(x, y);
  }
  x = fabs(x);
  y = fabs(y);
  const double ax = x < y ? y : x, ay = x < y ? x : y;
  if (ax > 0x1p+511) {
    if (ay <= __dmul_rn(ax, 0x1p-54)) return __dadd_rn(ax, ay);
    return __ddiv_rn(d_hypot_kernel(__dmul_rn(ax, 0x1p-600), __dmul_rn(ay, 0x1p-600)), 0x1p-600);
  }
  if (ay < 0x1p-511) {
    if (ax >= __ddiv_rn(ay, 0x1p-54)) return __dadd_rn(ax, ay);
    return __dmul_rn(d_hypot_kernel(__ddiv_rn(ax, 0x1p-600), __ddiv_rn(ay, 0x1p-600)), 0x1p-600);
  }
  if (ay <= __dmul_rn(ax, 0x1p-54)) return __dadd_rn(ax, ay);
  return d_hypot_kernel(ax, ay);
}

// One correlate1d pass with mode="nearest".  AXIS 0 runs along y (rows),
// AXIS 1 along x.  w[0..r]: w[0] centre tap, w[j] the tap at distance j.
template <int AXIS>
__global__ void __launch_bounds__(kMeshBlock) k_gauss_axis(int W, int H, const double* __restrict__ in,
                                                           double* __restrict__ out, int r,
                                                           const double* __restrict__ w) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= int64_t(W) * H) return;
  const int y = int(i / W), x = int(i - int64_t(y) * W);
  const int n = AXIS == 0 ? H : W;
  const int c = AXIS == 0 ? y : x;
  auto at = [&](int k) {
    k = k < 0 ? 0 : (k >= n ? n - 1 : k);
    return AXIS == 0 ? __ldg(in + int64_t(k) * W + x) : __ldg(in + int64_t(y) * W + k);
  };
  double acc = __dmul_rn(at(c), w[0]);
  for (int j = r; j >= 1; --j) acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(at(c - j), at(c + j)), w[j]));
  out[i] = acc;
}

// np.gradient (unit spacing, edge_order 1) of the smoothed image, np.hypot,
// and the Canny sector floor((mod(atan2(gy, gx), pi) + pi/8) / (pi/4)) % 4
// (meshgen.py:99-118).
__global__ void __launch_bounds__(kMeshBlock) k_grad_mag(int W, int H, const double* __restrict__ sm,
                                                         double* __restrict__ mag,
                                                         uint8_t* __restrict__ sector) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= int64_t(W) * H) return;
  const int y = int(i / W), x = int(i - int64_t(y) * W);
  auto f = [&](int yy, int xx) { return __ldg(sm + int64_t(yy) * W + xx); };
  double gy, gx;
  if (y == 0) gy = __dsub_rn(f(1, x), f(0, x));
  else if (y == H - 1) gy = __dsub_rn(f(H - 1, x), f(H - 2, x));
  else gy = __ddiv_rn(__dsub_rn(f(y + 1, x), f(y - 1, x)), 2.0);
  if (x == 0) gx = __dsub_rn(f(y, 1), f(y, 0));
  else if (x == W - 1) gx = __dsub_rn(f(y, W - 1), f(y, W - 2));
  else gx = __ddiv_rn(__dsub_rn(f(y, x + 1), f(y, x - 1)), 2.0);
  mag[i] = d_glibc_hypot(gx, gy);
  if (sector) {
    const double pi = 3.141592653589793;
    double a = atan2(gy, gx);
    double md = fmod(a, pi);  // npy_divmod's remainder
    if (md != 0.0) {
      if ((pi < 0) != (md < 0)) md = __dadd_rn(md, pi);
    } else {
      md = copysign(0.0, pi);
    }
    const double s = floor(__ddiv_rn(__dadd_rn(md, pi / 8), pi / 4));
    int si = int(s) % 4;
    if (si < 0) si += 4;
    sector[i] = uint8_t(si);
  }
}

// Non-maximum suppression against the two sector neighbours (out of image:
// -1, the reference's padding) and the hysteresis thresholds.  state: 0 none,
// 1 weak, 3 weak + strong.
__global__ void __launch_bounds__(kMeshBlock) k_nms(int W, int H, const double* __restrict__ mag,
                                                    const uint8_t* __restrict__ sector, double low,
                                                    double high, uint8_t* __restrict__ state) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= int64_t(W) * H) return;
  const int y = int(i / W), x = int(i - int64_t(y) * W);
  // pairs (meshgen.py:115): 0: (0,1),(0,-1)  1: (1,1),(-1,-1)  2: (1,0),(-1,0)  3: (1,-1),(-1,1)
  const int dy[4] = {0, 1, 1, 1}, dx[4] = {1, 1, 0, -1};
  const int s = sector[i];
  auto m = [&](int yy, int xx) {
    return (yy < 0 || yy >= H || xx < 0 || xx >= W) ? -1.0 : __ldg(mag + int64_t(yy) * W + xx);
  };
  const double v = mag[i];
  const bool keep = v >= m(y + dy[s], x + dx[s]) && v >= m(y - dy[s], x - dx[s]);
  uint8_t st = 0;
  if (keep && v >= low) st = 1;
  if (keep && v >= high) st = 3;
  state[i] = st;
}

__device__ __forceinline__ int uf_find(const int* p, int x) {
  int y;
  while ((y = __ldcg(p + x)) != x) x = y;
  return x;
}

__device__ void uf_union(int* p, int a, int b) {
  while (true) {
    a = uf_find(p, a);
    b = uf_find(p, b);
    if (a == b) return;
    if (a < b) {
      const int t = a;
      a = b;
      b = t;
    }
    const int old = atomicCAS(p + a, a, b);
    if (old == a) return;
    a = old;
  }
}

__global__ void __launch_bounds__(kMeshBlock) k_uf_init(int n, const uint8_t* __restrict__ state,
                                                        int* __restrict__ parent) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) parent[i] = state[i] ? i : -1;
}

// 8-connectivity (structure = ones((3, 3))): link to the four earlier neighbours
__global__ void __launch_bounds__(kMeshBlock) k_uf_merge(int W, int H, const uint8_t* __restrict__ state,
                                                         int* parent) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= W * H || !state[i]) return;
  const int y = i / W, x = i - y * W;
  const int ny[4] = {y - 1, y - 1, y - 1, y}, nx[4] = {x - 1, x, x + 1, x - 1};
  for (int k = 0; k < 4; ++k) {
    if (ny[k] < 0 || nx[k] < 0 || nx[k] >= W) continue;
    const int j = ny[k] * W + nx[k];
    if (state[j]) uf_union(parent, i, j);
  }
}

__global__ void __launch_bounds__(kMeshBlock) k_uf_strong(int n, const uint8_t* __restrict__ state,
                                                          const int* parent, int* __restrict__ good) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && state[i] == 3) good[uf_find(parent, i)] = 1;
}

__global__ void __launch_bounds__(kMeshBlock) k_uf_edges(int n, const uint8_t* __restrict__ state,
                                                         const int* parent, const int* __restrict__ good,
                                                         uint8_t* __restrict__ edges) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) edges[i] = state[i] ? uint8_t(good[uf_find(parent, i)] != 0) : uint8_t(0);
}

// circumcircles (delaunay.py:54-72) with numpy's rounding (no contraction).
__device__ void d_circumcircle(double2 a, double2 b, double2 c, double& cx, double& cy,
                               double& r2) {
  const double ab0 = __dsub_rn(b.x, a.x), ab1 = __dsub_rn(b.y, a.y);
  const double ac0 = __dsub_rn(c.x, a.x), ac1 = __dsub_rn(c.y, a.y);
  const double d = __dmul_rn(2.0, __dsub_rn(__dmul_rn(ab0, ac1), __dmul_rn(ab1, ac0)));
  const double ab2 = __dadd_rn(__dmul_rn(ab0, ab0), __dmul_rn(ab1, ab1));
  const double ac2 = __dadd_rn(__dmul_rn(ac0, ac0), __dmul_rn(ac1, ac1));
  const double ux = __ddiv_rn(__dsub_rn(__dmul_rn(ac1, ab2), __dmul_rn(ab1, ac2)), d);
  const double uy = __ddiv_rn(__dsub_rn(__dmul_rn(ab0, ac2), __dmul_rn(ac0, ab2)), d);
  if (!isfinite(ux) || !isfinite(uy)) {
    cx = a.x;
    cy = a.y;
    r2 = __longlong_as_double(0x7ff0000000000000LL);
    return;
  }
  r2 = __dadd_rn(__dmul_rn(ux, ux), __dmul_rn(uy, uy));
  cx = __dadd_rn(a.x, ux);
  cy = __dadd_rn(a.y, uy);
}

// delaunay_violations (delaunay.py:290-309): (triangle, vertex) pairs with
// hypot(v - c) < sqrt(max(r2, 0)) - margin, own corners excluded.  One
// thread per triangle, vertices streamed through shared memory; a squared-
// distance test with a 1e-9 relative band settles all but near-boundary
// pairs, which take the exact glibc-hypot comparison.
constexpr int kViolTile = 1024;
__global__ void __launch_bounds__(kMeshBlock) k_delaunay_violations(
    int64_t n, const double2* __restrict__ V, int64_t m, const int64_t* __restrict__ T,
    double margin, unsigned long long* __restrict__ total) {
  __shared__ double2 tile[kViolTile];
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  double cx = 0, cy = 0, thr = -1, thr2 = 0;
  int64_t c0 = -1, c1 = -1, c2 = -1;
  if (t < m) {
    c0 = T[3 * t], c1 = T[3 * t + 1], c2 = T[3 * t + 2];
    double r2;
    d_circumcircle(V[c0], V[c1], V[c2], cx, cy, r2);
    thr = __dsub_rn(__dsqrt_rn(fmax(r2, 0.0)), margin);
    thr2 = thr * thr;
  }
  unsigned long long cnt = 0;
  for (int64_t base = 0; base < n; base += kViolTile) {
    const int64_t len = (n - base) < kViolTile ? (n - base) : int64_t(kViolTile);
    __syncthreads();
    for (int k = threadIdx.x; k < len; k += blockDim.x) tile[k] = V[base + k];
    __syncthreads();
    if (thr <= 0) continue;
    for (int k = 0; k < len; ++k) {
      const double dx = __dsub_rn(tile[k].x, cx), dy = __dsub_rn(tile[k].y, cy);
      const double d2 = dx * dx + dy * dy;
      bool inside;
      if (d2 > thr2 * (1 + 1e-9)) inside = false;
      else if (d2 < thr2 * (1 - 1e-9)) inside = true;
      else inside = d_glibc_hypot(dx, dy) < thr;
      if (inside) {
        const int64_t v = base + k;
        if (v != c0 && v != c1 && v != c2) ++cnt;
      }
    }
  }
  if (cnt) atomicAdd(total, cnt);
}

inline unsigned mesh_blocks(int64_t n) { return unsigned((n + kMeshBlock - 1) / kMeshBlock); }

// Gaussian (both axes) + gradient magnitude (+ sector) into device buffers.
void run_grad_mag(cudaStream_t s, Tmp& t, int W, int H, const double* d_img, int r,
                  const double* h_w, double* d_mag, uint8_t* d_sector) {
  const int64_t n = int64_t(W) * H;
  // taps w[0] (centre) .. w[r]; the caller passes the full 2r+1 kernel
  std::vector<double> half(size_t(r) + 1);
  for (int j = 0; j <= r; ++j) half[j] = h_w[r + j];
  const double* d_w = t.up(half.data(), half.size());
  double* tmp = t.get<double>(size_t(n));
  double* sm = t.get<double>(size_t(n));
  k_gauss_axis<0><<<mesh_blocks(n), kMeshBlock, 0, s>>>(W, H, d_img, tmp, r, d_w);
  k_gauss_axis<1><<<mesh_blocks(n), kMeshBlock, 0, s>>>(W, H, tmp, sm, r, d_w);
  k_grad_mag<<<mesh_blocks(n), kMeshBlock, 0, s>>>(W, H, sm, d_mag, d_sector);
  ck(cudaGetLastError());
}

std::string check_taps(int W, int H, int r, const double* w) {
  if (W < 2 || H < 2) return "gradient needs an image of at least 2x2 pixels";
  if (r < 0 || !w) return "gaussian taps missing";
  for (int j = 0; j < r; ++j)
    if (w[j] != w[2 * r - j]) return "gaussian taps must be symmetric";
  return "";
}

void run_canny(cudaStream_t s, Tmp& t, int W, int H, const double* d_img, int r, const double* h_w,
               double low, double high, double* d_mag, uint8_t* d_edges) {
  const int n = W * H;
  uint8_t* sector = t.get<uint8_t>(size_t(n));
  uint8_t* state = t.get<uint8_t>(size_t(n));
  int* parent = t.get<int>(size_t(n));
  int* good = t.get<int>(size_t(n));
  run_grad_mag(s, t, W, H, d_img, r, h_w, d_mag, sector);
  k_nms<<<mesh_blocks(n), kMeshBlock, 0, s>>>(W, H, d_mag, sector, low, high, state);
  k_uf_init<<<mesh_blocks(n), kMeshBlock, 0, s>>>(n, state, parent);
  k_uf_merge<<<mesh_blocks(n), kMeshBlock, 0, s>>>(W, H, state, parent);
  ck(cudaMemsetAsync(good, 0, sizeof(int) * size_t(n), s));
  k_uf_strong<<<mesh_blocks(n), kMeshBlock, 0, s>>>(n, state, parent, good);
  k_uf_edges<<<mesh_blocks(n), kMeshBlock, 0, s>>>(n, state, parent, good, d_edges);
  ck(cudaGetLastError());
}

void put_err(const std::string& msg, char* err, int32_t err_len) {
  if (err && err_len > 0) {
    std::strncpy(err, msg.c_str(), size_t(err_len) - 1);
    err[err_len - 1] = 0;
  }
}

}  // namespace

struct mrb_tris {
  mrb::Tris t;
};

extern "C" {

int mrb_gradient_magnitude(mrb_ctx* ctx, int32_t width, int32_t height, const double* image,
                           int32_t radius, const double* taps, double* mag) {
  if (!ctx || !image || !mag) return MRB_E_VALUE;
  const std::string e = check_taps(width, height, radius, taps);
  if (!e.empty()) return fail(ctx, MRB_E_VALUE, e);
  if (int64_t(width) * height >= (int64_t(1) << 31))
    return fail(ctx, MRB_E_VALUE, "image too large for 32-bit pixel indexing");
  try {
    ck(cudaSetDevice(ctx->device));
    Tmp t(ctx->stream);
    const size_t n = size_t(width) * height;
    const double* d_img = t.up(image, n);
    double* d_mag = t.get<double>(n);
    run_grad_mag(ctx->stream, t, width, height, d_img, radius, taps, d_mag, nullptr);
    ck(mrb_copy_async(mag, d_mag, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ck(cudaStreamSynchronize(ctx->stream));
  } catch (const CudaError& ce) {
    return cuda_fail(ctx, ce.e);
  }
  return MRB_OK;
}

int mrb_canny_edges(mrb_ctx* ctx, int32_t width, int32_t height, const double* image,
                    int32_t radius, const double* taps, double low, double high, uint8_t* edges,
                    double* mag) {
  if (!ctx || !image || !edges) return MRB_E_VALUE;
  const std::string e = check_taps(width, height, radius, taps);
  if (!e.empty()) return fail(ctx, MRB_E_VALUE, e);
  if (int64_t(width) * height >= (int64_t(1) << 31))
    return fail(ctx, MRB_E_VALUE, "image too large for 32-bit pixel indexing");
  try {
    ck(cudaSetDevice(ctx->device));
    Tmp t(ctx->stream);
    const size_t n = size_t(width) * height;
    const double* d_img = t.up(image, n);
    double* d_mag = t.get<double>(n);
    uint8_t* d_edges = t.get<uint8_t>(n);
    run_canny(ctx->stream, t, width, height, d_img, radius, taps, low, high, d_mag, d_edges);
    ck(mrb_copy_async(edges, d_edges, n, cudaMemcpyDeviceToHost, ctx->stream));
    if (mag) ck(mrb_copy_async(mag, d_mag, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ck(cudaStreamSynchronize(ctx->stream));
  } catch (const CudaError& ce) {
    return cuda_fail(ctx, ce.e);
  }
  return MRB_OK;
}

int mrb_canny_sample(mrb_ctx* ctx, int32_t width, int32_t height, const double* image,
                     int32_t radius, const double* taps, double low, double high, double spacing,
                     int64_t budget, double* points, int64_t* count) {
  if (!ctx || !image || !count) return MRB_E_VALUE;
  *count = 0;
  if (budget <= 0) return MRB_OK;
  if (!points) return MRB_E_VALUE;
  const size_t n = size_t(width) * height;
  std::vector<uint8_t> edges(n);
  std::vector<double> mag(n);
  const int rc = mrb_canny_edges(ctx, width, height, image, radius, taps, low, high, edges.data(),
                                 mag.data());
  if (rc != MRB_OK) return rc;
  // lexsort((xs, ys, -mag)): strongest first, then row-major
  std::vector<int64_t> idx;
  for (size_t i = 0; i < n; ++i)
    if (edges[i]) idx.push_back(int64_t(i));
  if (idx.empty()) return MRB_OK;
  std::stable_sort(idx.begin(), idx.end(),
                   [&](int64_t a, int64_t b) { return -mag[size_t(a)] < -mag[size_t(b)]; });
  std::vector<double> xy(2 * idx.size());
  for (size_t k = 0; k < idx.size(); ++k) {
    xy[2 * k] = double(idx[k] % width);
    xy[2 * k + 1] = double(idx[k] / width);
  }
  std::vector<double> out;
  mrb::spacing_thin(xy.data(), int64_t(idx.size()), nullptr, spacing, budget, out);
  std::copy(out.begin(), out.end(), points);
  *count = int64_t(out.size() / 2);
  return MRB_OK;
}

int mrb_halftone_dots(int32_t width, int32_t height, const double* mag, int64_t budget,
                      int32_t serpentine_start, uint8_t* dots, double* total) {
  if (!mag || !dots || width < 1 || height < 1) return MRB_E_VALUE;
  const double tot = mrb::np_pairwise_sum(mag, int64_t(width) * height);
  if (total) *total = tot;
  if (tot <= 1e-12) {
    std::memset(dots, 0, size_t(width) * height);
    return MRB_OK;
  }
  mrb::floyd_steinberg(mag, double(budget) / tot, width, height, serpentine_start, dots);
  return MRB_OK;
}

int mrb_floyd_steinberg(int32_t width, int32_t height, const double* density,
                        int32_t serpentine_start, uint8_t* dots) {
  if (!density || !dots || width < 1 || height < 1) return MRB_E_VALUE;
  mrb::floyd_steinberg(density, 1.0, width, height, serpentine_start, dots);
  return MRB_OK;
}

int mrb_spacing_thin(int64_t n, const double* xy, const int64_t* order, double spacing,
                     int64_t budget, double* out, int64_t* count) {
  if (!count || (n > 0 && !xy) || (budget > 0 && !out)) return MRB_E_VALUE;
  std::vector<double> kept;
  if (budget > 0) mrb::spacing_thin(xy, n, order, spacing, budget, kept);
  std::copy(kept.begin(), kept.end(), out);
  *count = int64_t(kept.size() / 2);
  return MRB_OK;
}

int mrb_uniform_sample(int32_t width, int32_t height, int64_t budget, double* out, int64_t cap,
                       int64_t* count, char* err, int32_t err_len) {
  if (!count) return MRB_E_VALUE;
  std::vector<double> pts;
  const std::string e = mrb::uniform_sample(width, height, budget, pts);
  if (!e.empty()) {
    put_err(e, err, err_len);
    return MRB_E_VALUE;
  }
  *count = int64_t(pts.size() / 2);
  if (*count > cap || !out) return MRB_E_VALUE;
  std::copy(pts.begin(), pts.end(), out);
  return MRB_OK;
}

int mrb_dedupe_points(int64_t n, const double* points, double tol, double* out, int64_t* count,
                      char* err, int32_t err_len) {
  if (!count || (n > 0 && (!points || !out))) return MRB_E_VALUE;
  std::vector<double> P;
  const std::string e = mrb::dedupe_points(points, n, tol, P);
  if (!e.empty()) {
    put_err(e, err, err_len);
    return MRB_E_VALUE;
  }
  std::copy(P.begin(), P.end(), out);
  *count = int64_t(P.size() / 2);
  return MRB_OK;
}

int mrb_tris_create(int64_t n_vertices, const double* vertices, int64_t n_triangles,
                    const int64_t* triangles, mrb_tris** out, char* err, int32_t err_len) {
  if (!out || n_vertices < 0 || n_triangles < 0) return MRB_E_VALUE;
  *out = nullptr;
  auto* m = new mrb_tris();
  m->t.V.assign(vertices, vertices + 2 * n_vertices);
  m->t.T.assign(triangles, triangles + 3 * n_triangles);
  const std::string e = mrb::trimesh_init(m->t);
  if (!e.empty()) {
    put_err(e, err, err_len);
    delete m;
    return MRB_E_VALUE;
  }
  *out = m;
  return MRB_OK;
}

int mrb_delaunay(int64_t n, const double* points, mrb_tris** out, char* err, int32_t err_len) {
  if (!out || (n > 0 && !points)) return MRB_E_VALUE;
  *out = nullptr;
  auto* m = new mrb_tris();
  int kind = 1;
  std::string e;
  try {
    e = mrb::delaunay(points, n, m->t, kind);
  } catch (const std::exception& ex) {
    e = std::string("internal error: ") + ex.what();
    kind = 2;
  }
  if (!e.empty()) {
    put_err(e, err, err_len);
    delete m;
    return kind == 2 ? MRB_E_INTERNAL : MRB_E_VALUE;
  }
  *out = m;
  return MRB_OK;
}

int mrb_flip_edges(mrb_tris* mesh, int32_t passes, int32_t* changed, char* err, int32_t err_len) {
  if (!mesh) return MRB_E_VALUE;
  std::string e;
  const int c = mrb::flip_edges(mesh->t, passes, e);
  if (changed) *changed = c;
  if (!e.empty()) {
    put_err(e, err, err_len);
    return MRB_E_VALUE;
  }
  return MRB_OK;
}

int mrb_smooth_mesh(mrb_tris* mesh, int32_t width, int32_t height, const double* mag,
                    int32_t cvt_iterations, int32_t odt_iterations, char* err, int32_t err_len) {
  if (!mesh || !mag || width < 1 || height < 1) return MRB_E_VALUE;
  const std::string e =
      mrb::smooth_mesh(mesh->t, width, height, mag, cvt_iterations, odt_iterations);
  if (!e.empty()) {
    put_err(e, err, err_len);
    return MRB_E_VALUE;
  }
  return MRB_OK;
}

int mrb_tris_counts(const mrb_tris* mesh, int64_t* n_vertices, int64_t* n_triangles) {
  if (!mesh) return MRB_E_VALUE;
  if (n_vertices) *n_vertices = mesh->t.n();
  if (n_triangles) *n_triangles = mesh->t.m();
  return MRB_OK;
}

int mrb_tris_export(const mrb_tris* mesh, double* vertices, int64_t* triangles) {
  if (!mesh) return MRB_E_VALUE;
  if (vertices) std::copy(mesh->t.V.begin(), mesh->t.V.end(), vertices);
  if (triangles) std::copy(mesh->t.T.begin(), mesh->t.T.end(), triangles);
  return MRB_OK;
}

int mrb_delaunay_violations(mrb_ctx* ctx, int64_t n_vertices, const double* vertices,
                            int64_t n_triangles, const int64_t* triangles, double margin,
                            int64_t* count) {
  if (!ctx || !count || n_vertices < 0 || n_triangles < 0) return MRB_E_VALUE;
  *count = 0;
  for (int64_t k = 0; k < 3 * n_triangles; ++k)
    if (triangles[k] < 0 || triangles[k] >= n_vertices)
      return fail(ctx, MRB_E_VALUE, "triangle index out of range");
  if (n_triangles == 0 || n_vertices == 0) return MRB_OK;
  try {
    ck(cudaSetDevice(ctx->device));
    Tmp t(ctx->stream);
    const double2* dV = reinterpret_cast<const double2*>(t.up(vertices, size_t(2 * n_vertices)));
    const int64_t* dT = t.up(triangles, size_t(3 * n_triangles));
    unsigned long long* dtot = t.get<unsigned long long>(1);
    ck(cudaMemsetAsync(dtot, 0, sizeof(unsigned long long), ctx->stream));
    k_delaunay_violations<<<mesh_blocks(n_triangles), kMeshBlock, 0, ctx->stream>>>(
        n_vertices, dV, n_triangles, dT, margin, dtot);
    ck(cudaGetLastError());
    unsigned long long h = 0;
    ck(mrb_copy_async(&h, dtot, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    ck(cudaStreamSynchronize(ctx->stream));
    *count = int64_t(h);
  } catch (const CudaError& ce) {
    return cuda_fail(ctx, ce.e);
  }
  return MRB_OK;
}

int mrb_tris_destroy(mrb_tris* mesh) {
  delete mesh;
  return MRB_OK;
}

}  // extern "C"
