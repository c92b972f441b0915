// Host mesh setup: validation, CCW orientation, connectivity, CSR operators
// and geometry, bit-exact with the reference (compiled with
// -ffp-contract=off so every product/sum rounds exactly like numpy's).
//
// Reference: pkg/src/meshreg/mesh.py
//   TriMesh.__init__            58-89   validation + orientation
//   TriMesh._build_connectivity 91-123  edges / rings / incident / boundary
//   _signed_area2               153-159
//   TriangleGeometry            173-213 areas, Eq. 9 coefficients, CSR ops
//   build_laplacian             254-265
// and densefield.py PointLocator/locate 62-127 for the coverage fallback.
#include "mesh_host.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>
#ifdef __SSE2__
#include <immintrin.h>
#endif

namespace mrb {

namespace {

constexpr double kDegenerateArea = 1e-9;  // mesh.py:28
constexpr double kBaryEps = 1e-9;         // densefield.py:31

inline double area2(const double* V, int64_t a, int64_t b, int64_t c) {
  // (b0-a0)*(c1-a1) - (c0-a0)*(b1-a1)
  const double ax = V[2 * a], ay = V[2 * a + 1];
  const double bx = V[2 * b], by = V[2 * b + 1];
  const double cx = V[2 * c], cy = V[2 * c + 1];
  const double p = (bx - ax) * (cy - ay);
  const double q = (cx - ax) * (by - ay);
  return p - q;
}

std::string fmt_g(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%g", v);
  return buf;
}

uint32_t spread16(uint32_t x) {
  x &= 0xFFFF;
  x = (x | (x << 8)) & 0x00FF00FF;
  x = (x | (x << 4)) & 0x0F0F0F0F;
  x = (x | (x << 2)) & 0x33333333;
  x = (x | (x << 1)) & 0x55555555;
  return x;
}

}  // namespace

void barycentric(const double* a, const double* b, const double* c, double px, double py,
                 double w[3]) {
  const double d = (b[0] - a[0]) * (c[1] - a[1]) - (c[0] - a[0]) * (b[1] - a[1]);
  const double w1 = ((b[0] - px) * (c[1] - py) - (c[0] - px) * (b[1] - py)) / d;
  const double w2 = ((c[0] - px) * (a[1] - py) - (a[0] - px) * (c[1] - py)) / d;
  w[0] = w1;
  w[1] = w2;
  w[2] = 1.0 - w1 - w2;
}

namespace {

// mesh.py:61-86: validation that needs no connectivity (shape checks happen
// in the binding) and the CCW reorientation into Tout (rows [0, 2, 1] where
// the signed area is negative)
// Deferred meshes are written once here and then only read by the GPU's DMA:
// non-temporal stores keep them out of the CPU caches (the upload then reads
// DRAM instead of snooping freshly written cache lines)
inline void store_nt(double* p, double v) {
#ifdef __SSE2__
  _mm_stream_si64(reinterpret_cast<long long*>(p), __builtin_bit_cast(long long, v));
#else
  *p = v;
#endif
}
inline void store_nt(int32_t* p, int32_t v) {
#ifdef __SSE2__
  _mm_stream_si32(reinterpret_cast<int*>(p), v);
#else
  *p = v;
#endif
}
inline void store_nt(int64_t* p, int64_t v) { *p = v; }  // host build: stays cached
inline void store_fence() {
#ifdef __SSE2__
  _mm_sfence();
#endif
}

template <typename TI>
std::string validate_core(int64_t n, const double* Vin, int64_t m, const int64_t* Tin, TI* Tout,
                          double* Vout = nullptr, int32_t* max_inc = nullptr) {
  // one pass over V (copied to Vout if given) and one over T; the errors are
  // reported in the reference's order whatever triangle trips them
  if (m < 1) return "triangles must be (m, 3) with m >= 1, got (0, 3)";
  bool finite = true;
  for (int64_t i = 0; i < 2 * n; ++i) {
    finite = finite && std::isfinite(Vin[i]);
    if (Vout) store_nt(Vout + i, Vin[i]);
  }
  if (!finite) return "vertex coordinates must be finite";
  std::vector<int32_t> inc(max_inc ? static_cast<size_t>(n) : 0, 0);
  bool range = false, repeated = false, bad = false;
  int64_t worst = 0;
  double worst_abs = INFINITY;
  int32_t mx = 0;
  for (int64_t t = 0; t < m; ++t) {
    const int64_t* r = Tin + 3 * t;
    if (uint64_t(r[0]) >= uint64_t(n) || uint64_t(r[1]) >= uint64_t(n) ||
        uint64_t(r[2]) >= uint64_t(n)) {
      range = true;
      continue;
    }
    repeated = repeated || r[0] == r[1] || r[1] == r[2] || r[0] == r[2];
    const double a2 = area2(Vin, r[0], r[1], r[2]);
    const double ab = std::fabs(a2);
    if (ab <= 2.0 * kDegenerateArea) bad = true;
    if (ab < worst_abs) {  // np.argmin: first minimum
      worst_abs = ab;
      worst = t;
    }
    const bool flip = a2 < 0;  // [0, 2, 1]
    store_nt(Tout + 3 * t, TI(r[0]));
    store_nt(Tout + 3 * t + 1, TI(flip ? r[2] : r[1]));
    store_nt(Tout + 3 * t + 2, TI(flip ? r[1] : r[2]));
    if (max_inc)
      for (int c = 0; c < 3; ++c) mx = std::max(mx, ++inc[size_t(r[c])]);
  }
  store_fence();
  if (range) return "triangle index out of range";
  if (repeated) return "triangle with repeated vertex index";
  if (bad)
    return "degenerate triangle " + std::to_string(worst) + " (area " + fmt_g(worst_abs / 2.0) +
           ")";
  if (max_inc) *max_inc = mx;
  return "";
}

// validate_core into the host mesh (M.n, M.m, M.V, M.T)
std::string validate_orient(int64_t n, const double* Vin, int64_t m, const int64_t* Tin,
                            HostMesh& M) {
  M.T.resize(size_t(std::max<int64_t>(m, 0)) * 3);
  const std::string e = validate_core(n, Vin, m, Tin, M.T.data());
  if (!e.empty()) return e;
  M.n = n;
  M.m = m;
  M.V.assign(Vin, Vin + 2 * n);
  return "";
}

}  // namespace

std::string create_mesh(int64_t n, const double* Vin, int64_t m, const int64_t* Tin,
                        double* Vout, int32_t* Tout, HostMesh& M) {
  if (n >= (int64_t(1) << 31)) return "mesh too large for the device setup (n >= 2^31)";
  int32_t mx = 0;
  const std::string e = validate_core(n, Vin, m, Tin, Tout, Vout, &mx);
  if (!e.empty()) return e;
  M.n = n;
  M.m = m;
  M.dV = Vout;
  M.dT = Tout;
  M.deferred = true;
  // fast-path eligibility estimate (valence = incident triangles, + 1 on the
  // boundary); the device build reports the exact value
  M.max_deg = mx + 1;
  return "";
}

void validate_part(int64_t n, const double* Vin, int64_t v0, int64_t v1, int64_t m,
                   const int64_t* Tin, int64_t t0, int64_t t1, double* Vout, int32_t* Tout,
                   int32_t* inc, ValidatePart& out) {
  (void)m;
  // locals, written to `out` once (neighbouring parts share cache lines)
  ValidatePart p;
  for (int64_t i = 2 * v0; i < 2 * v1; ++i) {
    p.finite = p.finite && std::isfinite(Vin[i]);
    store_nt(Vout + i, Vin[i]);
  }
  for (int64_t t = t0; t < t1; ++t) {
    const int64_t* r = Tin + 3 * t;
    if (uint64_t(r[0]) >= uint64_t(n) || uint64_t(r[1]) >= uint64_t(n) ||
        uint64_t(r[2]) >= uint64_t(n)) {
      p.range = true;
      continue;
    }
    p.repeated = p.repeated || r[0] == r[1] || r[1] == r[2] || r[0] == r[2];
    const double a2 = area2(Vin, r[0], r[1], r[2]);
    const double ab = std::fabs(a2);
    if (ab <= 2.0 * kDegenerateArea) p.bad = true;
    if (ab < p.worst_abs) {  // np.argmin: first minimum (parts merged in order)
      p.worst_abs = ab;
      p.worst = t;
    }
    const bool flip = a2 < 0;
    store_nt(Tout + 3 * t, int32_t(r[0]));
    store_nt(Tout + 3 * t + 1, int32_t(flip ? r[2] : r[1]));
    store_nt(Tout + 3 * t + 2, int32_t(flip ? r[1] : r[2]));
    // incidence counts for the fast-path eligibility estimate: relaxed
    // load + store, not a locked RMW (those ran 40x slower here); a count two
    // parts bump at once may come out low, harmless for an estimate the
    // device build replaces with the exact valence
    for (int c = 0; c < 3; ++c) {
      const int32_t v = __atomic_load_n(inc + r[c], __ATOMIC_RELAXED) + 1;
      __atomic_store_n(inc + r[c], v, __ATOMIC_RELAXED);
      p.max_inc = std::max(p.max_inc, v);
    }
  }
  store_fence();
  out = p;
}

std::string finish_create(const std::vector<ValidatePart>& parts, int64_t n, int64_t m,
                          double* Vout, int32_t* Tout, HostMesh& M) {
  if (m < 1) return "triangles must be (m, 3) with m >= 1, got (0, 3)";
  bool finite = true, range = false, repeated = false, bad = false;
  int64_t worst = 0;
  double worst_abs = INFINITY;
  int32_t mx = 0;
  for (const ValidatePart& p : parts) {  // in triangle order
    finite = finite && p.finite;
    range = range || p.range;
    repeated = repeated || p.repeated;
    bad = bad || p.bad;
    if (p.worst_abs < worst_abs) {
      worst_abs = p.worst_abs;
      worst = p.worst;
    }
    mx = std::max(mx, p.max_inc);
  }
  if (!finite) return "vertex coordinates must be finite";
  if (range) return "triangle index out of range";
  if (repeated) return "triangle with repeated vertex index";
  if (bad)
    return "degenerate triangle " + std::to_string(worst) + " (area " + fmt_g(worst_abs / 2.0) +
           ")";
  M.n = n;
  M.m = m;
  M.dV = Vout;
  M.dT = Tout;
  M.deferred = true;
  M.max_deg = mx + 1;
  return "";
}

const std::string& ensure_host(HostMesh& M) {
  std::call_once(M.host_once, [&M] {
    if (!M.deferred) return;
    const std::vector<int64_t> T(M.dT, M.dT + 3 * M.m);  // already oriented
    M.host_err = build_mesh(M.n, M.dV, M.m, T.data(), M);
    if (M.host_err.empty()) M.deferred = false;
  });
  return M.host_err;
}

std::string build_mesh(int64_t n, const double* Vin, int64_t m, const int64_t* Tin,
                       HostMesh& M) {
  {
    const std::string e = validate_orient(n, Vin, m, Tin, M);
    if (!e.empty()) return e;
  }

  // ---- connectivity, mesh.py:91-123 ----
  // Unique undirected edges in np.unique's lexicographic (lo, hi) order with
  // their use counts: a counting sort on lo, then an insertion sort of each
  // (short) bucket on hi — O(m) instead of a comparison sort of 3m pairs.
  std::vector<int64_t> counts;
  {
    std::vector<int64_t> bptr(n + 1, 0), bhi(3 * m);
    for (int64_t t = 0; t < m; ++t) {
      const int64_t* r = &M.T[3 * t];
      bptr[std::min(r[0], r[1]) + 1]++;
      bptr[std::min(r[1], r[2]) + 1]++;
      bptr[std::min(r[2], r[0]) + 1]++;
    }
    for (int64_t i = 0; i < n; ++i) bptr[i + 1] += bptr[i];
    std::vector<int64_t> fill(bptr.begin(), bptr.end() - 1);
    for (int64_t t = 0; t < m; ++t) {
      const int64_t* r = &M.T[3 * t];
      const int64_t pr[3][2] = {{r[0], r[1]}, {r[1], r[2]}, {r[2], r[0]}};
      for (auto& e : pr) bhi[fill[std::min(e[0], e[1])]++] = std::max(e[0], e[1]);
    }
    M.edges.clear();
    M.edges.reserve(3 * m);
    counts.reserve(3 * m / 2 + n);
    for (int64_t lo = 0; lo < n; ++lo) {
      int64_t* b = bhi.data() + bptr[lo];
      const int64_t len = bptr[lo + 1] - bptr[lo];
      for (int64_t a = 1; a < len; ++a) {
        const int64_t v = b[a];
        int64_t c = a - 1;
        for (; c >= 0 && b[c] > v; --c) b[c + 1] = b[c];
        b[c + 1] = v;
      }
      for (int64_t k = 0; k < len;) {
        int64_t j = k;
        while (j < len && b[j] == b[k]) ++j;
        M.edges.push_back(lo);
        M.edges.push_back(b[k]);
        counts.push_back(j - k);
        k = j;
      }
    }
  }
  M.ne = int64_t(counts.size());
  for (int64_t c : counts)
    if (c > 2) return "non-manifold edge shared by more than two triangles";

  M.valence.assign(n, 0);
  for (int64_t e = 0; e < M.ne; ++e) {
    M.valence[M.edges[2 * e]]++;
    M.valence[M.edges[2 * e + 1]]++;
  }
  M.ring_ptr.assign(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) M.ring_ptr[i + 1] = M.ring_ptr[i] + M.valence[i];
  M.ring_idx.assign(M.ring_ptr[n], 0);
  {
    std::vector<int64_t> fill(M.ring_ptr.begin(), M.ring_ptr.end() - 1);
    for (int64_t e = 0; e < M.ne; ++e) {
      const int64_t a = M.edges[2 * e], b = M.edges[2 * e + 1];
      M.ring_idx[fill[a]++] = b;
      M.ring_idx[fill[b]++] = a;
    }
    // Already ascending: edges arrive in (lo, hi) order, so a vertex first
    // receives its lower neighbours (ascending lo), then its higher ones.
  }
  M.inc_ptr.assign(n + 1, 0);
  for (int64_t k = 0; k < 3 * m; ++k) M.inc_ptr[M.T[k] + 1]++;
  for (int64_t i = 0; i < n; ++i) M.inc_ptr[i + 1] += M.inc_ptr[i];
  M.inc_idx.assign(3 * m, 0);
  {
    std::vector<int64_t> fill(M.inc_ptr.begin(), M.inc_ptr.end() - 1);
    for (int64_t t = 0; t < m; ++t)
      for (int c = 0; c < 3; ++c) M.inc_idx[fill[M.T[3 * t + c]]++] = t;
  }
  M.boundary.assign(n, 0);
  for (int64_t e = 0; e < M.ne; ++e)
    if (counts[e] == 1) M.boundary[M.edges[2 * e]] = M.boundary[M.edges[2 * e + 1]] = 1;
  {
    int64_t lone = 0;
    for (int64_t i = 1; i < n; ++i)
      if (M.valence[i] < M.valence[lone]) lone = i;
    if (n > 0 && M.valence[lone] < 2)
      return "vertex " + std::to_string(lone) + " has valence " +
             std::to_string(M.valence[lone]) + " (< 2)";
  }

  // ---- geometry, mesh.py:173-213 ----
  const double* V = M.V.data();
  M.areas.resize(m);
  M.coeffs.resize(6 * m);
  for (int64_t t = 0; t < m; ++t) {
    const int64_t ia = M.T[3 * t], ib = M.T[3 * t + 1], ic = M.T[3 * t + 2];
    M.areas[t] = 0.5 * area2(V, ia, ib, ic);
  }
  for (int64_t t = 0; t < m; ++t)
    if (M.areas[t] <= kDegenerateArea) return "zero-area triangle in geometry";
  for (int64_t t = 0; t < m; ++t) {
    const double* a = V + 2 * M.T[3 * t];
    const double* b = V + 2 * M.T[3 * t + 1];
    const double* c = V + 2 * M.T[3 * t + 2];
    const double vij[2] = {b[0] - a[0], b[1] - a[1]};
    const double vjk[2] = {c[0] - b[0], c[1] - b[1]};
    const double vik[2] = {c[0] - a[0], c[1] - a[1]};
    auto dot = [](const double* u, double w0, double w1) { return u[0] * w0 + u[1] * w1; };
    // Eq. 9 (mesh.py:193-195): each corner pairs dot products of its edges
    const double di1 = dot(vij, vjk[0], vjk[1]), di2 = dot(vik, -vjk[0], -vjk[1]);
    const double nvij[2] = {-vij[0], -vij[1]}, nvjk[2] = {-vjk[0], -vjk[1]};
    const double nvik[2] = {-vik[0], -vik[1]};
    const double dj1 = dot(nvij, vik[0], vik[1]), dj2 = dot(vjk, -vik[0], -vik[1]);
    const double dk1 = dot(nvjk, -vij[0], -vij[1]), dk2 = dot(nvik, vij[0], vij[1]);
    const double ar = M.areas[t];
    const double inv4a2 = 1.0 / (4.0 * (ar * ar));
    double* co = &M.coeffs[6 * t];
    for (int d = 0; d < 2; ++d) {
      const double ti = di1 * (c[d] - a[d]) + di2 * (b[d] - a[d]);
      const double tj = dj1 * (c[d] - b[d]) + dj2 * (a[d] - b[d]);
      const double tk = dk1 * (a[d] - c[d]) + dk2 * (b[d] - c[d]);
      co[0 * 2 + d] = ti * inv4a2;
      co[1 * 2 + d] = tj * inv4a2;
      co[2 * 2 + d] = tk * inv4a2;
    }
  }
  M.vertex_areas.assign(n, 0.0);  // np.add.at in (t, corner) order
  for (int64_t k = 0; k < 3 * m; ++k) M.vertex_areas[M.T[k]] += M.areas[k / 3];

  // ---- device-facing layout ----
  // Morton (Z-order) relabelling so a warp's nodes gather nearby image taps.
  {
    double lo[2] = {INFINITY, INFINITY}, hi[2] = {-INFINITY, -INFINITY};
    for (int64_t i = 0; i < n; ++i)
      for (int d = 0; d < 2; ++d) {
        lo[d] = std::min(lo[d], V[2 * i + d]);
        hi[d] = std::max(hi[d], V[2 * i + d]);
      }
    const double span = std::max(std::max(hi[0] - lo[0], hi[1] - lo[1]), 1e-12);
    std::vector<uint32_t> key(n);
    for (int64_t i = 0; i < n; ++i) {
      const uint32_t qx = uint32_t(std::min(65535.0, (V[2 * i] - lo[0]) / span * 65535.0));
      const uint32_t qy = uint32_t(std::min(65535.0, (V[2 * i + 1] - lo[1]) / span * 65535.0));
      key[i] = spread16(qx) | (spread16(qy) << 1);
    }
    M.perm.resize(n);
    std::iota(M.perm.begin(), M.perm.end(), 0);
    std::stable_sort(M.perm.begin(), M.perm.end(),
                     [&](int32_t x, int32_t y) { return key[x] < key[y]; });
    M.iperm.resize(n);
    for (int64_t k = 0; k < n; ++k) M.iperm[M.perm[k]] = int32_t(k);
  }
  // Fused gradient operator G = avg∘grad on the {self} ∪ one-ring pattern:
  // grad_v = sum_t w_vt * sum_c coeff[t,c] f[T[t,c]]  (mesh.py:236-241).
  M.nb_ptr.assign(n + 1, 0);
  M.nb_idx.resize(M.ring_idx.size());
  M.g_nb.assign(2 * M.ring_idx.size(), 0.0);
  M.g_self.assign(2 * n, 0.0);
  M.inv_val.resize(n);
  M.Vn.resize(2 * n);
  for (int64_t k = 0; k < n; ++k) {
    const int64_t i = M.perm[k];
    M.nb_ptr[k + 1] = M.nb_ptr[k] + int32_t(M.valence[i]);
    M.max_deg = std::max(M.max_deg, int32_t(M.valence[i]));
  }
  for (int64_t k = 0; k < n; ++k) {
    const int64_t i = M.perm[k];
    M.inv_val[k] = 1.0 / double(M.valence[i]);
    M.Vn[2 * k] = V[2 * i];
    M.Vn[2 * k + 1] = V[2 * i + 1];
    const int64_t r0 = M.ring_ptr[i], r1 = M.ring_ptr[i + 1];
    const int32_t base = M.nb_ptr[k];
    for (int64_t r = r0; r < r1; ++r) M.nb_idx[base + (r - r0)] = M.iperm[M.ring_idx[r]];
    // accumulate fused coefficients over incident triangles (ascending id)
    const int64_t* ring = &M.ring_idx[r0];
    double* g = &M.g_nb[2 * int64_t(base)];
    double sx = 0.0, sy = 0.0;
    for (int64_t q = M.inc_ptr[i]; q < M.inc_ptr[i + 1]; ++q) {
      const int64_t t = M.inc_idx[q];
      const double w = M.areas[t] / M.vertex_areas[i];
      for (int c = 0; c < 3; ++c) {
        const int64_t j = M.T[3 * t + c];
        const double cx = w * M.coeffs[6 * t + 2 * c];
        const double cy = w * M.coeffs[6 * t + 2 * c + 1];
        if (j == i) {
          sx += cx;
          sy += cy;
        } else {
          int64_t pos = 0;
          while (ring[pos] != j) ++pos;  // j is a one-ring neighbour of i
          g[2 * pos] += cx;
          g[2 * pos + 1] += cy;
        }
      }
    }
    M.g_self[2 * k] = sx;
    M.g_self[2 * k + 1] = sy;
  }
  M.Tn.resize(4 * m);
  for (int64_t t = 0; t < m; ++t) {
    for (int c = 0; c < 3; ++c) M.Tn[4 * t + c] = M.iperm[M.T[3 * t + c]];
    M.Tn[4 * t + 3] = 0;
  }
  return "";
}

void ensure_reference_csr(HostMesh& M) {
  std::call_once(M.csr_once, [&M] {
    const int64_t n = M.n, m = M.m;
    // Gx, Gy (m x n, one row per triangle, its 3 corners by ascending vertex id)
    // and avg (n x m, row i = the incident triangles, ascending id: exactly
    // inc_ptr / inc_idx) — the canonical CSR scipy builds from the triplets.
    M.gx.indptr.resize(m + 1);
    M.gy.indptr.resize(m + 1);
    M.gx.indices.resize(3 * m);
    M.gy.indices.resize(3 * m);
    M.gx.data.resize(3 * m);
    M.gy.data.resize(3 * m);
    for (int64_t t = 0; t <= m; ++t) M.gx.indptr[t] = M.gy.indptr[t] = 3 * t;
    for (int64_t t = 0; t < m; ++t) {
      int o[3] = {0, 1, 2};
      const int64_t* r = &M.T[3 * t];
      if (r[o[1]] < r[o[0]]) std::swap(o[0], o[1]);
      if (r[o[2]] < r[o[1]]) std::swap(o[1], o[2]);
      if (r[o[1]] < r[o[0]]) std::swap(o[0], o[1]);
      for (int c = 0; c < 3; ++c) {
        M.gx.indices[3 * t + c] = M.gy.indices[3 * t + c] = r[o[c]];
        M.gx.data[3 * t + c] = M.coeffs[6 * t + 2 * o[c]];
        M.gy.data[3 * t + c] = M.coeffs[6 * t + 2 * o[c] + 1];
      }
    }
    M.avg.indptr = M.inc_ptr;
    M.avg.indices = M.inc_idx;
    M.avg.data.resize(3 * m);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t q = M.inc_ptr[i]; q < M.inc_ptr[i + 1]; ++q)
        M.avg.data[q] = M.areas[M.inc_idx[q]] / M.vertex_areas[i];
    // Laplacian (mesh.py:254-265): rows = one-rings, values 1/valence
    M.lap.indptr = M.ring_ptr;
    M.lap.indices = M.ring_idx;
    M.lap.data.resize(M.ring_idx.size());
    for (int64_t i = 0; i < n; ++i) {
      const double v = 1.0 / double(M.valence[i]);
      for (int64_t k = M.ring_ptr[i]; k < M.ring_ptr[i + 1]; ++k) M.lap.data[k] = v;
    }
  });
}

// ---- PointLocator / locate (densefield.py:62-127) ----
Locator::Locator(const HostMesh& M) {
  lo[0] = lo[1] = INFINITY;
  hi[0] = hi[1] = -INFINITY;
  for (int64_t i = 0; i < M.n; ++i)
    for (int d = 0; d < 2; ++d) {
      lo[d] = std::min(lo[d], M.V[2 * i + d]);
      hi[d] = std::max(hi[d], M.V[2 * i + d]);
    }
  const double s0 = std::max(hi[0] - lo[0], 1e-9), s1 = std::max(hi[1] - lo[1], 1e-9);
  cell = std::max(2.0, std::sqrt(2.0 * s0 * s1 / double(std::max<int64_t>(M.m, 1))));
  nx = int64_t(std::ceil(s0 / cell)) + 1;
  ny = int64_t(std::ceil(s1 / cell)) + 1;
  bins.assign(nx * ny, {});
  for (int64_t t = 0; t < M.m; ++t) {
    double mn[2] = {INFINITY, INFINITY}, mx[2] = {-INFINITY, -INFINITY};
    for (int c = 0; c < 3; ++c)
      for (int d = 0; d < 2; ++d) {
        mn[d] = std::min(mn[d], M.V[2 * M.T[3 * t + c] + d]);
        mx[d] = std::max(mx[d], M.V[2 * M.T[3 * t + c] + d]);
      }
    int64_t bx0, by0, bx1, by1;
    cell_of(mn[0], mn[1], bx0, by0);
    cell_of(mx[0], mx[1], bx1, by1);
    for (int64_t by = by0; by <= by1; ++by)
      for (int64_t bx = bx0; bx <= bx1; ++bx) bins[by * nx + bx].push_back(t);
  }
}

void Locator::cell_of(double x, double y, int64_t& bx, int64_t& by) const {
  bx = int64_t((std::min(std::max(x, lo[0]), hi[0]) - lo[0]) / cell);
  by = int64_t((std::min(std::max(y, lo[1]), hi[1]) - lo[1]) / cell);
  bx = std::min(bx, nx - 1);
  by = std::min(by, ny - 1);
}

int64_t Locator::locate(const HostMesh& M, double px, double py, double w[3]) const {
  int64_t bx, by;
  cell_of(px, py, bx, by);
  auto test = [&](int64_t t) {
    barycentric(&M.V[2 * M.T[3 * t]], &M.V[2 * M.T[3 * t + 1]], &M.V[2 * M.T[3 * t + 2]], px,
                py, w);
    return std::min(std::min(w[0], w[1]), w[2]) >= -kBaryEps;
  };
  for (int64_t t : bins[by * nx + bx])
    if (test(t)) return t;
  for (int64_t t = 0; t < M.m; ++t)
    if (test(t)) return t;
  return -1;
}

}  // namespace mrb
