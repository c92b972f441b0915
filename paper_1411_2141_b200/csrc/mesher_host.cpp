// Host side of the content-adaptive mesher: the sequential stages of the
// reference's generate_mesh (meshgen.py:365-396) and delaunay.py, in C++.
//
// The reference runs these in Python (Bowyer-Watson scans every triangle
// ever created per insertion: O(n^2), about 30 s for a 12k-node mesh and
// hours at 500k).  Here the insertion walks to the point and grows the
// cavity through triangle adjacency, the flip sweeps and the CVT/ODT
// relaxation are plain loops, and every floating-point expression keeps the
// reference's operation order (compiled with -ffp-contract=off), so the
// result is bit-identical to the reference mesh:
//   * triangle ids follow the reference's creation order, including the
//     iteration order of the Python set the cavity edges are collected in
//     (delaunay.py:162-168), which is reproduced from CPython 3.12's tuple
//     hash and set probing;
//   * sums follow numpy's pairwise (1-D) and sequential (axis 0) orders.
// The image-space stages (Gaussian, gradient magnitude, Canny) run on the
// GPU (mesher.cuh); this file receives their outputs.
#include "mesher_host.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <unordered_map>

namespace mrb {

namespace {

std::string fmt_g(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%g", v);
  return buf;
}

inline double orient(const double* a, const double* b, const double* c) {
  return (b[0] - a[0]) * (c[1] - a[1]) - (c[0] - a[0]) * (b[1] - a[1]);
}

// circumcircles (delaunay.py:54-72) for one triangle (a, b, c).
inline void circumcircle(const double* a, const double* b, const double* c, double& cx,
                         double& cy, double& r2) {
  const double ab0 = b[0] - a[0], ab1 = b[1] - a[1];
  const double ac0 = c[0] - a[0], ac1 = c[1] - a[1];
  const double d = 2.0 * (ab0 * ac1 - ab1 * ac0);
  const double ab2 = ab0 * ab0 + ab1 * ab1;
  const double ac2 = ac0 * ac0 + ac1 * ac1;
  double ux = (ac1 * ab2 - ab1 * ac2) / d;
  double uy = (ab0 * ac2 - ac0 * ab2) / d;
  if (!std::isfinite(ux) || !std::isfinite(uy)) {
    cx = a[0] + 0.0;
    cy = a[1] + 0.0;
    r2 = INFINITY;
    return;
  }
  r2 = ux * ux + uy * uy;
  cx = a[0] + ux;
  cy = a[1] + uy;
}

// Python's float floor division (Objects/floatobject.c float_floor_div).
double py_floordiv(double vx, double wx) {
  double mod = std::fmod(vx, wx);
  double div = (vx - mod) / wx;
  if (mod != 0.0) {
    if ((wx < 0) != (mod < 0)) div -= 1.0;
  }
  double fd;
  if (div != 0.0) {
    fd = std::floor(div);
    if (div - fd > 0.5) fd += 1.0;
  } else {
    fd = std::copysign(0.0, vx / wx);
  }
  return fd;
}

// ---- CPython 3.12 set iteration order for a set of 2-tuples of ints ------
// tuplehash (Objects/tupleobject.c, xxHash-based since 3.8) and
// set_add_entry / set_table_resize / set_insert_clean (Objects/setobject.c).
constexpr uint64_t kXXP1 = 11400714785074694791ULL;
constexpr uint64_t kXXP2 = 14029467366897019727ULL;
constexpr uint64_t kXXP5 = 2870177450012600261ULL;

inline uint64_t py_int_hash(int64_t v) {
  // ints in [0, 2^61 - 1) hash to themselves (all vertex ids here)
  return uint64_t(v);
}

inline int64_t py_tuple2_hash(int64_t a, int64_t b) {
  uint64_t acc = kXXP5;
  for (uint64_t lane : {py_int_hash(a), py_int_hash(b)}) {
    acc += lane * kXXP2;
    acc = (acc << 31) | (acc >> 33);
    acc *= kXXP1;
  }
  acc += uint64_t(2) ^ (kXXP5 ^ 3527539ULL);
  if (acc == ~uint64_t(0)) return 1546275796;
  return int64_t(acc);
}

struct PySet2 {
  struct Entry {
    int64_t hash;
    int32_t key;  // index into the key list, -1 = empty
  };
  const std::vector<std::pair<int64_t, int64_t>>* keys = nullptr;
  std::vector<Entry> table;
  size_t mask = 7, fill = 0, used = 0;
  static constexpr size_t kLinearProbes = 9;
  static constexpr int kPerturbShift = 5;

  void reset(const std::vector<std::pair<int64_t, int64_t>>* k) {
    keys = k;
    table.assign(8, Entry{0, -1});
    mask = 7;
    fill = used = 0;
  }
  void insert_clean(std::vector<Entry>& tab, size_t msk, int32_t key, int64_t hash) {
    size_t perturb = size_t(hash);
    size_t i = size_t(hash) & msk;
    while (true) {
      if (tab[i].key < 0) break;
      bool found = false;
      if (i + kLinearProbes <= msk) {
        for (size_t j = 1; j <= kLinearProbes; ++j) {
          if (tab[i + j].key < 0) {
            i += j;
            found = true;
            break;
          }
        }
      }
      if (found) break;
      perturb >>= kPerturbShift;
      i = (i * 5 + 1 + perturb) & msk;
    }
    tab[i] = Entry{hash, key};
  }
  void resize(size_t minused) {
    size_t newsize = 8;
    while (newsize <= minused) newsize <<= 1;
    std::vector<Entry> nt(newsize, Entry{0, -1});
    for (size_t i = 0; i <= mask; ++i)
      if (table[i].key >= 0) insert_clean(nt, newsize - 1, table[i].key, table[i].hash);
    table.swap(nt);
    mask = newsize - 1;
    fill = used;
  }
  bool eq(int32_t a, int32_t b) const { return (*keys)[a] == (*keys)[b]; }
  void add(int32_t key) {
    const auto& kv = (*keys)[key];
    const int64_t hash = py_tuple2_hash(kv.first, kv.second);
    size_t perturb = size_t(hash);
    size_t i = size_t(hash) & mask;
    while (true) {
      size_t probes = (i + kLinearProbes <= mask) ? kLinearProbes : 0;
      size_t j = i;
      while (true) {
        Entry& e = table[j];
        if (e.key < 0) {
          e = Entry{hash, key};
          ++fill;
          ++used;
          if (fill * 5 < mask * 3) return;
          resize(used > 50000 ? used * 2 : used * 4);
          return;
        }
        if (e.hash == hash && eq(e.key, key)) return;  // already present
        if (probes-- == 0) break;
        ++j;
      }
      perturb >>= kPerturbShift;
      i = (i * 5 + 1 + perturb) & mask;
    }
  }
  bool contains(int64_t a, int64_t b) const {
    const int64_t hash = py_tuple2_hash(a, b);
    size_t perturb = size_t(hash);
    size_t i = size_t(hash) & mask;
    while (true) {
      size_t probes = (i + kLinearProbes <= mask) ? kLinearProbes : 0;
      size_t j = i;
      while (true) {
        const Entry& e = table[j];
        if (e.key < 0) return false;
        if (e.hash == hash && (*keys)[e.key] == std::make_pair(a, b)) return true;
        if (probes-- == 0) break;
        ++j;
      }
      perturb >>= kPerturbShift;
      i = (i * 5 + 1 + perturb) & mask;
    }
  }
};

// numpy pairwise summation (numpy/_core/src/umath/loops_utils.h.src).
double pairwise_rec(const double* a, int64_t n) {
  if (n < 8) {
    double res = -0.0;
    for (int64_t i = 0; i < n; ++i) res += a[i];
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise_rec(a, n2) + pairwise_rec(a + n2, n - n2);
}

// glibc hypot kernel (sysdeps/ieee754/dbl-64/e_hypot.c, non-FMA build).
inline double hypot_kernel(double ax, double ay) {
  double t1, t2;
  double h = std::sqrt(ax * ax + ay * ay);
  if (h <= 2.0 * ay) {
    double delta = h - ay;
    t1 = ax * (2.0 * delta - ax);
    t2 = (delta - 2.0 * (ax - ay)) * delta;
  } else {
    double delta = h - ax;
    t1 = 2.0 * delta * (ax - 2.0 * ay);
    t2 = (4.0 * delta - ay) * ay + delta * delta;
  }
  h -= (t1 + t2) / (2.0 * h);
  return h;
}

}  // namespace

double np_pairwise_sum(const double* a, int64_t n) { return pairwise_rec(a, n); }

double glibc_hypot(double x, double y) {
  if (!std::isfinite(x) || !std::isfinite(y)) {
    if (std::isinf(x) || std::isinf(y)) return INFINITY;
    return x + y;
  }
  x = std::fabs(x);
  y = std::fabs(y);
  double ax = x < y ? y : x, ay = x < y ? x : y;
  if (ax > 0x1p+511) {
    if (ay <= ax * 0x1p-54) return ax + ay;
    return hypot_kernel(ax * 0x1p-600, ay * 0x1p-600) / 0x1p-600;
  }
  if (ay < 0x1p-511) {
    if (ax >= ay / 0x1p-54) return ax + ay;
    return hypot_kernel(ax / 0x1p-600, ay / 0x1p-600) * 0x1p-600;
  }
  if (ay <= ax * 0x1p-54) return ax + ay;
  return hypot_kernel(ax, ay);
}

// ---------------------------------------------------------------------------
// TriMesh(V, T), mesh.py:59-123
std::string trimesh_init(Tris& t) {
  const int64_t n = t.n(), m = t.m();
  if (m < 1) return "triangles must be (m, 3) with m >= 1, got (" + std::to_string(m) + ", 3)";
  for (double v : t.V)
    if (!std::isfinite(v)) return "vertex coordinates must be finite";
  for (int64_t v : t.T)
    if (v < 0 || v >= n) return "triangle index out of range";
  for (int64_t k = 0; k < m; ++k) {
    const int64_t* r = &t.T[3 * k];
    if (r[0] == r[1] || r[1] == r[2] || r[0] == r[2]) return "triangle with repeated vertex index";
  }
  int64_t worst = -1;
  double worst_abs = INFINITY;
  bool degenerate = false;
  std::vector<double> a2(m);
  for (int64_t k = 0; k < m; ++k) {
    const int64_t* r = &t.T[3 * k];
    a2[k] = orient(&t.V[2 * r[0]], &t.V[2 * r[1]], &t.V[2 * r[2]]);
    const double ab = std::fabs(a2[k]);
    if (ab <= 2.0 * 1e-9) degenerate = true;
    if (ab < worst_abs) {
      worst_abs = ab;
      worst = k;
    }
  }
  if (degenerate)
    return "degenerate triangle " + std::to_string(worst) + " (area " + fmt_g(worst_abs / 2.0) +
           ")";
  for (int64_t k = 0; k < m; ++k)
    if (a2[k] < 0) std::swap(t.T[3 * k + 1], t.T[3 * k + 2]);
  // edges with multiplicity (np.unique of sorted pairs)
  std::vector<uint64_t> e;
  e.reserve(3 * m);
  for (int64_t k = 0; k < m; ++k) {
    const int64_t* r = &t.T[3 * k];
    for (int j = 0; j < 3; ++j) {
      int64_t a = r[j], b = r[(j + 1) % 3];
      if (a > b) std::swap(a, b);
      e.push_back((uint64_t(a) << 32) | uint64_t(b));
    }
  }
  std::sort(e.begin(), e.end());
  std::vector<int64_t> valence(n, 0);
  t.boundary.assign(n, 0);
  for (size_t i = 0; i < e.size();) {
    size_t j = i;
    while (j < e.size() && e[j] == e[i]) ++j;
    if (j - i > 2) return "non-manifold edge shared by more than two triangles";
    const int64_t a = int64_t(e[i] >> 32), b = int64_t(e[i] & 0xffffffffu);
    valence[a]++;
    valence[b]++;
    if (j - i == 1) t.boundary[a] = t.boundary[b] = 1;
    i = j;
  }
  t.inc_ptr.assign(n + 1, 0);
  for (int64_t v : t.T) t.inc_ptr[v + 1]++;
  for (int64_t i = 0; i < n; ++i) t.inc_ptr[i + 1] += t.inc_ptr[i];
  t.inc_idx.assign(3 * m, 0);
  std::vector<int64_t> fillp(t.inc_ptr.begin(), t.inc_ptr.end() - 1);
  for (int64_t k = 0; k < m; ++k)
    for (int j = 0; j < 3; ++j) t.inc_idx[fillp[t.T[3 * k + j]]++] = k;
  int64_t lone = -1, lv = INT64_MAX;
  for (int64_t i = 0; i < n; ++i)
    if (valence[i] < lv) {
      lv = valence[i];
      lone = i;
    }
  if (lv < 2)
    return "vertex " + std::to_string(lone) + " has valence " + std::to_string(lv) + " (< 2)";
  return "";
}

// ---------------------------------------------------------------------------
// dedupe_points, delaunay.py:30-51
std::string dedupe_points(const double* P, int64_t n, double tol, std::vector<double>& out) {
  out.clear();
  for (int64_t i = 0; i < 2 * n; ++i)
    if (!std::isfinite(P[i])) return "points must be finite";
  if (n == 0) return "";
  std::vector<int64_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    if (P[2 * a] != P[2 * b]) return P[2 * a] < P[2 * b];
    return P[2 * a + 1] < P[2 * b + 1];
  });
  out.reserve(2 * n);
  out.push_back(P[2 * order[0]]);
  out.push_back(P[2 * order[0] + 1]);
  for (int64_t s = 1; s < n; ++s) {
    const double px = P[2 * order[s]], py = P[2 * order[s] + 1];
    bool dup = false;
    for (int64_t q = int64_t(out.size() / 2) - 1; q >= 0; --q) {
      const double qx = out[2 * q], qy = out[2 * q + 1];
      if (px - qx > tol) break;
      if (std::fabs(py - qy) <= tol && std::fabs(px - qx) <= tol) {
        dup = true;
        break;
      }
    }
    if (!dup) {
      out.push_back(px);
      out.push_back(py);
    }
  }
  return "";
}

namespace {

bool all_collinear(const std::vector<double>& P) {  // delaunay.py:94-104
  const int64_t n = int64_t(P.size() / 2);
  const double tol = 1e-12;
  std::vector<double> d(2 * n), norms(n);
  int64_t k = 0;
  double nmax = -INFINITY;
  for (int64_t i = 0; i < n; ++i) {
    d[2 * i] = P[2 * i] - P[0];
    d[2 * i + 1] = P[2 * i + 1] - P[1];
    norms[i] = glibc_hypot(d[2 * i], d[2 * i + 1]);
    if (norms[i] > nmax) {
      nmax = norms[i];
      k = i;
    }
  }
  if (norms[k] == 0.0) return true;
  const double r0 = d[2 * k] / norms[k], r1 = d[2 * k + 1] / norms[k];
  const double scale = std::max(nmax, 1.0);
  for (int64_t i = 0; i < n; ++i) {
    const double cross = std::fabs(d[2 * i] * r1 - d[2 * i + 1] * r0);
    if (!(cross <= tol * scale + 1e-12)) return false;
  }
  return true;
}

// Bowyer-Watson with the reference's triangle ids (delaunay.py:107-178).
struct BowyerWatson {
  int64_t n = 0;
  std::vector<double> X;      // (n+3)*2: points then the three super vertices
  std::vector<int64_t> tris;  // count*3
  std::vector<double> circ;   // count*3: cx, cy, r2
  std::vector<uint8_t> alive;
  std::vector<int64_t> nbr;   // count*3: triangle across edge k = (t[k], t[k+1])
  std::vector<uint32_t> stamp;
  uint32_t epoch = 0;
  bool check_full = false;    // MESHREG_B200_BW_CHECK: compare with the full scan
  mutable int64_t st_steps = 0, st_walk_fail = 0, st_scan = 0, st_cavity = 0;

  int64_t count() const { return int64_t(alive.size()); }

  int64_t push(int64_t a, int64_t b, int64_t c) {
    const int64_t t = count();
    tris.insert(tris.end(), {a, b, c});
    double cx, cy, r2;
    circumcircle(&X[2 * a], &X[2 * b], &X[2 * c], cx, cy, r2);
    circ.insert(circ.end(), {cx, cy, r2});
    alive.push_back(1);
    nbr.insert(nbr.end(), {-1, -1, -1});
    stamp.push_back(0);
    return t;
  }

  bool bad(int64_t t, double px, double py) const {
    if (!alive[t]) return false;
    const double dx = px - circ[3 * t], dy = py - circ[3 * t + 1];
    const double r2 = circ[3 * t + 2];
    const double tol = 4e-9 * std::sqrt(std::max(r2, 0.0)) + 1e-12;
    return dx * dx + dy * dy < r2 - tol;
  }

  bool contains_tol(int64_t t, const double* p) const {
    const double* a = &X[2 * tris[3 * t]];
    const double* b = &X[2 * tris[3 * t + 1]];
    const double* c = &X[2 * tris[3 * t + 2]];
    return orient(a, b, p) >= -1e-12 && orient(b, c, p) >= -1e-12 && orient(c, a, p) >= -1e-12;
  }

  // Straight walk to a triangle containing p; -1 when it leaves the hull or
  // cycles (fp), in which case the caller scans.
  int64_t walk(int64_t t, const double* p) const {
    const int64_t limit = count() + 16;
    for (int64_t s = 0; s < limit && t >= 0; ++s) {
      ++st_steps;
      if (!alive[t]) return -1;
      int64_t next = -2;
      for (int k = 0; k < 3; ++k) {
        const double* a = &X[2 * tris[3 * t + k]];
        const double* b = &X[2 * tris[3 * t + (k + 1) % 3]];
        if (orient(a, b, p) < 0) {
          next = nbr[3 * t + k];
          break;
        }
      }
      if (next == -2) return t;
      t = next;
    }
    return -1;
  }

  std::string run(const std::vector<double>& P, std::vector<int64_t>& T_out) {
    n = int64_t(P.size() / 2);
    double lo[2] = {P[0], P[1]}, hi[2] = {P[0], P[1]};
    for (int64_t i = 1; i < n; ++i)
      for (int j = 0; j < 2; ++j) {
        lo[j] = std::min(lo[j], P[2 * i + j]);
        hi[j] = std::max(hi[j], P[2 * i + j]);
      }
    const double center[2] = {0.5 * (lo[0] + hi[0]), 0.5 * (lo[1] + hi[1])};
    double span = hi[0] - lo[0];
    if (hi[1] - lo[1] > span) span = hi[1] - lo[1];
    if (1.0 > span) span = 1.0;
    const double big = 100.0 * span;
    // np.cos / np.sin of pi/2, 7pi/6, 11pi/6 (delaunay.py:117-119)
    static const double cs[3][2] = {{0x1.1a62633145c07p-54, 0x1.0000000000000p+0},
                                    {-0x1.bb67ae8584cacp-1, -0x1.ffffffffffffbp-2},
                                    {0x1.bb67ae8584ca8p-1, -0x1.0000000000004p-1}};
    X.assign(P.begin(), P.end());
    for (int s = 0; s < 3; ++s)
      for (int j = 0; j < 2; ++j) X.push_back(center[j] + 2.0 * big * cs[s][j]);
    const size_t cap = size_t(std::max<int64_t>(4 * n + 16, 64)) * 2 + 16;
    tris.reserve(3 * cap);
    circ.reserve(3 * cap);
    alive.reserve(cap);
    nbr.reserve(3 * cap);
    stamp.reserve(cap);
    if (orient(&X[2 * n], &X[2 * (n + 1)], &X[2 * (n + 2)]) < 0)
      push(n, n + 2, n + 1);
    else
      push(n, n + 1, n + 2);

    std::vector<int64_t> cavity, queue;
    std::vector<std::pair<int64_t, int64_t>> dedges;  // cavity directed edges
    std::vector<int64_t> dedge_outside;               // triangle across each
    PySet2 set;
    std::vector<int64_t> scan_bad;
    int64_t last = 0;
    // Walk start (jump-and-walk): a coarse grid over the points remembers a
    // triangle made by the latest insertion in each cell.  The points come in
    // lexicographic (x, y) order, so `last` alone can be a whole column away.
    // The start does not change the result, only the walk length.
    const int64_t G = std::max<int64_t>(1, int64_t(std::sqrt(double(n) / 2.0)));
    const double gw = std::max(hi[0] - lo[0], 1e-300), gh = std::max(hi[1] - lo[1], 1e-300);
    std::vector<int64_t> cell_tri(size_t(G * G), -1);
    auto cell_of = [&](const double* q) {
      int64_t cx = int64_t((q[0] - lo[0]) / gw * double(G));
      int64_t cy = int64_t((q[1] - lo[1]) / gh * double(G));
      cx = std::min(std::max<int64_t>(cx, 0), G - 1);
      cy = std::min(std::max<int64_t>(cy, 0), G - 1);
      return cy * G + cx;
    };
    auto start_for = [&](const double* q) {
      const int64_t c = cell_of(q), cx = c % G, cy = c / G;
      for (int64_t r = 0; r <= 2; ++r)
        for (int64_t dy = -r; dy <= r; ++dy)
          for (int64_t dx = -r; dx <= r; ++dx) {
            if (std::max(std::llabs(dx), std::llabs(dy)) != r) continue;
            const int64_t x = cx + dx, y = cy + dy;
            if (x < 0 || y < 0 || x >= G || y >= G) continue;
            const int64_t t = cell_tri[size_t(y * G + x)];
            if (t >= 0 && alive[t]) return t;
          }
      return last;
    };
    for (int64_t idx = 0; idx < n; ++idx) {
      const double* p = &X[2 * idx];
      const double px = p[0], py = p[1];
      cavity.clear();
      ++epoch;
      int64_t t0 = walk(start_for(p), p);
      if (t0 < 0 && alive[last]) t0 = walk(last, p);
      if (t0 < 0) ++st_walk_fail;
      if (t0 < 0) {
        for (int64_t t = 0; t < count(); ++t)
          if (alive[t] && contains_tol(t, p)) {
            t0 = t;
            break;
          }
      }
      // seeds: the containing triangle, else its bad neighbours
      queue.clear();
      if (t0 >= 0) {
        if (bad(t0, px, py)) {
          queue.push_back(t0);
          stamp[t0] = epoch;
        } else {
          stamp[t0] = epoch;
          for (int k = 0; k < 3; ++k) {
            const int64_t u = nbr[3 * t0 + k];
            if (u >= 0 && stamp[u] != epoch) {
              stamp[u] = epoch;
              if (bad(u, px, py)) queue.push_back(u);
            }
          }
        }
      }
      bool scanned = false;
      if (queue.empty()) {
        // the reference's full scan decides (and its containing-triangle fallback)
        scanned = true;
        ++st_scan;
        for (int64_t t = 0; t < count(); ++t)
          if (bad(t, px, py)) cavity.push_back(t);
        if (cavity.empty()) {
          int64_t c = -1;
          for (int64_t t = 0; t < count(); ++t)
            if (alive[t] && contains_tol(t, p)) {
              c = t;
              break;
            }
          if (c < 0) return "insertion point not covered by current triangulation";
          cavity.push_back(c);
        }
      } else {
        for (size_t q = 0; q < queue.size(); ++q) {
          const int64_t t = queue[q];
          cavity.push_back(t);
          for (int k = 0; k < 3; ++k) {
            const int64_t u = nbr[3 * t + k];
            if (u >= 0 && stamp[u] != epoch) {
              stamp[u] = epoch;
              if (bad(u, px, py)) queue.push_back(u);
            }
          }
        }
        std::sort(cavity.begin(), cavity.end());
      }
      if (check_full && !scanned) {
        scan_bad.clear();
        for (int64_t t = 0; t < count(); ++t)
          if (bad(t, px, py)) scan_bad.push_back(t);
        if (scan_bad != cavity) {
          std::fprintf(stderr, "meshreg_b200: Bowyer-Watson cavity differs from the full scan at "
                               "point %lld\n", (long long)idx);
          std::abort();
        }
      }
      // cavity edges into the emulated Python set, in the reference's order
      dedges.clear();
      dedge_outside.clear();
      for (int64_t t : cavity) {
        alive[t] = 0;
        for (int k = 0; k < 3; ++k) {
          dedges.emplace_back(tris[3 * t + k], tris[3 * t + (k + 1) % 3]);
          dedge_outside.push_back(nbr[3 * t + k]);
        }
      }
      set.reset(&dedges);
      for (size_t e = 0; e < dedges.size(); ++e) set.add(int32_t(e));
      const int64_t first_new = count();
      for (size_t s = 0; s <= set.mask; ++s) {
        const int32_t e = set.table[s].key;
        if (e < 0) continue;
        const int64_t u = dedges[e].first, v = dedges[e].second;
        if (set.contains(v, u)) continue;
        const int64_t t = push(u, v, idx);
        // adjacency: across (u, v) the outside triangle (which now points here)
        const int64_t o = dedge_outside[e];
        nbr[3 * t] = o;
        if (o >= 0) {
          for (int k = 0; k < 3; ++k)
            if (tris[3 * o + k] == v && tris[3 * o + (k + 1) % 3] == u) nbr[3 * o + k] = t;
        }
      }
      // adjacency among the new fan: (v, idx) meets the triangle starting at
      // v, (idx, u) the one ending at u
      const int64_t k_new = count() - first_new;
      if (k_new <= 64) {
        for (int64_t a = first_new; a < count(); ++a)
          for (int64_t b = first_new; b < count(); ++b) {
            if (tris[3 * b] == tris[3 * a + 1]) nbr[3 * a + 1] = b;
            if (tris[3 * b + 1] == tris[3 * a]) nbr[3 * a + 2] = b;
          }
      } else {
        std::unordered_map<int64_t, int64_t> by_start, by_end;
        for (int64_t b = first_new; b < count(); ++b) {
          by_start[tris[3 * b]] = b;
          by_end[tris[3 * b + 1]] = b;
        }
        for (int64_t a = first_new; a < count(); ++a) {
          auto i1 = by_start.find(tris[3 * a + 1]);
          if (i1 != by_start.end()) nbr[3 * a + 1] = i1->second;
          auto i2 = by_end.find(tris[3 * a]);
          if (i2 != by_end.end()) nbr[3 * a + 2] = i2->second;
        }
      }
      if (k_new > 0) {
        last = count() - 1;
        cell_tri[size_t(cell_of(p))] = last;
      }
    }
    if (std::getenv("MESHREG_B200_DEBUG"))
      std::fprintf(stderr, "meshreg_b200: bowyer-watson walk steps %lld, walk fallbacks %lld, "
                   "full scans %lld\n", (long long)st_steps, (long long)st_walk_fail,
                   (long long)st_scan);
    T_out.clear();
    for (int64_t t = 0; t < count(); ++t) {
      if (!alive[t]) continue;
      const int64_t* r = &tris[3 * t];
      if (r[0] < n && r[1] < n && r[2] < n) T_out.insert(T_out.end(), {r[0], r[1], r[2]});
    }
    if (T_out.empty()) return "triangulation collapsed (points nearly collinear)";
    return "";
  }
};

// One flip sweep (delaunay.py:202-287).  Returns the number of flips.
int64_t flip_sweep(const std::vector<double>& V, std::vector<int64_t>& T) {
  const int64_t m = int64_t(T.size() / 3);
  struct Ent {
    int64_t u, v;
    int64_t t[2], w[2];
    int cnt;
  };
  // The reference's edge_map is an insertion-ordered dict keyed by (min, max)
  // over the half-edges h = 3t + j in order.  Here: bucket the half-edges by
  // their low vertex (counting sort), pair equal keys inside each bucket, and
  // order the edges by their first half-edge.
  const int64_t nv = m > 0 ? *std::max_element(T.begin(), T.end()) + 1 : 0;
  std::vector<int64_t> start(size_t(nv) + 1, 0), hv(size_t(3 * m)), hid(size_t(3 * m));
  auto half = [&](int64_t h, int64_t& u, int64_t& v, int64_t& w) {
    const int64_t t = h / 3, j = h - 3 * t;
    const int64_t a = T[3 * t + j], b = T[3 * t + (j + 1) % 3];
    w = T[3 * t + (j + 2) % 3];
    u = std::min(a, b);
    v = std::max(a, b);
  };
  for (int64_t h = 0; h < 3 * m; ++h) {
    int64_t u, v, w;
    half(h, u, v, w);
    start[size_t(u) + 1]++;
  }
  for (int64_t i = 0; i < nv; ++i) start[size_t(i) + 1] += start[size_t(i)];
  {
    std::vector<int64_t> fillp(start.begin(), start.end() - 1);
    for (int64_t h = 0; h < 3 * m; ++h) {
      int64_t u, v, w;
      half(h, u, v, w);
      const int64_t k = fillp[size_t(u)]++;
      hv[size_t(k)] = v;
      hid[size_t(k)] = h;  // ascending within a bucket
    }
  }
  std::vector<int64_t> first_of(size_t(3 * m), -1);  // first half-edge -> edge slot
  std::vector<Ent> ents;
  ents.reserve(size_t(1.6 * double(m)) + 8);
  for (int64_t u = 0; u < nv; ++u) {
    const int64_t b0 = start[size_t(u)], b1 = start[size_t(u) + 1];
    for (int64_t k = b0; k < b1; ++k) {
      if (hv[size_t(k)] < 0) continue;  // consumed by an earlier half-edge
      const int64_t v = hv[size_t(k)];
      Ent e{u, v, {-1, -1}, {-1, -1}, 0};
      for (int64_t q = k; q < b1; ++q) {
        if (hv[size_t(q)] != v) continue;
        int64_t uu, vv, w;
        half(hid[size_t(q)], uu, vv, w);
        if (e.cnt < 2) {
          e.t[e.cnt] = hid[size_t(q)] / 3;
          e.w[e.cnt] = w;
        }
        e.cnt++;
        if (q != k) hv[size_t(q)] = -1;
      }
      first_of[size_t(hid[size_t(k)])] = int64_t(ents.size());
      ents.push_back(e);
    }
  }
  {  // insertion order of the reference's dict: by first half-edge
    std::vector<Ent> ordered;
    ordered.reserve(ents.size());
    for (int64_t h = 0; h < 3 * m; ++h)
      if (first_of[size_t(h)] >= 0) ordered.push_back(ents[size_t(first_of[size_t(h)])]);
    ents.swap(ordered);
  }
  struct Cand {
    int64_t u, v, c, q, t1, t2;
    double key;
  };
  std::vector<Cand> cands;
  bool any_interior = false;
  for (const Ent& e : ents) {
    if (e.cnt != 2) continue;
    any_interior = true;
    const int64_t u = e.u, v = e.v, c = e.w[0], q = e.w[1];
    double cx, cy, r2;
    circumcircle(&V[2 * u], &V[2 * v], &V[2 * c], cx, cy, r2);
    const double dist = glibc_hypot(V[2 * q] - cx, V[2 * q + 1] - cy);
    const double depth = std::sqrt(std::max(r2, 0.0)) - dist;
    const bool violate = depth > 1e-9;
    bool want = false;
    if (!violate && std::fabs(depth) <= 1e-9) {
      int64_t best = u;
      for (int64_t j : {v, c, q}) {
        const double jx = V[2 * j], jy = V[2 * j + 1], bx = V[2 * best], by = V[2 * best + 1];
        if (jx < bx || (jx == bx && (jy < by || (jy == by && j < best)))) best = j;
      }
      want = best != u && best != v;
    }
    if (violate || want) cands.push_back(Cand{u, v, c, q, e.t[0], e.t[1], violate ? depth : 0.0});
  }
  if (!any_interior || cands.empty()) return 0;
  std::stable_sort(cands.begin(), cands.end(),
                   [](const Cand& a, const Cand& b) { return -a.key < -b.key; });
  std::vector<uint8_t> dirty(m, 0);
  int64_t flips = 0;
  for (const Cand& k : cands) {
    if (dirty[k.t1] || dirty[k.t2]) continue;
    const double a1 = orient(&V[2 * k.u], &V[2 * k.q], &V[2 * k.c]);
    const double a2 = orient(&V[2 * k.q], &V[2 * k.v], &V[2 * k.c]);
    if (std::fabs(a1) <= 2.0 * 1e-9 || std::fabs(a2) <= 2.0 * 1e-9) continue;
    if ((a1 > 0) != (a2 > 0)) continue;
    int64_t* r1 = &T[3 * k.t1];
    int64_t* r2 = &T[3 * k.t2];
    if (a1 > 0) {
      r1[0] = k.u, r1[1] = k.q, r1[2] = k.c;
      r2[0] = k.q, r2[1] = k.v, r2[2] = k.c;
    } else {
      r1[0] = k.u, r1[1] = k.c, r1[2] = k.q;
      r2[0] = k.q, r2[1] = k.c, r2[2] = k.v;
    }
    dirty[k.t1] = dirty[k.t2] = 1;
    ++flips;
  }
  return flips;
}

}  // namespace

int flip_edges(Tris& t, int passes, std::string& err) {
  err.clear();
  int changed = 0;
  for (int p = 0; p < std::max(passes, 0); ++p) {
    if (flip_sweep(t.V, t.T) == 0) break;
    ++changed;
  }
  if (changed) err = trimesh_init(t);
  return changed;
}

std::string delaunay(const double* points, int64_t n, Tris& out, int& err_kind) {
  err_kind = 1;
  std::vector<double> P;
  std::string e = dedupe_points(points, n, 1e-9, P);
  if (!e.empty()) return e;
  const int64_t np_ = int64_t(P.size() / 2);
  if (np_ < 3) return "need at least 3 distinct points, got " + std::to_string(np_);
  if (all_collinear(P)) return "all points are collinear";
  BowyerWatson bw;
  const char* chk = std::getenv("MESHREG_B200_BW_CHECK");
  bw.check_full = chk && chk[0] == '1';
  const bool dbg = std::getenv("MESHREG_B200_DEBUG") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto tick = [&](const char* what) {
    if (!dbg) return;
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "meshreg_b200: delaunay %-14s %8.1f ms\n", what,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  std::vector<int64_t> T;
  e = bw.run(P, T);
  tick("bowyer-watson");
  if (!e.empty()) {
    err_kind = e.rfind("insertion", 0) == 0 ? 2 : 1;
    return e;
  }
  out.V = std::move(P);
  out.T = std::move(T);
  e = trimesh_init(out);
  tick("trimesh");
  if (!e.empty()) return e;
  const int sweeps = flip_edges(out, 100, e);
  if (dbg) std::fprintf(stderr, "meshreg_b200: delaunay %d flip sweeps\n", sweeps);
  tick("flips");
  return e;
}

// ---------------------------------------------------------------------------
// smooth_mesh, meshgen.py:269-351
namespace {

enum { kFree = 0, kSlideX = 1, kSlideY = 2, kFixed = 3 };

double bilinear(const double* arr, int w, int h, double x, double y) {  // meshgen.py:251-266
  x = std::min(std::max(x, 0.0), w - 1.0);
  y = std::min(std::max(y, 0.0), h - 1.0);
  const int64_t x0 = int64_t(std::min(std::floor(x), double(w > 1 ? w - 2 : 0)));
  const int64_t y0 = int64_t(std::min(std::floor(y), double(h > 1 ? h - 2 : 0)));
  const double tx = x - double(x0), ty = y - double(y0);
  const int64_t x1 = std::min<int64_t>(x0 + 1, w - 1), y1 = std::min<int64_t>(y0 + 1, h - 1);
  const double A = arr[y0 * w + x0], B = arr[y0 * w + x1], C = arr[y1 * w + x0],
               D = arr[y1 * w + x1];
  return A * (1 - tx) * (1 - ty) + B * tx * (1 - ty) + C * (1 - tx) * ty + D * tx * ty;
}

}  // namespace

std::string smooth_mesh(Tris& t, int width, int height, const double* mag, int cvt, int odt) {
  if (cvt == 0 && odt == 0) return "";
  const double w = double(width - 1), h = double(height - 1);
  double mmax = -INFINITY;
  for (int64_t i = 0; i < int64_t(width) * height; ++i) mmax = std::max(mmax, mag[i]);
  double floor_ = 1e-3 * mmax;
  if (1e-6 > floor_) floor_ = 1e-6;
  const int64_t n = t.n();
  std::vector<double>& V = t.V;
  const std::vector<int64_t>& T = t.T;
  std::vector<int> kind(n, kFree);
  const double tol = 1e-6;
  for (int64_t i = 0; i < n; ++i) {
    if (!t.boundary[i]) continue;
    const double x = V[2 * i], y = V[2 * i + 1];
    const bool on_v = x <= tol || x >= w - tol;
    const bool on_h = y <= tol || y >= h - tol;
    kind[i] = (on_v && on_h) ? kFixed : on_v ? kSlideY : on_h ? kSlideX : kFixed;
  }
  std::vector<double> wgt, tx, ty;
  auto relax = [&](bool circum) {
    for (int64_t i = 0; i < n; ++i) {
      if (kind[i] == kFixed) continue;
      const int64_t b0 = t.inc_ptr[i], b1 = t.inc_ptr[i + 1], k = b1 - b0;
      wgt.resize(k);
      tx.resize(k);
      ty.resize(k);
      bool finite = true;
      for (int64_t s = 0; s < k; ++s) {
        const int64_t* r = &T[3 * t.inc_idx[b0 + s]];
        const double *a = &V[2 * r[0]], *b = &V[2 * r[1]], *c = &V[2 * r[2]];
        const double area = 0.5 * ((b[0] - a[0]) * (c[1] - a[1]) - (c[0] - a[0]) * (b[1] - a[1]));
        if (circum) {
          double r2;
          circumcircle(a, b, c, tx[s], ty[s], r2);
        } else {
          tx[s] = (a[0] + b[0] + c[0]) / 3.0;
          ty[s] = (a[1] + b[1] + c[1]) / 3.0;
        }
        if (!std::isfinite(tx[s]) || !std::isfinite(ty[s])) finite = false;
        const double dens = bilinear(mag, width, height, tx[s], ty[s]) + floor_;
        wgt[s] = std::fabs(area) * dens;
      }
      const double total = np_pairwise_sum(wgt.data(), k);
      if (total <= 0 || !finite) continue;
      double sx = wgt[0] * tx[0], sy = wgt[0] * ty[0];
      for (int64_t s = 1; s < k; ++s) {
        sx += wgt[s] * tx[s];
        sy += wgt[s] * ty[s];
      }
      double pos[2] = {sx / total, sy / total};
      // min(max(p, 0.0), w) with Python's builtin semantics
      for (int j = 0; j < 2; ++j) {
        const double hi = j == 0 ? w : h;
        double p = pos[j];
        if (0.0 > p) p = 0.0;
        if (hi < p) p = hi;
        pos[j] = p;
      }
      if (kind[i] == kSlideX) pos[1] = V[2 * i + 1];
      else if (kind[i] == kSlideY) pos[0] = V[2 * i];
      bool inverts = false;
      for (int64_t s = 0; s < k && !inverts; ++s) {
        const int64_t* r = &T[3 * t.inc_idx[b0 + s]];
        const double* p3[3];
        for (int j = 0; j < 3; ++j) p3[j] = r[j] == i ? pos : &V[2 * r[j]];
        const double a2 = (p3[1][0] - p3[0][0]) * (p3[2][1] - p3[0][1]) -
                          (p3[2][0] - p3[0][0]) * (p3[1][1] - p3[0][1]);
        if (a2 <= 2.0 * 1e-9) inverts = true;
      }
      if (inverts) continue;
      V[2 * i] = pos[0];
      V[2 * i + 1] = pos[1];
    }
  };
  for (int s = 0; s < cvt; ++s) relax(false);
  for (int s = 0; s < odt; ++s) relax(true);
  return trimesh_init(t);
}

// ---------------------------------------------------------------------------
void floyd_steinberg(const double* mag, double scale, int width, int height, int serpentine_start,
                     uint8_t* dots) {
  const int64_t W = width, H = height;
  std::vector<double> acc(size_t(W * H));
  for (int64_t i = 0; i < W * H; ++i) acc[i] = mag[i] * scale;
  for (int64_t row = 0; row < H; ++row) {
    const bool reverse = (row + serpentine_start) % 2 == 1;
    const int64_t step = reverse ? -1 : 1;
    for (int64_t s = 0; s < W; ++s) {
      const int64_t col = reverse ? W - 1 - s : s;
      const double v = acc[row * W + col];
      const bool on = v >= 0.5;
      dots[row * W + col] = on;
      const double err = on ? v - 1.0 : v;
      const int64_t ahead = col + step;
      if (0 <= ahead && ahead < W) acc[row * W + ahead] += err * (7.0 / 16.0);
      if (row + 1 < H) {
        const int64_t behind = col - step;
        if (0 <= behind && behind < W) acc[(row + 1) * W + behind] += err * (3.0 / 16.0);
        acc[(row + 1) * W + col] += err * (5.0 / 16.0);
        if (0 <= ahead && ahead < W) acc[(row + 1) * W + ahead] += err * (1.0 / 16.0);
      }
    }
  }
}

void spacing_thin(const double* xy, int64_t n, const int64_t* order, double spacing,
                  int64_t budget, std::vector<double>& out) {
  out.clear();
  const double s = spacing;
  std::unordered_map<uint64_t, std::vector<std::pair<double, double>>> cells;
  auto key = [](int64_t i, int64_t j) {
    return (uint64_t(uint32_t(int32_t(i))) << 32) | uint64_t(uint32_t(int32_t(j)));
  };
  for (int64_t q = 0; q < n; ++q) {
    const int64_t k = order ? order[q] : q;
    const double x = xy[2 * k], y = xy[2 * k + 1];
    const int64_t cx = int64_t(py_floordiv(x, s)), cy = int64_t(py_floordiv(y, s));
    bool ok = true;
    for (int64_t i = cx - 1; i <= cx + 1 && ok; ++i)
      for (int64_t j = cy - 1; j <= cy + 1 && ok; ++j) {
        auto it = cells.find(key(i, j));
        if (it == cells.end()) continue;
        for (const auto& p : it->second)
          if (std::pow(p.first - x, 2.0) + std::pow(p.second - y, 2.0) < s * s) {
            ok = false;
            break;
          }
      }
    if (!ok) continue;
    cells[key(cx, cy)].emplace_back(x, y);
    out.push_back(x);
    out.push_back(y);
    if (int64_t(out.size() / 2) >= budget) break;
  }
}

std::string uniform_sample(int width, int height, int64_t budget, std::vector<double>& out) {
  out.clear();
  if (budget < 4) return "uniform budget must be >= 4, got " + std::to_string(budget);
  int64_t kf = int64_t(std::sqrt(double(budget)));
  while (kf * kf > budget) --kf;
  while ((kf + 1) * (kf + 1) <= budget) ++kf;
  kf = std::max<int64_t>(2, kf);
  const int64_t count_f = kf * kf + std::min(budget - kf * kf, (kf - 1) * (kf - 1));
  const int64_t kc = kf + 1, count_c = kc * kc;
  int64_t k, extra;
  if (std::llabs(count_c - budget) < std::llabs(count_f - budget)) {
    k = kc;
    extra = 0;
  } else {
    k = kf;
    extra = std::min(budget - kf * kf, (kf - 1) * (kf - 1));
  }
  auto linspace = [](double start, double stop, int64_t num) {  // np.linspace
    std::vector<double> y(num);
    const int64_t div = num - 1;
    const double delta = stop - start;
    const double step = delta / double(div);
    for (int64_t i = 0; i < num; ++i)
      y[i] = (step == 0 ? (double(i) / double(div)) * delta : double(i) * step) + start;
    if (num > 1) y[num - 1] = stop;
    return y;
  };
  const std::vector<double> xs = linspace(0.0, width - 1.0, k), ys = linspace(0.0, height - 1.0, k);
  for (int64_t i = 0; i < k; ++i)
    for (int64_t j = 0; j < k; ++j) {
      out.push_back(xs[j]);
      out.push_back(ys[i]);
    }
  if (extra > 0) {
    int64_t c = 0;
    for (int64_t i = 0; i + 1 < k && c < extra; ++i)
      for (int64_t j = 0; j + 1 < k && c < extra; ++j, ++c) {
        out.push_back(0.5 * (xs[j] + xs[j + 1]));
        out.push_back(0.5 * (ys[i] + ys[i + 1]));
      }
  }
  return "";
}

}  // namespace mrb
