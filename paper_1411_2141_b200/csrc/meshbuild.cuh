// Device-side mesh setup for deferred mesh handles (mrb_mesh_create_many).
//
// The reference builds a TriMesh and its TriangleGeometry on the host before
// registering (mesh.py:58-123 connectivity, 153-159 signed area, 173-213
// areas / Eq. 9 coefficients / vertex areas, 236-241 the gradient operators
// avg∘grad, 254-265 the one-ring Laplacian).  For a batch of meshes whose
// handles were only validated and oriented on the host, this file builds on
// the GPU everything the fp32 cluster fast path reads, bit-identical to the
// host build (mesh_host.cpp build_mesh, meshreg_b200.cu plan_topo/write_topo):
//
//   k_mesh_build_a (one 8-CTA cluster per mesh: cluster barriers between the
//       phases, scans and reductions through distributed shared memory)
//       areas + coefficients (exact fp64 op order: explicit _rn intrinsics,
//       never a contracted FMA), incident
//       lists (ascending triangle id), vertex areas in np.add.at order, the
//       sorted one-rings with their use counts (non-manifold / valence
//       checks), Morton keys of the vertices
//   cub radix sort (stable) of (mesh << 32 | Morton key, vertex)  = the host's
//       std::stable_sort of the node order
//   k_mesh_build_b (one 8-CTA cluster per mesh)  iperm, one-ring CSR in
//       device ids, the fused operator G accumulated over incident triangles
//       in the host's order, 1/valence, device-order vertices and triangles
//   k_topo_count / k_topo_write / k_topo_send (one CTA per (mesh, cluster
//       rank))  the paired SELL-32 topology of a cluster shape: slice pair
//       rows, halo lists in first-reference order (shared-memory hash with
//       atomicMin of the first entry), 16-bit codes, fp32 coefficients, push
//       send lists
//
// Every kernel is integer / gather work bound by latency on a few MB per mesh.
#pragma once

#include <cstdint>

#include <cooperative_groups.h>

#include "cluster.cuh"

namespace mrb {

constexpr int kBuildThreads = 512;
constexpr int kBuildMaxInc = 24;  // incident triangles per vertex (else: host build)
constexpr int kTopoThreads = 512;
constexpr int kTopoHash = 2048;   // distinct remote nodes per CTA (else: host plan)
constexpr int kTopoMaxSlices = 256;  // 8192 slots per CTA (grid shapes: 768 x 8)

enum BuildFlag : int {
  kBuildOverflow = 1,     // a vertex with more than kBuildMaxInc triangles
  kBuildNonManifold = 2,  // an edge of more than two triangles (mesh.py:99-100)
  kBuildLone = 4,         // a vertex of valence < 2 (mesh.py:119-122)
};

struct BuildJob {
  int n, m, mesh;
  int ring_cap;      // capacity of ring_idx / nb_idx / g_nb (3m + n >= 2e when manifold)
  const double2* V;  // original order
  const int* T;      // m*3, CCW-oriented, original ids
  // scratch
  double* areas;     // m
  double* coeffs;    // m*6  [t][corner][xy]
  int* cnt;          // n
  int* inc_ptr;      // n+1
  int* inc_idx;      // 3m
  unsigned char* cpos;  // 6m: ring position of the two other corners of each incident triangle
  int* valence;      // n
  int* ring_ptr;     // n+1
  int* ring_idx;     // ring_cap
  double* varea;     // n
  int* iperm;        // n
  unsigned long long* key;  // n  (segment of the sort input)
  int* val;                 // n
  const int* sorted;        // n  (segment of the sort output: vertex per device id)
  // kept for topology builds
  int* nb_ptr;       // n+1
  int* nb_idx;       // ring_cap
  double2* g_nb;     // ring_cap
  // DeviceMesh arrays
  double2* Vn;
  int4* tri;
  int* perm;
  float2* g_self_f;
  float* inv_val_f;
  double2* g_self_d;  // fp64 self terms and 1/valence (k_cluster64), or null
  double* inv_val_d;
  int* stats;        // [0] flags, [1] max valence, [2] nnz one-ring (2e)
};

// ---- cluster helpers: one thread-block cluster of kBuildCluster CTAs per mesh ----

constexpr int kBuildCluster = 8;

// one CTA: out[i] = carry + value(b0) + ... + value(i-1) for i in [b0, b1)
template <typename F>
__device__ int cta_scan_range(int b0, int b1, int carry, F value, int* out, int* s_tmp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int base = b0; base < b1; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int v = i < b1 ? value(i) : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_tmp[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int w = lane < nw ? s_tmp[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      if (lane < nw) s_tmp[lane] = w;
    }
    __syncthreads();
    if (i < b1) out[i] = carry + (warp ? s_tmp[warp - 1] : 0) + x - v;
    carry += s_tmp[nw - 1];
    __syncthreads();
  }
  return carry;
}

template <typename T, typename Op>
__device__ T cta_reduce(T v, Op op, T* s_tmp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) s_tmp[warp] = v;
  __syncthreads();
  T r = s_tmp[0];
  for (int k = 1; k < nw; ++k) r = op(r, s_tmp[k]);
  __syncthreads();
  return r;
}

// exclusive scan over [0, n) by the whole cluster: CTA r owns the r-th
// segment; segment totals are exchanged through distributed shared memory.
// out[n] = total.  Ends with a cluster barrier.
template <typename F>
__device__ void cluster_exclusive_scan(int n, F value, int* out, int* s_tmp, int* s_tot) {
  cg::cluster_group cluster = cg::this_cluster();
  const int r = int(cluster.block_rank());
  const int seg = (n + kBuildCluster - 1) / kBuildCluster;
  const int b0 = min(n, r * seg), b1 = min(n, b0 + seg);
  int part = 0;
  for (int i = b0 + int(threadIdx.x); i < b1; i += blockDim.x) part += value(i);
  part = cta_reduce(part, [](int x, int y) { return x + y; }, s_tmp);
  if (threadIdx.x == 0) *s_tot = part;
  cluster.sync();
  int carry = 0;
  for (int q = 0; q < r; ++q) carry += *cluster.map_shared_rank(s_tot, q);
  carry = cta_scan_range(b0, b1, carry, value, out, s_tmp);
  if (r == kBuildCluster - 1 && threadIdx.x == 0) out[n] = carry;
  cluster.sync();
}

// min / max of a double over the cluster (every CTA gets the result)
template <typename Op>
__device__ double cluster_reduce(double v, Op op, double* s_red, double* s_out) {
  cg::cluster_group cluster = cg::this_cluster();
  v = cta_reduce(v, op, s_red);
  if (threadIdx.x == 0) *s_out = v;
  cluster.sync();
  double r = *cluster.map_shared_rank(s_out, 0);
  for (unsigned q = 1; q < kBuildCluster; ++q) r = op(r, *cluster.map_shared_rank(s_out, q));
  cluster.sync();  // s_out may be reused
  return r;
}

__device__ __forceinline__ uint32_t spread16_d(uint32_t x) {
  x &= 0xFFFF;
  x = (x | (x << 8)) & 0x00FF00FF;
  x = (x | (x << 4)) & 0x0F0F0F0F;
  x = (x | (x << 2)) & 0x33333333;
  x = (x | (x << 1)) & 0x55555555;
  return x;
}

template <typename T>
__device__ __forceinline__ void insertion_sort(T* a, int k) {
  for (int x = 1; x < k; ++x) {
    const T v = a[x];
    int c = x - 1;
    for (; c >= 0 && a[c] > v; --c) a[c + 1] = a[c];
    a[c + 1] = v;
  }
}

// one-ring of vertex v from its (sorted) incident triangles: sorted neighbour
// list with duplicates (each neighbour once per triangle sharing the edge)
__device__ __forceinline__ int gather_ring(const BuildJob& J, int v, int b0, int k,
                                           int (&nb)[2 * kBuildMaxInc]) {
  int c = 0;
  for (int q = 0; q < k; ++q) {
    const int t = J.inc_idx[b0 + q];
#pragma unroll
    for (int x = 0; x < 3; ++x) {
      const int j = J.T[3 * t + x];
      if (j != v) nb[c++] = j;
    }
  }
  insertion_sort(nb, c);
  return c;
}

// ---- per-element steps (shared by the cluster kernels and the grid kernels) ----

// TriangleGeometry (mesh.py:173-197; host: mesh_host.cpp build_mesh) of
// triangle t and its three incidence counts
__device__ __forceinline__ void build_tri(const BuildJob& J, int t) {
  const int ia = J.T[3 * t], ib = J.T[3 * t + 1], ic = J.T[3 * t + 2];
  const double2 A = J.V[ia], B = J.V[ib], Cc = J.V[ic];
  const double a[2] = {A.x, A.y}, b[2] = {B.x, B.y}, c[2] = {Cc.x, Cc.y};
  const double a2 = __dsub_rn(__dmul_rn(__dsub_rn(b[0], a[0]), __dsub_rn(c[1], a[1])),
                              __dmul_rn(__dsub_rn(c[0], a[0]), __dsub_rn(b[1], a[1])));
  const double ar = __dmul_rn(0.5, a2);
  J.areas[t] = ar;
  const double vij[2] = {__dsub_rn(b[0], a[0]), __dsub_rn(b[1], a[1])};
  const double vjk[2] = {__dsub_rn(c[0], b[0]), __dsub_rn(c[1], b[1])};
  const double vik[2] = {__dsub_rn(c[0], a[0]), __dsub_rn(c[1], a[1])};
  auto dot = [](const double* u, double w0, double w1) {
    return __dadd_rn(__dmul_rn(u[0], w0), __dmul_rn(u[1], w1));
  };
  const double di1 = dot(vij, vjk[0], vjk[1]), di2 = dot(vik, -vjk[0], -vjk[1]);
  const double nvij[2] = {-vij[0], -vij[1]}, nvjk[2] = {-vjk[0], -vjk[1]};
  const double nvik[2] = {-vik[0], -vik[1]};
  const double dj1 = dot(nvij, vik[0], vik[1]), dj2 = dot(vjk, -vik[0], -vik[1]);
  const double dk1 = dot(nvjk, -vij[0], -vij[1]), dk2 = dot(nvik, vij[0], vij[1]);
  const double inv4a2 = __ddiv_rn(1.0, __dmul_rn(4.0, __dmul_rn(ar, ar)));
  double* co = J.coeffs + 6 * size_t(t);
#pragma unroll
  for (int d = 0; d < 2; ++d) {
    const double ti = __dadd_rn(__dmul_rn(di1, __dsub_rn(c[d], a[d])),
                                __dmul_rn(di2, __dsub_rn(b[d], a[d])));
    const double tj = __dadd_rn(__dmul_rn(dj1, __dsub_rn(c[d], b[d])),
                                __dmul_rn(dj2, __dsub_rn(a[d], b[d])));
    const double tk = __dadd_rn(__dmul_rn(dk1, __dsub_rn(a[d], c[d])),
                                __dmul_rn(dk2, __dsub_rn(b[d], c[d])));
    co[0 * 2 + d] = __dmul_rn(ti, inv4a2);
    co[1 * 2 + d] = __dmul_rn(tj, inv4a2);
    co[2 * 2 + d] = __dmul_rn(tk, inv4a2);
  }
  atomicAdd(J.cnt + ia, 1);
  atomicAdd(J.cnt + ib, 1);
  atomicAdd(J.cnt + ic, 1);
}

__device__ __forceinline__ void build_fill(const BuildJob& J, int t) {
#pragma unroll
  for (int x = 0; x < 3; ++x) {
    const int v = J.T[3 * t + x];
    J.inc_idx[J.inc_ptr[v] + atomicAdd(J.cnt + v, 1)] = t;
  }
}

// vertex v: incident list ascending (mesh.py:106-110), vertex area in
// np.add.at's (triangle, corner) order (mesh.py:209-211), valence, edge use
// counts, ring positions of the incident triangles' corners; returns flags
__device__ __forceinline__ int build_vertex(const BuildJob& J, int v) {
  const int b0 = J.inc_ptr[v], k = J.inc_ptr[v + 1] - b0;
  if (k > kBuildMaxInc) {
    J.valence[v] = 0;
    J.varea[v] = 0.0;
    return kBuildOverflow;
  }
  int flags = 0;
  int tl[kBuildMaxInc];
  for (int q = 0; q < k; ++q) tl[q] = J.inc_idx[b0 + q];
  insertion_sort(tl, k);
  double va = 0.0;
  for (int q = 0; q < k; ++q) {
    J.inc_idx[b0 + q] = tl[q];
    va = __dadd_rn(va, J.areas[tl[q]]);
  }
  J.varea[v] = va;
  // neighbour id << 6 | origin (2 q + s: the s-th other corner of the q-th
  // incident triangle): sorted, equal ids adjacent; the ring position of
  // every origin (cpos) spares pass B a search per corner
  int nb[2 * kBuildMaxInc];
  int c = 0;
  for (int q = 0; q < k; ++q) {
    int sidx = 0;
#pragma unroll
    for (int x = 0; x < 3; ++x) {
      const int j = J.T[3 * tl[q] + x];
      if (j != v) nb[c++] = j << 6 | (2 * q + sidx++);
    }
  }
  insertion_sort(nb, c);
  int val = 0;
  for (int x = 0; x < c;) {
    int y = x;
    while (y < c && (nb[y] >> 6) == (nb[x] >> 6)) {
      J.cpos[2 * size_t(b0) + (nb[y] & 63)] = (unsigned char)val;
      ++y;
    }
    if (y - x > 2) flags |= kBuildNonManifold;
    ++val;
    x = y;
  }
  J.valence[v] = val;
  if (val < 2) flags |= kBuildLone;
  return flags;
}

// sorted one-ring of v (mesh.py:101-104,116) at ring_ptr[v]
__device__ __forceinline__ void build_ring(const BuildJob& J, int v) {
  const int b0 = J.inc_ptr[v], k = J.inc_ptr[v + 1] - b0;
  if (k > kBuildMaxInc) return;
  int nb[2 * kBuildMaxInc];
  const int c = gather_ring(J, v, b0, k, nb);
  int* out = J.ring_idx + J.ring_ptr[v];
  int w = 0;
  for (int x = 0; x < c; ++x)
    if (x == 0 || nb[x] != nb[x - 1]) out[w++] = nb[x];
}

// Morton (Z-order) key of v for the node relabelling (host: build_mesh)
__device__ __forceinline__ void build_key(const BuildJob& J, int v, double lo0, double lo1,
                                          double span) {
  const double2 p = J.V[v];
  const uint32_t qx = __double2uint_rz(
      fmin(65535.0, __dmul_rn(__ddiv_rn(__dsub_rn(p.x, lo0), span), 65535.0)));
  const uint32_t qy = __double2uint_rz(
      fmin(65535.0, __dmul_rn(__ddiv_rn(__dsub_rn(p.y, lo1), span), 65535.0)));
  J.key[v] = (static_cast<unsigned long long>(J.mesh) << 32) |
             (spread16_d(qx) | (spread16_d(qy) << 1));
  J.val[v] = v;
}

__device__ __forceinline__ void build_perm(const BuildJob& J, int k) {
  const int i = J.sorted[k];
  J.perm[k] = i;
  J.iperm[i] = k;
}

// device id k: one-ring CSR row and the fused operator G = avg∘grad on
// {self} ∪ one-ring (mesh.py:199-213,236-241), incident triangles ascending,
// corners in order, as the host accumulates; returns the valence
__device__ __forceinline__ int build_row(const BuildJob& J, int k) {
  const int i = J.perm[k];
  const int deg = J.valence[i], rb = J.ring_ptr[i], base = J.nb_ptr[k];
  const int* ring = J.ring_idx + rb;
  double gx[2 * kBuildMaxInc], gy[2 * kBuildMaxInc];
  for (int r = 0; r < deg; ++r) {
    J.nb_idx[base + r] = J.iperm[ring[r]];
    gx[r] = gy[r] = 0.0;
  }
  double sx = 0.0, sy = 0.0;
  const int q0 = J.inc_ptr[i], q1 = J.inc_ptr[i + 1];
  const double va = J.varea[i];
  for (int q = q0; q < q1 && q1 - q0 <= kBuildMaxInc; ++q) {
    const int t = J.inc_idx[q];
    const double w = __ddiv_rn(J.areas[t], va);
    const double* co = J.coeffs + 6 * size_t(t);
    int sidx = 0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int j = J.T[3 * t + c];
      const double cx = __dmul_rn(w, co[2 * c]);
      const double cy = __dmul_rn(w, co[2 * c + 1]);
      if (j == i) {
        sx = __dadd_rn(sx, cx);
        sy = __dadd_rn(sy, cy);
      } else {
        const int pos = min(int(J.cpos[2 * size_t(q) + sidx++]), max(deg - 1, 0));
        gx[pos] = __dadd_rn(gx[pos], cx);
        gy[pos] = __dadd_rn(gy[pos], cy);
      }
    }
  }
  for (int r = 0; r < deg; ++r) J.g_nb[base + r] = make_double2(gx[r], gy[r]);
  J.g_self_f[k] = make_float2(__double2float_rn(sx), __double2float_rn(sy));
  const double iv = __ddiv_rn(1.0, double(max(deg, 1)));
  J.inv_val_f[k] = __double2float_rn(iv);
  if (J.g_self_d) {
    J.g_self_d[k] = make_double2(sx, sy);
    J.inv_val_d[k] = iv;
  }
  J.Vn[k] = J.V[i];
  return deg;
}

__device__ __forceinline__ void build_tri_out(const BuildJob& J, int t) {
  J.tri[t] = make_int4(J.iperm[J.T[3 * t]], J.iperm[J.T[3 * t + 1]], J.iperm[J.T[3 * t + 2]], 0);
}

// ---- pass A: geometry, incidence, one-rings, Morton keys ---------------------
__global__ void __cluster_dims__(kBuildCluster, 1, 1) __launch_bounds__(kBuildThreads)
    k_mesh_build_a(const BuildJob* __restrict__ jobs) {
  cg::cluster_group cluster = cg::this_cluster();
  const BuildJob J = jobs[blockIdx.x / kBuildCluster];
  __shared__ int s_tmp[33];
  __shared__ int s_tot;
  __shared__ double s_red[32];
  __shared__ double s_out;
  __shared__ int s_flags;
  const int n = J.n, m = J.m;
  const int nt = kBuildCluster * int(blockDim.x);
  const int tid = int(cluster.block_rank()) * int(blockDim.x) + int(threadIdx.x);
  if (threadIdx.x == 0) s_flags = 0;
  for (int v = tid; v < n; v += nt) J.cnt[v] = 0;
  cluster.sync();
  for (int t = tid; t < m; t += nt) build_tri(J, t);
  cluster.sync();
  cluster_exclusive_scan(n, [&](int v) { return J.cnt[v]; }, J.inc_ptr, s_tmp, &s_tot);
  for (int v = tid; v < n; v += nt) J.cnt[v] = 0;
  cluster.sync();
  for (int t = tid; t < m; t += nt) build_fill(J, t);
  cluster.sync();
  int flags = 0;
  for (int v = tid; v < n; v += nt) flags |= build_vertex(J, v);
  if (flags) atomicOr(&s_flags, flags);
  cluster.sync();
  cluster_exclusive_scan(n, [&](int v) { return J.valence[v]; }, J.ring_ptr, s_tmp, &s_tot);
  const bool ring_fits = J.ring_ptr[n] <= J.ring_cap;  // else non-manifold: flagged
  if (!ring_fits && tid == 0) atomicOr(J.stats, kBuildOverflow);
  for (int v = tid; v < n && ring_fits; v += nt) build_ring(J, v);
  double lo0 = INFINITY, lo1 = INFINITY, hi0 = -INFINITY, hi1 = -INFINITY;
  for (int v = tid; v < n; v += nt) {
    const double2 p = J.V[v];
    lo0 = fmin(lo0, p.x);
    lo1 = fmin(lo1, p.y);
    hi0 = fmax(hi0, p.x);
    hi1 = fmax(hi1, p.y);
  }
  auto mn = [](double x, double y) { return fmin(x, y); };
  auto mx = [](double x, double y) { return fmax(x, y); };
  lo0 = cluster_reduce(lo0, mn, s_red, &s_out);
  lo1 = cluster_reduce(lo1, mn, s_red, &s_out);
  hi0 = cluster_reduce(hi0, mx, s_red, &s_out);
  hi1 = cluster_reduce(hi1, mx, s_red, &s_out);
  const double span = fmax(fmax(__dsub_rn(hi0, lo0), __dsub_rn(hi1, lo1)), 1e-12);
  for (int v = tid; v < n; v += nt) build_key(J, v, lo0, lo1, span);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_flags) atomicOr(J.stats, s_flags);
    if (cluster.block_rank() == 0) J.stats[2] = J.ring_ptr[n];
  }
}

// ---- pass B: device order, one-ring CSR, fused operator G ---------------------
__global__ void __cluster_dims__(kBuildCluster, 1, 1) __launch_bounds__(kBuildThreads)
    k_mesh_build_b(const BuildJob* __restrict__ jobs) {
  cg::cluster_group cluster = cg::this_cluster();
  const BuildJob J = jobs[blockIdx.x / kBuildCluster];
  __shared__ int s_tmp[33];
  __shared__ int s_tot;
  __shared__ int s_red[32];
  const int n = J.n, m = J.m;
  if (J.ring_ptr[n] > J.ring_cap) return;  // flagged by pass A (uniform over the cluster)
  const int nt = kBuildCluster * int(blockDim.x);
  const int tid = int(cluster.block_rank()) * int(blockDim.x) + int(threadIdx.x);
  for (int k = tid; k < n; k += nt) build_perm(J, k);
  cluster.sync();
  cluster_exclusive_scan(n, [&](int k) { return J.valence[J.perm[k]]; }, J.nb_ptr, s_tmp, &s_tot);
  int dmax = 0;
  for (int k = tid; k < n; k += nt) dmax = max(dmax, build_row(J, k));
  for (int t = tid; t < m; t += nt) build_tri_out(J, t);
  dmax = cta_reduce(dmax, [](int x, int y) { return max(x, y); }, s_red);
  if (threadIdx.x == 0) atomicMax(J.stats + 1, dmax);
}

// ---- the same steps as grid-wide kernels, for one large mesh ------------------
// (a single cluster of kBuildCluster CTAs per mesh would serialise a C5-size
// mesh; the scans between the steps are CUB device scans)
__global__ void k_bg_tri(const BuildJob* __restrict__ j) {
  const BuildJob& J = *j;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < J.m; t += gridDim.x * blockDim.x)
    build_tri(J, t);
}
__global__ void k_bg_fill(const BuildJob* __restrict__ j) {
  const BuildJob& J = *j;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < J.m; t += gridDim.x * blockDim.x)
    build_fill(J, t);
}
// vertices; block partials of the coordinate bounds into bounds[block][4]
__global__ void k_bg_vertex(const BuildJob* __restrict__ j, double4* __restrict__ bounds) {
  const BuildJob& J = *j;
  __shared__ double s_red[32];
  int flags = 0;
  double lo0 = INFINITY, lo1 = INFINITY, hi0 = -INFINITY, hi1 = -INFINITY;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < J.n; v += gridDim.x * blockDim.x) {
    flags |= build_vertex(J, v);
    const double2 p = J.V[v];
    lo0 = fmin(lo0, p.x);
    lo1 = fmin(lo1, p.y);
    hi0 = fmax(hi0, p.x);
    hi1 = fmax(hi1, p.y);
  }
  if (flags) atomicOr(J.stats, flags);
  auto mn = [](double x, double y) { return fmin(x, y); };
  auto mx = [](double x, double y) { return fmax(x, y); };
  lo0 = cta_reduce(lo0, mn, s_red);
  lo1 = cta_reduce(lo1, mn, s_red);
  hi0 = cta_reduce(hi0, mx, s_red);
  hi1 = cta_reduce(hi1, mx, s_red);
  if (threadIdx.x == 0) bounds[blockIdx.x] = make_double4(lo0, lo1, hi0, hi1);
}
// rings + keys (bounds reduced by every block in the same order)
__global__ void k_bg_ring_key(const BuildJob* __restrict__ j, const double4* __restrict__ bounds,
                              int nbounds) {
  const BuildJob& J = *j;
  double lo0 = INFINITY, lo1 = INFINITY, hi0 = -INFINITY, hi1 = -INFINITY;
  for (int b = 0; b < nbounds; ++b) {
    const double4 q = bounds[b];
    lo0 = fmin(lo0, q.x);
    lo1 = fmin(lo1, q.y);
    hi0 = fmax(hi0, q.z);
    hi1 = fmax(hi1, q.w);
  }
  const double span = fmax(fmax(__dsub_rn(hi0, lo0), __dsub_rn(hi1, lo1)), 1e-12);
  const bool ring_fits = J.ring_ptr[J.n] <= J.ring_cap;
  const int first = blockIdx.x * blockDim.x + threadIdx.x;
  if (first == 0) {
    if (!ring_fits) atomicOr(J.stats, kBuildOverflow);
    J.stats[2] = J.ring_ptr[J.n];
  }
  for (int v = first; v < J.n; v += gridDim.x * blockDim.x) {
    if (ring_fits) build_ring(J, v);
    build_key(J, v, lo0, lo1, span);
  }
}
// device order; the permuted valences into cnt (scanned into nb_ptr next)
__global__ void k_bg_perm(const BuildJob* __restrict__ j) {
  const BuildJob& J = *j;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < J.n; k += gridDim.x * blockDim.x) {
    build_perm(J, k);
    J.cnt[k] = J.valence[J.sorted[k]];
  }
}
__global__ void k_bg_rows(const BuildJob* __restrict__ j) {
  const BuildJob& J = *j;
  __shared__ int s_red[32];
  if (J.ring_ptr[J.n] > J.ring_cap) return;
  int dmax = 0;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < J.n; k += gridDim.x * blockDim.x)
    dmax = max(dmax, build_row(J, k));
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < J.m; t += gridDim.x * blockDim.x)
    build_tri_out(J, t);
  dmax = cta_reduce(dmax, [](int x, int y) { return max(x, y); }, s_red);
  if (threadIdx.x == 0) atomicMax(J.stats + 1, dmax);
}

// ---- cluster topology (host twin: plan_topo + write_topo) --------------------
struct TopoJob {
  int n, cs, chunk, slices, slots;
  const int* nb_ptr;
  const int* nb_idx;
  const double2* g_nb;
  int* stat;  // [cs][3] stride_r, n_halo_r, flags; then n_send [cs]
  // write pass (slab zeroed beforehand)
  uint16_t* codes;
  float2* g;
  double2* g64;      // fp64 coefficients instead (k_cluster64 topologies), or null
  uint32_t* soff;
  uint32_t* halo;
  int* n_halo;
  unsigned char* deg;
  uint32_t* send;
  int* n_send;
  int stride, hstride, sstride;
};

__device__ __forceinline__ int topo_hash(int j) {
  return int((uint32_t(j) * 2654435761u) >> (32 - 11)) & (kTopoHash - 1);
}

// slice pair rows of CTA r (warp per slice) into s_pairs; returns nothing
__device__ __forceinline__ void topo_slices(const TopoJob& J, int r, int* s_pairs) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int sl = warp; sl < J.slices; sl += nw) {
    const int s = sl * 32 + lane;
    const int i = r * J.chunk + s;
    const int d = (s < J.chunk && i < J.n) ? J.nb_ptr[i + 1] - J.nb_ptr[i] : 0;
    const int mx = __reduce_max_sync(0xffffffffu, d);
    if (lane == 0) s_pairs[sl] = (mx + 1) / 2;
  }
}

// insert remote node j; returns its hash slot (-1: table full)
__device__ __forceinline__ int topo_insert(int* s_key, int j, bool* fresh) {
  int h = topo_hash(j);
  *fresh = false;
  for (int p = 0; p < kTopoHash; ++p) {
    const int prev = atomicCAS(s_key + h, -1, j);
    if (prev == -1) {
      *fresh = true;
      return h;
    }
    if (prev == j) return h;
    h = (h + 1) & (kTopoHash - 1);
  }
  return -1;
}

__device__ __forceinline__ int topo_find(const int* s_key, int j) {
  int h = topo_hash(j);
  for (int p = 0; p < kTopoHash; ++p) {
    if (s_key[h] == j) return h;
    h = (h + 1) & (kTopoHash - 1);
  }
  return -1;
}

// pass 1: per (mesh, rank) the block stride, the number of distinct remote
// nodes (halo size) and, per owner, the send-list counts
__global__ void __launch_bounds__(kTopoThreads) k_topo_count(const TopoJob* __restrict__ jobs) {
  const TopoJob J = jobs[blockIdx.y];
  const int r = blockIdx.x;
  if (r >= J.cs) return;
  __shared__ int s_key[kTopoHash];
  __shared__ int s_pairs[kTopoMaxSlices];
  __shared__ int s_cnt, s_flag;
  for (int h = threadIdx.x; h < kTopoHash; h += blockDim.x) s_key[h] = -1;
  if (threadIdx.x == 0) s_cnt = s_flag = 0;
  if (J.slices > kTopoMaxSlices) {
    if (threadIdx.x == 0) J.stat[3 * r + 2] = 1;
    return;
  }
  topo_slices(J, r, s_pairs);
  __syncthreads();
  const int k0 = min(J.n, r * J.chunk), k1 = min(J.n, r * J.chunk + J.chunk);
  const int q0 = J.nb_ptr[k0], q1 = J.nb_ptr[k1];
  for (int q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
    const int j = J.nb_idx[q];
    if (unsigned(j) >= unsigned(J.n)) {
      s_flag = 1;
      continue;
    }
    const int rj = j / J.chunk;
    if (rj == r) continue;
    bool fresh;
    if (topo_insert(s_key, j, &fresh) < 0) {
      s_flag = 1;
    } else if (fresh) {
      atomicAdd(&s_cnt, 1);
      atomicAdd(J.stat + 3 * J.cs + rj, 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int sl = 0; sl < J.slices; ++sl) acc += 32 * s_pairs[sl];
    J.stat[3 * r] = 2 * acc;
    J.stat[3 * r + 1] = s_cnt;
    J.stat[3 * r + 2] = s_flag || s_cnt > kTopoHash * 3 / 4;
  }
}

// pass 2: slice offsets, halo list (first-reference order), codes +
// coefficients in the paired SELL-32 layout, degrees
__global__ void __launch_bounds__(kTopoThreads) k_topo_write(const TopoJob* __restrict__ jobs) {
  const TopoJob J = jobs[blockIdx.y];
  const int r = blockIdx.x;
  if (r >= J.cs) return;
  __shared__ int s_key[kTopoHash];
  __shared__ int s_pos[kTopoHash];
  __shared__ int s_list[kTopoHash];
  __shared__ uint32_t s_soff[kTopoMaxSlices];
  __shared__ int s_pairs[kTopoMaxSlices];
  __shared__ int s_cnt;
  const uint16_t zero = uint16_t(J.slots + J.hstride - 1);
  for (int e = threadIdx.x; e < J.stride; e += blockDim.x)
    J.codes[size_t(r) * J.stride + e] = zero;
  for (int h = threadIdx.x; h < kTopoHash; h += blockDim.x) {
    s_key[h] = -1;
    s_pos[h] = INT_MAX;
  }
  if (threadIdx.x == 0) s_cnt = 0;
  topo_slices(J, r, s_pairs);
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int sl = 0; sl < J.slices; ++sl) {
      s_soff[sl] = uint32_t(s_pairs[sl]) << 24 | uint32_t(acc);
      J.soff[size_t(r) * J.slices + sl] = s_soff[sl];
      acc += 32 * s_pairs[sl];
    }
  }
  const int k0 = min(J.n, r * J.chunk), k1 = min(J.n, r * J.chunk + J.chunk);
  const int q0 = J.nb_ptr[k0], q1 = J.nb_ptr[k1];
  for (int q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
    const int j = J.nb_idx[q];
    if (j / J.chunk == r) continue;
    bool fresh;
    const int h = topo_insert(s_key, j, &fresh);
    atomicMin(s_pos + h, q);
  }
  __syncthreads();
  for (int h = threadIdx.x; h < kTopoHash; h += blockDim.x)
    if (s_key[h] >= 0) s_list[atomicAdd(&s_cnt, 1)] = h;
  __syncthreads();
  // halo index = rank of the node's first reference among the CTA's entries
  const int cnt = s_cnt;
  constexpr int kPer = kTopoHash / kTopoThreads;
  int rank[kPer];
#pragma unroll
  for (int x = 0; x < kPer; ++x) {
    const int a = threadIdx.x + x * blockDim.x;
    rank[x] = 0;
    if (a >= cnt) continue;
    const int pa = s_pos[s_list[a]];
    int rk = 0;
    for (int b = 0; b < cnt; ++b) rk += s_pos[s_list[b]] < pa;
    rank[x] = rk;
  }
  __syncthreads();
#pragma unroll
  for (int x = 0; x < kPer; ++x) {
    const int a = threadIdx.x + x * blockDim.x;
    if (a >= cnt) continue;
    const int h = s_list[a];
    const int j = s_key[h], rj = j / J.chunk;
    s_pos[h] = rank[x];
    J.halo[size_t(r) * J.hstride + rank[x]] = uint32_t(rj << 16 | (j - rj * J.chunk));
  }
  if (threadIdx.x == 0) J.n_halo[r] = cnt;
  __syncthreads();
  for (int s = threadIdx.x; s < J.chunk; s += blockDim.x) {
    const int i = r * J.chunk + s;
    if (i >= J.n) break;
    const int b = J.nb_ptr[i], e = J.nb_ptr[i + 1];
    J.deg[i] = (unsigned char)(e - b);
    const size_t base =
        size_t(r) * J.stride + 2 * size_t((s_soff[s / 32] & 0xffffffu) + (s % 32));
    for (int q = b; q < e; ++q) {
      const int k = q - b, j = J.nb_idx[q];
      const size_t at = base + 64 * size_t(k >> 1) + (k & 1);
      const uint16_t code = j / J.chunk == r ? uint16_t(j - r * J.chunk)
                                             : uint16_t(J.slots + s_pos[topo_find(s_key, j)]);
      J.codes[at] = code;
      const double2 gq = J.g_nb[q];
      if (J.g64)
        J.g64[at] = gq;
      else
        J.g[at] = make_float2(__double2float_rn(gq.x), __double2float_rn(gq.y));
    }
  }
}

// pass 3: push send lists, the inverse of the halo lists in (consumer CTA,
// halo index) order
__global__ void __launch_bounds__(256) k_topo_send(const TopoJob* __restrict__ jobs) {
  const TopoJob J = jobs[blockIdx.y];
  const int r = blockIdx.x;
  if (r >= J.cs || J.sstride == 0) return;
  __shared__ int s_w[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int out = 0;
  for (int c = 0; c < J.cs; ++c) {
    const int nh = J.n_halo[c];
    for (int base = 0; base < nh; base += blockDim.x) {
      const int hh = base + threadIdx.x;
      const uint32_t e = hh < nh ? J.halo[size_t(c) * J.hstride + hh] : 0u;
      const bool f = hh < nh && int(e >> 16) == r;
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      if (lane == 0) s_w[warp] = __popc(bal);
      __syncthreads();
      int before = 0, tot = 0;
      for (int w = 0; w < nw; ++w) {
        if (w < warp) before += s_w[w];
        tot += s_w[w];
      }
      if (f)
        J.send[size_t(r) * J.sstride + out + before + __popc(bal & ((1u << lane) - 1))] =
            (e & 0xffffu) << 20 | uint32_t(c) << 16 | uint32_t(hh);
      out += tot;
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) J.n_send[r] = out;
}

}  // namespace mrb
