// Persistent thread-block-cluster registration kernel (fp32 fast path).
//
// One cluster of CS CTAs (CS <= 16) owns one pair for the whole descent loop
// (solver.py:171-195).  CTA r owns the contiguous chunk [r*chunk, (r+1)*chunk)
// of the device (Morton) node order; thread t owns slots t, t+768, ... (NPT
// slots).  Per-node constants live in shared memory; u and r in registers.
//
// Neighbour exchange = ghost (halo) exchange over DSMEM: each CTA keeps its
// own values followed by a halo region holding copies of the remote nodes its
// one-rings reference.  After each cluster barrier the CTA pulls exactly its
// halo (one ld.shared::cluster per halo node), so every one-ring gather of the
// fused gradient operator G = avg∘grad (mesh.py:236-241) and of the umbrella
// Laplacian (mesh.py:254-282) is a local LDS through a 16-bit index.  The
// one-ring topology is staged once in a SELL-32 layout (entry-major per 32-slot
// slice, padded to the slice's largest one-ring): bank-conflict-free.
//
// Per iteration k:
//   A  sample (Te, Re) at V+u: 4 rows x one 256-bit load from one of four
//      32-byte-aligned shifted copies of the padded image; residual; energy
//      partial per warp (double-buffered by k & 1).
//   == cluster barrier; read the decision of iteration k-1 (stop -> the field
//      after step k-1 is final); pull the s_te halo; CTA barrier
//   B  grad = r * G s_te, u0 = u - tau*grad (solver.py:133,189)
//   == cluster barrier; pull u0 halo; CTA barrier
//   C  umbrella smoothing (one more exchange per extra pass) + domain clamp;
//      then the control warp reduces every CTA's energy partials of iteration
//      k in one fixed order (identical in every CTA) and runs the divergence /
//      tolerance logic of solver.py:174-195 off the critical path.
#pragma once

#include <cooperative_groups.h>

#include "kernels.cuh"

namespace mrb {

namespace cg = cooperative_groups;

#ifndef MRB_CLUSTER_THREADS
#define MRB_CLUSTER_THREADS 768
#endif
#ifndef MRB_CLUSTER_MINB
#define MRB_CLUSTER_MINB 1
#endif
constexpr int kClusterThreads = MRB_CLUSTER_THREADS;  // threads per CTA
constexpr int kClusterMinBlocks = MRB_CLUSTER_MINB;   // resident CTAs per SM (launch bounds)
constexpr int kMaxDeg = 16;           // largest one-ring the fast path accepts
constexpr int kWarps = kClusterThreads / 32;
constexpr int kCtlWarp = kWarps - 1;  // owns the fewest nodes when chunk < SLOTS

struct ClusterPair {
  const double2* V;           // device-order vertices
  const float2* g_self;       // [n]
  const float* inv_val;       // [n]
  // SELL-32 topology, CTA r's block at r * topo_stride entries:
  const uint16_t* codes;      // local index: own slot, or SLOTS + halo index
  const float2* g;            // fused gradient coefficients
  const uint32_t* slice_off;  // [CS][slices]: entry offset of each 32-slot slice
  const uint32_t* halo;       // [CS][halo_stride]: rank << 16 | slot to pull
  const int* n_halo;          // [CS]
  const unsigned char* deg;   // [n]
  const float2* img4;         // 4 shifted copies of the padded (Te, Re) image
  float2* u;                  // [n] final displacement (device order)
  double2* u_out;             // [n] reference order
  const int* perm;
  double* trace;
  long long* prof;            // optional phase timestamps (MESHREG_B200_PROFILE_PHASES)
  // dense pass (k_dense_fast)
  const int* tri_of;          // pixel -> triangle
  const int4* tri;            // triangles (device node ids)
  float *ux, *uy, *warped;
  int pix_blk_begin;
  int n, chunk, W, H;
  int topo_stride, slices, halo_stride, pitch;
  int plane;
  // push exchange (k_cluster_push): per CTA send list, slot << 20 | dst << 16 | halo idx
  const uint32_t* send;       // [CS][send_stride]
  const int* n_send;          // [CS]
  int send_stride;
  unsigned* flags;            // k_grid_flags: energy-partial counters (zeroed per launch)
  // grid path only (k_grid_register): global exchange buffers
  float* xg_s;                // [CS][SLOTS] s_te of every slot
  float2* xg_u;               // [2][CS][SLOTS] smoothing ping-pong
  double* wpart;              // [2][CS][kWarps] energy partials by parity
  int* gbad;                  // [CS] sticky non-finite gradient flags
  unsigned* bar;              // grid barrier counter (zeroed before each launch)
  // k_grid_flags: [CS][SLOTS/32] bit per slot read by another CTA's halo
  // (only those slots publish exchange words); null = publish every slot
  const uint32_t* exports;
  int tap_evict_first;        // k_grid_flags: L2 policy of the tap loads (see ld_row4_pol)
  int rowpair;                // img4 in the row-pair layout (k_pad_planar_rp): grid path, images beyond L2
};

// Four copies of the padded (H+2)x(W+2) (Te, Re) image; copy s holds padded
// element x at column x + s of a row of `pitch` (a multiple of 4) float2, so
// any 4-tap row starting at column cx is one 32-byte-aligned 256-bit load in
// copy (4 - cx % 4) % 4.  The ring holds the reference's extrapolation
// (image.py:62-71,134-148), computed in fp64 and rounded to fp32.
__global__ void k_pad_image4(const float* __restrict__ img, size_t img_stride, int W, int H,
                             float2* __restrict__ out, int pitch, size_t plane,
                             size_t out_stride) {
  const int Wp = W + 2, Hp = H + 2;
  const float* src = img + blockIdx.y * img_stride;
  float2* dst = out + blockIdx.y * out_stride;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < Wp * Hp; q += gridDim.x * blockDim.x) {
    const int r = q / Wp, c = q - r * Wp;
    const Px<float, double, 2> v = ext_tap<float, double, 2>(src, W, H, r, c);
    const float2 f = make_float2(float(v.v[0]), float(v.v[1]));
#pragma unroll
    for (int s = 0; s < 4; ++s) dst[s * plane + size_t(r) * pitch + c + s] = f;
  }
}

// Same four padded copies built straight from the planar fp32 inputs
// (reference / template stacks) — the fast path needs no other image layout.
__global__ void k_pad_planar4(const float* const* __restrict__ re, const float* const* __restrict__ te,
                              int W, int H, float2* __restrict__ out, int pitch, size_t plane,
                              size_t out_stride) {
  const int Wp = W + 2, Hp = H + 2;
  const float* r_img = re[blockIdx.y];
  const float* t_img = te[blockIdx.y];
  float2* dst = out + blockIdx.y * out_stride;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < Wp * Hp; q += gridDim.x * blockDim.x) {
    const int r = q / Wp, c = q - r * Wp;
    const double vt = ext_tap<float, double, 1>(t_img, W, H, r, c).v[0];
    const double vr = ext_tap<float, double, 1>(r_img, W, H, r, c).v[0];
    const float2 f = make_float2(float(vt), float(vr));
#pragma unroll
    for (int s = 0; s < 4; ++s) dst[s * plane + size_t(r) * pitch + c + s] = f;
  }
}

// Row-pair layout of the padded image for images that stream from DRAM (the
// whole-GPU grid path beyond L2, C5): eight copies, x shift s = 0..3 and row
// parity p = 0..1.  Padded element (r, c) of copy (s, p) sits at
//   (2s + p) * plane + ((r + p) / 2) * 2 pitch + ((c + s) / 4) * 8 + ((r + p) % 2) * 4 + (c + s) % 4
// so the 4-tap rows r and r+1 of a window (r + p even) fill one 64-byte
// aligned block: a 4x4 window is exactly two 64-byte DRAM fetches (the four
// 32-byte rows of the shifted layout cost four, half of each wasted).
__device__ __forceinline__ size_t rp_index(int s, int p, int r, int c, int pitch, size_t plane) {
  const int rr = r + p, cc = c + s;
  return size_t(2 * s + p) * plane + size_t(rr >> 1) * (2 * size_t(pitch)) + size_t(cc >> 2) * 8 +
         (rr & 1) * 4 + (cc & 3);
}

__global__ void k_pad_planar_rp(const float* const* __restrict__ re,
                                const float* const* __restrict__ te, int W, int H,
                                float2* __restrict__ out, int pitch, size_t plane,
                                size_t out_stride) {
  const int Wp = W + 2, Hp = H + 2;
  const float* r_img = re[blockIdx.y];
  const float* t_img = te[blockIdx.y];
  float2* dst = out + blockIdx.y * out_stride;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < Wp * Hp; q += gridDim.x * blockDim.x) {
    const int r = q / Wp, c = q - r * Wp;
    const double vt = ext_tap<float, double, 1>(t_img, W, H, r, c).v[0];
    const double vr = ext_tap<float, double, 1>(r_img, W, H, r, c).v[0];
    const float2 f = make_float2(float(vt), float(vr));
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
      for (int p = 0; p < 2; ++p) dst[rp_index(s, p, r, c, pitch, plane)] = f;
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(addr), "r"(rank));
  return out;
}

__device__ __forceinline__ float ld_dsmem_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}

__device__ __forceinline__ float2 ld_dsmem_f32x2(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];"
               : "=f"(v.x), "=f"(v.y)
               : "r"(addr)
               : "memory");
  return v;
}

__device__ __forceinline__ double ld_dsmem_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}

__device__ __forceinline__ int ld_dsmem_s32(uint32_t addr) {
  int v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}

__device__ __forceinline__ void cluster_sync_all() {
  // barrier.cluster.arrive.release + wait.acquire (orders DSMEM traffic)
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// one 4-tap (Te, Re) row: a single 256-bit read-only load
// L1::no_allocate: a node's taps are not re-read by its CTA within an
// iteration, so they would only evict the L1-resident topology / halo lines
// (C4 7.96 -> 7.63 ms).
__device__ __forceinline__ void ld_row4(const float2* p, float2 (&t)[4]) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(t[0].x), "=f"(t[0].y), "=f"(t[1].x), "=f"(t[1].y), "=f"(t[2].x),
                 "=f"(t[2].y), "=f"(t[3].x), "=f"(t[3].y)
               : "l"(p));
}

// ld_row4 with an L2 cache-eviction policy (createpolicy): the whole-GPU
// kernel marks the taps evict_first when the image copies exceed L2, so the
// per-iteration constants (topology, coordinates) stay resident instead.
__device__ __forceinline__ void ld_row4_pol(const float2* p, float2 (&t)[4], uint64_t pol) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
               : "=f"(t[0].x), "=f"(t[0].y), "=f"(t[1].x), "=f"(t[1].y), "=f"(t[2].x),
                 "=f"(t[2].y), "=f"(t[3].x), "=f"(t[3].y)
               : "l"(p), "l"(pol));
}

// Catmull-Rom window of (Te, Re) at (x, y) (ImageGrid.sample, image.py:73-84,
// _locate 105-116) in the aligned padded copies: base row pointer + weights.
struct Window {
  const float2* base;
  float wx[4], wy[4];
};

// the image fields locate() needs, held in registers across the loop
struct ImgView {
  const float2* img4;
  int W, H, pitch, plane;
};

__device__ __forceinline__ ImgView img_view(const ClusterPair& d) {
  return ImgView{d.img4, d.W, d.H, d.pitch, d.plane};
}

// Catmull-Rom weights (image.py:151-164) in Horner form with FMAs for the
// fp32 fast path: 11 instructions per axis instead of the reference's 18
// separately rounded operations; the same polynomials, within a few ulp.
__device__ __forceinline__ void cr_weights_fma(float t, float w[4]) {
  const float t2 = t * t;
  w[0] = t * fmaf(t, fmaf(-0.5f, t, 1.0f), -0.5f);  // 0.5 (-t^3 + 2t^2 - t)
  w[1] = fmaf(t2, fmaf(1.5f, t, -2.5f), 1.0f);     // 0.5 (3t^3 - 5t^2 + 2)
  w[2] = t * fmaf(t, fmaf(-1.5f, t, 2.0f), 0.5f);  // 0.5 (-3t^3 + 4t^2 + t)
  w[3] = t2 * fmaf(0.5f, t, -0.5f);                // 0.5 (t^3 - t^2)
}

template <bool RP = false, typename D>
__device__ __forceinline__ Window locate(const D& d, double x, double y) {
  const double xc = fmin(fmax(x, 0.0), double(d.W) - 1.0);
  const double yc = fmin(fmax(y, 0.0), double(d.H) - 1.0);
  const int cx = min(int(xc), d.W - 2);  // xc >= 0: truncation == floor
  const int cy = min(int(yc), d.H - 2);
  Window w;
  cr_weights_fma(float(xc - double(cx)), w.wx);
  cr_weights_fma(float(yc - double(cy)), w.wy);
  const int s = (4 - (cx & 3)) & 3;
  if constexpr (RP)  // padded window rows cy..cy+3, columns cx..cx+3
    w.base = d.img4 + rp_index(s, cy & 1, cy, cx, d.pitch, size_t(d.plane));
  else
    w.base = d.img4 + size_t(s) * d.plane + size_t(cy) * d.pitch + cx + s;
  return w;
}

// offset of window row j from Window::base
template <bool RP>
__device__ __forceinline__ size_t row_off(int pitch, int j) {
  return RP ? size_t(j >> 1) * (2 * size_t(pitch)) + (j & 1) * 4 : size_t(j) * pitch;
}

__device__ __forceinline__ float2 combine(const Window& w, const float2 (&t)[4][4]) {
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float rt = w.wx[0] * t[j][0].x, rr = w.wx[0] * t[j][0].y;
#pragma unroll
    for (int i = 1; i < 4; ++i) {
      rt = fmaf(w.wx[i], t[j][i].x, rt);
      rr = fmaf(w.wx[i], t[j][i].y, rr);
    }
    acc.x = fmaf(w.wy[j], rt, acc.x);
    acc.y = fmaf(w.wy[j], rr, acc.y);
  }
  return acc;
}

// np.clip(u1, -V, (W-1) - V) (solver.py:140-144) evaluated in fp64 and
// rounded to fp32 equals the fp32 clip against the rounded bounds (rounding
// is monotonic), which is what this computes.
__device__ __forceinline__ float2 clamp_dom(float2 v, double2 V, int W, int H) {
  const float lox = float(-V.x), hix = float((double(W) - 1.0) - V.x);
  const float loy = float(-V.y), hiy = float((double(H) - 1.0) - V.y);
  return make_float2(fminf(fmaxf(v.x, lox), hix), fminf(fmaxf(v.y, loy), hiy));
}

// Dynamic shared memory layout (host: cluster_dyn_smem).  The coefficient
// pairs (float4) come first so they are 16-byte aligned.
struct ClusterSmem {
  float4* g4;      // paired SELL coefficients (gx, gy) of entries 2p, 2p+1
  double2* V;
  float2 *gs, *xu0, *xu1;
  float *iv, *xs;
  uint32_t* halo;
  uint32_t* code2;  // paired SELL codes: entry 2p in the low half, 2p+1 in the high
  uint32_t* soff;
};

template <int NPT>
__device__ __forceinline__ ClusterSmem carve(unsigned char* p, const ClusterPair& d, bool two) {
  constexpr int SLOTS = kClusterThreads * NPT;
  const int X = SLOTS + d.halo_stride;  // own slots followed by the halo (last: ZERO slot)
  ClusterSmem s;
  s.g4 = reinterpret_cast<float4*>(p);
  s.V = reinterpret_cast<double2*>(s.g4 + d.topo_stride / 2);  // topo_stride % 8 == 0
  s.gs = reinterpret_cast<float2*>(s.V + SLOTS);
  s.xu0 = s.gs + SLOTS;
  s.xu1 = s.xu0 + X;
  s.iv = reinterpret_cast<float*>(s.xu1 + (two ? X : 0));
  s.xs = s.iv + SLOTS;
  s.halo = reinterpret_cast<uint32_t*>(s.xs + X);
  s.code2 = s.halo + d.halo_stride;
  s.soff = s.code2 + d.topo_stride / 2;
  return s;
}

// One-ring gather over the paired SELL layout (see write_topo): for the pair
// rows of this slot's slice (a warp-uniform count, the slice's largest
// one-ring rounded up), f(codes of entries 2p | 2p+1 << 16, row index).
// Padding entries point at the ZERO slot with coefficient 0, so they add
// exactly nothing and no lane needs a predicate.
template <int NP, typename F>
__device__ __forceinline__ void ring_pairs_n(const uint32_t* code2, uint32_t base, F&& f) {
  uint32_t cc[NP];
#pragma unroll
  for (int q = 0; q < NP; ++q) cc[q] = code2[base + 32u * q];  // all codes first
#pragma unroll
  for (int q = 0; q < NP; ++q) f(cc[q], base + 32u * q);
}

template <typename F>
__device__ __forceinline__ void ring_pairs(const uint32_t* code2, uint32_t sw, int lane, F&& f) {
  const uint32_t base = (sw & 0xffffffu) + uint32_t(lane);
  const int np = int(sw >> 24);
  // warp-uniform pair-row count: fully unrolled bodies for the usual counts
  // (the codes of every row loaded before the gathers that depend on them)
  switch (np) {
    case 2: ring_pairs_n<2>(code2, base, f); return;
    case 3: ring_pairs_n<3>(code2, base, f); return;
    case 4: ring_pairs_n<4>(code2, base, f); return;
    case 5: ring_pairs_n<5>(code2, base, f); return;
    default: break;
  }
#pragma unroll 2
  for (int q = 0; q < np; ++q) {
    const uint32_t at = base + 32u * uint32_t(q);
    f(code2[at], at);
  }
}

template <int NPT>
__global__ void __launch_bounds__(kClusterThreads, kClusterMinBlocks)
    k_cluster_register(const ClusterPair* __restrict__ pairs, PairStatus* __restrict__ st,
                       int max_iter, double tol, float tau, float lam, int passes) {
  constexpr int SLOTS = kClusterThreads * NPT;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = int(cluster.block_rank());
  const int CS = int(cluster.num_blocks());  // runtime cluster size (1..16)
  const int p = blockIdx.x / CS;
  const ClusterPair& d = pairs[p];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;

  __shared__ double s_wpart[2][kWarps];  // per-warp energy partials, by iteration parity
  __shared__ double s_cpart[2];          // CTA energy partial (fixed-order sum of s_wpart)
  __shared__ int s_gradbad;              // non-finite gradient seen in this CTA
  __shared__ int s_stop;                 // decision so far: 0 go, 1 error, 2 converged
  __shared__ int s_nhalo;
  // descent control state (control warp lane 0 only; identical in every CTA)
  __shared__ double s_hist[6];
  __shared__ double s_prev;
  __shared__ int s_cs[4];                // rises, iters, err, err_iter
  extern __shared__ __align__(16) unsigned char s_dyn[];
  const ClusterSmem sm = carve<NPT>(s_dyn, d, passes >= 2);
  const int zero = SLOTS + d.halo_stride - 1;  // ZERO slot of the padding entries

  if (t == 0) {
    s_gradbad = 0;
    s_stop = 0;
    s_prev = 0.0;
    s_cs[0] = s_cs[1] = s_cs[2] = s_cs[3] = 0;
    s_nhalo = d.n_halo[rank];
  }
  // ---- stage this CTA's topology and halo list (coalesced block copies)
  {
    const size_t tb = size_t(rank) * d.topo_stride;
    const float4* g4 = reinterpret_cast<const float4*>(d.g + tb);
    const uint32_t* c2 = reinterpret_cast<const uint32_t*>(d.codes + tb);
    for (int q = t; q < d.topo_stride / 2; q += kClusterThreads) {
      sm.g4[q] = g4[q];
      sm.code2[q] = c2[q];
    }
    for (int q = t; q < d.slices; q += kClusterThreads)
      sm.soff[q] = d.slice_off[size_t(rank) * d.slices + q];
    for (int q = t; q < d.halo_stride; q += kClusterThreads)
      sm.halo[q] = d.halo[size_t(rank) * d.halo_stride + q];
    if (t == 0) {
      sm.xs[zero] = 0.f;
      sm.xu0[zero] = make_float2(0.f, 0.f);
      if (passes >= 2) sm.xu1[zero] = make_float2(0.f, 0.f);
    }
  }
  // ---- per-node constants into shared memory, evolving state in registers
  float2 u[NPT];
  float r[NPT];
  unsigned own_mask = 0;
#pragma unroll
  for (int j = 0; j < NPT; ++j) {
    const int slot = t + j * kClusterThreads;
    const int nd = rank * d.chunk + slot;
    const bool o = slot < d.chunk && nd < d.n;
    own_mask |= unsigned(o) << j;
    sm.V[slot] = o ? d.V[nd] : make_double2(0.0, 0.0);
    sm.gs[slot] = o ? d.g_self[nd] : make_float2(0.f, 0.f);
    sm.iv[slot] = o ? d.inv_val[nd] : 0.f;
    u[j] = make_float2(0.f, 0.f);
    r[j] = 0.f;
  }
#define OWN(j) ((own_mask >> (j)) & 1u)
  const uint32_t cpart_addr = smem_u32(&s_cpart[0]), bad_addr = smem_u32(&s_gradbad);
  const uint32_t xs_addr = smem_u32(sm.xs), xu0_addr = smem_u32(sm.xu0),
                 xu1_addr = smem_u32(sm.xu1);
  cluster_sync_all();  // every CTA started and staged
  const int nhalo = s_nhalo;

#ifdef MRB_PHASE_PROFILE  // phase timestamps (build flag; MESHREG_B200_PROFILE_PHASES)
  long long* const prof =
      (d.prof && t == 0) ? d.prof + (size_t(rank) * 8) * 16 : nullptr;  // d.prof: this pair's
#define PROF(k, slot) \
  if (prof && (k) < 8) prof[(k) * 16 + (slot)] = clock64();
#else
#define PROF(k, slot)
#endif

  // Control step of iteration kk (control warp, all CTAs identically):
  // fixed-order cluster reduction of the energy partials, then the logic of
  // solver.py:176-195 in the reference's order (energy checks, the step's
  // gradient check, tolerance).
  auto control = [&](int kk) {
    // one DSMEM load per lane: the CTA partials of iteration kk (each CTA
    // reduced its own warp partials after the first barrier of kk)
    double v = lane < CS ? ld_dsmem_f64(mapa_u32(cpart_addr, lane) + 8u * (kk & 1)) : 0.0;
    int gb = lane < CS ? ld_dsmem_s32(mapa_u32(bad_addr, lane)) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v += __shfl_down_sync(0xffffffffu, v, o);
      gb |= __shfl_down_sync(0xffffffffu, gb, o);
    }
    if (lane == 0 && s_stop == 0) {
      int stop = 0, rises = s_cs[0], err = ERR_NONE, err_iter = 0;
      const double e = 0.5 * v;
      const double prev = s_prev;
      if (!isfinite(e)) {  // solver.py:176-177
        err = ERR_NONFINITE_ENERGY;
        err_iter = kk;
        stop = 1;
      } else if (kk > 0 && e > __dadd_rn(__dmul_rn(prev, 1.0 + 1e-4), 1e-12)) {
        if (++rises >= 10) {  // material_rise, solver.py:43-44,178-184
          err = ERR_RISES;
          err_iter = kk;
          stop = 1;
        }
      } else if (kk > 0 && e <= prev) {
        rises = 0;  // solver.py:185-186
      }
      if (!stop && gb) {  // step(): non-finite gradient, solver.py:131-132
        err = ERR_NONFINITE_GRAD;
        err_iter = kk;
        stop = 1;
      }
      if (!stop) {
        s_cs[1] = kk + 1;
        s_hist[kk % 6] = e;
        if (kk + 1 >= 6) {  // solver.py:192-195; trace[-6] == hist[(kk+1)%6]
          const double base = s_hist[(kk + 1) % 6];
          if (fabs(__dsub_rn(e, base)) <= __dmul_rn(tol, fmax(fabs(base), 1e-12))) stop = 2;
        }
      }
      if (rank == 0) d.trace[kk] = e;
      s_prev = e;
      s_cs[0] = rises;
      s_cs[2] = err;
      s_cs[3] = err_iter;
      s_stop = stop;
    }
  };

  const ImgView img = img_view(d);
  int k = 0;
  for (; k < max_iter; ++k) {
    PROF(k, 0)
    // -------- phase A: sample Te, Re at V + u; residual; energy partial
    {
      double e2 = 0.0;
#pragma unroll
      for (int j = 0; j < NPT; ++j) {  // one node at a time: no register spills
        if (OWN(j)) {
          const double2 V = sm.V[t + j * kClusterThreads];
          const Window w = locate(img, V.x + double(u[j].x), V.y + double(u[j].y));
          float2 tap[4][4];
#pragma unroll
          for (int row = 0; row < 4; ++row) ld_row4(w.base + size_t(row) * img.pitch, tap[row]);
          const float2 s = combine(w, tap);
          r[j] = s.x - s.y;
          sm.xs[t + j * kClusterThreads] = s.x;
          e2 = fma(double(r[j]), double(r[j]), e2);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) e2 += __shfl_down_sync(0xffffffffu, e2, o);
      if (lane == 0) s_wpart[k & 1][warp] = e2;
    }
    PROF(k, 1)
    cluster_sync_all();  // s_te, energy partials (and the k-1 decision) visible
    PROF(k, 2)
    if (s_stop) break;   // iteration k-1 was the last one (u untouched since)
    for (int h = t; h < nhalo; h += kClusterThreads) {  // pull the s_te halo
      const uint32_t c = sm.halo[h];
      sm.xs[SLOTS + h] = ld_dsmem_f32(mapa_u32(xs_addr, c >> 16) + 4u * (c & 0xffffu));
    }
    PROF(k, 3)
    __syncthreads();  // s_te halo complete
    if (warp == kCtlWarp) {  // CTA energy partial of iteration k, fixed order
      double v = lane < kWarps ? s_wpart[k & 1][lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      if (lane == 0) s_cpart[k & 1] = v;  // read remotely after the next cluster barrier
    }
    PROF(k, 4)

    // -------- phase B: gradient via the fused one-ring operator, descent
    bool bad = false;
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
      if (OWN(j)) {
        const int slot = t + j * kClusterThreads;
        const float si = sm.xs[slot];
        const float2 gs = sm.gs[slot];
        float gx = gs.x * si, gy = gs.y * si;
        ring_pairs(sm.code2, sm.soff[slot >> 5], lane, [&](uint32_t cc, uint32_t at) {
          const float s0 = sm.xs[cc & 0xffffu], s1 = sm.xs[cc >> 16];
          const float4 ge = sm.g4[at];
          gx = fmaf(ge.x, s0, gx);
          gy = fmaf(ge.y, s0, gy);
          gx = fmaf(ge.z, s1, gx);
          gy = fmaf(ge.w, s1, gy);
        });
        const float dx = r[j] * gx, dy = r[j] * gy;  // solver.py:189
        bad |= !isfinite(dx) || !isfinite(dy);
        sm.xu0[slot] = make_float2(u[j].x - tau * dx, u[j].y - tau * dy);  // solver.py:133
      }
    }
    PROF(k, 5)
    if (__syncthreads_or(bad) && t == 0) s_gradbad = 1;
    PROF(k, 6)

    // -------- phase C: umbrella smoothing passes + domain clamp
    if (passes == 0) {
      cluster_sync_all();  // gradbad flags visible; s_te halo reads of all CTAs done
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        if (OWN(j)) {
          const int slot = t + j * kClusterThreads;
          u[j] = clamp_dom(sm.xu0[slot], sm.V[slot], img.W, img.H);
        }
      }
    }
    for (int q = 0; q < passes; ++q) {
      float2* src = (q & 1) ? sm.xu1 : sm.xu0;
      const uint32_t src_addr = (q & 1) ? xu1_addr : xu0_addr;
      PROF(k, 7)
      cluster_sync_all();  // src (and the gradbad flags) visible cluster-wide
      PROF(k, 8)
      for (int h = t; h < nhalo; h += kClusterThreads) {  // pull the halo of src
        const uint32_t c = sm.halo[h];
        src[SLOTS + h] = ld_dsmem_f32x2(mapa_u32(src_addr, c >> 16) + 8u * (c & 0xffffu));
      }
      PROF(k, 9)
      __syncthreads();
      PROF(k, 10)
      float2 v[NPT];
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        v[j] = make_float2(0.f, 0.f);
        if (OWN(j)) {
          const int slot = t + j * kClusterThreads;
          const float iv = sm.iv[slot];
          float ax = 0.f, ay = 0.f;
          // (L u)_i, L_ij = 1/val_i
          ring_pairs(sm.code2, sm.soff[slot >> 5], lane, [&](uint32_t cc, uint32_t) {
            const float2 u0 = src[cc & 0xffffu], u1 = src[cc >> 16];
            ax = fmaf(iv, u0.x, ax);
            ay = fmaf(iv, u0.y, ay);
            ax = fmaf(iv, u1.x, ax);
            ay = fmaf(iv, u1.y, ay);
          });
          const float2 si = src[slot];
          const float om = 1.f - lam;  // (1 - lam) u + lam (L u), mesh.py:281
          v[j] = make_float2(om * si.x + lam * ax, om * si.y + lam * ay);
        }
      }
      if (q == passes - 1) {
#pragma unroll
        for (int j = 0; j < NPT; ++j)
          if (OWN(j)) u[j] = clamp_dom(v[j], sm.V[t + j * kClusterThreads], img.W, img.H);
      } else {
        float2* dst = (q & 1) ? sm.xu0 : sm.xu1;
#pragma unroll
        for (int j = 0; j < NPT; ++j)
          if (OWN(j)) dst[t + j * kClusterThreads] = v[j];
      }
    }
    // -------- control of iteration k, off the critical path; its decision is
    // read by every thread after the next cluster barrier
    if (warp == kCtlWarp) control(k);
    PROF(k, 11)
  }
#undef PROF
#pragma unroll
  for (int j = 0; j < NPT; ++j) {
    if (OWN(j)) {
      const int nd = rank * d.chunk + t + j * kClusterThreads;
      d.u[nd] = u[j];
      d.u_out[d.perm[nd]] = make_double2(double(u[j].x), double(u[j].y));
    }
  }
#undef OWN
  __syncthreads();
  if (rank == 0 && t == 0) {
    PairStatus s{};
    s.stop_iter = k;
    s.err = s_cs[2];
    s.err_iter = s_cs[3];
    s.rises = s_cs[0];
    s.iters = s_cs[1];
    st[p] = s;
  }
  cluster_sync_all();  // keep every CTA's smem alive until all remote reads are done
}

// Dense pass of the fp32 fast path: densify (densefield.py:130-187; fp64
// barycentric weights in numpy's operation order), backward warp
// (densefield.py:190-199) from the aligned padded copies, and the fp64 MSD
// partials of msd(Te, Re) and msd(warped, Re) (image.py:181-186), with the
// same block partition as k_dense so k_msd_final reduces them unchanged.
__global__ void __launch_bounds__(kPixBlock)
    k_dense_fast(const ClusterPair* __restrict__ pairs, PairStatus* __restrict__ st,
                 const int* __restrict__ blk_pair, double2* __restrict__ partials, int blk0) {
  __shared__ double sh[2 * kPixBlock / 32];
  const int blk = blk0 + int(blockIdx.x);  // launched per group of pairs
  const int p = blk_pair[blk];
  const ClusterPair& d = pairs[p];
  if (st[p].err) return;
  const int q = (blk - d.pix_blk_begin) * kPixBlock + threadIdx.x;
  double2 acc = make_double2(0.0, 0.0);
  const int ti = q < d.W * d.H ? __ldg(d.tri_of + q) : kUnassigned;
  if (ti == kUnassigned && q < d.W * d.H) {
    // not yet assigned: the deferred coverage check (mrb_batch_sync) either
    // raises MeshCoverageError or reruns the batch with the located pixels
    d.ux[q] = d.uy[q] = d.warped[q] = 0.f;
  } else if (q < d.W * d.H) {
    const int y = q / d.W, x = q - y * d.W;
    const int4 tv = __ldg(d.tri + ti);
    // barycentric weights (densefield.py:99-107) in fp64 with one reciprocal
    // instead of two divisions: within an ulp of the exact-rounding form,
    // far inside the fp32 path's tolerance (the exact form is bary_rn, used
    // by the fp64 dense pass and the pixel_map export)
    double w[3];
    {
      const double2 a = __ldg(d.V + tv.x), b = __ldg(d.V + tv.y), c = __ldg(d.V + tv.z);
      const double px = double(x), py = double(y);
      const double inv = 1.0 / ((b.x - a.x) * (c.y - a.y) - (c.x - a.x) * (b.y - a.y));
      w[0] = ((b.x - px) * (c.y - py) - (c.x - px) * (b.y - py)) * inv;
      w[1] = ((c.x - px) * (a.y - py) - (a.x - px) * (c.y - py)) * inv;
      w[2] = (1.0 - w[0]) - w[1];
    }
    const float2 ua = d.u[tv.x], ub = d.u[tv.y], uc = d.u[tv.z];
    // (w * u[T]).sum(axis=2) = (w1 ua + w2 ub) + w3 uc, densefield.py:184-187
    const float rx = float(__dadd_rn(__dadd_rn(__dmul_rn(w[0], double(ua.x)), __dmul_rn(w[1], double(ub.x))),
                                     __dmul_rn(w[2], double(uc.x))));
    const float ry = float(__dadd_rn(__dadd_rn(__dmul_rn(w[0], double(ua.y)), __dmul_rn(w[1], double(ub.y))),
                                     __dmul_rn(w[2], double(uc.y))));
    d.ux[q] = rx;
    d.uy[q] = ry;
    float2 tap[4][4];
    Window win;
    float2 own;  // (Te, Re) at the pixel: padded (y + 1, x + 1) of copy 0
    if (d.rowpair) {
      win = locate<true>(d, double(x) + double(rx), double(y) + double(ry));
#pragma unroll
      for (int row = 0; row < 4; ++row) ld_row4(win.base + row_off<true>(d.pitch, row), tap[row]);
      own = __ldg(d.img4 + rp_index(0, 0, y + 1, x + 1, d.pitch, size_t(d.plane)));
    } else {
      win = locate(d, double(x) + double(rx), double(y) + double(ry));
#pragma unroll
      for (int row = 0; row < 4; ++row) ld_row4(win.base + size_t(row) * d.pitch, tap[row]);
      own = __ldg(d.img4 + size_t(y + 1) * d.pitch + (x + 1));
    }
    const float wv = combine(win, tap).x;
    d.warped[q] = wv;
    const double d0 = double(own.x) - double(own.y);
    const double d1 = double(wv) - double(own.y);
    acc.x = d0 * d0;
    acc.y = d1 * d1;
    if (!isfinite(rx) || !isfinite(ry)) atomicOr(&st[p].dense_nonfinite, 1);
    if (!isfinite(wv)) atomicOr(&st[p].dense_nonfinite, 2);
  }
  const double2 bs = block_sum2<kPixBlock>(acc, sh);
  if (threadIdx.x == 0) partials[blk] = bs;
}

}  // namespace mrb
