// Persistent thread-block-cluster loop in fp64: the reference's arithmetic
// width (solver.py:148-208 computes in float64) and the API's default
// precision.  Same structure as k_cluster_register (cluster.cuh) — one
// cluster of CS CTAs owns one pair for the whole descent loop, per-node
// constants and the paired SELL-32 topology in shared memory, halo exchange
// over DSMEM between two cluster barriers per iteration, control deferred one
// phase — with fp64 state, coefficients and arithmetic:
//   * taps: a padded (H+2) x (W+2) fp64 (Te, Re) image whose ring holds the
//     reference's extrapolation in fp64 (image.py:62-71,134-148; the padded
//     fp32 copies of the fp32 path would round it), built once per run by
//     k_pad_pair64 from the generic path's interleaved image: every window,
//     border or not, is 16 double2 loads with cr_sample's arithmetic;
//   * coefficients: one double2 per SELL entry (16 B; one 768-node CTA per
//     SM, so NPT = 1);
//   * the loop writes the final u into the generic path's state, whose dense
//     pass (k_dense), MSD and un-permutation then run unchanged.
#pragma once

#include "cluster.cuh"

namespace mrb {

struct ClusterPair64 {
  const double2* V;           // device-order vertices
  const double2* g_self;      // [n] fused operator, self term
  const double* inv_val;      // [n] 1/valence
  const uint16_t* codes;      // paired SELL codes (write_topo layout)
  const double2* g;           // paired SELL coefficients, one double2 per entry
  const uint32_t* slice_off;  // [CS][slices]
  const uint32_t* halo;       // [CS][halo_stride]: rank << 16 | slot
  const int* n_halo;          // [CS]
  const uint32_t* send;       // push exchange: [CS][send_stride] slot << 20 | dst << 16 | halo idx
  const int* n_send;          // [CS]
  int send_stride;
  const void* img;            // interleaved (Te, Re), H x W: float, or double (tap_d)
  const double2* pad;         // padded (H+2) x (W+2) (Te, Re), exact fp64 ring
  const float2* img4;         // fp32-exact inputs: the fp32 path's 4 shifted padded copies
  int pitch, plane;           //   (interior windows only: their ring is rounded)
  double2* u;                 // [n] final displacement, device order
  double* trace;
  int n, chunk, W, H, tap_d;
  int topo_stride, slices, halo_stride;
};

// padded fp64 (Te, Re) images of a batch (grid.y = pair): the stored pixels
// and the reference's extrapolated ring, exactly as ext_tap computes them
template <typename TapT>
__global__ void k_pad_pair64(const ClusterPair64* __restrict__ pairs) {
  const ClusterPair64& d = pairs[blockIdx.y];
  const int Wp = d.W + 2, Hp = d.H + 2;
  const TapT* img = static_cast<const TapT*>(d.img);
  double2* out = const_cast<double2*>(d.pad);
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < Wp * Hp; q += gridDim.x * blockDim.x) {
    const int r = q / Wp, c = q - r * Wp;
    const Px<TapT, double, 2> v = ext_tap<TapT, double, 2>(img, d.W, d.H, r, c);
    out[q] = make_double2(v.v[0], v.v[1]);
  }
}

// Catmull-Rom (Te, Re) at (x, y) from the padded fp64 image: cr_sample's
// clamp, cell, weights and accumulation order (image.py:73-84,105-123)
__device__ __forceinline__ double2 sample_pad64(const double2* __restrict__ pad, int W, int H,
                                                double x, double y) {
  const double xc = fmin(fmax(x, 0.0), double(W) - 1.0);
  const double yc = fmin(fmax(y, 0.0), double(H) - 1.0);
  const int cx = min(int(xc), W - 2);  // xc >= 0: truncation == floor
  const int cy = min(int(yc), H - 2);
  double wx[4], wy[4];
  cr_weights<double>(xc - double(cx), wx);
  cr_weights<double>(yc - double(cy), wy);
  // padded row cy + j, column cx + i holds image pixel (cy - 1 + j, cx - 1 + i)
  const double2* base = pad + size_t(cy) * (W + 2) + cx;
  double te = 0.0, re = 0.0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    double2 tp[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) tp[i] = __ldg(base + size_t(j) * (W + 2) + i);
    double rt = wx[0] * tp[0].x, rr = wx[0] * tp[0].y;
#pragma unroll
    for (int i = 1; i < 4; ++i) {
      rt = fma(wx[i], tp[i].x, rt);
      rr = fma(wx[i], tp[i].y, rr);
    }
    te = fma(wy[j], rt, te);
    re = fma(wy[j], rr, re);
  }
  return make_double2(te, re);
}

// fp32-exact inputs: an interior window (no ring tap) reads the fp32 path's
// aligned shifted copies — 4 x 32-byte rows instead of 16 x 16-byte taps —
// with the same fp64 weights and accumulation as sample_pad64; a window
// touching the ring reads the exact fp64 padded image
__device__ __forceinline__ double2 sample_int64(const ClusterPair64& d, double x, double y) {
  const double xc = fmin(fmax(x, 0.0), double(d.W) - 1.0);
  const double yc = fmin(fmax(y, 0.0), double(d.H) - 1.0);
  const int cx = min(int(xc), d.W - 2);
  const int cy = min(int(yc), d.H - 2);
  if (cx < 1 || cx > d.W - 3 || cy < 1 || cy > d.H - 3) return sample_pad64(d.pad, d.W, d.H, x, y);
  double wx[4], wy[4];
  cr_weights<double>(xc - double(cx), wx);
  cr_weights<double>(yc - double(cy), wy);
  const int s = (4 - (cx & 3)) & 3;
  const float2* base = d.img4 + size_t(s) * d.plane + size_t(cy) * d.pitch + cx + s;
  double te = 0.0, re = 0.0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float2 tp[4];
    ld_row4(base + size_t(j) * d.pitch, tp);
    double rt = wx[0] * double(tp[0].x), rr = wx[0] * double(tp[0].y);
#pragma unroll
    for (int i = 1; i < 4; ++i) {
      rt = fma(wx[i], double(tp[i].x), rt);
      rr = fma(wx[i], double(tp[i].y), rr);
    }
    te = fma(wy[j], rt, te);
    re = fma(wy[j], rr, re);
  }
  return make_double2(te, re);
}

__device__ __forceinline__ double2 ld_dsmem_f64x2(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y)
               : "r"(addr)
               : "memory");
  return v;
}

// np.clip(u1, -V, (W-1, H-1) - V), solver.py:138-144, in fp64
__device__ __forceinline__ double2 clamp_dom64(double2 v, double2 V, int W, int H) {
  return make_double2(fmin(fmax(v.x, -V.x), (double(W) - 1.0) - V.x),
                      fmin(fmax(v.y, -V.y), (double(H) - 1.0) - V.y));
}

// Dynamic shared memory (host: cluster64_dyn_smem): coefficients first
// (16-byte aligned), then per-slot constants and state, halo list, codes.
struct Cluster64Smem {
  double2* g;
  double2 *V, *gs, *xu0, *xu1;
  double *iv, *xs;
  uint32_t *halo, *code2, *soff;
};

template <int NPT>
__device__ __forceinline__ Cluster64Smem carve64(unsigned char* p, const ClusterPair64& d,
                                                 bool two) {
  constexpr int SLOTS = kClusterThreads * NPT;
  const int X = SLOTS + d.halo_stride;
  Cluster64Smem s;
  s.g = reinterpret_cast<double2*>(p);
  s.V = s.g + d.topo_stride;
  s.gs = s.V + SLOTS;
  s.xu0 = s.gs + SLOTS;
  s.xu1 = s.xu0 + X;
  s.iv = reinterpret_cast<double*>(s.xu1 + (two ? X : 0));
  s.xs = s.iv + SLOTS;
  s.halo = reinterpret_cast<uint32_t*>(s.xs + X);
  s.code2 = s.halo + d.halo_stride;
  s.soff = s.code2 + d.topo_stride / 2;
  return s;
}

template <int NPT>
__global__ void __launch_bounds__(kClusterThreads, 1)
    k_cluster64(const ClusterPair64* __restrict__ pairs, PairStatus* __restrict__ st,
                int max_iter, double tol, double tau, double lam, int passes) {
  constexpr int SLOTS = kClusterThreads * NPT;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = int(cluster.block_rank());
  const int CS = int(cluster.num_blocks());
  const int p = blockIdx.x / CS;
  const ClusterPair64& d = pairs[p];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;

  __shared__ double s_wpart[2][kWarps];
  __shared__ double s_cpart[2];
  __shared__ int s_gradbad;
  __shared__ int s_stop;
  __shared__ int s_nhalo;
  __shared__ double s_hist[6];
  __shared__ double s_prev;
  __shared__ int s_cs[4];  // rises, iters, err, err_iter
  extern __shared__ __align__(16) unsigned char s_dyn[];
  const Cluster64Smem sm = carve64<NPT>(s_dyn, d, passes >= 2);
  const int zero = SLOTS + d.halo_stride - 1;  // ZERO slot of the padding entries

  if (t == 0) {
    s_gradbad = 0;
    s_stop = 0;
    s_prev = 0.0;
    s_cs[0] = s_cs[1] = s_cs[2] = s_cs[3] = 0;
    s_nhalo = d.n_halo[rank];
  }
  {
    const size_t tb = size_t(rank) * d.topo_stride;
    const uint32_t* c2 = reinterpret_cast<const uint32_t*>(d.codes + tb);
    for (int q = t; q < d.topo_stride; q += kClusterThreads) sm.g[q] = d.g[tb + q];
    for (int q = t; q < d.topo_stride / 2; q += kClusterThreads) sm.code2[q] = c2[q];
    for (int q = t; q < d.slices; q += kClusterThreads)
      sm.soff[q] = d.slice_off[size_t(rank) * d.slices + q];
    for (int q = t; q < d.halo_stride; q += kClusterThreads)
      sm.halo[q] = d.halo[size_t(rank) * d.halo_stride + q];
    if (t == 0) {
      sm.xs[zero] = 0.0;
      sm.xu0[zero] = make_double2(0.0, 0.0);
      if (passes >= 2) sm.xu1[zero] = make_double2(0.0, 0.0);
    }
  }
  double2 u[NPT];
  double r[NPT];
  unsigned own_mask = 0;
#pragma unroll
  for (int j = 0; j < NPT; ++j) {
    const int slot = t + j * kClusterThreads;
    const int nd = rank * d.chunk + slot;
    const bool o = slot < d.chunk && nd < d.n;
    own_mask |= unsigned(o) << j;
    sm.V[slot] = o ? d.V[nd] : make_double2(0.0, 0.0);
    sm.gs[slot] = o ? d.g_self[nd] : make_double2(0.0, 0.0);
    sm.iv[slot] = o ? d.inv_val[nd] : 0.0;
    u[j] = make_double2(0.0, 0.0);
    r[j] = 0.0;
  }
#define OWN(j) ((own_mask >> (j)) & 1u)
  const uint32_t cpart_addr = smem_u32(&s_cpart[0]), bad_addr = smem_u32(&s_gradbad);
  const uint32_t xs_addr = smem_u32(sm.xs), xu0_addr = smem_u32(sm.xu0),
                 xu1_addr = smem_u32(sm.xu1);
  cluster_sync_all();  // every CTA started and staged
  const int nhalo = s_nhalo;

  // control step of iteration kk: as in k_cluster_register (solver.py:174-195)
  auto control = [&](int kk) {
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
      if (!isfinite(e)) {
        err = ERR_NONFINITE_ENERGY;
        err_iter = kk;
        stop = 1;
      } else if (kk > 0 && e > __dadd_rn(__dmul_rn(prev, 1.0 + 1e-4), 1e-12)) {
        if (++rises >= 10) {
          err = ERR_RISES;
          err_iter = kk;
          stop = 1;
        }
      } else if (kk > 0 && e <= prev) {
        rises = 0;
      }
      if (!stop && gb) {
        err = ERR_NONFINITE_GRAD;
        err_iter = kk;
        stop = 1;
      }
      if (!stop) {
        s_cs[1] = kk + 1;
        s_hist[kk % 6] = e;
        if (kk + 1 >= 6) {
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

  int k = 0;
  for (; k < max_iter; ++k) {
    // -------- phase A: sample Te, Re at V + u (fp64 weights, exact ring)
    {
      double e2 = 0.0;
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        if (OWN(j)) {
          const double2 V = sm.V[t + j * kClusterThreads];
          const double2 s = d.img4 ? sample_int64(d, V.x + u[j].x, V.y + u[j].y)
                                   : sample_pad64(d.pad, d.W, d.H, V.x + u[j].x, V.y + u[j].y);
          r[j] = s.x - s.y;
          sm.xs[t + j * kClusterThreads] = s.x;
          e2 = fma(r[j], r[j], e2);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) e2 += __shfl_down_sync(0xffffffffu, e2, o);
      if (lane == 0) s_wpart[k & 1][warp] = e2;
    }
    cluster_sync_all();  // s_te, energy partials (and the k-1 decision) visible
    if (s_stop) break;
    for (int h = t; h < nhalo; h += kClusterThreads) {
      const uint32_t c = sm.halo[h];
      sm.xs[SLOTS + h] = ld_dsmem_f64(mapa_u32(xs_addr, c >> 16) + 8u * (c & 0xffffu));
    }
    __syncthreads();
    if (warp == kCtlWarp) {
      double v = lane < kWarps ? s_wpart[k & 1][lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      if (lane == 0) s_cpart[k & 1] = v;
    }

    // -------- phase B: grad = r * G s_te, u0 = u - tau * grad (solver.py:133,189)
    bool bad = false;
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
      if (OWN(j)) {
        const int slot = t + j * kClusterThreads;
        const double si = sm.xs[slot];
        const double2 gs = sm.gs[slot];
        double gx = gs.x * si, gy = gs.y * si;
        ring_pairs(sm.code2, sm.soff[slot >> 5], lane, [&](uint32_t cc, uint32_t at) {
          const double s0 = sm.xs[cc & 0xffffu], s1 = sm.xs[cc >> 16];
          const double2 g0 = sm.g[2 * at], g1 = sm.g[2 * at + 1];
          gx = fma(g0.x, s0, gx);
          gy = fma(g0.y, s0, gy);
          gx = fma(g1.x, s1, gx);
          gy = fma(g1.y, s1, gy);
        });
        const double dx = r[j] * gx, dy = r[j] * gy;
        bad |= !isfinite(dx) || !isfinite(dy);
        sm.xu0[slot] = make_double2(u[j].x - tau * dx, u[j].y - tau * dy);
      }
    }
    if (__syncthreads_or(bad) && t == 0) s_gradbad = 1;

    // -------- phase C: umbrella smoothing passes + domain clamp (mesh.py:268-282)
    if (passes == 0) {
      cluster_sync_all();
#pragma unroll
      for (int j = 0; j < NPT; ++j)
        if (OWN(j)) {
          const int slot = t + j * kClusterThreads;
          u[j] = clamp_dom64(sm.xu0[slot], sm.V[slot], d.W, d.H);
        }
    }
    for (int q = 0; q < passes; ++q) {
      double2* src = (q & 1) ? sm.xu1 : sm.xu0;
      const uint32_t src_addr = (q & 1) ? xu1_addr : xu0_addr;
      cluster_sync_all();
      for (int h = t; h < nhalo; h += kClusterThreads) {
        const uint32_t c = sm.halo[h];
        src[SLOTS + h] = ld_dsmem_f64x2(mapa_u32(src_addr, c >> 16) + 16u * (c & 0xffffu));
      }
      __syncthreads();
      double2 v[NPT];
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        v[j] = make_double2(0.0, 0.0);
        if (OWN(j)) {
          const int slot = t + j * kClusterThreads;
          const double iv = sm.iv[slot];
          double ax = 0.0, ay = 0.0;
          ring_pairs(sm.code2, sm.soff[slot >> 5], lane, [&](uint32_t cc, uint32_t) {
            const double2 u0 = src[cc & 0xffffu], u1 = src[cc >> 16];
            ax = fma(iv, u0.x, ax);
            ay = fma(iv, u0.y, ay);
            ax = fma(iv, u1.x, ax);
            ay = fma(iv, u1.y, ay);
          });
          const double2 si = src[slot];
          const double om = 1.0 - lam;
          v[j] = make_double2(om * si.x + lam * ax, om * si.y + lam * ay);
        }
      }
      if (q == passes - 1) {
#pragma unroll
        for (int j = 0; j < NPT; ++j)
          if (OWN(j)) u[j] = clamp_dom64(v[j], sm.V[t + j * kClusterThreads], d.W, d.H);
      } else {
        double2* dst = (q & 1) ? sm.xu0 : sm.xu1;
#pragma unroll
        for (int j = 0; j < NPT; ++j)
          if (OWN(j)) dst[t + j * kClusterThreads] = v[j];
      }
    }
    if (warp == kCtlWarp) control(k);
  }
#pragma unroll
  for (int j = 0; j < NPT; ++j)
    if (OWN(j)) d.u[rank * d.chunk + t + j * kClusterThreads] = u[j];
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

}  // namespace mrb
