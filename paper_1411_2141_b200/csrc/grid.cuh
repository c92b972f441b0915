// Whole-GPU persistent registration kernel for meshes larger than one
// thread-block cluster holds (BASELINE configs 3 and 5; fp32 fast path).
//
// Same iteration as k_cluster_register (cluster.cuh) with the cluster swapped
// for the whole grid: CTA r of CS co-resident CTAs (cooperative launch, one
// per SM) owns the Morton chunk [r*chunk, (r+1)*chunk) of one pair.  Owners
// publish s_te / u0 to global exchange arrays; after a grid barrier each CTA
// pulls its halo (L2, bypassing L1) into shared memory, so the one-ring
// gathers of the fused gradient operator and of the umbrella Laplacian stay
// shared-memory loads.  The SELL-32 topology and the per-node constants are
// read through the read-only path (L1/L2 resident across iterations), so the
// kernel has no per-CTA topology size limit.  Every CTA reduces all energy
// partials in one fixed order and runs the control logic itself (identical
// decisions, no broadcast); the decision of iteration k is read after the
// first barrier of iteration k+1, as in the cluster kernel.
#pragma once

#include "cluster.cuh"

namespace mrb {

// Sense-free grid barrier on a monotonic counter: the n-th barrier of a launch
// waits until the counter reaches n * gridDim.x.  Release/acquire at gpu scope
// order the exchange-array writes before the halo reads of other CTAs.
__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// one-ring gather over this CTA's paired SELL topology in global memory
// (read through L1; layout in write_topo): f(codes of entries 2p | 2p+1 <<
// 16, row index) for the slice's warp-uniform pair-row count
template <int NP, typename F>
__device__ __forceinline__ void ring_pairs_gn(const uint32_t* __restrict__ code2, uint32_t base,
                                              F&& f) {
  uint32_t cc[NP];
#pragma unroll
  for (int q = 0; q < NP; ++q) cc[q] = __ldg(code2 + base + 32u * q);  // all codes first
#pragma unroll
  for (int q = 0; q < NP; ++q) f(cc[q], base + 32u * q);
}

template <typename F>
__device__ __forceinline__ void ring_pairs_g(const uint32_t* __restrict__ code2, uint32_t sw,
                                             int lane, F&& f) {
  const uint32_t base = (sw & 0xffffffu) + uint32_t(lane);
  const int np = int(sw >> 24);
  switch (np) {  // warp-uniform: fully unrolled bodies for the usual counts
    case 2: ring_pairs_gn<2>(code2, base, f); return;
    case 3: ring_pairs_gn<3>(code2, base, f); return;
    case 4: ring_pairs_gn<4>(code2, base, f); return;
    case 5: ring_pairs_gn<5>(code2, base, f); return;
    default: break;
  }
#pragma unroll 2
  for (int q = 0; q < np; ++q) {
    const uint32_t at = base + 32u * uint32_t(q);
    f(__ldg(code2 + at), at);
  }
}

template <int NPT>
__global__ void __launch_bounds__(kClusterThreads, kClusterMinBlocks)
    k_grid_register(const ClusterPair* __restrict__ pairs, PairStatus* __restrict__ st,
                    int max_iter, double tol, float tau, float lam, int passes) {
  constexpr int SLOTS = kClusterThreads * NPT;
  const int rank = blockIdx.x, CS = gridDim.x;
  const ClusterPair& d = pairs[0];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  __shared__ int s_stop, s_nhalo;
  __shared__ double s_hist[6];
  __shared__ double s_prev;
  __shared__ int s_cs[4];  // rises, iters, err, err_iter
  extern __shared__ __align__(16) unsigned char s_dyn[];
  const int X = SLOTS + d.halo_stride;
  float* xs = reinterpret_cast<float*>(s_dyn);             // [X] s_te, own + halo
  float2* xu0 = reinterpret_cast<float2*>(xs + X + (X & 1));
  float2* xu1 = xu0 + X;                                   // [X] when passes >= 2
  uint32_t* halo = reinterpret_cast<uint32_t*>(xu1 + (passes >= 2 ? X : 0));

  if (t == 0) {
    s_stop = 0;
    s_prev = 0.0;
    s_cs[0] = s_cs[1] = s_cs[2] = s_cs[3] = 0;
    s_nhalo = d.n_halo[rank];
  }
  for (int q = t; q < d.halo_stride; q += kClusterThreads)
    halo[q] = d.halo[size_t(rank) * d.halo_stride + q];
  const uint32_t* code2 = reinterpret_cast<const uint32_t*>(d.codes + size_t(rank) * d.topo_stride);
  const float4* g4 = reinterpret_cast<const float4*>(d.g + size_t(rank) * d.topo_stride);
  if (t == 0) {  // ZERO slot of the padding entries
    xs[X - 1] = 0.f;
    xu0[X - 1] = make_float2(0.f, 0.f);
    if (passes >= 2) xu1[X - 1] = make_float2(0.f, 0.f);
  }
  const uint32_t* soff = d.slice_off + size_t(rank) * d.slices;
  float* xg_s = d.xg_s;
  float2* xg_u0 = d.xg_u;
  float2* xg_u1 = d.xg_u + size_t(CS) * SLOTS;

  float2 u[NPT];
  float r[NPT];
  unsigned own_mask = 0;
#pragma unroll
  for (int j = 0; j < NPT; ++j) {
    const int slot = t + j * kClusterThreads;
    own_mask |= unsigned(slot < d.chunk && rank * d.chunk + slot < d.n) << j;
    u[j] = make_float2(0.f, 0.f);
    r[j] = 0.f;
  }
#define OWN(j) ((own_mask >> (j)) & 1u)
  unsigned nbar = 0;
  auto gsync = [&]() { grid_barrier(d.bar, ++nbar * unsigned(CS)); };
  __syncthreads();
  const int nhalo = s_nhalo;

  __shared__ double s_wpart[kWarps];
  // control step of iteration kk: the CS CTA partials in one fixed order
  auto control = [&](int kk) {
    double v = 0.0;
    const double* wp = d.wpart + size_t(kk & 1) * CS;
    for (int idx = lane; idx < CS; idx += 32) v += __ldcg(wp + idx);
    int gb = 0;
    for (int idx = lane; idx < CS; idx += 32) gb |= __ldcg(d.gbad + idx);
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
        if (kk + 1 >= 6) {  // solver.py:192-195
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
    // -------- phase A: sample Te, Re at V + u; residual; energy partial
    {
      double e2 = 0.0;
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        if (OWN(j)) {
          const int slot = t + j * kClusterThreads;
          const int nd = rank * d.chunk + slot;
          const double2 V = __ldg(d.V + nd);
          const Window w = locate(d, V.x + double(u[j].x), V.y + double(u[j].y));
          float2 tap[4][4];
#pragma unroll
          for (int row = 0; row < 4; ++row) ld_row4(w.base + size_t(row) * d.pitch, tap[row]);
          const float2 s = combine(w, tap);
          r[j] = s.x - s.y;
          xs[slot] = s.x;
          __stcg(xg_s + size_t(rank) * SLOTS + slot, s.x);
          e2 = fma(double(r[j]), double(r[j]), e2);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) e2 += __shfl_down_sync(0xffffffffu, e2, o);
      if (lane == 0) s_wpart[warp] = e2;
    }
    gsync();            // s_te, energy partials (and the k-1 decision) visible
    if (s_stop) break;  // iteration k-1 was the last one (u untouched since)
    for (int h = t; h < nhalo; h += kClusterThreads) {  // pull the s_te halo
      const uint32_t c = halo[h];
      xs[SLOTS + h] = __ldcg(xg_s + size_t(c >> 16) * SLOTS + (c & 0xffffu));
    }
    if (warp == kCtlWarp) {  // CTA energy partial of iteration k, fixed order; read by
      // every CTA's control(k) after the next grid barrier
      double v = lane < kWarps ? s_wpart[lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      if (lane == 0) __stcg(d.wpart + size_t(k & 1) * CS + rank, v);
    }
    __syncthreads();

    // -------- phase B: gradient via the fused one-ring operator, descent
    bool bad = false;
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
      if (OWN(j)) {
        const int slot = t + j * kClusterThreads;
        const int nd = rank * d.chunk + slot;
        const float si = xs[slot];
        const float2 gs = __ldg(d.g_self + nd);
        float gx = gs.x * si, gy = gs.y * si;
        ring_pairs_g(code2, __ldg(soff + (slot >> 5)), lane, [&](uint32_t cc, uint32_t at) {
          const float s0 = xs[cc & 0xffffu], s1 = xs[cc >> 16];
          const float4 ge = __ldg(g4 + at);
          gx = fmaf(ge.x, s0, gx);
          gy = fmaf(ge.y, s0, gy);
          gx = fmaf(ge.z, s1, gx);
          gy = fmaf(ge.w, s1, gy);
        });
        const float dx = r[j] * gx, dy = r[j] * gy;  // solver.py:189
        bad |= !isfinite(dx) || !isfinite(dy);
        const float2 v = make_float2(u[j].x - tau * dx, u[j].y - tau * dy);  // solver.py:133
        xu0[slot] = v;
        __stcg(xg_u0 + size_t(rank) * SLOTS + slot, v);
      }
    }
    if (__syncthreads_or(bad) && t == 0) __stcg(d.gbad + rank, 1);

    // -------- phase C: umbrella smoothing passes + domain clamp
    if (passes == 0) {
      gsync();  // gradbad flags visible
#pragma unroll
      for (int j = 0; j < NPT; ++j)
        if (OWN(j)) {
          const int slot = t + j * kClusterThreads;
          u[j] = clamp_dom(xu0[slot], __ldg(d.V + rank * d.chunk + slot), d.W, d.H);
        }
    }
    for (int q = 0; q < passes; ++q) {
      float2* src = (q & 1) ? xu1 : xu0;
      const float2* gsrc = (q & 1) ? xg_u1 : xg_u0;
      gsync();  // src (and the gradbad flags) visible grid-wide
      for (int h = t; h < nhalo; h += kClusterThreads) {  // pull the halo of src
        const uint32_t c = halo[h];
        src[SLOTS + h] = __ldcg(gsrc + size_t(c >> 16) * SLOTS + (c & 0xffffu));
      }
      __syncthreads();
      float2 v[NPT];
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        v[j] = make_float2(0.f, 0.f);
        if (OWN(j)) {
          const int slot = t + j * kClusterThreads;
          const int nd = rank * d.chunk + slot;
          const float iv = __ldg(d.inv_val + nd);
          float ax = 0.f, ay = 0.f;
          ring_pairs_g(code2, __ldg(soff + (slot >> 5)), lane, [&](uint32_t cc, uint32_t) {
            const float2 u0 = src[cc & 0xffffu], u1 = src[cc >> 16];  // (L u)_i, L_ij = 1/val_i
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
          if (OWN(j))
            u[j] = clamp_dom(v[j], __ldg(d.V + rank * d.chunk + t + j * kClusterThreads), d.W,
                             d.H);
      } else {
        float2* dst = (q & 1) ? xu0 : xu1;
        float2* gdst = (q & 1) ? xg_u0 : xg_u1;
#pragma unroll
        for (int j = 0; j < NPT; ++j)
          if (OWN(j)) {
            const int slot = t + j * kClusterThreads;
            dst[slot] = v[j];
            __stcg(gdst + size_t(rank) * SLOTS + slot, v[j]);
          }
      }
    }
    if (warp == kCtlWarp) control(k);
  }
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
    st[0] = s;
  }
}

}  // namespace mrb

namespace mrb {

constexpr int kFlagStride = 32;  // unsigned words between flags (one 128-byte line)

// Epoch-tagged exchange words: a value and the epoch it belongs to packed in
// ONE 64-bit scalar (epoch << 32 | value bits), written and polled with a
// single b64 relaxed access.  A scalar access is single-copy atomic in the
// PTX memory model (a .v2.u32 access is not: its halves are separate
// accesses in unspecified order, so a torn (new epoch, old value) read would
// be allowed).  A consumer polls the data itself: one L2 round trip instead
// of flag + data.
__device__ __forceinline__ void put_tagged(uint2* p, float v, unsigned e) {
  const unsigned long long w =
      (static_cast<unsigned long long>(e) << 32) | __float_as_uint(v);
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ float get_tagged(const uint2* p, unsigned e) {
  unsigned long long w;
  do {
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  } while (static_cast<unsigned>(w >> 32) != e);
  return __uint_as_float(static_cast<unsigned>(w));
}

// Release-store / acquire-load of an epoch flag at gpu scope.
__device__ __forceinline__ void flag_release(unsigned* f, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned flag_acquire(const unsigned* f) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
  return v;
}

// k_grid_register with the two grid barriers per iteration replaced by
// epoch-tagged exchange words (smoothing_passes <= 1):
//   * each published s_te / u0 value carries the epoch k+1 in the same 8-byte
//     word; a consumer thread polls exactly the halo words it needs until
//     their epoch matches — no flag, no barrier, one L2 round trip;
//   * exchange arrays are double-buffered by iteration parity — the halo
//     relation is symmetric, so no CTA runs more than one iteration ahead of
//     a CTA that reads it;
//   * the CTA energy partial + non-finite-gradient flag of iteration k are
//     published after phase B into buffer k & 3 with a release-increment of
//     that buffer's counter; the control of iteration k runs one iteration
//     late (end of k+1), waits until the counter holds all CS contributions
//     and reduces the CS partials in one fixed order (identical decisions in
//     every CTA); the decision is read after phase A of k+2, before any CTA
//     waits on a word of k+2, so all CTAs stop together, and the field is
//     rolled back to the one the reference returns (u before step k+1).  Four
//     buffers: a CTA writing buffer k & 3 again at k+4 has waited for all
//     partials of k+2, so every CTA finished control(k).
template <int NPT, bool RP = false>  // RP: taps in the row-pair layout (k_pad_planar_rp)
__global__ void __launch_bounds__(kClusterThreads, kClusterMinBlocks)
    k_grid_flags(const ClusterPair* __restrict__ pairs, PairStatus* __restrict__ st, int max_iter,
                 double tol, float tau, float lam, int passes) {
  constexpr int SLOTS = kClusterThreads * NPT;
  const int rank = blockIdx.x, CS = gridDim.x;
  const ClusterPair& d = pairs[0];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  __shared__ int s_stop, s_nhalo;
  __shared__ double s_hist[6];
  __shared__ double s_prev;
  __shared__ double s_wpart[kWarps];
  __shared__ int s_cs[4];  // rises, iters, err, err_iter
  extern __shared__ __align__(16) unsigned char s_dyn[];
  const int X = SLOTS + d.halo_stride;
  float* xs = reinterpret_cast<float*>(s_dyn);
  float2* xu0 = reinterpret_cast<float2*>(xs + X + (X & 1));
  uint32_t* halo = reinterpret_cast<uint32_t*>(xu0 + X);
  // per-slot state kept in SMEM, not registers (NPT = 8 spilled it to local
  // memory, whose traffic competed with the taps for L2): u at the start of
  // the previous iteration (deferred control) and the residual
  float2* xsave = reinterpret_cast<float2*>(halo + d.halo_stride + (d.halo_stride & 1));
  float* xr = reinterpret_cast<float*>(xsave + SLOTS);

  if (t == 0) {
    s_stop = 0;
    s_prev = 0.0;
    s_cs[0] = s_cs[1] = s_cs[2] = s_cs[3] = 0;
    s_nhalo = d.n_halo[rank];
  }
  for (int q = t; q < d.halo_stride; q += kClusterThreads)
    halo[q] = d.halo[size_t(rank) * d.halo_stride + q];
  const uint32_t* code2 = reinterpret_cast<const uint32_t*>(d.codes + size_t(rank) * d.topo_stride);
  const float4* g4 = reinterpret_cast<const float4*>(d.g + size_t(rank) * d.topo_stride);
  if (t == 0) {  // ZERO slot of the padding entries
    xs[X - 1] = 0.f;
    xu0[X - 1] = make_float2(0.f, 0.f);
  }
  const uint32_t* soff = d.slice_off + size_t(rank) * d.slices;
  // one 128-byte line per flag: polled lines are never shared by two flags
  constexpr int FS = kFlagStride;
  unsigned* const flag_p = d.flags;  // [4] energy-partial counters, one line each
  double* const wpart = d.wpart;       // [4][CS] by iteration mod 4
  int* const gbad = d.gbad;            // [4][CS]

  float2 u[NPT];
  // NPT = 8 keeps u_save / r in SMEM (in registers they spill); smaller NPT
  // keeps them in registers
  constexpr bool kSmemState = NPT >= 8;  // NPT = 8: u_save / r in SMEM (registers spill)
  float2 u_save[kSmemState ? 1 : NPT];
  float r_reg[kSmemState ? 1 : NPT];
  auto save_u = [&](int j, float2 v) {
    if constexpr (kSmemState) xsave[t + j * kClusterThreads] = v; else u_save[j] = v;
  };
  auto saved_u = [&](int j) {
    if constexpr (kSmemState) return xsave[t + j * kClusterThreads]; else return u_save[j];
  };
  auto set_r = [&](int j, float v) {
    if constexpr (kSmemState) xr[t + j * kClusterThreads] = v; else r_reg[j] = v;
  };
  auto get_r = [&](int j) {
    if constexpr (kSmemState) return xr[t + j * kClusterThreads]; else return r_reg[j];
  };
  uint64_t tap_pol;
  if (d.tap_evict_first)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(tap_pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(tap_pol));
  unsigned own_mask = 0, exp_mask = 0;
  constexpr int WORDS = SLOTS / 32;
#pragma unroll
  for (int j = 0; j < NPT; ++j) {
    const int slot = t + j * kClusterThreads;
    own_mask |= unsigned(slot < d.chunk && rank * d.chunk + slot < d.n) << j;
    const unsigned ex =
        d.exports ? (__ldg(d.exports + size_t(rank) * WORDS + (slot >> 5)) >> (slot & 31)) & 1u
                  : 1u;
    exp_mask |= ex << j;
    u[j] = make_float2(0.f, 0.f);
    save_u(j, u[j]);
    set_r(j, 0.f);
  }
#define OWN(j) ((own_mask >> (j)) & 1u)
#define EXPORTED(j) ((exp_mask >> (j)) & 1u)
  __syncthreads();
  const int nhalo = s_nhalo;
  auto control = [&](int kk) {  // control warp, every CTA identically
    const int par = kk & 3;
    // all CS partials of iteration kk: the counter of buffer kk & 3 counts
    // every CTA's release-increment, so one polled word replaces CS flags
    const unsigned target = unsigned(CS) * (unsigned(kk >> 2) + 1u);
    if (lane == 0)
      while (flag_acquire(flag_p + size_t(par) * FS) < target) __nanosleep(20);
    __syncwarp();
    double v = 0.0;
    int gb = 0;
    for (int idx = lane; idx < CS; idx += 32) {
      v += __ldcg(wpart + size_t(par) * CS + idx);
      gb |= __ldcg(gbad + size_t(par) * CS + idx);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v += __shfl_down_sync(0xffffffffu, v, o);
      gb |= __shfl_down_sync(0xffffffffu, gb, o);
    }
    if (lane == 0 && s_stop == 0) {
      int stop = 0, rises = s_cs[0], err = ERR_NONE, err_iter = 0;
      const double en = 0.5 * v;
      const double prev = s_prev;
      if (!isfinite(en)) {  // solver.py:176-177
        err = ERR_NONFINITE_ENERGY;
        err_iter = kk;
        stop = 1;
      } else if (kk > 0 && en > __dadd_rn(__dmul_rn(prev, 1.0 + 1e-4), 1e-12)) {
        if (++rises >= 10) {  // material_rise, solver.py:43-44,178-184
          err = ERR_RISES;
          err_iter = kk;
          stop = 1;
        }
      } else if (kk > 0 && en <= prev) {
        rises = 0;  // solver.py:185-186
      }
      if (!stop && gb) {  // step(): non-finite gradient, solver.py:131-132
        err = ERR_NONFINITE_GRAD;
        err_iter = kk;
        stop = 1;
      }
      if (!stop) {
        s_cs[1] = kk + 1;
        s_hist[kk % 6] = en;
        if (kk + 1 >= 6) {  // solver.py:192-195
          const double base = s_hist[(kk + 1) % 6];
          if (fabs(__dsub_rn(en, base)) <= __dmul_rn(tol, fmax(fabs(base), 1e-12))) stop = 2;
        }
      }
      if (rank == 0) d.trace[kk] = en;
      s_prev = en;
      s_cs[0] = rises;
      s_cs[2] = err;
      s_cs[3] = err_iter;
      s_stop = stop;
    }
  };

  int k = 0;
  for (; k < max_iter; ++k) {
    const int par = k & 1;
    const unsigned e = unsigned(k) + 1u;
    // tagged exchange words: s_te [2][CS][SLOTS], u0 [2][CS][SLOTS][2] (x, y)
    uint2* xg_s = reinterpret_cast<uint2*>(d.xg_s) + size_t(par) * CS * SLOTS;
    uint2* xg_u = reinterpret_cast<uint2*>(d.xg_u) + size_t(par) * CS * SLOTS * 2;
    // -------- phase A: sample Te, Re at V + u; residual; energy partial
    {
      double e2 = 0.0;
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        if (OWN(j)) {
          const int slot = t + j * kClusterThreads;
          const int nd = rank * d.chunk + slot;
          const double2 V = __ldg(d.V + nd);
          float2 tap[4][4];
          Window w;
          w = locate<RP>(d, V.x + double(u[j].x), V.y + double(u[j].y));
#pragma unroll
          for (int row = 0; row < 4; ++row)  // row-pair layout: two 64-byte blocks per window
            ld_row4_pol(w.base + row_off<RP>(d.pitch, row), tap[row], tap_pol);
          const float2 s = combine(w, tap);
          const float rj = s.x - s.y;
          set_r(j, rj);
          xs[slot] = s.x;
          if (EXPORTED(j)) put_tagged(xg_s + size_t(rank) * SLOTS + slot, s.x, e);
          e2 = fma(double(rj), double(rj), e2);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) e2 += __shfl_down_sync(0xffffffffu, e2, o);
      if (lane == 0) s_wpart[warp] = e2;
    }
    __syncthreads();   // s_te published by all threads; decision of k-2
    // Control runs one iteration late (its all-CTA wait is then almost never
    // on the critical path).  If iteration k-2 ended the reference's loop, the
    // field it returns is the one before step k-1: restore it.  Identical in
    // every CTA, so no flag of iteration k is published.
    if (s_stop) {
#pragma unroll
      for (int j = 0; j < NPT; ++j) u[j] = saved_u(j);
      break;
    }
#pragma unroll
    for (int j = 0; j < NPT; ++j) save_u(j, u[j]);
    for (int h = t; h < nhalo; h += kClusterThreads) {  // the s_te halo, as it arrives
      const uint32_t c = halo[h];
      xs[SLOTS + h] = get_tagged(xg_s + size_t(c >> 16) * SLOTS + (c & 0xffffu), e);
    }
    __syncthreads();
    // -------- phase B: gradient via the fused one-ring operator, descent
    bool bad = false;
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
      if (OWN(j)) {
        const int slot = t + j * kClusterThreads;
        const int nd = rank * d.chunk + slot;
        const float si = xs[slot];
        const float2 gs = __ldg(d.g_self + nd);
        float gx = gs.x * si, gy = gs.y * si;
        ring_pairs_g(code2, __ldg(soff + (slot >> 5)), lane, [&](uint32_t cc, uint32_t at) {
          const float s0 = xs[cc & 0xffffu], s1 = xs[cc >> 16];
          const float4 ge = __ldg(g4 + at);
          gx = fmaf(ge.x, s0, gx);
          gy = fmaf(ge.y, s0, gy);
          gx = fmaf(ge.z, s1, gx);
          gy = fmaf(ge.w, s1, gy);
        });
        const float rj = get_r(j);
        const float dx = rj * gx, dy = rj * gy;  // solver.py:189
        bad |= !isfinite(dx) || !isfinite(dy);
        const float2 v = make_float2(u[j].x - tau * dx, u[j].y - tau * dy);  // solver.py:133
        xu0[slot] = v;
        if (passes > 0 && EXPORTED(j)) {
          uint2* w = xg_u + (size_t(rank) * SLOTS + slot) * 2;
          put_tagged(w, v.x, e);
          put_tagged(w + 1, v.y, e);
        }
      }
    }
    const int anybad = __syncthreads_or(bad);  // also: u0 published by all threads
    if (warp == kCtlWarp) {  // CTA partial + flag of iteration k, then its epoch
      double v = lane < kWarps ? s_wpart[lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      if (lane == 0) {
        const int q4 = k & 3;
        __stcg(wpart + size_t(q4) * CS + rank, v);
        __stcg(gbad + size_t(q4) * CS + rank, anybad);
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(flag_p + size_t(q4) * FS)
                     : "memory");
      }
    }
    // -------- phase C: umbrella smoothing (one pass) + domain clamp
    if (passes == 0) {
#pragma unroll
      for (int j = 0; j < NPT; ++j)
        if (OWN(j)) {
          const int slot = t + j * kClusterThreads;
          u[j] = clamp_dom(xu0[slot], __ldg(d.V + rank * d.chunk + slot), d.W, d.H);
        }
    } else {
      for (int h = t; h < nhalo; h += kClusterThreads) {  // the u0 halo, as it arrives
        const uint32_t c = halo[h];
        const uint2* w = xg_u + (size_t(c >> 16) * SLOTS + (c & 0xffffu)) * 2;
        xu0[SLOTS + h] = make_float2(get_tagged(w, e), get_tagged(w + 1, e));
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        if (OWN(j)) {
          const int slot = t + j * kClusterThreads;
          const int nd = rank * d.chunk + slot;
          const float iv = __ldg(d.inv_val + nd);
          float ax = 0.f, ay = 0.f;
          ring_pairs_g(code2, __ldg(soff + (slot >> 5)), lane, [&](uint32_t cc, uint32_t) {
            const float2 u0 = xu0[cc & 0xffffu], u1 = xu0[cc >> 16];  // (L u)_i, L_ij = 1/val_i
            ax = fmaf(iv, u0.x, ax);
            ay = fmaf(iv, u0.y, ay);
            ax = fmaf(iv, u1.x, ax);
            ay = fmaf(iv, u1.y, ay);
          });
          const float2 si = xu0[slot];
          const float om = 1.f - lam;  // (1 - lam) u + lam (L u), mesh.py:281
          u[j] = clamp_dom(make_float2(om * si.x + lam * ax, om * si.y + lam * ay),
                           __ldg(d.V + nd), d.W, d.H);
        }
      }
    }
    if (warp == kCtlWarp && k > 0) control(k - 1);
  }
  __syncthreads();
  if (k == max_iter) {  // the loop ran out: settle the last two decisions
    if (s_stop) {       // control(max_iter - 2) stopped: undo step max_iter - 1
#pragma unroll
      for (int j = 0; j < NPT; ++j) u[j] = saved_u(j);
    } else if (warp == kCtlWarp) {
      control(k - 1);
    }
  }
#pragma unroll
  for (int j = 0; j < NPT; ++j) {
    if (OWN(j)) {
      const int nd = rank * d.chunk + t + j * kClusterThreads;
      d.u[nd] = u[j];
      d.u_out[d.perm[nd]] = make_double2(double(u[j].x), double(u[j].y));
    }
  }
#undef OWN
#undef EXPORTED
  __syncthreads();
  if (rank == 0 && t == 0) {
    PairStatus s{};
    s.stop_iter = k;
    s.err = s_cs[2];
    s.err_iter = s_cs[3];
    s.rises = s_cs[0];
    s.iters = s_cs[1];
    st[0] = s;
  }
}

}  // namespace mrb
