// Cluster registration kernel with a PUSH halo exchange (fp32 fast path,
// smoothing_passes <= 1).  Same iteration and numerics as k_cluster_register
// (cluster.cuh); what changes is how neighbour values move:
//
//   pull (cluster.cuh): write own values, cluster barrier, every CTA loads its
//        halo from the owners' shared memory (a DSMEM round trip per value).
//   push (here):        the owner stores each value straight into every
//        consumer's halo slot with st.async, which also credits the bytes to
//        the consumer's mbarrier; a consumer waits only for its own halo bytes.
//
// There is no cluster barrier inside the loop.  Halo buffers and mbarriers are
// double-buffered by iteration parity; since the neighbour relation is
// symmetric, a CTA can run at most one iteration ahead of any neighbour, so a
// parity buffer is never overwritten while it is read.  The energy partial
// and the non-finite-gradient flag of iteration k go to every CTA as one
// 16-byte message after phase B; each CTA's control warp reduces the CS
// messages in rank order (the same fixed order as the pull kernel) and
// decides; the decision is read after phase A of iteration k+1, before that
// iteration sends anything, so all CTAs stop on the same iteration with no
// message in flight.
#pragma once

#include "cluster.cuh"

namespace mrb {

__device__ __forceinline__ void mbar_init(uint32_t mb, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mb), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect(uint32_t mb, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t mb, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n W_%=:\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W_%=;\n}" ::"r"(mb),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void st_async_f32(uint32_t addr, float v, uint32_t mb) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
                   addr),
               "r"(__float_as_uint(v)), "r"(mb)
               : "memory");
}

__device__ __forceinline__ void st_async_f32x2(uint32_t addr, float2 v, uint32_t mb) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1, %2}, [%3];" ::"r"(
          addr),
      "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y)), "r"(mb)
      : "memory");
}

__device__ __forceinline__ void st_async_v4(uint32_t addr, uint4 v, uint32_t mb) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, "
      "[%5];" ::"r"(addr),
      "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(mb)
      : "memory");
}

// Dynamic shared memory of k_cluster_push (host: push_dyn_smem).
// The paired SELL coefficients (float4) come first: 16-byte aligned.
struct PushSmem {
  float4* g4;
  double2* V;
  float2 *gs, *xu[2];  // xu[p]: u0 of iteration parity p, own slots then halo
  float *iv, *xs[2];   // xs[p]: s_te of iteration parity p, own slots then halo
  uint32_t* send;
  uint32_t* code2;
  uint32_t* soff;
};

template <int NPT>
__device__ __forceinline__ PushSmem push_carve(unsigned char* p, const ClusterPair& d) {
  constexpr int SLOTS = kClusterThreads * NPT;
  const int X = SLOTS + d.halo_stride;
  PushSmem s;
  s.g4 = reinterpret_cast<float4*>(p);
  s.V = reinterpret_cast<double2*>(s.g4 + d.topo_stride / 2);  // topo_stride % 8 == 0
  s.gs = reinterpret_cast<float2*>(s.V + SLOTS);
  s.xu[0] = s.gs + SLOTS;
  s.xu[1] = s.xu[0] + X;
  s.iv = reinterpret_cast<float*>(s.xu[1] + X);
  s.xs[0] = s.iv + SLOTS;
  s.xs[1] = s.xs[0] + X;
  s.send = reinterpret_cast<uint32_t*>(s.xs[1] + X);
  s.code2 = s.send + d.send_stride;
  s.soff = s.code2 + d.topo_stride / 2;
  return s;
}

template <int NPT>
__global__ void __launch_bounds__(kClusterThreads, kClusterMinBlocks)
    k_cluster_push(const ClusterPair* __restrict__ pairs, PairStatus* __restrict__ st,
                   int max_iter, double tol, float tau, float lam, int passes) {
  constexpr int SLOTS = kClusterThreads * NPT;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = int(cluster.block_rank());
  const int CS = int(cluster.num_blocks());
  const int p = blockIdx.x / CS;
  const ClusterPair& d = pairs[p];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;

  __shared__ double s_wpart[kWarps];
  __shared__ __align__(16) uint4 s_msg[2][16];  // [parity][rank]: energy partial, bad flag
  __shared__ __align__(8) unsigned long long s_mb[6];  // s_te[2], u0[2], msg[2]
  __shared__ int s_stop, s_nhalo, s_nsend;
  __shared__ double s_hist[6];
  __shared__ double s_prev;
  __shared__ int s_cs[4];  // rises, iters, err, err_iter
  extern __shared__ __align__(16) unsigned char s_dyn[];
  const PushSmem sm = push_carve<NPT>(s_dyn, d);

  const uint32_t mb0 = smem_u32(&s_mb[0]);
  auto mb_s = [&](int par) { return mb0 + 8u * par; };
  auto mb_u = [&](int par) { return mb0 + 8u * (2 + par); };
  auto mb_m = [&](int par) { return mb0 + 8u * (4 + par); };
  if (t == 0) {
    s_stop = 0;
    s_prev = 0.0;
    s_cs[0] = s_cs[1] = s_cs[2] = s_cs[3] = 0;
    s_nhalo = d.n_halo[rank];
    s_nsend = d.n_send[rank];
    for (int q = 0; q < 6; ++q) mbar_init(mb0 + 8u * q, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {  // this CTA's topology and send list
    const size_t tb = size_t(rank) * d.topo_stride;
    const float4* g4 = reinterpret_cast<const float4*>(d.g + tb);
    const uint32_t* c2 = reinterpret_cast<const uint32_t*>(d.codes + tb);
    for (int q = t; q < d.topo_stride / 2; q += kClusterThreads) {
      sm.g4[q] = g4[q];
      sm.code2[q] = c2[q];
    }
    if (t == 0) {  // the ZERO slot of the padding entries, both parities
      const int zero = SLOTS + d.halo_stride - 1;
      sm.xs[0][zero] = sm.xs[1][zero] = 0.f;
      sm.xu[0][zero] = sm.xu[1][zero] = make_float2(0.f, 0.f);
    }
    for (int q = t; q < d.slices; q += kClusterThreads)
      sm.soff[q] = d.slice_off[size_t(rank) * d.slices + q];
    for (int q = t; q < d.send_stride; q += kClusterThreads)
      sm.send[q] = d.send[size_t(rank) * d.send_stride + q];
  }
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
  // every CTA's mbarriers are initialised before anyone pushes into them
  cluster_sync_all();
  const int nhalo = s_nhalo, nsend = s_nsend;
  const unsigned halo_s_bytes = 4u * unsigned(nhalo), halo_u_bytes = 8u * unsigned(nhalo);
  const ImgView img = img_view(d);
  const uint32_t xs_a0 = smem_u32(sm.xs[0]), xs_a1 = smem_u32(sm.xs[1]);
  const uint32_t xu_a0 = smem_u32(sm.xu[0]), xu_a1 = smem_u32(sm.xu[1]);
  const uint32_t msg_addr = smem_u32(&s_msg[0][0]);

  // control step of iteration kk on the control warp: CS messages, rank order
  auto control = [&](int kk) {
    const int par = kk & 1;
    mbar_wait(mb_m(par), unsigned(kk >> 1) & 1u);
    double v = 0.0;
    int gb = 0;
    if (lane < CS) {
      const uint4 m = s_msg[par][lane];
      v = __hiloint2double(int(m.y), int(m.x));
      gb = int(m.z);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v += __shfl_down_sync(0xffffffffu, v, o);
      gb |= __shfl_down_sync(0xffffffffu, gb, o);
    }
    if (lane == 0) {
      if (s_stop == 0) {
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
      // re-arm this parity's message barrier for iteration kk + 2
      mbar_expect(mb_m(par), 16u * unsigned(CS));
    }
  };

  if (t == 0) {  // arm both parities of every exchange
    for (int par = 0; par < 2; ++par) {
      mbar_expect(mb_s(par), halo_s_bytes);
      mbar_expect(mb_u(par), halo_u_bytes);
      mbar_expect(mb_m(par), 16u * unsigned(CS));
    }
  }

  // debug: per-CTA stamps of the first 8 iterations (MESHREG_B200_PROFILE_PHASES;
  // "mapped": iteration numbers readable during a hang, else clock64 cycles)
#ifdef MRB_PHASE_PROFILE  // build flag
  volatile long long* const trace_pt =
      (d.prof && t == 0) ? d.prof + size_t(rank) * 128 : nullptr;
#define TRACE(slot) \
  if (trace_pt && k < 8) trace_pt[k * 16 + (slot)] = clock64();
#else
#define TRACE(slot)
#endif
  int k = 0;
  for (; k < max_iter; ++k) {
    const int par = k & 1;
    TRACE(0)
    const unsigned ph = unsigned(k >> 1) & 1u;  // phase of this parity's barriers
    float* xs = par ? sm.xs[1] : sm.xs[0];
    float2* xu = par ? sm.xu[1] : sm.xu[0];
    const uint32_t xs_addr = par ? xs_a1 : xs_a0, xu_addr = par ? xu_a1 : xu_a0;
    // -------- phase A: sample Te, Re at V + u; residual; energy partial
    {
      double e2 = 0.0;
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        if (OWN(j)) {
          const double2 V = sm.V[t + j * kClusterThreads];
          const Window w = locate(img, V.x + double(u[j].x), V.y + double(u[j].y));
          float2 tap[4][4];
#pragma unroll
          for (int row = 0; row < 4; ++row) ld_row4(w.base + size_t(row) * img.pitch, tap[row]);
          const float2 s = combine(w, tap);
          r[j] = s.x - s.y;
          xs[t + j * kClusterThreads] = s.x;
          e2 = fma(double(r[j]), double(r[j]), e2);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) e2 += __shfl_down_sync(0xffffffffu, e2, o);
      if (lane == 0) s_wpart[warp] = e2;
    }
    TRACE(7)
    __syncthreads();     // own s_te, warp partials, the decision of k-1
    // Re-arm the u0 barrier of iteration k-1's parity (used again by k+1) only
    // now that every thread has passed its wait: with an empty halo the
    // re-armed phase completes at once, and a thread still waiting on the old
    // phase would then wait for the next one forever.
    if (t == 0 && k > 0 && passes > 0) mbar_expect(mb_u(par ^ 1), halo_u_bytes);
    TRACE(6)
    if (s_stop) break;  // decision of k-1, identical in every CTA: nobody sends for k
    for (int q = t; q < nsend; q += kClusterThreads) {  // push s_te to its consumers
      const uint32_t e = sm.send[q];
      const uint32_t dst = e >> 16 & 0xfu;
      st_async_f32(mapa_u32(xs_addr, dst) + 4u * (SLOTS + (e & 0xffffu)),
                   xs[e >> 20], mapa_u32(mb_s(par), dst));
    }
    TRACE(1)
    mbar_wait(mb_s(par), ph);  // my s_te halo has arrived
    TRACE(2)
    // -------- phase B: gradient via the fused one-ring operator, descent
    bool bad = false;
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
      if (OWN(j)) {
        const int slot = t + j * kClusterThreads;
        const float si = xs[slot];
        const float2 gs = sm.gs[slot];
        float gx = gs.x * si, gy = gs.y * si;
        ring_pairs(sm.code2, sm.soff[slot >> 5], lane, [&](uint32_t cc, uint32_t at) {
          const float s0 = xs[cc & 0xffffu], s1 = xs[cc >> 16];
          const float4 ge = sm.g4[at];
          gx = fmaf(ge.x, s0, gx);
          gy = fmaf(ge.y, s0, gy);
          gx = fmaf(ge.z, s1, gx);
          gy = fmaf(ge.w, s1, gy);
        });
        const float dx = r[j] * gx, dy = r[j] * gy;  // solver.py:189
        bad |= !isfinite(dx) || !isfinite(dy);
        xu[slot] = make_float2(u[j].x - tau * dx, u[j].y - tau * dy);  // solver.py:133
      }
    }
    const int anybad = __syncthreads_or(bad);  // also: own u0 complete
    // re-arm for iteration k + 2: every thread passed its wait (barrier above)
    if (t == 0) mbar_expect(mb_s(par), halo_s_bytes);
    if (warp == kCtlWarp) {  // energy partial + flag of iteration k to every CTA
      double v = lane < kWarps ? s_wpart[lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      v = __shfl_sync(0xffffffffu, v, 0);
      if (lane < CS) {
        const uint4 m = make_uint4(unsigned(__double2loint(v)), unsigned(__double2hiint(v)),
                                   unsigned(anybad), 0u);
        st_async_v4(mapa_u32(msg_addr, lane) + 16u * (par * 16 + rank), m,
                    mapa_u32(mb_m(par), lane));
      }
    }
    // -------- phase C: umbrella smoothing (one pass) + domain clamp
    if (passes == 0) {
#pragma unroll
      for (int j = 0; j < NPT; ++j)
        if (OWN(j)) {
          const int slot = t + j * kClusterThreads;
          u[j] = clamp_dom(xu[slot], sm.V[slot], img.W, img.H);
        }
    } else {
      for (int q = t; q < nsend; q += kClusterThreads) {  // push u0 to its consumers
        const uint32_t e = sm.send[q];
        const uint32_t dst = e >> 16 & 0xfu;
        st_async_f32x2(mapa_u32(xu_addr, dst) + 8u * (SLOTS + (e & 0xffffu)),
                       xu[e >> 20], mapa_u32(mb_u(par), dst));
      }
      TRACE(3)
      mbar_wait(mb_u(par), ph);  // my u0 halo has arrived
      TRACE(4)
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        if (OWN(j)) {
          const int slot = t + j * kClusterThreads;
          const float ivs = sm.iv[slot];
          float ax = 0.f, ay = 0.f;
          // (L u)_i, L_ij = 1/val_i
          ring_pairs(sm.code2, sm.soff[slot >> 5], lane, [&](uint32_t cc, uint32_t) {
            const float2 u0 = xu[cc & 0xffffu], u1 = xu[cc >> 16];
            ax = fmaf(ivs, u0.x, ax);
            ay = fmaf(ivs, u0.y, ay);
            ax = fmaf(ivs, u1.x, ax);
            ay = fmaf(ivs, u1.y, ay);
          });
          const float2 si = xu[slot];
          const float om = 1.f - lam;  // (1 - lam) u + lam (L u), mesh.py:281
          u[j] = clamp_dom(make_float2(om * si.x + lam * ax, om * si.y + lam * ay), sm.V[slot],
                           img.W, img.H);
        }
      }
    }
    // -------- control of iteration k (waits for the CS messages of k); its
    // decision is read after phase A of k+1.  Every message is consumed here,
    // so none can still be in flight into this CTA when it exits.
    if (warp == kCtlWarp) control(k);
    TRACE(5)
  }
#undef TRACE
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
  cluster_sync_all();  // no CTA leaves while a peer could still address its memory
}

}  // namespace mrb
