// fp64 cluster loop with the PUSH halo exchange (smoothing_passes <= 1):
// k_cluster64's state, coefficients and sampling (cluster64.cuh) moved by
// k_cluster_push's exchange (push.cuh) — each owner st.async-stores its
// boundary s_te / u0 values into the consumers' halo slots, crediting their
// mbarriers; halo buffers and mbarriers double-buffered by iteration parity;
// energy partials and gradient flags travel as one 16-byte message per CTA;
// no cluster barrier inside the loop.  Same per-node arithmetic as the pull
// kernel, same fixed reduction order, so the fields are bit-identical.
#pragma once

#include "cluster64.cuh"
#include "push.cuh"

namespace mrb {

__device__ __forceinline__ void st_async_f64(uint32_t addr, double v, uint32_t mb) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(
                   addr),
               "d"(v), "r"(mb)
               : "memory");
}

__device__ __forceinline__ void st_async_f64x2(uint32_t addr, double2 v, uint32_t mb) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
          addr),
      "d"(v.x), "d"(v.y), "r"(mb)
      : "memory");
}

// Dynamic shared memory (host: push64_dyn_smem)
struct Push64Smem {
  double2* g;
  double2 *V, *gs, *xu[2];
  double *iv, *xs[2];
  uint32_t *send, *code2, *soff;
};

__device__ __forceinline__ Push64Smem push64_carve(unsigned char* p, const ClusterPair64& d) {
  constexpr int SLOTS = kClusterThreads;
  const int X = SLOTS + d.halo_stride;
  Push64Smem s;
  s.g = reinterpret_cast<double2*>(p);
  s.V = s.g + d.topo_stride;
  s.gs = s.V + SLOTS;
  s.xu[0] = s.gs + SLOTS;
  s.xu[1] = s.xu[0] + X;
  s.iv = reinterpret_cast<double*>(s.xu[1] + X);
  s.xs[0] = s.iv + SLOTS;
  s.xs[1] = s.xs[0] + X;
  s.send = reinterpret_cast<uint32_t*>(s.xs[1] + X);
  s.code2 = s.send + d.send_stride;
  s.soff = s.code2 + d.topo_stride / 2;
  return s;
}

__global__ void __launch_bounds__(kClusterThreads, 1)
    k_cluster64_push(const ClusterPair64* __restrict__ pairs, PairStatus* __restrict__ st,
                     int max_iter, double tol, double tau, double lam, int passes) {
  constexpr int SLOTS = kClusterThreads;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = int(cluster.block_rank());
  const int CS = int(cluster.num_blocks());
  const int p = blockIdx.x / CS;
  const ClusterPair64& d = pairs[p];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;

  __shared__ double s_wpart[kWarps];
  __shared__ __align__(16) uint4 s_msg[2][16];  // [parity][rank]: energy partial, bad flag
  __shared__ __align__(8) unsigned long long s_mb[6];  // s_te[2], u0[2], msg[2]
  __shared__ int s_stop, s_nhalo, s_nsend;
  __shared__ double s_hist[6];
  __shared__ double s_prev;
  __shared__ int s_cs[4];  // rises, iters, err, err_iter
  extern __shared__ __align__(16) unsigned char s_dyn[];
  const Push64Smem sm = push64_carve(s_dyn, d);

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
    const uint32_t* c2 = reinterpret_cast<const uint32_t*>(d.codes + tb);
    for (int q = t; q < d.topo_stride; q += kClusterThreads) sm.g[q] = d.g[tb + q];
    for (int q = t; q < d.topo_stride / 2; q += kClusterThreads) sm.code2[q] = c2[q];
    if (t == 0) {  // the ZERO slot of the padding entries, both parities
      const int zero = SLOTS + d.halo_stride - 1;
      sm.xs[0][zero] = sm.xs[1][zero] = 0.0;
      sm.xu[0][zero] = sm.xu[1][zero] = make_double2(0.0, 0.0);
    }
    for (int q = t; q < d.slices; q += kClusterThreads)
      sm.soff[q] = d.slice_off[size_t(rank) * d.slices + q];
    for (int q = t; q < d.send_stride; q += kClusterThreads)
      sm.send[q] = d.send[size_t(rank) * d.send_stride + q];
  }
  const int slot = t;
  const int nd = rank * d.chunk + slot;
  const bool own = slot < d.chunk && nd < d.n;
  sm.V[slot] = own ? d.V[nd] : make_double2(0.0, 0.0);
  sm.gs[slot] = own ? d.g_self[nd] : make_double2(0.0, 0.0);
  sm.iv[slot] = own ? d.inv_val[nd] : 0.0;
  double2 u = make_double2(0.0, 0.0);
  double r = 0.0;
  // every CTA's mbarriers are initialised before anyone pushes into them
  cluster_sync_all();
  const int nhalo = s_nhalo, nsend = s_nsend;
  const unsigned halo_s_bytes = 8u * unsigned(nhalo), halo_u_bytes = 16u * unsigned(nhalo);
  const uint32_t xs_a0 = smem_u32(sm.xs[0]), xs_a1 = smem_u32(sm.xs[1]);
  const uint32_t xu_a0 = smem_u32(sm.xu[0]), xu_a1 = smem_u32(sm.xu[1]);
  const uint32_t msg_addr = smem_u32(&s_msg[0][0]);

  // control step of iteration kk on the control warp: CS messages, rank
  // order (k_cluster_push's; solver.py:174-195)
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
      mbar_expect(mb_m(par), 16u * unsigned(CS));  // re-arm for iteration kk + 2
    }
  };

  if (t == 0) {  // arm both parities of every exchange
    for (int par = 0; par < 2; ++par) {
      mbar_expect(mb_s(par), halo_s_bytes);
      mbar_expect(mb_u(par), halo_u_bytes);
      mbar_expect(mb_m(par), 16u * unsigned(CS));
    }
  }

  int k = 0;
  for (; k < max_iter; ++k) {
    const int par = k & 1;
    const unsigned ph = unsigned(k >> 1) & 1u;  // phase of this parity's barriers
    double* xs = par ? sm.xs[1] : sm.xs[0];
    double2* xu = par ? sm.xu[1] : sm.xu[0];
    const uint32_t xs_addr = par ? xs_a1 : xs_a0, xu_addr = par ? xu_a1 : xu_a0;
    // -------- phase A: sample Te, Re at V + u; residual; energy partial
    {
      double e2 = 0.0;
      if (own) {
        const double2 V = sm.V[slot];
        const double2 s = d.img4 ? sample_int64(d, V.x + u.x, V.y + u.y)
                                 : sample_pad64(d.pad, d.W, d.H, V.x + u.x, V.y + u.y);
        r = s.x - s.y;
        xs[slot] = s.x;
        e2 = r * r;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) e2 += __shfl_down_sync(0xffffffffu, e2, o);
      if (lane == 0) s_wpart[warp] = e2;
    }
    __syncthreads();  // own s_te, warp partials, the decision of k-1
    if (t == 0 && k > 0 && passes > 0) mbar_expect(mb_u(par ^ 1), halo_u_bytes);
    if (s_stop) break;  // decision of k-1, identical in every CTA: nobody sends for k
    for (int q = t; q < nsend; q += kClusterThreads) {  // push s_te to its consumers
      const uint32_t e = sm.send[q];
      const uint32_t dst = e >> 16 & 0xfu;
      st_async_f64(mapa_u32(xs_addr, dst) + 8u * (SLOTS + (e & 0xffffu)), xs[e >> 20],
                   mapa_u32(mb_s(par), dst));
    }
    mbar_wait(mb_s(par), ph);  // my s_te halo has arrived
    // -------- phase B: grad = r * G s_te, u0 = u - tau * grad (solver.py:133,189)
    bool bad = false;
    if (own) {
      const double si = xs[slot];
      const double2 gs = sm.gs[slot];
      double gx = gs.x * si, gy = gs.y * si;
      ring_pairs(sm.code2, sm.soff[slot >> 5], lane, [&](uint32_t cc, uint32_t at) {
        const double s0 = xs[cc & 0xffffu], s1 = xs[cc >> 16];
        const double2 g0 = sm.g[2 * at], g1 = sm.g[2 * at + 1];
        gx = fma(g0.x, s0, gx);
        gy = fma(g0.y, s0, gy);
        gx = fma(g1.x, s1, gx);
        gy = fma(g1.y, s1, gy);
      });
      const double dx = r * gx, dy = r * gy;
      bad = !isfinite(dx) || !isfinite(dy);
      xu[slot] = make_double2(u.x - tau * dx, u.y - tau * dy);
    }
    const int anybad = __syncthreads_or(bad);  // also: own u0 complete
    if (t == 0) mbar_expect(mb_s(par), halo_s_bytes);  // re-arm for k + 2
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
      if (own) u = clamp_dom64(xu[slot], sm.V[slot], d.W, d.H);
    } else {
      for (int q = t; q < nsend; q += kClusterThreads) {  // push u0 to its consumers
        const uint32_t e = sm.send[q];
        const uint32_t dst = e >> 16 & 0xfu;
        st_async_f64x2(mapa_u32(xu_addr, dst) + 16u * (SLOTS + (e & 0xffffu)), xu[e >> 20],
                       mapa_u32(mb_u(par), dst));
      }
      mbar_wait(mb_u(par), ph);  // my u0 halo has arrived
      if (own) {
        const double iv = sm.iv[slot];
        double ax = 0.0, ay = 0.0;
        ring_pairs(sm.code2, sm.soff[slot >> 5], lane, [&](uint32_t cc, uint32_t) {
          const double2 u0 = xu[cc & 0xffffu], u1 = xu[cc >> 16];
          ax = fma(iv, u0.x, ax);
          ay = fma(iv, u0.y, ay);
          ax = fma(iv, u1.x, ax);
          ay = fma(iv, u1.y, ay);
        });
        const double2 si = xu[slot];
        const double om = 1.0 - lam;
        u = clamp_dom64(make_double2(om * si.x + lam * ax, om * si.y + lam * ay), sm.V[slot],
                        d.W, d.H);
      }
    }
    if (warp == kCtlWarp) control(k);
  }
  if (own) d.u[nd] = u;
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
