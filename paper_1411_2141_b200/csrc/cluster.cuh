// Persistent thread-block-cluster registration kernel (fast path).
//
// One cluster of CS CTAs (CS <= 16) owns one pair for the whole descent loop
// (solver.py:171-195).  Each thread owns one mesh node (device/Morton order);
// its one-ring topology — neighbour codes and the fused gradient operator
// G = avg∘grad (mesh.py:236-241) — is staged once into shared memory in an
// entry-major [entry][thread] layout (bank-conflict-free) and reused for all
// iterations; the node state (V, u, r) stays in registers.
// The two neighbour exchanges per iteration (s_te for the gradient, u0 for the
// umbrella smoothing) go through distributed shared memory, ordered by
// hardware cluster barriers; nothing round-trips through global memory except
// the image taps.  The fp64 energy partial of every CTA is reduced in a fixed
// order by every CTA, so all CTAs take the same divergence / tolerance
// decision (solver.py:174-195) without another barrier.
#pragma once

#include <cooperative_groups.h>

#include "kernels.cuh"

namespace mrb {

namespace cg = cooperative_groups;

constexpr int kClusterThreads = 768;  // nodes per CTA (one per thread)
constexpr int kMaxDeg = 12;           // one-ring entries staged per node
// dynamic shared memory of the kernel: G coefficients + neighbour codes
constexpr size_t kClusterDynSmem =
    size_t(kMaxDeg) * kClusterThreads * (sizeof(float2) + sizeof(uint16_t));

struct ClusterPair {
  const double2* V;           // device-order vertices
  const uint16_t* codes;      // [kMaxDeg][n]: rank << 12 | local index
  const float2* g;            // [kMaxDeg][n]: fused gradient coefficients
  const float2* g_self;       // [n]
  const float* inv_val;       // [n]
  const unsigned char* deg;   // [n]
  const float* img;           // interleaved (Te, Re), H*W*2
  float2* u;                  // [n] final displacement (device order)
  double2* u_out;             // [n] reference order
  const int* perm;
  double* trace;
  int n, chunk, W, H;
};

// Sampling with the border path kept out of line (register pressure).
__device__ __noinline__ Px<float, float, 2> cr_sample_border(const float* img, int W, int H,
                                                             double x, double y) {
  return cr_sample<float, float, 2>(img, W, H, x, y);
}

__device__ __forceinline__ Px<float, float, 2> cr_sample_fast(const float* __restrict__ img,
                                                             int W, int H, double x, double y) {
  const double xc = fmin(fmax(x, 0.0), double(W) - 1.0);
  const double yc = fmin(fmax(y, 0.0), double(H) - 1.0);
  const int cx = min(int(floor(xc)), W - 2);
  const int cy = min(int(floor(yc)), H - 2);
  if (!(cx >= 1 && cx <= W - 3 && cy >= 1 && cy <= H - 3)) return cr_sample_border(img, W, H, x, y);
  float wx[4], wy[4];
  cr_weights<float>(float(xc - double(cx)), wx);
  cr_weights<float>(float(yc - double(cy)), wy);
  const float2* base = reinterpret_cast<const float2*>(img) + (size_t(cy - 1) * W + (cx - 1));
  Px<float, float, 2> acc;
  acc.v[0] = acc.v[1] = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2* row = base + size_t(j) * W;
    const float2 t0 = __ldg(row), t1 = __ldg(row + 1), t2 = __ldg(row + 2), t3 = __ldg(row + 3);
    float rt = wx[0] * t0.x;
    rt = fmaf(wx[1], t1.x, rt);
    rt = fmaf(wx[2], t2.x, rt);
    rt = fmaf(wx[3], t3.x, rt);
    float rr = wx[0] * t0.y;
    rr = fmaf(wx[1], t1.y, rr);
    rr = fmaf(wx[2], t2.y, rr);
    rr = fmaf(wx[3], t3.y, rr);
    acc.v[0] = fmaf(wy[j], rt, acc.v[0]);
    acc.v[1] = fmaf(wy[j], rr, acc.v[1]);
  }
  return acc;
}

__device__ __forceinline__ void cluster_sync_all() {
  // barrier.cluster.arrive.release + wait.acquire (orders DSMEM traffic)
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <int CS>
__global__ void __launch_bounds__(kClusterThreads, 1)
    k_cluster_register(const ClusterPair* __restrict__ pairs, PairStatus* __restrict__ st,
                       int max_iter, double tol, float tau, float lam, int passes) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = int(cluster.block_rank());
  const int p = blockIdx.x / CS;
  const ClusterPair& d = pairs[p];
  const int t = threadIdx.x;
  const int i = rank * d.chunk + t;
  const bool own = (t < d.chunk) && (i < d.n);

  __shared__ float s_ste[kClusterThreads];
  __shared__ float2 s_u0[kClusterThreads];
  __shared__ float2 s_u1[kClusterThreads];
  __shared__ double s_part;     // this CTA's energy partial
  __shared__ int s_gradbad;     // non-finite gradient seen in this CTA
  __shared__ double s_warp[kClusterThreads / 32];
  __shared__ int s_ctl[2];      // [0] = stop after this iteration, [1] = error
  // descent control state (thread 0 only; identical in every CTA)
  __shared__ double s_hist[6];
  __shared__ double s_prev;
  __shared__ int s_cs[4];       // rises, iters, err, err_iter
  __shared__ const float* s_rste[CS];
  __shared__ const float2* s_ru0[CS];
  __shared__ const float2* s_ru1[CS];
  extern __shared__ __align__(16) unsigned char s_dyn[];
  float2* s_g = reinterpret_cast<float2*>(s_dyn);                          // [e][t]
  uint16_t* s_code = reinterpret_cast<uint16_t*>(s_g + kMaxDeg * kClusterThreads);  // [e][t]

  if (t < CS) {
    s_rste[t] = cluster.map_shared_rank(s_ste, t);
    s_ru0[t] = cluster.map_shared_rank(s_u0, t);
    s_ru1[t] = cluster.map_shared_rank(s_u1, t);
  }
  if (t == 0) {
    s_gradbad = 0;
    s_prev = 0.0;
    s_cs[0] = s_cs[1] = s_cs[2] = s_cs[3] = 0;
  }

  // ---- node state into registers, one-ring topology into shared memory
  double2 V = make_double2(0.0, 0.0);
  float2 gs = make_float2(0.f, 0.f);
  float iv = 0.f;
  int deg = 0;
  if (own) {
    V = d.V[i];
    gs = d.g_self[i];
    iv = d.inv_val[i];
    deg = d.deg[i];
    for (int e = 0; e < deg; ++e) {
      s_code[e * kClusterThreads + t] = d.codes[size_t(e) * d.n + i];
      s_g[e * kClusterThreads + t] = d.g[size_t(e) * d.n + i];
    }
  }
  float2 u = make_float2(0.f, 0.f);
  float r = 0.f;
  cluster_sync_all();  // remote smem pointers / flags initialised everywhere

  int k = 0;
  for (; k < max_iter; ++k) {
    // -------- phase A: sample Te, Re at V + u; residual; energy partial
    double e2 = 0.0;
    if (own) {
      const Px<float, float, 2> s = cr_sample_fast(d.img, d.W, d.H, V.x + double(u.x),
                                                   V.y + double(u.y));
      r = s.v[0] - s.v[1];
      s_ste[t] = s.v[0];
      e2 = double(r) * double(r);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e2 += __shfl_down_sync(0xffffffffu, e2, o);
    if ((t & 31) == 0) s_warp[t >> 5] = e2;
    __syncthreads();
    if (t == 0) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kClusterThreads / 32; ++w) s += s_warp[w];
      s_part = s;
    }
    cluster_sync_all();  // #1: s_ste and partials visible cluster-wide
    if (t < 32) {
      // fixed-order cluster reduction, identical in every CTA
      double v = 0.0;
      int gb = 0;
      if (t < CS) {
        v = *cluster.map_shared_rank(&s_part, t);
        gb = *cluster.map_shared_rank(&s_gradbad, t);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        v += __shfl_down_sync(0xffffffffu, v, o);
        gb |= __shfl_down_sync(0xffffffffu, gb, o);
      }
      if (t == 0) {
        int stop = 0;
        int rises = s_cs[0], err = s_cs[2];
        if (gb) {  // non-finite gradient in the previous step (solver.py:131-132)
          err = ERR_NONFINITE_GRAD;
          s_cs[3] = k - 1;
          stop = 1;
        } else {
          const double e = 0.5 * v;
          const double prev = s_prev;
          if (!isfinite(e)) {  // solver.py:176-177
            err = ERR_NONFINITE_ENERGY;
            s_cs[3] = k;
            stop = 1;
          } else {
            if (k > 0) {  // material_rise, solver.py:43-44,178-186
              const double thr = __dadd_rn(__dmul_rn(prev, 1.0 + 1e-4), 1e-12);
              if (e > thr) {
                if (++rises >= 10) {
                  err = ERR_RISES;
                  s_cs[3] = k;
                  stop = 1;
                }
              } else if (e <= prev) {
                rises = 0;
              }
            }
            if (!stop) {
              s_cs[1] = k + 1;
              s_hist[k % 6] = e;
              if (k + 1 >= 6) {  // solver.py:192-195; trace[-6] == hist[(k+1)%6]
                const double base = s_hist[(k + 1) % 6];
                if (fabs(__dsub_rn(e, base)) <= __dmul_rn(tol, fmax(fabs(base), 1e-12)))
                  stop = 2;  // take this step, then stop
              }
            }
          }
          if (rank == 0) d.trace[k] = e;
          s_prev = e;
        }
        s_cs[0] = rises;
        s_cs[2] = err;
        s_ctl[0] = stop;
      }
    }
    __syncthreads();
    const int stop = s_ctl[0];
    if (stop == 1) break;

    // -------- phase B: gradient via the fused one-ring operator, descent
    bool bad = false;
    if (own) {
      const float si = s_ste[t];
      float gx = gs.x * si, gy = gs.y * si;
      for (int e = 0; e < deg; ++e) {
        const uint32_t c = s_code[e * kClusterThreads + t];
        const float2 ge = s_g[e * kClusterThreads + t];
        const float sj = s_rste[c >> 12][c & 0xfff];
        gx = fmaf(ge.x, sj, gx);
        gy = fmaf(ge.y, sj, gy);
      }
      const float dx = r * gx, dy = r * gy;
      bad = !isfinite(dx) || !isfinite(dy);
      s_u0[t] = make_float2(u.x - tau * dx, u.y - tau * dy);
    }
    if (__syncthreads_or(bad) && t == 0) s_gradbad = 1;
    cluster_sync_all();  // #2: u0 visible cluster-wide

    // -------- phase C: umbrella smoothing passes + domain clamp
    if (passes == 0) {
      if (own) {
        const float2 v = s_u0[t];
        u.x = float(fmin(fmax(double(v.x), -V.x), (double(d.W) - 1.0) - V.x));
        u.y = float(fmin(fmax(double(v.y), -V.y), (double(d.H) - 1.0) - V.y));
      }
    }
    for (int q = 0; q < passes; ++q) {
      const float2* const* src = (q & 1) ? s_ru1 : s_ru0;
      float2 v = make_float2(0.f, 0.f);
      if (own) {
        float ax = 0.f, ay = 0.f;
        for (int e = 0; e < deg; ++e) {
          const uint32_t c = s_code[e * kClusterThreads + t];
          const float2 uj = src[c >> 12][c & 0xfff];
          ax = fmaf(iv, uj.x, ax);
          ay = fmaf(iv, uj.y, ay);
        }
        const float2 si = src[rank][t];
        const float om = 1.f - lam;
        v = make_float2(om * si.x + lam * ax, om * si.y + lam * ay);
      }
      if (q == passes - 1) {
        if (own) {
          u.x = float(fmin(fmax(double(v.x), -V.x), (double(d.W) - 1.0) - V.x));
          u.y = float(fmin(fmax(double(v.y), -V.y), (double(d.H) - 1.0) - V.y));
        }
      } else {
        if (own) ((q & 1) ? s_u0 : s_u1)[t] = v;
        cluster_sync_all();
      }
    }
    if (stop == 2) {
      ++k;
      break;
    }
  }
  // final gradient-finiteness check of the last step taken
  cluster_sync_all();
  if (t == 0 && s_cs[2] == ERR_NONE) {
    int gb = 0;
    for (int c = 0; c < CS; ++c) gb |= *cluster.map_shared_rank(&s_gradbad, c);
    if (gb) {
      s_cs[2] = ERR_NONFINITE_GRAD;
      s_cs[3] = k - 1;
    }
  }
  if (own) {
    d.u[i] = u;
    d.u_out[d.perm[i]] = make_double2(double(u.x), double(u.y));
  }
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
