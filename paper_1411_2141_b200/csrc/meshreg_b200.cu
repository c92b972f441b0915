// C ABI + launch orchestration of the B200 mesh-registration path.
// Public interface: include/meshreg_b200.h.  Device code: kernels.cuh.
//
// Environment hooks (tests and diagnostics only; none changes a result):
//   MESHREG_B200_PATH=cluster|grid|generic, MESHREG_B200_EXCHANGE=push|pull
//     force a loop path (cross-path parity tests);
//   MESHREG_B200_NO_TAIL, MESHREG_B200_NO_GROUPS  run the C4 job without the
//     latency-shape tail wave / as one launch (equivalence tests);
//   MESHREG_B200_DEBUG  host/device timeline on stderr;
//   MESHREG_B200_PROFILE_PHASES  per-phase clock64 stamps of the cluster
//     kernels (tools/phase_profile.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <type_traits>
#include <atomic>
#include <pthread.h>
#include <thread>
#include <tuple>
#include <mutex>
#include <chrono>
#include <climits>
#include <condition_variable>
#include <functional>
#include <vector>

#include "../../include/meshreg_b200.h"
#include "cluster.cuh"
#include "grid.cuh"
#include "push.cuh"
#include "cluster64.cuh"
#include "push64.cuh"
#include "pixel.cuh"
#include "kernels.cuh"
#include "meshbuild.cuh"
#include "mesh_host.h"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

using namespace mrb;

struct mrb_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  mrb_ctx* sub[2] = {nullptr, nullptr};  // pipeline streams of mrb_register_many
  // host staging buffers for uploads (grow): [0] meshes, [1] fast-path
  // topologies, so planning the topologies never waits for the mesh copies
  // pinned staging: [0] meshes, [1] topologies, [2] tail-shape topologies
  void* pinned[3] = {nullptr, nullptr, nullptr};
  size_t pinned_cap[3] = {0, 0, 0};
  cudaEvent_t stage_done[3] = {nullptr, nullptr, nullptr};  // last async copy out of pinned[i]
  cudaStream_t copy = nullptr;       // input copies of mrb_register_many
  cudaEvent_t copy_done = nullptr;
  cudaStream_t aux = nullptr;        // rasters of mrb_register_many (beside the run), lowest priority
  cudaStream_t aux_hi = nullptr;     // the same at the loop streams' priority (fill_idle off)
  // register_many without dense outputs: rasters and dense passes run at the
  // lowest priority in the SMs the loop kernels leave idle.  With dense
  // outputs requested they keep the loops' priority, so each group's dense
  // field is ready (and its D2H under way) while later groups compute.
  bool fill_idle = false;
  cudaEvent_t aux_ev = nullptr;
  unsigned long long* counts = nullptr;  // pinned uncovered-pixel counts
  size_t counts_cap = 0;
  // pinned arena for the small descriptor uploads of a batch creation: a
  // pageable cudaMemcpyAsync synchronises the stream first, a pinned one not
  unsigned char* arena = nullptr;
  size_t arena_cap = 0, arena_off = 0;
  cudaEvent_t arena_done = nullptr;
  bool arena_used = false;
  // device-side mesh setup (meshbuild.cuh): small pinned scratch for job
  // descriptors and stats, and the builds whose stats are not yet checked
  void* small_pin = nullptr;
  size_t small_cap = 0;
  cudaEvent_t small_ev = nullptr;
  std::vector<HostMesh*> build_pending;
  int* build_stats = nullptr;  // pinned, [mesh][4]
  size_t build_stats_cap = 0;
  cudaEvent_t build_ev = nullptr;
  cudaEvent_t build_in = nullptr;  // V / T of the pending build uploaded
  // Large per-call buffers of mrb_register_many kept on the context (its
  // batches on one context run in turn): a fresh stream-ordered allocation
  // of a few hundred MB maps new pool memory, ~1 ms of host time each.
  struct Kept {
    void* p = nullptr;
    size_t cap = 0;
  } kept[5];  // see KeptSlot
  // side streams of this context's batches (wave groups, tail wave, topology
  // copies): created once; a stream creation costs ~0.1 ms of host time
  cudaStream_t side[4] = {nullptr, nullptr, nullptr, nullptr};
};

enum KeptSlot { kKeptPad, kKeptDense, kKeptState, kKeptImages, kKeptVT };

struct mrb_mesh {
  HostMesh h;
  std::unique_ptr<Locator> locator;  // built on first mrb_mesh_locate
};

namespace mrb {

// Stream-ordered device memory from the pool allocator: allocations made
// inside an API call are ordered on that call's context stream (AllocScope),
// so building and tearing down batches costs no device synchronisation.
inline thread_local cudaStream_t t_alloc_stream = nullptr;

inline void dev_free(void* p, cudaStream_t s) {
  if (!p) return;
  if (s)
    cudaFreeAsync(p, s);
  else
    cudaFree(p);
}

struct AllocScope {
  cudaStream_t prev;
  explicit AllocScope(cudaStream_t s) : prev(t_alloc_stream) { t_alloc_stream = s; }
  ~AllocScope() { t_alloc_stream = prev; }
};

struct DeviceMesh {
  int device = -1;
  cudaStream_t stream = nullptr;  // stream its memory is ordered on
  unsigned char* slab = nullptr;
  std::shared_ptr<unsigned char> slab_hold;  // set when `slab` is a slice of a shared upload
  unsigned char* slab64 = nullptr;
  std::shared_ptr<unsigned char> slab64_hold;  // set when slab64 is a shared upload's slice
  unsigned char* slab_ring = nullptr;
  double2* V = nullptr;
  int* nb_ptr = nullptr;
  int* nb_idx = nullptr;
  int4* tri = nullptr;
  int* perm = nullptr;
  float2* g_self_f = nullptr;
  float2* g_nb_f = nullptr;
  float* inv_val_f = nullptr;
  double2* g_self_d = nullptr;
  double2* g_nb_d = nullptr;
  double* inv_val_d = nullptr;
  // device-built meshes (meshbuild.cuh): the one-ring CSR in device ids and
  // the fp64 fused operator, kept for topology builds of any cluster shape
  const int* b_nb_ptr = nullptr;
  const int* b_nb_idx = nullptr;
  const double2* b_g_nb = nullptr;
  std::shared_ptr<unsigned char> build_hold;
  std::map<std::pair<int, int>, int*> pixel_maps;
  // owners of pixel maps that are slices of a batch's shared slab
  std::map<std::pair<int, int>, std::shared_ptr<unsigned char>> pixel_map_hold;
  // cluster fast path: register topology packed for a given chunk size
  struct Topo {  // SELL-32 one-ring layout for one (cluster size, nodes/thread)
    unsigned char* slab = nullptr;  // every array below lives in it
    std::shared_ptr<unsigned char> hold;  // owner when the slab is a shared upload's slice
    uint16_t* codes = nullptr;
    float2* g = nullptr;
    double2* g64 = nullptr;  // fp64 coefficients (k_cluster64 topologies)
    uint32_t* slice_off = nullptr;
    uint32_t* halo = nullptr;
    int* n_halo = nullptr;
    unsigned char* deg = nullptr;
    uint32_t* send = nullptr;
    int* n_send = nullptr;
    int chunk = 0, topo_stride = 0, slices = 0, halo_stride = 0, send_stride = 0;
  };
  std::map<int64_t, Topo> topo;  // key: topo_key(cluster size, chunk, nodes/thread, fp64)
  int max_deg = 0;
  ~DeviceMesh() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (device >= 0) cudaSetDevice(device);
    if (slab_hold)  // every per-mesh array lives in the slabs
      slab_hold.reset();
    else
      dev_free(slab, stream);
    if (slab64_hold)
      slab64_hold.reset();
    else
      dev_free(slab64, stream);
    dev_free(slab_ring, stream);
    build_hold.reset();
    for (auto& kv : pixel_maps)
      if (!pixel_map_hold.count(kv.first)) dev_free(kv.second, stream);
    pixel_map_hold.clear();
    for (auto& kv : topo) {
      if (kv.second.hold)
        kv.second.hold.reset();
      else
        dev_free(kv.second.slab, stream);
    }
    if (cur >= 0) cudaSetDevice(cur);
  }
};

HostMesh::~HostMesh() = default;

}  // namespace mrb

namespace {

const char* kVersion = "meshreg_b200 0.1.0 (sm_100a)";

inline size_t al256(size_t b) { return (b + 255) / 256 * 256; }

struct CudaError {
  cudaError_t e;
  int line = 0;  // source line of the failing call (reported under MESHREG_B200_DEBUG)
};

inline void ck_at(cudaError_t e, int line) {
  if (e != cudaSuccess) throw CudaError{e, line};
}
#define ck(e) ck_at((e), __LINE__)

// host<->device bytes moved by the library (reported by the benchmark)
std::atomic<long long> g_h2d_bytes{0}, g_d2h_bytes{0};

inline void count_copy(size_t bytes, cudaMemcpyKind kind) {
  if (kind == cudaMemcpyHostToDevice) g_h2d_bytes += (long long)bytes;
  if (kind == cudaMemcpyDeviceToHost) g_d2h_bytes += (long long)bytes;
}

inline cudaError_t mrb_copy_async(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind,
                                  cudaStream_t s) {
  count_copy(bytes, kind);
  return cudaMemcpyAsync(dst, src, bytes, kind, s);
}

inline cudaError_t mrb_copy2d_async(void* dst, size_t dpitch, const void* src, size_t spitch,
                                    size_t width, size_t height, cudaMemcpyKind kind,
                                    cudaStream_t s) {
  count_copy(width * height, kind);
  return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, kind, s);
}

inline cudaError_t mrb_copy(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
  count_copy(bytes, kind);
  return cudaMemcpy(dst, src, bytes, kind);
}

template <typename T>
T* dalloc(size_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  if (t_alloc_stream)
    ck(cudaMallocAsync(&p, n * sizeof(T), t_alloc_stream));
  else
    ck(cudaMalloc(&p, n * sizeof(T)));
  return static_cast<T*>(p);
}

// side stream `which` of the context (0 wave groups, 1 tail wave, 2 copies)
// Stream priorities: the streams the persistent loop kernels (and the device
// mesh setup ahead of them) run on get the highest priority; the rasters'
// stream (ctx->aux) and the dense passes' stream (side 3) stay at the
// default, lowest one.  The setup rasters and the dense passes of earlier
// wave groups then fill the SMs the loop kernels leave idle (13 of 148 during
// a C4 wave, 84 during the tail wave) instead of holding back a cluster
// launch, which needs whole SMs: C4 e2e 9.40 -> 9.15 ms.
cudaError_t create_stream(cudaStream_t* s, bool high) {
  if (!high) return cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
  int least = 0, greatest = 0;
  cudaDeviceGetStreamPriorityRange(&least, &greatest);
  return cudaStreamCreateWithPriority(s, cudaStreamNonBlocking, greatest);
}
cudaStream_t side_stream(mrb_ctx* ctx, int which) {  // 3: the dense passes' stream (low)
  if (!ctx->side[which]) ck(create_stream(&ctx->side[which], which != 3));
  return ctx->side[which];
}

// A kept buffer of the context (grows; stream-ordered on ctx->stream, or
// the AllocScope's stream)
void* kept_buffer(mrb_ctx* ctx, int slot, size_t bytes) {
  mrb_ctx::Kept& k = ctx->kept[slot];
  if (k.cap < bytes) {
    dev_free(k.p, ctx->stream);
    k.p = dalloc<unsigned char>(bytes);
    k.cap = bytes;
  }
  return k.p;
}

// One device allocation shared by the meshes of an upload (freed, stream
// ordered, with the last mesh that uses it).
std::shared_ptr<unsigned char> shared_slab(size_t bytes, cudaStream_t s) {
  unsigned char* p = dalloc<unsigned char>(bytes);
  return std::shared_ptr<unsigned char>(p, [s](unsigned char* q) { dev_free(q, s); });
}

// Descriptor arena (mrb_ctx::arena): arena_begin waits until the previous
// creation's copies left the arena, then hands out slices (each upload
// records arena_done after its copy).
void arena_begin(mrb_ctx* ctx, size_t need) {
  if (ctx->arena_used) ck(cudaEventSynchronize(ctx->arena_done));
  ctx->arena_used = false;
  ctx->arena_off = 0;
  if (need > ctx->arena_cap) {
    if (ctx->arena) cudaFreeHost(ctx->arena);
    ctx->arena = nullptr;
    ctx->arena_cap = 0;
    const size_t cap = std::max<size_t>(need + need / 2, size_t(1) << 20);
    ck(cudaHostAlloc(reinterpret_cast<void**>(&ctx->arena), cap, cudaHostAllocMapped));
    ctx->arena_cap = cap;
  }
  if (!ctx->arena_done) ck(cudaEventCreateWithFlags(&ctx->arena_done, cudaEventDisableTiming));
}

template <typename T>
T* dupload(const T* h, size_t n, cudaStream_t s);

// Zero-copy read of pinned host memory by a kernel: the descriptor uploads
// of a batch are small, and as DMA copies they would queue behind the bulk
// image / mesh copies of mrb_register_many on the copy engine.
__global__ void k_copy_from_host(unsigned char* __restrict__ dst,
                                 const unsigned char* __restrict__ src, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n / 16;
       i += size_t(gridDim.x) * blockDim.x)
    reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
  const size_t tail = n & ~size_t(15);
  if (blockIdx.x == 0 && threadIdx.x < n - tail) dst[tail + threadIdx.x] = src[tail + threadIdx.x];
}

// device copy of h[0..n) through the arena (pageable fallback when full)
template <typename T>
T* aupload(mrb_ctx* ctx, const T* h, size_t n) {
  const size_t bytes = n * sizeof(T), at = (ctx->arena_off + 255) / 256 * 256;
  if (!ctx->arena || at + bytes > ctx->arena_cap) return dupload(h, n, ctx->stream);
  std::memcpy(ctx->arena + at, h, bytes);
  ctx->arena_off = at + bytes;
  T* d = dalloc<T>(n);  // 256-byte aligned, as is the arena slice
  if (n) {
    unsigned char* src = nullptr;
    ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&src), ctx->arena + at, 0));
    const unsigned blocks = unsigned(std::min<size_t>((bytes / 16 + 255) / 256 + 1, 64));
    k_copy_from_host<<<blocks, 256, 0, ctx->stream>>>(reinterpret_cast<unsigned char*>(d), src,
                                                     bytes);
    ck(cudaGetLastError());
  }
  ck(cudaEventRecord(ctx->arena_done, ctx->stream));  // arena slice free after this
  ctx->arena_used = true;
  return d;
}

template <typename T>
T* dupload(const T* h, size_t n, cudaStream_t s) {
  T* d = dalloc<T>(n);
  if (n) ck(mrb_copy_async(d, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
  return d;
}

// Scoped stream-ordered temporaries for the single-operation entry points.
struct Tmp {
  cudaStream_t s;
  std::vector<void*> ptrs;
  explicit Tmp(cudaStream_t st) : s(st) {}
  template <typename T>
  T* get(size_t n) {
    void* p = nullptr;
    ck(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), s));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  template <typename T>
  T* up(const T* h, size_t n) {
    T* d = get<T>(n);
    if (n) ck(mrb_copy_async(d, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
    return d;
  }
  ~Tmp() {
    for (void* p : ptrs) cudaFreeAsync(p, s);
  }
};

int fail(mrb_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

int cuda_fail(mrb_ctx* ctx, cudaError_t e, int line = 0) {
  if (line && std::getenv("MESHREG_B200_DEBUG"))
    std::fprintf(stderr, "meshreg_b200: CUDA error %s at meshreg_b200.cu:%d\n",
                 cudaGetErrorString(e), line);
  return fail(ctx, MRB_E_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e));
}

// Python float repr (shortest round-trip digits; fixed for 1e-4 <= |x| < 1e16)
std::string py_repr(double v) {
  if (std::isnan(v)) return "nan";
  if (std::isinf(v)) return v > 0 ? "inf" : "-inf";
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  char buf[64];
  int prec = 1;
  for (; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*e", prec - 1, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  // buf = [-]d.ddde[+-]XX
  std::string s(buf);
  const bool neg = s[0] == '-';
  if (neg) s = s.substr(1);
  const size_t epos = s.find('e');
  std::string mant = s.substr(0, epos);
  const int exp10 = std::atoi(s.c_str() + epos + 1);
  std::string digits;
  for (char c : mant)
    if (c != '.') digits += c;
  while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
  std::string out;
  if (exp10 >= -5 && exp10 < 16) {
    const int decpt = exp10 + 1;  // digits before the point
    if (decpt <= 0) {
      out = "0." + std::string(-decpt, '0') + digits;
    } else if (decpt >= int(digits.size())) {
      out = digits + std::string(decpt - digits.size(), '0') + ".0";
    } else {
      out = digits.substr(0, decpt) + "." + digits.substr(decpt);
    }
    if (exp10 == -5) {  // Python switches to exponent below 1e-4
      out.clear();
    }
  }
  if (out.empty()) {
    out = digits.substr(0, 1);
    if (digits.size() > 1) out += "." + digits.substr(1);
    char e[16];
    std::snprintf(e, sizeof e, "e%c%02d", exp10 < 0 ? '-' : '+', std::abs(exp10));
    out += e;
  }
  return neg ? "-" + out : out;
}

// Host staging memory owned by the context (pinned, grows, reused once the
// previous copy out of it has completed).
void* pinned_stage(mrb_ctx* ctx, size_t bytes, int which) {
  if (ctx->stage_done[which]) ck(cudaEventSynchronize(ctx->stage_done[which]));
  if (bytes > ctx->pinned_cap[which]) {
    if (ctx->pinned[which]) cudaFreeHost(ctx->pinned[which]);
    ctx->pinned[which] = nullptr;
    ctx->pinned_cap[which] = 0;
    const size_t cap = std::max<size_t>(bytes + bytes / 4, size_t(16) << 20);
    ck(cudaHostAlloc(&ctx->pinned[which], cap, cudaHostAllocDefault));
    ctx->pinned_cap[which] = cap;
  }
  return ctx->pinned[which];
}

// Persistent host worker pool: parallel_for(n, f) runs f(0..n-1) on up to 16
// threads (the caller participates).  Thread start-up is paid once per
// process, not per call — batch setup calls it several times per chunk.
// The pool is never destroyed (its threads end with the process), and a
// forked child, which inherits no threads, runs everything on the caller.
class WorkerPool {
 public:
  static WorkerPool& get() {
    static WorkerPool* pool = new WorkerPool();
    return *pool;
  }
  template <typename F>
  void run(size_t n, F&& f) {
    if (n == 0) return;
    if (workers_.empty() || n == 1 || forked_) {
      for (size_t i = 0; i < n; ++i) f(i);
      return;
    }
    std::unique_lock<std::mutex> job_lock(job_mu_);  // one parallel_for at a time
    std::function<void(size_t)> fn = std::forward<F>(f);
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      n_ = n;
      next_ = 0;
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return done_ == n_; });
    fn_ = nullptr;
  }

 private:
  WorkerPool() {
    pthread_atfork(nullptr, nullptr, [] { get().forked_ = true; });
    const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency())) - 1;
    for (unsigned k = 0; k < nt; ++k)
      workers_.emplace_back([this] {
        size_t seen = 0;
        for (;;) {
          {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
          }
          work();
        }
      });
  }
  void work() {
    for (;;) {
      size_t i;
      std::function<void(size_t)>* fn;
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (!fn_ || next_ >= n_) return;
        i = next_++;
        fn = fn_;
      }
      (*fn)(i);
      std::lock_guard<std::mutex> lk(mu_);
      if (++done_ == n_) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, job_mu_;
  std::condition_variable cv_, done_cv_;
  std::function<void(size_t)>* fn_ = nullptr;
  size_t n_ = 0, next_ = 0, done_ = 0, gen_ = 0;
  bool stop_ = false;
  volatile bool forked_ = false;
};

template <typename F>
void parallel_for(size_t n, F&& f) {
  WorkerPool::get().run(n, std::forward<F>(f));
}

// MESHREG_B200_DEBUG: named device timestamps, printed (relative to the
// call's start) by mrb_register_many
std::vector<std::pair<std::string, cudaEvent_t>>& dev_marks() {
  static std::vector<std::pair<std::string, cudaEvent_t>> v;
  return v;
}
void dev_mark(cudaStream_t s, const char* what) {
  static const bool on = std::getenv("MESHREG_B200_DEBUG") != nullptr;
  if (!on) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, s);
  dev_marks().emplace_back(what, e);
}

// Upload the per-mesh device arrays of every mesh in `meshes` that has none
// yet.  Each mesh gets one device slab; the slabs are filled on a host thread
// pool into a context-owned pinned staging buffer and copied asynchronously.
// The fp64 operator arrays are uploaded only when an fp64 batch needs them
// (ensure_device_mesh_f64).
void ensure_device_meshes(mrb_ctx* ctx, const std::vector<HostMesh*>& meshes, bool with_ring) {
  std::vector<HostMesh*> todo;
  for (HostMesh* h : meshes)
    if (!(h->dev && h->dev->device == ctx->device) &&
        std::find(todo.begin(), todo.end(), h) == todo.end())
      todo.push_back(h);
  if (todo.empty()) return;
  parallel_for(todo.size(), [&](size_t i) { ensure_host(*todo[i]); });
  AllocScope scope(ctx->stream);
  const bool dbg = std::getenv("MESHREG_B200_DEBUG") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto tick = [&](const char* what) {
    if (!dbg) return;
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "meshreg_b200:   meshes %-18s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  struct Plan {
    size_t off[8], tot, base;
  };
  std::vector<Plan> plan(todo.size());
  size_t total = 0;
  for (size_t i = 0; i < todo.size(); ++i) {
    const HostMesh& h = *todo[i];
    const size_t n = size_t(h.n), m = size_t(h.m), ne2 = h.nb_idx.size();
    // 1, 2, 6: one-ring CSR + fused operator of the generic path (optional)
    const size_t r = with_ring ? 1 : 0;
    const size_t sizes[8] = {n * 16, r * (n + 1) * 4, r * ne2 * 4, m * 16, n * 4, n * 8,
                             r * ne2 * 8, n * 4};
    Plan& pl = plan[i];
    pl.tot = 0;
    for (int k = 0; k < 8; ++k) {
      pl.off[k] = pl.tot;
      pl.tot += (sizes[k] + 255) / 256 * 256;
    }
    pl.base = total;
    total += pl.tot;
  }
  unsigned char* stage = static_cast<unsigned char*>(pinned_stage(ctx, total, 0));
  tick("stage wait");
  auto fill = [&](size_t i) {
    const HostMesh& h = *todo[i];
    const Plan& pl = plan[i];
    unsigned char* dst = stage + pl.base;
    const size_t n = size_t(h.n), m = size_t(h.m), ne2 = h.nb_idx.size();
    std::memcpy(dst + pl.off[0], h.Vn.data(), n * 16);
    if (with_ring) {
      std::memcpy(dst + pl.off[1], h.nb_ptr.data(), (n + 1) * 4);
      std::memcpy(dst + pl.off[2], h.nb_idx.data(), ne2 * 4);
      float* gn = reinterpret_cast<float*>(dst + pl.off[6]);
      for (size_t k = 0; k < 2 * ne2; ++k) gn[k] = float(h.g_nb[k]);
    }
    std::memcpy(dst + pl.off[3], h.Tn.data(), m * 16);
    std::memcpy(dst + pl.off[4], h.perm.data(), n * 4);
    float* gs = reinterpret_cast<float*>(dst + pl.off[5]);
    for (size_t k = 0; k < 2 * n; ++k) gs[k] = float(h.g_self[k]);
    float* iv = reinterpret_cast<float*>(dst + pl.off[7]);
    for (size_t k = 0; k < n; ++k) iv[k] = float(h.inv_val[k]);
  };
  parallel_for(todo.size(), fill);
  tick("host fill");
  // one allocation and one large copy for every mesh of the upload (large
  // copies run at full PCIe rate, ~1 MB ones at less than half of it)
  const std::shared_ptr<unsigned char> all = shared_slab(total, ctx->stream);
  ck(mrb_copy_async(all.get(), stage, total, cudaMemcpyHostToDevice, ctx->stream));
  dev_mark(ctx->stream, "mesh upload done");
  for (size_t i = 0; i < todo.size(); ++i) {
    HostMesh& h = *todo[i];
    const Plan& pl = plan[i];
    h.dev.reset(new DeviceMesh());
    DeviceMesh& d = *h.dev;
    d.device = ctx->device;
    d.stream = ctx->stream;
    unsigned char* slab = all.get() + pl.base;
    d.slab = slab;
    d.slab_hold = all;
    d.V = reinterpret_cast<double2*>(slab + pl.off[0]);
    if (with_ring) {
      d.nb_ptr = reinterpret_cast<int*>(slab + pl.off[1]);
      d.nb_idx = reinterpret_cast<int*>(slab + pl.off[2]);
      d.g_nb_f = reinterpret_cast<float2*>(slab + pl.off[6]);
    }
    d.tri = reinterpret_cast<int4*>(slab + pl.off[3]);
    d.perm = reinterpret_cast<int*>(slab + pl.off[4]);
    d.g_self_f = reinterpret_cast<float2*>(slab + pl.off[5]);
    d.inv_val_f = reinterpret_cast<float*>(slab + pl.off[7]);
    d.max_deg = h.max_deg;
  }
  ck(cudaEventRecord(ctx->stage_done[0], ctx->stream));  // staging buffer reusable after this
  tick("copies issued");
}

// one-ring CSR + fp32 operator of the generic path, when a mesh was uploaded
// without them (cluster-path batches)
void ensure_device_mesh_ring(mrb_ctx* ctx, HostMesh& h) {
  DeviceMesh& d = *h.dev;
  if (d.nb_ptr) return;
  ensure_host(h);
  AllocScope scope(ctx->stream);
  const size_t n = size_t(h.n), ne2 = h.nb_idx.size();
  const size_t o1 = ((n + 1) * 4 + 255) / 256 * 256, o2 = o1 + (ne2 * 4 + 255) / 256 * 256;
  std::vector<unsigned char> host(o2 + ne2 * 8);
  std::memcpy(host.data(), h.nb_ptr.data(), (n + 1) * 4);
  std::memcpy(host.data() + o1, h.nb_idx.data(), ne2 * 4);
  float* gn = reinterpret_cast<float*>(host.data() + o2);
  for (size_t k = 0; k < 2 * ne2; ++k) gn[k] = float(h.g_nb[k]);
  d.slab_ring = dalloc<unsigned char>(host.size());
  ck(mrb_copy_async(d.slab_ring, host.data(), host.size(), cudaMemcpyHostToDevice, ctx->stream));
  d.nb_ptr = reinterpret_cast<int*>(d.slab_ring);
  d.nb_idx = reinterpret_cast<int*>(d.slab_ring + o1);
  d.g_nb_f = reinterpret_cast<float2*>(d.slab_ring + o2);
}

void ensure_device_mesh(mrb_ctx* ctx, HostMesh& h) {
  ensure_device_meshes(ctx, {&h}, true);
  ensure_device_mesh_ring(ctx, h);
}

// fp64 operator arrays, uploaded on first use by an fp64 batch / single op
void ensure_device_mesh_f64(mrb_ctx* ctx, HostMesh& h) {
  ensure_device_mesh(ctx, h);  // includes the one-ring arrays
  ensure_host(h);
  DeviceMesh& d = *h.dev;
  if (d.slab64 && d.g_nb_d) return;
  if (d.slab64_hold) d.slab64_hold.reset();  // the self-term-only slice
  else if (d.slab64) dev_free(d.slab64, ctx->stream);
  AllocScope scope(ctx->stream);
  const size_t n = size_t(h.n), ne2 = h.nb_idx.size();
  const size_t o1 = (n * 16 + 255) / 256 * 256, o2 = o1 + (ne2 * 16 + 255) / 256 * 256;
  std::vector<unsigned char> host(o2 + n * 8);
  std::memcpy(host.data(), h.g_self.data(), n * 16);
  std::memcpy(host.data() + o1, h.g_nb.data(), ne2 * 16);
  std::memcpy(host.data() + o2, h.inv_val.data(), n * 8);
  d.slab64 = dalloc<unsigned char>(host.size());
  ck(mrb_copy_async(d.slab64, host.data(), host.size(), cudaMemcpyHostToDevice, ctx->stream));
  d.g_self_d = reinterpret_cast<double2*>(d.slab64);
  d.g_nb_d = reinterpret_cast<double2*>(d.slab64 + o1);
  d.inv_val_d = reinterpret_cast<double*>(d.slab64 + o2);
}

// fp64 self terms and 1/valence only (what k_cluster64 reads besides its
// topology), for many meshes: one pinned-staged copy
void ensure_device_meshes_f64_self(mrb_ctx* ctx, const std::vector<HostMesh*>& meshes) {
  std::vector<HostMesh*> todo;
  for (HostMesh* h : meshes)
    if (!h->dev->g_self_d && std::find(todo.begin(), todo.end(), h) == todo.end())
      todo.push_back(h);
  if (todo.empty()) return;
  parallel_for(todo.size(), [&](size_t i) { ensure_host(*todo[i]); });
  std::vector<size_t> base(todo.size());
  size_t total = 0;
  for (size_t i = 0; i < todo.size(); ++i) {
    base[i] = total;
    total += (size_t(todo[i]->n) * 16 + 255) / 256 * 256 + (size_t(todo[i]->n) * 8 + 255) / 256 * 256;
  }
  unsigned char* stage = static_cast<unsigned char*>(pinned_stage(ctx, total, 0));
  parallel_for(todo.size(), [&](size_t i) {
    const HostMesh& h = *todo[i];
    const size_t n = size_t(h.n), o = (n * 16 + 255) / 256 * 256;
    std::memcpy(stage + base[i], h.g_self.data(), n * 16);
    std::memcpy(stage + base[i] + o, h.inv_val.data(), n * 8);
  });
  AllocScope scope(ctx->stream);
  const std::shared_ptr<unsigned char> all = shared_slab(total, ctx->stream);
  ck(mrb_copy_async(all.get(), stage, total, cudaMemcpyHostToDevice, ctx->stream));
  ck(cudaEventRecord(ctx->stage_done[0], ctx->stream));
  for (size_t i = 0; i < todo.size(); ++i) {
    DeviceMesh& d = *todo[i]->dev;
    const size_t o = (size_t(todo[i]->n) * 16 + 255) / 256 * 256;
    d.slab64 = all.get() + base[i];
    d.slab64_hold = all;
    d.g_self_d = reinterpret_cast<double2*>(d.slab64);
    d.inv_val_d = reinterpret_cast<double*>(d.slab64 + o);
  }
}

// Shared-memory topology of the cluster kernel for `cs` CTAs of `chunk` nodes
// and `npt` slots per thread:
//  * SELL-32 one-rings — for every 32-slot slice of a CTA's chunk, entry e of
//    slot s sits at slice_off[slice] + 32 e + s % 32, padded to the slice's
//    largest one-ring; every CTA block is padded to the same stride;
//  * codes are CTA-local indices into [own slots (SLOTS = 768*npt) | halo];
//  * halo[r] lists (owner rank << 16 | owner slot) of every remote node CTA r's
//    one-rings reference, in first-reference order.
// Host plan of one fast-path topology (cluster of cs CTAs, `chunk` nodes per
// CTA): SELL-32 slice offsets, halo lists and the code of every one-ring
// entry.  write_topo() then packs it straight into (pinned) memory.
// A topology's arrays depend on the cluster size as well as the chunk (two
// sizes can give the same chunk for a small mesh), so both are in the key.
inline int64_t topo_key(int cs, int chunk, int npt, bool f64 = false) {
  return (int64_t(cs) << 40) | (int64_t(chunk) << 8) | (int64_t(npt) << 1) | int64_t(f64);
}

struct TopoHost {
  int cs = 0;
  int chunk = 0, stride = 0, slices = 0, hstride = 0, sstride = 0;
  size_t off[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  size_t total = 0;                  // packed bytes
  std::vector<uint32_t> soff;        // [cs][slices]
  std::vector<uint32_t> halo;        // [cs][hstride]
  std::vector<int> n_halo;           // [cs]
  std::vector<uint16_t> code;        // per one-ring entry (CSR order)
  // push exchange (cluster kernel): what CTA r sends where, the inverse of the
  // halo lists: slot << 20 | dst CTA << 16 | dst halo index
  std::vector<uint32_t> send;        // [cs][sstride]
  std::vector<int> n_send;           // [cs]
};

// gbytes: bytes per SELL coefficient entry (float2 8, double2 16 for k_cluster64)
TopoHost plan_topo(const HostMesh& h, int cs, int chunk, int npt, int gbytes = 8) {
  ensure_host(const_cast<HostMesh&>(h));  // deferred handles: host arrays first
  const int n = int(h.n);
  const int SLOTS = kClusterThreads * npt;
  TopoHost t;
  t.cs = cs;
  t.chunk = chunk;
  t.slices = (chunk + 31) / 32;
  t.soff.assign(size_t(cs) * t.slices, 0);
  t.code.resize(size_t(h.nb_ptr[n]));
  std::vector<std::vector<uint32_t>> halos(cs);
  std::vector<int> stamp(static_cast<size_t>(n), -1), hidx(static_cast<size_t>(n), 0);
  int stride = 0;
  for (int r = 0; r < cs; ++r) {
    int acc = 0;  // pair rows x 32 so far in this CTA's block
    for (int sl = 0; sl < t.slices; ++sl) {
      const size_t si = size_t(r) * t.slices + sl;
      int mx = 0;
      for (int s = sl * 32; s < std::min(chunk, sl * 32 + 32); ++s) {
        const int i = r * chunk + s;
        if (i >= n) break;
        mx = std::max(mx, h.nb_ptr[i + 1] - h.nb_ptr[i]);
        for (int q = h.nb_ptr[i]; q < h.nb_ptr[i + 1]; ++q) {
          const int j = h.nb_idx[q];
          const int rj = j / chunk;
          if (rj == r) {
            t.code[q] = uint16_t(j - rj * chunk);
            continue;
          }
          if (stamp[j] != r) {  // first reference of remote node j by CTA r
            stamp[j] = r;
            hidx[j] = int(halos[r].size());
            halos[r].push_back(uint32_t(rj << 16 | (j - rj * chunk)));
          }
          t.code[q] = uint16_t(SLOTS + hidx[j]);
        }
      }
      const int pairs = (mx + 1) / 2;  // warp-uniform trip count of the gathers
      t.soff[si] = uint32_t(pairs) << 24 | uint32_t(acc);
      acc += 32 * pairs;
    }
    stride = std::max(stride, 2 * acc);  // entries (uint16 codes / float2 coefficients)
  }
  t.stride = std::max((stride + 7) / 8 * 8, 8);
  // halo slots, plus one: the last slot of the halo region is the ZERO slot
  // (always 0) every padding entry of the SELL layout points at
  int hstride = 2;
  for (auto& hl : halos) hstride = std::max<int>(hstride, int(hl.size()) + 1);
  t.hstride = (hstride + 31) / 32 * 32;
  t.halo.assign(size_t(cs) * t.hstride, 0);
  t.n_halo.resize(cs);
  for (int r = 0; r < cs; ++r) {
    t.n_halo[r] = int(halos[r].size());
    std::copy(halos[r].begin(), halos[r].end(), t.halo.begin() + size_t(r) * t.hstride);
  }
  t.n_send.assign(cs, 0);
  if (cs <= 16 && SLOTS <= 4096) {  // cluster shapes only
    std::vector<std::vector<uint32_t>> sends(cs);
    for (int c = 0; c < cs; ++c)
      for (size_t hh = 0; hh < halos[c].size(); ++hh) {
        const uint32_t e = halos[c][hh];
        sends[e >> 16].push_back((e & 0xffffu) << 20 | uint32_t(c) << 16 | uint32_t(hh));
      }
    int ss = 2;
    for (auto& v : sends) ss = std::max<int>(ss, int(v.size()));
    t.sstride = (ss + 31) / 32 * 32;
    t.send.assign(size_t(cs) * t.sstride, 0);
    for (int r = 0; r < cs; ++r) {
      t.n_send[r] = int(sends[r].size());
      std::copy(sends[r].begin(), sends[r].end(), t.send.begin() + size_t(r) * t.sstride);
    }
  }
  const size_t bytes[8] = {size_t(cs) * t.stride * 2, size_t(cs) * t.stride * gbytes,
                           t.soff.size() * 4, t.halo.size() * 4, size_t(cs) * 4, size_t(n),
                           t.send.size() * 4, size_t(cs) * 4};
  for (int k = 0; k < 8; ++k) {
    t.off[k] = t.total;
    t.total += (bytes[k] + 255) / 256 * 256;
  }
  return t;
}

// packed layout: codes | g | slice_off | halo | n_halo | deg | send | n_send
//
// Paired SELL-32: the one-ring entries of a 32-slot slice (one warp) are
// stored in pair rows; entry e of slot s sits at entry index
//   2 * (pair_off(slice) + 32 * (e / 2) + s % 32) + e % 2
// so one 32-bit load fetches the codes of entries (2p, 2p+1) and one 128-bit
// load their two coefficient pairs.  slice_off = pair rows << 24 | pair_off;
// the pair-row count is the slice's largest one-ring, rounded up, so every
// gather loop is warp-uniform.  Padding entries point at the ZERO slot
// (halo_stride - 1 past the own slots) with coefficient 0.
inline uint16_t zero_slot(int npt, int hstride) {
  return uint16_t(kClusterThreads * npt + hstride - 1);
}

void write_topo(const HostMesh& h, int cs, const TopoHost& t, unsigned char* dst, int npt,
                bool f64 = false) {
  const int n = int(h.n), chunk = t.chunk;
  uint16_t* codes = reinterpret_cast<uint16_t*>(dst + t.off[0]);
  float2* g = reinterpret_cast<float2*>(dst + t.off[1]);
  double2* g64 = reinterpret_cast<double2*>(dst + t.off[1]);
  std::fill(codes, codes + size_t(cs) * t.stride, zero_slot(npt, t.hstride));
  std::memset(g, 0, size_t(cs) * t.stride * (f64 ? 16 : 8));
  unsigned char* deg = dst + t.off[5];
  for (int i = 0; i < n; ++i) {
    const int r = i / chunk, s = i - r * chunk;
    const int b = h.nb_ptr[i], e = h.nb_ptr[i + 1];
    deg[i] = (unsigned char)(e - b);
    const size_t base =
        size_t(r) * t.stride + 2 * size_t((t.soff[size_t(r) * t.slices + s / 32] & 0xffffffu) + (s % 32));
    for (int q = b; q < e; ++q) {
      const int k = q - b;
      const size_t at = base + 64 * size_t(k >> 1) + (k & 1);
      codes[at] = t.code[q];
      if (f64)
        g64[at] = make_double2(h.g_nb[2 * q], h.g_nb[2 * q + 1]);
      else
        g[at] = make_float2(float(h.g_nb[2 * q]), float(h.g_nb[2 * q + 1]));
    }
  }
  std::memcpy(dst + t.off[2], t.soff.data(), t.soff.size() * 4);
  std::memcpy(dst + t.off[3], t.halo.data(), t.halo.size() * 4);
  std::memcpy(dst + t.off[4], t.n_halo.data(), t.n_halo.size() * 4);
  std::memcpy(dst + t.off[6], t.send.data(), t.send.size() * 4);
  std::memcpy(dst + t.off[7], t.n_send.data(), t.n_send.size() * 4);
}

// device arrays of a packed topology, carved out of one slab
// f64: a k_cluster64 topology (double2 coefficients, its own cache key)
DeviceMesh::Topo& install_topo(HostMesh& h, int npt, const TopoHost& th,
                                     unsigned char* slab, bool f64 = false) {
  DeviceMesh::Topo t;
  t.chunk = th.chunk;
  t.topo_stride = th.stride;
  t.slices = th.slices;
  t.halo_stride = th.hstride;
  t.slab = slab;
  t.codes = reinterpret_cast<uint16_t*>(slab + th.off[0]);
  t.g = reinterpret_cast<float2*>(slab + th.off[1]);
  t.slice_off = reinterpret_cast<uint32_t*>(slab + th.off[2]);
  t.halo = reinterpret_cast<uint32_t*>(slab + th.off[3]);
  t.n_halo = reinterpret_cast<int*>(slab + th.off[4]);
  t.deg = slab + th.off[5];
  t.send = reinterpret_cast<uint32_t*>(slab + th.off[6]);
  t.n_send = reinterpret_cast<int*>(slab + th.off[7]);
  t.send_stride = th.sstride;
  if (f64) {
    t.g64 = reinterpret_cast<double2*>(t.g);
    t.g = nullptr;
    return h.dev->topo[topo_key(th.cs, th.chunk, 1, true)] = t;
  }
  return h.dev->topo[topo_key(th.cs, th.chunk, npt)] = t;
}

// ---- device-side mesh setup (deferred handles, meshbuild.cuh) --------------
//
// Deferred handles (mrb_mesh_create_many) carry only V and the oriented T.
// device_build_meshes stages them through pinned memory, copies them on the
// given stream and runs the connectivity / geometry / node-order / fused
// operator build on ctx->stream; device_cluster_topos plans and writes the
// fast-path topology of any cluster shape on the GPU.  Both produce the bytes
// the host build (build_mesh, plan_topo + write_topo) produces.

// Process-wide cache of host blocks for deferred mesh handles: pinned when
// the driver allows it (else plain memory, e.g. without a GPU), recycled when
// the last mesh of a creation is destroyed.
struct BlockCache {
  std::mutex mu;
  std::multimap<size_t, std::pair<void*, bool>> free;  // size -> (ptr, pinned)
  size_t cached = 0;
  static BlockCache& get() {
    static BlockCache* c = new BlockCache();
    return *c;
  }
};

std::shared_ptr<unsigned char> pinned_block(size_t bytes) {
  BlockCache& c = BlockCache::get();
  void* p = nullptr;
  bool pinned = false;
  size_t size = bytes;
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.free.lower_bound(bytes);
    if (it != c.free.end() && it->first <= 2 * bytes) {
      size = it->first;
      p = it->second.first;
      pinned = it->second.second;
      c.cached -= size;
      c.free.erase(it);
    }
  }
  if (!p) {
    size = al256(bytes);
    pinned = cudaHostAlloc(&p, size, cudaHostAllocDefault) == cudaSuccess;
    if (!pinned) {
      cudaGetLastError();  // no device: plain host memory
      p = std::malloc(size);
      if (!p) throw std::bad_alloc();
    }
  }
  return std::shared_ptr<unsigned char>(static_cast<unsigned char*>(p), [size, pinned](unsigned char* q) {
    BlockCache& cc = BlockCache::get();
    std::lock_guard<std::mutex> lk(cc.mu);
    if (cc.cached + size <= (size_t(1) << 30)) {
      cc.free.emplace(size, std::make_pair(static_cast<void*>(q), pinned));
      cc.cached += size;
    } else if (pinned) {
      cudaFreeHost(q);
    } else {
      std::free(q);
    }
  });
}

// MESHREG_B200_DEBUG: host time since the previous call (what: label)
void host_tick(const char* what) {
  static const bool on = std::getenv("MESHREG_B200_DEBUG") != nullptr;
  if (!on) return;
  static thread_local auto last = std::chrono::steady_clock::now();
  const auto now = std::chrono::steady_clock::now();
  std::fprintf(stderr, "meshreg_b200:     host %-28s %8.3f ms\n", what,
               std::chrono::duration<double, std::milli>(now - last).count());
  last = now;
}

// pinned scratch for descriptors and stats (the previous use must be done)
unsigned char* small_pinned(mrb_ctx* ctx, size_t bytes) {
  if (ctx->small_ev) ck(cudaEventSynchronize(ctx->small_ev));
  if (bytes > ctx->small_cap) {
    if (ctx->small_pin) cudaFreeHost(ctx->small_pin);
    ctx->small_pin = nullptr;
    ctx->small_cap = 0;
    const size_t cap = std::max<size_t>(2 * bytes, size_t(1) << 16);
    ck(cudaHostAlloc(&ctx->small_pin, cap, cudaHostAllocMapped));
    ctx->small_cap = cap;
  }
  if (!ctx->small_ev) ck(cudaEventCreateWithFlags(&ctx->small_ev, cudaEventDisableTiming));
  return static_cast<unsigned char*>(ctx->small_pin);
}

// device copy of `bytes` of mapped pinned memory by a kernel: as a DMA copy a
// descriptor upload would queue behind the bulk image copies on the engine
void upload_zero_copy(void* dst, const unsigned char* pinned, size_t bytes, cudaStream_t s) {
  count_copy(bytes, cudaMemcpyHostToDevice);
  unsigned char* src = nullptr;
  ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&src), const_cast<unsigned char*>(pinned),
                              0));
  const unsigned blocks = unsigned(std::min<size_t>((bytes / 16 + 255) / 256 + 1, 64));
  k_copy_from_host<<<blocks, 256, 0, s>>>(static_cast<unsigned char*>(dst), src, bytes);
  ck(cudaGetLastError());
}

// a deferred mesh the device build takes (cluster-sized, not yet on a device)
bool device_buildable(const HostMesh& h) {
  return h.deferred && h.dV && !h.dev && h.n >= 3;
}

// with64: also the fp64 self terms and 1/valence (the fp64 cluster path)
int device_sms();

// Meshes above this size are built by grid-wide kernels (k_bg_*), the rest
// by one 8-CTA cluster each (k_mesh_build_a/b), all sorted together.
constexpr int64_t kBuildGridNodes = 32768;

void device_build_meshes(mrb_ctx* ctx, const std::vector<HostMesh*>& todo_in, cudaStream_t copy,
                         bool with64 = false) {
  if (todo_in.empty()) return;
  // cluster-built meshes first, then the large ones
  std::vector<HostMesh*> todo = todo_in;
  std::stable_partition(todo.begin(), todo.end(),
                        [](const HostMesh* h) { return h->n <= kBuildGridNodes; });
  const size_t K = todo.size();
  size_t K_small = 0;
  while (K_small < K && todo[K_small]->n <= kBuildGridNodes) ++K_small;
  // inputs: V (double2) and T (int3) per mesh, one pinned stage, one copy
  std::vector<size_t> in_off(K), out_off(K), b_off(K), key_off(K);
  size_t in_tot = 0, out_tot = 0, b_tot = 0, keys = 0;
  for (size_t i = 0; i < K; ++i) {
    const size_t n = size_t(todo[i]->n), m = size_t(todo[i]->m);
    in_off[i] = in_tot;
    in_tot += al256(n * 16) + al256(m * 12);
    out_off[i] = out_tot;  // DeviceMesh slab: V, tri, perm, g_self_f, inv_val_f (+ fp64)
    out_tot += al256(n * 16) + al256(m * 16) + al256(n * 4) + al256(n * 8) + al256(n * 4) +
               (with64 ? al256(n * 16) + al256(n * 8) : 0);
    b_off[i] = b_tot;  // build slab (kept: nb_ptr, nb_idx, g_nb)
    const size_t e2 = 3 * m + n;  // one-ring entries of a manifold mesh (2e <= 3m + n)
    b_tot += al256(m * 8) + al256(m * 48) + 3 * al256((n + 1) * 4) + 2 * al256((n + 1) * 4) +
             al256(3 * m * 4) + al256(6 * m) + 2 * al256(e2 * 4) + al256(n * 8) +
             al256((n + 1) * 4) + al256(e2 * 16);
    key_off[i] = keys;
    keys += n;
  }
  // V / T straight from the creation blocks (same layout): one copy per run
  // of meshes adjacent in their block
  unsigned char* din = nullptr;
  {
    AllocScope scope(copy);
    if (ctx->kept[kKeptVT].cap >= in_tot && ctx->build_ev)
      ck(cudaStreamWaitEvent(copy, ctx->build_ev, 0));  // the previous build read it
    din = static_cast<unsigned char*>(kept_buffer(ctx, kKeptVT, in_tot));
    dev_mark(copy, "mesh V/T upload start");
    auto region = [&](size_t i) { return (i + 1 < K ? in_off[i + 1] : in_tot) - in_off[i]; };
    for (size_t i = 0; i < K;) {
      const unsigned char* src = reinterpret_cast<const unsigned char*>(todo[i]->dV);
      size_t j = i + 1, bytes = region(i);
      while (j < K && reinterpret_cast<const unsigned char*>(todo[j]->dV) == src + bytes &&
             todo[j]->def_hold == todo[i]->def_hold)
        bytes += region(j++);
      ck(mrb_copy_async(din + in_off[i], src, bytes, cudaMemcpyHostToDevice, copy));
      i = j;
    }
    if (!ctx->build_in) ck(cudaEventCreateWithFlags(&ctx->build_in, cudaEventDisableTiming));
    ck(cudaEventRecord(ctx->build_in, copy));
    dev_mark(copy, "mesh V/T upload done");
  }
  cudaStream_t s = ctx->stream;
  ck(cudaStreamWaitEvent(s, ctx->build_in, 0));
  AllocScope scope(s);
  const std::shared_ptr<unsigned char> out = shared_slab(out_tot, s);
  const std::shared_ptr<unsigned char> bld = shared_slab(b_tot + al256(K * 16), s);
  int* dstats = reinterpret_cast<int*>(bld.get() + b_tot);
  unsigned long long* kin = dalloc<unsigned long long>(2 * keys);
  int* vin = dalloc<int>(2 * keys);
  std::vector<BuildJob> jobs(K);
  for (size_t i = 0; i < K; ++i) {
    HostMesh& h = *todo[i];
    const size_t n = size_t(h.n), m = size_t(h.m);
    BuildJob& J = jobs[i];
    J.n = int(n);
    J.m = int(m);
    J.mesh = int(i);
    unsigned char* p = din + in_off[i];
    J.V = reinterpret_cast<const double2*>(p);
    J.T = reinterpret_cast<const int*>(p + al256(n * 16));
    unsigned char* b = bld.get() + b_off[i];
    auto take = [&](size_t bytes) {
      unsigned char* q = b;
      b += al256(bytes);
      return q;
    };
    J.areas = reinterpret_cast<double*>(take(m * 8));
    J.coeffs = reinterpret_cast<double*>(take(m * 48));
    J.cnt = reinterpret_cast<int*>(take((n + 1) * 4));      // + 1: device scans of the
    J.valence = reinterpret_cast<int*>(take((n + 1) * 4));  // grid kernels (last entry 0)
    J.iperm = reinterpret_cast<int*>(take((n + 1) * 4));
    J.inc_ptr = reinterpret_cast<int*>(take((n + 1) * 4));
    J.ring_ptr = reinterpret_cast<int*>(take((n + 1) * 4));
    J.inc_idx = reinterpret_cast<int*>(take(3 * m * 4));
    J.cpos = take(6 * m);
    J.ring_cap = int(3 * m + n);
    J.ring_idx = reinterpret_cast<int*>(take(size_t(J.ring_cap) * 4));
    J.nb_idx = reinterpret_cast<int*>(take(size_t(J.ring_cap) * 4));
    J.varea = reinterpret_cast<double*>(take(n * 8));
    J.nb_ptr = reinterpret_cast<int*>(take((n + 1) * 4));
    J.g_nb = reinterpret_cast<double2*>(take(size_t(J.ring_cap) * 16));
    J.key = kin + key_off[i];
    J.val = vin + key_off[i];
    J.sorted = vin + keys + key_off[i];
    unsigned char* o = out.get() + out_off[i];
    J.Vn = reinterpret_cast<double2*>(o);
    J.tri = reinterpret_cast<int4*>(o + al256(n * 16));
    J.perm = reinterpret_cast<int*>(o + al256(n * 16) + al256(m * 16));
    J.g_self_f = reinterpret_cast<float2*>(o + al256(n * 16) + al256(m * 16) + al256(n * 4));
    J.inv_val_f = reinterpret_cast<float*>(o + al256(n * 16) + al256(m * 16) + al256(n * 4) +
                                           al256(n * 8));
    J.g_self_d = nullptr;
    J.inv_val_d = nullptr;
    if (with64) {
      unsigned char* o64 = o + al256(n * 16) + al256(m * 16) + al256(n * 4) + al256(n * 8) +
                           al256(n * 4);
      J.g_self_d = reinterpret_cast<double2*>(o64);
      J.inv_val_d = reinterpret_cast<double*>(o64 + al256(n * 16));
    }
    J.stats = dstats + 4 * i;
  }
  unsigned char* pin = small_pinned(ctx, K * sizeof(BuildJob));
  std::memcpy(pin, jobs.data(), K * sizeof(BuildJob));
  BuildJob* djobs = dalloc<BuildJob>(K);
  upload_zero_copy(djobs, pin, K * sizeof(BuildJob), s);
  ck(cudaEventRecord(ctx->small_ev, s));
  ck(cudaMemsetAsync(dstats, 0, K * 16, s));
  if (K_small) k_mesh_build_a<<<unsigned(K_small * kBuildCluster), kBuildThreads, 0, s>>>(djobs);
  // large meshes: the same steps as grid-wide kernels with CUB scans between
  const int bg_blocks = 4 * device_sms(), bg_threads = 256;
  double4* bounds = K > K_small ? dalloc<double4>(bg_blocks) : nullptr;
  auto scan = [&](const int* in, int* out, int count) {  // exclusive, count = n + 1
    size_t tb = 0;
    ck(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, count, s));
    void* tmp = dalloc<unsigned char>(tb);
    ck(cub::DeviceScan::ExclusiveSum(tmp, tb, in, out, count, s));
    dev_free(tmp, s);
  };
  for (size_t i = K_small; i < K; ++i) {
    const BuildJob& J = jobs[i];
    const BuildJob* dj = djobs + i;
    ck(cudaMemsetAsync(J.cnt, 0, size_t(J.n + 1) * 4, s));
    k_bg_tri<<<bg_blocks, bg_threads, 0, s>>>(dj);
    scan(J.cnt, J.inc_ptr, J.n + 1);
    ck(cudaMemsetAsync(J.cnt, 0, size_t(J.n + 1) * 4, s));
    k_bg_fill<<<bg_blocks, bg_threads, 0, s>>>(dj);
    ck(cudaMemsetAsync(J.valence + J.n, 0, 4, s));
    k_bg_vertex<<<bg_blocks, bg_threads, 0, s>>>(dj, bounds);
    scan(J.valence, J.ring_ptr, J.n + 1);
    k_bg_ring_key<<<bg_blocks, bg_threads, 0, s>>>(dj, bounds, bg_blocks);
  }
  dev_mark(s, "  build pass A done");
  // the node order: a stable sort of (mesh << 32 | Morton key) = the host's
  // std::stable_sort of each mesh's keys
  int end_bit = 32;
  while ((size_t(1) << (end_bit - 32)) < K) ++end_bit;
  size_t temp = 0;
  ck(cub::DeviceRadixSort::SortPairs(nullptr, temp, kin, kin + keys, vin, vin + keys, int(keys),
                                     0, end_bit, s));
  void* dtemp = dalloc<unsigned char>(temp);
  ck(cub::DeviceRadixSort::SortPairs(dtemp, temp, kin, kin + keys, vin, vin + keys, int(keys), 0,
                                     end_bit, s));
  dev_mark(s, "  node order sorted");
  if (K_small) k_mesh_build_b<<<unsigned(K_small * kBuildCluster), kBuildThreads, 0, s>>>(djobs);
  for (size_t i = K_small; i < K; ++i) {
    const BuildJob& J = jobs[i];
    const BuildJob* dj = djobs + i;
    ck(cudaMemsetAsync(J.cnt + J.n, 0, 4, s));
    k_bg_perm<<<bg_blocks, bg_threads, 0, s>>>(dj);
    scan(J.cnt, J.nb_ptr, J.n + 1);
    k_bg_rows<<<bg_blocks, bg_threads, 0, s>>>(dj);
  }
  if (bounds) dev_free(bounds, s);
  ck(cudaGetLastError());
  dev_free(dtemp, s);
  dev_free(kin, s);
  dev_free(vin, s);
  dev_free(djobs, s);
  if (ctx->build_stats_cap < K) {
    if (ctx->build_stats) cudaFreeHost(ctx->build_stats);
    ctx->build_stats = nullptr;
    ctx->build_stats_cap = 0;
    const size_t cap = std::max<size_t>(K, 256);
    ck(cudaHostAlloc(reinterpret_cast<void**>(&ctx->build_stats), cap * 16, cudaHostAllocDefault));
    ctx->build_stats_cap = cap;
  }
  ck(mrb_copy_async(ctx->build_stats, dstats, K * 16, cudaMemcpyDeviceToHost, s));
  if (!ctx->build_ev) ck(cudaEventCreateWithFlags(&ctx->build_ev, cudaEventDisableTiming));
  ck(cudaEventRecord(ctx->build_ev, s));
  dev_mark(s, "mesh build done");
  for (size_t i = 0; i < K; ++i) {
    HostMesh& h = *todo[i];
    const BuildJob& J = jobs[i];
    h.dev.reset(new DeviceMesh());
    DeviceMesh& d = *h.dev;
    d.device = ctx->device;
    d.stream = s;
    d.slab = out.get() + out_off[i];
    d.slab_hold = out;
    d.V = J.Vn;
    d.tri = J.tri;
    d.perm = J.perm;
    d.g_self_f = J.g_self_f;
    d.inv_val_f = J.inv_val_f;
    d.g_self_d = J.g_self_d;  // slab64 stays null: these live in the shared slab
    d.inv_val_d = J.inv_val_d;
    d.max_deg = h.max_deg;
    d.b_nb_ptr = J.nb_ptr;
    d.b_nb_idx = J.nb_idx;
    d.b_g_nb = J.g_nb;
    d.build_hold = bld;
  }
  ctx->build_pending = todo;
}

// Check the pending device builds (waits for them): exact max_deg and edge
// counts; a mesh the build flagged loses its device arrays and gets the host
// build.  Returns "" or the first failing mesh's ValueError text.
std::string device_build_finish(mrb_ctx* ctx) {
  if (ctx->build_pending.empty()) return "";
  ck(cudaEventSynchronize(ctx->build_ev));
  std::vector<HostMesh*> todo;
  todo.swap(ctx->build_pending);
  std::string err;
  for (size_t i = 0; i < todo.size(); ++i) {
    HostMesh& h = *todo[i];
    const int* st = ctx->build_stats + 4 * i;
    if (st[0] == 0) {
      h.max_deg = st[1];
      h.ne = st[2] / 2;
      if (h.dev) h.dev->max_deg = st[1];
      continue;
    }
    h.dev.reset();  // stream-ordered frees
    const std::string& e = ensure_host(h);
    if (!e.empty() && err.empty()) err = e;
  }
  return err;
}

// Fast-path topologies of device-built meshes for the requested (mesh,
// cluster size, nodes/thread) shapes, planned and written on stream s
// (k_topo_count, one sync for the sizes, k_topo_write, k_topo_send).
// Returns false, installing nothing, when a mesh needs the host planner.
bool device_cluster_topos(mrb_ctx* ctx, const std::vector<std::tuple<HostMesh*, int, int>>& req,
                          cudaStream_t s, bool f64 = false) {
  struct Item {
    HostMesh* h;
    int npt;
    TopoHost th;
    size_t base;
  };
  std::vector<Item> items;
  for (const auto& r : req) {
    HostMesh* h = std::get<0>(r);
    const int cs = std::get<1>(r), npt = std::get<2>(r);
    // cluster shapes (<= 16 CTAs) and whole-GPU grid shapes (SMs CTAs, 768 x npt slots)
    if (!h->dev || !h->dev->b_nb_ptr || cs < 1 || cs > 1024 || kClusterThreads * npt > 8192)
      return false;
    const int chunk = int((h->n + cs - 1) / cs);
    if (h->dev->topo.count(topo_key(cs, chunk, f64 ? 1 : npt, f64))) continue;
    bool dup = false;
    for (const Item& it : items)
      dup = dup || (it.h == h && it.th.cs == cs && it.npt == npt);
    if (dup) continue;
    Item it;
    it.h = h;
    it.npt = npt;
    it.th.cs = cs;
    it.th.chunk = chunk;
    it.th.slices = (chunk + 31) / 32;
    if (it.th.slices > kTopoMaxSlices) return false;
    items.push_back(std::move(it));
  }
  if (items.empty()) return true;
  const size_t K = items.size();
  AllocScope scope(s);
  std::vector<size_t> soff(K);
  size_t stat_ints = 0;
  for (size_t k = 0; k < K; ++k) {
    soff[k] = stat_ints;
    stat_ints += 4 * size_t(items[k].th.cs);
  }
  int* dstat = dalloc<int>(stat_ints);
  ck(cudaMemsetAsync(dstat, 0, stat_ints * 4, s));
  std::vector<TopoJob> jobs(K);
  for (size_t k = 0; k < K; ++k) {
    const Item& it = items[k];
    TopoJob& J = jobs[k];
    J = TopoJob{};
    J.n = int(it.h->n);
    J.cs = it.th.cs;
    J.chunk = it.th.chunk;
    J.slices = it.th.slices;
    J.slots = kClusterThreads * it.npt;
    J.nb_ptr = it.h->dev->b_nb_ptr;
    J.nb_idx = it.h->dev->b_nb_idx;
    J.g_nb = it.h->dev->b_g_nb;
    J.stat = dstat + soff[k];
  }
  const size_t jb = al256(K * sizeof(TopoJob));
  unsigned char* pin = small_pinned(ctx, 2 * jb + stat_ints * 4);
  std::memcpy(pin, jobs.data(), K * sizeof(TopoJob));
  TopoJob* djobs = dalloc<TopoJob>(K);
  upload_zero_copy(djobs, pin, K * sizeof(TopoJob), s);
  int cs_max = 1;
  for (const Item& it : items) cs_max = std::max(cs_max, it.th.cs);
  k_topo_count<<<dim3(unsigned(cs_max), unsigned(K)), kTopoThreads, 0, s>>>(djobs);
  int* hstat = reinterpret_cast<int*>(pin + 2 * jb);
  ck(mrb_copy_async(hstat, dstat, stat_ints * 4, cudaMemcpyDeviceToHost, s));
  dev_mark(s, "  topology sizes");
  host_tick("topo: count enqueued");
  ck(cudaStreamSynchronize(s));
  host_tick("topo: sizes synced");
  size_t total = 0;
  bool ok = true;
  for (size_t k = 0; k < K && ok; ++k) {
    TopoHost& t = items[k].th;
    const int cs = t.cs;
    const int* st = hstat + soff[k];
    int stride = 0, hs = 2, ss = 2;
    for (int r = 0; r < cs; ++r) {
      ok = ok && st[3 * r + 2] == 0;
      stride = std::max(stride, st[3 * r]);
      hs = std::max(hs, st[3 * r + 1] + 1);
      ss = std::max(ss, st[3 * cs + r]);
    }
    t.stride = std::max((stride + 7) / 8 * 8, 8);
    t.hstride = (hs + 31) / 32 * 32;
    // push send lists for cluster shapes only (plan_topo)
    t.sstride = cs <= 16 && kClusterThreads * items[k].npt <= 4096 ? (ss + 31) / 32 * 32 : 0;
    const size_t n = size_t(items[k].h->n);
    const size_t bytes[8] = {size_t(cs) * t.stride * 2, size_t(cs) * t.stride * (f64 ? 16 : 8),
                             size_t(cs) * t.slices * 4, size_t(cs) * t.hstride * 4,
                             size_t(cs) * 4,           n,
                             size_t(cs) * t.sstride * 4, size_t(cs) * 4};
    t.total = 0;
    for (int q = 0; q < 8; ++q) {
      t.off[q] = t.total;
      t.total += al256(bytes[q]);
    }
    items[k].base = total;
    total += t.total;
  }
  if (!ok) {
    ck(cudaEventRecord(ctx->small_ev, s));
    dev_free(djobs, s);
    dev_free(dstat, s);
    return false;
  }
  const std::shared_ptr<unsigned char> all = shared_slab(total, ctx->stream);
  ck(cudaMemsetAsync(all.get(), 0, total, s));
  host_tick("topo: slab");
  for (size_t k = 0; k < K; ++k) {
    const TopoHost& t = items[k].th;
    unsigned char* slab = all.get() + items[k].base;
    TopoJob& J = jobs[k];
    J.codes = reinterpret_cast<uint16_t*>(slab + t.off[0]);
    J.g = reinterpret_cast<float2*>(slab + t.off[1]);
    J.g64 = f64 ? reinterpret_cast<double2*>(slab + t.off[1]) : nullptr;
    J.soff = reinterpret_cast<uint32_t*>(slab + t.off[2]);
    J.halo = reinterpret_cast<uint32_t*>(slab + t.off[3]);
    J.n_halo = reinterpret_cast<int*>(slab + t.off[4]);
    J.deg = slab + t.off[5];
    J.send = reinterpret_cast<uint32_t*>(slab + t.off[6]);
    J.n_send = reinterpret_cast<int*>(slab + t.off[7]);
    J.stride = t.stride;
    J.hstride = t.hstride;
    J.sstride = t.sstride;
  }
  std::memcpy(pin + jb, jobs.data(), K * sizeof(TopoJob));
  dev_mark(s, "  topology slab zeroed");
  upload_zero_copy(djobs, pin + jb, K * sizeof(TopoJob), s);
  dev_mark(s, "  topology jobs uploaded");
  ck(cudaEventRecord(ctx->small_ev, s));
  k_topo_write<<<dim3(unsigned(cs_max), unsigned(K)), kTopoThreads, 0, s>>>(djobs);
  dev_mark(s, "  topology written");
  k_topo_send<<<dim3(unsigned(cs_max), unsigned(K)), 256, 0, s>>>(djobs);
  ck(cudaGetLastError());
  dev_mark(s, "device topologies done");
  dev_free(djobs, s);
  dev_free(dstat, s);
  host_tick("topo: write enqueued");
  for (size_t k = 0; k < K; ++k)
    install_topo(*items[k].h, items[k].npt, items[k].th, all.get() + items[k].base, f64).hold =
        all;
  host_tick("topo: installed");
  return true;
}

const DeviceMesh::Topo& ensure_cluster_topo(mrb_ctx* ctx, HostMesh& h, int cs, int chunk,
                                            int npt) {
  auto it = h.dev->topo.find(topo_key(cs, chunk, npt));
  if (it != h.dev->topo.end()) return it->second;
  if (h.dev->b_nb_ptr && device_cluster_topos(ctx, {std::make_tuple(&h, cs, npt)}, ctx->stream))
    return h.dev->topo.at(topo_key(cs, chunk, npt));
  AllocScope scope(ctx->stream);
  const TopoHost th = plan_topo(h, cs, chunk, npt);
  std::vector<unsigned char> packed(th.total);
  write_topo(h, cs, th, packed.data(), npt);
  unsigned char* slab = dalloc<unsigned char>(th.total);
  ck(mrb_copy_async(slab, packed.data(), th.total, cudaMemcpyHostToDevice,
                    ctx->stream));  // pageable: staged before return
  return install_topo(h, npt, th, slab);
}

// topologies of many meshes: built on a host thread pool, uploaded through
// the pinned staging buffer
// Topologies of many meshes in two halves.  plan_cluster_topos plans them on
// the host thread pool, allocates one shared device slab and installs every
// topology's device pointers (so descriptors can be built at once); the data
// is packed straight into the pinned staging buffer and copied by
// upload_cluster_topos, all at once or (mrb_register_many) one wave group at
// a time, ahead of that group's launch.
struct TopoUpload {
  std::vector<HostMesh*> meshes;
  std::vector<TopoHost> th;
  std::vector<size_t> base;
  int cs = 0, npt = 1;
  int slot = 1;                    // pinned staging slot
  unsigned char* stage = nullptr;  // pinned, ctx->pinned[slot]
  unsigned char* dev = nullptr;    // shared slab
  bool device = false;             // planned + written on the GPU (device_cluster_topos)
};

TopoUpload plan_cluster_topos(mrb_ctx* ctx, const std::vector<HostMesh*>& todo, int cs, int npt,
                              int slot = 1, cudaStream_t alloc_s = nullptr) {
  TopoUpload up;
  up.meshes = todo;
  up.cs = cs;
  up.npt = npt;
  up.slot = slot;
  {  // device-built meshes: planned and written on the GPU
    bool dev = !todo.empty();
    std::vector<std::tuple<HostMesh*, int, int>> req;
    for (HostMesh* h : todo) {
      dev = dev && h->dev && h->dev->b_nb_ptr;
      req.emplace_back(h, cs, npt);
    }
    if (dev && device_cluster_topos(ctx, req, alloc_s ? alloc_s : ctx->stream)) {
      up.device = true;
      return up;
    }
  }
  up.th.resize(todo.size());
  parallel_for(todo.size(), [&](size_t i) {
    const HostMesh& h = *todo[i];
    up.th[i] = plan_topo(h, cs, int((h.n + cs - 1) / cs), npt);
  });
  size_t total = 0;
  up.base.resize(todo.size());
  for (size_t i = 0; i < todo.size(); ++i) {
    up.base[i] = total;
    total += up.th[i].total;
  }
  up.stage = static_cast<unsigned char*>(pinned_stage(ctx, std::max<size_t>(total, 1), slot));
  // allocated in `alloc_s` order (the copy stream of a lazily planned group:
  // ctx->stream may hold running groups), freed in ctx->stream order
  AllocScope scope(alloc_s ? alloc_s : ctx->stream);
  const std::shared_ptr<unsigned char> all = shared_slab(std::max<size_t>(total, 1), ctx->stream);
  up.dev = all.get();
  for (size_t i = 0; i < todo.size(); ++i)
    install_topo(*todo[i], npt, up.th[i], all.get() + up.base[i]).hold = all;
  return up;
}

// pack meshes [i0, i1) of an upload and copy them on `stream` (one copy)
void upload_cluster_topos(mrb_ctx* ctx, const TopoUpload& up, size_t i0, size_t i1,
                          cudaStream_t stream) {
  if (i0 >= i1 || up.device) return;
  parallel_for(i1 - i0, [&](size_t k) {
    const size_t i = i0 + k;
    write_topo(*up.meshes[i], up.cs, up.th[i], up.stage + up.base[i], up.npt);
  });
  const size_t b0 = up.base[i0];
  const size_t b1 = i1 < up.meshes.size() ? up.base[i1] : up.base.back() + up.th.back().total;
  if (std::getenv("MESHREG_B200_DEBUG")) {
    char what[64];
    std::snprintf(what, sizeof what, "topology copy %.1f MB", (b1 - b0) / 1e6);
    dev_mark(stream, what);
  }
  ck(mrb_copy_async(up.dev + b0, up.stage + b0, b1 - b0, cudaMemcpyHostToDevice, stream));
  dev_mark(stream, "topology copy done");
  ck(cudaEventRecord(ctx->stage_done[up.slot], stream));  // staging reusable after this
}

void ensure_cluster_topos(mrb_ctx* ctx, const std::vector<HostMesh*>& meshes, int cs, int npt,
                          int slot = 1) {
  std::vector<HostMesh*> todo;
  for (HostMesh* h : meshes) {
    const int chunk = int((h->n + cs - 1) / cs);
    if (!h->dev->topo.count(topo_key(cs, chunk, npt)) &&
        std::find(todo.begin(), todo.end(), h) == todo.end())
      todo.push_back(h);
  }
  if (todo.empty()) return;
  const bool dbg = std::getenv("MESHREG_B200_DEBUG") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto tick = [&](const char* what) {
    if (!dbg) return;
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "meshreg_b200:   topologies %-14s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  TopoUpload up = plan_cluster_topos(ctx, todo, cs, npt, slot);
  tick("host plan");
  upload_cluster_topos(ctx, up, 0, up.meshes.size(), ctx->stream);
  tick("fill + copy");
}

// fp64 topologies of k_cluster64 (one node per thread): the same paired
// SELL layout with double2 coefficients, cached under their own key; planned
// and packed on the worker pool, uploaded as one copy
int64_t topo64_key(int cs, int chunk) { return topo_key(cs, chunk, 1, true); }

void ensure_cluster_topos64(mrb_ctx* ctx, const std::vector<HostMesh*>& meshes, int cs) {
  std::vector<HostMesh*> todo;
  for (HostMesh* h : meshes) {
    const int chunk = int((h->n + cs - 1) / cs);
    if (!h->dev->topo.count(topo64_key(cs, chunk)) &&
        std::find(todo.begin(), todo.end(), h) == todo.end())
      todo.push_back(h);
  }
  if (todo.empty()) return;
  {  // device-built meshes: planned and written on the GPU
    bool dev = true;
    std::vector<std::tuple<HostMesh*, int, int>> req;
    for (HostMesh* h : todo) {
      dev = dev && h->dev->b_nb_ptr;
      req.emplace_back(h, cs, 1);
    }
    if (dev && device_cluster_topos(ctx, req, ctx->stream, true)) return;
  }
  std::vector<TopoHost> th(todo.size());
  parallel_for(todo.size(), [&](size_t i) {
    th[i] = plan_topo(*todo[i], cs, int((todo[i]->n + cs - 1) / cs), 1, 16);
  });
  std::vector<size_t> base(todo.size());
  size_t total = 0;
  for (size_t i = 0; i < todo.size(); ++i) {
    base[i] = total;
    total += th[i].total;
  }
  // packed straight into the pinned staging buffer (a pageable copy of the
  // ~2 MB per C2-size mesh would stage synchronously)
  unsigned char* packed =
      static_cast<unsigned char*>(pinned_stage(ctx, std::max<size_t>(total, 1), 1));
  parallel_for(todo.size(), [&](size_t i) {
    write_topo(*todo[i], cs, th[i], packed + base[i], 1, true);
  });
  AllocScope scope(ctx->stream);
  const std::shared_ptr<unsigned char> all = shared_slab(std::max<size_t>(total, 1), ctx->stream);
  ck(mrb_copy_async(all.get(), packed, total, cudaMemcpyHostToDevice, ctx->stream));
  ck(cudaEventRecord(ctx->stage_done[1], ctx->stream));  // staging reusable after this
  for (size_t i = 0; i < todo.size(); ++i) {
    DeviceMesh::Topo t;
    unsigned char* slab = all.get() + base[i];
    t.chunk = th[i].chunk;
    t.topo_stride = th[i].stride;
    t.slices = th[i].slices;
    t.halo_stride = th[i].hstride;
    t.slab = slab;
    t.hold = all;
    t.codes = reinterpret_cast<uint16_t*>(slab + th[i].off[0]);
    t.g64 = reinterpret_cast<double2*>(slab + th[i].off[1]);
    t.slice_off = reinterpret_cast<uint32_t*>(slab + th[i].off[2]);
    t.halo = reinterpret_cast<uint32_t*>(slab + th[i].off[3]);
    t.n_halo = reinterpret_cast<int*>(slab + th[i].off[4]);
    t.deg = slab + th[i].off[5];
    t.send = reinterpret_cast<uint32_t*>(slab + th[i].off[6]);
    t.n_send = reinterpret_cast<int*>(slab + th[i].off[7]);
    t.send_stride = th[i].sstride;
    todo[i]->dev->topo[topo64_key(cs, t.chunk)] = t;
  }
}

// bytes of dynamic shared memory of k_cluster64_push (Push64Smem carve)
size_t push64_dyn_smem(int topo_stride, int slices, int halo_stride, int send_stride) {
  const size_t S = size_t(kClusterThreads), X = S + halo_stride;
  return size_t(topo_stride) * (16 + 2) + S * (16 + 16 + 8) + X * (2 * 16 + 2 * 8) +
         size_t(send_stride) * 4 + size_t(slices) * 4;
}

// bytes of dynamic shared memory of k_cluster64 (Cluster64Smem carve)
size_t cluster64_dyn_smem(int topo_stride, int slices, int halo_stride, bool two_u) {
  const size_t S = size_t(kClusterThreads), X = S + halo_stride;
  return size_t(topo_stride) * (16 + 2) + S * (16 + 16 + 8) + X * (16 * (two_u ? 2 : 1) + 8) +
         size_t(halo_stride) * 4 + size_t(slices) * 4;
}

// bytes of dynamic shared memory of k_cluster_register (ClusterSmem carve)
size_t cluster_dyn_smem(int npt, int topo_stride, int slices, int halo_stride, bool two_u) {
  const size_t S = size_t(kClusterThreads) * npt, X = S + halo_stride;
  return S * (sizeof(double2) + sizeof(float2) + sizeof(float) + 1) +
         X * (sizeof(float2) * (two_u ? 2 : 1) + sizeof(float)) + size_t(halo_stride) * 4 +
         size_t(topo_stride) * (sizeof(float2) + sizeof(uint16_t)) + size_t(slices) * 4;
}

// bytes of dynamic shared memory of k_cluster_push (PushSmem carve)
size_t push_dyn_smem(int npt, int topo_stride, int slices, int halo_stride, int send_stride) {
  const size_t S = size_t(kClusterThreads) * npt, X = S + halo_stride;
  return S * (sizeof(double2) + sizeof(float2) + sizeof(float) + 1) +
         2 * X * (sizeof(float2) + sizeof(float)) + size_t(send_stride) * 4 +
         size_t(topo_stride) * (sizeof(float2) + sizeof(uint16_t)) + size_t(slices) * 4;
}

// Pixel->triangle map for (W, H): GPU raster + host locate fallback, in two
// halves so host work can run while the rasters do: issue_pixel_maps enqueues
// the rasters and the uncovered-pixel counts (into pinned memory) and records
// an event; finish_pixel_maps waits for that event only and runs the
// reference's binned locate for uncovered pixels.  Returns "" or the
// MeshCoverageError message.
struct PixelMapJob {
  std::vector<HostMesh*> todo;
  std::vector<int*> maps;
  int W = 0, H = 0;
  unsigned long long* missing = nullptr;  // pinned, one count per map
  cudaEvent_t done = nullptr;
  std::shared_ptr<unsigned char> slab;    // the maps, when rasterised together
};

// side = true: the rasters run on ctx->aux after the mesh uploads on
// ctx->stream, so a run enqueued on ctx->stream need not wait for them (its
// dense passes wait for job.done instead)
PixelMapJob issue_pixel_maps(mrb_ctx* ctx, const std::vector<HostMesh*>& meshes, int W, int H,
                             bool side = false, cudaEvent_t after = nullptr) {
  PixelMapJob job;
  job.W = W;
  job.H = H;
  const auto key = std::make_pair(W, H);
  ensure_device_meshes(ctx, meshes, false);
  cudaStream_t s = ctx->stream;
  if (side) {
    cudaStream_t& ax = ctx->fill_idle ? ctx->aux : ctx->aux_hi;
    if (!ax) ck(create_stream(&ax, !ctx->fill_idle));
    if (!ctx->aux_ev) ck(cudaEventCreateWithFlags(&ctx->aux_ev, cudaEventDisableTiming));
    if (after) {  // the meshes are ready at `after` (device build)
      ck(cudaStreamWaitEvent(ax, after, 0));
    } else {
      ck(cudaEventRecord(ctx->aux_ev, ctx->stream));  // meshes uploaded
      ck(cudaStreamWaitEvent(ax, ctx->aux_ev, 0));
    }
    s = ax;
  }
  AllocScope scope(s);
  for (HostMesh* h : meshes) {
    if (!h->dev->pixel_maps.count(key) &&
        std::find(job.todo.begin(), job.todo.end(), h) == job.todo.end())
      job.todo.push_back(h);
  }
  if (job.todo.empty()) return job;
  const size_t npx = size_t(W) * size_t(H);
  if (ctx->counts_cap < job.todo.size()) {  // pinned count slots (grow)
    if (ctx->counts) cudaFreeHost(ctx->counts);
    ctx->counts = nullptr;
    ctx->counts_cap = 0;
    const size_t cap = std::max<size_t>(job.todo.size(), 1024);
    ck(cudaHostAlloc(reinterpret_cast<void**>(&ctx->counts), cap * sizeof(unsigned long long),
                     cudaHostAllocDefault));
    ctx->counts_cap = cap;
  }
  job.missing = ctx->counts;
  unsigned long long* cnt = nullptr;
  ck(cudaMallocAsync(&cnt, job.todo.size() * sizeof(unsigned long long), s));
  ck(cudaMemsetAsync(cnt, 0, job.todo.size() * sizeof(unsigned long long), s));
  job.maps.resize(job.todo.size());
  if (job.todo.size() == 1) {
    const HostMesh& h = *job.todo[0];
    job.maps[0] = dalloc<int>(npx);
    ck(cudaMemsetAsync(job.maps[0], 0x7f, npx * sizeof(int), s));
    k_raster<<<unsigned((h.m * kRasterLanes + 255) / 256), 256, 0, s>>>(h.dev->V, h.dev->tri, int(h.m), W, H,
                                                          job.maps[0]);
    k_count_uncovered<<<unsigned(std::min<size_t>((npx + 255) / 256, 1184)), 256, 0, s>>>(
        job.maps[0], int(npx), cnt);
  } else {
    // every map in one slab: one memset, then one raster and one count launch
    // per kRasterJobs meshes
    const size_t map_bytes = (npx * sizeof(int) + 255) / 256 * 256;
    job.slab = shared_slab(map_bytes * job.todo.size(), ctx->stream);
    ck(cudaMemsetAsync(job.slab.get(), 0x7f, map_bytes * job.todo.size(), s));
    for (size_t i0 = 0; i0 < job.todo.size(); i0 += kRasterJobs) {
      const size_t nj = std::min<size_t>(kRasterJobs, job.todo.size() - i0);
      RasterJobs rj{};
      int64_t mmax = 0;
      for (size_t j = 0; j < nj; ++j) {
        const HostMesh& h = *job.todo[i0 + j];
        job.maps[i0 + j] = reinterpret_cast<int*>(job.slab.get() + (i0 + j) * map_bytes);
        rj.V[j] = h.dev->V;
        rj.tri[j] = h.dev->tri;
        rj.map[j] = job.maps[i0 + j];
        rj.m[j] = int(h.m);
        mmax = std::max(mmax, h.m);
      }
      k_raster_many<<<dim3(unsigned((mmax * kRasterLanes + 255) / 256), unsigned(nj)), 256, 0, s>>>(rj, W, H);
      k_count_uncovered_many<<<dim3(unsigned(std::min<size_t>((npx + 255) / 256, 296)),
                                    unsigned(nj)), 256, 0, s>>>(rj, int(npx), cnt + i0);
    }
  }
  ck(cudaGetLastError());
  // installed now so descriptors can be built while the rasters run;
  // finish_pixel_maps removes the maps of meshes that fail the coverage check
  for (size_t i = 0; i < job.todo.size(); ++i) {
    job.todo[i]->dev->pixel_maps[key] = job.maps[i];
    if (job.slab) job.todo[i]->dev->pixel_map_hold[key] = job.slab;
  }
  ck(mrb_copy_async(job.missing, cnt, job.todo.size() * sizeof(unsigned long long),
                    cudaMemcpyDeviceToHost, s));
  ck(cudaFreeAsync(cnt, s));
  dev_mark(s, "rasters done");
  ck(cudaEventCreateWithFlags(&job.done, cudaEventDisableTiming));
  ck(cudaEventRecord(job.done, s));
  return job;
}

// rasters issued early by mrb_register_many (its device setup), handed to
// chunk 0's batch creation on this thread
inline thread_local PixelMapJob* t_early_pm = nullptr;

// a batch whose maps the early rasters already installed takes over their
// job (event + uncovered counts): its dense passes wait for them and its
// coverage check covers them
void adopt_early_rasters(PixelMapJob& pmj, int W, int H) {
  if (!pmj.todo.empty() || !t_early_pm || t_early_pm->todo.empty() || t_early_pm->W != W ||
      t_early_pm->H != H)
    return;
  pmj = std::move(*t_early_pm);
  t_early_pm->todo.clear();
  t_early_pm->done = nullptr;
}

std::string finish_pixel_maps(mrb_ctx* ctx, PixelMapJob& job) {
  if (job.todo.empty()) return "";
  const int W = job.W, H = job.H;
  const size_t npx = size_t(W) * size_t(H);
  const auto ts = std::chrono::steady_clock::now();
  ck(cudaEventSynchronize(job.done));
  cudaEventDestroy(job.done);
  job.done = nullptr;
  if (std::getenv("MESHREG_B200_DEBUG"))
    std::fprintf(stderr, "meshreg_b200:   pixel maps: %zu rasters, wait %.2f ms\n",
                 job.todo.size(),
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ts)
                     .count());
  std::string err;
  for (size_t i = 0; i < job.todo.size(); ++i) {
    HostMesh& h = *job.todo[i];
    const unsigned long long missing = job.missing[i];
    if (missing && err.empty()) {
      // densefield.py:176-182: binned locate for each unassigned pixel, row-major
      ensure_host(h);
      std::vector<int> host(npx);
      ck(mrb_copy(host.data(), job.maps[i], npx * sizeof(int), cudaMemcpyDeviceToHost));
      Locator loc(h);
      for (size_t q = 0; q < npx && err.empty(); ++q) {
        if (host[q] != kUnassigned) continue;
        const double px = double(q % W), py = double(q / W);
        double w[3];
        const int64_t t = loc.locate(h, px, py, w);
        if (t < 0) {
          char buf[128];
          std::snprintf(buf, sizeof buf, "point (%s, %s) not covered by any triangle",
                        py_repr(px).c_str(), py_repr(py).c_str());
          err = buf;
        }
        host[q] = int(t);
      }
      if (err.empty())
        ck(mrb_copy(job.maps[i], host.data(), npx * sizeof(int), cudaMemcpyHostToDevice));
    }
    if (missing && !err.empty()) {
      h.dev->pixel_maps.erase(std::make_pair(W, H));
      h.dev->pixel_map_hold.erase(std::make_pair(W, H));
      if (!job.slab) dev_free(job.maps[i], ctx->stream);
      continue;
    }
  }
  return err;
}

std::string ensure_pixel_maps(mrb_ctx* ctx, const std::vector<HostMesh*>& meshes, int W, int H) {
  PixelMapJob job = issue_pixel_maps(ctx, meshes, W, H);
  return finish_pixel_maps(ctx, job);
}

std::string ensure_pixel_map(mrb_ctx* ctx, HostMesh& h, int W, int H, int** out) {
  const std::string err = ensure_pixel_maps(ctx, {&h}, W, H);
  if (err.empty()) *out = h.dev->pixel_maps.at(std::make_pair(W, H));
  return err;
}

}  // namespace

// =========================================================================
// batch
// =========================================================================
struct mrb_batch {
  mrb_ctx* ctx = nullptr;
  int n_pairs = 0, W = 0, H = 0, in_dtype = MRB_F32;
  mrb_config cfg{};
  bool tap_d = false, real_d = false;
  std::vector<mrb_mesh*> meshes;
  std::vector<int> node_off;  // offsets into the concatenated u_out (nodes)
  int n_node_blocks = 0, n_pix_blocks = 0;
  int64_t total_nodes = 0;
  // device
  void* pairs = nullptr;  // PairDev<TapT,Real>[n_pairs]
  PairStatus* st = nullptr;
  int* blk_pair = nullptr;
  int* pix_blk_pair = nullptr;
  double* partials = nullptr;
  double2* pix_partials = nullptr;
  void* state = nullptr;
  double* traces = nullptr;
  void* img = nullptr;
  void* stage = nullptr;  // H2D staging (re stack, te stack)
  void** src_ptrs = nullptr;  // device: [re_0..re_{P-1}, te_0..te_{P-1}]
  void** img_ptrs = nullptr;  // device: interleaved tap buffer per pair
  std::vector<const void*> src_host;  // current sources (for graph validity)
  void* dense = nullptr;       // ux, uy, warped (Real)
  double2* u_out = nullptr;
  void* conv = nullptr;        // dtype conversion scratch for get_results
  cudaGraphExec_t graph = nullptr;
  std::vector<const void*> graph_src;
  // cluster fast path (0 = generic three-kernel loop)
  int cluster_cs = 0, cluster_npt = 1;
  int forced_cs = 0, forced_npt = 0;  // shape imposed by mrb_register_many
  bool grid_mode = false;  // k_grid_register (cluster_cs = CTAs of the whole-GPU grid)
  bool grid_flags = false; // ... with the epoch-tagged exchange (k_grid_flags)
  size_t xbytes = 0;       // exchange-word bytes of xbuf (zeroed per grid launch)
  bool push_mode = false;  // k_cluster_push (smoothing_passes <= 1): push halo exchange
  size_t push_smem = 0;
  // Tail of a throughput-mode batch: the pairs of the last, partial wave
  // [tail_p0, n_pairs) run in a second launch with the latency shape (more
  // CTAs per pair, one node per thread), which finishes the partial wave
  // sooner than the throughput shape would.
  int tail_p0 = 1 << 30;
  int tail_cs = 0, tail_npt = 0;
  size_t tail_smem = 0;
  bool tail_push = false;
  void* xbuf = nullptr;    // grid path exchange buffers (shared by the pairs, run in turn)
  uint32_t* xexports = nullptr;  // grid path: per pair [CS][SLOTS/32] export bitmaps
  unsigned* xbar = nullptr;  // grid barrier counter + gbad flags [1 + CS]
  // wave groups (mrb_register_many): the first run launches the fast path per
  // group of pairs and records group_ev[g]; get_results then copies group g
  // back on copy_stream while later groups still compute
  std::vector<int> groups;  // pair boundaries, size G + 1 (empty: one launch)
  // deferred topology upload (mrb_register_many): planned at creation, data
  // packed and copied one wave group at a time ahead of that group's launch
  std::unique_ptr<TopoUpload> topo_up;
  std::map<const HostMesh*, size_t> topo_index;  // mesh -> position in topo_up
  size_t topo_done = 0;                           // meshes of topo_up uploaded
  cudaEvent_t topo_ev = nullptr;
  std::unique_ptr<TopoUpload> tail_up;  // the tail pairs' latency-shape topologies
  bool tail_done = false;
  int planned_end = 1 << 30;  // pairs past this got no throughput-shape topology planned
  // fp64 batches: the generic path's state, image and dense pass, with the
  // descent loop in one persistent k_cluster64 launch (c64_cs CTAs per pair)
  int c64_cs = 0;
  size_t c64_smem = 0;
  bool c64_push = false;  // k_cluster64_push (smoothing_passes <= 1, fits)
  void* c64_pairs = nullptr;  // ClusterPair64[n_pairs]
  double2* pad64 = nullptr;   // padded fp64 images [pair][(H+2) x (W+2)]
  // mrb_register_many: main-shape pairs [lazy_from, planned_end) are planned
  // per wave group in the run (flush_topo), while earlier groups compute
  int lazy_from = 1 << 30;
  std::vector<std::unique_ptr<TopoUpload>> lazy_ups;
  std::vector<ClusterPair> cp_host;      // descriptors (patched for lazy pairs)
  ClusterPair* cp_pinned = nullptr;      // their pinned copy-out buffer
  std::vector<cudaEvent_t> dbg_group_ev;  // MESHREG_B200_DEBUG: start of each group launch
  std::vector<cudaEvent_t> group_ev;
  // per wave group: its images arrived (mrb_register_many; not owned).  The
  // group's padded copies are then made on the group's stream after it.
  std::vector<cudaEvent_t> img_ev;
  cudaStream_t copy_stream = nullptr;
  // tail wave + its dense pass on a side stream, concurrent with the main
  // launch's dense pass (enqueue_run)
  cudaStream_t tail_stream = nullptr;
  cudaEvent_t tail_fork = nullptr, tail_join = nullptr;
  // wave groups alternate between ctx->stream and grp_stream, so group g+1's
  // clusters fill the SMs group g's retiring clusters free (one launch per
  // group on one stream would drain the GPU between groups)
  cudaStream_t grp_stream = nullptr;
  cudaEvent_t grp_fork = nullptr, grp_join = nullptr;
  // mrb_register_many: the pixel maps' coverage check (host wait for the
  // rasters) is deferred to mrb_batch_sync, off the launch path; the dense
  // kernels skip unassigned pixels (flag 4) until then
  std::unique_ptr<PixelMapJob> pending_pm;
  bool redo = false;  // a located (not rasterised) pixel: rerun undeferred
  cudaStream_t lstream = nullptr;  // launch stream override (nullptr: ctx->stream)
  bool groups_recorded = false;
  size_t cluster_smem = 0;
  int pad_pitch = 0;
  size_t pad_plane = 0;
  int pad_copies = 4;       // 4 shifted copies, or 8 in the row-pair layout
  bool pad_rowpair = false;  // k_pad_planar_rp layout (grid path, images beyond L2)
  bool tap_evict_first = false;
  void* cpairs = nullptr;     // ClusterPair[n_pairs]
  std::vector<unsigned char> pairs_host;  // host copy of the PairDev array
  long long* phase_prof = nullptr;  // MESHREG_B200_PROFILE_PHASES
  long long* prof_host = nullptr;   // ... = "mapped": host pointer of phase_prof
  float2* img_pad = nullptr;  // 4 shifted padded (H+2)x(W+2) (Te, Re) copies per pair
  bool img_pad_borrowed = false;  // ctx kept buffers (mrb_register_many batches)
  bool pairs_borrowed = false;    // state + dense from the ctx kept buffers
  size_t state_bytes = 0;
  int runs = 0;
  // host results
  std::vector<PairStatus> h_st;
  std::vector<double> h_trace;
  bool synced = false;
  ~mrb_batch() {
    try {  // topologies installed in the meshes' caches must hold data
      if (topo_up && topo_done < topo_up->meshes.size())
        upload_cluster_topos(ctx, *topo_up, topo_done, topo_up->meshes.size(), ctx->stream);
      if (tail_up && !tail_done)
        upload_cluster_topos(ctx, *tail_up, 0, tail_up->meshes.size(), ctx->stream);
    } catch (const CudaError&) {
    }
    if (graph) cudaGraphExecDestroy(graph);
    if (pending_pm && pending_pm->done) cudaEventDestroy(pending_pm->done);
    if (cp_pinned) {
      cudaStreamSynchronize(ctx->stream);
      if (copy_stream) cudaStreamSynchronize(copy_stream);
      cudaFreeHost(cp_pinned);
    }
    for (cudaEvent_t e : group_ev) cudaEventDestroy(e);
    if (topo_ev) cudaEventDestroy(topo_ev);
    for (cudaEvent_t e : dbg_group_ev) cudaEventDestroy(e);
    if (copy_stream) cudaStreamSynchronize(copy_stream);  // context-owned streams
    if (tail_stream) cudaStreamSynchronize(tail_stream);
    if (tail_fork) cudaEventDestroy(tail_fork);
    if (tail_join) cudaEventDestroy(tail_join);
    if (grp_stream) cudaStreamSynchronize(grp_stream);
    if (grp_fork) cudaEventDestroy(grp_fork);
    if (grp_join) cudaEventDestroy(grp_join);
    void* ptrs[] = {pairs, st, blk_pair, pix_blk_pair, partials, pix_partials,
                    pairs_borrowed ? nullptr : state, traces, img, stage, src_ptrs, img_ptrs,
                    pairs_borrowed ? nullptr : dense, u_out, conv, cpairs,
                    img_pad_borrowed ? nullptr : img_pad, c64_pairs, pad64,
                    prof_host ? nullptr : phase_prof, xbuf, xbar, xexports};
    if (prof_host) cudaFreeHost(prof_host);
    for (void* p : ptrs) dev_free(p, ctx ? ctx->stream : nullptr);
  }
};

namespace {

size_t tap_size(const mrb_batch* b) { return b->tap_d ? sizeof(double) : sizeof(float); }
size_t real_size(const mrb_batch* b) { return b->real_d ? sizeof(double) : sizeof(float); }
size_t in_size(int dtype) { return dtype == MRB_F64 ? sizeof(double) : sizeof(float); }

void free_pairs(mrb_batch* b) {
  if (b->pairs_borrowed) b->state = b->dense = nullptr;
  void** ptrs[] = {&b->state, &b->dense, &b->pairs, reinterpret_cast<void**>(&b->blk_pair),
                   reinterpret_cast<void**>(&b->pix_blk_pair),
                   reinterpret_cast<void**>(&b->partials),
                   reinterpret_cast<void**>(&b->pix_partials)};
  for (void** p : ptrs) {
    dev_free(*p, b->ctx->stream);
    *p = nullptr;
  }
}

template <typename TapT, typename Real>
void build_pairs(mrb_batch* b) {
  using PD = PairDev<TapT, Real>;
  using R2 = typename V2<Real>::type;
  std::vector<PD> pd(b->n_pairs);
  const size_t npx = size_t(b->W) * b->H;
  // state layout: per pair u, ua, ub (R2 * n) then ste, r (Real * n)
  size_t state_bytes = 0;
  std::vector<size_t> st_off(b->n_pairs);
  for (int p = 0; p < b->n_pairs; ++p) {
    st_off[p] = state_bytes;
    const size_t n = size_t(b->meshes[p]->h.n);
    state_bytes += (3 * n * sizeof(R2) + 2 * n * sizeof(Real) + 255) / 256 * 256;
  }
  if (b->forced_cs) {  // mrb_register_many
    b->state = kept_buffer(b->ctx, kKeptState, state_bytes);
    b->dense = kept_buffer(b->ctx, kKeptDense, 3 * npx * b->n_pairs * sizeof(Real));
    b->pairs_borrowed = true;
  } else {
    b->state = dalloc<char>(state_bytes);
    b->dense = dalloc<Real>(3 * npx * b->n_pairs);
  }
  b->state_bytes = state_bytes;
  int blk = 0, pblk = 0;
  std::vector<int> bp, pbp;
  const int pix_nblk = int((npx + kPixBlock - 1) / kPixBlock);
  pbp.reserve(size_t(b->n_pairs) * pix_nblk);  // 64 x 1024 entries at C4: bulk-filled
  for (int p = 0; p < b->n_pairs; ++p) {
    HostMesh& h = b->meshes[p]->h;
    DeviceMesh& dm = *h.dev;
    PD& d = pd[p];
    d.V = dm.V;
    d.nb_ptr = dm.nb_ptr;
    d.nb_idx = dm.nb_idx;
    if constexpr (sizeof(Real) == 8) {
      d.g_self = dm.g_self_d;
      d.g_nb = dm.g_nb_d;
      d.inv_val = dm.inv_val_d;
    } else {
      d.g_self = dm.g_self_f;
      d.g_nb = dm.g_nb_f;
      d.inv_val = dm.inv_val_f;
    }
    d.tri = dm.tri;
    d.tri_of = dm.pixel_maps.at(std::make_pair(b->W, b->H));
    d.perm = dm.perm;
    d.img = static_cast<const TapT*>(b->img) + size_t(p) * 2 * npx;
    const size_t n = size_t(h.n);
    char* base = static_cast<char*>(b->state) + st_off[p];
    d.u = reinterpret_cast<R2*>(base);
    d.ua = d.u + n;
    d.ub = d.ua + n;
    d.ste = reinterpret_cast<Real*>(d.ub + n);
    d.r = d.ste + n;
    d.trace = b->traces + size_t(p) * b->cfg.max_iterations;
    d.grad_out = nullptr;
    Real* dense = static_cast<Real*>(b->dense);
    d.ux = dense + (3 * size_t(p) + 0) * npx;
    d.uy = dense + (3 * size_t(p) + 1) * npx;
    d.warped = dense + (3 * size_t(p) + 2) * npx;
    d.u_out = b->u_out + b->node_off[p];
    d.W = b->W;
    d.H = b->H;
    d.n = int(n);
    d.blk_begin = blk;
    d.nblk = int((n + kNodeBlock - 1) / kNodeBlock);
    d.pix_blk_begin = pblk;
    d.pix_nblk = pix_nblk;
    bp.insert(bp.end(), size_t(d.nblk), p);
    pbp.insert(pbp.end(), size_t(pix_nblk), p);
    blk += d.nblk;
    pblk += pix_nblk;
  }
  b->n_node_blocks = blk;
  b->n_pix_blocks = pblk;
  cudaStream_t s = b->ctx->stream;
  b->pairs = aupload(b->ctx, pd.data(), pd.size());
  b->blk_pair = aupload(b->ctx, bp.data(), bp.size());
  b->pix_blk_pair = aupload(b->ctx, pbp.data(), pbp.size());
  b->partials = dalloc<double>(blk);
  b->pix_partials = dalloc<double2>(pblk);
  b->pairs_host.assign(reinterpret_cast<const unsigned char*>(pd.data()),
                       reinterpret_cast<const unsigned char*>(pd.data() + pd.size()));
}

template <typename InT, typename TapT>
void launch_interleave(mrb_batch* b) {
  const int npx = b->W * b->H;
  dim3 grid(std::min((npx + 255) / 256, 1024), b->n_pairs);
  k_interleave<InT, TapT><<<grid, 256, 0, b->ctx->stream>>>(
      reinterpret_cast<const InT* const*>(b->src_ptrs),
      reinterpret_cast<const InT* const*>(b->src_ptrs + b->n_pairs),
      reinterpret_cast<TapT* const*>(b->img_ptrs), npx);
}

struct KernelTimer {
  cudaStream_t s;
  std::vector<cudaEvent_t> ev;
  std::vector<int> kind;
  bool on = false;
  void mark(int k) {
    if (!on) return;
    cudaEvent_t e;
    ck(cudaEventCreate(&e));
    ck(cudaEventRecord(e, s));
    ev.push_back(e);
    kind.push_back(k);
  }
  ~KernelTimer() {
    for (auto e : ev) cudaEventDestroy(e);
  }
};

template <int NPT>
void launch_cluster_t(mrb_batch* b, int p0, int np, int CS, size_t smem) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(unsigned(np * CS));
  lc.blockDim = dim3(kClusterThreads);
  lc.dynamicSmemBytes = smem;
  lc.stream = b->lstream ? b->lstream : b->ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  ck(cudaLaunchKernelEx(&lc, k_cluster_register<NPT>,
                        static_cast<const ClusterPair*>(b->cpairs) + p0, b->st + p0,
                        int(b->cfg.max_iterations), double(b->cfg.energy_tolerance),
                        float(b->cfg.tau), float(b->cfg.lam), int(b->cfg.smoothing_passes)));
}

// A kernel's dynamic-smem limit only ever grows (per device and kernel), so
// every batch created so far can still launch.
template <typename K>
bool raise_smem_limit_of(K kern, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> cur;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  size_t& c = cur[std::make_pair(reinterpret_cast<const void*>(kern), dev)];
  if (smem <= c) return true;
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) !=
      cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  c = smem;
  return true;
}

template <int NPT>
bool raise_smem_limit(size_t smem) {
  return raise_smem_limit_of(k_cluster_register<NPT>, smem);
}

template <int NPT>
int cluster_occupancy(int CS, size_t smem) {
  auto kern = k_cluster_register<NPT>;
  if (!raise_smem_limit<NPT>(smem)) return 0;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(unsigned(CS));
  lc.blockDim = dim3(kClusterThreads);
  lc.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  int n = 0;
  const cudaError_t e = cudaOccupancyMaxActiveClusters(&n, kern, &lc);
  if (e != cudaSuccess) {
    if (std::getenv("MESHREG_B200_DEBUG"))
      std::fprintf(stderr, "meshreg_b200: cudaOccupancyMaxActiveClusters(%d,%d): %s\n", CS, NPT,
                   cudaGetErrorString(e));
    cudaGetLastError();
    return 0;
  }
  return n;
}

int cluster_occupancy_cs(int cs, int npt, size_t smem) {
  // the answer only depends on (cs, npt, smem): cached (queries are not free)
  static std::mutex mu;
  static std::map<std::tuple<int, int, size_t, int>, int> memo;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(cs, npt, smem, dev);
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
  }
  const int occ = npt == 2 ? cluster_occupancy<2>(cs, smem) : cluster_occupancy<1>(cs, smem);
  std::lock_guard<std::mutex> lock(mu);
  return memo[key] = occ;
}

template <int NPT>
void launch_grid_t(mrb_batch* b, int p) {
  cudaStream_t s = b->ctx->stream;
  // barrier counter, sticky gradient flags / partial counters start at zero
  // per pair; epoch-tagged exchange words too (a stale word of an earlier
  // launch must never carry a current epoch)
  ck(cudaMemsetAsync(b->xbar, 0, (1 + 3 * size_t(b->cluster_cs) * kFlagStride) * sizeof(unsigned),
                     s));
  if (b->grid_flags) ck(cudaMemsetAsync(b->xbuf, 0, b->xbytes, s));
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(unsigned(b->cluster_cs));
  lc.blockDim = dim3(kClusterThreads);
  lc.dynamicSmemBytes = b->cluster_smem;
  lc.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // co-residency for the grid barrier
  attr[0].val.cooperative = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  ck(cudaLaunchKernelEx(&lc,
                        !b->grid_flags   ? k_grid_register<NPT>
                        : b->pad_rowpair ? k_grid_flags<NPT, true>
                                         : k_grid_flags<NPT, false>,
                        static_cast<const ClusterPair*>(b->cpairs) + p, b->st + p,
                        int(b->cfg.max_iterations), double(b->cfg.energy_tolerance),
                        float(b->cfg.tau), float(b->cfg.lam), int(b->cfg.smoothing_passes)));
}

int64_t launch_grid(mrb_batch* b, int p0, int np) {
  for (int p = p0; p < p0 + np; ++p) {  // one whole-GPU launch per pair
    switch (b->cluster_npt) {
      case 1: launch_grid_t<1>(b, p); break;
      case 2: launch_grid_t<2>(b, p); break;
      case 4: launch_grid_t<4>(b, p); break;
      default: launch_grid_t<8>(b, p); break;
    }
  }
  return np;
}

template <int NPT>
int push_occupancy_t(int CS, size_t smem) {
  auto kern = k_cluster_push<NPT>;
  if (!raise_smem_limit_of(kern, smem)) return 0;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(unsigned(CS));
  lc.blockDim = dim3(kClusterThreads);
  lc.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &lc) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int push_occupancy(int cs, int npt, size_t smem) {
  return npt == 2 ? push_occupancy_t<2>(cs, smem) : push_occupancy_t<1>(cs, smem);
}

template <int NPT>
void launch_push_t(mrb_batch* b, int p0, int np, int CS, size_t smem) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(unsigned(np * CS));
  lc.blockDim = dim3(kClusterThreads);
  lc.dynamicSmemBytes = smem;
  lc.stream = b->lstream ? b->lstream : b->ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  ck(cudaLaunchKernelEx(&lc, k_cluster_push<NPT>,
                        static_cast<const ClusterPair*>(b->cpairs) + p0, b->st + p0,
                        int(b->cfg.max_iterations), double(b->cfg.energy_tolerance),
                        float(b->cfg.tau), float(b->cfg.lam), int(b->cfg.smoothing_passes)));
}

void launch_shape(mrb_batch* b, int p0, int np, int cs, int npt, bool push, size_t smem) {
  if (np <= 0) return;
  if (push) {
    if (npt == 2)
      launch_push_t<2>(b, p0, np, cs, smem);
    else
      launch_push_t<1>(b, p0, np, cs, smem);
  } else {
    if (npt == 2)
      launch_cluster_t<2>(b, p0, np, cs, smem);
    else
      launch_cluster_t<1>(b, p0, np, cs, smem);
  }
}

// pairs [p0, p0 + np): the batch shape, and the tail shape past tail_p0
int64_t launch_cluster(mrb_batch* b, int p0, int np) {
  if (b->grid_mode) return launch_grid(b, p0, np);
  const int p1 = p0 + np, split = std::min(std::max(b->tail_p0, p0), p1);
  launch_shape(b, p0, split - p0, b->cluster_cs, b->cluster_npt, b->push_mode,
               b->push_mode ? b->push_smem : b->cluster_smem);
  launch_shape(b, split, p1 - split, b->tail_cs, b->tail_npt, b->tail_push, b->tail_smem);
  return (split > p0) + (p1 > split);
}

// Deferred topologies (mrb_register_many): pack and copy, on `copy`, the
// meshes pairs [0, p1) need and make `s` wait for them.
void patch_descriptors(mrb_batch* b, int p0, int p1);

void flush_topo(mrb_batch* b, int p1, cudaStream_t copy, cudaStream_t s) {
  bool copied = false;
  const int pe = std::min(p1, b->planned_end);
  if (b->lazy_from < pe) {
    // plan the main-shape topologies of pairs [lazy_from, pe) now (this host
    // work overlaps the previous group's run), copy them and the patched
    // descriptors on `copy`
    const int cs = b->cluster_cs, npt = b->cluster_npt;
    std::vector<HostMesh*> todo;
    for (int p = b->lazy_from; p < pe; ++p) {
      HostMesh* h = &b->meshes[p]->h;
      const int chunk = int((h->n + cs - 1) / cs);
      if (!h->dev->topo.count(topo_key(cs, chunk, npt)) &&
          std::find(todo.begin(), todo.end(), h) == todo.end())
        todo.push_back(h);
    }
    if (!b->topo_ev) ck(cudaEventCreateWithFlags(&b->topo_ev, cudaEventDisableTiming));
    if (!todo.empty()) {
      b->lazy_ups.emplace_back(
          new TopoUpload(plan_cluster_topos(b->ctx, todo, cs, npt, 1, copy)));
      upload_cluster_topos(b->ctx, *b->lazy_ups.back(), 0, todo.size(), copy);
    }
    patch_descriptors(b, b->lazy_from, pe);
    ck(mrb_copy_async(static_cast<ClusterPair*>(b->cpairs) + b->lazy_from,
                      b->cp_pinned + b->lazy_from, sizeof(ClusterPair) * size_t(pe - b->lazy_from),
                      cudaMemcpyHostToDevice, copy));
    b->lazy_from = pe;
    copied = true;
  }
  if (!b->topo_up) {
    if (copied && copy != s) {
      ck(cudaEventRecord(b->topo_ev, copy));
      ck(cudaStreamWaitEvent(s, b->topo_ev, 0));
    }
    return;
  }
  size_t need = b->topo_done;
  for (int p = 0; p < p1; ++p) {
    auto it = b->topo_index.find(&b->meshes[p]->h);
    if (it != b->topo_index.end()) need = std::max(need, it->second + 1);
  }
  if (need <= b->topo_done && !copied) return;
  if (need > b->topo_done) upload_cluster_topos(b->ctx, *b->topo_up, b->topo_done, need, copy);
  b->topo_done = std::max(b->topo_done, need);
  if (copy != s) {
    if (!b->topo_ev) ck(cudaEventCreateWithFlags(&b->topo_ev, cudaEventDisableTiming));
    ck(cudaEventRecord(b->topo_ev, copy));
    ck(cudaStreamWaitEvent(s, b->topo_ev, 0));
  }
}

// Deferred tail-shape topologies: pack and copy on `copy` before the tail's
// launch and make `s` wait for them.
void flush_tail_topo(mrb_batch* b, cudaStream_t copy, cudaStream_t s) {
  if (!b->tail_up || b->tail_done) return;
  upload_cluster_topos(b->ctx, *b->tail_up, 0, b->tail_up->meshes.size(), copy);
  b->tail_done = true;
  if (copy != s) {
    if (!b->topo_ev) ck(cudaEventCreateWithFlags(&b->topo_ev, cudaEventDisableTiming));
    ck(cudaEventRecord(b->topo_ev, copy));
    ck(cudaStreamWaitEvent(s, b->topo_ev, 0));
  }
}

void setup_cluster64(mrb_batch* b);
void launch_cluster64(mrb_batch* b);

// fp64 batch k_cluster64 can run: every mesh fits 16 CTAs x 768 nodes with
// one-rings of <= kMaxDeg (MESHREG_B200_PATH=generic keeps the 3-kernel loop)
bool cluster64_candidate(const mrb_batch* b) {
  const char* env = std::getenv("MESHREG_B200_PATH");
  if (env && std::string(env) == "generic") return false;
  for (const mrb_mesh* m : b->meshes)
    if (m->h.n > 16 * kClusterThreads || m->h.max_deg > kMaxDeg) return false;
  return true;
}

template <typename TapT, typename Real>
int64_t enqueue_run(mrb_batch* b, KernelTimer* tm = nullptr) {
  KernelTimer dummy;
  if (!tm) tm = &dummy;
  using PD = PairDev<TapT, Real>;
  cudaStream_t s = b->ctx->stream;
  const PD* pairs = static_cast<const PD*>(b->pairs);
  int64_t launches = 0;
  if (b->cluster_cs) {
    if constexpr (std::is_same<TapT, float>::value && std::is_same<Real, float>::value) {
      // fast path: padded aligned copies straight from the planar inputs,
      // one persistent cluster launch for every iteration of every pair,
      // then the fused dense pass
      const size_t npad = size_t(b->W + 2) * (b->H + 2);
      auto pad = [&](int p0, int p1, cudaStream_t st_) {
        const dim3 grid(unsigned(std::min<size_t>((npad + 255) / 256, 1024)), unsigned(p1 - p0));
        const float* const* re = reinterpret_cast<const float* const*>(b->src_ptrs) + p0;
        const float* const* te =
            reinterpret_cast<const float* const*>(b->src_ptrs + b->n_pairs) + p0;
        const size_t per = size_t(b->pad_copies) * b->pad_plane;
        if (b->pad_rowpair)
          k_pad_planar_rp<<<grid, 256, 0, st_>>>(re, te, b->W, b->H, b->img_pad + p0 * per,
                                                 b->pad_pitch, b->pad_plane, per);
        else
          k_pad_planar4<<<grid, 256, 0, st_>>>(re, te, b->W, b->H, b->img_pad + p0 * per,
                                               b->pad_pitch, b->pad_plane, per);
        ++launches;
      };
      const bool grouped_run = b->groups.size() > 2 && tm == &dummy && b->runs == 0;
      // images per wave group (mrb_register_many): each group pads its own
      // pairs once their copy landed, so group 0 need not wait for the rest
      const bool group_pads = grouped_run && b->img_ev.size() + 1 == b->groups.size();
      if (!group_pads) {
        for (cudaEvent_t e : b->img_ev) ck(cudaStreamWaitEvent(s, e, 0));
        pad(0, b->n_pairs, s);
      }
      if (grouped_run) {
        // per wave group: loop + dense pass + MSD, then an event for the
        // group's device-to-host copies (mrb_batch_get_results)
        const PD* host = reinterpret_cast<const PD*>(b->pairs_host.data());
        const size_t ng = b->groups.size() - 1;
        // the last group is the tail wave (latency shape, a third of the
        // SMs): it runs on a side stream from the end of the previous group's
        // loop, beside that group's dense pass
        const bool tail_side = !b->grid_mode && ng >= 2 &&
                               b->groups[ng - 1] >= b->tail_p0 && b->tail_p0 < b->n_pairs;
        if (tail_side && !b->tail_stream) {
          b->tail_stream = side_stream(b->ctx, 1);
          ck(cudaEventCreateWithFlags(&b->tail_fork, cudaEventDisableTiming));
          ck(cudaEventCreateWithFlags(&b->tail_join, cudaEventDisableTiming));
        }
        auto dense_msd = [&](int p0, int p1, cudaStream_t st_) {
          if (b->pending_pm && b->pending_pm->done)  // rasters on the side stream
            ck(cudaStreamWaitEvent(st_, b->pending_pm->done, 0));
          const int blk0 = host[p0].pix_blk_begin;
          const int blk1 = p1 < b->n_pairs ? host[p1].pix_blk_begin : b->n_pix_blocks;
          k_dense_fast<<<blk1 - blk0, kPixBlock, 0, st_>>>(
              static_cast<const ClusterPair*>(b->cpairs), b->st, b->pix_blk_pair, b->pix_partials,
              blk0);
          k_msd_final<TapT, Real><<<p1 - p0, kPixBlock, 0, st_>>>(pairs + p0, b->st + p0,
                                                                 b->pix_partials);
          launches += 2;
        };
        if (!b->grp_stream) {
          b->grp_stream = side_stream(b->ctx, 0);
          ck(cudaEventCreateWithFlags(&b->grp_fork, cudaEventDisableTiming));
          ck(cudaEventCreateWithFlags(&b->grp_join, cudaEventDisableTiming));
        }
        ck(cudaEventRecord(b->grp_fork, s));  // descriptors (and unless group_pads, images) ready
        ck(cudaStreamWaitEvent(b->grp_stream, b->grp_fork, 0));
        const cudaStream_t gst[2] = {s, b->grp_stream};
        for (size_t g = 0; g < ng; ++g) {
          const int p0 = b->groups[g], p1 = b->groups[g + 1];
          if (tail_side && g == ng - 1) {  // launched beside group ng - 2's dense pass
            ck(cudaEventRecord(b->group_ev[g], b->tail_stream));
            continue;
          }
          // (grid mode: whole-GPU cooperative launches sharing one exchange
          // buffer must stay serial on one stream)
          const cudaStream_t gs = b->grid_mode ? s : gst[g & 1];
          if (group_pads) {
            ck(cudaStreamWaitEvent(gs, b->img_ev[g], 0));
            pad(p0, p1, gs);
          }
          // this group's topologies (host packing overlaps the previous group)
          flush_topo(b, p1, b->copy_stream, gs);
          if (p1 > b->tail_p0) flush_tail_topo(b, b->copy_stream, gs);
          if (std::getenv("MESHREG_B200_DEBUG")) {  // device timeline of the groups
            cudaEvent_t e;
            cudaEventCreate(&e);
            cudaEventRecord(e, gs);
            b->dbg_group_ev.push_back(e);
          }
          b->lstream = gs;
          launches += launch_cluster(b, p0, p1 - p0);
          b->lstream = nullptr;
          if (tail_side && g == ng - 2) {
            const int t0 = b->groups[ng - 1], t1 = b->groups[ng];
            ck(cudaEventRecord(b->tail_fork, gs));
            ck(cudaStreamWaitEvent(b->tail_stream, b->tail_fork, 0));
            if (group_pads) {
              ck(cudaStreamWaitEvent(b->tail_stream, b->img_ev[ng - 1], 0));
              pad(t0, t1, b->tail_stream);
            }
            flush_topo(b, t1, b->copy_stream, b->tail_stream);
            flush_tail_topo(b, b->copy_stream, b->tail_stream);
            b->lstream = b->tail_stream;
            launches += launch_cluster(b, t0, t1 - t0);
            b->lstream = nullptr;
            dense_msd(t0, t1, b->tail_stream);
            ck(cudaEventRecord(b->tail_join, b->tail_stream));
          }
          if (!b->grid_mode && b->ctx->fill_idle) {  // dense pass + MSD off the loop streams (see create_stream)
            const cudaStream_t ds = side_stream(b->ctx, 3);
            cudaEvent_t loop_done;
            ck(cudaEventCreateWithFlags(&loop_done, cudaEventDisableTiming));
            ck(cudaEventRecord(loop_done, gs));
            ck(cudaStreamWaitEvent(ds, loop_done, 0));
            cudaEventDestroy(loop_done);
            dense_msd(p0, p1, ds);
            ck(cudaEventRecord(b->group_ev[g], ds));
          } else {
            dense_msd(p0, p1, gs);
            ck(cudaEventRecord(b->group_ev[g], gs));
          }
        }
        // everything later on ctx->stream (results, sync) follows every group
        if (!b->grid_mode && b->ctx->fill_idle) {
          cudaEvent_t dense_done;
          ck(cudaEventCreateWithFlags(&dense_done, cudaEventDisableTiming));
          ck(cudaEventRecord(dense_done, side_stream(b->ctx, 3)));
          ck(cudaStreamWaitEvent(s, dense_done, 0));
          cudaEventDestroy(dense_done);
        }
        ck(cudaEventRecord(b->grp_join, b->grp_stream));
        ck(cudaStreamWaitEvent(s, b->grp_join, 0));
        if (tail_side) ck(cudaStreamWaitEvent(s, b->tail_join, 0));
        b->groups_recorded = true;
        ck(cudaGetLastError());
        return launches;
      }
      if (b->pending_pm && b->pending_pm->done)  // side-stream rasters (pixel maps)
        ck(cudaStreamWaitEvent(s, b->pending_pm->done, 0));
      flush_topo(b, b->n_pairs, s, s);  // deferred topologies not yet uploaded
      flush_tail_topo(b, s, s);
      if (tm == &dummy && !b->grid_mode && b->tail_p0 > 0 && b->tail_p0 < b->n_pairs) {
        // the tail wave holds a third of the SMs for ~1 ms after the main
        // launch: run it, and then its pairs' dense pass, on a side stream
        // while the main pairs' dense pass fills the idle SMs
        const PD* host = reinterpret_cast<const PD*>(b->pairs_host.data());
        const int tb = host[b->tail_p0].pix_blk_begin;
        if (!b->tail_stream) {
          b->tail_stream = side_stream(b->ctx, 1);
          ck(cudaEventCreateWithFlags(&b->tail_fork, cudaEventDisableTiming));
          ck(cudaEventCreateWithFlags(&b->tail_join, cudaEventDisableTiming));
        }
        launch_shape(b, 0, b->tail_p0, b->cluster_cs, b->cluster_npt, b->push_mode,
                     b->push_mode ? b->push_smem : b->cluster_smem);
        ck(cudaEventRecord(b->tail_fork, s));
        ck(cudaStreamWaitEvent(b->tail_stream, b->tail_fork, 0));
        b->lstream = b->tail_stream;
        launch_shape(b, b->tail_p0, b->n_pairs - b->tail_p0, b->tail_cs, b->tail_npt,
                     b->tail_push, b->tail_smem);
        b->lstream = nullptr;
        k_dense_fast<<<b->n_pix_blocks - tb, kPixBlock, 0, b->tail_stream>>>(
            static_cast<const ClusterPair*>(b->cpairs), b->st, b->pix_blk_pair, b->pix_partials,
            tb);
        ck(cudaEventRecord(b->tail_join, b->tail_stream));
        k_dense_fast<<<tb, kPixBlock, 0, s>>>(static_cast<const ClusterPair*>(b->cpairs), b->st,
                                             b->pix_blk_pair, b->pix_partials, 0);
        ck(cudaStreamWaitEvent(s, b->tail_join, 0));
        k_msd_final<TapT, Real><<<b->n_pairs, kPixBlock, 0, s>>>(pairs, b->st, b->pix_partials);
        launches += 5;
        ck(cudaGetLastError());
        return launches;
      }
      tm->mark(-1);
      launches += launch_cluster(b, 0, b->n_pairs);
      tm->mark(0);
      k_dense_fast<<<b->n_pix_blocks, kPixBlock, 0, s>>>(
          static_cast<const ClusterPair*>(b->cpairs), b->st, b->pix_blk_pair, b->pix_partials, 0);
      tm->mark(3);
      k_msd_final<TapT, Real><<<b->n_pairs, kPixBlock, 0, s>>>(pairs, b->st, b->pix_partials);
      launches += 2;
      ck(cudaGetLastError());
      return launches;
    }
  }
  if (b->in_dtype == MRB_F64)
    launch_interleave<double, TapT>(b);
  else
    launch_interleave<float, TapT>(b);
  ++launches;
  k_reset_status<<<(b->n_pairs + 127) / 128, 128, 0, s>>>(b->st, b->n_pairs,
                                                         b->cfg.max_iterations);
  ++launches;
  const int nb = b->n_node_blocks;
  const double tol = b->cfg.energy_tolerance;
  const Real tau = Real(b->cfg.tau), lam = Real(b->cfg.lam);
  const int passes = b->cfg.smoothing_passes;
  tm->mark(-1);
  if (b->c64_cs) {  // fp64: the whole descent loop in one persistent cluster launch
    const size_t padn = size_t(b->W + 2) * (b->H + 2);
    const dim3 pg(unsigned(std::min<size_t>((padn + 255) / 256, 1024)), b->n_pairs);
    if (b->tap_d)
      k_pad_pair64<double><<<pg, 256, 0, s>>>(static_cast<const ClusterPair64*>(b->c64_pairs));
    else
      k_pad_pair64<float><<<pg, 256, 0, s>>>(static_cast<const ClusterPair64*>(b->c64_pairs));
    ++launches;
    if (b->img_pad) {  // the fp32 shifted copies for interior windows
      k_pad_planar4<<<pg, 256, 0, s>>>(reinterpret_cast<const float* const*>(b->src_ptrs),
                                       reinterpret_cast<const float* const*>(b->src_ptrs +
                                                                             b->n_pairs),
                                       b->W, b->H, b->img_pad, b->pad_pitch, b->pad_plane,
                                       4 * b->pad_plane);
      ++launches;
    }
    launch_cluster64(b);
    tm->mark(0);
    ++launches;
  }
  for (int k = 0; k < (b->c64_cs ? 0 : b->cfg.max_iterations); ++k) {
    k_sample<TapT, Real><<<nb, kNodeBlock, 0, s>>>(pairs, b->st, b->blk_pair, b->partials, k, tol);
    tm->mark(0);
    k_grad<TapT, Real><<<nb, kNodeBlock, 0, s>>>(pairs, b->st, b->blk_pair, k, tau, passes);
    tm->mark(1);
    launches += 2;
    for (int q = 0; q < passes; ++q) {
      k_smooth<TapT, Real><<<nb, kNodeBlock, 0, s>>>(pairs, b->st, b->blk_pair, k, lam, q, passes);
      tm->mark(2);
      ++launches;
    }
  }
  k_dense<TapT, Real><<<b->n_pix_blocks, kPixBlock, 0, s>>>(pairs, b->st, b->pix_blk_pair,
                                                            b->pix_partials);
  tm->mark(3);
  k_msd_final<TapT, Real><<<b->n_pairs, kPixBlock, 0, s>>>(pairs, b->st, b->pix_partials);
  k_unpermute<TapT, Real><<<nb, kNodeBlock, 0, s>>>(pairs, b->blk_pair);
  launches += 3;
  ck(cudaGetLastError());
  return launches;
}

template <typename TapT, typename Real>
void enqueue_zero_u(mrb_batch* b) {
  // u = 0 for every pair (solver.py:168): u is the first slab of each pair's
  // state (layout of build_pairs); the rest is scratch, so one memset of the
  // whole state (one API call instead of one per pair)
  ck(cudaMemsetAsync(b->state, 0, b->state_bytes, b->ctx->stream));
}

template <typename TapT, typename Real>
int64_t enqueue_all(mrb_batch* b, KernelTimer* tm) {
  enqueue_zero_u<TapT, Real>(b);
  return enqueue_run<TapT, Real>(b, tm);
}

int64_t dispatch_enqueue(mrb_batch* b, KernelTimer* tm = nullptr) {
  if (b->tap_d) return enqueue_all<double, double>(b, tm);
  if (b->real_d) return enqueue_all<float, double>(b, tm);
  return enqueue_all<float, float>(b, tm);
}

int64_t launches_per_run(const mrb_batch* b) {
  if (b->grid_mode) return 3 + b->n_pairs;  // pad, one grid loop per pair, dense, msd
  if (b->cluster_cs) return 4 + (b->tail_p0 < b->n_pairs);  // pad, loop(s), dense, msd
  if (b->c64_cs) return b->img_pad ? 8 : 7;  // interleave, reset, pad(s), loop, dense, msd, unpermute
  return 2 + int64_t(b->cfg.max_iterations) * (2 + b->cfg.smoothing_passes) + 3;
}

// Choose the cluster fast path when it applies: fp32, every pair fits one
// cluster of <= 16 CTAs x 768 nodes, one-rings of <= kMaxDeg entries.
// Cluster shape (CS CTAs per pair, NPT nodes per thread) for a batch of
// n_pairs pairs whose largest mesh is `big`.  Cost model = waves x nodes per
// CTA = ceil(P / max active clusters(CS)) * ceil(n / CS), evaluated with the
// largest mesh's topology; the occupancy API sees the GPC structure (e.g.
// clusters of 9 pack two per 18/19-SM GPC where clusters of 8 leave SMs
// idle).  The decision is cached per (shape, device).  Returns false when no
// candidate fits; *occ = active clusters of the choice (pairs per wave).
bool choose_cluster_shape(mrb_ctx* ctx, HostMesh& big, int n_pairs, bool two_u, int* cs_out,
                          int* npt_out, int* occ_out, int npt_pref = 0) {
  const bool dbg = std::getenv("MESHREG_B200_DEBUG") != nullptr;
  const int64_t nmax = big.n;
  // latency mode (few pairs): one node per thread, more CTAs per pair;
  // throughput mode: two nodes per thread, fewer CTAs per pair
  int npt = npt_pref ? npt_pref : (n_pairs >= 4 ? 2 : 1);
  static std::mutex cache_mu;
  static std::map<std::tuple<int, int, int64_t, bool, int>, std::tuple<int, int, int>> cache;
  const auto key = std::make_tuple(npt, n_pairs, int64_t(nmax), two_u, ctx->device);
  {
    std::lock_guard<std::mutex> lock(cache_mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      std::tie(*cs_out, *npt_out, *occ_out) = it->second;
      return true;
    }
  }
  for (; npt >= 1; --npt) {
    const int cap = kClusterThreads * npt;
    const int cs_min = int((nmax + cap - 1) / cap);
    if (cs_min > 16) continue;
    double best = 1e300;
    int best_cs = 0, best_occ = 0;
    for (int cs = cs_min; cs <= 16; ++cs) {
      const int chunk = int((big.n + cs - 1) / cs);
      const DeviceMesh::Topo& t = ensure_cluster_topo(ctx, big, cs, chunk, npt);
      const size_t smem =
          cluster_dyn_smem(npt, t.topo_stride, t.slices, t.halo_stride, two_u) + 4096;
      const int occ = cluster_occupancy_cs(cs, npt, smem);
      if (occ < 1) continue;
      const double cost = double((n_pairs + occ - 1) / occ) * double((nmax + cs - 1) / cs);
      if (dbg)
        std::fprintf(stderr,
                     "meshreg_b200: candidate cluster %d x %d nodes/thread: %zu B smem, "
                     "%d active clusters, cost %.0f\n",
                     cs, npt, smem, occ, cost);
      if (cost < best) {
        best = cost;
        best_cs = cs;
        best_occ = occ;
      }
    }
    if (best_cs) {
      *cs_out = best_cs;
      *npt_out = npt;
      *occ_out = best_occ;
      std::lock_guard<std::mutex> lock(cache_mu);
      cache[key] = std::make_tuple(best_cs, npt, best_occ);
      return true;
    }
  }
  return false;
}

// SMs of the current device (whole-GPU grid size of k_grid_register)
int device_sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return std::max(n, 1);
}

size_t device_l2_bytes() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrL2CacheSize, dev);
  return size_t(std::max(n, 1));
}

constexpr int kGridMaxNpt = 8;
// A single pair with at least this many nodes runs faster on the whole-GPU
// grid than on one 16-CTA cluster (measured: C2, 12k nodes, 0.79 vs 0.98 ms;
// C1, 3k nodes, 0.43 vs 0.28 ms).
constexpr int64_t kGridSinglePairNodes = 6000;

// Fast-path mode of a batch: 1 = thread-block cluster per pair (every mesh
// fits 16 CTAs x 768 x 2 nodes), 2 = whole-GPU grid per pair (larger meshes,
// up to SMs x 768 x 8 nodes, and a single pair of >= kGridSinglePairNodes),
// 0 = generic path (*why says why).  Both fast modes need fp32 state and
// images and one-rings within kMaxDeg.  MESHREG_B200_PATH=cluster|grid|generic
// forces a mode.
int fast_mode(bool real_d, bool tap_d, int in_dtype, const std::vector<mrb_mesh*>& meshes,
              const char** why) {
  const char* env = std::getenv("MESHREG_B200_PATH");
  const std::string path = env ? env : "";
  *why = nullptr;
  if (path == "generic") return (*why = "MESHREG_B200_PATH=generic"), 0;
  if (real_d || tap_d) return (*why = "fp64 precision"), 0;
  if (in_dtype != MRB_F32) return (*why = "fp64 image storage"), 0;
  int64_t nmax = 0;
  for (mrb_mesh* m : meshes) {
    nmax = std::max<int64_t>(nmax, m->h.n);
    if (m->h.max_deg > kMaxDeg) return (*why = "one-ring larger than kMaxDeg"), 0;
  }
  const bool single_big = meshes.size() == 1 && nmax >= kGridSinglePairNodes;
  if (path == "cluster" || (path != "grid" && !single_big))
    if (nmax <= 16 * 2 * kClusterThreads) return 1;
  if (nmax <= int64_t(device_sms()) * kClusterThreads * kGridMaxNpt) return 2;
  return (*why = "mesh larger than the whole-GPU grid holds"), 0;
}

const char* cluster_ineligible(bool real_d, bool tap_d, int in_dtype,
                               const std::vector<mrb_mesh*>& meshes) {
  const char* why = nullptr;
  return fast_mode(real_d, tap_d, in_dtype, meshes, &why) == 1
             ? nullptr
             : (why ? why : "mesh larger than one cluster");
}

// grid shape for the largest mesh: CS = SMs, NPT = smallest of 1/2/4/8 with
// CS * 768 * NPT >= n
void grid_shape(int64_t nmax, int* cs, int* npt) {
  *cs = device_sms();
  const int64_t per = (nmax + *cs - 1) / *cs;
  *npt = 1;
  while (int64_t(*npt) * kClusterThreads < per) *npt *= 2;
}

size_t grid_dyn_smem(int npt, int halo_stride, bool two_u, bool flags = false) {
  const size_t slots = size_t(kClusterThreads) * npt, X = slots + halo_stride;
  // k_grid_flags adds u_save (float2) + residual (float) per slot
  return X * 4 + 8 + X * 8 * (two_u ? 2 : 1) + size_t(halo_stride) * 4 + 64 +
         (flags && npt >= 8 ? slots * 12 + 8 : 0);
}

// exports[src][slot >> 5] |= bit: slots some other CTA's halo reads
__global__ void k_mark_exports(const uint32_t* __restrict__ halo, const int* __restrict__ n_halo,
                               int hs, int cs, int words, uint32_t* __restrict__ exports) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cs * hs; i += gridDim.x * blockDim.x) {
    const int r = i / hs, h = i - r * hs;
    if (h >= __ldg(n_halo + r)) continue;
    const uint32_t c = __ldg(halo + i);
    const uint32_t slot = c & 0xffffu;
    atomicOr(exports + size_t(c >> 16) * words + (slot >> 5), 1u << (slot & 31));
  }
}

void build_fast_descriptors(mrb_batch* b);
void setup_grid_path(mrb_batch* b, int64_t nmax);
void setup_tail(mrb_batch* b, size_t main_smem);

void setup_cluster_path(mrb_batch* b) {
  b->cluster_cs = 0;
  const bool dbg = std::getenv("MESHREG_B200_DEBUG") != nullptr;
  auto why = [&](const char* m) {
    if (dbg) std::fprintf(stderr, "meshreg_b200: generic path (%s)\n", m);
  };
  auto t0 = std::chrono::steady_clock::now();
  auto tick = [&](const char* what) {
    if (!dbg) return;
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "meshreg_b200:   cluster setup %-18s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  const char* reason = nullptr;
  const int mode = fast_mode(b->real_d, b->tap_d, b->in_dtype, b->meshes, &reason);
  if (mode == 0) return why(reason);
  const bool two_u = b->cfg.smoothing_passes >= 2;
  mrb_mesh* big = *std::max_element(b->meshes.begin(), b->meshes.end(),
                                    [](mrb_mesh* x, mrb_mesh* y) { return x->h.n < y->h.n; });
  int cs = 0, npt = 0, occ = 0;
  if (mode == 2) {
    setup_grid_path(b, big->h.n);
    if (!b->cluster_cs) return why("grid kernel does not fit");
    return;
  }
  if (b->forced_cs) {  // shape decided for the whole queue (mrb_register_many)
    cs = b->forced_cs;
    npt = b->forced_npt;
  } else if (!choose_cluster_shape(b->ctx, big->h, b->n_pairs, two_u, &cs, &npt, &occ)) {
    return why("no cluster configuration fits");
  }
  // pairs past planned_end (the expected tail wave of a deferred batch) have
  // no throughput-shape topology unless setup_tail turns the tail down
  const int main_end = std::min(b->n_pairs, b->planned_end);
  // pairs [lazy_from, main_end) are planned in the run (mrb_register_many)
  const int plan_end = std::min(main_end, b->lazy_from);
  {  // per-mesh topologies: host thread pool + pinned staged upload
    std::vector<HostMesh*> hm;
    for (int p = 0; p < plan_end; ++p) hm.push_back(&b->meshes[p]->h);
    ensure_cluster_topos(b->ctx, hm, cs, npt);
  }
  tick("topologies");
  auto main_smem = [&](int p0, int p1, size_t smem) {
    for (int p = p0; p < p1; ++p) {
      HostMesh& h = b->meshes[p]->h;
      const int chunk = int((h.n + cs - 1) / cs);
      const DeviceMesh::Topo& t = ensure_cluster_topo(b->ctx, h, cs, chunk, npt);
      smem = std::max(smem, cluster_dyn_smem(npt, t.topo_stride, t.slices, t.halo_stride, two_u));
    }
    return smem;
  };
  size_t smem = main_smem(0, plan_end, 0);
  if (cluster_occupancy_cs(cs, npt, smem) < 1) return why("no cluster configuration fits");
  b->cluster_cs = cs;
  b->cluster_npt = npt;
  b->cluster_smem = smem;
  // Push exchange whenever it fits (smoothing_passes <= 1, send lists, no
  // occupancy loss): no cluster barrier inside the loop.  Latency mode
  // measured C1 -25%, C2 -18% time; throughput mode with the paired SELL
  // gathers C4 6.90 -> 6.27 ms (before them the pull kernel was faster there:
  // 8.4 vs 9.5 ms).  MESHREG_B200_EXCHANGE=push|pull overrides.
  const char* xenv = std::getenv("MESHREG_B200_EXCHANGE");
  const bool want_push = xenv ? std::string(xenv) == "push" : true;
  if (b->cfg.smoothing_passes <= 1 && want_push) {
    size_t ps = 0;
    bool lists = true;
    // the main shape's pairs only: the expected tail's pairs have no topology
    // of this shape (setup_tail decides them; planning one here would cost a
    // synchronous host plan + upload per tail mesh)
    for (int p = 0; p < plan_end; ++p) {
      HostMesh& h = b->meshes[p]->h;
      const int chunk = int((h.n + cs - 1) / cs);
      const DeviceMesh::Topo& t = ensure_cluster_topo(b->ctx, h, cs, chunk, npt);
      lists = lists && t.send_stride > 0;
      ps = std::max(ps, push_dyn_smem(npt, t.topo_stride, t.slices, t.halo_stride,
                                      t.send_stride));
    }
    if (lists && push_occupancy(cs, npt, ps) >= cluster_occupancy_cs(cs, npt, smem)) {
      b->push_mode = true;
      b->push_smem = ps;
    }
  }
  tick("shape + exchange");
  if (dbg)
    std::fprintf(stderr, "meshreg_b200: cluster %d CTAs x %d nodes/thread, %zu B smem, %s exchange\n",
                 cs, npt, b->push_mode ? b->push_smem : smem, b->push_mode ? "push" : "pull");
  setup_tail(b, smem);
  tick("tail");
  if (b->tail_p0 > main_end && main_end < b->n_pairs) {
    // no tail after all: the remaining pairs need the main shape (staging
    // slot 2, slot 1 still backs the deferred groups)
    std::vector<HostMesh*> rest;
    for (int p = main_end; p < b->n_pairs; ++p) rest.push_back(&b->meshes[p]->h);
    ensure_cluster_topos(b->ctx, rest, cs, npt, 2);
    b->cluster_smem = smem = main_smem(main_end, b->n_pairs, smem);
    if (cluster_occupancy_cs(cs, npt, smem) < 1) {
      b->cluster_cs = 0;
      return why("no cluster configuration fits");
    }
  }
  build_fast_descriptors(b);
  tick("descriptors");
}

// Tail split of a throughput-mode batch (see mrb_batch::tail_p0): with W
// clusters per wave and r = P mod W > 0 pairs left for the last wave, run
// those r pairs in the latency shape when it holds all r in one wave
// (measured C4: 60 pairs 6.93 ms + 4 pairs 1.07 ms vs 8.41 ms for 64).
void setup_tail(mrb_batch* b, size_t main_smem) {
  b->tail_p0 = 1 << 30;
  if (b->cluster_npt != 2 || std::getenv("MESHREG_B200_NO_TAIL")) return;
  const int W = cluster_occupancy_cs(b->cluster_cs, b->cluster_npt, main_smem);
  const int P = b->n_pairs;
  if (W < 1 || P <= W || P % W == 0) return;
  const int r = P % W, p0 = P - r;
  std::vector<mrb_mesh*> tm(b->meshes.begin() + p0, b->meshes.end());
  mrb_mesh* big = *std::max_element(tm.begin(), tm.end(),
                                    [](mrb_mesh* x, mrb_mesh* y) { return x->h.n < y->h.n; });
  const bool two_u = b->cfg.smoothing_passes >= 2;
  int cs = 0, npt = 0, occ = 0;
  if (!choose_cluster_shape(b->ctx, big->h, r, two_u, &cs, &npt, &occ, 1) || npt != 1 || occ < r)
    return;
  std::vector<HostMesh*> hm;
  for (mrb_mesh* m : tm) hm.push_back(&m->h);
  // own staging slot: slot 1 may still hold deferred wave-group topologies.
  // With deferred topologies (mrb_register_many) only plan now; the data is
  // packed and copied just before the tail's launch (flush_tail_topo).
  if (b->topo_up) {
    std::vector<HostMesh*> todo;
    for (HostMesh* h : hm) {
      const int chunk = int((h->n + cs - 1) / cs);
      if (!h->dev->topo.count(topo_key(cs, chunk, npt)) &&
          std::find(todo.begin(), todo.end(), h) == todo.end())
        todo.push_back(h);
    }
    if (!todo.empty()) b->tail_up.reset(new TopoUpload(plan_cluster_topos(b->ctx, todo, cs, npt, 2)));
  } else {
    ensure_cluster_topos(b->ctx, hm, cs, npt, 2);
  }
  size_t smem = 0, ps = 0;
  bool lists = true;
  for (mrb_mesh* m : tm) {
    const int chunk = int((m->h.n + cs - 1) / cs);
    const DeviceMesh::Topo& t = ensure_cluster_topo(b->ctx, m->h, cs, chunk, npt);
    smem = std::max(smem, cluster_dyn_smem(npt, t.topo_stride, t.slices, t.halo_stride, two_u));
    ps = std::max(ps, push_dyn_smem(npt, t.topo_stride, t.slices, t.halo_stride, t.send_stride));
    lists = lists && t.send_stride > 0;
  }
  if (cluster_occupancy_cs(cs, npt, smem) < r) return;
  const char* xenv = std::getenv("MESHREG_B200_EXCHANGE");
  const bool want_push = !(xenv && std::string(xenv) == "pull") && b->cfg.smoothing_passes <= 1;
  b->tail_push = want_push && lists && push_occupancy(cs, npt, ps) >= r;
  b->tail_cs = cs;
  b->tail_npt = npt;
  b->tail_smem = b->tail_push ? ps : smem;
  b->tail_p0 = p0;
  if (std::getenv("MESHREG_B200_DEBUG"))
    std::fprintf(stderr, "meshreg_b200: tail of %d pairs: cluster %d CTAs x %d nodes/thread, %s\n",
                 r, cs, npt, b->tail_push ? "push" : "pull");
}

void set_topology(ClusterPair& c, const DeviceMesh::Topo& t) {
  c.codes = t.codes;
  c.g = t.g;
  c.slice_off = t.slice_off;
  c.halo = t.halo;
  c.n_halo = t.n_halo;
  c.halo_stride = t.halo_stride;
  c.deg = t.deg;
  c.send = t.send;
  c.n_send = t.n_send;
  c.send_stride = t.send_stride;
  c.topo_stride = t.topo_stride;
  c.slices = t.slices;
}

// ClusterPair descriptors + padded image copies of a fast-path batch
void build_fast_descriptors(mrb_batch* b) {
  const int cs = b->cluster_cs;
  b->pad_pitch = (b->W + 5 + 3) / 4 * 4;
  b->pad_plane = size_t(b->H + 2) * b->pad_pitch;
  // taps evict_first when the four image copies exceed half of L2 (C5); the
  // whole-GPU grid path then streams the taps from DRAM and reads them in the
  // row-pair layout (one 64-byte fetch per two tap rows instead of one per
  // row)
  b->tap_evict_first = 4 * b->pad_plane * sizeof(float2) > device_l2_bytes() / 2;
  b->pad_rowpair = b->grid_mode && b->grid_flags && b->tap_evict_first;
  if (b->pad_rowpair) {
    b->pad_copies = 8;
    b->pad_plane = size_t((b->H + 2) / 2 + 1) * 2 * b->pad_pitch;
  }
  // columns of a copy that the pad kernel does not write are never read
  {
    const size_t need = size_t(b->pad_copies) * b->pad_plane * b->n_pairs;
    if (b->forced_cs) {  // mrb_register_many: its batches on a context run in turn
      b->img_pad = static_cast<float2*>(kept_buffer(b->ctx, kKeptPad, need * sizeof(float2)));
      b->img_pad_borrowed = true;
    } else {
      b->img_pad = dalloc<float2>(need);
    }
  }
  const PairDev<float, float>* host =
      reinterpret_cast<const PairDev<float, float>*>(b->pairs_host.data());
  std::vector<ClusterPair> cp(b->n_pairs);
  const DeviceMesh::Topo none{};
  for (int p = 0; p < b->n_pairs; ++p) {
    HostMesh& h = b->meshes[p]->h;
    const bool tail = p >= b->tail_p0;
    const int pcs = tail ? b->tail_cs : cs, pnpt = tail ? b->tail_npt : b->cluster_npt;
    const int chunk = int((h.n + pcs - 1) / pcs);
    // pairs planned lazily in the run get their topology fields then
    // (patch_descriptors)
    const bool lazy = !tail && p >= b->lazy_from && p < b->planned_end;
    const DeviceMesh::Topo& t = lazy ? none : ensure_cluster_topo(b->ctx, h, pcs, chunk, pnpt);
    ClusterPair& c = cp[p];
    c.V = h.dev->V;
    c.g_self = h.dev->g_self_f;
    c.inv_val = h.dev->inv_val_f;
    set_topology(c, t);
    c.img4 = b->img_pad + size_t(b->pad_copies) * b->pad_plane * p;
    c.rowpair = b->pad_rowpair;
    c.tri_of = host[p].tri_of;
    c.tri = host[p].tri;
    c.ux = host[p].ux;
    c.uy = host[p].uy;
    c.warped = host[p].warped;
    c.pix_blk_begin = host[p].pix_blk_begin;
    c.u = host[p].u;
    c.u_out = host[p].u_out;
    c.perm = h.dev->perm;
    c.trace = host[p].trace;
    c.prof = nullptr;
    if (std::getenv("MESHREG_B200_PROFILE_PHASES")) {
      if (!b->phase_prof) {
        const size_t cnt = size_t(b->n_pairs) * cs * 8 * 16;
        if (std::string(std::getenv("MESHREG_B200_PROFILE_PHASES")) == "mapped") {
          // debug: host-mapped, readable while the kernel runs (progress of a hang)
          ck(cudaHostAlloc(reinterpret_cast<void**>(&b->prof_host), cnt * sizeof(long long),
                           cudaHostAllocMapped));
          std::memset(b->prof_host, 0xff, cnt * sizeof(long long));
          ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&b->phase_prof), b->prof_host, 0));
        } else {
          b->phase_prof = dalloc<long long>(cnt);
          ck(cudaMemset(b->phase_prof, 0, cnt * sizeof(long long)));
        }
      }
      c.prof = b->phase_prof + size_t(p) * cs * 8 * 16;
    }
    c.n = int(h.n);
    c.chunk = chunk;
    c.W = b->W;
    c.H = b->H;
    c.pitch = b->pad_pitch;
    c.plane = int(b->pad_plane);
    c.xg_s = nullptr;
    c.xg_u = nullptr;
    c.wpart = nullptr;
    c.gbad = nullptr;
    c.bar = nullptr;
    c.flags = nullptr;
    c.exports = nullptr;
    c.tap_evict_first = b->tap_evict_first;
    if (b->grid_mode && b->grid_flags && !b->xexports) {
      const int words = kClusterThreads * b->cluster_npt / 32;
      b->xexports = dalloc<uint32_t>(size_t(b->n_pairs) * cs * words);
      ck(cudaMemsetAsync(b->xexports, 0, sizeof(uint32_t) * b->n_pairs * cs * words,
                         b->ctx->stream));
    }
    if (b->grid_mode && b->grid_flags) {
      const int words = kClusterThreads * b->cluster_npt / 32;
      k_mark_exports<<<std::max(1, std::min(1024, (cs * t.halo_stride + 255) / 256)), 256, 0,
                       b->ctx->stream>>>(t.halo, t.n_halo, t.halo_stride, cs, words,
                                         b->xexports + size_t(p) * cs * words);
      ck(cudaGetLastError());
    }
    if (b->grid_mode) {  // exchange buffers shared by the pairs (launched in turn)
      const size_t slots = size_t(cs) * kClusterThreads * b->cluster_npt;
      char* x = static_cast<char*>(b->xbuf);
      c.xg_s = reinterpret_cast<float*>(x);
      c.xg_u = reinterpret_cast<float2*>(x + (2 * slots * 8 + 255) / 256 * 256);
      c.wpart = reinterpret_cast<double*>(reinterpret_cast<char*>(c.xg_u) +
                                          (2 * slots * 16 + 255) / 256 * 256);
      c.bar = b->xbar;
      if (b->grid_flags) {
        // export bitmap of this pair's topology (built below, once per batch)
        const int words = kClusterThreads * b->cluster_npt / 32;
        // publish only exported slots at NPT = 8 (C5: 2% faster); smaller
        // NPT publishes every slot (measured faster, C2/C3)
        const bool sel = b->cluster_npt >= 8;
        c.exports = sel ? b->xexports + size_t(p) * cs * words : nullptr;
        c.flags = b->xbar + 1;
        c.gbad = reinterpret_cast<int*>(b->xbar + 1 + 3 * size_t(cs) * kFlagStride);
      } else {
        c.gbad = reinterpret_cast<int*>(b->xbar + 1);
      }
    }
  }
  b->cpairs = aupload(b->ctx, cp.data(), cp.size());
  if (b->lazy_from < std::min(b->planned_end, b->n_pairs)) {
    b->cp_host = cp;
    ck(cudaHostAlloc(reinterpret_cast<void**>(&b->cp_pinned), sizeof(ClusterPair) * cp.size(),
                     cudaHostAllocDefault));
  }
}

// Topology fields of the lazily planned pairs [p0, p1) (main shape), into
// the pinned descriptor copy flush_topo uploads; the launch's dynamic shared
// memory grows to what they need.
void patch_descriptors(mrb_batch* b, int p0, int p1) {
  const int cs = b->cluster_cs, npt = b->cluster_npt;
  const bool two_u = b->cfg.smoothing_passes >= 2;
  for (int p = p0; p < p1; ++p) {
    HostMesh& h = b->meshes[p]->h;
    const DeviceMesh::Topo& t = ensure_cluster_topo(b->ctx, h, cs, int((h.n + cs - 1) / cs), npt);
    set_topology(b->cp_host[p], t);
    b->cp_pinned[p] = b->cp_host[p];
    const size_t sm = cluster_dyn_smem(npt, t.topo_stride, t.slices, t.halo_stride, two_u);
    if (sm > b->cluster_smem) {
      b->cluster_smem = sm;
      cluster_occupancy_cs(cs, npt, sm);  // raises the kernel's smem limit
    }
    if (b->push_mode) {
      const size_t ps =
          push_dyn_smem(npt, t.topo_stride, t.slices, t.halo_stride, t.send_stride);
      if (ps > b->push_smem) {
        b->push_smem = ps;
        push_occupancy(cs, npt, ps);
      }
    }
  }
}

// Whole-GPU grid path (meshes larger than one cluster): CS = SMs CTAs per
// pair, NPT nodes per thread, topology read from global memory.
void setup_grid_path(mrb_batch* b, int64_t nmax) {
  int cs = 0, npt = 0;
  grid_shape(nmax, &cs, &npt);
  std::vector<HostMesh*> hm;
  for (mrb_mesh* m : b->meshes) hm.push_back(&m->h);
  ensure_cluster_topos(b->ctx, hm, cs, npt);
  int hs = 0;
  for (mrb_mesh* m : b->meshes) {
    const int chunk = int((m->h.n + cs - 1) / cs);
    hs = std::max(hs, ensure_cluster_topo(b->ctx, m->h, cs, chunk, npt).halo_stride);
  }
  size_t smem = grid_dyn_smem(npt, hs, b->cfg.smoothing_passes >= 2, true);
  auto fit = [&](auto kern) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) !=
        cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kClusterThreads, smem) !=
        cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    return per_sm;
  };
  // epoch-tagged exchange (no grid barrier) for at most one smoothing pass
  bool flags = b->cfg.smoothing_passes <= 1;
  int per_sm = 0;
  auto fit2 = [&](auto k1, auto k2) { return std::min(fit(k1), fit(k2)); };  // both tap layouts
  if (flags)
    per_sm = npt == 1   ? fit2(k_grid_flags<1, false>, k_grid_flags<1, true>)
             : npt == 2 ? fit2(k_grid_flags<2, false>, k_grid_flags<2, true>)
             : npt == 4 ? fit2(k_grid_flags<4, false>, k_grid_flags<4, true>)
                        : fit2(k_grid_flags<8, false>, k_grid_flags<8, true>);
  if (per_sm < 1) {
    flags = false;
    smem = grid_dyn_smem(npt, hs, b->cfg.smoothing_passes >= 2, false);
    per_sm = npt == 1 ? fit(k_grid_register<1>) : npt == 2 ? fit(k_grid_register<2>)
             : npt == 4 ? fit(k_grid_register<4>) : fit(k_grid_register<8>);
  }
  if (per_sm < 1) return;
  b->grid_mode = true;
  b->grid_flags = flags;
  b->cluster_cs = cs;
  b->cluster_npt = npt;
  b->cluster_smem = smem;
  // exchange arrays: s_te [2][slots] x 8 B (epoch-tagged words; the barrier
  // kernel uses floats), u [2][slots] x 16 B (tagged x, y; barrier kernel:
  // u0/u1 float2), energy partials [4][CS]; xbar: barrier counter, the
  // partial counters (one line each) and gradient flags [4][CS]
  const size_t slots = size_t(cs) * kClusterThreads * npt;
  b->xbytes = (2 * slots * 8 + 255) / 256 * 256 + (2 * slots * 16 + 255) / 256 * 256;
  b->xbuf = dalloc<char>(b->xbytes + size_t(4) * cs * kWarps * 8);
  b->xbar = dalloc<unsigned>(1 + 3 * size_t(cs) * kFlagStride + 4 * size_t(cs));
  if (std::getenv("MESHREG_B200_DEBUG"))
    std::fprintf(stderr, "meshreg_b200: grid %d CTAs x %d nodes/thread, %zu B smem, %s\n", cs,
                 npt, smem, flags ? "epoch-tagged exchange" : "grid barriers");
  build_fast_descriptors(b);
}

// src_ptrs[p] = re + p * stride, src_ptrs[n + p] = te + p * stride
__global__ void k_fill_ptrs(void** __restrict__ out, const char* re, const char* te,
                            size_t stride, int n) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  out[p] = const_cast<char*>(re + size_t(p) * stride);
  out[n + p] = const_cast<char*>(te + size_t(p) * stride);
}

template <typename From, typename To>
__global__ void k_convert(const From* __restrict__ a, To* __restrict__ o, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    o[i] = To(a[i]);
}

std::string config_error(const mrb_config* c) {
  // SolverConfig.__post_init__, solver.py:55-65
  if (!(c->tau > 0)) return "tau must be positive, got " + py_repr(c->tau);
  if (!(0.0 < c->lam && c->lam < 1.0)) return "lambda must be in (0, 1), got " + py_repr(c->lam);
  if (c->max_iterations < 1) return "max_iterations must be >= 1";
  if (c->smoothing_passes < 0) return "smoothing_passes must be >= 0";
  if (!(c->energy_tolerance >= 0)) return "energy_tolerance must be >= 0";
  return "";
}

std::string pair_message(const mrb_batch* b, int p, int* code) {
  const PairStatus& s = b->h_st[p];
  const double* tr = b->h_trace.data() + size_t(p) * b->cfg.max_iterations;
  *code = MRB_OK;
  switch (s.err) {
    case ERR_NONFINITE_ENERGY:
      *code = MRB_E_DIVERGED;
      return "energy became non-finite; reduce tau";
    case ERR_RISES: {
      *code = MRB_E_DIVERGED;
      const int k = s.err_iter;
      std::string vals = "[";
      for (int j = std::max(0, k - 3); j <= k; ++j) {
        if (j > std::max(0, k - 3)) vals += ", ";
        vals += py_repr(tr[j]);
      }
      vals += "]";
      return "energy increased for 10 consecutive iterations (last values " + vals +
             "); reduce tau";
    }
    case ERR_NONFINITE_GRAD:
      *code = MRB_E_DIVERGED;
      return "non-finite gradient; reduce the step size tau";
    default:
      break;
  }
  if (s.dense_nonfinite) {
    *code = MRB_E_VALUE;
    return (s.dense_nonfinite & 1) ? "displacement planes must be finite"
                                   : "image intensities must be finite";
  }
  return "";
}

// deferred handles reaching a host-side consumer: the full host build first
// (the reference validates the whole mesh in TriMesh.__init__, mesh.py:58-123)
int host_ready(mrb_ctx* ctx, mrb_mesh* const* meshes, int64_t count) {
  parallel_for(size_t(count), [&](size_t k) { ensure_host(meshes[k]->h); });  // worker pool
  for (int64_t k = 0; k < count; ++k) {
    const std::string& e = ensure_host(meshes[k]->h);  // first failing mesh, in order
    if (!e.empty()) return fail(ctx, MRB_E_VALUE, e);
  }
  return MRB_OK;
}

}  // namespace

extern "C" {

const char* mrb_version(void) { return kVersion; }

int mrb_ctx_create(int32_t device, mrb_ctx** out) {
  if (!out) return MRB_E_VALUE;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return MRB_E_CUDA;
  if (device < 0 || device >= count) return MRB_E_VALUE;
  auto* c = new mrb_ctx();
  c->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = create_stream(&c->stream, true);
  for (auto& ev : c->stage_done)
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e == cudaSuccess) {  // keep freed pool memory for reuse by later batches
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  if (e != cudaSuccess) {
    delete c;
    return MRB_E_CUDA;
  }
  *out = c;
  return MRB_OK;
}

int mrb_ctx_destroy(mrb_ctx* ctx) {
  if (!ctx) return MRB_OK;
  for (mrb_ctx*& c : ctx->sub) {
    mrb_ctx_destroy(c);
    c = nullptr;
  }
  cudaSetDevice(ctx->device);
  if (ctx->stream) {
    cudaStreamSynchronize(ctx->stream);
    cudaStreamDestroy(ctx->stream);
  }
  for (cudaEvent_t ev : ctx->stage_done)
    if (ev) cudaEventDestroy(ev);
  if (ctx->copy) {
    cudaStreamSynchronize(ctx->copy);
    cudaStreamDestroy(ctx->copy);
  }
  if (ctx->copy_done) cudaEventDestroy(ctx->copy_done);
  if (ctx->aux_hi) {
    cudaStreamSynchronize(ctx->aux_hi);
    cudaStreamDestroy(ctx->aux_hi);
  }
  if (ctx->aux) {
    cudaStreamSynchronize(ctx->aux);
    cudaStreamDestroy(ctx->aux);
  }
  if (ctx->aux_ev) cudaEventDestroy(ctx->aux_ev);
  for (void* pin : ctx->pinned)
    if (pin) cudaFreeHost(pin);
  if (ctx->counts) cudaFreeHost(ctx->counts);
  if (ctx->arena) cudaFreeHost(ctx->arena);
  if (ctx->arena_done) cudaEventDestroy(ctx->arena_done);
  if (ctx->small_pin) cudaFreeHost(ctx->small_pin);
  if (ctx->small_ev) cudaEventDestroy(ctx->small_ev);
  if (ctx->build_stats) cudaFreeHost(ctx->build_stats);
  if (ctx->build_ev) cudaEventDestroy(ctx->build_ev);
  if (ctx->build_in) cudaEventDestroy(ctx->build_in);
  for (auto& k : ctx->kept)
    if (k.p) cudaFree(k.p);
  for (cudaStream_t st : ctx->side)
    if (st) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
  delete ctx;
  return MRB_OK;
}

const char* mrb_last_error(const mrb_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

void* mrb_ctx_stream(mrb_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int mrb_ctx_synchronize(mrb_ctx* ctx) {
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  return e == cudaSuccess ? MRB_OK : cuda_fail(ctx, e);
}

// ---------------------------------------------------------------- mesh
int mrb_mesh_build(int64_t n, const double* V, int64_t m, const int64_t* T, mrb_mesh** out,
                   char* err, int32_t err_len) {
  if (!out) return MRB_E_VALUE;
  *out = nullptr;
  auto* mesh = new mrb_mesh();
  std::string msg;
  try {
    msg = build_mesh(n, V, m, T, mesh->h);
  } catch (const std::exception& ex) {
    msg = std::string("internal error: ") + ex.what();
  }
  if (!msg.empty()) {
    if (err && err_len > 0) {
      std::strncpy(err, msg.c_str(), size_t(err_len) - 1);
      err[err_len - 1] = 0;
    }
    delete mesh;
    return MRB_E_VALUE;
  }
  *out = mesh;
  return MRB_OK;
}

int mrb_mesh_build_many(int32_t count, const int64_t* n, const double* const* V, const int64_t* m,
                        const int64_t* const* T, mrb_mesh** out, int32_t* first_bad, char* err,
                        int32_t err_len) {
  if (first_bad) *first_bad = -1;
  if (count < 0 || (count > 0 && (!n || !V || !m || !T || !out))) return MRB_E_VALUE;
  std::vector<std::string> msg(static_cast<size_t>(count));
  for (int32_t k = 0; k < count; ++k) out[k] = nullptr;
  WorkerPool::get().run(size_t(count), [&](size_t k) {
    auto* mesh = new mrb_mesh();
    try {
      msg[k] = build_mesh(n[k], V[k], m[k], T[k], mesh->h);
    } catch (const std::exception& ex) {
      msg[k] = std::string("internal error: ") + ex.what();
    }
    if (msg[k].empty())
      out[k] = mesh;
    else
      delete mesh;
  });
  for (int32_t k = 0; k < count; ++k)
    if (!msg[k].empty()) {
      if (first_bad) *first_bad = k;
      if (err && err_len > 0) {
        std::strncpy(err, msg[k].c_str(), size_t(err_len) - 1);
        err[err_len - 1] = 0;
      }
      for (int32_t j = 0; j < count; ++j) {  // all or nothing
        delete out[j];
        out[j] = nullptr;
      }
      return MRB_E_VALUE;
    }
  return MRB_OK;
}

int mrb_mesh_create_many(int32_t count, const int64_t* n, const double* const* V, const int64_t* m,
                         const int64_t* const* T, mrb_mesh** out, int32_t* first_bad, char* err,
                         int32_t err_len) {
  if (first_bad) *first_bad = -1;
  if (count < 0 || (count > 0 && (!n || !V || !m || !T || !out))) return MRB_E_VALUE;
  for (int32_t k = 0; k < count; ++k) out[k] = nullptr;
  if (count == 0) return MRB_OK;
  // one block for every mesh of the call, laid out as the device build
  // uploads it (V, then the oriented int32 T, 256-byte aligned): pinned and
  // recycled, so neither page faults nor a staging copy
  std::vector<size_t> off(static_cast<size_t>(count) + 1, 0);
  for (int32_t k = 0; k < count; ++k)
    off[k + 1] = off[k] + al256(size_t(std::max<int64_t>(n[k], 0)) * 16) +
                 al256(size_t(std::max<int64_t>(m[k], 0)) * 12);
  const std::shared_ptr<unsigned char> block = pinned_block(std::max<size_t>(off[count], 256));
  std::vector<std::string> msg(static_cast<size_t>(count));
  // a large mesh is validated in parts on the whole worker pool, the others
  // one mesh per worker
  auto large = [&](int32_t k) { return m[k] >= 200000 && n[k] < (int64_t(1) << 31); };
  WorkerPool::get().run(size_t(count), [&](size_t k) {
    if (large(int32_t(k))) return;
    auto* mesh = new mrb_mesh();
    unsigned char* at = block.get() + off[k];
    try {
      msg[k] = create_mesh(n[k], V[k], m[k], T[k], reinterpret_cast<double*>(at),
                           reinterpret_cast<int32_t*>(at + al256(size_t(n[k]) * 16)), mesh->h);
    } catch (const std::exception& ex) {
      msg[k] = std::string("internal error: ") + ex.what();
    }
    if (msg[k].empty()) {
      mesh->h.def_hold = block;
      out[k] = mesh;
    } else {
      delete mesh;
    }
  });
  for (int32_t k = 0; k < count; ++k) {
    if (!large(k)) continue;
    auto* mesh = new mrb_mesh();
    unsigned char* at = block.get() + off[k];
    double* Vout = reinterpret_cast<double*>(at);
    int32_t* Tout = reinterpret_cast<int32_t*>(at + al256(size_t(n[k]) * 16));
    constexpr int kParts = 64;
    std::vector<ValidatePart> parts(kParts);
    std::vector<int32_t> inc(size_t(n[k]), 0);
    try {
      WorkerPool::get().run(kParts, [&](size_t c) {
        validate_part(n[k], V[k], n[k] * int64_t(c) / kParts, n[k] * int64_t(c + 1) / kParts,
                      m[k], T[k], m[k] * int64_t(c) / kParts, m[k] * int64_t(c + 1) / kParts,
                      Vout, Tout, inc.data(), parts[c]);
      });
      msg[k] = finish_create(parts, n[k], m[k], Vout, Tout, mesh->h);
    } catch (const std::exception& ex) {
      msg[k] = std::string("internal error: ") + ex.what();
    }
    if (msg[k].empty()) {
      mesh->h.def_hold = block;
      out[k] = mesh;
    } else {
      delete mesh;
    }
  }
  for (int32_t k = 0; k < count; ++k)
    if (!msg[k].empty()) {
      if (first_bad) *first_bad = k;
      if (err && err_len > 0) {
        std::strncpy(err, msg[k].c_str(), size_t(err_len) - 1);
        err[err_len - 1] = 0;
      }
      for (int32_t j = 0; j < count; ++j) {  // all or nothing
        delete out[j];
        out[j] = nullptr;
      }
      return MRB_E_VALUE;
    }
  return MRB_OK;
}

int mrb_mesh_destroy(mrb_mesh* mesh) {
  delete mesh;
  return MRB_OK;
}

int mrb_mesh_device_check(mrb_ctx* ctx, mrb_mesh* mesh, int32_t cs, int32_t npt, int64_t* out) {
  // test hook: the device build of a deferred mesh against the host build
  // (element mismatches per array; see the header)
  if (!ctx || !mesh || !out) return MRB_E_VALUE;
  HostMesh& h = mesh->h;
  if (!h.deferred || !(h.dev ? h.dev->b_nb_ptr != nullptr : device_buildable(h)))
    return fail(ctx, MRB_E_VALUE, "not a device-buildable deferred mesh");
  try {
    ck(cudaSetDevice(ctx->device));
    AllocScope scope(ctx->stream);
    if (!h.dev) device_build_meshes(ctx, {&h}, ctx->stream);
    {
      const std::string e = device_build_finish(ctx);
      if (!e.empty()) return fail(ctx, MRB_E_VALUE, e);
    }
    if (!h.dev || !h.dev->b_nb_ptr) return fail(ctx, MRB_E_INTERNAL, "device build flagged");
    const int chunk = int((h.n + cs - 1) / cs);
    if (!device_cluster_topos(ctx, {std::make_tuple(&h, int(cs), int(npt))}, ctx->stream))
      return fail(ctx, MRB_E_INTERNAL, "device topology needs the host planner");
    ck(cudaStreamSynchronize(ctx->stream));
    // the host build of the same mesh (a copy: h keeps its device arrays)
    HostMesh H;
    {
      const std::vector<int64_t> T64(h.dT, h.dT + 3 * h.m);
      const std::string e = build_mesh(h.n, h.dV, h.m, T64.data(), H);
      if (!e.empty()) return fail(ctx, MRB_E_VALUE, e);
    }
    const size_t n = size_t(h.n), m = size_t(h.m), e2 = H.nb_idx.size();
    const DeviceMesh& d = *h.dev;
    auto fetch = [&](const void* src, size_t bytes) {
      std::vector<unsigned char> v(bytes);
      ck(cudaMemcpy(v.data(), src, bytes, cudaMemcpyDeviceToHost));
      return v;
    };
    auto diff = [](const void* a, const void* b, size_t count, size_t size) {
      int64_t c = 0;
      for (size_t i = 0; i < count; ++i)
        c += std::memcmp(static_cast<const char*>(a) + i * size,
                         static_cast<const char*>(b) + i * size, size) != 0;
      return c;
    };
    std::vector<float> gs(2 * n), iv(n);
    for (size_t k = 0; k < 2 * n; ++k) gs[k] = float(H.g_self[k]);
    for (size_t k = 0; k < n; ++k) iv[k] = float(H.inv_val[k]);
    out[0] = diff(fetch(d.V, n * 16).data(), H.Vn.data(), n, 16);
    out[1] = diff(fetch(d.tri, m * 16).data(), H.Tn.data(), m, 16);
    out[2] = diff(fetch(d.perm, n * 4).data(), H.perm.data(), n, 4);
    out[3] = diff(fetch(d.g_self_f, n * 8).data(), gs.data(), n, 8);
    out[4] = diff(fetch(d.inv_val_f, n * 4).data(), iv.data(), n, 4);
    out[5] = int64_t(h.max_deg != H.max_deg) + int64_t(h.ne != H.ne);
    out[6] = diff(fetch(d.b_nb_ptr, (n + 1) * 4).data(), H.nb_ptr.data(), n + 1, 4);
    out[7] = diff(fetch(d.b_nb_idx, e2 * 4).data(), H.nb_idx.data(), e2, 4);
    out[8] = diff(fetch(d.b_g_nb, e2 * 16).data(), H.g_nb.data(), e2, 16);
    const DeviceMesh::Topo& t = d.topo.at(topo_key(cs, chunk, npt));
    const TopoHost th = plan_topo(H, cs, chunk, npt);
    std::vector<unsigned char> packed(th.total, 0);
    write_topo(H, cs, th, packed.data(), npt);
    if (t.topo_stride != th.stride || t.halo_stride != th.hstride ||
        t.send_stride != th.sstride || t.slices != th.slices) {
      out[9] = -1;
    } else {
      out[9] = diff(fetch(t.slab, th.total).data(), packed.data(), th.total, 1);
    }
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e, e.line);
  }
  return MRB_OK;
}

int mrb_mesh_counts(const mrb_mesh* mesh, int64_t* c) {
  if (!ensure_host(const_cast<mrb_mesh*>(mesh)->h).empty()) return MRB_E_VALUE;
  const HostMesh& h = mesh->h;
  c[0] = h.n;
  c[1] = h.m;
  c[2] = h.ne;
  c[3] = int64_t(h.ring_idx.size());  // nnz(L) = 2 n_edges
  c[4] = 3 * h.m;                      // nnz(Gx) = nnz(Gy)
  c[5] = 3 * h.m;                      // nnz(avg)
  return MRB_OK;
}

int mrb_mesh_export_connectivity(const mrb_mesh* mesh, int64_t* tri, int64_t* edges,
                                 int64_t* valence, uint8_t* boundary, int64_t* ring_ptr,
                                 int64_t* ring_idx, int64_t* inc_ptr, int64_t* inc_idx) {
  if (!ensure_host(const_cast<mrb_mesh*>(mesh)->h).empty()) return MRB_E_VALUE;
  const HostMesh& h = mesh->h;
  auto cp = [](int64_t* dst, const std::vector<int64_t>& v) {
    if (dst) std::memcpy(dst, v.data(), v.size() * sizeof(int64_t));
  };
  cp(tri, h.T);
  cp(edges, h.edges);
  cp(valence, h.valence);
  if (boundary) std::memcpy(boundary, h.boundary.data(), h.boundary.size());
  cp(ring_ptr, h.ring_ptr);
  cp(ring_idx, h.ring_idx);
  cp(inc_ptr, h.inc_ptr);
  cp(inc_idx, h.inc_idx);
  return MRB_OK;
}

int mrb_mesh_export_csr(const mrb_mesh* mesh, int32_t which, int64_t* indptr, int64_t* indices,
                        double* data) {
  HostMesh& h = const_cast<mrb_mesh*>(mesh)->h;  // the CSR cache is built on first use
  if (!ensure_host(h).empty()) return MRB_E_VALUE;
  ensure_reference_csr(h);
  const Csr* c = which == MRB_CSR_LAPLACIAN  ? &h.lap
                 : which == MRB_CSR_GRAD_X   ? &h.gx
                 : which == MRB_CSR_GRAD_Y   ? &h.gy
                 : which == MRB_CSR_VERTEX_AVG ? &h.avg
                                               : nullptr;
  if (!c) return MRB_E_VALUE;
  if (indptr) std::memcpy(indptr, c->indptr.data(), c->indptr.size() * sizeof(int64_t));
  if (indices) std::memcpy(indices, c->indices.data(), c->indices.size() * sizeof(int64_t));
  if (data) std::memcpy(data, c->data.data(), c->data.size() * sizeof(double));
  return MRB_OK;
}

int mrb_mesh_export_geometry(const mrb_mesh* mesh, double* areas, double* coeffs,
                             double* vertex_areas) {
  if (!ensure_host(const_cast<mrb_mesh*>(mesh)->h).empty()) return MRB_E_VALUE;
  const HostMesh& h = mesh->h;
  if (areas) std::memcpy(areas, h.areas.data(), h.areas.size() * sizeof(double));
  if (coeffs) std::memcpy(coeffs, h.coeffs.data(), h.coeffs.size() * sizeof(double));
  if (vertex_areas)
    std::memcpy(vertex_areas, h.vertex_areas.data(), h.vertex_areas.size() * sizeof(double));
  return MRB_OK;
}

int mrb_mesh_locate(mrb_mesh* mesh, int64_t n, const double* pts, int64_t* tri, double* w) {
  // PointLocator + locate, densefield.py:62-127: lowest-index containing
  // triangle and its barycentric weights in numpy's order; -1 if uncovered
  if (!ensure_host(mesh->h).empty()) return MRB_E_VALUE;
  if (!mesh->locator) mesh->locator.reset(new Locator(mesh->h));
  for (int64_t i = 0; i < n; ++i) {
    double wi[3] = {0.0, 0.0, 0.0};
    tri[i] = mesh->locator->locate(mesh->h, pts[2 * i], pts[2 * i + 1], wi);
    if (w) std::memcpy(w + 3 * i, wi, sizeof wi);
  }
  return MRB_OK;
}

int mrb_pixel_map(mrb_ctx* ctx, mrb_mesh* mesh, int32_t W, int32_t H, int64_t* tri_of,
                  double* weights) {
  if (const int rc = host_ready(ctx, &mesh, 1)) return rc;
  try {
    AllocScope scope(ctx->stream);
    ck(cudaSetDevice(ctx->device));
    int* map = nullptr;
    const std::string msg = ensure_pixel_map(ctx, mesh->h, W, H, &map);
    if (!msg.empty()) return fail(ctx, MRB_E_COVERAGE, msg);
    const size_t npx = size_t(W) * H;
    if (tri_of) {
      std::vector<int> host(npx);
      ck(mrb_copy_async(host.data(), map, npx * sizeof(int), cudaMemcpyDeviceToHost,
                         ctx->stream));
      ck(cudaStreamSynchronize(ctx->stream));
      for (size_t q = 0; q < npx; ++q) tri_of[q] = host[q];
    }
    if (weights) {
      Tmp t(ctx->stream);
      double* w = t.get<double>(3 * npx);
      k_pixel_weights<<<unsigned((npx + 255) / 256), 256, 0, ctx->stream>>>(
          mesh->h.dev->V, mesh->h.dev->tri, map, W, int(npx), w);
      ck(cudaGetLastError());
      ck(mrb_copy_async(weights, w, 3 * npx * sizeof(double), cudaMemcpyDeviceToHost,
                         ctx->stream));
      ck(cudaStreamSynchronize(ctx->stream));
    }
    return MRB_OK;
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e, e.line);
  }
}

// ---------------------------------------------------------------- batch
}  // extern "C"

namespace {
// mrb_batch_create with an optional imposed cluster shape (forced_cs > 0)
int batch_create_impl(mrb_ctx* ctx, int32_t n_pairs, mrb_mesh* const* meshes, int32_t W,
                      int32_t H, int32_t img_dtype, const mrb_config* cfg, int forced_cs,
                      int forced_npt, mrb_batch** out, int defer_topo = 0) {
  // defer_topo > 0: topologies are planned here, the first `defer_topo` pairs'
  // data uploaded here too (they gate the first launch), the rest per wave
  // group by the run (flush_topo)
  *out = nullptr;
  const std::string ce = config_error(cfg);
  if (!ce.empty()) return fail(ctx, MRB_E_VALUE, ce);
  if (n_pairs < 1) return fail(ctx, MRB_E_VALUE, "batch needs at least one pair");
  if (W < 2 || H < 2)
    return fail(ctx, MRB_E_VALUE, "bicubic sampling needs an image of at least 2x2 pixels");
  if (int64_t(W) * H >= (int64_t(1) << 31) / 2)
    return fail(ctx, MRB_E_VALUE, "image too large for 32-bit pixel indexing");
  std::unique_ptr<mrb_batch> b(new mrb_batch());
  b->ctx = ctx;
  b->n_pairs = n_pairs;
  b->W = W;
  b->H = H;
  b->in_dtype = img_dtype;
  b->cfg = *cfg;
  b->real_d = cfg->precision == MRB_PREC_F64;
  b->tap_d = img_dtype == MRB_F64 && b->real_d;
  b->meshes.assign(meshes, meshes + n_pairs);
  AllocScope scope(ctx->stream);
  try {
    ck(cudaSetDevice(ctx->device));
    {
      size_t nodes = 0;
      for (int p = 0; p < n_pairs; ++p) nodes += size_t(meshes[p]->h.n);
      const size_t pix_blocks = size_t(n_pairs) * ((size_t(W) * H + kPixBlock - 1) / kPixBlock);
      arena_begin(ctx, size_t(n_pairs) * 2048 + 4 * (pix_blocks + nodes / kNodeBlock + n_pairs) +
                           (64 << 10));
    }
    int64_t off = 0;
    const bool dbg = std::getenv("MESHREG_B200_DEBUG") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    const bool dbg_sync = dbg && std::string(std::getenv("MESHREG_B200_DEBUG")) != "2";
    auto tick = [&](const char* what) {
      if (!dbg) return;
      if (dbg_sync) cudaStreamSynchronize(ctx->stream);  // MESHREG_B200_DEBUG=2: host time only
      const auto t1 = std::chrono::steady_clock::now();
      std::fprintf(stderr, "meshreg_b200: batch_create %-22s %8.2f ms\n", what,
                   std::chrono::duration<double, std::milli>(t1 - t0).count());
      t0 = t1;
    };
    std::vector<HostMesh*> hm;
    for (int p = 0; p < n_pairs; ++p) {
      b->node_off.push_back(int(off));
      off += meshes[p]->h.n;
      hm.push_back(&meshes[p]->h);
    }
    // the fast path never reads the generic one-ring arrays: upload them only
    // when the batch is not eligible for it
    const char* why_not = nullptr;
    const int mode = fast_mode(b->real_d, b->tap_d, img_dtype, b->meshes, &why_not);
    const bool eligible = mode != 0;
    b->forced_cs = forced_cs;
    b->forced_npt = forced_npt;
    // fp64 batches that k_cluster64 can run need neither the generic path's
    // one-ring arrays nor its fp64 ring operator (setup_cluster64 falls back)
    const bool c64 = b->real_d && cluster64_candidate(b.get());
    ensure_device_meshes(ctx, hm, !eligible && !c64);
    if (!eligible && !c64)  // meshes uploaded earlier by a fast-path batch lack them
      for (HostMesh* h : hm) ensure_device_mesh_ring(ctx, *h);
    if (b->real_d) {
      if (c64)
        ensure_device_meshes_f64_self(ctx, hm);
      else
        for (HostMesh* h : hm) ensure_device_mesh_f64(ctx, *h);
    }
    tick("mesh upload");
    PixelMapJob pmj;
    bool rasters_issued = false;
    const bool defer = eligible && defer_topo && mode == 1;
    if (!defer) {  // rasters run while the host plans the topologies
      pmj = issue_pixel_maps(ctx, hm, W, H);
      adopt_early_rasters(pmj, W, H);
      rasters_issued = true;
    }
    if (eligible) {
      // fast-path topologies: their host planning overlaps the mesh and image
      // uploads still in flight (finish_pixel_maps synchronises)
      mrb_mesh* big = *std::max_element(b->meshes.begin(), b->meshes.end(),
                                        [](mrb_mesh* x, mrb_mesh* y) { return x->h.n < y->h.n; });
      int cs = forced_cs, npt = forced_npt, occ = 0;
      if (mode == 2)
        grid_shape(big->h.n, &cs, &npt);
      if (cs || choose_cluster_shape(ctx, big->h, n_pairs, cfg->smoothing_passes >= 2, &cs, &npt,
                                     &occ)) {
        if (defer) {  // plan now, pack + copy per wave group in the run
          // pairs of the expected tail wave (setup_tail) run in the latency
          // shape: no throughput-shape topology for them
          int planned = n_pairs;
          if (npt == 2 && n_pairs > defer_topo && n_pairs % defer_topo &&
              !std::getenv("MESHREG_B200_NO_TAIL"))
            planned = n_pairs - n_pairs % defer_topo;
          b->planned_end = planned;
          // only the first wave group is planned here; later groups are
          // planned in the run, ahead of their launch (flush_topo) — unless
          // every topology exists already (device-built meshes)
          b->lazy_from = std::min(defer_topo, planned);
          {
            bool all = true;
            for (int p = b->lazy_from; p < planned && all; ++p) {
              HostMesh* h = hm[p];
              all = h->dev->topo.count(topo_key(cs, int((h->n + cs - 1) / cs), npt)) > 0;
            }
            if (all) b->lazy_from = planned;
          }
          std::vector<HostMesh*> todo;
          for (int p = 0; p < b->lazy_from; ++p) {
            HostMesh* h = hm[p];
            const int chunk = int((h->n + cs - 1) / cs);
            if (!h->dev->topo.count(topo_key(cs, chunk, npt)) &&
                std::find(todo.begin(), todo.end(), h) == todo.end())
              todo.push_back(h);
          }
          cudaEvent_t slab_ev = nullptr;
          if (!todo.empty()) {
            b->topo_up.reset(new TopoUpload(plan_cluster_topos(ctx, todo, cs, npt)));
            for (size_t i = 0; i < todo.size(); ++i) b->topo_index[todo[i]] = i;
            ck(cudaEventCreateWithFlags(&slab_ev, cudaEventDisableTiming));
            ck(cudaEventRecord(slab_ev, ctx->stream));  // the slab exists from here on
          }
          // rasters on the side stream: the first group's loop and topology
          // copy need not wait for them (its dense pass does)
          pmj = issue_pixel_maps(ctx, hm, W, H, true);
          adopt_early_rasters(pmj, W, H);
          rasters_issued = true;
          if (!todo.empty()) {
            if (!b->copy_stream)
              b->copy_stream = side_stream(ctx, 2);
            ck(cudaStreamWaitEvent(b->copy_stream, slab_ev, 0));
            cudaEventDestroy(slab_ev);
            flush_topo(b.get(), std::min(defer_topo, n_pairs), b->copy_stream, ctx->stream);
          }
        } else {
          ensure_cluster_topos(ctx, hm, cs, npt);
        }
      }
      tick("topologies");
    }
    if (!rasters_issued) {
      pmj = issue_pixel_maps(ctx, hm, W, H);
      adopt_early_rasters(pmj, W, H);
    }
    b->total_nodes = off;
    const size_t npx = size_t(W) * H;
    b->st = dalloc<PairStatus>(n_pairs);
    b->traces = dalloc<double>(size_t(n_pairs) * cfg->max_iterations);
    b->u_out = dalloc<double2>(off);
    b->src_ptrs = dalloc<void*>(2 * n_pairs);
    // the interleaved image copy of the generic / fp64 loops (the fp32
    // cluster path reads the planar inputs): allocated when a path needs it
    auto alloc_img = [&](mrb_batch* bb) {
      bb->img = dalloc<char>(size_t(n_pairs) * 2 * npx * tap_size(bb));
      std::vector<void*> ip(n_pairs);
      for (int p = 0; p < n_pairs; ++p)
        ip[p] = static_cast<char*>(bb->img) + size_t(p) * 2 * npx * tap_size(bb);
      bb->img_ptrs = aupload(ctx, ip.data(), ip.size());
    };
    if (!(eligible && mode == 1 && !b->real_d)) alloc_img(b.get());
    if (b->tap_d)
      build_pairs<double, double>(b.get());
    else if (b->real_d)
      build_pairs<float, double>(b.get());
    else
      build_pairs<float, float>(b.get());
    tick("buffers + descriptors");
    if (eligible) setup_cluster_path(b.get());
    if (b->real_d) setup_cluster64(b.get());
    if (c64 && !b->c64_cs) {  // no cluster shape after all: the generic loop's arrays
      for (HostMesh* h : hm) {
        ensure_device_mesh_ring(ctx, *h);
        ensure_device_mesh_f64(ctx, *h);
      }
      free_pairs(b.get());
      if (b->tap_d)
        build_pairs<double, double>(b.get());
      else
        build_pairs<float, double>(b.get());
    }
    tick("cluster path setup");
    if (eligible && !b->cluster_cs) {
      // predicted fast path did not fit after all: generic path needs the rings
      for (HostMesh* h : hm) ensure_device_mesh_ring(ctx, *h);
      if (!b->img) alloc_img(b.get());
      free_pairs(b.get());
      if (b->real_d)
        build_pairs<float, double>(b.get());
      else
        build_pairs<float, float>(b.get());
    }
    // coverage check last: the host work above overlapped the rasters.
    // mrb_register_many (defer_topo) defers it to mrb_batch_sync.
    if (defer_topo > 0 && eligible && b->cluster_cs && !b->grid_mode) {
      b->pending_pm.reset(new PixelMapJob(std::move(pmj)));
    } else {
      const std::string msg = finish_pixel_maps(ctx, pmj);
      if (!msg.empty()) return fail(ctx, MRB_E_COVERAGE, msg);
    }
    tick("pixel maps");
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e, e.line);
  }
  *out = b.release();
  return MRB_OK;
}
// fp64 persistent cluster loop (k_cluster64) for a batch on the generic path
// (fp64 state, fp32-exact images): every mesh fits 16 CTAs x 768 nodes with
// one-rings of <= kMaxDeg.  Cluster size by the cost model of
// choose_cluster_shape (waves x nodes per CTA).  MESHREG_B200_PATH=generic
// keeps the three-kernel loop.
template <int NPT>
int cluster64_occupancy(int CS, size_t smem) {
  auto kern = k_cluster64<NPT>;
  if (!raise_smem_limit_of(kern, smem)) return 0;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(unsigned(CS));
  lc.blockDim = dim3(kClusterThreads);
  lc.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &lc) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

std::string env_exchange() {
  const char* x = std::getenv("MESHREG_B200_EXCHANGE");
  return x ? std::string(x) : std::string();
}

int cluster64_push_occupancy(int CS, size_t smem) {
  auto kern = k_cluster64_push;
  if (!raise_smem_limit_of(kern, smem)) return 0;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(unsigned(CS));
  lc.blockDim = dim3(kClusterThreads);
  lc.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &lc) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void setup_cluster64(mrb_batch* b) {
  const char* env = std::getenv("MESHREG_B200_PATH");
  const bool dbg = std::getenv("MESHREG_B200_DEBUG") != nullptr;
  if (env && std::string(env) == "generic") return;
  int64_t nmax = 0;
  for (mrb_mesh* m : b->meshes) {
    nmax = std::max<int64_t>(nmax, m->h.n);
    if (m->h.max_deg > kMaxDeg) return;
  }
  const int cs_min = int((nmax + kClusterThreads - 1) / kClusterThreads);
  if (cs_min > 16) return;
  const bool two_u = b->cfg.smoothing_passes >= 2;
  std::vector<HostMesh*> hm;
  for (mrb_mesh* m : b->meshes) hm.push_back(&m->h);
  double best = 1e300;
  int best_cs = 0;
  size_t best_smem = 0;
  // mrb_register_many's device setup decides the cluster size (forced_cs)
  const int cs_lo = b->forced_cs ? std::max(cs_min, b->forced_cs) : cs_min;
  const int cs_hi = b->forced_cs ? cs_lo : 16;
  for (int cs = cs_lo; cs <= cs_hi; ++cs) {
    ensure_cluster_topos64(b->ctx, hm, cs);
    size_t smem = 0;
    for (HostMesh* h : hm) {
      const DeviceMesh::Topo& t = h->dev->topo.at(topo64_key(cs, int((h->n + cs - 1) / cs)));
      smem = std::max(smem, cluster64_dyn_smem(t.topo_stride, t.slices, t.halo_stride, two_u));
    }
    const int occ = cluster64_occupancy<1>(cs, smem);
    if (occ < 1) continue;
    const double cost = double((b->n_pairs + occ - 1) / occ) * double((nmax + cs - 1) / cs);
    if (cost < best) {
      best = cost;
      best_cs = cs;
      best_smem = smem;
    }
  }
  if (!best_cs) {
    if (dbg) std::fprintf(stderr, "meshreg_b200: fp64 generic loop (no cluster shape fits)\n");
    return;
  }
  // the generic path's descriptors: PairDev<float, double> or, with fp64
  // image storage, PairDev<double, double> (same fields, taps differ)
  const PairDev<float, double>* host32 =
      reinterpret_cast<const PairDev<float, double>*>(b->pairs_host.data());
  const PairDev<double, double>* host64 =
      reinterpret_cast<const PairDev<double, double>*>(b->pairs_host.data());
  std::vector<ClusterPair64> cp(b->n_pairs);
  const size_t padn = size_t(b->W + 2) * (b->H + 2);
  b->pad64 = dalloc<double2>(padn * b->n_pairs);
  if (!b->tap_d && b->in_dtype == MRB_F32) {  // fp32-exact inputs: the shifted fp32 copies too
    b->pad_pitch = (b->W + 5 + 3) / 4 * 4;
    b->pad_plane = size_t(b->H + 2) * b->pad_pitch;
    b->img_pad = dalloc<float2>(4 * b->pad_plane * b->n_pairs);
  }
  for (int p = 0; p < b->n_pairs; ++p) {
    HostMesh& h = b->meshes[p]->h;
    const int chunk = int((h.n + best_cs - 1) / best_cs);
    const DeviceMesh::Topo& t = h.dev->topo.at(topo64_key(best_cs, chunk));
    ClusterPair64& c = cp[p];
    c.tap_d = b->tap_d ? 1 : 0;
    c.pad = b->pad64 + padn * p;
    c.img4 = b->img_pad ? b->img_pad + 4 * b->pad_plane * p : nullptr;
    c.pitch = b->pad_pitch;
    c.plane = int(b->pad_plane);
    c.V = b->tap_d ? host64[p].V : host32[p].V;
    c.g_self = b->tap_d ? host64[p].g_self : host32[p].g_self;
    c.inv_val = b->tap_d ? host64[p].inv_val : host32[p].inv_val;
    c.codes = t.codes;
    c.g = t.g64;
    c.slice_off = t.slice_off;
    c.halo = t.halo;
    c.n_halo = t.n_halo;
    c.send = t.send;
    c.n_send = t.n_send;
    c.send_stride = t.send_stride;
    c.img = b->tap_d ? static_cast<const void*>(host64[p].img)
                     : static_cast<const void*>(host32[p].img);
    c.u = b->tap_d ? host64[p].u : host32[p].u;
    c.trace = b->tap_d ? host64[p].trace : host32[p].trace;
    c.n = int(h.n);
    c.chunk = chunk;
    c.W = b->W;
    c.H = b->H;
    c.topo_stride = t.topo_stride;
    c.slices = t.slices;
    c.halo_stride = t.halo_stride;
  }
  b->c64_pairs = aupload(b->ctx, cp.data(), cp.size());
  b->c64_cs = best_cs;
  b->c64_smem = best_smem;
  // push exchange when it fits without losing resident clusters (no cluster
  // barrier in the loop; the pull kernel measured barrier-bound)
  if (b->cfg.smoothing_passes <= 1 && env_exchange() != "pull") {
    size_t ps = 0;
    bool lists = true;
    for (HostMesh* h : hm) {
      const DeviceMesh::Topo& t = h->dev->topo.at(topo64_key(best_cs, int((h->n + best_cs - 1) / best_cs)));
      lists = lists && t.send_stride > 0;
      ps = std::max(ps, push64_dyn_smem(t.topo_stride, t.slices, t.halo_stride, t.send_stride));
    }
    if (lists && cluster64_push_occupancy(best_cs, ps) >= cluster64_occupancy<1>(best_cs, best_smem)) {
      b->c64_push = true;
      b->c64_smem = ps;
    }
  }
  if (std::getenv("MESHREG_B200_DEBUG"))
    std::fprintf(stderr, "meshreg_b200: fp64 cluster %d CTAs x 1 node/thread, %zu B smem, %s\n",
                 best_cs, b->c64_smem, b->c64_push ? "push" : "pull");
}

void launch_cluster64(mrb_batch* b) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(unsigned(b->n_pairs * b->c64_cs));
  lc.blockDim = dim3(kClusterThreads);
  lc.dynamicSmemBytes = b->c64_smem;
  lc.stream = b->ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = b->c64_cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  ck(cudaLaunchKernelEx(&lc, b->c64_push ? k_cluster64_push : k_cluster64<1>,
                        static_cast<const ClusterPair64*>(b->c64_pairs), b->st,
                        int(b->cfg.max_iterations), double(b->cfg.energy_tolerance),
                        double(b->cfg.tau), double(b->cfg.lam), int(b->cfg.smoothing_passes)));
}

// Split a fast-path batch into wave groups of `per` pairs (see mrb_batch).
void batch_set_groups(mrb_batch* b, int per) {
  if (!b->cluster_cs || per <= 0 || per >= b->n_pairs) return;
  b->groups.clear();
  for (int p = 0; p < b->n_pairs; p += per) b->groups.push_back(p);
  b->groups.push_back(b->n_pairs);
  b->group_ev.resize(b->groups.size());
  for (auto& e : b->group_ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  if (!b->copy_stream) b->copy_stream = side_stream(b->ctx, 2);
}
}  // namespace

extern "C" {

int mrb_batch_create(mrb_ctx* ctx, int32_t n_pairs, mrb_mesh* const* meshes, int32_t W,
                     int32_t H, int32_t img_dtype, const mrb_config* cfg, mrb_batch** out) {
  if (n_pairs > 0 && meshes)
    if (const int rc = host_ready(ctx, meshes, n_pairs)) return rc;
  return batch_create_impl(ctx, n_pairs, meshes, W, H, img_dtype, cfg, 0, 0, out);
}

int mrb_batch_destroy(mrb_batch* b) {
  if (!b) return MRB_OK;
  cudaSetDevice(b->ctx->device);
  cudaStreamSynchronize(b->ctx->stream);
  delete b;
  return MRB_OK;
}

int mrb_batch_set_images(mrb_batch* b, const void* re, const void* te, int32_t on_device) {
  mrb_ctx* ctx = b->ctx;
  AllocScope scope(ctx->stream);
  try {
    ck(cudaSetDevice(ctx->device));
    const size_t npx = size_t(b->W) * b->H, es = in_size(b->in_dtype);
    const size_t bytes = size_t(b->n_pairs) * npx * es;
    const char *rs, *ts;
    if (on_device) {
      rs = static_cast<const char*>(re);
      ts = static_cast<const char*>(te);
    } else {
      if (!b->stage) b->stage = dalloc<char>(2 * bytes);
      char* st = static_cast<char*>(b->stage);
      ck(mrb_copy_async(st, re, bytes, cudaMemcpyHostToDevice, ctx->stream));
      ck(mrb_copy_async(st + bytes, te, bytes, cudaMemcpyHostToDevice, ctx->stream));
      rs = st;
      ts = st + bytes;
    }
    std::vector<const void*> ptrs(2 * b->n_pairs);
    for (int p = 0; p < b->n_pairs; ++p) {
      ptrs[p] = rs + size_t(p) * npx * es;
      ptrs[b->n_pairs + p] = ts + size_t(p) * npx * es;
    }
    if (ptrs != b->src_host) {  // filled on the device: no host buffer, no stream sync
      b->src_host = ptrs;
      k_fill_ptrs<<<(b->n_pairs + 255) / 256, 256, 0, ctx->stream>>>(
          b->src_ptrs, rs, ts, npx * es, b->n_pairs);
      ck(cudaGetLastError());
    }
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e, e.line);
  }
  return MRB_OK;
}

int mrb_batch_run(mrb_batch* b) {
  mrb_ctx* ctx = b->ctx;
  try {
    ck(cudaSetDevice(ctx->device));
    b->synced = false;
    if (b->runs == 0) {
      dispatch_enqueue(b);  // first run: direct launches
    } else {
      if (!b->graph) {
        cudaGraph_t g;
        ck(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
        dispatch_enqueue(b);
        ck(cudaStreamEndCapture(ctx->stream, &g));
        ck(cudaGraphInstantiate(&b->graph, g, 0));
        cudaGraphDestroy(g);
      }
      ck(cudaGraphLaunch(b->graph, ctx->stream));
    }
    b->runs++;
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e, e.line);
  }
  return MRB_OK;
}

int mrb_batch_get_results(mrb_batch* b, int32_t out_dtype, double* u, void* ux, void* uy,
                          void* warped) {
  mrb_ctx* ctx = b->ctx;
  AllocScope scope(ctx->stream);
  try {
    ck(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const bool same_dtype = (out_dtype == MRB_F64) == b->real_d;
    if (b->groups_recorded && same_dtype) {
      // wave groups: group g's results leave while later groups compute
      b->groups_recorded = false;
      const size_t npx = size_t(b->W) * b->H, os = in_size(out_dtype);
      void* outs[3] = {ux, uy, warped};
      for (size_t g = 0; g + 1 < b->groups.size(); ++g) {
        const int p0 = b->groups[g], p1 = b->groups[g + 1];
        ck(cudaStreamWaitEvent(b->copy_stream, b->group_ev[g], 0));
        if (u) {
          const size_t n0 = size_t(b->node_off[p0]);
          const size_t n1 = p1 < b->n_pairs ? size_t(b->node_off[p1]) : size_t(b->total_nodes);
          ck(mrb_copy_async(u + 2 * n0, b->u_out + n0, (n1 - n0) * sizeof(double2),
                            cudaMemcpyDeviceToHost, b->copy_stream));
        }
        for (int c = 0; c < 3; ++c) {  // one strided copy per plane and group
          if (!outs[c]) continue;
          ck(mrb_copy2d_async(static_cast<char*>(outs[c]) + size_t(p0) * npx * os, npx * os,
                              static_cast<const char*>(b->dense) + (3 * size_t(p0) + c) * npx * os,
                              3 * npx * os, npx * os, size_t(p1 - p0), cudaMemcpyDeviceToHost,
                              b->copy_stream));
        }
      }
      ck(cudaEventRecord(b->group_ev.back(), b->copy_stream));
      ck(cudaStreamWaitEvent(s, b->group_ev.back(), 0));  // sync on ctx->stream covers it
      return MRB_OK;
    }
    if (u)
      ck(mrb_copy_async(u, b->u_out, size_t(b->total_nodes) * sizeof(double2),
                         cudaMemcpyDeviceToHost, s));
    const size_t npx = size_t(b->W) * b->H;
    const bool same = (out_dtype == MRB_F64) == b->real_d;
    const size_t os = in_size(out_dtype);
    void* outs[3] = {ux, uy, warped};
    for (int c = 0; c < 3; ++c) {
      if (!outs[c]) continue;
      for (int p = 0; p < b->n_pairs; ++p) {
        const char* src = static_cast<const char*>(b->dense) + (3 * size_t(p) + c) * npx * real_size(b);
        char* dst = static_cast<char*>(outs[c]) + size_t(p) * npx * os;
        if (same) {
          ck(mrb_copy_async(dst, src, npx * os, cudaMemcpyDeviceToHost, s));
        } else {
          if (!b->conv) b->conv = dalloc<char>(3 * size_t(b->n_pairs) * npx * os);
          char* cv = static_cast<char*>(b->conv) + (3 * size_t(p) + c) * npx * os;
          const unsigned g = unsigned(std::min<size_t>((npx + 255) / 256, 2048));
          if (b->real_d)
            k_convert<double, float><<<g, 256, 0, s>>>(reinterpret_cast<const double*>(src),
                                                       reinterpret_cast<float*>(cv), npx);
          else
            k_convert<float, double><<<g, 256, 0, s>>>(reinterpret_cast<const float*>(src),
                                                       reinterpret_cast<double*>(cv), npx);
          ck(cudaGetLastError());
          ck(mrb_copy_async(dst, cv, npx * os, cudaMemcpyDeviceToHost, s));
        }
      }
    }
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e, e.line);
  }
  return MRB_OK;
}

int mrb_batch_sync(mrb_batch* b) {
  mrb_ctx* ctx = b->ctx;
  try {
    ck(cudaSetDevice(ctx->device));
    ck(cudaStreamSynchronize(ctx->stream));
    if (b->pending_pm) {  // deferred coverage check (mrb_register_many)
      PixelMapJob& job = *b->pending_pm;
      bool located = false;
      ck(cudaEventSynchronize(job.done));
      for (size_t i = 0; i < job.todo.size(); ++i) located = located || job.missing[i] > 0;
      const std::string msg = finish_pixel_maps(ctx, job);
      b->pending_pm.reset();
      if (!msg.empty()) return fail(ctx, MRB_E_COVERAGE, msg);
      // a pixel the rasters left and the binned locate assigned: the dense
      // pass skipped it, so the caller reruns the batch undeferred
      if (located) b->redo = true;
    }
    b->h_st.resize(b->n_pairs);
    b->h_trace.resize(size_t(b->n_pairs) * b->cfg.max_iterations);
    ck(mrb_copy(b->h_st.data(), b->st, b->n_pairs * sizeof(PairStatus),
                  cudaMemcpyDeviceToHost));
    ck(mrb_copy(b->h_trace.data(), b->traces, b->h_trace.size() * sizeof(double),
                  cudaMemcpyDeviceToHost));
    b->synced = true;
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e, e.line);
  }
  for (int p = 0; p < b->n_pairs; ++p) {
    int code;
    const std::string msg = pair_message(b, p, &code);
    if (code != MRB_OK) return fail(ctx, code, msg);
  }
  return MRB_OK;
}

int mrb_batch_pair_status(mrb_batch* b, int32_t p, int32_t* iters, double* msd_before,
                          double* msd_after, double* trace, char* msg, int32_t msg_len) {
  if (!b->synced || p < 0 || p >= b->n_pairs) return MRB_E_VALUE;
  const PairStatus& s = b->h_st[p];
  if (iters) *iters = s.iters;
  if (msd_before) *msd_before = s.msd_before;
  if (msd_after) *msd_after = s.msd_after;
  if (trace)
    std::memcpy(trace, b->h_trace.data() + size_t(p) * b->cfg.max_iterations,
                size_t(b->cfg.max_iterations) * sizeof(double));
  int code;
  const std::string m = pair_message(b, p, &code);
  if (msg && msg_len > 0) {
    std::strncpy(msg, m.c_str(), size_t(msg_len) - 1);
    msg[msg_len - 1] = 0;
  }
  return code;
}

int64_t mrb_batch_launches_per_run(const mrb_batch* b) { return launches_per_run(b); }

const char* mrb_batch_loop_kernel(const mrb_batch* b) {
  if (b->c64_cs) return b->c64_push ? "k_cluster64_push" : "k_cluster64";
  if (!b->cluster_cs) return "k_sample";
  if (b->grid_mode) return b->grid_flags ? "k_grid_flags" : "k_grid_register";
  return b->push_mode ? "k_cluster_push" : "k_cluster_register";
}

int32_t mrb_batch_path(const mrb_batch* b) {
  if (b->c64_cs) return b->c64_cs;
  return b->grid_mode ? -b->cluster_cs : b->cluster_cs;
}

int mrb_transfer_bytes(int64_t* h2d, int64_t* d2h, int32_t reset) {
  if (h2d) *h2d = g_h2d_bytes.load();
  if (d2h) *d2h = g_d2h_bytes.load();
  if (reset) {
    g_h2d_bytes = 0;
    g_d2h_bytes = 0;
  }
  return MRB_OK;
}

// debug: phase timestamps of the cluster kernel (MESHREG_B200_PROFILE_PHASES)
int mrb_batch_phase_profile(mrb_batch* b, long long* out, int64_t n) {
  if (!b->phase_prof) return MRB_E_VALUE;
  const size_t cnt = std::min<size_t>(size_t(n), size_t(b->n_pairs) * b->cluster_cs * 8 * 16);
  if (b->prof_host) {  // mapped debug buffer: no CUDA call, usable during a hang
    std::memcpy(out, const_cast<const long long*>(b->prof_host), cnt * sizeof(long long));
    return MRB_OK;
  }
  try {
    ck(mrb_copy(out, b->phase_prof, cnt * sizeof(long long), cudaMemcpyDeviceToHost));
  } catch (const CudaError& e) {
    return cuda_fail(b->ctx, e.e, e.line);
  }
  return MRB_OK;
}

double mrb_batch_algorithmic_bytes(const mrb_batch* b) {
  // iterations*(184 n_V + 60 n_T + 8 n_E) + 128 W H per pair
  double tot = 0;
  for (const mrb_mesh* m : b->meshes)
    tot += double(b->cfg.max_iterations) *
               (184.0 * m->h.n + 60.0 * m->h.m + 8.0 * m->h.ne) +
           128.0 * double(b->W) * b->H;
  return tot;
}

int mrb_batch_kernel_bytes(const mrb_batch* b, double* out) {
  // SURVEY.md §8(d) per-unit figures split by the kernel that moves them:
  //   k_sample 148 B/node  (V 8, u 8, Te+Re 16 taps x 2 x 4 = 128, s_te 4)
  //   k_grad    16 B/node + 60 B/triangle (s_te read 4, avg indptr 4, u0 8;
  //             3 corner ids 12, 6 coefficients 24, 3 avg entries 24)
  //   k_smooth  20 B/node + 8 B/edge (u0 read 8, L indptr 4, u write 8; 2 ids)
  //   k_dense  128 B/pixel (B_final)
  double nv = 0, nt = 0, ne = 0;
  for (const mrb_mesh* m : b->meshes) {
    nv += double(m->h.n);
    nt += double(m->h.m);
    ne += double(m->h.ne);
  }
  out[0] = 148.0 * nv;
  out[1] = 16.0 * nv + 60.0 * nt;
  out[2] = 20.0 * nv + 8.0 * ne;
  out[3] = 128.0 * double(b->W) * b->H * b->n_pairs;
  if (b->cluster_cs || b->c64_cs) {  // one launch runs every iteration of every pair
    out[0] = double(b->cfg.max_iterations) * (184.0 * nv + 60.0 * nt + 8.0 * ne);
    out[1] = out[2] = 0.0;
  }
  return MRB_OK;
}

int mrb_batch_kernel_times(mrb_batch* b, double* out) {
  mrb_ctx* ctx = b->ctx;
  try {
    ck(cudaSetDevice(ctx->device));
    KernelTimer tm;
    tm.s = ctx->stream;
    tm.on = true;
    cudaEvent_t e0, e1;
    ck(cudaEventCreate(&e0));
    ck(cudaEventCreate(&e1));
    ck(cudaEventRecord(e0, ctx->stream));
    dispatch_enqueue(b, &tm);
    ck(cudaEventRecord(e1, ctx->stream));
    ck(cudaStreamSynchronize(ctx->stream));
    double sum[4] = {0, 0, 0, 0};
    int cnt[4] = {0, 0, 0, 0};
    for (size_t k = 1; k < tm.ev.size(); ++k) {
      float ms = 0;
      ck(cudaEventElapsedTime(&ms, tm.ev[k - 1], tm.ev[k]));
      sum[tm.kind[k]] += ms;
      cnt[tm.kind[k]]++;
    }
    for (int k = 0; k < 4; ++k) out[k] = cnt[k] ? sum[k] / cnt[k] : 0.0;
    float tot = 0;
    ck(cudaEventElapsedTime(&tot, e0, e1));
    out[4] = tot;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    b->synced = false;
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e, e.line);
  }
  return MRB_OK;
}

// ---------------------------------------------------------------- pipeline
static int register_many_impl(mrb_ctx* ctx, int32_t n_pairs, mrb_mesh* const* meshes, int32_t W,
                              int32_t H, int32_t img_dtype, const void* reference,
                              const void* tmpl, const mrb_config* cfg, int32_t chunk_pairs,
                              int32_t out_dtype, double* u, void* ux, void* uy, void* warped,
                              int32_t* iterations_run, double* msd_before, double* msd_after,
                              double* trace, int32_t* codes, char* messages, int32_t msg_len,
                              bool defer = true) {
  constexpr int kRedo = -1000;
  // Pipeline: chunk 0 is set up and launched on pipeline stream A.  For every
  // later chunk k the per-mesh device setup (mesh upload, pixel maps,
  // fast-path topologies) runs on the context's own stream while chunk k-1
  // computes on the other pipeline stream; the chunk's pipeline stream then
  // waits for that setup (event) and its batch creation is cheap.
  if (n_pairs < 1) return fail(ctx, MRB_E_VALUE, "batch needs at least one pair");
  const bool dbg = std::getenv("MESHREG_B200_DEBUG") != nullptr;
  const auto T0 = std::chrono::steady_clock::now();
  auto stamp = [&](const char* what, int k) {
    if (dbg)
      std::fprintf(stderr, "meshreg_b200: many %8.2f ms  %s %d\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - T0)
                       .count(),
                   what, k);
  };
  cudaEvent_t dbg_t0 = nullptr;  // device timeline origin (MESHREG_B200_DEBUG)
  if (dbg) {
    cudaSetDevice(ctx->device);
    cudaEventCreate(&dbg_t0);
    cudaEventRecord(dbg_t0, ctx->stream);
  }
  for (auto& c : ctx->sub)
    if (!c) {
      const int rc = mrb_ctx_create(ctx->device, &c);
      if (rc != MRB_OK) return fail(ctx, rc, "cannot create a pipeline stream");
    }
  // Deferred handles (mrb_mesh_create_many): the per-mesh setup runs on the
  // GPU (meshbuild.cuh) when the batch takes the fp32 cluster fast path; any
  // other batch gets the host build first.
  bool dev_setup = false, dev64 = false;  // dev64: the fp64 cluster path (k_cluster64)
  PixelMapJob early_pm;  // rasters of the device setup (chunk 0's batch adopts them)
  struct EarlyPmScope {
    PixelMapJob* prev;
    PixelMapJob* job;
    explicit EarlyPmScope(PixelMapJob* j) : prev(t_early_pm), job(j) { t_early_pm = j; }
    ~EarlyPmScope() {
      t_early_pm = prev;
      if (job->done) cudaEventDestroy(job->done);  // neither adopted nor finished (error)
    }
  } early_pm_scope(&early_pm);
  {
    bool any = false, fits = true;
    for (int p = 0; p < n_pairs; ++p) {
      const HostMesh& h = meshes[p]->h;
      if (!h.deferred) continue;
      any = true;
      fits = fits && (h.dev ? h.dev->b_nb_ptr != nullptr : device_buildable(h));
    }
    if (any) {
      std::vector<mrb_mesh*> all(meshes, meshes + n_pairs);
      const char* penv = std::getenv("MESHREG_B200_PATH");
      bool f64_ok = cfg->precision == MRB_PREC_F64 && !(penv && std::string(penv) == "generic");
      for (int p = 0; p < n_pairs && f64_ok; ++p)  // k_cluster64's limits (cluster64_candidate)
        f64_ok = meshes[p]->h.n <= 16 * kClusterThreads && meshes[p]->h.max_deg <= kMaxDeg;
      const char* why = nullptr;  // cluster (1) or whole-GPU grid (2) fp32 path
      const bool f32_ok = cfg->precision == MRB_PREC_F32 &&
                          fast_mode(false, false, img_dtype, all, &why) != 0;
      dev_setup = fits && config_error(cfg).empty() &&
                  img_dtype == MRB_F32 && (f32_ok || f64_ok);
      dev64 = dev_setup && f64_ok;
      if (!dev_setup) {
        if (const int rc = host_ready(ctx, meshes, n_pairs)) return rc;
      } else {
        std::vector<HostMesh*> todo;
        for (int p = 0; p < n_pairs; ++p) {
          HostMesh* h = &meshes[p]->h;
          if (device_buildable(*h) && std::find(todo.begin(), todo.end(), h) == todo.end())
            todo.push_back(h);
        }
        try {
          ck(cudaSetDevice(ctx->device));
          if (!ctx->copy) {
            ck(cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking));
            ck(cudaEventCreateWithFlags(&ctx->copy_done, cudaEventDisableTiming));
          }
          // V / T go first on the copy stream, ahead of the images
          device_build_meshes(ctx, todo, ctx->copy, dev64);
          stamp("device mesh build enqueued", 0);
        } catch (const CudaError& e) {
          return cuda_fail(ctx, e.e, e.line);
        }
      }
    }
  }
  // The fast-path cluster shape is decided once for the whole queue (cost
  // model with P = n_pairs) and imposed on every chunk.  Default chunk = one
  // wave of that shape (the pairs one launch keeps resident), so the chunks'
  // runs add up to the single-launch time while chunk k's host setup and
  // transfers overlap chunk k-1's run.
  int forced_cs = 0, forced_npt = 0, wave = 0;
  {
    std::vector<mrb_mesh*> all(meshes, meshes + n_pairs);
    const bool real_d = cfg->precision == MRB_PREC_F64;
    if (config_error(cfg).empty() && !cluster_ineligible(real_d, img_dtype == MRB_F64 && real_d,
                                                         img_dtype, all)) {
      mrb_mesh* big = *std::max_element(all.begin(), all.end(), [](mrb_mesh* x, mrb_mesh* y) {
        return x->h.n < y->h.n;
      });
      int occ = 0;
      try {
        AllocScope scope(ctx->stream);
        ck(cudaSetDevice(ctx->device));
        ensure_device_meshes(ctx, {&big->h}, false);
        if (!choose_cluster_shape(ctx, big->h, n_pairs, cfg->smoothing_passes >= 2, &forced_cs,
                                  &forced_npt, &occ))
          forced_cs = forced_npt = occ = 0;
      } catch (const CudaError& e) {
        return cuda_fail(ctx, e.e, e.line);
      }
      wave = occ;
    }
  }
  // default: one chunk (the per-chunk host setup costs more than a wave's
  // device time); within it, wave groups overlap results D2H with compute
  if (chunk_pairs <= 0) chunk_pairs = n_pairs;
  const size_t npx = size_t(W) * H, es = in_size(img_dtype), os = in_size(out_dtype);
  // Chunk 0's images: H2D issued now on the copy stream (behind the meshes'
  // V / T), one copy pair per wave group with an event each, so the device
  // setup overlaps them and group g's loop waits only for its own images.
  struct EarlyImages {
    char* dimg = nullptr;
    std::vector<cudaEvent_t> ev;
    ~EarlyImages() {
      for (cudaEvent_t e : ev) cudaEventDestroy(e);
    }
  } early;
  const bool no_groups = std::getenv("MESHREG_B200_NO_GROUPS") != nullptr;
  try {
    ck(cudaSetDevice(ctx->device));
    if (!ctx->copy) {
      ck(cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking));
      ck(cudaEventCreateWithFlags(&ctx->copy_done, cudaEventDisableTiming));
    }
    const int P0 = std::min<int>(chunk_pairs, n_pairs);
    const size_t img_bytes = size_t(P0) * npx * es;
    const int per = wave > 0 && P0 > wave && !no_groups ? wave : P0;
    AllocScope scope(ctx->copy);
    early.dimg = static_cast<char*>(kept_buffer(ctx, kKeptImages, 2 * img_bytes));
    for (int a = 0; a < P0; a += per) {
      const int e = std::min(P0, a + per);
      const size_t o = size_t(a) * npx * es, len = size_t(e - a) * npx * es;
      ck(mrb_copy_async(early.dimg + o, static_cast<const char*>(reference) + o, len,
                        cudaMemcpyHostToDevice, ctx->copy));
      ck(mrb_copy_async(early.dimg + img_bytes + o, static_cast<const char*>(tmpl) + o, len,
                        cudaMemcpyHostToDevice, ctx->copy));
      cudaEvent_t ev;
      ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      early.ev.push_back(ev);
      ck(cudaEventRecord(ev, ctx->copy));
    }
    ck(cudaEventRecord(ctx->copy_done, ctx->copy));
    dev_mark(ctx->copy, "images H2D done");
    stamp("images enqueued", 0);
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e, e.line);
  }
  if (dev_setup) {
    // every fast-path topology the run uses, planned and written on the GPU
    // now: the main shape for the pairs of full waves, the latency shape of
    // the tail wave (setup_tail) for the rest
    try {
      AllocScope scope(ctx->stream);
      if (forced_cs) {
        int planned = n_pairs;
        if (chunk_pairs >= n_pairs && forced_npt == 2 && wave > 0 && n_pairs > wave &&
            n_pairs % wave && !std::getenv("MESHREG_B200_NO_TAIL"))
          planned = n_pairs - n_pairs % wave;
        std::vector<std::tuple<HostMesh*, int, int>> req;
        for (int p = 0; p < planned; ++p) req.emplace_back(&meshes[p]->h, forced_cs, forced_npt);
        if (planned < n_pairs) {
          mrb_mesh* big = *std::max_element(
              meshes + planned, meshes + n_pairs,
              [](mrb_mesh* x, mrb_mesh* y) { return x->h.n < y->h.n; });
          int tcs = 0, tnpt = 0, tocc = 0;
          const bool tail = choose_cluster_shape(ctx, big->h, n_pairs - planned,
                                                 cfg->smoothing_passes >= 2, &tcs, &tnpt, &tocc,
                                                 1) &&
                            tnpt == 1;
          for (int p = planned; p < n_pairs; ++p)
            req.emplace_back(&meshes[p]->h, tail ? tcs : forced_cs, tail ? 1 : forced_npt);
        }
        device_cluster_topos(ctx, req, ctx->stream);  // false: planned later (host)
        stamp("device topologies", 0);
      } else if (!dev64) {
        // whole-GPU grid path (setup_grid_path): the grid shape of the
        // largest mesh, every mesh's topology of it
        std::vector<mrb_mesh*> all(meshes, meshes + n_pairs);
        const char* why = nullptr;
        if (fast_mode(false, false, img_dtype, all, &why) == 2) {
          int64_t nmax = 0;
          for (mrb_mesh* m : all) nmax = std::max<int64_t>(nmax, m->h.n);
          int gcs = 0, gnpt = 0;
          grid_shape(nmax, &gcs, &gnpt);
          std::vector<std::tuple<HostMesh*, int, int>> req;
          for (int p = 0; p < n_pairs; ++p) req.emplace_back(&meshes[p]->h, gcs, gnpt);
          device_cluster_topos(ctx, req, ctx->stream);
          stamp("device grid topologies", 0);
        }
      } else if (dev64) {
        // fp64 cluster size by setup_cluster64's cost model on the largest
        // mesh (waves x nodes per CTA), then every mesh's topology of it
        mrb_mesh* big = *std::max_element(meshes, meshes + n_pairs,
                                          [](mrb_mesh* x, mrb_mesh* y) { return x->h.n < y->h.n; });
        const int64_t nmax = big->h.n;
        const int cs_min = int((nmax + kClusterThreads - 1) / kClusterThreads);
        std::vector<std::tuple<HostMesh*, int, int>> cand;
        for (int cs = cs_min; cs <= 16; ++cs) cand.emplace_back(&big->h, cs, 1);
        if (device_cluster_topos(ctx, cand, ctx->stream, true)) {
          double best = 1e300;
          int best_cs = 0;
          const bool two_u = cfg->smoothing_passes >= 2;
          for (int cs = cs_min; cs <= 16; ++cs) {
            const DeviceMesh::Topo& t =
                big->h.dev->topo.at(topo64_key(cs, int((nmax + cs - 1) / cs)));
            const int occ = cluster64_occupancy<1>(
                cs, cluster64_dyn_smem(t.topo_stride, t.slices, t.halo_stride, two_u));
            if (occ < 1) continue;
            const double cost = double((n_pairs + occ - 1) / occ) * double((nmax + cs - 1) / cs);
            if (cost < best) {
              best = cost;
              best_cs = cs;
            }
          }
          if (best_cs) {
            std::vector<std::tuple<HostMesh*, int, int>> req;
            for (int p = 0; p < n_pairs; ++p) req.emplace_back(&meshes[p]->h, best_cs, 1);
            device_cluster_topos(ctx, req, ctx->stream, true);
            forced_cs = best_cs;  // setup_cluster64 takes it
            forced_npt = 1;
          }
        }
        stamp("device fp64 topologies", 0);
      }
      const std::string e = device_build_finish(ctx);
      if (!e.empty()) return fail(ctx, MRB_E_VALUE, e);
      {  // pixel maps: rasters on the side stream now, beside the topology
         // writes and the host's batch setup (chunk 0's batch adopts them)
        std::vector<HostMesh*> all_h;
        bool built = true;
        for (int p = 0; p < n_pairs; ++p) {
          all_h.push_back(&meshes[p]->h);
          built = built && meshes[p]->h.dev;
        }
        if (built) early_pm = issue_pixel_maps(ctx, all_h, W, H, true, ctx->build_ev);
      }
      // the build arrays go back to the pool now (stream-ordered) for this
      // call's batch buffers; a later topology of another shape for these
      // meshes is planned on the host
      for (int p = 0; p < n_pairs; ++p) {
        HostMesh& h = meshes[p]->h;
        if (h.dev && h.dev->b_nb_ptr) {
          h.dev->b_nb_ptr = nullptr;
          h.dev->b_nb_idx = nullptr;
          h.dev->b_g_nb = nullptr;
          h.dev->build_hold.reset();
        }
      }
    } catch (const CudaError& e) {
      return cuda_fail(ctx, e.e, e.line);
    }
  }
  std::vector<mrb_batch*> live;  // batches in flight, freed once harvested
  std::vector<std::pair<int, int>> span;
  int first_err = MRB_OK;
  std::string first_msg;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> dbg_events;  // run of each chunk
  std::vector<cudaEvent_t> dbg_done;                             // results of each chunk
  auto harvest = [&](size_t k) {  // wait for chunk k and collect its statuses
    mrb_batch* b = live[k];
    if (!b) return;
    stamp("harvest begin", int(k));
    const int rc = mrb_batch_sync(b);
    if (dbg && k < dbg_events.size()) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, dbg_events[k].first, dbg_events[k].second);
      float t_start = 0.f, t_end = 0.f, t_done = 0.f;
      cudaEventElapsedTime(&t_start, dbg_t0, dbg_events[k].first);
      cudaEventElapsedTime(&t_end, dbg_t0, dbg_events[k].second);
      if (k < dbg_done.size()) cudaEventElapsedTime(&t_done, dbg_t0, dbg_done[k]);
      std::fprintf(stderr,
                   "meshreg_b200: many chunk %zu run %.2f ms (path %d x %d); device timeline: "
                   "run %.2f -> %.2f ms, results %.2f ms\n",
                   k, ms, b->cluster_cs, b->cluster_npt, t_start, t_end, t_done);
      for (size_t g = 0; g < b->dbg_group_ev.size(); ++g) {
        float tg = 0.f;
        cudaEventElapsedTime(&tg, dbg_t0, b->dbg_group_ev[g]);
        std::fprintf(stderr, "meshreg_b200:   group %zu launch reached at %.2f ms\n", g, tg);
      }
      for (auto& mk : dev_marks()) {
        float tm = 0.f;
        if (cudaEventElapsedTime(&tm, dbg_t0, mk.second) == cudaSuccess)
          std::fprintf(stderr, "meshreg_b200:   device: %-20s at %.2f ms\n", mk.first.c_str(), tm);
        cudaEventDestroy(mk.second);
      }
      dev_marks().clear();
    }
    if ((rc == MRB_E_CUDA || rc == MRB_E_COVERAGE || b->redo) && first_err == MRB_OK) {
      first_err = b->redo ? kRedo : rc;
      first_msg = b->ctx->err;
    }
    if (b->synced) {
      for (int q = 0; q < b->n_pairs; ++q) {
        const int p = span[k].first + q;
        char buf[512];
        const int code = mrb_batch_pair_status(
            b, q, iterations_run ? iterations_run + p : nullptr,
            msd_before ? msd_before + p : nullptr, msd_after ? msd_after + p : nullptr,
            trace ? trace + size_t(p) * cfg->max_iterations : nullptr, buf, sizeof buf);
        if (codes) codes[p] = code;
        if (messages && msg_len > 0) {
          std::strncpy(messages + size_t(p) * msg_len, buf, size_t(msg_len) - 1);
          messages[size_t(p) * msg_len + msg_len - 1] = 0;
        }
        if (code != MRB_OK && first_err == MRB_OK) {
          first_err = code;
          first_msg = buf;
        }
      }
    }
    mrb_batch_destroy(b);
    live[k] = nullptr;
  };
  cudaEvent_t setup_done = nullptr;
  int cs = 0, npt = 0;
  size_t node_off = 0;
  try {
    ck(cudaSetDevice(ctx->device));
    ck(cudaEventCreateWithFlags(&setup_done, cudaEventDisableTiming));
    for (int p0 = 0, k = 0; p0 < n_pairs; p0 += chunk_pairs, ++k) {
      const int P = std::min<int>(chunk_pairs, n_pairs - p0);
      mrb_ctx* sc = ctx->sub[k & 1];
      std::vector<HostMesh*> hm;
      for (int q = 0; q < P; ++q) hm.push_back(&meshes[p0 + q]->h);
      if (k > 0) {
        // per-mesh setup on the context stream, overlapping chunk k-1's run
        stamp("setup begin", k);
        AllocScope scope(ctx->stream);
        ensure_device_meshes(ctx, hm, cs == 0);
        stamp("  meshes", k);
        if (cs == 0)
          for (HostMesh* h : hm) ensure_device_mesh_ring(ctx, *h);
        const std::string msg = ensure_pixel_maps(ctx, hm, W, H);
        stamp("  pixel maps", k);
        if (!msg.empty()) {
          for (size_t j = 0; j < live.size(); ++j) harvest(j);
          cudaEventDestroy(setup_done);
          return fail(ctx, MRB_E_COVERAGE, msg);
        }
        if (cs) ensure_cluster_topos(ctx, hm, cs, npt);
        ck(cudaEventRecord(setup_done, ctx->stream));
        stamp("setup end", k);
        if (k >= 2) harvest(size_t(k - 2));  // the pipeline stream's previous chunk
        ck(cudaStreamWaitEvent(sc->stream, setup_done, 0));
      }
      // images: their H2D starts on the context's copy stream before the
      // (host-bound) batch setup, so the copy overlaps it; the pipeline
      // stream waits for it just before the run
      const size_t img_bytes = size_t(P) * npx * es;
      char* dimg = k == 0 ? early.dimg : nullptr;
      if (!dimg) {
        if (!ctx->copy) {
          ck(cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking));
          ck(cudaEventCreateWithFlags(&ctx->copy_done, cudaEventDisableTiming));
        }
        AllocScope scope(ctx->copy);
        dimg = dalloc<char>(2 * img_bytes);
        ck(mrb_copy_async(dimg, static_cast<const char*>(reference) + size_t(p0) * npx * es,
                          img_bytes, cudaMemcpyHostToDevice, ctx->copy));
        ck(mrb_copy_async(dimg + img_bytes, static_cast<const char*>(tmpl) + size_t(p0) * npx * es,
                          img_bytes, cudaMemcpyHostToDevice, ctx->copy));
        ck(cudaEventRecord(ctx->copy_done, ctx->copy));
        dev_mark(ctx->copy, "images H2D done");
      }
      mrb_batch* b = nullptr;
      stamp("create begin", k);
      const bool grouped = wave > 0 && P > wave && !no_groups;
      int rc = batch_create_impl(sc, P, meshes + p0, W, H, img_dtype, cfg, forced_cs, forced_npt,
                                 &b, grouped && defer ? wave : 0);
      stamp("create end", k);
      if (rc == MRB_OK && k == 0) {
        cs = b->cluster_cs;
        npt = b->cluster_npt;
      }
      // chunk 0's per-group image events go to the batch (its run waits for
      // them); otherwise the run waits for all images
      const bool group_images = k == 0 && early.ev.size() > 1;
      if (!group_images) cudaStreamWaitEvent(sc->stream, ctx->copy_done, 0);
      if (rc == MRB_OK) rc = mrb_batch_set_images(b, dimg, dimg + img_bytes, 1);
      if (rc == MRB_OK && grouped) {
        try {
          batch_set_groups(b, wave);
        } catch (const CudaError& e) {
          rc = cuda_fail(sc, e.e, e.line);
        }
      }
      if (group_images) {  // only the fp32 fast path pads per group (enqueue_run)
        if (rc == MRB_OK && b->cluster_cs && !b->real_d && b->in_dtype == MRB_F32)
          b->img_ev = early.ev;
        else
          cudaStreamWaitEvent(sc->stream, ctx->copy_done, 0);
      }
      cudaEvent_t ev_run[2] = {nullptr, nullptr};
      if (dbg && rc == MRB_OK) {
        for (auto& e : ev_run) cudaEventCreate(&e);
        cudaEventRecord(ev_run[0], sc->stream);
      }
      if (rc == MRB_OK) rc = mrb_batch_run(b);
      if (dbg && ev_run[1]) {
        cudaEventRecord(ev_run[1], sc->stream);
        dbg_events.push_back({ev_run[0], ev_run[1]});
      }
      // stream-ordered free after the run consumed it; unconditionally after
      // the H2D into it, even when the batch could not be created
      if (group_images) cudaStreamWaitEvent(sc->stream, ctx->copy_done, 0);
      if (dimg != early.dimg) cudaFreeAsync(dimg, sc->stream);  // chunk 0's are kept
      if (rc == MRB_OK) {
        auto off = [&](void* base) -> void* {
          return base ? static_cast<char*>(base) + size_t(p0) * npx * os : nullptr;
        };
        rc = mrb_batch_get_results(b, out_dtype, u ? u + 2 * node_off : nullptr, off(ux), off(uy),
                                   off(warped));
        if (dbg) {
          cudaEvent_t e;
          cudaEventCreate(&e);
          cudaEventRecord(e, sc->stream);
          dbg_done.push_back(e);
        }
      }
      stamp("enqueued", k);
      for (int q = 0; q < P; ++q) node_off += size_t(meshes[p0 + q]->h.n);
      live.push_back(b);
      span.emplace_back(p0, P);
      if (rc != MRB_OK) {
        const std::string m = sc->err;
        for (size_t j = 0; j < live.size(); ++j) harvest(j);
        cudaEventDestroy(setup_done);
        return fail(ctx, rc, m);
      }
    }
  } catch (const CudaError& e) {
    for (size_t j = 0; j < live.size(); ++j) harvest(j);
    if (setup_done) cudaEventDestroy(setup_done);
    return cuda_fail(ctx, e.e, e.line);
  }
  for (size_t j = 0; j < live.size(); ++j) harvest(j);
  cudaEventDestroy(setup_done);
  if (!early_pm.todo.empty()) {  // early rasters no batch took over: check them here
    try {
      const std::string m = finish_pixel_maps(ctx, early_pm);
      if (!m.empty() && first_err == MRB_OK) {
        first_err = MRB_E_COVERAGE;
        first_msg = m;
      }
    } catch (const CudaError& e) {
      return cuda_fail(ctx, e.e, e.line);
    }
  }
  for (auto& e : dbg_events) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  for (cudaEvent_t e : dbg_done) cudaEventDestroy(e);
  if (dbg_t0) cudaEventDestroy(dbg_t0);
  if (first_err == kRedo)  // see mrb_batch::redo: rerun with the blocking coverage check
    return register_many_impl(ctx, n_pairs, meshes, W, H, img_dtype, reference, tmpl, cfg,
                              chunk_pairs, out_dtype, u, ux, uy, warped, iterations_run,
                              msd_before, msd_after, trace, codes, messages, msg_len, false);
  if (first_err != MRB_OK) return fail(ctx, first_err, first_msg);
  return MRB_OK;
}

// Every pair gets a status: pairs the run never reached (an early failure —
// invalid config, coverage, a CUDA error in the shape probe or a later
// chunk) carry the call's own error code and message instead of a stale
// zero (MRB_OK) that would read as success.
int mrb_register_many(mrb_ctx* ctx, int32_t n_pairs, mrb_mesh* const* meshes, int32_t W,
                      int32_t H, int32_t img_dtype, const void* reference, const void* tmpl,
                      const mrb_config* cfg, int32_t chunk_pairs, int32_t out_dtype, double* u,
                      void* ux, void* uy, void* warped, int32_t* iterations_run,
                      double* msd_before, double* msd_after, double* trace, int32_t* codes,
                      char* messages, int32_t msg_len) {
  constexpr int32_t kUnset = INT32_MIN;
  if (codes)
    for (int32_t p = 0; p < n_pairs; ++p) codes[p] = kUnset;
  // no dense outputs wanted: rasters and dense passes fill the idle SMs (ctx->fill_idle)
  const bool fill = !ux && !uy && !warped;
  auto set_fill = [&](bool v) {
    ctx->fill_idle = v;
    for (mrb_ctx* c : ctx->sub)
      if (c) c->fill_idle = v;
  };
  for (auto& c : ctx->sub)  // the pipeline contexts exist before the flag is set on them
    if (!c && mrb_ctx_create(ctx->device, &c) != MRB_OK) c = nullptr;
  set_fill(fill);
  const int rc = register_many_impl(ctx, n_pairs, meshes, W, H, img_dtype, reference, tmpl, cfg,
                                    chunk_pairs, out_dtype, u, ux, uy, warped, iterations_run,
                                    msd_before, msd_after, trace, codes, messages, msg_len);
  set_fill(false);
  if (codes) {
    const std::string msg =
        rc != MRB_OK ? std::string(ctx->err) : std::string("internal error: pair not run");
    for (int32_t p = 0; p < n_pairs; ++p) {
      if (codes[p] != kUnset) continue;
      codes[p] = rc != MRB_OK ? rc : MRB_E_INTERNAL;
      if (messages && msg_len > 0) {
        std::strncpy(messages + size_t(p) * msg_len, msg.c_str(), size_t(msg_len) - 1);
        messages[size_t(p) * msg_len + msg_len - 1] = 0;
      }
    }
  }
  return rc;
}

// ---------------------------------------------------------------- register
int mrb_register(mrb_ctx* ctx, mrb_mesh* mesh, int32_t W, int32_t H, int32_t img_dtype,
                 const void* re, const void* te, const mrb_config* cfg, double* u,
                 double* trace, int32_t* iters, double* msd_before, double* msd_after,
                 double* ux, double* uy, double* warped) {
  mrb_batch* b = nullptr;
  int rc = mrb_batch_create(ctx, 1, &mesh, W, H, img_dtype, cfg, &b);
  if (rc != MRB_OK) return rc;
  std::unique_ptr<mrb_batch> guard(b);
  if ((rc = mrb_batch_set_images(b, re, te, 0)) != MRB_OK) return rc;
  if ((rc = mrb_batch_run(b)) != MRB_OK) return rc;
  if ((rc = mrb_batch_get_results(b, MRB_F64, u, ux, uy, warped)) != MRB_OK) return rc;
  rc = mrb_batch_sync(b);
  if (b->synced) mrb_batch_pair_status(b, 0, iters, msd_before, msd_after, trace, nullptr, 0);
  return rc;
}

// ---------------------------------------------------------------- single ops
int mrb_warp_sample(mrb_ctx* ctx, int32_t W, int32_t H, int32_t dtype, const void* image,
                    int64_t n, const double* V, const double* u, double* out) {
  if (W < 2 || H < 2)
    return fail(ctx, MRB_E_VALUE, "bicubic sampling needs an image of at least 2x2 pixels");
  try {
    ck(cudaSetDevice(ctx->device));
    Tmp t(ctx->stream);
    const size_t npx = size_t(W) * H;
    const double* dV = t.up(V, 2 * n);
    const double* du = t.up(u, 2 * n);
    double* dout = t.get<double>(n);
    const unsigned g = unsigned((n + 255) / 256);
    if (n > 0) {
      if (dtype == MRB_F64)
        k_sample_points<double><<<g, 256, 0, ctx->stream>>>(
            t.up(static_cast<const double*>(image), npx), W, H, int(n), dV, du, dout);
      else
        k_sample_points<float><<<g, 256, 0, ctx->stream>>>(
            t.up(static_cast<const float*>(image), npx), W, H, int(n), dV, du, dout);
      ck(cudaGetLastError());
    }
    ck(mrb_copy_async(out, dout, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ck(cudaStreamSynchronize(ctx->stream));
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e, e.line);
  }
  return MRB_OK;
}

namespace {

// One-pair f64 evaluation of (energy, grad) at a given u through the same
// k_sample / k_grad kernels the registration loop uses.
int unit_eval(mrb_ctx* ctx, mrb_mesh* mesh, int32_t W, int32_t H, int32_t dtype, const void* re,
              const void* te, const double* u, const double* f_override, double* energy,
              double* grad) {
  if (W < 2 || H < 2)
    return fail(ctx, MRB_E_VALUE, "bicubic sampling needs an image of at least 2x2 pixels");
  if (const int rc = host_ready(ctx, &mesh, 1)) return rc;
  try {
    ck(cudaSetDevice(ctx->device));
    HostMesh& h = mesh->h;
    ensure_device_mesh_f64(ctx, h);
    DeviceMesh& dm = *h.dev;
    cudaStream_t s = ctx->stream;
    Tmp t(s);
    const size_t n = size_t(h.n), npx = size_t(W) * H;
    using PD = PairDev<double, double>;
    PD d{};
    d.V = dm.V;
    d.nb_ptr = dm.nb_ptr;
    d.nb_idx = dm.nb_idx;
    d.g_self = dm.g_self_d;
    d.g_nb = dm.g_nb_d;
    d.inv_val = dm.inv_val_d;
    d.W = W;
    d.H = H;
    d.n = int(n);
    d.blk_begin = 0;
    d.nblk = int((n + kNodeBlock - 1) / kNodeBlock);
    std::vector<double> tmp(2 * n);
    if (u)
      for (size_t k = 0; k < n; ++k) {
        tmp[2 * k] = u[2 * h.perm[k]];
        tmp[2 * k + 1] = u[2 * h.perm[k] + 1];
      }
    d.u = reinterpret_cast<double2*>(t.up(tmp.data(), 2 * n));
    d.ste = t.get<double>(n);
    d.r = t.get<double>(n);
    d.trace = t.get<double>(1);
    d.grad_out = grad ? t.get<double2>(n) : nullptr;
    PairStatus st0{};
    st0.stop_iter = 1;
    PairStatus* st = t.up(&st0, 1);
    std::vector<int> bp(d.nblk, 0);
    int* blk_pair = t.up(bp.data(), bp.size());
    double* partials = t.get<double>(d.nblk);
    if (f_override) {  // vertex_gradient_all: ste = f, r = 1
      std::vector<double> f(n), one(n, 1.0);
      for (size_t k = 0; k < n; ++k) f[k] = f_override[h.perm[k]];
      ck(mrb_copy_async(d.ste, f.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
      ck(mrb_copy_async(d.r, one.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
      PD* dd = t.up(&d, 1);
      k_grad<double, double><<<d.nblk, kNodeBlock, 0, s>>>(dd, st, blk_pair, 0, 0.0, 0);
      ck(cudaGetLastError());
    } else {
      // interleave (Te, Re) into f64 taps
      double* img = t.get<double>(2 * npx);
      std::vector<double> inter(2 * npx);
      for (size_t q = 0; q < npx; ++q) {
        inter[2 * q] = dtype == MRB_F64 ? static_cast<const double*>(te)[q]
                                        : double(static_cast<const float*>(te)[q]);
        inter[2 * q + 1] = dtype == MRB_F64 ? static_cast<const double*>(re)[q]
                                            : double(static_cast<const float*>(re)[q]);
      }
      ck(mrb_copy_async(img, inter.data(), 2 * npx * sizeof(double), cudaMemcpyHostToDevice, s));
      d.img = img;
      PD* dd = t.up(&d, 1);
      k_sample<double, double><<<d.nblk, kNodeBlock, 0, s>>>(dd, st, blk_pair, partials, 0, 0.0);
      ck(cudaGetLastError());
      if (grad) {
        // k_grad skips pairs whose status says stop; force it to run
        ck(mrb_copy_async(st, &st0, sizeof st0, cudaMemcpyHostToDevice, s));
        k_grad<double, double><<<d.nblk, kNodeBlock, 0, s>>>(dd, st, blk_pair, 0, 0.0, 0);
        ck(cudaGetLastError());
      }
    }
    if (energy) ck(mrb_copy_async(energy, d.trace, sizeof(double), cudaMemcpyDeviceToHost, s));
    if (grad) {
      ck(mrb_copy_async(tmp.data(), d.grad_out, 2 * n * sizeof(double), cudaMemcpyDeviceToHost, s));
      ck(cudaStreamSynchronize(s));
      for (size_t k = 0; k < n; ++k) {
        grad[2 * h.perm[k]] = tmp[2 * k];
        grad[2 * h.perm[k] + 1] = tmp[2 * k + 1];
      }
    }
    ck(cudaStreamSynchronize(s));
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e, e.line);
  }
  return MRB_OK;
}

}  // namespace

int mrb_energy(mrb_ctx* ctx, mrb_mesh* mesh, int32_t W, int32_t H, int32_t dtype,
               const void* re, const void* te, const double* u, double* out) {
  return unit_eval(ctx, mesh, W, H, dtype, re, te, u, nullptr, out, nullptr);
}

int mrb_energy_gradient(mrb_ctx* ctx, mrb_mesh* mesh, int32_t W, int32_t H, int32_t dtype,
                        const void* re, const void* te, const double* u, double* grad) {
  return unit_eval(ctx, mesh, W, H, dtype, re, te, u, nullptr, nullptr, grad);
}

int mrb_vertex_gradient_all(mrb_ctx* ctx, mrb_mesh* mesh, const double* f, double* out) {
  return unit_eval(ctx, mesh, 2, 2, MRB_F64, nullptr, nullptr, nullptr, f, nullptr, out);
}

namespace {
int csr_smooth_impl(mrb_ctx* ctx, Tmp& t, int64_t n, const int64_t* indptr,
                    const int64_t* indices, const double* data, double2* cur, double lam,
                    int32_t passes, double2** result) {
  const int64_t nnz = indptr[n];
  const int64_t* dp = t.up(indptr, n + 1);
  const int64_t* di = t.up(indices, nnz);
  const double* dd = t.up(data, nnz);
  double2* other = t.get<double2>(n);
  const unsigned g = unsigned((n + 255) / 256);
  for (int q = 0; q < passes; ++q) {
    if (n > 0) k_csr_smooth<<<g, 256, 0, ctx->stream>>>(int(n), dp, di, dd, cur, lam, other);
    std::swap(cur, other);
  }
  ck(cudaGetLastError());
  *result = cur;
  return MRB_OK;
}
}  // namespace

int mrb_smooth_csr(mrb_ctx* ctx, int64_t n, const int64_t* indptr, const int64_t* indices,
                   const double* data, const double* u0, double lam, int32_t passes,
                   double* out) {
  if (!(0.0 < lam && lam < 1.0))
    return fail(ctx, MRB_E_VALUE, "smoothing weight must be in (0, 1), got " + py_repr(lam));
  if (passes < 0) return fail(ctx, MRB_E_VALUE, "iterations must be >= 0");
  try {
    ck(cudaSetDevice(ctx->device));
    Tmp t(ctx->stream);
    double2* cur = reinterpret_cast<double2*>(t.up(u0, 2 * n));
    double2* res = nullptr;
    csr_smooth_impl(ctx, t, n, indptr, indices, data, cur, lam, passes, &res);
    ck(mrb_copy_async(out, res, n * sizeof(double2), cudaMemcpyDeviceToHost, ctx->stream));
    ck(cudaStreamSynchronize(ctx->stream));
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e, e.line);
  }
  return MRB_OK;
}

int mrb_step_csr(mrb_ctx* ctx, int64_t n, const int64_t* indptr, const int64_t* indices,
                 const double* data, const double* u, const double* grad, double tau, double lam,
                 int32_t passes, const double* V, int32_t W, int32_t H, double* out) {
  try {
    ck(cudaSetDevice(ctx->device));
    Tmp t(ctx->stream);
    const double2* du = reinterpret_cast<const double2*>(t.up(u, 2 * n));
    const double2* dg = reinterpret_cast<const double2*>(t.up(grad, 2 * n));
    double2* u0 = t.get<double2>(n);
    int* bad = t.get<int>(1);
    ck(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
    const unsigned g = unsigned((n + 255) / 256);
    if (n > 0) k_descent<<<g, 256, 0, ctx->stream>>>(int(n), du, dg, tau, u0, bad);
    ck(cudaGetLastError());
    int hbad = 0;
    ck(mrb_copy_async(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    ck(cudaStreamSynchronize(ctx->stream));
    if (hbad) return fail(ctx, MRB_E_DIVERGED, "non-finite gradient; reduce the step size tau");
    double2* res = u0;
    if (passes > 0) {
      if (!(0.0 < lam && lam < 1.0))
        return fail(ctx, MRB_E_VALUE, "smoothing weight must be in (0, 1), got " + py_repr(lam));
      csr_smooth_impl(ctx, t, n, indptr, indices, data, u0, lam, passes, &res);
    }
    if (V && n > 0) {
      k_clamp<<<g, 256, 0, ctx->stream>>>(int(n), reinterpret_cast<const double2*>(t.up(V, 2 * n)),
                                          W, H, res);
      ck(cudaGetLastError());
    }
    ck(mrb_copy_async(out, res, n * sizeof(double2), cudaMemcpyDeviceToHost, ctx->stream));
    ck(cudaStreamSynchronize(ctx->stream));
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e, e.line);
  }
  return MRB_OK;
}

int mrb_densify(mrb_ctx* ctx, mrb_mesh* mesh, int32_t W, int32_t H, const double* u, double* ux,
                double* uy) {
  if (const int rc = host_ready(ctx, &mesh, 1)) return rc;
  try {
    AllocScope scope(ctx->stream);
    ck(cudaSetDevice(ctx->device));
    HostMesh& h = mesh->h;
    int* map = nullptr;
    const std::string msg = ensure_pixel_map(ctx, h, W, H, &map);
    if (!msg.empty()) return fail(ctx, MRB_E_COVERAGE, msg);
    Tmp t(ctx->stream);
    std::vector<double> un(2 * h.n);
    for (int64_t k = 0; k < h.n; ++k) {
      un[2 * k] = u[2 * h.perm[k]];
      un[2 * k + 1] = u[2 * h.perm[k] + 1];
    }
    const double2* du = reinterpret_cast<const double2*>(t.up(un.data(), un.size()));
    const size_t npx = size_t(W) * H;
    double* dx = t.get<double>(npx);
    double* dy = t.get<double>(npx);
    k_densify<<<unsigned((npx + 255) / 256), 256, 0, ctx->stream>>>(h.dev->V, h.dev->tri, map, du,
                                                                    W, int(npx), dx, dy);
    ck(cudaGetLastError());
    ck(mrb_copy_async(ux, dx, npx * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ck(mrb_copy_async(uy, dy, npx * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ck(cudaStreamSynchronize(ctx->stream));
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e, e.line);
  }
  return MRB_OK;
}

int mrb_warp_image(mrb_ctx* ctx, int32_t W, int32_t H, int32_t dtype, const void* te,
                   const double* ux, const double* uy, double* out) {
  if (W < 2 || H < 2)
    return fail(ctx, MRB_E_VALUE, "bicubic sampling needs an image of at least 2x2 pixels");
  try {
    ck(cudaSetDevice(ctx->device));
    Tmp t(ctx->stream);
    const size_t npx = size_t(W) * H;
    const double* dx = t.up(ux, npx);
    const double* dy = t.up(uy, npx);
    double* dout = t.get<double>(npx);
    const unsigned g = unsigned((npx + 255) / 256);
    if (dtype == MRB_F64)
      k_warp_image<double><<<g, 256, 0, ctx->stream>>>(t.up(static_cast<const double*>(te), npx),
                                                       W, H, dx, dy, dout);
    else
      k_warp_image<float><<<g, 256, 0, ctx->stream>>>(t.up(static_cast<const float*>(te), npx), W,
                                                      H, dx, dy, dout);
    ck(cudaGetLastError());
    ck(mrb_copy_async(out, dout, npx * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ck(cudaStreamSynchronize(ctx->stream));
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e, e.line);
  }
  return MRB_OK;
}

int mrb_msd(mrb_ctx* ctx, int64_t n, const double* a, const double* b, double* out) {
  try {
    ck(cudaSetDevice(ctx->device));
    Tmp t(ctx->stream);
    const double* da = t.up(a, n);
    const double* db = t.up(b, n);
    const int nb = int((n + kPixBlock - 1) / kPixBlock);
    double* partials = t.get<double>(std::max(nb, 1));
    double* dout = t.get<double>(1);
    if (nb > 0) k_sqdiff_partials<<<nb, kPixBlock, 0, ctx->stream>>>(int(n), da, db, partials);
    k_sum_final<<<1, kPixBlock, 0, ctx->stream>>>(nb, partials, double(n), dout);
    ck(cudaGetLastError());
    ck(mrb_copy_async(out, dout, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ck(cudaStreamSynchronize(ctx->stream));
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e, e.line);
  }
  return MRB_OK;
}

}  // extern "C"

// pixel-grid engine (baseline.py)
#include "pixel_api.cuh"

// content-adaptive mesher (meshgen.py, delaunay.py)
#include "mesher.cuh"
