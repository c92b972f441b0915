// Host side of the pixel-grid engine (reference baseline.py:46-118).  Part of
// the meshreg_b200.cu translation unit (included at its end) so it shares the
// allocator, copy counters and error helpers.
#pragma once

struct mrb_pixel_batch {
  mrb_ctx* ctx = nullptr;
  int n_pairs = 0, W = 0, H = 0, in_dtype = MRB_F32;
  mrb_pixel_config cfg{};
  bool real_d = false;
  int tiles_x = 0, tiles = 0, warp_blocks = 0;
  void* pairs = nullptr;       // PixelDev<Real>[n_pairs]
  PairStatus* st = nullptr;
  double* partials = nullptr;  // [pair][iteration][tile]
  double2* msd_partials = nullptr;
  double* traces = nullptr;
  void* img = nullptr;         // padded (Te, Re) per pair
  int pitch = 0;               // padded row pitch (R2 elements)
  size_t img_stride = 0;       // R2 elements between pairs
  CUtensorMap* tmaps = nullptr;  // device: TMA descriptors, image + planes per pair
  void* u = nullptr;           // [pair][H*W] final (ux, uy)
  void* wbuf = nullptr;        // [2][pair][H*wpitch] descended (ux, uy)
  int wpitch = 0;
  void* warped = nullptr;      // [pair][H*W]
  void* stage = nullptr;
  void* conv = nullptr;
  const void** src_ptrs = nullptr;  // device: re[0..P), te[0..P)
  std::vector<const void*> src_host;
  cudaGraphExec_t graph = nullptr;
  int runs = 0, final_src = 0;
  std::vector<PairStatus> h_st;
  std::vector<double> h_trace;
  bool synced = false;
  ~mrb_pixel_batch() {
    if (graph) cudaGraphExecDestroy(graph);
    void* ptrs[] = {pairs, st, partials, msd_partials, traces, img, u, wbuf, warped, stage, conv,
                    const_cast<void**>(src_ptrs), tmaps};
    for (void* p : ptrs) dev_free(p, ctx ? ctx->stream : nullptr);
  }
};

namespace {

std::string pixel_config_error(const mrb_pixel_config* c) {
  // baseline.py:59-64
  if (!(c->tau > 0)) return "tau must be positive, got " + py_repr(c->tau);
  if (!(0.0 <= c->lam && c->lam < 1.0)) return "lambda must be in [0, 1), got " + py_repr(c->lam);
  if (c->iterations < 1) return "iterations must be >= 1";
  return "";
}

// smoothing passes applied per iteration (range(negative) is empty)
int pixel_passes(const mrb_pixel_config& c) {
  return c.lam > 0.0 ? std::max(c.smoothing_passes, 0) : 0;
}

// extra smoothing launches (passes beyond kPixMaxR) before each step launch
// after the first
int pixel_extra_launches(const mrb_pixel_config& c) {
  const int p = pixel_passes(c);
  return p <= kPixMaxR ? 0 : (p - kPixMaxR + kPixMaxR - 1) / kPixMaxR;
}

// k_pixel_step launches per run: iteration 0 (sample only), iterations
// 1..n-1 and the final smoothing (each after its extra launches)
int64_t pixel_step_launches(const mrb_pixel_config& c) {
  return int64_t(c.iterations) + 1 + int64_t(c.iterations) * pixel_extra_launches(c);
}

template <typename Real>
size_t pixel_tile_counts(int W, int H, int* tiles_x) {
  *tiles_x = (W + PixTile<Real>::TX - 1) / PixTile<Real>::TX;
  return size_t(*tiles_x) * ((H + PixTile<Real>::TY - 1) / PixTile<Real>::TY);
}

template <typename Real>
PixelStepArgs<Real> pixel_step_args(const mrb_pixel_batch* b) {
  using R2 = typename V2<Real>::type;
  PixelStepArgs<Real> a{};
  a.img = static_cast<const R2*>(b->img);
  a.tmap = b->tmaps;
  a.w = static_cast<R2*>(b->wbuf);
  a.u = static_cast<R2*>(b->u);
  a.partials = b->partials;
  a.img_stride = b->img_stride;
  a.wplane = size_t(b->wpitch) * b->H;
  a.n = b->n_pairs;
  a.iterations = b->cfg.iterations;
  a.W = b->W;
  a.H = b->H;
  a.pitch = b->pitch;
  a.wpitch = b->wpitch;
  a.tiles_x = b->tiles_x;
  a.tiles = b->tiles;
  return a;
}

template <typename Real>
void launch_pixel_step(const mrb_pixel_batch* b, const PixelStepArgs<Real>& pairs, int k, int src,
                       Real tau, Real lam, int r, int load, int clamp, int sample,
                       int final_out) {
  const dim3 grid(b->tiles_x, b->tiles / b->tiles_x, b->n_pairs);
  cudaStream_t s = b->ctx->stream;
#define MRB_PIX_LAUNCH(RR)                                                          \
  k_pixel_step<Real, RR><<<grid, kPixThreads, PixPatch<Real>::smem_bytes, s>>>(     \
      pairs, k, src, tau, lam, load, clamp, sample, final_out)
  switch (r) {
    case 0: MRB_PIX_LAUNCH(0); break;
    case 1: MRB_PIX_LAUNCH(1); break;
    case 2: MRB_PIX_LAUNCH(2); break;
    default: MRB_PIX_LAUNCH(3); break;
  }
#undef MRB_PIX_LAUNCH
}

template <typename Real, int RR>
void pixel_smem_attr() {
  ck(cudaFuncSetAttribute(k_pixel_step<Real, RR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          int(PixPatch<Real>::smem_bytes)));
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    ck(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw CudaError{cudaErrorNotSupported};
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

template <typename Real>
void pixel_enqueue_t(mrb_pixel_batch* b, KernelTimer* tm) {
  using R2 = typename V2<Real>::type;
  cudaStream_t s = b->ctx->stream;
  const int n = b->n_pairs, W = b->W, H = b->H;
  const size_t npx = size_t(W) * H, npad = size_t(W + 2) * (H + 2);
  const auto* pairs = static_cast<const PixelDev<Real>*>(b->pairs);
  const PixelStepArgs<Real> args = pixel_step_args<Real>(b);
  {
    const unsigned g = unsigned(std::min<size_t>((npad + 255) / 256, 1024));
    if (b->in_dtype == MRB_F64)
      k_pixel_pad<double, Real><<<dim3(g, n), 256, 0, s>>>(
          reinterpret_cast<const double* const*>(b->src_ptrs),
          reinterpret_cast<const double* const*>(b->src_ptrs) + n, W, H, b->pitch,
          static_cast<R2*>(b->img), b->img_stride);
    else
      k_pixel_pad<float, Real><<<dim3(g, n), 256, 0, s>>>(
          reinterpret_cast<const float* const*>(b->src_ptrs),
          reinterpret_cast<const float* const*>(b->src_ptrs) + n, W, H, b->pitch,
          static_cast<R2*>(b->img), b->img_stride);
    ck(cudaGetLastError());
  }
  const int passes = pixel_passes(b->cfg);
  const Real tau = Real(b->cfg.tau), lam = Real(b->cfg.lam);
  const int r_last = std::min(passes, kPixMaxR);  // passes of each step launch
  const bool dbg = std::getenv("MESHREG_B200_DEBUG") != nullptr;
  int src = 1;  // descended planes of the previous launch: w[src]
  for (int k = 0; k <= b->cfg.iterations; ++k) {
    if (k > 0) {  // extra smoothing launches (passes beyond kPixMaxR)
      for (int rem = passes - r_last; rem > 0;) {
        const int r = std::min(rem, kPixMaxR);
        rem -= r;
        launch_pixel_step<Real>(b, args, k, src, tau, lam, r, 1, 0, 0, 0);
        src ^= 1;
      }
    }
    const bool last = k == b->cfg.iterations;
    if (tm && !last) tm->mark(0);
    // iteration 0 samples u = 0; iteration k > 0 smooths + clamps the
    // previous descent first; the final launch only smooths + clamps
    launch_pixel_step<Real>(b, args, k, src, tau, lam, k > 0 ? r_last : 0, k > 0, k > 0,
                            !last, last);
    if (tm && !last) tm->mark(1);
    if (dbg) {
      ck(cudaStreamSynchronize(s));
      ck(cudaGetLastError());
    }
    src ^= 1;
  }
  ck(cudaGetLastError());
  b->final_src = 0;
  k_pixel_trace<Real><<<n, kPixBlock, 0, s>>>(pairs, b->cfg.iterations, b->traces, b->st);
  k_pixel_warp<Real><<<dim3(b->warp_blocks, n), kPixBlock, 0, s>>>(pairs, 0, b->st,
                                                                   b->msd_partials,
                                                                   b->warp_blocks);
  k_pixel_msd<<<n, kPixBlock, 0, s>>>(b->msd_partials, b->warp_blocks, double(npx), b->st);
  ck(cudaGetLastError());
}

void pixel_enqueue(mrb_pixel_batch* b, KernelTimer* tm = nullptr) {
  if (b->real_d)
    pixel_enqueue_t<double>(b, tm);
  else
    pixel_enqueue_t<float>(b, tm);
}

template <typename Real>
void pixel_setup_t(mrb_pixel_batch* b) {
  using R2 = typename V2<Real>::type;
  cudaStream_t s = b->ctx->stream;
  const int n = b->n_pairs;
  const size_t npx = size_t(b->W) * b->H, npad = size_t(b->W + 2) * (b->H + 2);
  b->tiles = int(pixel_tile_counts<Real>(b->W, b->H, &b->tiles_x));
  b->warp_blocks = int((npx + kPixBlock - 1) / kPixBlock);
  // rows padded to a 16-byte multiple (TMA global stride rule)
  b->pitch = sizeof(R2) == 8 ? (b->W + 2 + 1) / 2 * 2 : b->W + 2;
  b->img_stride = size_t(b->pitch) * (b->H + 2);
  b->img = dalloc<R2>(size_t(n) * b->img_stride);
  ck(cudaMemsetAsync(b->img, 0, size_t(n) * b->img_stride * sizeof(R2), s));  // pitch pad
  pixel_smem_attr<Real, 0>();
  pixel_smem_attr<Real, 1>();
  pixel_smem_attr<Real, 2>();
  pixel_smem_attr<Real, 3>();
  b->u = dalloc<R2>(size_t(n) * npx);
  // descended planes: rows padded to a 16-byte multiple (TMA global stride)
  b->wpitch = sizeof(R2) == 8 ? (b->W + 1) / 2 * 2 : b->W;
  const size_t wplane = size_t(b->wpitch) * b->H;
  b->wbuf = dalloc<R2>(2 * size_t(n) * wplane);
  b->warped = dalloc<Real>(size_t(n) * npx);
  b->partials = dalloc<double>(size_t(n) * b->cfg.iterations * b->tiles);
  b->msd_partials = dalloc<double2>(size_t(n) * b->warp_blocks);
  b->traces = dalloc<double>(size_t(n) * b->cfg.iterations);
  b->st = dalloc<PairStatus>(n);
  b->src_ptrs = dalloc<const void*>(2 * size_t(n));
  std::vector<PixelDev<Real>> h(n);
  std::vector<CUtensorMap> maps(2 * size_t(n));
  b->tmaps = dalloc<CUtensorMap>(2 * size_t(n));
  for (int p = 0; p < n; ++p) {
    PixelDev<Real>& d = h[p];
    d.img = static_cast<const R2*>(b->img) + size_t(p) * b->img_stride;
    // 2-D view of the padded image in Real elements, (2 * pitch) x (H + 2);
    // box = the k_pixel_step image patch (same for every halo R)
    // (8-byte elements: one per float2, two per double2)
    constexpr int epr = int(sizeof(R2) / 8);
    const cuuint64_t gdim[2] = {cuuint64_t(epr) * b->pitch, cuuint64_t(b->H + 2)};
    const cuuint64_t gstride[1] = {cuuint64_t(b->pitch) * sizeof(R2)};
    const cuuint32_t box[2] = {cuuint32_t(epr * PixPatch<Real>::PW),
                               cuuint32_t(PixPatch<Real>::PH)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult cr = encode_tiled()(
        &maps[p], CU_TENSOR_MAP_DATA_TYPE_UINT64,
        2, const_cast<R2*>(d.img), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) throw CudaError{cudaErrorInvalidValue};
    d.tmap = b->tmaps + p;
    // 3-D view of the descended planes (x, y, buffer): W x H x 2 with the row
    // pitch wpitch (columns >= W read as zero), box = the state buffer
    R2* w0 = static_cast<R2*>(b->wbuf) + size_t(p) * wplane;
    const cuuint64_t udim[3] = {cuuint64_t(epr) * b->W, cuuint64_t(b->H), 2};
    const cuuint64_t ustride[2] = {cuuint64_t(b->wpitch) * sizeof(R2),
                                   cuuint64_t(n) * wplane * sizeof(R2)};
    const cuuint32_t ubox[3] = {cuuint32_t(epr * PixPatch<Real>::BW),
                                cuuint32_t(PixPatch<Real>::BH), 1};
    const cuuint32_t ustr[3] = {1, 1, 1};
    const CUresult cu = encode_tiled()(
        &maps[n + p], CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, w0, udim, ustride, ubox, ustr,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cu != CUDA_SUCCESS) throw CudaError{cudaErrorInvalidValue};

    d.pitch = b->pitch;
    d.u = static_cast<R2*>(b->u) + size_t(p) * npx;
    d.warped = static_cast<Real*>(b->warped) + size_t(p) * npx;
    d.partials = b->partials + size_t(p) * b->cfg.iterations * b->tiles;
    d.W = b->W;
    d.H = b->H;
    d.tiles_x = b->tiles_x;
    d.tiles = b->tiles;
  }
  b->pairs = dalloc<PixelDev<Real>>(n);
  ck(mrb_copy_async(b->pairs, h.data(), n * sizeof(PixelDev<Real>), cudaMemcpyHostToDevice, s));
  ck(mrb_copy_async(b->tmaps, maps.data(), 2 * n * sizeof(CUtensorMap), cudaMemcpyHostToDevice,
                    s));
  ck(cudaStreamSynchronize(s));  // h is a stack temporary
}

template <typename Real, typename Out>
__global__ void k_pixel_split(const typename V2<Real>::type* __restrict__ u, Out* __restrict__ ux,
                              Out* __restrict__ uy, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const auto v = u[i];
    if (ux) ux[i] = Out(v.x);
    if (uy) uy[i] = Out(v.y);
  }
}

std::string pixel_message(const mrb_pixel_batch* b, int p, int* code) {
  const PairStatus& s = b->h_st[p];
  *code = MRB_OK;
  switch (s.err) {  // baseline.py:81-88
    case ERR_NONFINITE_ENERGY:
      *code = MRB_E_DIVERGED;
      return "energy became non-finite; reduce tau";
    case ERR_RISES:
      *code = MRB_E_DIVERGED;
      return "energy increased for 10 consecutive iterations; reduce tau";
    default:
      break;
  }
  if (s.dense_nonfinite) {  // PixelField(ux, uy) / warp_image, baseline.py:103-104
    *code = MRB_E_VALUE;
    return (s.dense_nonfinite & 1) ? "displacement planes must be finite"
                                   : "image intensities must be finite";
  }
  return "";
}

}  // namespace

extern "C" {

int mrb_pixel_batch_create(mrb_ctx* ctx, int32_t n_pairs, int32_t W, int32_t H,
                           int32_t img_dtype, const mrb_pixel_config* cfg,
                           mrb_pixel_batch** out) {
  *out = nullptr;
  const std::string ce = pixel_config_error(cfg);
  if (!ce.empty()) return fail(ctx, MRB_E_VALUE, ce);
  if (n_pairs < 1) return fail(ctx, MRB_E_VALUE, "n_pairs must be >= 1");
  if (W < 2 || H < 2)
    return fail(ctx, MRB_E_VALUE, "bicubic sampling needs an image of at least 2x2 pixels");
  if (img_dtype != MRB_F32 && img_dtype != MRB_F64)
    return fail(ctx, MRB_E_VALUE, "image dtype must be MRB_F32 or MRB_F64");
  auto b = std::make_unique<mrb_pixel_batch>();
  b->ctx = ctx;
  b->n_pairs = n_pairs;
  b->W = W;
  b->H = H;
  b->in_dtype = img_dtype;
  b->cfg = *cfg;
  b->real_d = cfg->precision == MRB_PREC_F64;
  AllocScope scope(ctx->stream);
  try {
    ck(cudaSetDevice(ctx->device));
    if (b->real_d)
      pixel_setup_t<double>(b.get());
    else
      pixel_setup_t<float>(b.get());
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e);
  }
  *out = b.release();
  return MRB_OK;
}

int mrb_pixel_batch_destroy(mrb_pixel_batch* b) {
  delete b;
  return MRB_OK;
}

int mrb_pixel_batch_set_images(mrb_pixel_batch* b, const void* re, const void* te,
                               int32_t on_device) {
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
    if (ptrs != b->src_host) {
      ck(mrb_copy_async(b->src_ptrs, ptrs.data(), ptrs.size() * sizeof(void*),
                        cudaMemcpyHostToDevice, ctx->stream));
      ck(cudaStreamSynchronize(ctx->stream));  // ptrs is a stack temporary
      b->src_host = ptrs;
    }
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e);
  }
  return MRB_OK;
}

int mrb_pixel_batch_run(mrb_pixel_batch* b) {
  mrb_ctx* ctx = b->ctx;
  if (b->src_host.empty()) return fail(ctx, MRB_E_VALUE, "images not set");
  try {
    ck(cudaSetDevice(ctx->device));
    b->synced = false;
    if (b->runs == 0) {
      pixel_enqueue(b);  // first run: direct launches
    } else {
      if (!b->graph) {  // the iteration loop as one CUDA graph
        cudaGraph_t g;
        ck(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
        pixel_enqueue(b);
        ck(cudaStreamEndCapture(ctx->stream, &g));
        ck(cudaGraphInstantiate(&b->graph, g, 0));
        cudaGraphDestroy(g);
      }
      ck(cudaGraphLaunch(b->graph, ctx->stream));
    }
    b->runs++;
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e);
  }
  return MRB_OK;
}

int mrb_pixel_batch_get_results(mrb_pixel_batch* b, int32_t out_dtype, void* ux, void* uy,
                                void* warped) {
  mrb_ctx* ctx = b->ctx;
  AllocScope scope(ctx->stream);
  try {
    ck(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const size_t n = size_t(b->n_pairs) * b->W * b->H, os = in_size(out_dtype);
    const size_t rs = b->real_d ? sizeof(double) : sizeof(float);
    if (!b->conv) b->conv = dalloc<char>(3 * n * sizeof(double));
    char* cv = static_cast<char*>(b->conv);
    const unsigned g = unsigned(std::min<size_t>((n + 255) / 256, 4096));
    const void* u = static_cast<const char*>(b->u) + size_t(b->final_src) * n * 2 * rs;
    if (ux || uy) {
      void* cx = ux ? cv : nullptr;
      void* cy = uy ? cv + n * os : nullptr;
      if (b->real_d && out_dtype == MRB_F64)
        k_pixel_split<double, double><<<g, 256, 0, s>>>(static_cast<const double2*>(u),
                                                        static_cast<double*>(cx),
                                                        static_cast<double*>(cy), n);
      else if (b->real_d)
        k_pixel_split<double, float><<<g, 256, 0, s>>>(static_cast<const double2*>(u),
                                                       static_cast<float*>(cx),
                                                       static_cast<float*>(cy), n);
      else if (out_dtype == MRB_F64)
        k_pixel_split<float, double><<<g, 256, 0, s>>>(static_cast<const float2*>(u),
                                                       static_cast<double*>(cx),
                                                       static_cast<double*>(cy), n);
      else
        k_pixel_split<float, float><<<g, 256, 0, s>>>(static_cast<const float2*>(u),
                                                      static_cast<float*>(cx),
                                                      static_cast<float*>(cy), n);
      ck(cudaGetLastError());
      if (ux) ck(mrb_copy_async(ux, cx, n * os, cudaMemcpyDeviceToHost, s));
      if (uy) ck(mrb_copy_async(uy, cy, n * os, cudaMemcpyDeviceToHost, s));
    }
    if (warped) {
      const void* src = b->warped;
      if ((out_dtype == MRB_F64) != b->real_d) {
        char* cw = cv + 2 * n * os;
        if (b->real_d)
          k_convert<double, float><<<g, 256, 0, s>>>(static_cast<const double*>(b->warped),
                                                     reinterpret_cast<float*>(cw), n);
        else
          k_convert<float, double><<<g, 256, 0, s>>>(static_cast<const float*>(b->warped),
                                                     reinterpret_cast<double*>(cw), n);
        ck(cudaGetLastError());
        src = cw;
      }
      ck(mrb_copy_async(warped, src, n * os, cudaMemcpyDeviceToHost, s));
    }
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e);
  }
  return MRB_OK;
}

int mrb_pixel_batch_sync(mrb_pixel_batch* b) {
  mrb_ctx* ctx = b->ctx;
  try {
    ck(cudaSetDevice(ctx->device));
    ck(cudaStreamSynchronize(ctx->stream));
    b->h_st.resize(b->n_pairs);
    b->h_trace.resize(size_t(b->n_pairs) * b->cfg.iterations);
    ck(mrb_copy(b->h_st.data(), b->st, b->n_pairs * sizeof(PairStatus), cudaMemcpyDeviceToHost));
    ck(mrb_copy(b->h_trace.data(), b->traces, b->h_trace.size() * sizeof(double),
                cudaMemcpyDeviceToHost));
    b->synced = true;
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e);
  }
  for (int p = 0; p < b->n_pairs; ++p) {
    int code;
    const std::string msg = pixel_message(b, p, &code);
    if (code != MRB_OK) return fail(ctx, code, msg);
  }
  return MRB_OK;
}

int mrb_pixel_batch_pair_status(mrb_pixel_batch* b, int32_t p, int32_t* iters,
                                double* msd_before, double* msd_after, double* trace, char* msg,
                                int32_t msg_len) {
  if (!b->synced || p < 0 || p >= b->n_pairs) return MRB_E_VALUE;
  const PairStatus& s = b->h_st[p];
  // len(trace): iterations completed before a DivergenceError
  const int n_tr = s.err ? s.err_iter : s.iters;
  if (iters) *iters = n_tr;
  if (msd_before) *msd_before = s.msd_before;
  if (msd_after) *msd_after = s.msd_after;
  if (trace)
    std::memcpy(trace, b->h_trace.data() + size_t(p) * b->cfg.iterations,
                size_t(b->cfg.iterations) * sizeof(double));
  int code;
  const std::string m = pixel_message(b, p, &code);
  if (msg && msg_len > 0) {
    std::strncpy(msg, m.c_str(), size_t(msg_len) - 1);
    msg[msg_len - 1] = 0;
  }
  return code;
}

int64_t mrb_pixel_batch_launches_per_run(const mrb_pixel_batch* b) {
  return 4 + pixel_step_launches(b->cfg);
}

int mrb_pixel_batch_kernel_times(mrb_pixel_batch* b, double* out) {
  mrb_ctx* ctx = b->ctx;
  try {
    ck(cudaSetDevice(ctx->device));
    KernelTimer tm{ctx->stream};
    tm.on = true;
    cudaEvent_t e0, e1;
    ck(cudaEventCreate(&e0));
    ck(cudaEventCreate(&e1));
    ck(cudaEventRecord(e0, ctx->stream));
    pixel_enqueue(b, &tm);
    ck(cudaEventRecord(e1, ctx->stream));
    ck(cudaEventSynchronize(e1));
    double it = 0;
    int cnt = 0;
    for (size_t i = 0; i + 1 < tm.ev.size(); ++i)
      if (tm.kind[i] == 0 && tm.kind[i + 1] == 1) {
        float ms;
        ck(cudaEventElapsedTime(&ms, tm.ev[i], tm.ev[i + 1]));
        it += ms;
        ++cnt;
      }
    float tot;
    ck(cudaEventElapsedTime(&tot, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    out[0] = cnt ? it / cnt : 0.0;
    out[1] = tot;
    b->synced = false;
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e);
  }
  return MRB_OK;
}

int mrb_register_pixelwise(mrb_ctx* ctx, int32_t W, int32_t H, int32_t img_dtype,
                           const void* re, const void* te, const mrb_pixel_config* cfg,
                           double* ux, double* uy, double* warped, double* trace,
                           int32_t* iters, double* msd_before, double* msd_after) {
  mrb_pixel_batch* b = nullptr;
  int rc = mrb_pixel_batch_create(ctx, 1, W, H, img_dtype, cfg, &b);
  if (rc != MRB_OK) return rc;
  std::unique_ptr<mrb_pixel_batch> guard(b);
  if ((rc = mrb_pixel_batch_set_images(b, re, te, 0)) != MRB_OK) return rc;
  if ((rc = mrb_pixel_batch_run(b)) != MRB_OK) return rc;
  if ((rc = mrb_pixel_batch_get_results(b, MRB_F64, ux, uy, warped)) != MRB_OK) return rc;
  rc = mrb_pixel_batch_sync(b);
  if (b->synced) mrb_pixel_batch_pair_status(b, 0, iters, msd_before, msd_after, trace, nullptr, 0);
  return rc;
}

int mrb_sample_gradient(mrb_ctx* ctx, int32_t W, int32_t H, int32_t dtype, const void* image,
                        int64_t n, const double* pts, double* gx, double* gy) {
  if (W < 2 || H < 2)
    return fail(ctx, MRB_E_VALUE, "bicubic sampling needs an image of at least 2x2 pixels");
  try {
    ck(cudaSetDevice(ctx->device));
    Tmp t(ctx->stream);
    const size_t npx = size_t(W) * H;
    const double* dp = t.up(pts, 2 * n);
    double* dgx = t.get<double>(n);
    double* dgy = t.get<double>(n);
    if (n > 0) {
      const unsigned g = unsigned((n + 255) / 256);
      if (dtype == MRB_F64)
        k_sample_gradient_points<double><<<g, 256, 0, ctx->stream>>>(
            t.up(static_cast<const double*>(image), npx), W, H, int(n), dp, dgx, dgy);
      else
        k_sample_gradient_points<float><<<g, 256, 0, ctx->stream>>>(
            t.up(static_cast<const float*>(image), npx), W, H, int(n), dp, dgx, dgy);
      ck(cudaGetLastError());
    }
    ck(mrb_copy_async(gx, dgx, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ck(mrb_copy_async(gy, dgy, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ck(cudaStreamSynchronize(ctx->stream));
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e);
  }
  return MRB_OK;
}

int mrb_grid_umbrella_smooth(mrb_ctx* ctx, int32_t W, int32_t H, const double* plane, double lam,
                             double* out) {
  if (W < 1 || H < 1) return fail(ctx, MRB_E_VALUE, "plane must be non-empty");
  try {
    ck(cudaSetDevice(ctx->device));
    Tmp t(ctx->stream);
    const size_t npx = size_t(W) * H;
    const double* dp = t.up(plane, npx);
    double* dout = t.get<double>(npx);
    k_grid_umbrella<<<unsigned((npx + 255) / 256), 256, 0, ctx->stream>>>(dp, W, H, lam, dout);
    ck(cudaGetLastError());
    ck(mrb_copy_async(out, dout, npx * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ck(cudaStreamSynchronize(ctx->stream));
  } catch (const CudaError& e) {
    return cuda_fail(ctx, e.e);
  }
  return MRB_OK;
}

}  // extern "C"
