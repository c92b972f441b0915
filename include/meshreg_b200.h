/*
 * meshreg_b200.h — C ABI of the B200-native mesh-registration hot path.
 *
 * The reference (`meshreg`, a pure-Python package) has no plugin/FFI layer:
 * its boundary for this path is the Python API re-exported by
 * pkg/src/meshreg/__init__.py:12-60.  Each entry point here
 * is what a ctypes binding of that API would call; the Python package
 * `paper_1411_2141_b200` is that binding and mirrors the reference names,
 * argument meaning and exceptions.  All pointers are plain host pointers
 * unless an argument says "device"; sizes are element counts.
 *
 * Return codes map 1:1 onto the reference's exceptions:
 *   MRB_OK            success
 *   MRB_E_VALUE       ValueError          (solver.py:158-161, mesh.py:61-123,
 *                                          densefield.py:139-140,192-193,
 *                                          image.py:183-184)
 *   MRB_E_DIVERGED    DivergenceError     (solver.py:33-34,131-132,176-184)
 *   MRB_E_COVERAGE    MeshCoverageError   (densefield.py:58-59,127)
 *   MRB_E_CUDA        CUDA runtime failure / no device
 * The human-readable message (same text as the reference exception) is
 * available from mrb_last_error(ctx) or the per-pair status call.
 */
#ifndef MESHREG_B200_H
#define MESHREG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MRB_OK 0
#define MRB_E_VALUE 1
#define MRB_E_DIVERGED 2
#define MRB_E_COVERAGE 3
#define MRB_E_CUDA 4
#define MRB_E_INTERNAL 5

/* image / output element types */
#define MRB_F32 0
#define MRB_F64 1

/* arithmetic precision of the iteration state (mrb_config.precision) */
#define MRB_PREC_F32 0 /* fp32 state + fp32 math, fp64 energy/MSD reductions */
#define MRB_PREC_F64 1 /* fp64 state + fp64 math (fp32 taps when exact)      */

/* which CSR operator mrb_mesh_export_csr returns */
#define MRB_CSR_LAPLACIAN 0 /* build_laplacian, mesh.py:254-265              */
#define MRB_CSR_GRAD_X 1    /* TriangleGeometry.grad_x_op, mesh.py:203-205    */
#define MRB_CSR_GRAD_Y 2    /* TriangleGeometry.grad_y_op, mesh.py:206-208    */
#define MRB_CSR_VERTEX_AVG 3 /* TriangleGeometry.vertex_average_op, 210-213   */

typedef struct mrb_ctx mrb_ctx;
typedef struct mrb_mesh mrb_mesh;
typedef struct mrb_batch mrb_batch;
typedef struct mrb_pixel_batch mrb_pixel_batch;

/* SolverConfig, reference solver.py:47-68 (validated the same way). */
typedef struct mrb_config {
  double tau;
  double lam;
  double energy_tolerance;
  int32_t max_iterations;
  int32_t smoothing_passes;
  int32_t precision; /* MRB_PREC_* */
  int32_t reserved;
} mrb_config;

/* register_pixelwise keyword arguments, reference baseline.py:46-64 */
typedef struct mrb_pixel_config {
  double tau;
  double lam;                /* [0, 1); 0 disables smoothing               */
  int32_t iterations;
  int32_t smoothing_passes;  /* grid_umbrella_smooth passes per iteration   */
  int32_t precision;         /* MRB_PREC_*                                  */
  int32_t reserved;
} mrb_pixel_config;

/* ---- library / context ------------------------------------------------ */
const char* mrb_version(void);
/* One context per GPU: owns a non-blocking CUDA stream.  Not thread-safe;
 * separate contexts may be driven from separate threads or processes. */
int mrb_ctx_create(int32_t device, mrb_ctx** out);
int mrb_ctx_destroy(mrb_ctx* ctx);
const char* mrb_last_error(const mrb_ctx* ctx);
/* the cudaStream_t every call of this ctx is enqueued on (for CUDA events) */
void* mrb_ctx_stream(mrb_ctx* ctx);
int mrb_ctx_synchronize(mrb_ctx* ctx);

/* ---- mesh (replaces TriMesh + TriangleGeometry + build_laplacian) ------ */
/* Validates, orients CCW and builds connectivity/CSR/geometry on the host,
 * bit-exact with TriMesh.__init__ (mesh.py:58-123) and TriangleGeometry
 * (mesh.py:173-213).  Host-only: works without a GPU.  On failure returns
 * MRB_E_VALUE and writes the reference's message into err (if non-NULL). */
int mrb_mesh_build(int64_t n_vertices, const double* vertices /* n*2 */,
                   int64_t n_triangles, const int64_t* triangles /* m*3 */,
                   mrb_mesh** out, char* err, int32_t err_len);
/* mrb_mesh_build for `count` meshes at once on the library's host worker
 * pool (no reference counterpart: the reference builds one TriMesh at a time,
 * mesh.py:58).  All or nothing: on the first failing mesh (lowest index) every
 * out[k] is NULL, *first_bad = its index and err holds its message. */
int mrb_mesh_build_many(int32_t count, const int64_t* n_vertices,
                        const double* const* vertices, const int64_t* n_triangles,
                        const int64_t* const* triangles, mrb_mesh** out,
                        int32_t* first_bad, char* err, int32_t err_len);
int mrb_mesh_destroy(mrb_mesh* mesh);
/* Deferred mesh handles (no reference counterpart: the reference builds a
 * TriMesh per mesh on the host, mesh.py:58-123).  Only the checks that need no
 * connectivity run here (mesh.py:61-86: finite coordinates, index range,
 * repeated indices, degenerate area; same messages), plus the CCW
 * reorientation.  The connectivity, geometry, node order, fused operator and
 * fast-path topology are built on the GPU by the first mrb_register_many that
 * runs the handle on the fp32 cluster fast path (bit-identical to
 * mrb_mesh_build's); every other consumer (exports, single operations,
 * mrb_batch_create, other paths) runs the host build first, and a mesh the
 * reference would reject (non-manifold edge, valence < 2) fails there with the
 * reference's message.  All or nothing, like mrb_mesh_build_many. */
int mrb_mesh_create_many(int32_t count, const int64_t* n_vertices,
                         const double* const* vertices, const int64_t* n_triangles,
                         const int64_t* const* triangles, mrb_mesh** out,
                         int32_t* first_bad, char* err, int32_t err_len);
/* Test hook: builds a deferred mesh and its (cs, npt) cluster topology on the
 * GPU and compares them with the host build.  out[0..9] = mismatching
 * elements of: device-order vertices, triangles, node order, fp32 G self
 * terms, fp32 1/valence, (max valence, edge count), one-ring CSR row
 * pointers, one-ring CSR indices, fp64 G ring terms, topology bytes (-1 if
 * the layout sizes differ). */
int mrb_mesh_device_check(mrb_ctx* ctx, mrb_mesh* mesh, int32_t cluster_size,
                          int32_t nodes_per_thread, int64_t* out);
/* counts[0..5] = n_vertices, n_triangles, n_edges, nnz(L), nnz(grad), nnz(avg) */
int mrb_mesh_counts(const mrb_mesh* mesh, int64_t* counts);
/* oriented triangles (m*3), edges (e*2), valence (n), boundary (n bytes),
 * rings CSR (n+1, 2e) and incident-triangle CSR (n+1, 3m); any may be NULL */
int mrb_mesh_export_connectivity(const mrb_mesh* mesh, int64_t* triangles, int64_t* edges,
                                 int64_t* valence, uint8_t* boundary, int64_t* ring_ptr,
                                 int64_t* ring_idx, int64_t* inc_ptr, int64_t* inc_idx);
/* canonical scipy CSR (indptr, indices, data) of one MRB_CSR_* operator */
int mrb_mesh_export_csr(const mrb_mesh* mesh, int32_t which, int64_t* indptr,
                        int64_t* indices, double* data);
/* areas (m), coeffs (m*3*2), vertex_areas (n) */
int mrb_mesh_export_geometry(const mrb_mesh* mesh, double* areas, double* coeffs,
                             double* vertex_areas);
/* Pixel -> lowest-index containing triangle and barycentric weights
 * (densefield.py:148-182), rasterised on the GPU with fp64 predicates that
 * reproduce numpy's operation order; binned-locate fallback on the host. */
/* PointLocator + locate, densefield.py:62-127 (host, binned): for n points
 * (x, y) the lowest-index containing triangle (reference ids) or -1, and its
 * barycentric weights (n*3, may be NULL) */
int mrb_mesh_locate(mrb_mesh* mesh, int64_t n, const double* pts, int64_t* tri, double* w);
int mrb_pixel_map(mrb_ctx* ctx, mrb_mesh* mesh, int32_t width, int32_t height,
                  int64_t* tri_of /* H*W */, double* weights /* H*W*3, may be NULL */);

/* ---- the registration path (solver.register, solver.py:148-208) -------- */
/* One pair.  Images are row-major H*W in img_dtype.  Outputs (caller-owned
 * host memory, any may be NULL except u):
 *   u (n*2 f64, reference vertex order), trace (max_iterations f64),
 *   ux, uy, warped (H*W f64) — the dense field and warped template
 *   (densefield.py:130-199).  Returns MRB_E_DIVERGED / MRB_E_VALUE /
 *   MRB_E_COVERAGE with the reference's message on failure. */
int mrb_register(mrb_ctx* ctx, mrb_mesh* mesh, int32_t width, int32_t height,
                 int32_t img_dtype, const void* reference, const void* tmpl,
                 const mrb_config* cfg, double* u, double* trace, int32_t* iterations_run,
                 double* msd_before, double* msd_after, double* ux, double* uy,
                 double* warped);

/* Batched pairs (the pair queue of one GPU).  All pairs of a
 * batch share width/height/config; each has its own mesh.  Typical use:
 *   create -> set_images -> run -> get_results -> sync -> status   */
int mrb_batch_create(mrb_ctx* ctx, int32_t n_pairs, mrb_mesh* const* meshes, int32_t width,
                     int32_t height, int32_t img_dtype, const mrb_config* cfg,
                     mrb_batch** out);
int mrb_batch_destroy(mrb_batch* batch);
/* reference/template stacks (n_pairs*H*W, img_dtype).  on_device=0: host
 * memory (pinned for async), copied H2D on the ctx stream; on_device=1:
 * device pointers, copied D2D. */
int mrb_batch_set_images(mrb_batch* batch, const void* reference, const void* tmpl,
                         int32_t on_device);
/* enqueue the whole registration of every pair (loop + dense pass) */
int mrb_batch_run(mrb_batch* batch);
/* enqueue D2H copies of the results.  out_dtype applies to ux/uy/warped;
 * u is n_i*2 f64 per pair (concatenated in pair order).  NULL skips. */
int mrb_batch_get_results(mrb_batch* batch, int32_t out_dtype, double* u, void* ux, void* uy,
                          void* warped);
/* wait for the stream; returns the first pair error code (MRB_OK if none) */
int mrb_batch_sync(mrb_batch* batch);
/* per-pair outcome after sync: iterations_run, MSDs, trace (max_iterations),
 * message (reference text) — returns that pair's MRB_* code */
int mrb_batch_pair_status(mrb_batch* batch, int32_t pair, int32_t* iterations_run,
                          double* msd_before, double* msd_after, double* trace, char* msg,
                          int32_t msg_len);
/* execution path chosen for the batch: 0 = generic three-kernel loop; > 0 =
 * the cluster size of the persistent cluster kernel (fp32, <= 16 x 1536
 * nodes); < 0 = minus the CTA count of the whole-GPU persistent grid kernel
 * (fp32, larger meshes, one cooperative launch per pair) */
int32_t mrb_batch_path(const mrb_batch* batch);
/* name of the kernel that runs the descent loop: "k_cluster_register" (pull
 * halo exchange), "k_cluster_push" (push exchange), "k_grid_flags" /
 * "k_grid_register" (whole-GPU grid), "k_sample" (generic three-kernel loop) */
const char* mrb_batch_loop_kernel(const mrb_batch* batch);
/* debug: per-CTA phase timestamps of the cluster kernel (first 8 iterations,
 * 16 slots each) when MESHREG_B200_PROFILE_PHASES is set at batch creation */
int mrb_batch_phase_profile(mrb_batch* batch, long long* out, int64_t n);
/* host->device and device->host bytes copied by the library in this process
 * since the last reset (the benchmark's e2e transfer accounting) */
int mrb_transfer_bytes(int64_t* h2d, int64_t* d2h, int32_t reset);
/* device kernels launched by one mrb_batch_run (for the bench's launch count) */
int64_t mrb_batch_launches_per_run(const mrb_batch* batch);
/* algorithmic bytes of one run, SURVEY.md §8(d) byte model */
double mrb_batch_algorithmic_bytes(const mrb_batch* batch);
/* algorithmic bytes per launch of each kernel (same model):
 * out[0] k_sample, out[1] k_grad, out[2] k_smooth, out[3] k_dense */
int mrb_batch_kernel_bytes(const mrb_batch* batch, double* out);
/* Enqueue one full run with CUDA events around every kernel launch and
 * return the mean device time per launch in ms: out[0] k_sample, out[1]
 * k_grad, out[2] k_smooth, out[3] k_dense, out[4] whole run.  Synchronises. */
int mrb_batch_kernel_times(mrb_batch* batch, double* out);

/* Pipelined registration of many pairs (the per-GPU pair queue end to end):
 * pairs are processed in chunks of `chunk_pairs` on two internal streams, so
 * the host-side setup of chunk k overlaps the device work of chunk k-1 and
 * transfers overlap kernels.  Inputs are n_pairs*H*W stacks (host memory,
 * pinned for overlap).  Outputs (host, any may be NULL): u (concatenated
 * n_i*2 f64), ux/uy/warped (n_pairs*H*W in out_dtype), per-pair
 * iterations_run, MSDs, trace (n_pairs*max_iterations), MRB_* codes and
 * messages (n_pairs*msg_len).  Returns the first pair error (or MRB_OK).
 * Every pair's code is written: a pair the call never reached (an early
 * failure — invalid configuration, a mesh that does not cover the image, a
 * CUDA error) carries the call's own code and mrb_last_error message, never
 * a stale MRB_OK.  When one mesh fails the coverage check the call returns
 * MRB_E_COVERAGE for the whole batch (the caller may retry pair by pair).
 * With ux, uy and warped all NULL (what the reference's register() returns:
 * u and the report, solver.py:148-208) the dense passes, still needed for
 * msd_after, run at low stream priority in the SMs the loop kernels leave
 * idle; with a dense output requested they keep the loops' priority so each
 * group's field is copied back while later groups compute. */
int mrb_register_many(mrb_ctx* ctx, int32_t n_pairs, mrb_mesh* const* meshes, int32_t width,
                      int32_t height, int32_t img_dtype, const void* reference, const void* tmpl,
                      const mrb_config* cfg, int32_t chunk_pairs, int32_t out_dtype, double* u,
                      void* ux, void* uy, void* warped, int32_t* iterations_run,
                      double* msd_before, double* msd_after, double* trace, int32_t* codes,
                      char* messages, int32_t msg_len);

/* ---- single operations (reference functions of the same name) ---------- */
/* warp_sample, solver.py:91-97 / ImageGrid.sample image.py:73-84 */
int mrb_warp_sample(mrb_ctx* ctx, int32_t width, int32_t height, int32_t img_dtype,
                    const void* image, int64_t n, const double* vertices, const double* u,
                    double* out);
/* energy, solver.py:100-106 */
int mrb_energy(mrb_ctx* ctx, mrb_mesh* mesh, int32_t width, int32_t height,
               int32_t img_dtype, const void* reference, const void* tmpl, const double* u,
               double* out);
/* energy_gradient, solver.py:109-121 */
int mrb_energy_gradient(mrb_ctx* ctx, mrb_mesh* mesh, int32_t width, int32_t height,
                        int32_t img_dtype, const void* reference, const void* tmpl,
                        const double* u, double* grad);
/* vertex_gradient_all, mesh.py:236-241 */
int mrb_vertex_gradient_all(mrb_ctx* ctx, mrb_mesh* mesh, const double* f, double* out);
/* smooth_displacement, mesh.py:268-282, on an arbitrary CSR matrix */
int mrb_smooth_csr(mrb_ctx* ctx, int64_t n, const int64_t* indptr, const int64_t* indices,
                   const double* data, const double* u0, double lam, int32_t passes,
                   double* out);
/* step, solver.py:124-145 (clamp when vertices != NULL) */
int mrb_step_csr(mrb_ctx* ctx, int64_t n, const int64_t* indptr, const int64_t* indices,
                 const double* data, const double* u, const double* grad, double tau,
                 double lam, int32_t passes, const double* vertices, int32_t width,
                 int32_t height, double* out);
/* densify, densefield.py:130-187 */
int mrb_densify(mrb_ctx* ctx, mrb_mesh* mesh, int32_t width, int32_t height, const double* u,
                double* ux, double* uy);
/* warp_image, densefield.py:190-199 */
int mrb_warp_image(mrb_ctx* ctx, int32_t width, int32_t height, int32_t img_dtype,
                   const void* tmpl, const double* ux, const double* uy, double* out);
/* msd, image.py:181-186 */
int mrb_msd(mrb_ctx* ctx, int64_t n, const double* a, const double* b, double* out);

/* ---- pixel-grid engine (reference baseline.py) ---- */
/* register_pixelwise, baseline.py:46-118, one pair.  Outputs are f64 host
 * arrays (any may be NULL): ux/uy/warped H*W, trace[iterations].  Returns
 * MRB_E_VALUE for the ValueErrors of baseline.py:57-64 / DenseField, and
 * MRB_E_DIVERGED with the reference's DivergenceError message. */
int mrb_register_pixelwise(mrb_ctx* ctx, int32_t width, int32_t height, int32_t img_dtype,
                           const void* reference, const void* tmpl, const mrb_pixel_config* cfg,
                           double* ux, double* uy, double* warped, double* trace,
                           int32_t* iterations_run, double* msd_before, double* msd_after);
/* A resident batch of equally sized pairs for the pixel engine (same life
 * cycle as mrb_batch: set_images -> run -> get_results -> sync). */
int mrb_pixel_batch_create(mrb_ctx* ctx, int32_t n_pairs, int32_t width, int32_t height,
                           int32_t img_dtype, const mrb_pixel_config* cfg,
                           mrb_pixel_batch** out);
int mrb_pixel_batch_destroy(mrb_pixel_batch* batch);
int mrb_pixel_batch_set_images(mrb_pixel_batch* batch, const void* reference, const void* tmpl,
                               int32_t on_device);
int mrb_pixel_batch_run(mrb_pixel_batch* batch);
int mrb_pixel_batch_get_results(mrb_pixel_batch* batch, int32_t out_dtype, void* ux, void* uy,
                                void* warped);
int mrb_pixel_batch_sync(mrb_pixel_batch* batch);
int mrb_pixel_batch_pair_status(mrb_pixel_batch* batch, int32_t pair, int32_t* iterations_run,
                                double* msd_before, double* msd_after, double* trace, char* msg,
                                int32_t msg_len);
/* kernel launches per run; mean device ms: out[0] fused iteration kernel,
 * out[1] whole run (synchronises) */
int64_t mrb_pixel_batch_launches_per_run(const mrb_pixel_batch* batch);
int mrb_pixel_batch_kernel_times(mrb_pixel_batch* batch, double* out);
/* ImageGrid.sample_gradient, image.py:86-103: pts = n (x, y) pairs */
int mrb_sample_gradient(mrb_ctx* ctx, int32_t width, int32_t height, int32_t img_dtype,
                        const void* image, int64_t n, const double* pts, double* gx,
                        double* gy);
/* grid_umbrella_smooth, baseline.py:27-43 (one pass, f64 plane) */
int mrb_grid_umbrella_smooth(mrb_ctx* ctx, int32_t width, int32_t height, const double* plane,
                             double lam, double* out);

/* ---- content-adaptive mesher (meshgen.py, delaunay.py) -----------------
 * SURVEY.md §8(f) rows 3-4.  Images are (height, width) row-major float64.
 * `taps` is the full 2*radius+1 Gaussian kernel the reference's
 * scipy.ndimage.gaussian_filter builds (_gaussian_kernel1d: np.exp taps
 * normalised by their sum, radius = int(4*sigma + 0.5)); the Python layer
 * computes it with numpy so it is bit-identical.  Outputs match the
 * reference bit for bit. */
typedef struct mrb_tris mrb_tris;  /* a (V, T) triangulation + TriMesh connectivity */

/* _gradient_magnitude, meshgen.py:99-102 (GPU): hypot of np.gradient of the
 * Gaussian-smoothed image */
int mrb_gradient_magnitude(mrb_ctx* ctx, int32_t width, int32_t height, const double* image,
                           int32_t radius, const double* taps, double* mag);
/* _canny_edges, meshgen.py:105-132 (GPU): edges = H*W bytes (0/1); mag
 * (optional) = the gradient magnitude it thresholds */
int mrb_canny_edges(mrb_ctx* ctx, int32_t width, int32_t height, const double* image,
                    int32_t radius, const double* taps, double low, double high, uint8_t* edges,
                    double* mag);
/* canny_sample, meshgen.py:135-154: up to budget edge points (x, y),
 * strongest first, thinned to `spacing` (points: budget*2) */
int mrb_canny_sample(mrb_ctx* ctx, int32_t width, int32_t height, const double* image,
                     int32_t radius, const double* taps, double low, double high, double spacing,
                     int64_t budget, double* points, int64_t* count);
/* halftone_sample's dot mask, meshgen.py:157-203 (host): total = numpy's
 * pairwise mag.sum(); dots = Floyd-Steinberg of mag*budget/total (all zero
 * when total <= 1e-12) */
int mrb_halftone_dots(int32_t width, int32_t height, const double* mag, int64_t budget,
                      int32_t serpentine_start, uint8_t* dots, double* total);
/* _floyd_steinberg, meshgen.py:157-185 (host): dots of a density map */
int mrb_floyd_steinberg(int32_t width, int32_t height, const double* density,
                        int32_t serpentine_start, uint8_t* dots);
/* _SpacingGrid thinning, meshgen.py:80-96 (host): points xy (n*2) visited in
 * `order` (NULL = 0..n-1), kept while count < budget; out: budget*2 */
int mrb_spacing_thin(int64_t n, const double* xy, const int64_t* order, double spacing,
                     int64_t budget, double* out, int64_t* count);
/* uniform_sample, meshgen.py:219-248 (host); out capacity `cap` points */
int mrb_uniform_sample(int32_t width, int32_t height, int64_t budget, double* out, int64_t cap,
                       int64_t* count, char* err, int32_t err_len);
/* dedupe_points, delaunay.py:30-51 (host); out capacity n points */
int mrb_dedupe_points(int64_t n, const double* points, double tol, double* out, int64_t* count,
                      char* err, int32_t err_len);
/* TriMesh(V, T), mesh.py:59-123: validate + orient (host) */
int mrb_tris_create(int64_t n_vertices, const double* vertices, int64_t n_triangles,
                    const int64_t* triangles, mrb_tris** out, char* err, int32_t err_len);
/* delaunay, delaunay.py:75-91 (host): dedupe, Bowyer-Watson (same triangle
 * ids as the reference), flip_edges(passes=100).  MRB_E_VALUE = ValueError,
 * MRB_E_INTERNAL = RuntimeError (insertion point not covered) */
int mrb_delaunay(int64_t n, const double* points, mrb_tris** out, char* err, int32_t err_len);
/* flip_edges, delaunay.py:181-199 (host, in place); *changed = sweeps that flipped */
int mrb_flip_edges(mrb_tris* mesh, int32_t passes, int32_t* changed, char* err, int32_t err_len);
/* smooth_mesh, meshgen.py:269-327 (host, in place); mag = gradient magnitude
 * at sigma 1.5 (mrb_gradient_magnitude) */
int mrb_smooth_mesh(mrb_tris* mesh, int32_t width, int32_t height, const double* mag,
                    int32_t cvt_iterations, int32_t odt_iterations, char* err, int32_t err_len);
int mrb_tris_counts(const mrb_tris* mesh, int64_t* n_vertices, int64_t* n_triangles);
int mrb_tris_export(const mrb_tris* mesh, double* vertices, int64_t* triangles);
int mrb_tris_destroy(mrb_tris* mesh);
/* delaunay_violations, delaunay.py:290-309 (GPU): (triangle, vertex) pairs
 * with the vertex deeper than `margin` inside the circumcircle */
int mrb_delaunay_violations(mrb_ctx* ctx, int64_t n_vertices, const double* vertices,
                            int64_t n_triangles, const int64_t* triangles, double margin,
                            int64_t* count);

#ifdef __cplusplus
}
#endif
#endif /* MESHREG_B200_H */
