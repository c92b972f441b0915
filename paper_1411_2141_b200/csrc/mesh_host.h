// Host-side mesh setup shared by the C ABI and the CUDA launch code.
// Internal header (not part of the public ABI in include/meshreg_b200.h).
#pragma once

#include <cmath>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

namespace mrb {

// Canonical CSR as scipy builds it (rows ascending, columns ascending).
struct Csr {
  std::vector<int64_t> indptr, indices;
  std::vector<double> data;
};

struct DeviceMesh;  // defined in the .cu (per-device buffers)

struct HostMesh {
  int64_t n = 0, m = 0, ne = 0;
  // reference-order data (mesh.py TriMesh / TriangleGeometry)
  std::vector<double> V;         // n*2
  std::vector<int64_t> T;        // m*3, CCW-oriented
  std::vector<int64_t> edges;    // ne*2, lexicographically sorted unique pairs
  std::vector<int64_t> valence;  // n
  std::vector<uint8_t> boundary; // n
  std::vector<int64_t> ring_ptr, ring_idx;  // sorted one-rings
  std::vector<int64_t> inc_ptr, inc_idx;    // ascending incident triangles
  std::vector<double> areas, coeffs, vertex_areas;  // m, m*3*2, n
  Csr lap, gx, gy, avg;          // built on first export (ensure_reference_csr)
  std::once_flag csr_once;

  // device-facing layout (node relabelling by Morton order of V)
  std::vector<int32_t> perm;   // new -> old
  std::vector<int32_t> iperm;  // old -> new
  std::vector<int32_t> nb_ptr; // n+1, one-ring CSR in new ids (entries keep
  std::vector<int32_t> nb_idx; //   the reference's per-row order)
  std::vector<double> g_self;  // n*2   fused operator avg∘grad, self term
  std::vector<double> g_nb;    // 2e*2  fused operator, ring terms
  std::vector<double> inv_val; // n     1/valence (Laplacian row value)
  std::vector<double> Vn;      // n*2   vertices in new order
  std::vector<int32_t> Tn;     // m*4   triangles in new ids (+pad)
  int32_t max_deg = 0;         // largest one-ring (fast-path eligibility)

  // Deferred handles (mrb_mesh_create_many): only V, T (oriented), n, m and
  // an estimate of max_deg are set at creation; the rest is built on the GPU
  // (meshbuild.cuh) or, for any host consumer, by ensure_host.
  bool deferred = false;
  const double* dV = nullptr;   // deferred storage: V (n*2) and the oriented
  const int32_t* dT = nullptr;  // T (m*3) in the creation's block (pinned)
  std::shared_ptr<unsigned char> def_hold;
  std::once_flag host_once;
  std::string host_err;        // ensure_host's build_mesh message ("" = ok)

  std::unique_ptr<DeviceMesh> dev;  // lazily created per device
  ~HostMesh();
};

// Build + validate; returns "" on success, else the reference's ValueError text.
std::string build_mesh(int64_t n, const double* V, int64_t m, const int64_t* T, HostMesh& out);

// Validation that needs no connectivity (mesh.py:61-86: shapes, finite
// coordinates, index range, repeated indices, degenerate area) and the CCW
// orientation; writes V and the oriented T into Vout / Tout (the creation's
// block, the device build's upload source) and marks the mesh deferred.
// Returns "" or the reference's ValueError text.
std::string create_mesh(int64_t n, const double* V, int64_t m, const int64_t* T, double* Vout,
                        int32_t* Tout, HostMesh& out);

// create_mesh of one large mesh in parts on several threads: validate_part
// over vertex range [v0, v1) and triangle range [t0, t1) (incidence counts
// into inc, atomically), finish_create merges the parts in order.
struct ValidatePart {
  bool finite = true, range = false, repeated = false, bad = false;
  int64_t worst = 0;
  double worst_abs = INFINITY;
  int32_t max_inc = 0;
};
void validate_part(int64_t n, const double* V, int64_t v0, int64_t v1, int64_t m,
                   const int64_t* T, int64_t t0, int64_t t1, double* Vout, int32_t* Tout,
                   int32_t* inc, ValidatePart& out);
std::string finish_create(const std::vector<ValidatePart>& parts, int64_t n, int64_t m,
                          double* Vout, int32_t* Tout, HostMesh& out);

// Full host build of a deferred mesh (no-op otherwise); returns its error.
const std::string& ensure_host(HostMesh& M);

// The reference's CSR operators L, Gx, Gy, avg (mesh.py:199-213, 254-265):
// only the export entry points need them, so they are built on first use.
void ensure_reference_csr(HostMesh& M);

// PointLocator + locate (densefield.py:62-127) for pixels the raster pass
// left unassigned.  Returns triangle id or -1 (uncovered), fills w[3].
struct Locator {
  double lo[2], hi[2], cell;
  int64_t nx, ny;
  std::vector<std::vector<int64_t>> bins;
  explicit Locator(const HostMesh& mesh);
  void cell_of(double x, double y, int64_t& bx, int64_t& by) const;
  int64_t locate(const HostMesh& mesh, double px, double py, double w[3]) const;
};

// Barycentric weights with numpy's operation order (densefield.py:99-107).
void barycentric(const double* a, const double* b, const double* c, double px, double py,
                 double w[3]);

}  // namespace mrb
