// Host side of the content-adaptive mesher (reference meshgen.py, delaunay.py;
// SURVEY.md §8(f) rows 3-4).  Internal header: the public entry points are
// the mrb_mesher_* / mrb_tris_* functions of include/meshreg_b200.h.
//
// Every routine reproduces the reference's floating-point operation order
// (the build uses -ffp-contract=off), so a mesh generated here is
// bit-identical to the reference's generate_mesh on the same image.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace mrb {

// numpy's pairwise summation (the float64 add reduction of a contiguous
// array: 8 accumulators per <=128 block, halves split at multiples of 8).
double np_pairwise_sum(const double* a, int64_t n);

// glibc 2.35+ hypot (the libm numpy's np.hypot calls; not correctly rounded,
// so the device kernels replicate this exact sequence).
double glibc_hypot(double x, double y);

// A triangulation as the mesher passes it between stages: V (n,2), T (m,3)
// counter-clockwise, plus the TriMesh connectivity the stages read.
struct Tris {
  std::vector<double> V;
  std::vector<int64_t> T;
  // TriMesh connectivity (mesh.py:91-123), rebuilt by trimesh_init
  std::vector<int64_t> inc_ptr, inc_idx;  // ascending incident triangles
  std::vector<uint8_t> boundary;
  int64_t n() const { return int64_t(V.size() / 2); }
  int64_t m() const { return int64_t(T.size() / 3); }
};

// TriMesh(V, T) (mesh.py:59-123): validation with the reference's messages,
// clockwise rows reoriented, incident lists and boundary flags.  Returns ""
// or the ValueError text.
std::string trimesh_init(Tris& t);

// dedupe_points (delaunay.py:30-51).  Returns "" or the ValueError text.
std::string dedupe_points(const double* P, int64_t n, double tol, std::vector<double>& out);

// delaunay (delaunay.py:75-91): dedupe, Bowyer-Watson, TriMesh, flip_edges(100).
// Returns "" or the ValueError / RuntimeError text (err_kind 1 = ValueError,
// 2 = RuntimeError).
std::string delaunay(const double* points, int64_t n, Tris& out, int& err_kind);

// flip_edges (delaunay.py:181-199); returns the number of sweeps that
// changed the triangulation (0 = mesh unchanged).
int flip_edges(Tris& t, int passes, std::string& err);

// smooth_mesh (meshgen.py:269-327) on a (height, width) gradient-magnitude
// map (sigma 1.5, computed on the device).
std::string smooth_mesh(Tris& t, int width, int height, const double* mag, int cvt, int odt);

// Floyd-Steinberg error diffusion (meshgen.py:157-185) of mag * scale.
void floyd_steinberg(const double* mag, double scale, int width, int height, int serpentine_start,
                     uint8_t* dots);

// _SpacingGrid thinning (meshgen.py:80-96) of points visited in order,
// capped at budget.  Returns the kept points (x, y).
void spacing_thin(const double* xy, int64_t n, const int64_t* order, double spacing,
                  int64_t budget, std::vector<double>& out);

// uniform_sample (meshgen.py:219-248).
std::string uniform_sample(int width, int height, int64_t budget, std::vector<double>& out);

}  // namespace mrb
