// =============================================================================
// TEST INFRASTRUCTURE ONLY — NOT PART OF THE PRODUCT.
//
// CPU oracle: an Eigen-free C++ restatement of the reference `galerk` hot path
// (/root/reference/proj, Gypsilab-in-C++).  The reference itself cannot be
// compiled here (it hard-codes /usr/include/eigen3, which is absent, and needs
// the git-ignored doctest), so this file restates, function by function, the
// algorithm of:
//   mesh.cpp:47-94 (measure/centroid/radius), :253-309 (build_sphere),
//   :535-567 (unique_edges/edge_stats); quadrature.cpp:40-75, :138-189;
//   femspace.cpp:211-234, :254-277, :347-391, :460-494; kernels.cpp:14-19,
//   :21-54, :76-131, :151-207; assembly.cpp:135-222, :313-320, :358-697;
//   tests/support/oracles.cpp:106-245, :332-360.
// Every function cites the reference lines it follows.  Only tests/,
// __graft_entry__.smoke() and bench.py's CPU-baseline / reference legs may load
// it; the product (paper_1804_00995_b200) never links or calls it.
//
// Parity pinning: no reference binary can run here, so the oracle is pinned to
// the reference's own known-answer tests (ported in tests/test_oracle_*.py).
// =============================================================================
#pragma once

#include <array>
#include <complex>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace oracle {

using cplx = std::complex<double>;

struct V3 {
  double x = 0, y = 0, z = 0;
  V3() = default;
  V3(double a, double b, double c) : x(a), y(b), z(c) {}
  double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
  double& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
};
inline V3 operator+(const V3& a, const V3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 operator-(const V3& a, const V3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 operator*(double s, const V3& a) { return {s * a.x, s * a.y, s * a.z}; }
inline V3 operator/(const V3& a, double s) { return {a.x / s, a.y / s, a.z / s}; }
inline double dot(const V3& a, const V3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 cross(const V3& a, const V3& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
double norm(const V3& a);

// ---- RNG shared by all harness inputs (SplitMix64 -> U[0,1) -> Box-Muller) ----
struct SplitMix64 {
  uint64_t s;
  explicit SplitMix64(uint64_t seed) : s(seed) {}
  uint64_t next();
  double uniform01();  // 53-bit, [0,1)
};

// ---- mesh (mesh.cpp) ---------------------------------------------------------
struct Mesh {
  std::vector<V3> vertices;
  std::vector<std::array<int, 3>> elements;
  int nv() const { return (int)vertices.size(); }
  int ne() const { return (int)elements.size(); }
  double element_measure(int e) const;   // mesh.cpp:53-56
  V3 element_centroid(int e) const;      // mesh.cpp:73-78
  double element_radius(int e) const;    // mesh.cpp:80-86
};
Mesh build_sphere(int n_target, double radius);  // mesh.cpp:253-309
void perturb_radial(Mesh& m, uint64_t seed, double amp);  // BASELINE cfg 3
struct EdgeStats { double min_len = 0, max_len = 0, mean_len = 0, std_len = 0; };
EdgeStats edge_stats(const Mesh& m);  // mesh.cpp:535-567

// ---- quadrature (quadrature.cpp) ---------------------------------------------
struct Rule {
  int n = 0;
  std::vector<std::array<double, 3>> bary;
  std::vector<double> w;
};
const Rule& triangle_rule(int n);  // 1,3,7 (quadrature.cpp:40-75) + new 6
struct Quad {
  std::vector<V3> pts;
  std::vector<double> w;
  std::vector<int> elem;
};
Quad quadrature(const Mesh& m, int g);  // quadrature.cpp:167-189

// ---- FEM spaces P0/P1, Id operator (femspace.cpp) -----------------------------
enum Family { P0 = 0, P1 = 1 };
int dof_count(const Mesh& m, Family f);
std::vector<int> element_dofs(const Mesh& m, Family f, int e);  // femspace.cpp:211-234
// basis value of local dof l at barycentric point (femspace.cpp:368-380)
double basis_value(Family f, const std::array<double, 3>& bary, int l);
// tangential barycentric gradients, rows = local vertices (femspace.cpp:254-277)
std::array<V3, 3> barycentric_gradients(const Mesh& m, int e);

// Sparse eval matrix in CSR-by-point form: for each quadrature point, the
// (dof, value) nonzeros in ascending dof order (femspace.cpp:460-494 +
// setFromTriplets; exact zeros skipped, :482).
struct PointRows {
  std::vector<int64_t> start;  // M+1
  std::vector<int> dof;
  std::vector<double> val;
};
PointRows eval_rows(const Mesh& m, Family f, int g);

// ---- kernels (kernels.cpp) ----------------------------------------------------
double singular_guard_radius(const std::vector<V3>& X, const std::vector<V3>& Y);  // :14-19
struct Kernel {
  int kind = 1;      // 1 = Helmholtz e^{ikr}/r, 0 = "[1/r]" (k forced 0),
                     // 2 = constant 1 (test_assembly.cpp:140-143 custom kernel)
  double k = 0.0;
  std::string name;
};
Kernel green_kernel(const std::string& name, double k);  // kernels.cpp:21-54 (scalar names)
// out: len x ny col-major complex panel (kernels.cpp:76-131)
void evaluate_blocks(const Kernel& K, const V3* X, int64_t nx, const std::vector<V3>& Y,
                     std::vector<cplx>& out, double eps, bool mask);

struct TriangleNewton {
  double newton = 0.0;
  V3 grad, moment, rho;
  double height = 0.0;
};
TriangleNewton analytic_triangle_integrals(const V3& a, const V3& b, const V3& c,
                                           const V3& x);  // kernels.cpp:151-207

// ---- dense BEM (assembly.cpp:135-222, 313-320) --------------------------------
struct BemOptions {
  size_t memory_cap_bytes = size_t(8) * 1000 * 1000 * 1000;
  int64_t chunk = 1024;
};
// Full matrix, col-major N_t x N_u.  `rows` (optional): restrict to those test
// dofs (complete rows, identical arithmetic to the full computation).
std::vector<cplx> bem_dense(const Mesh& mx, int gx, Family fx, const Mesh& my, int gy,
                            Family fy, const Kernel& K, const BemOptions& opt,
                            const std::vector<int>* rows = nullptr, int threads = 1);
// radiation_dense (assembly.cpp:173-190, 334-341): point side x dom_y side
std::vector<cplx> radiation_dense(const std::vector<V3>& points, const Mesh& my, int gy, Family fy,
                                  const Kernel& K, const BemOptions& opt);
// GalerkinEvaluator::eval (assembly.cpp:225-291): rows x cols block, col-major
std::vector<cplx> block_eval(const Mesh& mx, int gx, Family fx, const Mesh& my, int gy, Family fy,
                             const Kernel& K, const std::vector<int>& rows, const std::vector<int>& cols);
// the same with a point test side (radiation_h, assembly.cpp:343-356)
std::vector<cplx> block_eval_points(const std::vector<V3>& points, const Mesh& my, int gy, Family fy,
                                    const Kernel& K, const std::vector<int>& rows, const std::vector<int>& cols);
// tests/support/oracles.cpp:332-360
std::vector<cplx> naive_bem(const Mesh& mx, int gx, Family fx, const Mesh& my, int gy,
                            Family fy, const Kernel& K);

// Matrix-free Green matvec (cfg 5 semantics): y_i = sum_j [r_ij>eps] G(x_i,y_j) q_j
std::vector<cplx> green_matvec(const Kernel& K, const std::vector<V3>& targets,
                               const std::vector<V3>& sources, const std::vector<cplx>& q,
                               double eps, const std::vector<int64_t>& target_ids,
                               int threads = 1);
// y = A x (col-major zgemv)
std::vector<cplx> matvec(const cplx* A, int64_t rows, int64_t cols, int64_t lda,
                         const cplx* x, int threads = 1);

// ---- near-field correction (assembly.cpp:358-697) ------------------------------
struct Triplet { int row, col; double val; };
struct RegStats {
  int64_t pairs = 0;
  int64_t analytic_calls = 0;
  int64_t gauss_evals = 0;
  std::array<int64_t, 8> depth_hist{};  // leaves accepted per depth
  // per near pair, in pair order: the accepted leaves of accurate_adaptive
  // (a different accept/split decision anywhere changes the count)
  std::vector<int32_t> pair_ex, pair_ey, pair_leaves;
};
enum class NearRule { Ref = 0, TwoHbar = 1 };
std::vector<std::pair<int, int>> close_pairs(const std::vector<V3>& xc, const std::vector<double>& xr,
                                             const std::vector<V3>& yc, const std::vector<double>& yr);
// Returns the summed triplets (setFromTriplets semantics), sorted col-major.
std::vector<Triplet> regularize(const Mesh& mx, int gx, Family fx, const Mesh& my, int gy,
                                Family fy, const std::string& singular_name,
                                RegStats* stats = nullptr, NearRule rule = NearRule::Ref,
                                double hbar = 0.0, const std::vector<int>* only_x = nullptr,
                                int threads = 1);
// regularize_radiation (assembly.cpp:699-750): point x trial-element pairs.
std::vector<Triplet> regularize_radiation(const std::vector<V3>& points, const Mesh& my, int gy, Family fy,
                                          const std::string& singular_name);
// Per-pair local values in pair order (P0 x P0 only) -> (ex, ey, value)
struct PairValue { int ex, ey; double val; };
std::vector<PairValue> regularize_pairs_p0(const Mesh& mx, int gx, const Mesh& my, int gy,
                                           NearRule rule, double hbar,
                                           const std::vector<int>* only_x, int threads,
                                           RegStats* stats);
std::vector<std::pair<int, int>> near_pairs(const Mesh& mx, const Mesh& my, NearRule rule,
                                            double hbar);

// ---- FEM helpers for the capacity pin (assembly.cpp:59-126) ---------------------
std::vector<double> linear_form_ones(const Mesh& m, Family f, int g);
std::vector<double> mass_dense(const Mesh& m, Family f, int g);  // N x N col-major

// ---- reference test-support oracles (tests/support/oracles.cpp) ----------------
double simplex_monomial(int dim, int a, int b, int c);
double newton_oracle(const V3& a, const V3& b, const V3& c, const V3& x, double tol);
V3 newton_moment_oracle(const V3& a, const V3& b, const V3& c, const V3& x, double tol);
V3 newton_grad_oracle(const V3& a, const V3& b, const V3& c, const V3& x, double tol);
double double_newton_oracle(const V3& a, const V3& b, const V3& c, double tol);

}  // namespace oracle
