// galerk_b200 host API — an Eigen-free mirror of the reference operator API
// (/root/reference/proj/include/galerk/{mesh,quadrature,femspace,kernels,
// assembly}.hpp) for the dense BEM hot path.  Same function names, argument
// order, option structs and exception types/messages; the compute calls go
// through the C-ABI in include/galerk_b200.h to the sm_100a kernels.
//
// Scope: triangle surface meshes, P0/P1 Lagrange spaces with
// the identity operator, the scalar Green kernels "[1/r]" and
// "[exp(ikr)/r]", dense assembly, radiation (collocation) matrices, the
// near-field correction and the Green-kernel matvecs.
#pragma once

#include <array>
#include <complex>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/galerk_b200.h"

namespace galerk {

using cplx = std::complex<double>;

struct Vec3 {
  double x = 0, y = 0, z = 0;
};

// ---- mesh.hpp -------------------------------------------------------------------
struct Mesh {
  std::vector<double> vertices;  // nv x 3, row-major (x,y,z per vertex)
  std::vector<int32_t> elements; // ne x 3
  Mesh() = default;
  Mesh(std::vector<double> v, std::vector<int32_t> e);
  int64_t vertex_count() const { return (int64_t)vertices.size() / 3; }
  int64_t element_count() const { return (int64_t)elements.size() / 3; }
  int dim() const { return 2; }
  bool empty() const { return elements.empty(); }
  Vec3 vertex(int64_t i) const { return {vertices[3 * i], vertices[3 * i + 1], vertices[3 * i + 2]}; }
  double element_measure(int64_t e) const;   // mesh.cpp:53-56
  Vec3 element_centroid(int64_t e) const;    // mesh.cpp:73-78
  double element_radius(int64_t e) const;    // mesh.cpp:80-86
  double total_measure() const;
  double bounding_box_diagonal() const;
};

struct EdgeStats {
  double min_len = 0.0, max_len = 0.0, mean_len = 0.0, std_len = 0.0;
};

Mesh build_sphere(int n_target, double radius);       // mesh.cpp:253-309
EdgeStats edge_stats(const Mesh& mesh);                // mesh.cpp:547-567
std::vector<std::array<int, 2>> unique_edges(const Mesh& mesh);
// BASELINE cfg 3 input: v <- v (1 + amp U(-1,1)), SplitMix64(seed), vertex order.
Mesh perturb_radial(const Mesh& mesh, uint64_t seed, double amp);

// ---- quadrature.hpp -----------------------------------------------------------
struct Domain {
  Mesh mesh;
  int gauss_count = 1;
};
struct ReferenceRule {
  std::vector<std::array<double, 3>> barycentric;
  std::vector<double> weights;
};
struct QuadratureSet {
  std::vector<double> x, y, z;  // SoA points
  std::vector<double> weights;
  std::vector<int32_t> element_of;
  int64_t size() const { return (int64_t)weights.size(); }
};
const std::vector<int>& supported_rules(int dim);         // {1,3,7} + 6 (cfg 3)
const ReferenceRule& reference_rule(int dim, int count);  // quadrature.cpp:138-151
Domain make_domain(const Mesh& mesh, int gauss_count = 1);  // quadrature.cpp:153-165
QuadratureSet quadrature(const Domain& dom);                // quadrature.cpp:167-189

// ---- femspace.hpp ---------------------------------------------------------------
enum class Family { P0, P1 };
class FemSpace {
 public:
  FemSpace() = default;
  FemSpace(Mesh mesh, Family family);
  const Mesh& mesh() const { return mesh_; }
  Family family() const { return family_; }
  int dof_count() const { return dof_count_; }
  int free_count() const { return dof_count_; }
  int free_index(int dof) const { return dof; }
  int dofs_per_element() const { return family_ == Family::P0 ? 1 : 3; }
  std::vector<int> element_dofs(int64_t e) const;  // femspace.cpp:211-234
  std::vector<Vec3> dof_locations() const;
  int result_components() const { return 1; }

 private:
  Mesh mesh_;
  Family family_ = Family::P1;
  int dof_count_ = 0;
};
FemSpace make_fem(const Mesh& mesh, const std::string& family_name);  // P0 | P1

// ---- kernels.hpp ----------------------------------------------------------------
class MatrixXcd;
class Kernel {
 public:
  static Kernel green(const std::string& name, double wavenumber);  // kernels.cpp:21-54
  int components() const { return components_; }
  double wavenumber() const { return wavenumber_; }
  const std::string& name() const { return name_; }
  std::string singular_name() const;
  bool is_custom() const { return custom_; }
  // Custom (callback) kernels exist in the reference API (kernels.hpp:25); the
  // GPU path has no CPU fallback, so assembling with one raises invalid_argument.
  static Kernel custom(int components, const std::string& name = "custom");
  gk_kernel abi() const;
  // kernels.cpp:76-131 (kernels.hpp:37-39): all components at all point pairs,
  // pairs within eps_r zeroed (mask) or raising runtime_error "(i,j)" (no
  // mask); computed on the device (gk_evaluate_blocks).
  void evaluate_blocks(const std::vector<Vec3>& X, const std::vector<Vec3>& Y, std::vector<MatrixXcd>& out,
                       double eps_r, bool mask_singular) const;

 private:
  int kind_ = GK_HELMHOLTZ;
  int components_ = 1;
  double wavenumber_ = 0.0;
  std::string name_;
  bool custom_ = false;
};
Kernel green_kernel(const std::string& name, double wavenumber);
double singular_guard_radius(const QuadratureSet& X, const QuadratureSet& Y);  // kernels.cpp:14-19

// ---- assembly.hpp ---------------------------------------------------------------
struct BemOptions {
  size_t memory_cap_bytes = size_t(8) * 1000 * 1000 * 1000;
  int64_t chunk = 1024;
};

// Column-major complex128 matrix, storage identical to Eigen::MatrixXcd.
// Storage is left uninitialised (every producer writes all entries) and large
// matrices are 2 MB aligned and advised for transparent huge pages, so the
// first touch of a 1.7 GB matrix takes ~800 page faults instead of ~400k.
class MatrixXcd {
 public:
  MatrixXcd() = default;
  MatrixXcd(int64_t r, int64_t c);
  int64_t rows() const { return rows_; }
  int64_t cols() const { return cols_; }
  cplx& operator()(int64_t i, int64_t j) { return data_[(size_t)(i + j * rows_)]; }
  const cplx& operator()(int64_t i, int64_t j) const { return data_[(size_t)(i + j * rows_)]; }
  cplx* data() { return data_.get(); }
  const cplx* data() const { return data_.get(); }

 private:
  struct Free {
    void operator()(cplx* p) const;
  };
  int64_t rows_ = 0, cols_ = 0;
  std::unique_ptr<cplx[], Free> data_;
};

// CSC sparse matrix with setFromTriplets semantics (duplicates summed in order).
struct SpMat {
  int64_t rows = 0, cols = 0;
  std::vector<int64_t> col_ptr;
  std::vector<int32_t> row_idx;
  std::vector<double> values;
  double coeff(int64_t i, int64_t j) const;
  int64_t nonZeros() const { return (int64_t)values.size(); }
};

MatrixXcd bem_dense(const Domain& dom_x, const Domain& dom_y, const FemSpace& test, const Kernel& kernel,
                    const FemSpace& trial, const BemOptions& opts = {});      // assembly.cpp:313-320
MatrixXcd radiation_dense(const std::vector<Vec3>& points, const Domain& dom_y, const Kernel& kernel,
                          const FemSpace& trial, const BemOptions& opts = {});  // assembly.cpp:334-341
SpMat regularize(const Domain& dom_x, const Domain& dom_y, const FemSpace& test,
                 const std::string& singular_name, const FemSpace& trial);   // assembly.cpp:609-697
SpMat regularize_radiation(const std::vector<Vec3>& points, const Domain& dom_y,
                           const std::string& singular_name, const FemSpace& trial);  // assembly.cpp:699-750

// ---- device-resident forms (the B200 data path; no reference counterpart) -----------
// The quadrature/dof tables of one side in the C-ABI layout (owns its arrays).
struct SideTables {
  QuadratureSet qs;
  std::vector<int32_t> elem_dofs;
  std::vector<double> basis;
  int g = 0, nloc = 0;
  int64_t nelem = 0, nfree = 0;
  gk_side abi() const;
};
SideTables make_side_tables(const Domain& dom, const FemSpace& space);  // make_side, assembly.cpp:144-171
SideTables make_point_side_tables(const std::vector<Vec3>& points);      // make_point_side, :173-190
// Row slab [r0, r1) of a test side (SURVEY 8e, row-slab sharding): the elements
// touching those dofs, their dofs renumbered to d - r0 and every other dof
// constrained (-1, skipped like femspace.cpp:476-484).  A plan on it assembles
// rows r0..r1-1 of the operator; with the trial side replicated, row slabs on
// different GPUs need no exchange.
SideTables row_slab(const SideTables& t, int64_t r0, int64_t r1);

class AssemblyPlan {
 public:
  // row_begin/row_end: assemble only rows [row_begin, row_end) of A into an
  // (row_end - row_begin) x cols matrix (row_end < 0: all rows)
  AssemblyPlan(const Domain& dom_x, const Domain& dom_y, const FemSpace& test, const Kernel& kernel,
               const FemSpace& trial, const BemOptions& opts = {}, int symmetric = -1, int64_t row_begin = 0,
               int64_t row_end = -1);
  ~AssemblyPlan();
  AssemblyPlan(const AssemblyPlan&) = delete;
  AssemblyPlan& operator=(const AssemblyPlan&) = delete;
  void assemble(gk_cplx* A_device, int64_t lda, gk_stream stream = nullptr);
  // frequency sweeps: the same tables at another wavenumber ("[1/r]" stays k = 0)
  void set_wavenumber(double k);
  gk_plan_info info() const;
  int launches() const;

 private:
  gk_plan* plan_ = nullptr;
};

// BlockEvaluator (hmatrix.hpp:45-52) backed by the device: the Galerkin entry
// generator of bem_h / radiation_h (assembly.cpp:225-299, 322-356).
class GalerkinEvaluator {
 public:
  GalerkinEvaluator(const Domain& dom_x, const Domain& dom_y, const FemSpace& test, const Kernel& kernel,
                    const FemSpace& trial);
  // radiation_h form: point rows (make_point_side, assembly.cpp:173-190)
  GalerkinEvaluator(const std::vector<Vec3>& points, const Domain& dom_y, const Kernel& kernel,
                    const FemSpace& trial);
  ~GalerkinEvaluator();
  GalerkinEvaluator(const GalerkinEvaluator&) = delete;
  GalerkinEvaluator& operator=(const GalerkinEvaluator&) = delete;
  int64_t rows() const;
  int64_t cols() const;
  void eval(const std::vector<int>& row_ids, const std::vector<int>& col_ids, MatrixXcd& out) const;
  // many eval() requests in one device round trip (ACA panels of many blocks, dense leaves)
  std::vector<MatrixXcd> eval_batch(const std::vector<std::pair<std::vector<int>, std::vector<int>>>& req) const;

 private:
  gk_evaluator* ev_ = nullptr;
};

// ---- harness RNG: SplitMix64 -> U[0,1) -> Box-Muller -------------
std::vector<double> uniform01(uint64_t seed, int64_t n);
std::vector<double> normal(uint64_t seed, int64_t n);          // cos branch first
std::vector<cplx> complex_normal(uint64_t seed, int64_t n);     // re, im consecutive draws

// Throws the exception type matching a gk_status (invalid_argument / runtime_error).
void throw_status(gk_status st);

}  // namespace galerk
