// TEST INFRASTRUCTURE ONLY.  Python binding of the REFERENCE's own sources,
// compiled unchanged from /root/reference/proj/src/{mesh,quadrature,kernels,
// femspace,assembly}.cpp and proj/tests/support/oracles.cpp against the
// Eigen-API shim in oracle/eigen_shim (recipe: oracle/Makefile target `ref`,
// output oracle/_ref/; the H-matrix engine is stubbed, ref_stubs.cpp).
// tests/test_ref_pins.py compares the oracle restatement and the product's
// host tables with these functions, which pins bit for bit:
//   build_sphere            mesh.cpp:253-309
//   edge_stats              mesh.cpp:535-567
//   element_measure         mesh.cpp:47-69
//   reference_rule (tri)    quadrature.cpp:40-75, 138-151
//   quadrature()            quadrature.cpp:167-189
//   singular_guard_radius   kernels.cpp:14-19
//   Kernel::green + evaluate_blocks   kernels.cpp:21-54, 76-131
//   analytic_triangle_integrals       kernels.cpp:151-207
// and to rounding (the shim's sparse products sum in their own order):
//   bem_dense / bem_product            assembly.cpp:144-222, 313-320
//   radiation_dense                    assembly.cpp:173-190, 334-341
//   regularize / regularize_radiation  assembly.cpp:355-750
//   naive_bem                          tests/support/oracles.cpp:332-360
#include <pybind11/complex.h>
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include "galerk/assembly.hpp"
#include "galerk/kernels.hpp"
#include "galerk/mesh.hpp"
#include "galerk/quadrature.hpp"
#include "oracles.hpp"

namespace py = pybind11;
using galerk::MatX3;
using galerk::Vec3;
using F64 = py::array_t<double, py::array::c_style | py::array::forcecast>;
using I32 = py::array_t<int32_t, py::array::c_style | py::array::forcecast>;

static MatX3 to_x3(F64 a) {
  auto v = a.unchecked<2>();
  MatX3 m(v.shape(0), 3);
  for (py::ssize_t i = 0; i < v.shape(0); ++i)
    for (int c = 0; c < 3; ++c) m(i, c) = v(i, c);
  return m;
}
static F64 from_x3(const MatX3& m) {
  F64 a({(py::ssize_t)m.rows(), (py::ssize_t)3});
  auto v = a.mutable_unchecked<2>();
  for (Eigen::Index i = 0; i < m.rows(); ++i)
    for (int c = 0; c < 3; ++c) v(i, c) = m(i, c);
  return a;
}
static galerk::Mesh to_mesh(F64 vtx, I32 elt) {
  auto e = elt.unchecked<2>();
  Eigen::MatrixXi E(e.shape(0), e.shape(1));
  for (py::ssize_t i = 0; i < e.shape(0); ++i)
    for (py::ssize_t c = 0; c < e.shape(1); ++c) E(i, c) = e(i, c);
  return galerk::Mesh(to_x3(vtx), E);
}
static py::tuple from_mesh(const galerk::Mesh& m) {
  I32 e({(py::ssize_t)m.elements.rows(), (py::ssize_t)m.elements.cols()});
  auto v = e.mutable_unchecked<2>();
  for (Eigen::Index i = 0; i < m.elements.rows(); ++i)
    for (Eigen::Index c = 0; c < m.elements.cols(); ++c) v(i, c) = m.elements(i, c);
  return py::make_tuple(from_x3(m.vertices), e);
}
static Vec3 v3(py::sequence s) { return Vec3(s[0].cast<double>(), s[1].cast<double>(), s[2].cast<double>()); }
static py::tuple t3(const Vec3& v) { return py::make_tuple(v(0), v(1), v(2)); }

PYBIND11_MODULE(_ref, m) {
  m.doc() = "the galerk reference's own mesh/quadrature/kernel sources (test infrastructure)";
  m.def("build_sphere", [](int n, double r) { return from_mesh(galerk::build_sphere(n, r)); });
  m.def("edge_stats", [](F64 v, I32 e) {
    const galerk::EdgeStats s = galerk::edge_stats(to_mesh(v, e));
    return py::make_tuple(s.min_len, s.max_len, s.mean_len, s.std_len);
  });
  m.def("element_measures", [](F64 v, I32 e) {
    const galerk::Mesh mm = to_mesh(v, e);
    std::vector<double> out(mm.element_count());
    for (Eigen::Index i = 0; i < mm.element_count(); ++i) out[i] = mm.element_measure(i);
    return out;
  });
  m.def("rule", [](int n) {
    const galerk::ReferenceRule& r = galerk::reference_rule(2, n);
    std::vector<double> b, w;
    for (Eigen::Index q = 0; q < r.barycentric.rows(); ++q)
      for (Eigen::Index c = 0; c < r.barycentric.cols(); ++c) b.push_back(r.barycentric(q, c));
    for (Eigen::Index q = 0; q < r.weights.size(); ++q) w.push_back(r.weights(q));
    return py::make_tuple(b, w);
  });
  m.def("quadrature", [](F64 v, I32 e, int g) {
    const galerk::QuadratureSet q = galerk::quadrature(galerk::make_domain(to_mesh(v, e), g));
    std::vector<double> w(q.weights.size());
    std::vector<int> el(q.element_of.size());
    for (Eigen::Index i = 0; i < q.weights.size(); ++i) w[i] = q.weights(i), el[i] = q.element_of(i);
    return py::make_tuple(from_x3(q.points), w, el);
  });
  m.def("singular_guard_radius", [](F64 X, F64 Y) { return galerk::singular_guard_radius(to_x3(X), to_x3(Y)); });
  m.def("evaluate", [](const std::string& name, double k, F64 X, F64 Y, bool mask, double eps) {
    const galerk::Kernel K = galerk::green_kernel(name, k);
    const MatX3 x = to_x3(X), y = to_x3(Y);
    if (eps < 0) eps = galerk::singular_guard_radius(x, y);
    std::vector<Eigen::MatrixXcd> out;
    K.evaluate_blocks(x, y, out, eps, mask);
    py::array_t<std::complex<double>> a({(py::ssize_t)x.rows(), (py::ssize_t)y.rows()});
    auto v = a.mutable_unchecked<2>();
    for (Eigen::Index i = 0; i < x.rows(); ++i)
      for (Eigen::Index j = 0; j < y.rows(); ++j) v(i, j) = out[0](i, j);
    return a;
  });
  m.def("kernel_info", [](const std::string& name, double k) {
    const galerk::Kernel K = galerk::green_kernel(name, k);
    return py::make_tuple(K.components(), K.wavenumber(), K.singular_name());
  });
  auto fem = [](const galerk::Mesh& mm, int fam) { return galerk::make_fem(mm, fam == 1 ? "P1" : "P0"); };
  auto dense_out = [](const Eigen::MatrixXcd& A) {
    py::array_t<std::complex<double>, py::array::f_style> out({(py::ssize_t)A.rows(), (py::ssize_t)A.cols()});
    std::copy(A.data(), A.data() + A.rows() * A.cols(), out.mutable_data());
    return out;
  };
  auto sparse_out = [](const galerk::SpMat& S) {  // col-major triplets
    std::vector<int> r, c;
    std::vector<double> v;
    for (Eigen::Index j = 0; j < S.outerSize(); ++j)
      for (galerk::SpMat::InnerIterator it(S, j); it; ++it) {
        r.push_back((int)it.row());
        c.push_back((int)j);
        v.push_back(it.value());
      }
    return py::make_tuple(r, c, v);
  };
  m.def("bem_dense", [=](F64 vx, I32 ex, int gx, int fx, F64 vy, I32 ey, int gy, int fy, const std::string& name,
                         double k, double cap) {
    const galerk::Mesh mx = to_mesh(vx, ex), my = to_mesh(vy, ey);
    galerk::BemOptions o;
    if (cap > 0) o.memory_cap_bytes = (size_t)cap;
    Eigen::MatrixXcd A;
    {
      py::gil_scoped_release rel;
      A = galerk::bem_dense(galerk::make_domain(mx, gx), galerk::make_domain(my, gy), fem(mx, fx),
                            galerk::green_kernel(name, k), fem(my, fy), o);
    }
    return dense_out(A);
  }, py::arg("vx"), py::arg("ex"), py::arg("gx"), py::arg("fx"), py::arg("vy"), py::arg("ey"), py::arg("gy"),
     py::arg("fy"), py::arg("name"), py::arg("k"), py::arg("cap") = -1.0);
  m.def("radiation_dense", [=](F64 pts, F64 vy, I32 ey, int gy, int fy, const std::string& name, double k) {
    const galerk::Mesh my = to_mesh(vy, ey);
    const MatX3 P = to_x3(pts);
    Eigen::MatrixXcd A;
    {
      py::gil_scoped_release rel;
      A = galerk::radiation_dense(P, galerk::make_domain(my, gy), galerk::green_kernel(name, k), fem(my, fy));
    }
    return dense_out(A);
  });
  m.def("naive_bem", [=](F64 vx, I32 ex, int gx, int fx, F64 vy, I32 ey, int gy, int fy, const std::string& name,
                         double k) {
    const galerk::Mesh mx = to_mesh(vx, ex), my = to_mesh(vy, ey);
    return dense_out(oracles::naive_bem(galerk::make_domain(mx, gx), galerk::make_domain(my, gy), fem(mx, fx),
                                        galerk::green_kernel(name, k), fem(my, fy)));
  });
  m.def("regularize", [=](F64 vx, I32 ex, int gx, int fx, F64 vy, I32 ey, int gy, int fy, const std::string& name) {
    const galerk::Mesh mx = to_mesh(vx, ex), my = to_mesh(vy, ey);
    galerk::SpMat S;
    {
      py::gil_scoped_release rel;
      S = galerk::regularize(galerk::make_domain(mx, gx), galerk::make_domain(my, gy), fem(mx, fx), name,
                             fem(my, fy));
    }
    return sparse_out(S);
  });
  m.def("regularize_radiation", [=](F64 pts, F64 vy, I32 ey, int gy, int fy, const std::string& name) {
    const galerk::Mesh my = to_mesh(vy, ey);
    return sparse_out(galerk::regularize_radiation(to_x3(pts), galerk::make_domain(my, gy), name, fem(my, fy)));
  });
  m.def("double_newton_oracle", [](py::sequence a, py::sequence b, py::sequence c, double tol) {
    return oracles::double_newton_oracle(v3(a), v3(b), v3(c), tol);
  });
  m.def("analytic", [](py::sequence a, py::sequence b, py::sequence c, py::sequence x) {
    const galerk::TriangleNewton t = galerk::analytic_triangle_integrals(v3(a), v3(b), v3(c), v3(x));
    return py::make_tuple(t.newton, t3(t.grad), t3(t.moment), t3(t.rho), t.height);
  });
}
