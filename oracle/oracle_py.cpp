// TEST INFRASTRUCTURE ONLY — Python binding of the CPU oracle (galerk_oracle.cpp)
// for tests/, __graft_entry__.smoke() and bench.py's CPU legs.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <chrono>

#include "galerk_oracle.hpp"

namespace py = pybind11;
using namespace oracle;

using F64 = py::array_t<double, py::array::c_style | py::array::forcecast>;
using I32 = py::array_t<int32_t, py::array::c_style | py::array::forcecast>;
using C128 = py::array_t<std::complex<double>, py::array::c_style | py::array::forcecast>;

static Mesh to_mesh(F64 v, I32 e) {
  Mesh m;
  auto vv = v.unchecked<2>();
  auto ee = e.unchecked<2>();
  m.vertices.resize(vv.shape(0));
  for (py::ssize_t i = 0; i < vv.shape(0); ++i) m.vertices[i] = V3(vv(i, 0), vv(i, 1), vv(i, 2));
  m.elements.resize(ee.shape(0));
  for (py::ssize_t i = 0; i < ee.shape(0); ++i) m.elements[i] = {ee(i, 0), ee(i, 1), ee(i, 2)};
  return m;
}

static py::tuple from_mesh(const Mesh& m) {
  F64 v({(py::ssize_t)m.nv(), (py::ssize_t)3});
  I32 e({(py::ssize_t)m.ne(), (py::ssize_t)3});
  auto vv = v.mutable_unchecked<2>();
  auto ee = e.mutable_unchecked<2>();
  for (int i = 0; i < m.nv(); ++i) {
    vv(i, 0) = m.vertices[i].x;
    vv(i, 1) = m.vertices[i].y;
    vv(i, 2) = m.vertices[i].z;
  }
  for (int i = 0; i < m.ne(); ++i)
    for (int c = 0; c < 3; ++c) ee(i, c) = m.elements[i][c];
  return py::make_tuple(v, e);
}

static std::vector<V3> to_pts(F64 p) {
  auto pp = p.unchecked<2>();
  std::vector<V3> out(pp.shape(0));
  for (py::ssize_t i = 0; i < pp.shape(0); ++i) out[i] = V3(pp(i, 0), pp(i, 1), pp(i, 2));
  return out;
}

static F64 pts_array(const std::vector<V3>& p) {
  F64 a({(py::ssize_t)p.size(), (py::ssize_t)3});
  auto m = a.mutable_unchecked<2>();
  for (size_t i = 0; i < p.size(); ++i) {
    m(i, 0) = p[i].x;
    m(i, 1) = p[i].y;
    m(i, 2) = p[i].z;
  }
  return a;
}

static py::array_t<std::complex<double>> colmajor(std::vector<cplx>&& A, int64_t rows, int64_t cols) {
  // returns a (rows, cols) Fortran-ordered array owning the buffer
  auto* buf = new std::vector<cplx>(std::move(A));
  py::capsule free_when_done(buf, [](void* f) { delete reinterpret_cast<std::vector<cplx>*>(f); });
  return py::array_t<std::complex<double>>(
      {(py::ssize_t)rows, (py::ssize_t)cols},
      {(py::ssize_t)sizeof(cplx), (py::ssize_t)(sizeof(cplx) * rows)}, buf->data(), free_when_done);
}

static V3 v3(py::sequence s) { return V3(s[0].cast<double>(), s[1].cast<double>(), s[2].cast<double>()); }
static py::tuple t3(const V3& v) { return py::make_tuple(v.x, v.y, v.z); }

PYBIND11_MODULE(_oracle, m) {
  m.doc() = "TEST INFRASTRUCTURE: CPU restatement of the galerk reference hot path";

  m.def("build_sphere", [](int n, double r) { return from_mesh(build_sphere(n, r)); });
  m.def("perturb_radial", [](F64 v, I32 e, uint64_t seed, double amp) {
    Mesh mm = to_mesh(v, e);
    perturb_radial(mm, seed, amp);
    return from_mesh(mm);
  });
  m.def("edge_stats", [](F64 v, I32 e) {
    EdgeStats s = edge_stats(to_mesh(v, e));
    return py::make_tuple(s.min_len, s.max_len, s.mean_len, s.std_len);
  });
  m.def("element_measures", [](F64 v, I32 e) {
    Mesh mm = to_mesh(v, e);
    std::vector<double> out(mm.ne());
    for (int i = 0; i < mm.ne(); ++i) out[i] = mm.element_measure(i);
    return out;
  });
  m.def("rule", [](int n) {
    const Rule& r = triangle_rule(n);
    return py::make_tuple(r.bary, r.w);
  });
  m.def("quadrature", [](F64 v, I32 e, int g) {
    Quad q = quadrature(to_mesh(v, e), g);
    return py::make_tuple(pts_array(q.pts), q.w, q.elem);
  });
  m.def("eval_rows", [](F64 v, I32 e, int fam, int g) {
    PointRows r = eval_rows(to_mesh(v, e), (Family)fam, g);
    return py::make_tuple(r.start, r.dof, r.val);
  });
  m.def("singular_guard_radius", [](F64 X, F64 Y) { return singular_guard_radius(to_pts(X), to_pts(Y)); });
  m.def("evaluate", [](const std::string& name, double k, F64 X, F64 Y, bool mask, double eps) {
    Kernel K = green_kernel(name, k);
    auto x = to_pts(X), y = to_pts(Y);
    if (eps < 0) eps = singular_guard_radius(x, y);
    std::vector<cplx> out;
    evaluate_blocks(K, x.data(), (int64_t)x.size(), y, out, eps, mask);
    return colmajor(std::move(out), (int64_t)x.size(), (int64_t)y.size());
  }, py::arg("name"), py::arg("k"), py::arg("X"), py::arg("Y"), py::arg("mask") = false,
     py::arg("eps") = -1.0);
  m.def("bem_dense",
        [](F64 vx, I32 ex, int gx, int fx, F64 vy, I32 ey, int gy, int fy, const std::string& name,
           double k, py::object rows, int threads, double cap, int64_t chunk) {
          Mesh mx = to_mesh(vx, ex), my = to_mesh(vy, ey);
          Kernel K = green_kernel(name, k);
          BemOptions o;
          if (cap > 0) o.memory_cap_bytes = (size_t)cap;
          o.chunk = chunk;
          std::vector<int> rr;
          const bool has_rows = !rows.is_none();
          if (has_rows) rr = rows.cast<std::vector<int>>();
          std::vector<cplx> A;
          {
            py::gil_scoped_release rel;
            A = bem_dense(mx, gx, (Family)fx, my, gy, (Family)fy, K, o, has_rows ? &rr : nullptr, threads);
          }
          const int64_t nt = has_rows ? (int64_t)rr.size() : dof_count(mx, (Family)fx);
          return colmajor(std::move(A), nt, dof_count(my, (Family)fy));
        },
        py::arg("vx"), py::arg("ex"), py::arg("gx"), py::arg("fx"), py::arg("vy"), py::arg("ey"),
        py::arg("gy"), py::arg("fy"), py::arg("name"), py::arg("k"), py::arg("rows") = py::none(),
        py::arg("threads") = 1, py::arg("cap") = -1.0, py::arg("chunk") = 1024);
  m.def("radiation_dense", [](F64 pts, F64 vy, I32 ey, int gy, int fy, const std::string& name, double k) {
    auto P = to_pts(pts);
    Mesh my = to_mesh(vy, ey);
    auto A = radiation_dense(P, my, gy, (Family)fy, green_kernel(name, k), BemOptions{});
    return colmajor(std::move(A), (int64_t)P.size(), dof_count(my, (Family)fy));
  });
  m.def("block_eval", [](F64 vx, I32 ex, int gx, int fx, F64 vy, I32 ey, int gy, int fy, const std::string& name,
                         double k, const std::vector<int>& rows, const std::vector<int>& cols) {
    Mesh mx = to_mesh(vx, ex), my = to_mesh(vy, ey);
    auto B = block_eval(mx, gx, (Family)fx, my, gy, (Family)fy, green_kernel(name, k), rows, cols);
    return colmajor(std::move(B), (int64_t)rows.size(), (int64_t)cols.size());
  });
  m.def("block_eval_points", [](F64 pts, F64 vy, I32 ey, int gy, int fy, const std::string& name, double k,
                                const std::vector<int>& rows, const std::vector<int>& cols) {
    Mesh my = to_mesh(vy, ey);
    auto B = block_eval_points(to_pts(pts), my, gy, (Family)fy, green_kernel(name, k), rows, cols);
    return colmajor(std::move(B), (int64_t)rows.size(), (int64_t)cols.size());
  });
  m.def("naive_bem", [](F64 vx, I32 ex, int gx, int fx, F64 vy, I32 ey, int gy, int fy,
                        const std::string& name, double k) {
    Mesh mx = to_mesh(vx, ex), my = to_mesh(vy, ey);
    auto A = naive_bem(mx, gx, (Family)fx, my, gy, (Family)fy, green_kernel(name, k));
    return colmajor(std::move(A), dof_count(mx, (Family)fx), dof_count(my, (Family)fy));
  });
  m.def("green_matvec", [](const std::string& name, double k, F64 T, F64 S, C128 q, double eps,
                           std::vector<int64_t> ids, int threads) {
    auto t = to_pts(T), s = to_pts(S);
    std::vector<cplx> qq(q.data(), q.data() + q.size());
    std::vector<cplx> y;
    {
      py::gil_scoped_release rel;
      y = green_matvec(green_kernel(name, k), t, s, qq, eps, ids, threads);
    }
    return y;
  });
  m.def("matvec", [](py::array_t<std::complex<double>, py::array::f_style | py::array::forcecast> A,
                     C128 x, int threads) {
    std::vector<cplx> y;
    {
      py::gil_scoped_release rel;
      y = matvec(A.data(), A.shape(0), A.shape(1), A.shape(0), x.data(), threads);
    }
    return y;
  });
  m.def("analytic", [](py::sequence a, py::sequence b, py::sequence c, py::sequence x) {
    TriangleNewton t = analytic_triangle_integrals(v3(a), v3(b), v3(c), v3(x));
    return py::make_tuple(t.newton, t3(t.grad), t3(t.moment), t3(t.rho), t.height);
  });
  m.def("newton_oracle", [](py::sequence a, py::sequence b, py::sequence c, py::sequence x, double tol) {
    return newton_oracle(v3(a), v3(b), v3(c), v3(x), tol);
  });
  m.def("newton_moment_oracle", [](py::sequence a, py::sequence b, py::sequence c, py::sequence x, double tol) {
    return t3(newton_moment_oracle(v3(a), v3(b), v3(c), v3(x), tol));
  });
  m.def("newton_grad_oracle", [](py::sequence a, py::sequence b, py::sequence c, py::sequence x, double tol) {
    return t3(newton_grad_oracle(v3(a), v3(b), v3(c), v3(x), tol));
  });
  m.def("double_newton_oracle", [](py::sequence a, py::sequence b, py::sequence c, double tol) {
    return double_newton_oracle(v3(a), v3(b), v3(c), tol);
  });
  m.def("simplex_monomial", &simplex_monomial);
  m.def("regularize",
        [](F64 vx, I32 ex, int gx, int fx, F64 vy, I32 ey, int gy, int fy, const std::string& name,
           int rule, double hbar, py::object only_x, int threads) {
          Mesh mx = to_mesh(vx, ex), my = to_mesh(vy, ey);
          std::vector<int> ox;
          const bool has = !only_x.is_none();
          if (has) ox = only_x.cast<std::vector<int>>();
          RegStats st;
          std::vector<Triplet> t;
          {
            py::gil_scoped_release rel;
            t = regularize(mx, gx, (Family)fx, my, gy, (Family)fy, name, &st, (NearRule)rule, hbar,
                           has ? &ox : nullptr, threads);
          }
          std::vector<int> r(t.size()), c(t.size());
          std::vector<double> v(t.size());
          for (size_t i = 0; i < t.size(); ++i) {
            r[i] = t[i].row;
            c[i] = t[i].col;
            v[i] = t[i].val;
          }
          py::dict stats;
          stats["pairs"] = st.pairs;
          stats["analytic_calls"] = st.analytic_calls;
          stats["gauss_evals"] = st.gauss_evals;
          stats["depth_hist"] = std::vector<int64_t>(st.depth_hist.begin(), st.depth_hist.end());
          stats["pair_ex"] = st.pair_ex;
          stats["pair_ey"] = st.pair_ey;
          stats["pair_leaves"] = st.pair_leaves;
          return py::make_tuple(r, c, v, stats);
        },
        py::arg("vx"), py::arg("ex"), py::arg("gx"), py::arg("fx"), py::arg("vy"), py::arg("ey"),
        py::arg("gy"), py::arg("fy"), py::arg("name"), py::arg("rule") = 0, py::arg("hbar") = 0.0,
        py::arg("only_x") = py::none(), py::arg("threads") = 1);
  m.def("regularize_radiation", [](F64 pts, F64 vy, I32 ey, int gy, int fy, const std::string& name) {
    auto t = regularize_radiation(to_pts(pts), to_mesh(vy, ey), gy, (Family)fy, name);
    std::vector<int> r(t.size()), c(t.size());
    std::vector<double> v(t.size());
    for (size_t i = 0; i < t.size(); ++i) {
      r[i] = t[i].row;
      c[i] = t[i].col;
      v[i] = t[i].val;
    }
    return py::make_tuple(r, c, v);
  });
  m.def("near_pairs", [](F64 vx, I32 ex, F64 vy, I32 ey, int rule, double hbar) {
    return near_pairs(to_mesh(vx, ex), to_mesh(vy, ey), (NearRule)rule, hbar);
  });
  m.def("linear_form_ones", [](F64 v, I32 e, int fam, int g) {
    return linear_form_ones(to_mesh(v, e), (Family)fam, g);
  });
  m.def("mass_dense", [](F64 v, I32 e, int fam, int g) {
    Mesh mm = to_mesh(v, e);
    const int64_t n = dof_count(mm, (Family)fam);
    auto M = mass_dense(mm, (Family)fam, g);
    std::vector<cplx> Mc(M.begin(), M.end());
    return colmajor(std::move(Mc), n, n);
  });
  m.def("uniform01_stream", [](uint64_t seed, int64_t n) {
    SplitMix64 r(seed);
    std::vector<double> out(n);
    for (auto& v : out) v = r.uniform01();
    return out;
  });
}
