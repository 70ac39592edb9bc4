// Python binding of the galerk_b200 host API (csrc/host/galerk.hpp).
// std::invalid_argument -> ValueError, std::runtime_error -> RuntimeError, so
// Python tests read like the reference's doctest cases.
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include "../host/galerk.hpp"
#include "../../../include/galerk_b200_diag.h"

namespace py = pybind11;
using namespace galerk;

using F64 = py::array_t<double, py::array::c_style | py::array::forcecast>;
using I32 = py::array_t<int32_t, py::array::c_style | py::array::forcecast>;

namespace {
py::array_t<std::complex<double>> to_numpy(MatrixXcd&& A) {
  auto* m = new MatrixXcd(std::move(A));
  py::capsule own(m, [](void* p) { delete reinterpret_cast<MatrixXcd*>(p); });
  return py::array_t<std::complex<double>>({(py::ssize_t)m->rows(), (py::ssize_t)m->cols()},
                                           {(py::ssize_t)16, (py::ssize_t)(16 * m->rows())}, m->data(), own);
}

std::vector<Vec3> to_points(F64 p) {
  auto a = p.unchecked<2>();
  std::vector<Vec3> out(a.shape(0));
  for (py::ssize_t i = 0; i < a.shape(0); ++i) out[i] = {a(i, 0), a(i, 1), a(i, 2)};
  return out;
}

Mesh mesh_from(F64 v, I32 e) {
  return Mesh(std::vector<double>(v.data(), v.data() + v.size()),
              std::vector<int32_t>(e.data(), e.data() + e.size()));
}

py::array_t<double> points_array(const QuadratureSet& q) {
  py::array_t<double> a({(py::ssize_t)q.size(), (py::ssize_t)3});
  auto m = a.mutable_unchecked<2>();
  for (int64_t i = 0; i < q.size(); ++i) {
    m(i, 0) = q.x[i];
    m(i, 1) = q.y[i];
    m(i, 2) = q.z[i];
  }
  return a;
}

py::dict info_dict(const gk_plan_info& i) {
  py::dict d;
  d["rows"] = i.rows;
  d["cols"] = i.cols;
  d["x_locations"] = i.x_locations;
  d["y_locations"] = i.y_locations;
  d["pairs_reference"] = i.pairs_reference;
  d["pairs_unique"] = i.pairs_unique;
  d["pairs_evaluated"] = i.pairs_evaluated;
  d["tiles"] = i.tiles;
  d["masked_tiles"] = i.masked_tiles;
  d["symmetric"] = (bool)i.symmetric;
  d["eps"] = i.eps;
  d["device_bytes"] = i.device_bytes;
  d["x_halo"] = i.x_halo;
  d["y_halo"] = i.y_halo;
  d["natural_order"] = (bool)i.natural_order;
  d["x_blocks"] = i.x_blocks;
  d["y_blocks"] = i.y_blocks;
  return d;
}

gk_stream as_stream(uintptr_t s) { return reinterpret_cast<gk_stream>(s); }

class GreenPlan {
 public:
  GreenPlan(F64 targets, F64 sources, const Kernel& kernel) {
    auto t = to_points(targets), s = to_points(sources);
    std::vector<double> tx(t.size()), ty(t.size()), tz(t.size()), sx(s.size()), sy(s.size()), sz(s.size());
    for (size_t i = 0; i < t.size(); ++i) {
      tx[i] = t[i].x;
      ty[i] = t[i].y;
      tz[i] = t[i].z;
    }
    for (size_t i = 0; i < s.size(); ++i) {
      sx[i] = s[i].x;
      sy[i] = s[i].y;
      sz[i] = s[i].z;
    }
    const gk_kernel k = kernel.abi();
    throw_status(gk_green_plan_create((int64_t)t.size(), tx.data(), ty.data(), tz.data(), (int64_t)s.size(),
                                      sx.data(), sy.data(), sz.data(), &k, &p_));
  }
  ~GreenPlan() {
    if (p_) gk_green_plan_destroy(p_);
  }
  void matvec(uintptr_t q, uintptr_t y, int precision, uintptr_t stream) {
    throw_status(gk_green_matvec(p_, reinterpret_cast<const gk_cplx*>(q), reinterpret_cast<gk_cplx*>(y), precision,
                                 as_stream(stream)));
  }
  int launches(int precision) const { return gk_green_plan_launches(p_, precision); }
  py::dict info() const {
    int64_t nt = 0, ns = 0;
    double eps = 0;
    throw_status(gk_green_plan_get_info(p_, &nt, &ns, &eps));
    py::dict d;
    d["symmetric"] = gk_green_plan_is_symmetric(p_) != 0;
    d["unique_targets"] = nt;
    d["unique_sources"] = ns;
    d["eps"] = eps;
    return d;
  }

 private:
  gk_green_plan* p_ = nullptr;
};

gk_mesh_side mesh_side(const Domain& d, const FemSpace& s) {
  gk_mesh_side m;
  m.nv = d.mesh.vertex_count();
  m.vertices = d.mesh.vertices.data();
  m.ne = d.mesh.element_count();
  m.elements = d.mesh.elements.data();
  m.family = s.family() == Family::P0 ? 0 : 1;
  m.g = d.gauss_count;
  m.nfree = s.free_count();
  return m;
}

// Device near-field correction (regularize) with in-place apply.
class NearField {
 public:
  NearField(const Domain& dx, const Domain& dy, const FemSpace& t, const std::string& name, const FemSpace& u,
            int rule, double hbar) {
    const gk_mesh_side a = mesh_side(dx, t), b = mesh_side(dy, u);
    throw_status(gk_nearfield_create(&a, &b, name.c_str(), rule, hbar, &p_));
  }
  ~NearField() {
    if (p_) gk_nearfield_destroy(p_);
  }
  void compute(uintptr_t stream) { throw_status(gk_nearfield_compute(p_, as_stream(stream))); }
  void apply(uintptr_t A, int64_t lda, uintptr_t stream) {
    throw_status(gk_nearfield_apply(p_, reinterpret_cast<gk_cplx*>(A), lda, as_stream(stream)));
  }
  py::tuple info() const {
    int64_t pairs = 0, entries = 0;
    throw_status(gk_nearfield_get_info(p_, &pairs, &entries));
    return py::make_tuple(pairs, entries);
  }
  py::tuple triplets() {
    int64_t pairs = 0, entries = 0;
    throw_status(gk_nearfield_get_info(p_, &pairs, &entries));
    std::vector<int32_t> r(entries), c(entries);
    std::vector<double> v(entries);
    throw_status(gk_stream_synchronize(nullptr));
    throw_status(gk_nearfield_triplets(p_, r.data(), c.data(), v.data()));
    return py::make_tuple(r, c, v);
  }
  // (ex, ey, leaves) per near pair (gk_diag_nearfield_pairs)
  py::tuple pair_leaves() const {
    int64_t pairs = 0, entries = 0;
    throw_status(gk_nearfield_get_info(p_, &pairs, &entries));
    std::vector<int32_t> ex(pairs), ey(pairs), lv(pairs);
    throw_status(gk_stream_synchronize(nullptr));
    throw_status(gk_diag_nearfield_pairs(p_, ex.data(), ey.data(), lv.data()));
    return py::make_tuple(ex, ey, lv);
  }
  py::tuple stats() const {
    int64_t calls = 0, hist[8] = {0};
    throw_status(gk_nearfield_stats(p_, &calls, hist));
    return py::make_tuple(calls, std::vector<int64_t>(hist, hist + 8));
  }

 private:
  gk_nearfield* p_ = nullptr;
};
}  // namespace

PYBIND11_MODULE(_galerk, m) {
  m.doc() = "galerk_b200: B200-native dense BEM assembly (host API over the C-ABI)";

  py::class_<Vec3>(m, "Vec3").def_readonly("x", &Vec3::x).def_readonly("y", &Vec3::y).def_readonly("z", &Vec3::z);

  py::class_<Mesh>(m, "Mesh")
      .def(py::init(&mesh_from), py::arg("vertices"), py::arg("elements"))
      .def_property_readonly("vertices",
                             [](const Mesh& s) {
                               return py::array_t<double>({(py::ssize_t)s.vertex_count(), (py::ssize_t)3},
                                                          s.vertices.data());
                             })
      .def_property_readonly("elements",
                             [](const Mesh& s) {
                               return py::array_t<int32_t>({(py::ssize_t)s.element_count(), (py::ssize_t)3},
                                                           s.elements.data());
                             })
      .def("vertex_count", &Mesh::vertex_count)
      .def("element_count", &Mesh::element_count)
      .def("element_measure", &Mesh::element_measure)
      .def("total_measure", &Mesh::total_measure)
      .def("bounding_box_diagonal", &Mesh::bounding_box_diagonal);

  py::class_<EdgeStats>(m, "EdgeStats")
      .def_readonly("min_len", &EdgeStats::min_len)
      .def_readonly("max_len", &EdgeStats::max_len)
      .def_readonly("mean_len", &EdgeStats::mean_len)
      .def_readonly("std_len", &EdgeStats::std_len);

  m.def("build_sphere", &build_sphere, py::arg("n_target"), py::arg("radius"));
  m.def("edge_stats", &edge_stats);
  m.def("perturb_radial", &perturb_radial, py::arg("mesh"), py::arg("seed"), py::arg("amp"));

  py::class_<Domain>(m, "Domain")
      .def_readonly("mesh", &Domain::mesh)
      .def_readonly("gauss_count", &Domain::gauss_count);
  m.def("make_domain", &make_domain, py::arg("mesh"), py::arg("gauss_count") = 1);
  m.def("supported_rules", &supported_rules);
  m.def("reference_rule", [](int dim, int count) {
    const ReferenceRule& r = reference_rule(dim, count);
    return py::make_tuple(r.barycentric, r.weights);
  });
  m.def("quadrature", [](const Domain& d) {
    QuadratureSet q = quadrature(d);
    return py::make_tuple(points_array(q), q.weights, q.element_of);
  });

  py::enum_<Family>(m, "Family").value("P0", Family::P0).value("P1", Family::P1);
  py::class_<FemSpace>(m, "FemSpace")
      .def("dof_count", &FemSpace::dof_count)
      .def("free_count", &FemSpace::free_count)
      .def("family", &FemSpace::family)
      .def("element_dofs", &FemSpace::element_dofs)
      .def_property_readonly("mesh", &FemSpace::mesh);
  m.def("make_fem", &make_fem, py::arg("mesh"), py::arg("family"));

  py::class_<Kernel>(m, "Kernel")
      .def_static("green", &Kernel::green)
      .def_static("custom", &Kernel::custom, py::arg("components"), py::arg("name") = "custom")
      .def("components", &Kernel::components)
      .def("wavenumber", &Kernel::wavenumber)
      .def("name", &Kernel::name)
      .def("singular_name", &Kernel::singular_name);
  m.def("green_kernel", &green_kernel, py::arg("name"), py::arg("wavenumber"));

  py::class_<BemOptions>(m, "BemOptions")
      .def(py::init<>())
      .def_readwrite("memory_cap_bytes", &BemOptions::memory_cap_bytes)
      .def_readwrite("chunk", &BemOptions::chunk);

  m.def(
      "bem_dense",
      [](const Domain& dx, const Domain& dy, const FemSpace& t, const Kernel& k, const FemSpace& u,
         const BemOptions& o) {
        MatrixXcd A;
        {
          py::gil_scoped_release rel;
          A = bem_dense(dx, dy, t, k, u, o);
        }
        return to_numpy(std::move(A));
      },
      py::arg("dom_x"), py::arg("dom_y"), py::arg("test"), py::arg("kernel"), py::arg("trial"),
      py::arg("opts") = BemOptions{});
  m.def(
      "radiation_dense",
      [](F64 pts, const Domain& dy, const Kernel& k, const FemSpace& u, const BemOptions& o) {
        auto P = to_points(pts);
        MatrixXcd A;
        {
          py::gil_scoped_release rel;
          A = radiation_dense(P, dy, k, u, o);
        }
        return to_numpy(std::move(A));
      },
      py::arg("points"), py::arg("dom_y"), py::arg("kernel"), py::arg("trial"), py::arg("opts") = BemOptions{});
  m.def("regularize", [](const Domain& dx, const Domain& dy, const FemSpace& t, const std::string& name,
                         const FemSpace& u) {
    SpMat S;
    {
      py::gil_scoped_release rel;
      S = regularize(dx, dy, t, name, u);
    }
    return py::make_tuple(S.col_ptr, S.row_idx, S.values, py::make_tuple(S.rows, S.cols));
  });
  m.def(
      "regularize_radiation",
      [](F64 pts, const Domain& dy, const std::string& name, const FemSpace& u) {
        auto P = to_points(pts);
        SpMat S;
        {
          py::gil_scoped_release rel;
          S = regularize_radiation(P, dy, name, u);
        }
        return py::make_tuple(S.col_ptr, S.row_idx, S.values, py::make_tuple(S.rows, S.cols));
      },
      py::arg("points"), py::arg("dom_y"), py::arg("singular_name"), py::arg("trial"));

  py::class_<AssemblyPlan>(m, "AssemblyPlan")
      .def(py::init<const Domain&, const Domain&, const FemSpace&, const Kernel&, const FemSpace&,
                    const BemOptions&, int, int64_t, int64_t>(),
           py::arg("dom_x"), py::arg("dom_y"), py::arg("test"), py::arg("kernel"), py::arg("trial"),
           py::arg("opts") = BemOptions{}, py::arg("symmetric") = -1, py::arg("row_begin") = 0,
           py::arg("row_end") = -1)
      .def(
          "assemble",
          [](AssemblyPlan& p, uintptr_t A, int64_t lda, uintptr_t stream) {
            py::gil_scoped_release rel;
            p.assemble(reinterpret_cast<gk_cplx*>(A), lda, as_stream(stream));
          },
          py::arg("A"), py::arg("lda"), py::arg("stream") = 0)
      .def("set_wavenumber", &AssemblyPlan::set_wavenumber, py::arg("k"))
      .def("info", [](const AssemblyPlan& p) { return info_dict(p.info()); })
      .def("launches", &AssemblyPlan::launches);

  m.def(
      "matvec",
      [](uintptr_t A, int64_t rows, int64_t cols, int64_t lda, uintptr_t x, uintptr_t y, uintptr_t stream) {
        throw_status(gk_matvec(reinterpret_cast<const gk_cplx*>(A), rows, cols, lda,
                               reinterpret_cast<const gk_cplx*>(x), reinterpret_cast<gk_cplx*>(y),
                               as_stream(stream)));
      },
      py::arg("A"), py::arg("rows"), py::arg("cols"), py::arg("lda"), py::arg("x"), py::arg("y"),
      py::arg("stream") = 0);
  m.def("matvec_launches", &gk_matvec_launches);
  m.def(
      "matvec_multi",
      [](uintptr_t A, int64_t rows, int64_t cols, int64_t lda, uintptr_t X, int64_t ldx, uintptr_t Y, int64_t ldy,
         int32_t nrhs, uintptr_t stream) {
        throw_status(gk_matvec_multi(reinterpret_cast<const gk_cplx*>(A), rows, cols, lda,
                                     reinterpret_cast<const gk_cplx*>(X), ldx, reinterpret_cast<gk_cplx*>(Y), ldy,
                                     nrhs, as_stream(stream)));
      },
      py::arg("A"), py::arg("rows"), py::arg("cols"), py::arg("lda"), py::arg("X"), py::arg("ldx"), py::arg("Y"),
      py::arg("ldy"), py::arg("nrhs"), py::arg("stream") = 0);
  m.def("matvec_multi_launches", &gk_matvec_multi_launches);
  m.def(
      "evaluate_blocks",
      [](F64 X, F64 Y, const Kernel& K, double eps, bool mask) {
        auto x = X.unchecked<2>();
        auto y = Y.unchecked<2>();
        if (x.shape(1) != 3 || y.shape(1) != 3) throw std::invalid_argument("evaluate_blocks: points must be n x 3");
        const gk_kernel kk = K.abi();
        const int64_t nx = x.shape(0), ny = y.shape(0);
        py::array_t<std::complex<double>, py::array::f_style> out({(py::ssize_t)nx, (py::ssize_t)ny});
        {
          py::gil_scoped_release rel;
          throw_status(gk_evaluate_blocks(nx, X.data(), ny, Y.data(), &kk, eps, mask ? 1 : 0,
                                          reinterpret_cast<gk_cplx*>(out.mutable_data()), std::max<int64_t>(1, nx),
                                          nullptr));
        }
        return out;
      },
      py::arg("X"), py::arg("Y"), py::arg("kernel"), py::arg("eps"), py::arg("mask") = true);
  m.def(
      "lu_factor",
      [](uintptr_t A, int64_t n, int64_t lda, uintptr_t ipiv, uintptr_t stream) {
        int64_t singular_at = 0;
        {
          py::gil_scoped_release rel;
          throw_status(gk_lu_factor(reinterpret_cast<gk_cplx*>(A), n, lda, reinterpret_cast<int64_t*>(ipiv),
                                    &singular_at, as_stream(stream)));
        }
        return singular_at;
      },
      py::arg("A"), py::arg("n"), py::arg("lda"), py::arg("ipiv"), py::arg("stream") = 0);
  m.def(
      "lu_solve",
      [](uintptr_t LU, int64_t n, int64_t lda, uintptr_t ipiv, uintptr_t B, int64_t ldb, int64_t nrhs,
         uintptr_t stream) {
        py::gil_scoped_release rel;
        throw_status(gk_lu_solve(reinterpret_cast<const gk_cplx*>(LU), n, lda, reinterpret_cast<const int64_t*>(ipiv),
                                 reinterpret_cast<gk_cplx*>(B), ldb, nrhs, as_stream(stream)));
      },
      py::arg("LU"), py::arg("n"), py::arg("lda"), py::arg("ipiv"), py::arg("B"), py::arg("ldb"), py::arg("nrhs"),
      py::arg("stream") = 0);
  m.def(
      "gmres",
      [](uintptr_t A, int64_t n, int64_t lda, uintptr_t b, uintptr_t x, double tol, int restart, int maxit,
         uintptr_t stream) {
        gk_solve_info info{};
        std::vector<double> hist(std::max(0, maxit));
        {
          py::gil_scoped_release rel;
          throw_status(gk_gmres(reinterpret_cast<const gk_cplx*>(A), n, lda, reinterpret_cast<const gk_cplx*>(b),
                                reinterpret_cast<gk_cplx*>(x), tol, restart, maxit, &info, hist.data(),
                                as_stream(stream)));
        }
        hist.resize(std::min<size_t>(hist.size(), (size_t)std::max(0, info.history_len)));
        py::dict d;
        d["converged"] = info.converged != 0;
        d["iterations"] = info.iterations;
        d["residual"] = info.residual;
        d["history"] = hist;
        return d;
      },
      py::arg("A"), py::arg("n"), py::arg("lda"), py::arg("b"), py::arg("x"), py::arg("tol") = 1e-6,
      py::arg("restart") = 50, py::arg("maxit") = 1000, py::arg("stream") = 0);

  py::class_<GreenPlan>(m, "GreenPlan")
      .def(py::init<F64, F64, const Kernel&>(), py::arg("targets"), py::arg("sources"), py::arg("kernel"))
      .def("matvec", &GreenPlan::matvec, py::arg("q"), py::arg("y"), py::arg("precision") = 0,
           py::arg("stream") = 0)
      .def("info", &GreenPlan::info)
      .def("launches", &GreenPlan::launches, py::arg("precision") = 0);

  py::class_<GalerkinEvaluator>(m, "GalerkinEvaluator")
      .def(py::init<const Domain&, const Domain&, const FemSpace&, const Kernel&, const FemSpace&>(),
           py::arg("dom_x"), py::arg("dom_y"), py::arg("test"), py::arg("kernel"), py::arg("trial"))
      .def_static(
          "points",
          [](F64 pts, const Domain& dy, const Kernel& k, const FemSpace& u) {
            return std::make_unique<GalerkinEvaluator>(to_points(pts), dy, k, u);
          },
          py::arg("points"), py::arg("dom_y"), py::arg("kernel"), py::arg("trial"))
      .def("rows", &GalerkinEvaluator::rows)
      .def("cols", &GalerkinEvaluator::cols)
      .def(
          "eval",
          [](const GalerkinEvaluator& e, const std::vector<int>& r, const std::vector<int>& c) {
            MatrixXcd out;
            {
              py::gil_scoped_release rel;
              e.eval(r, c, out);
            }
            return to_numpy(std::move(out));
          },
          py::arg("row_ids"), py::arg("col_ids"))
      .def(
          "eval_batch",
          [](const GalerkinEvaluator& e, const std::vector<std::pair<std::vector<int>, std::vector<int>>>& req) {
            std::vector<MatrixXcd> out;
            {
              py::gil_scoped_release rel;
              out = e.eval_batch(req);
            }
            py::list l;
            for (auto& M : out) l.append(to_numpy(std::move(M)));
            return l;
          },
          py::arg("requests"));

  py::class_<NearField>(m, "NearField")
      .def(py::init<const Domain&, const Domain&, const FemSpace&, const std::string&, const FemSpace&, int,
                    double>(),
           py::arg("dom_x"), py::arg("dom_y"), py::arg("test"), py::arg("singular_name"), py::arg("trial"),
           py::arg("rule") = 0, py::arg("hbar") = 0.0)
      .def("compute", &NearField::compute, py::arg("stream") = 0, py::call_guard<py::gil_scoped_release>())
      .def("apply", &NearField::apply, py::arg("A"), py::arg("lda"), py::arg("stream") = 0)
      .def("info", &NearField::info)
      .def("triplets", &NearField::triplets)
      .def("stats", &NearField::stats)
      .def("pair_leaves", &NearField::pair_leaves);
  m.attr("NEAR_REF") = GK_NEAR_REF;
  m.attr("NEAR_2HBAR") = GK_NEAR_2HBAR;

  m.def("side_tables", [](const Domain& d, const FemSpace& s) {
    SideTables t = make_side_tables(d, s);
    py::dict out;
    out["points"] = points_array(t.qs);
    out["weights"] = t.qs.weights;
    out["g"] = t.g;
    out["nelem"] = t.nelem;
    out["nloc"] = t.nloc;
    out["elem_dofs"] = t.elem_dofs;
    out["basis"] = t.basis;
    out["nfree"] = t.nfree;
    return out;
  });
  m.def("uniform01", &uniform01);
  m.def("normal", &normal);
  m.def("complex_normal", [](uint64_t seed, int64_t n) {
    auto v = complex_normal(seed, n);
    return py::array_t<std::complex<double>>((py::ssize_t)v.size(), v.data());
  });
  // one-shot C-ABI drop-in with a caller-provided (pinned) host output buffer
  m.def(
      "bem_dense_into",
      [](const Domain& dx, const Domain& dy, const FemSpace& t, const Kernel& k, const FemSpace& u,
         const BemOptions& o, uintptr_t host_ptr, int64_t lda) {
        py::gil_scoped_release rel;
        const auto t0 = std::chrono::steady_clock::now();
        // bem_dense(dom, dom, V, k, V): one side-table build serves both sides
        const bool same = &dx == &dy && &t == &u;
        const SideTables a = make_side_tables(dx, t);
        const SideTables b = same ? SideTables{} : make_side_tables(dy, u);
        const SideTables& bb = same ? a : b;
        if (std::getenv("GK_TIMING"))
          std::fprintf(stderr, "[bem_dense_into] side tables %8.2f ms\n",
                       std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        const gk_side sa = a.abi(), sb = bb.abi();
        const gk_kernel kk = k.abi();
        gk_options go;
        gk_options_default(&go);
        go.memory_cap_bytes = o.memory_cap_bytes;
        go.chunk = o.chunk;
        throw_status(gk_bem_dense(&sa, &sb, &kk, &go, reinterpret_cast<gk_cplx*>(host_ptr), lda));
        return (int64_t)(a.qs.size() * 32 + bb.qs.size() * 32 + a.elem_dofs.size() * 4 + bb.elem_dofs.size() * 4);
      },
      py::arg("dom_x"), py::arg("dom_y"), py::arg("test"), py::arg("kernel"), py::arg("trial"), py::arg("opts"),
      py::arg("host_ptr"), py::arg("lda"));
  m.def(
      "plan_info_dry",
      [](const Domain& dx, const Domain& dy, const FemSpace& t, const Kernel& k, const FemSpace& u,
         const BemOptions& o, int symmetric) {
        const SideTables a = make_side_tables(dx, t), b = make_side_tables(dy, u);
        const gk_side sa = a.abi(), sb = b.abi();
        const gk_kernel kk = k.abi();
        gk_options go;
        gk_options_default(&go);
        go.memory_cap_bytes = o.memory_cap_bytes;
        go.chunk = o.chunk;
        go.symmetric = symmetric;
        gk_plan_info info;
        throw_status(gk_diag_plan_info(&sa, &sb, &kk, &go, &info));
        return info_dict(info);
      },
      py::arg("dom_x"), py::arg("dom_y"), py::arg("test"), py::arg("kernel"), py::arg("trial"),
      py::arg("opts") = BemOptions{}, py::arg("symmetric") = -1);
  m.def(
      "location_ids",
      [](const Domain& d, const FemSpace& sp, bool serial) {
        const SideTables t = make_side_tables(d, sp);
        const gk_side s = t.abi();
        py::array_t<int64_t> loc(s.npts);
        py::array_t<double> xyz(3 * s.npts);
        int64_t n = 0;
        throw_status(gk_diag_location_ids(&s, serial ? 1 : 0, loc.mutable_data(), &n, xyz.mutable_data()));
        return py::make_tuple(loc, n, xyz);
      },
      py::arg("dom"), py::arg("space"), py::arg("serial") = false);
  m.def(
      "plan_info_dry_rows",
      [](const Domain& dx, const Domain& dy, const FemSpace& t, const Kernel& k, const FemSpace& u,
         const BemOptions& o, int64_t r0, int64_t r1) {
        const SideTables a = row_slab(make_side_tables(dx, t), r0, r1), b = make_side_tables(dy, u);
        const gk_side sa = a.abi(), sb = b.abi();
        const gk_kernel kk = k.abi();
        gk_options go;
        gk_options_default(&go);
        go.memory_cap_bytes = o.memory_cap_bytes;
        go.chunk = o.chunk;
        go.symmetric = 0;
        gk_plan_info info;
        throw_status(gk_diag_plan_info(&sa, &sb, &kk, &go, &info));
        return info_dict(info);
      },
      py::arg("dom_x"), py::arg("dom_y"), py::arg("test"), py::arg("kernel"), py::arg("trial"),
      py::arg("opts"), py::arg("row_begin"), py::arg("row_end"));
  m.def("diag_fp64_peak", [](int64_t iters, uintptr_t stream) {
    double g = 0;
    throw_status(gk_diag_fp64_peak(iters, &g, as_stream(stream)));
    return g;
  });
  m.def("diag_fp64_sustained", [](double seconds, uintptr_t scratch, uint64_t bytes, uintptr_t stream) {
    double gf = 0.0, ms = 0.0;
    {
      py::gil_scoped_release rel;
      throw_status(gk_diag_fp64_sustained(seconds, reinterpret_cast<void*>(scratch), bytes, &gf, &ms,
                                          as_stream(stream)));
    }
    return py::make_tuple(gf, ms);
  });
  m.def("diag_probe_pairs", [](int64_t n, uintptr_t x, uintptr_t y, uintptr_t z, double k, double eps, uintptr_t out,
                               bool fast, uintptr_t stream) {
    auto f = fast ? gk_diag_fast_pairs : gk_diag_probe_pairs;
    throw_status(f(n, reinterpret_cast<const double*>(x), reinterpret_cast<const double*>(y),
                   reinterpret_cast<const double*>(z), k, eps, reinterpret_cast<gk_cplx*>(out), as_stream(stream)));
  });
  m.def("diag_probe_analytic", [](int64_t n, uintptr_t tri, uintptr_t pts, int64_t ntri, uintptr_t out,
                                  uintptr_t stream) {
    throw_status(gk_diag_probe_analytic(n, reinterpret_cast<const double*>(tri), reinterpret_cast<const double*>(pts),
                                        ntri, reinterpret_cast<double*>(out), as_stream(stream)));
  });
  m.def("diag_math", [](int fn, int64_t n, uintptr_t a, uintptr_t b, uintptr_t out, uintptr_t stream) {
    throw_status(gk_diag_math(fn, n, reinterpret_cast<const double*>(a), reinterpret_cast<const double*>(b),
                              reinterpret_cast<double*>(out), as_stream(stream)));
  });
  m.def("last_error", []() { return std::string(gk_last_error()); });
  m.def("version", []() { return std::string(gk_version()); });
  m.attr("FP64") = GK_FP64;
  m.attr("FP32") = GK_FP32;
}
