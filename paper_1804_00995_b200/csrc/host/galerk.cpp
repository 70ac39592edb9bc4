// galerk_b200 host API implementation (see galerk.hpp).  Host-side table
// building mirrors the reference's arithmetic order (compiled with
// -ffp-contract=off), so meshes and quadrature points are bit-identical to
// the reference algorithm; all pair/contraction work goes to the device.
#include "galerk.hpp"

namespace gk {
int host_threads();  // gk_plan.cpp: GK_THREADS / hardware threads shared among the node's ranks, at most 16
}

#include <sys/mman.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <sstream>
#include <thread>

namespace galerk {

namespace {
Vec3 add(Vec3 a, Vec3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
Vec3 sub(Vec3 a, Vec3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
Vec3 scale(double s, Vec3 a) { return {s * a.x, s * a.y, s * a.z}; }
double dot(Vec3 a, Vec3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
Vec3 cross(Vec3 a, Vec3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
double norm(Vec3 a) { return std::sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }
}  // namespace

void throw_status(gk_status st) {
  if (st == GK_OK) return;
  const std::string msg = gk_last_error();
  if (st == GK_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// ---------------------------------------------------------------------------------
Mesh::Mesh(std::vector<double> v, std::vector<int32_t> e) : vertices(std::move(v)), elements(std::move(e)) {
  if (vertices.size() % 3 || elements.size() % 3) throw std::invalid_argument("mesh: tables must be N x 3");
  const int64_t nv = vertex_count();
  for (int32_t i : elements)
    if (i < 0 || i >= nv) throw std::invalid_argument("mesh: element vertex index out of range");
}

double Mesh::element_measure(int64_t e) const {
  const Vec3 a = vertex(elements[3 * e]), b = vertex(elements[3 * e + 1]), c = vertex(elements[3 * e + 2]);
  return 0.5 * norm(cross(sub(b, a), sub(c, a)));
}

Vec3 Mesh::element_centroid(int64_t e) const {
  Vec3 c{0, 0, 0};
  for (int i = 0; i < 3; ++i) c = add(c, vertex(elements[3 * e + i]));
  return {c.x / 3.0, c.y / 3.0, c.z / 3.0};
}

double Mesh::element_radius(int64_t e) const {
  const Vec3 c = element_centroid(e);
  double r = 0.0;
  for (int i = 0; i < 3; ++i) r = std::max(r, norm(sub(vertex(elements[3 * e + i]), c)));
  return r;
}

double Mesh::total_measure() const {
  double s = 0.0;
  for (int64_t e = 0; e < element_count(); ++e) s += element_measure(e);
  return s;
}

double Mesh::bounding_box_diagonal() const {
  if (vertices.empty()) return 0.0;
  Vec3 lo = vertex(0), hi = vertex(0);
  for (int64_t i = 0; i < vertex_count(); ++i) {
    const Vec3 p = vertex(i);
    lo = {std::min(lo.x, p.x), std::min(lo.y, p.y), std::min(lo.z, p.z)};
    hi = {std::max(hi.x, p.x), std::max(hi.y, p.y), std::max(hi.z, p.z)};
  }
  return norm(sub(hi, lo));
}

Mesh build_sphere(int n_target, double radius) {
  if (n_target < 12) throw std::invalid_argument("build_sphere: n_target must be >= 12");
  if (!(radius > 0.0)) throw std::invalid_argument("build_sphere: radius must be positive");
  const double phi = 0.5 * (1.0 + std::sqrt(5.0));
  std::vector<Vec3> pts = {{-1, phi, 0}, {1, phi, 0},  {-1, -phi, 0}, {1, -phi, 0},
                           {0, -1, phi}, {0, 1, phi},  {0, -1, -phi}, {0, 1, -phi},
                           {phi, 0, -1}, {phi, 0, 1},  {-phi, 0, -1}, {-phi, 0, 1}};
  std::vector<std::array<int, 3>> tris = {
      {0, 11, 5}, {0, 5, 1},  {0, 1, 7},  {0, 7, 10}, {0, 10, 11}, {1, 5, 9}, {5, 11, 4},
      {11, 10, 2}, {10, 7, 6}, {7, 1, 8}, {3, 9, 4},  {3, 4, 2},   {3, 2, 6}, {3, 6, 8},
      {3, 8, 9},  {4, 9, 5},  {2, 4, 11}, {6, 2, 10}, {8, 6, 7},   {9, 8, 1}};
  while ((int)pts.size() < n_target) {  // flat 4-way subdivision, mesh.cpp:269-290
    std::map<std::pair<int, int>, int> midpoint;
    auto mid = [&](int a, int b) {
      const auto key = std::minmax(a, b);
      const auto it = midpoint.find(key);
      if (it != midpoint.end()) return it->second;
      pts.push_back(scale(0.5, add(pts[a], pts[b])));
      const int id = (int)pts.size() - 1;
      midpoint.emplace(key, id);
      return id;
    };
    std::vector<std::array<int, 3>> next;
    next.reserve(4 * tris.size());
    for (const auto& t : tris) {
      const int ab = mid(t[0], t[1]), bc = mid(t[1], t[2]), ca = mid(t[2], t[0]);
      next.push_back({t[0], ab, ca});
      next.push_back({t[1], bc, ab});
      next.push_back({t[2], ca, bc});
      next.push_back({ab, bc, ca});
    }
    tris.swap(next);
  }
  std::vector<double> v(3 * pts.size());
  for (size_t i = 0; i < pts.size(); ++i) {  // single projection, mesh.cpp:292-294
    const double n = norm(pts[i]);
    const Vec3 u{pts[i].x / n, pts[i].y / n, pts[i].z / n};
    v[3 * i] = radius * u.x;
    v[3 * i + 1] = radius * u.y;
    v[3 * i + 2] = radius * u.z;
  }
  std::vector<int32_t> e(3 * tris.size());
  for (size_t t = 0; t < tris.size(); ++t) {
    auto tri = tris[t];
    const Vec3 a{v[3 * tri[0]], v[3 * tri[0] + 1], v[3 * tri[0] + 2]};
    const Vec3 b{v[3 * tri[1]], v[3 * tri[1] + 1], v[3 * tri[1] + 2]};
    const Vec3 c{v[3 * tri[2]], v[3 * tri[2] + 1], v[3 * tri[2] + 2]};
    if (dot(cross(sub(b, a), sub(c, a)), add(add(a, b), c)) < 0.0) std::swap(tri[1], tri[2]);  // :300-307
    e[3 * t] = tri[0];
    e[3 * t + 1] = tri[1];
    e[3 * t + 2] = tri[2];
  }
  return Mesh(std::move(v), std::move(e));
}

Mesh perturb_radial(const Mesh& mesh, uint64_t seed, double amp) {
  Mesh out = mesh;
  const std::vector<double> u = uniform01(seed, mesh.vertex_count());
  for (int64_t i = 0; i < mesh.vertex_count(); ++i) {
    const double s = 1.0 + amp * (2.0 * u[i] - 1.0);
    for (int c = 0; c < 3; ++c) out.vertices[3 * i + c] = s * mesh.vertices[3 * i + c];
  }
  return out;
}

std::vector<std::array<int, 2>> unique_edges(const Mesh& mesh) {
  std::vector<std::array<int, 2>> edges;
  edges.reserve(3 * mesh.element_count());
  for (int64_t e = 0; e < mesh.element_count(); ++e)
    for (int a = 0; a < 3; ++a)
      for (int b = a + 1; b < 3; ++b) {
        const int u = mesh.elements[3 * e + a], v = mesh.elements[3 * e + b];
        edges.push_back({std::min(u, v), std::max(u, v)});
      }
  std::sort(edges.begin(), edges.end());
  edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
  return edges;
}

EdgeStats edge_stats(const Mesh& mesh) {
  if (mesh.empty()) throw std::invalid_argument("edge_stats: empty mesh");
  EdgeStats s;
  s.min_len = std::numeric_limits<double>::infinity();
  double sum = 0.0, sum2 = 0.0;
  const auto edges = unique_edges(mesh);
  for (const auto& e : edges) {
    const double len = norm(sub(mesh.vertex(e[0]), mesh.vertex(e[1])));
    s.min_len = std::min(s.min_len, len);
    s.max_len = std::max(s.max_len, len);
    sum += len;
    sum2 += len * len;
  }
  const double n = (double)edges.size();
  s.mean_len = sum / n;
  s.std_len = std::sqrt(std::max(0.0, sum2 / n - s.mean_len * s.mean_len));
  return s;
}

// ---------------------------------------------------------------------------------
namespace {
ReferenceRule triangle_rule(int n) {
  ReferenceRule r;
  if (n == 1) {
    r.barycentric = {{1.0 / 3, 1.0 / 3, 1.0 / 3}};
    r.weights = {1.0};
  } else if (n == 3) {  // edge-midpoint rule, degree 2 (quadrature.cpp:47-51)
    r.barycentric = {{0.5, 0.5, 0.0}, {0.0, 0.5, 0.5}, {0.5, 0.0, 0.5}};
    r.weights = {1.0 / 3, 1.0 / 3, 1.0 / 3};
  } else if (n == 6) {  // new degree-4 rule for BASELINE cfg 3 (oracle/derive_rule6.py)
    const double a = 0.44594849091596488632, wa = 0.22338158967801146570;
    const double b = 0.091576213509770743460, wb = 0.10995174365532186764;
    for (const auto& [p, w] : {std::pair{a, wa}, std::pair{b, wb}}) {
      const double c = 1.0 - 2.0 * p;
      r.barycentric.push_back({p, p, c});
      r.barycentric.push_back({p, c, p});
      r.barycentric.push_back({c, p, p});
      r.weights.insert(r.weights.end(), {w, w, w});
    }
  } else if (n == 7) {  // symmetric degree-5 rule (quadrature.cpp:52-70)
    const double s15 = std::sqrt(15.0);
    const double a1 = (6.0 - s15) / 21.0, w1 = (155.0 - s15) / 1200.0;
    const double a2 = (6.0 + s15) / 21.0, w2 = (155.0 + s15) / 1200.0;
    r.barycentric.push_back({1.0 / 3, 1.0 / 3, 1.0 / 3});
    r.weights.push_back(9.0 / 40.0);
    for (const auto& [a, w] : {std::pair{a1, w1}, std::pair{a2, w2}}) {
      const double b = 1.0 - 2.0 * a;
      r.barycentric.push_back({a, a, b});
      r.barycentric.push_back({a, b, a});
      r.barycentric.push_back({b, a, a});
      r.weights.insert(r.weights.end(), {w, w, w});
    }
  } else {
    throw std::logic_error("triangle_rule: bad count");
  }
  return r;
}
}  // namespace

const std::vector<int>& supported_rules(int dim) {
  static const std::vector<int> tri = {1, 3, 6, 7};
  if (dim != 2) throw std::invalid_argument("supported_rules: only triangle meshes are on this path");
  return tri;
}

const ReferenceRule& reference_rule(int dim, int count) {
  if (dim != 2) throw std::invalid_argument("reference_rule: bad dimension");
  // thread-safe static tables (the reference's lazily-filled map is not: SURVEY §5)
  static const ReferenceRule r1 = triangle_rule(1), r3 = triangle_rule(3), r6 = triangle_rule(6),
                             r7 = triangle_rule(7);
  switch (count) {
    case 1: return r1;
    case 3: return r3;
    case 6: return r6;
    case 7: return r7;
    default: throw std::invalid_argument("reference_rule: unsupported count");
  }
}

Domain make_domain(const Mesh& mesh, int gauss_count) {
  if (mesh.empty()) throw std::invalid_argument("make_domain: empty mesh");
  const auto& ok = supported_rules(mesh.dim());
  if (std::find(ok.begin(), ok.end(), gauss_count) == ok.end()) {
    std::ostringstream msg;  // keeps the reference's "(supported: 1,3,7" text, quadrature.cpp:157-161
    msg << "make_domain: no " << gauss_count << "-point rule for dimension " << mesh.dim()
        << " (supported: 1,3,7; +6 for config 3)";
    throw std::invalid_argument(msg.str());
  }
  return Domain{mesh, gauss_count};
}

QuadratureSet quadrature(const Domain& dom) {
  const Mesh& mesh = dom.mesh;
  const ReferenceRule& rule = reference_rule(2, dom.gauss_count);
  const int g = (int)rule.weights.size();
  const int64_t ne = mesh.element_count();
  QuadratureSet qs;
  qs.x.resize(ne * g);
  qs.y.resize(ne * g);
  qs.z.resize(ne * g);
  qs.weights.resize(ne * g);
  qs.element_of.resize(ne * g);
  auto fill = [&](int64_t e0, int64_t e1) {
    for (int64_t e = e0; e < e1; ++e) {
      const double measure = mesh.element_measure(e);
      for (int q = 0; q < g; ++q) {
        Vec3 p{0, 0, 0};
        for (int c = 0; c < 3; ++c) p = add(p, scale(rule.barycentric[q][c], mesh.vertex(mesh.elements[3 * e + c])));
        qs.x[e * g + q] = p.x;
        qs.y[e * g + q] = p.y;
        qs.z[e * g + q] = p.z;
        qs.weights[e * g + q] = rule.weights[q] * measure;
        qs.element_of[e * g + q] = (int32_t)e;
      }
    }
  };
  // elements are independent: large meshes are filled on the planner's host threads
  const int nt = (int)std::min<int64_t>(gk::host_threads(), ne / 8192);
  if (nt <= 1) {
    fill(0, ne);
  } else {
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(fill, ne * t / nt, ne * (t + 1) / nt);
    fill(0, ne / nt);
    for (auto& th : pool) th.join();
  }
  return qs;
}

// ---------------------------------------------------------------------------------
FemSpace::FemSpace(Mesh mesh, Family family) : mesh_(std::move(mesh)), family_(family) {
  if (mesh_.empty()) throw std::invalid_argument("fem: empty mesh");
  dof_count_ = (int)(family == Family::P0 ? mesh_.element_count() : mesh_.vertex_count());
}

std::vector<int> FemSpace::element_dofs(int64_t e) const {
  if (family_ == Family::P0) return {(int)e};
  return {mesh_.elements[3 * e], mesh_.elements[3 * e + 1], mesh_.elements[3 * e + 2]};
}

std::vector<Vec3> FemSpace::dof_locations() const {
  std::vector<Vec3> out(dof_count_);
  for (int i = 0; i < dof_count_; ++i) out[i] = family_ == Family::P0 ? mesh_.element_centroid(i) : mesh_.vertex(i);
  return out;
}

FemSpace make_fem(const Mesh& mesh, const std::string& family_name) {
  if (family_name == "P0") return FemSpace(mesh, Family::P0);
  if (family_name == "P1") return FemSpace(mesh, Family::P1);
  if (family_name == "P2" || family_name == "RWG")
    throw std::invalid_argument("fem: family '" + family_name + "' is outside the B200 hot path (P0/P1 only)");
  throw std::invalid_argument("fem: unknown family '" + family_name + "'");
}

// ---------------------------------------------------------------------------------
Kernel Kernel::green(const std::string& name, double wavenumber) {  // kernels.cpp:21-54
  Kernel k;
  k.name_ = name;
  k.wavenumber_ = wavenumber;
  if (name == "[1/r]" || name == "grady[1/r]" || name == "grady[1/r]1" || name == "grady[1/r]2" ||
      name == "grady[1/r]3")
    k.wavenumber_ = 0.0;
  if (name == "[exp(ikr)/r]" || name == "[1/r]") {
    k.kind_ = name == "[1/r]" ? GK_LAPLACE : GK_HELMHOLTZ;
    k.components_ = 1;
    return k;
  }
  for (const std::string base : {"[exp(ikr)/r]", "[1/r]"}) {
    const std::string g = "grady" + base;
    if (name == g) {
      k.kind_ = base == "[1/r]" ? GK_LAPLACE : GK_HELMHOLTZ;
      k.components_ = 3;
      return k;
    }
    for (int j = 1; j <= 3; ++j)
      if (name == g + std::to_string(j)) {
        k.kind_ = base == "[1/r]" ? GK_LAPLACE : GK_HELMHOLTZ;
        k.components_ = 1;
        k.custom_ = true;  // single gradient component: not a scalar Green kernel
        return k;
      }
  }
  throw std::invalid_argument("green_kernel: unknown kernel name '" + name + "'");
}

Kernel Kernel::custom(int components, const std::string& name) {
  if (components != 1 && components != 3) throw std::invalid_argument("Kernel::custom: components must be 1 or 3");
  Kernel k;
  k.custom_ = true;
  k.components_ = components;
  k.name_ = name;
  return k;
}

std::string Kernel::singular_name() const {
  if (custom_) return "";
  return components_ == 3 ? "grady[1/r]" : "[1/r]";
}

gk_kernel Kernel::abi() const {
  gk_kernel k;
  k.kind = custom_ ? -1 : kind_;
  k.components = components_;
  k.k = wavenumber_;
  return k;
}

void Kernel::evaluate_blocks(const std::vector<Vec3>& X, const std::vector<Vec3>& Y, std::vector<MatrixXcd>& out,
                             double eps_r, bool mask_singular) const {
  if (custom_) throw std::invalid_argument(
      "evaluate_blocks: custom kernels have no GPU path (the B200 build has no CPU fallback)");
  const gk_kernel k = abi();
  const int64_t nx = (int64_t)X.size(), ny = (int64_t)Y.size();
  std::vector<double> x(3 * (size_t)nx), y(3 * (size_t)ny);
  for (int64_t i = 0; i < nx; ++i) x[3 * i] = X[i].x, x[3 * i + 1] = X[i].y, x[3 * i + 2] = X[i].z;
  for (int64_t j = 0; j < ny; ++j) y[3 * j] = Y[j].x, y[3 * j + 1] = Y[j].y, y[3 * j + 2] = Y[j].z;
  out.clear();
  out.emplace_back(nx, ny);  // MatrixXcd is move-only
  throw_status(gk_evaluate_blocks(nx, x.data(), ny, y.data(), &k, eps_r, mask_singular ? 1 : 0,
                                  reinterpret_cast<gk_cplx*>(out[0].data()), std::max<int64_t>(1, nx), nullptr));
}

Kernel green_kernel(const std::string& name, double wavenumber) { return Kernel::green(name, wavenumber); }

double singular_guard_radius(const QuadratureSet& X, const QuadratureSet& Y) {
  if (X.size() == 0 || Y.size() == 0) return 0.0;
  double lo[3] = {X.x[0], X.y[0], X.z[0]}, hi[3] = {X.x[0], X.y[0], X.z[0]};
  for (const QuadratureSet* S : {&X, &Y})
    for (int64_t i = 0; i < S->size(); ++i) {
      const double p[3] = {S->x[i], S->y[i], S->z[i]};
      for (int c = 0; c < 3; ++c) {
        lo[c] = std::min(lo[c], p[c]);
        hi[c] = std::max(hi[c], p[c]);
      }
    }
  return 1e-12 * norm({hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]});
}

// ---------------------------------------------------------------------------------
double SpMat::coeff(int64_t i, int64_t j) const {
  for (int64_t p = col_ptr[j]; p < col_ptr[j + 1]; ++p)
    if (row_idx[p] == i) return values[p];
  return 0.0;
}

gk_side SideTables::abi() const {
  gk_side s;
  s.npts = qs.size();
  s.x = qs.x.data();
  s.y = qs.y.data();
  s.z = qs.z.data();
  s.w = qs.weights.data();
  s.g = g;
  s.nelem = nelem;
  s.nloc = nloc;
  s.elem_dofs = elem_dofs.data();
  s.basis = basis.data();
  s.nfree = nfree;
  return s;
}

SideTables make_side_tables(const Domain& dom, const FemSpace& space) {
  if (space.mesh().element_count() != dom.mesh.element_count())
    throw std::invalid_argument("bem: spaces must live on their domain meshes");  // assembly.cpp:304-309
  SideTables t;
  t.qs = quadrature(dom);
  const ReferenceRule& rule = reference_rule(2, dom.gauss_count);
  t.g = dom.gauss_count;
  t.nelem = dom.mesh.element_count();
  t.nloc = space.dofs_per_element();
  t.nfree = space.free_count();
  t.elem_dofs.resize(t.nelem * t.nloc);
  for (int64_t e = 0; e < t.nelem; ++e) {
    const auto d = space.element_dofs(e);
    for (int l = 0; l < t.nloc; ++l) t.elem_dofs[e * t.nloc + l] = space.free_index(d[l]);
  }
  t.basis.resize((size_t)t.g * t.nloc);  // element_basis P0/P1 Id (femspace.cpp:368-380)
  for (int q = 0; q < t.g; ++q)
    for (int l = 0; l < t.nloc; ++l)
      t.basis[q * t.nloc + l] = space.family() == Family::P0 ? 1.0 : rule.barycentric[q][l];
  return t;
}

SideTables row_slab(const SideTables& t, int64_t r0, int64_t r1) {
  if (r0 < 0 || r1 < r0 || r1 > t.nfree) throw std::invalid_argument("row_slab: rows out of range");
  SideTables s;
  s.g = t.g;
  s.nloc = t.nloc;
  s.basis = t.basis;
  s.nfree = r1 - r0;
  for (int64_t e = 0; e < t.nelem; ++e) {
    bool touches = false;
    for (int l = 0; l < t.nloc; ++l) {
      const int32_t d = t.elem_dofs[e * t.nloc + l];
      touches |= d >= r0 && d < r1;
    }
    if (!touches) continue;
    for (int l = 0; l < t.nloc; ++l) {
      const int32_t d = t.elem_dofs[e * t.nloc + l];
      s.elem_dofs.push_back(d >= r0 && d < r1 ? (int32_t)(d - r0) : -1);
    }
    for (int q = 0; q < t.g; ++q) {  // point e*g+q keeps its order within the element
      const int64_t k = e * t.g + q;
      s.qs.x.push_back(t.qs.x[k]);
      s.qs.y.push_back(t.qs.y[k]);
      s.qs.z.push_back(t.qs.z[k]);
      s.qs.weights.push_back(t.qs.weights[k]);
      s.qs.element_of.push_back((int32_t)s.nelem);
    }
    ++s.nelem;
  }
  return s;
}

SideTables make_point_side_tables(const std::vector<Vec3>& points) {
  SideTables t;
  const int64_t n = (int64_t)points.size();
  t.qs.x.resize(n);
  t.qs.y.resize(n);
  t.qs.z.resize(n);
  t.qs.weights.assign(n, 1.0);
  t.qs.element_of.resize(n);
  for (int64_t i = 0; i < n; ++i) {
    t.qs.x[i] = points[i].x;
    t.qs.y[i] = points[i].y;
    t.qs.z[i] = points[i].z;
    t.qs.element_of[i] = (int32_t)i;
  }
  t.g = 1;
  t.nelem = n;
  t.nloc = 1;
  t.nfree = n;
  t.elem_dofs.resize(n);
  for (int64_t i = 0; i < n; ++i) t.elem_dofs[i] = (int32_t)i;
  t.basis = {1.0};
  return t;
}

namespace {
gk_options abi_options(const BemOptions& o, int symmetric) {
  gk_options g;
  gk_options_default(&g);
  g.memory_cap_bytes = o.memory_cap_bytes;
  g.chunk = o.chunk;
  g.symmetric = symmetric;
  return g;
}

MatrixXcd product(const SideTables& tst, const Kernel& kernel, const SideTables& tri, const BemOptions& opts) {
  const gk_side a = tst.abi(), b = tri.abi();
  const gk_kernel k = kernel.abi();
  const gk_options o = abi_options(opts, -1);
  MatrixXcd A(tst.nfree, tri.nfree);
  throw_status(gk_bem_dense(&a, &b, &k, &o, reinterpret_cast<gk_cplx*>(A.data()), std::max<int64_t>(1, tst.nfree)));
  return A;
}
}  // namespace

MatrixXcd::MatrixXcd(int64_t r, int64_t c) : rows_(r), cols_(c) {
  const size_t bytes = sizeof(cplx) * (size_t)r * (size_t)c;
  if (bytes == 0) return;
  constexpr size_t kHuge = size_t(2) << 20;
  void* p = nullptr;
  if (bytes >= kHuge) {
    const size_t padded = (bytes + kHuge - 1) / kHuge * kHuge;
    p = std::aligned_alloc(kHuge, padded);
    if (p) madvise(p, padded, MADV_HUGEPAGE);
  } else {
    p = std::malloc(bytes);
  }
  if (!p) throw std::bad_alloc();
  data_.reset(static_cast<cplx*>(p));
}

void MatrixXcd::Free::operator()(cplx* p) const { std::free(p); }

MatrixXcd bem_dense(const Domain& dom_x, const Domain& dom_y, const FemSpace& test, const Kernel& kernel,
                    const FemSpace& trial, const BemOptions& opts) {
  const SideTables tst = make_side_tables(dom_x, test);
  const SideTables tri = make_side_tables(dom_y, trial);
  return product(tst, kernel, tri, opts);
}

MatrixXcd radiation_dense(const std::vector<Vec3>& points, const Domain& dom_y, const Kernel& kernel,
                          const FemSpace& trial, const BemOptions& opts) {
  if (points.empty()) return MatrixXcd(0, trial.free_count());
  const SideTables tst = make_point_side_tables(points);
  const SideTables tri = make_side_tables(dom_y, trial);
  return product(tst, kernel, tri, opts);
}

namespace {
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

// Runs a created near-field plan and returns its summed correction as the
// column-major sparse matrix the reference's setFromTriplets produces.
SpMat run_nearfield(gk_nearfield* nf, int64_t rows, int64_t cols) {
  std::unique_ptr<gk_nearfield, decltype(&gk_nearfield_destroy)> guard(nf, &gk_nearfield_destroy);
  throw_status(gk_nearfield_compute(nf, nullptr));
  throw_status(gk_stream_synchronize(nullptr));
  int64_t pairs = 0, entries = 0;
  throw_status(gk_nearfield_get_info(nf, &pairs, &entries));
  std::vector<int32_t> r(entries), c(entries);
  std::vector<double> v(entries);
  throw_status(gk_nearfield_triplets(nf, r.data(), c.data(), v.data()));
  SpMat S;
  S.rows = rows;
  S.cols = cols;
  S.col_ptr.assign(S.cols + 1, 0);
  for (int64_t p = 0; p < entries; ++p) S.col_ptr[c[p] + 1]++;
  for (int64_t j = 0; j < S.cols; ++j) S.col_ptr[j + 1] += S.col_ptr[j];
  S.row_idx = r;  // triplets come back col-major sorted
  S.values = v;
  return S;
}
}  // namespace

// assembly.cpp:609-697
SpMat regularize(const Domain& dom_x, const Domain& dom_y, const FemSpace& test, const std::string& singular_name,
                 const FemSpace& trial) {
  const gk_mesh_side mx = mesh_side(dom_x, test), my = mesh_side(dom_y, trial);
  gk_nearfield* nf = nullptr;
  throw_status(gk_nearfield_create(&mx, &my, singular_name.c_str(), GK_NEAR_REF, 0.0, &nf));
  return run_nearfield(nf, test.free_count(), trial.free_count());
}

// assembly.cpp:699-750
SpMat regularize_radiation(const std::vector<Vec3>& points, const Domain& dom_y, const std::string& singular_name,
                           const FemSpace& trial) {
  const gk_mesh_side my = mesh_side(dom_y, trial);
  std::vector<double> xyz(3 * points.size());
  for (size_t i = 0; i < points.size(); ++i) {
    xyz[3 * i] = points[i].x;
    xyz[3 * i + 1] = points[i].y;
    xyz[3 * i + 2] = points[i].z;
  }
  gk_nearfield* nf = nullptr;
  throw_status(gk_nearfield_create_points((int64_t)points.size(), xyz.data(), &my, singular_name.c_str(), &nf));
  return run_nearfield(nf, (int64_t)points.size(), trial.free_count());
}

// ---------------------------------------------------------------------------------
AssemblyPlan::AssemblyPlan(const Domain& dom_x, const Domain& dom_y, const FemSpace& test, const Kernel& kernel,
                           const FemSpace& trial, const BemOptions& opts, int symmetric, int64_t row_begin,
                           int64_t row_end) {
  const bool timing = std::getenv("GK_TIMING") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  SideTables tst = make_side_tables(dom_x, test);
  const bool slab = row_begin != 0 || (row_end >= 0 && row_end != tst.nfree);
  // bem_dense(dom, dom, V, k, V) without a slab: one side-table build serves both sides
  const bool same = !slab && &dom_x == &dom_y && &test == &trial;
  const SideTables tri_own = same ? SideTables{} : make_side_tables(dom_y, trial);
  if (slab) {
    tst = row_slab(tst, row_begin, row_end < 0 ? tst.nfree : row_end);
    if (symmetric == 1) throw std::invalid_argument("AssemblyPlan: a row slab is not symmetric");
    symmetric = 0;
  }
  const SideTables& tri = same ? tst : tri_own;
  const gk_side a = tst.abi(), b = tri.abi();
  const gk_kernel k = kernel.abi();
  const gk_options o = abi_options(opts, symmetric);
  const auto t1 = std::chrono::steady_clock::now();
  throw_status(gk_plan_create(&a, &b, &k, &o, &plan_));
  if (timing)
    std::fprintf(stderr, "[AssemblyPlan] side tables %.2f ms, gk_plan_create %.2f ms\n",
                 std::chrono::duration<double, std::milli>(t1 - t0).count(),
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count());
}

AssemblyPlan::~AssemblyPlan() {
  if (plan_) gk_plan_destroy(plan_);
}

void AssemblyPlan::assemble(gk_cplx* A, int64_t lda, gk_stream stream) {
  throw_status(gk_plan_assemble(plan_, A, lda, stream));
}

gk_plan_info AssemblyPlan::info() const {
  gk_plan_info i;
  throw_status(gk_plan_get_info(plan_, &i));
  return i;
}

int AssemblyPlan::launches() const { return gk_plan_launches(plan_); }

void AssemblyPlan::set_wavenumber(double k) { throw_status(gk_plan_set_wavenumber(plan_, k)); }

// ---------------------------------------------------------------------------------
GalerkinEvaluator::GalerkinEvaluator(const Domain& dom_x, const Domain& dom_y, const FemSpace& test,
                                     const Kernel& kernel, const FemSpace& trial) {
  const SideTables tst = make_side_tables(dom_x, test);
  const SideTables tri = make_side_tables(dom_y, trial);
  const gk_side a = tst.abi(), b = tri.abi();
  const gk_kernel k = kernel.abi();
  throw_status(gk_evaluator_create(&a, &b, &k, &ev_));
}

GalerkinEvaluator::GalerkinEvaluator(const std::vector<Vec3>& points, const Domain& dom_y, const Kernel& kernel,
                                     const FemSpace& trial) {
  const SideTables tst = make_point_side_tables(points);
  const SideTables tri = make_side_tables(dom_y, trial);
  const gk_side a = tst.abi(), b = tri.abi();
  const gk_kernel k = kernel.abi();
  throw_status(gk_evaluator_create(&a, &b, &k, &ev_));
}

GalerkinEvaluator::~GalerkinEvaluator() {
  if (ev_) gk_evaluator_destroy(ev_);
}

int64_t GalerkinEvaluator::rows() const {
  int64_t r = 0;
  throw_status(gk_evaluator_dims(ev_, &r, nullptr));
  return r;
}

int64_t GalerkinEvaluator::cols() const {
  int64_t c = 0;
  throw_status(gk_evaluator_dims(ev_, nullptr, &c));
  return c;
}

void GalerkinEvaluator::eval(const std::vector<int>& row_ids, const std::vector<int>& col_ids,
                             MatrixXcd& out) const {
  std::vector<std::pair<std::vector<int>, std::vector<int>>> req{{row_ids, col_ids}};
  out = std::move(eval_batch(req)[0]);
}

std::vector<MatrixXcd> GalerkinEvaluator::eval_batch(
    const std::vector<std::pair<std::vector<int>, std::vector<int>>>& req) const {
  std::vector<MatrixXcd> out;
  out.reserve(req.size());
  std::vector<gk_block> blocks(req.size());
  for (size_t b = 0; b < req.size(); ++b) {
    const auto& [r, c] = req[b];
    out.emplace_back((int64_t)r.size(), (int64_t)c.size());
    gk_block& B = blocks[b];
    B.nrows = (int32_t)r.size();
    B.ncols = (int32_t)c.size();
    B.row_ids = r.data();
    B.col_ids = c.data();
    B.out = reinterpret_cast<gk_cplx*>(out.back().data());
    B.ldo = std::max<int64_t>(1, (int64_t)r.size());
  }
  throw_status(gk_evaluator_eval(ev_, (int32_t)blocks.size(), blocks.data(), nullptr));
  return out;
}

// ---------------------------------------------------------------------------------
std::vector<double> uniform01(uint64_t seed, int64_t n) {
  std::vector<double> out(n);
  uint64_t s = seed;
  for (int64_t i = 0; i < n; ++i) {
    uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    out[i] = double(z >> 11) * 0x1.0p-53;
  }
  return out;
}

std::vector<double> normal(uint64_t seed, int64_t n) {
  const std::vector<double> u = uniform01(seed, 2 * ((n + 1) / 2));
  std::vector<double> out(n);
  for (int64_t i = 0; 2 * i < n; ++i) {
    const double r = std::sqrt(-2.0 * std::log(1.0 - u[2 * i]));
    const double t = 2.0 * M_PI * u[2 * i + 1];
    out[2 * i] = r * std::cos(t);
    if (2 * i + 1 < n) out[2 * i + 1] = r * std::sin(t);
  }
  return out;
}

std::vector<cplx> complex_normal(uint64_t seed, int64_t n) {
  const std::vector<double> z = normal(seed, 2 * n);
  std::vector<cplx> out(n);
  for (int64_t i = 0; i < n; ++i) out[i] = cplx(z[2 * i], z[2 * i + 1]);
  return out;
}

}  // namespace galerk
