// TEST INFRASTRUCTURE ONLY — see galerk_oracle.hpp for scope and provenance.
// Compiled with -ffp-contract=off so the arithmetic order written here is the
// arithmetic order executed (the reference is built without FMA contraction:
// proj/src/CMakeLists.txt:19 uses -O3 -Wall -Wextra, no -march).
#include "galerk_oracle.hpp"

#include <algorithm>
#include <cmath>
#include <functional>
#include <limits>
#include <numeric>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace oracle {

double norm(const V3& a) { return std::sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }

// ---------------------------------------------------------------------------
// RNG (BASELINE.md §3 "repo's own portable RNG")
// ---------------------------------------------------------------------------
uint64_t SplitMix64::next() {
  uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
double SplitMix64::uniform01() { return double(next() >> 11) * 0x1.0p-53; }

// ---------------------------------------------------------------------------
// Mesh (mesh.cpp)
// ---------------------------------------------------------------------------
double Mesh::element_measure(int e) const {  // mesh.cpp:53-56
  const V3& a = vertices[elements[e][0]];
  const V3& b = vertices[elements[e][1]];
  const V3& c = vertices[elements[e][2]];
  return 0.5 * norm(cross(b - a, c - a));
}

V3 Mesh::element_centroid(int e) const {  // mesh.cpp:73-78
  V3 c(0, 0, 0);
  for (int i = 0; i < 3; ++i) c = c + vertices[elements[e][i]];
  return c / 3.0;
}

double Mesh::element_radius(int e) const {  // mesh.cpp:80-86
  V3 c = element_centroid(e);
  double r = 0.0;
  for (int i = 0; i < 3; ++i) r = std::max(r, norm(vertices[elements[e][i]] - c));
  return r;
}

Mesh build_sphere(int n_target, double radius) {  // mesh.cpp:253-309
  if (n_target < 12) throw std::invalid_argument("build_sphere: n_target must be >= 12");
  if (!(radius > 0.0)) throw std::invalid_argument("build_sphere: radius must be positive");
  const double phi = 0.5 * (1.0 + std::sqrt(5.0));
  // The regular icosahedron in its classic vertex/face order (the order fixes
  // the numbering of every subdivided mesh, so it is part of the input spec).
  std::vector<V3> pts = {{-1, phi, 0}, {1, phi, 0},  {-1, -phi, 0}, {1, -phi, 0},
                         {0, -1, phi}, {0, 1, phi},  {0, -1, -phi}, {0, 1, -phi},
                         {phi, 0, -1}, {phi, 0, 1},  {-phi, 0, -1}, {-phi, 0, 1}};
  std::vector<std::array<int, 3>> tris = {
      {0, 11, 5}, {0, 5, 1},  {0, 1, 7},   {0, 7, 10}, {0, 10, 11}, {1, 5, 9},  {5, 11, 4},
      {11, 10, 2}, {10, 7, 6}, {7, 1, 8},  {3, 9, 4},  {3, 4, 2},   {3, 2, 6},  {3, 6, 8},
      {3, 8, 9},  {4, 9, 5},  {2, 4, 11},  {6, 2, 10}, {8, 6, 7},   {9, 8, 1}};
  while ((int)pts.size() < n_target) {
    std::map<std::pair<int, int>, int> midpoint;
    auto mid = [&](int a, int b) {
      auto key = std::minmax(a, b);
      auto it = midpoint.find(key);
      if (it != midpoint.end()) return it->second;
      const V3 s = pts[a] + pts[b];
      pts.push_back(0.5 * s);
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
  Mesh m;
  m.vertices.resize(pts.size());
  for (size_t i = 0; i < pts.size(); ++i) {
    const double n = norm(pts[i]);
    const V3 u = pts[i] / n;  // Eigen normalized(): v / sqrt(squaredNorm)
    m.vertices[i] = radius * u;
  }
  m.elements = tris;
  for (auto& t : m.elements) {  // outward orientation, mesh.cpp:300-307
    const V3& a = m.vertices[t[0]];
    const V3& b = m.vertices[t[1]];
    const V3& c = m.vertices[t[2]];
    if (dot(cross(b - a, c - a), a + b + c) < 0.0) std::swap(t[1], t[2]);
  }
  return m;
}

void perturb_radial(Mesh& m, uint64_t seed, double amp) {
  // BASELINE cfg 3: v <- v * (1 + amp * U(-1,1)), one draw per vertex in index order.
  SplitMix64 rng(seed);
  for (auto& v : m.vertices) {
    const double u = 2.0 * rng.uniform01() - 1.0;
    const double s = 1.0 + amp * u;
    v = s * v;
  }
}

EdgeStats edge_stats(const Mesh& m) {  // mesh.cpp:535-567
  if (m.elements.empty()) throw std::invalid_argument("edge_stats: empty mesh");
  std::vector<std::array<int, 2>> edges;
  edges.reserve(3 * m.elements.size());
  for (const auto& t : m.elements)
    for (int a = 0; a < 3; ++a)
      for (int b = a + 1; b < 3; ++b) edges.push_back({std::min(t[a], t[b]), std::max(t[a], t[b])});
  std::sort(edges.begin(), edges.end());
  edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
  EdgeStats s;
  s.min_len = std::numeric_limits<double>::infinity();
  double sum = 0.0, sum2 = 0.0;
  for (const auto& e : edges) {
    const double len = norm(m.vertices[e[0]] - m.vertices[e[1]]);
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

// ---------------------------------------------------------------------------
// Quadrature (quadrature.cpp)
// ---------------------------------------------------------------------------
namespace {
Rule make_rule(int n) {
  Rule r;
  r.n = n;
  if (n == 1) {
    r.bary = {{1.0 / 3, 1.0 / 3, 1.0 / 3}};
    r.w = {1.0};
  } else if (n == 3) {  // edge-midpoint rule, quadrature.cpp:47-51
    r.bary = {{0.5, 0.5, 0.0}, {0.0, 0.5, 0.5}, {0.5, 0.0, 0.5}};
    r.w = {1.0 / 3, 1.0 / 3, 1.0 / 3};
  } else if (n == 6) {
    // NEW (not in the reference): symmetric degree-4 two-orbit rule, constants
    // derived by oracle/derive_rule6.py from the degree-4 moment equations.
    const double a = 0.44594849091596488632, wa = 0.22338158967801146570;
    const double b = 0.091576213509770743460, wb = 0.10995174365532186764;
    for (auto [p, w] : {std::pair{a, wa}, std::pair{b, wb}}) {
      const double c = 1.0 - 2.0 * p;
      r.bary.push_back({p, p, c});
      r.w.push_back(w);
      r.bary.push_back({p, c, p});
      r.w.push_back(w);
      r.bary.push_back({c, p, p});
      r.w.push_back(w);
    }
  } else if (n == 7) {  // quadrature.cpp:52-70 (Radon degree-5 rule)
    const double s15 = std::sqrt(15.0);
    const double a1 = (6.0 - s15) / 21.0, w1 = (155.0 - s15) / 1200.0;
    const double a2 = (6.0 + s15) / 21.0, w2 = (155.0 + s15) / 1200.0;
    r.bary.push_back({1.0 / 3, 1.0 / 3, 1.0 / 3});
    r.w.push_back(9.0 / 40.0);
    for (auto [a, w] : {std::pair{a1, w1}, std::pair{a2, w2}}) {
      const double b = 1.0 - 2.0 * a;
      r.bary.push_back({a, a, b});
      r.w.push_back(w);
      r.bary.push_back({a, b, a});
      r.w.push_back(w);
      r.bary.push_back({b, a, a});
      r.w.push_back(w);
    }
  } else {
    throw std::invalid_argument("make_domain: no " + std::to_string(n) +
                                "-point rule for dimension 2 (supported: 1,3,7; +6 for config 3)");
  }
  return r;
}
}  // namespace

const Rule& triangle_rule(int n) {
  static const Rule r1 = make_rule(1), r3 = make_rule(3), r6 = make_rule(6), r7 = make_rule(7);
  switch (n) {
    case 1: return r1;
    case 3: return r3;
    case 6: return r6;
    case 7: return r7;
    default: make_rule(n);  // throws
  }
  throw std::logic_error("unreachable");
}

Quad quadrature(const Mesh& m, int g) {  // quadrature.cpp:167-189
  const Rule& rule = triangle_rule(g);
  Quad q;
  const int64_t ne = m.ne();
  q.pts.resize(ne * g);
  q.w.resize(ne * g);
  q.elem.resize(ne * g);
  for (int64_t e = 0; e < ne; ++e) {
    const double measure = m.element_measure((int)e);
    for (int k = 0; k < g; ++k) {
      V3 p(0, 0, 0);
      for (int c = 0; c < 3; ++c) p = p + rule.bary[k][c] * m.vertices[m.elements[e][c]];
      q.pts[e * g + k] = p;
      q.w[e * g + k] = rule.w[k] * measure;
      q.elem[e * g + k] = (int)e;
    }
  }
  return q;
}

// ---------------------------------------------------------------------------
// FEM (femspace.cpp)
// ---------------------------------------------------------------------------
int dof_count(const Mesh& m, Family f) { return f == P0 ? m.ne() : m.nv(); }

std::vector<int> element_dofs(const Mesh& m, Family f, int e) {
  if (f == P0) return {e};
  return {m.elements[e][0], m.elements[e][1], m.elements[e][2]};
}

double basis_value(Family f, const std::array<double, 3>& bary, int l) {
  return f == P0 ? 1.0 : bary[l];
}

std::array<V3, 3> barycentric_gradients(const Mesh& m, int e) {  // femspace.cpp:254-277
  const V3 v0 = m.vertices[m.elements[e][0]];
  const V3 e1 = m.vertices[m.elements[e][1]] - v0;
  const V3 e2 = m.vertices[m.elements[e][2]] - v0;
  // gram = E^T E, G = E gram^{-1} (2x2 inverse by cofactors)
  const double g00 = dot(e1, e1), g01 = dot(e1, e2), g11 = dot(e2, e2);
  const double det = g00 * g11 - g01 * g01;
  const double i00 = g11 / det, i01 = -g01 / det, i11 = g00 / det;
  std::array<V3, 3> g;
  g[1] = V3(e1.x * i00 + e2.x * i01, e1.y * i00 + e2.y * i01, e1.z * i00 + e2.z * i01);
  g[2] = V3(e1.x * i01 + e2.x * i11, e1.y * i01 + e2.y * i11, e1.z * i01 + e2.z * i11);
  g[0] = V3(0, 0, 0) - g[1] - g[2];
  return g;
}

PointRows eval_rows(const Mesh& m, Family f, int g) {  // femspace.cpp:460-494
  const Rule& rule = triangle_rule(g);
  const int64_t M = (int64_t)m.ne() * g;
  PointRows pr;
  pr.start.assign(M + 1, 0);
  std::vector<std::vector<std::pair<int, double>>> rows(M);
  for (int e = 0; e < m.ne(); ++e) {
    auto dofs = element_dofs(m, f, e);
    for (size_t l = 0; l < dofs.size(); ++l)
      for (int q = 0; q < g; ++q) {
        const double v = basis_value(f, rule.bary[q], (int)l);
        if (v != 0.0) rows[(int64_t)e * g + q].push_back({dofs[l], v});
      }
  }
  for (int64_t k = 0; k < M; ++k) {
    std::sort(rows[k].begin(), rows[k].end(),
              [](const auto& a, const auto& b) { return a.first < b.first; });
    pr.start[k + 1] = pr.start[k] + (int64_t)rows[k].size();
    for (auto& [d, v] : rows[k]) {
      pr.dof.push_back(d);
      pr.val.push_back(v);
    }
  }
  return pr;
}

// ---------------------------------------------------------------------------
// Kernels (kernels.cpp)
// ---------------------------------------------------------------------------
double singular_guard_radius(const std::vector<V3>& X, const std::vector<V3>& Y) {
  if (X.empty() || Y.empty()) return 0.0;  // kernels.cpp:14-19
  V3 lo = X[0], hi = X[0];
  auto upd = [&](const V3& p) {
    for (int c = 0; c < 3; ++c) {
      lo[c] = std::min(lo[c], p[c]);
      hi[c] = std::max(hi[c], p[c]);
    }
  };
  for (const auto& p : X) upd(p);
  for (const auto& p : Y) upd(p);
  return 1e-12 * norm(hi - lo);
}

Kernel green_kernel(const std::string& name, double k) {  // kernels.cpp:21-54
  Kernel K;
  K.name = name;
  if (name == "[1/r]") {
    K.kind = 0;
    K.k = 0.0;
  } else if (name == "[exp(ikr)/r]") {
    K.kind = 1;
    K.k = k;
  } else if (name == "__ones__") {
    K.kind = 2;  // custom constant kernel of test_assembly.cpp:140-143 (no mask)
  } else {
    throw std::invalid_argument("green_kernel: unknown kernel name '" + name + "'");
  }
  return K;
}

void evaluate_blocks(const Kernel& K, const V3* X, int64_t nx, const std::vector<V3>& Y,
                     std::vector<cplx>& out, double eps, bool mask) {  // kernels.cpp:76-131
  const int64_t ny = (int64_t)Y.size();
  out.assign(nx * ny, cplx(0.0, 0.0));
  if (K.kind == 2) {
    for (auto& v : out) v = cplx(1.0, 0.0);
    return;
  }
  const double eps2 = eps * eps;
  const double k = K.k;
  // Singular pairs raise when !mask (kernels.cpp:104-108); that check runs
  // serially first because exceptions must not leave an OpenMP region.
  if (!mask)
    for (int64_t j = 0; j < ny; ++j)
      for (int64_t i = 0; i < nx; ++i) {
        const double dx = X[i].x - Y[j].x, dy = X[i].y - Y[j].y, dz = X[i].z - Y[j].z;
        const double r = std::sqrt(dx * dx + dy * dy + dz * dz);
        if (r * r <= eps2)
          throw std::runtime_error("kernel evaluation at singular point pair (" +
                                   std::to_string(i) + "," + std::to_string(j) +
                                   "), r=" + std::to_string(r));
      }
#pragma omp parallel for schedule(static) if (nx * ny > 65536)
  for (int64_t j = 0; j < ny; ++j) {
    const double yx = Y[j].x, yy = Y[j].y, yz = Y[j].z;
    for (int64_t i = 0; i < nx; ++i) {
      const double dx = X[i].x - yx, dy = X[i].y - yy, dz = X[i].z - yz;
      const double r = std::sqrt(dx * dx + dy * dy + dz * dz);
      double cv = 0.0, sv = 0.0;
      if (k != 0.0) {
        cv = std::cos(k * r);
        sv = std::sin(k * r);
      }
      if (r * r <= eps2) {
        out[j * nx + i] = 0.0;
        continue;
      }
      const cplx eikr = (k != 0.0) ? cplx(cv, sv) : cplx(1.0, 0.0);
      out[j * nx + i] = cplx(eikr.real() / r, eikr.imag() / r);
    }
  }
}

TriangleNewton analytic_triangle_integrals(const V3& a, const V3& b, const V3& c,
                                           const V3& x) {  // kernels.cpp:151-207
  const V3 cr = cross(b - a, c - a);
  const double area2 = norm(cr);
  const double diam = std::max({norm(b - a), norm(c - b), norm(a - c)});
  if (area2 <= 1e-14 * diam * diam)
    throw std::invalid_argument("analytic_triangle_integrals: degenerate triangle");
  const V3 n = cr / area2;
  TriangleNewton res;
  res.height = dot(x - a, n);
  const double w0 = res.height, aw0 = std::abs(w0);
  res.rho = x - w0 * n;
  const V3 verts[3] = {a, b, c};
  double newton = 0.0, beta_total = 0.0;
  V3 grad_inplane(0, 0, 0), moment(0, 0, 0);
  for (int i = 0; i < 3; ++i) {
    const V3 pm = verts[i];
    const V3 pp = verts[(i + 1) % 3];
    const double len = norm(pp - pm);
    if (len <= 1e-300) continue;
    const V3 s_hat = (pp - pm) / len;
    const V3 m_hat = cross(s_hat, n);
    const double t = dot(pm - res.rho, m_hat);
    const double sm = dot(pm - res.rho, s_hat);
    const double sp = dot(pp - res.rho, s_hat);
    const double rm = norm(x - pm);
    const double rp = norm(x - pp);
    const double r0sq = t * t + w0 * w0;
    double f = 0.0;
    if (r0sq > 1e-28 * len * len) {
      if (sm >= 0.0)
        f = std::log((rp + sp) / (rm + sm));
      else if (sp <= 0.0)
        f = std::log((rm - sm) / (rp - sp));
      else
        f = std::log((rp + sp) * (rm - sm) / r0sq);
    }
    const double beta =
        std::atan(t * sp / (r0sq + aw0 * rp)) - std::atan(t * sm / (r0sq + aw0 * rm));
    newton += t * f - aw0 * beta;
    beta_total += beta;
    grad_inplane = grad_inplane + f * m_hat;
    const double mom = r0sq * f + sp * rp - sm * rm;
    moment = moment + mom * (0.5 * m_hat);
  }
  const double sgn = (w0 > 0.0) ? 1.0 : (w0 < 0.0 ? -1.0 : 0.0);
  res.newton = newton;
  res.grad = grad_inplane + (sgn * beta_total) * n;
  res.moment = moment;
  return res;
}

// ---------------------------------------------------------------------------
// Dense BEM (assembly.cpp:135-222, 313-320)
// ---------------------------------------------------------------------------
namespace {
struct Side {  // BemSide, assembly.cpp:135-171 (dense-path members only)
  std::vector<V3> points;
  int64_t nfree = 0;
  PointRows wrows;  // per point: (dof, w_k * B_kj), ascending dof
};

Side make_side(const Mesh& m, int g, Family f) {
  Side s;
  Quad q = quadrature(m, g);
  s.points = q.pts;
  s.nfree = dof_count(m, f);
  s.wrows = eval_rows(m, f, g);
  for (int64_t k = 0; k + 1 < (int64_t)s.wrows.start.size(); ++k)
    for (int64_t p = s.wrows.start[k]; p < s.wrows.start[k + 1]; ++p)
      s.wrows.val[p] = q.w[k] * s.wrows.val[p];
  return s;
}

// right = weighted_y^T as CSC by trial dof: per dof j, (point l, value) ascending l
struct ColLists {
  std::vector<int64_t> start;
  std::vector<int64_t> pt;
  std::vector<double> val;
};
ColLists by_dof(const Side& s) {
  ColLists c;
  c.start.assign(s.nfree + 1, 0);
  const int64_t M = (int64_t)s.points.size();
  for (int64_t k = 0; k < M; ++k)
    for (int64_t p = s.wrows.start[k]; p < s.wrows.start[k + 1]; ++p) c.start[s.wrows.dof[p] + 1]++;
  for (int64_t j = 0; j < s.nfree; ++j) c.start[j + 1] += c.start[j];
  c.pt.resize(c.start.back());
  c.val.resize(c.start.back());
  std::vector<int64_t> fill(c.start.begin(), c.start.end() - 1);
  for (int64_t k = 0; k < M; ++k)
    for (int64_t p = s.wrows.start[k]; p < s.wrows.start[k + 1]; ++p) {
      const int j = s.wrows.dof[p];
      c.pt[fill[j]] = k;
      c.val[fill[j]] = s.wrows.val[p];
      fill[j]++;
    }
  return c;
}
}  // namespace

namespace {
Side make_point_side(const std::vector<V3>& points) {  // assembly.cpp:173-190
  Side s;
  s.points = points;
  s.nfree = (int64_t)points.size();
  s.wrows.start.resize(points.size() + 1);
  for (size_t i = 0; i <= points.size(); ++i) s.wrows.start[i] = (int64_t)i;
  s.wrows.dof.resize(points.size());
  s.wrows.val.assign(points.size(), 1.0);
  for (size_t i = 0; i < points.size(); ++i) s.wrows.dof[i] = (int)i;
  return s;
}

std::vector<cplx> bem_product(const Side& tst, const Side& tri, const Kernel& K,
                              const BemOptions& opt, const std::vector<int>* rows);
}  // namespace

std::vector<cplx> bem_dense(const Mesh& mx, int gx, Family fx, const Mesh& my, int gy, Family fy,
                            const Kernel& K, const BemOptions& opt, const std::vector<int>* rows,
                            int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
  return bem_product(make_side(mx, gx, fx), make_side(my, gy, fy), K, opt, rows);
}

std::vector<cplx> radiation_dense(const std::vector<V3>& points, const Mesh& my, int gy, Family fy,
                                  const Kernel& K, const BemOptions& opt) {
  if (points.empty()) return {};
  return bem_product(make_point_side(points), make_side(my, gy, fy), K, opt, nullptr);
}

namespace {
// GalerkinEvaluator::eval (assembly.cpp:227-233 constructor eps, :240-291):
// unique supporting points in first-seen order, K over them with mask=true,
// out = lt * (K * ru).  Dense products summed in ascending index order.
std::vector<cplx> galerkin_eval(const Side& tst, const Side& tri, const Kernel& K, const std::vector<int>& rows,
                                const std::vector<int>& cols) {
  const double eps = singular_guard_radius(tst.points, tri.points);
  const ColLists xs = by_dof(tst), ys = by_dof(tri);
  const int64_t nr = (int64_t)rows.size(), nc = (int64_t)cols.size();
  std::vector<int64_t> xlocal(tst.points.size(), -1), ylocal(tri.points.size(), -1);
  std::vector<int64_t> xids, yids;
  for (int a : rows)
    for (int64_t p = xs.start[a]; p < xs.start[a + 1]; ++p)
      if (xlocal[xs.pt[p]] < 0) {
        xlocal[xs.pt[p]] = (int64_t)xids.size();
        xids.push_back(xs.pt[p]);
      }
  for (int b : cols)
    for (int64_t p = ys.start[b]; p < ys.start[b + 1]; ++p)
      if (ylocal[ys.pt[p]] < 0) {
        ylocal[ys.pt[p]] = (int64_t)yids.size();
        yids.push_back(ys.pt[p]);
      }
  const int64_t nx = (int64_t)xids.size(), ny = (int64_t)yids.size();
  std::vector<V3> X(nx), Y(ny);
  for (int64_t i = 0; i < nx; ++i) X[i] = tst.points[xids[i]];
  for (int64_t i = 0; i < ny; ++i) Y[i] = tri.points[yids[i]];
  std::vector<cplx> Km;  // nx x ny col-major
  evaluate_blocks(K, X.data(), nx, Y, Km, eps, /*mask=*/true);
  std::vector<double> lt((size_t)(nr * nx), 0.0), ru((size_t)(ny * nc), 0.0);
  for (int64_t a = 0; a < nr; ++a)
    for (int64_t p = xs.start[rows[a]]; p < xs.start[rows[a] + 1]; ++p) lt[a + nr * xlocal[xs.pt[p]]] = xs.val[p];
  for (int64_t b = 0; b < nc; ++b)
    for (int64_t p = ys.start[cols[b]]; p < ys.start[cols[b] + 1]; ++p) ru[ylocal[ys.pt[p]] + ny * b] = ys.val[p];
  std::vector<cplx> tmp((size_t)(nx * nc), cplx(0.0, 0.0)), out((size_t)(nr * nc), cplx(0.0, 0.0));
  for (int64_t b = 0; b < nc; ++b)
    for (int64_t y = 0; y < ny; ++y) {
      const double r = ru[y + ny * b];
      if (r == 0.0) continue;
      for (int64_t x = 0; x < nx; ++x) tmp[x + nx * b] += Km[x + nx * y] * r;
    }
  for (int64_t b = 0; b < nc; ++b)
    for (int64_t x = 0; x < nx; ++x) {
      const cplx v = tmp[x + nx * b];
      for (int64_t a = 0; a < nr; ++a) {
        const double l = lt[a + nr * x];
        if (l != 0.0) out[a + nr * b] += l * v;
      }
    }
  return out;
}
}  // namespace

std::vector<cplx> block_eval(const Mesh& mx, int gx, Family fx, const Mesh& my, int gy, Family fy, const Kernel& K,
                             const std::vector<int>& rows, const std::vector<int>& cols) {
  return galerkin_eval(make_side(mx, gx, fx), make_side(my, gy, fy), K, rows, cols);
}

std::vector<cplx> block_eval_points(const std::vector<V3>& points, const Mesh& my, int gy, Family fy,
                                    const Kernel& K, const std::vector<int>& rows, const std::vector<int>& cols) {
  return galerkin_eval(make_point_side(points), make_side(my, gy, fy), K, rows, cols);
}

namespace {
std::vector<cplx> bem_product(const Side& tst, const Side& tri, const Kernel& K,
                              const BemOptions& opt, const std::vector<int>* rows) {  // :192-222
  const int64_t mxp = (int64_t)tst.points.size(), myp = (int64_t)tri.points.size();
  if (!rows) {  // memory cap, assembly.cpp:196-203
    const size_t need = 16u * (size_t(tst.nfree) * tri.nfree + size_t(opt.chunk) * myp +
                               size_t(opt.chunk) * tri.nfree);
    if (need > opt.memory_cap_bytes)
      throw std::runtime_error("bem_dense: estimated memory " + std::to_string(need / 1000000) +
                               " MB exceeds the cap of " +
                               std::to_string(opt.memory_cap_bytes / 1000000) +
                               " MB; use the tol (H-matrix) variant");
  }
  const double eps = singular_guard_radius(tst.points, tri.points);
  const ColLists right = by_dof(tri);
  const int64_t nu = tri.nfree;

  // Row selection: output row r <-> test dof rows[r]; x points restricted to
  // those supporting a selected row (same per-entry accumulation sequence).
  std::vector<int> row_of(tst.nfree, -1);
  int64_t nt = tst.nfree;
  std::vector<int64_t> xsel;
  if (rows) {
    nt = (int64_t)rows->size();
    for (int64_t r = 0; r < nt; ++r) row_of[(*rows)[r]] = (int)r;
    for (int64_t k = 0; k < mxp; ++k)
      for (int64_t p = tst.wrows.start[k]; p < tst.wrows.start[k + 1]; ++p)
        if (row_of[tst.wrows.dof[p]] >= 0) {
          xsel.push_back(k);
          break;
        }
  } else {
    for (int64_t i = 0; i < nt; ++i) row_of[i] = (int)i;
    xsel.resize(mxp);
    std::iota(xsel.begin(), xsel.end(), 0);
  }
  std::vector<cplx> A(nt * nu, cplx(0.0, 0.0));
  std::vector<cplx> panel, kr;
  std::vector<V3> xchunk;
  const int64_t nsel = (int64_t)xsel.size();
  for (int64_t lo = 0; lo < nsel; lo += opt.chunk) {  // assembly.cpp:212-220
    const int64_t len = std::min<int64_t>(opt.chunk, nsel - lo);
    xchunk.resize(len);
    for (int64_t i = 0; i < len; ++i) xchunk[i] = tst.points[xsel[lo + i]];
    evaluate_blocks(K, xchunk.data(), len, tri.points, panel, eps, /*mask=*/true);
    // kr = panel * right  (len x nu)
    kr.assign(len * nu, cplx(0.0, 0.0));
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < nu; ++j)
      for (int64_t p = right.start[j]; p < right.start[j + 1]; ++p) {
        const cplx* col = &panel[right.pt[p] * len];
        const double v = right.val[p];
        cplx* out = &kr[j * len];
        for (int64_t i = 0; i < len; ++i) out[i] += col[i] * v;
      }
    // A += weighted_x(:, chunk) * kr
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < nu; ++j) {
      cplx* acol = &A[j * nt];
      for (int64_t i = 0; i < len; ++i) {
        const int64_t k = xsel[lo + i];
        const cplx kv = kr[j * len + i];
        for (int64_t p = tst.wrows.start[k]; p < tst.wrows.start[k + 1]; ++p) {
          const int r = row_of[tst.wrows.dof[p]];
          if (r >= 0) acol[r] += tst.wrows.val[p] * kv;
        }
      }
    }
  }
  return A;
}
}  // namespace

std::vector<cplx> naive_bem(const Mesh& mx, int gx, Family fx, const Mesh& my, int gy, Family fy,
                            const Kernel& K) {  // tests/support/oracles.cpp:332-360
  Quad qx = quadrature(mx, gx), qy = quadrature(my, gy);
  PointRows bx = eval_rows(mx, fx, gx), by = eval_rows(my, fy, gy);
  const int64_t nt = dof_count(mx, fx), nu = dof_count(my, fy);
  const double eps = singular_guard_radius(qx.pts, qy.pts);
  std::vector<cplx> A(nt * nu, cplx(0.0, 0.0));
  std::vector<cplx> kv;
  for (int64_t kq = 0; kq < (int64_t)qx.pts.size(); ++kq)
    for (int64_t l = 0; l < (int64_t)qy.pts.size(); ++l) {
      const double r = norm(qx.pts[kq] - qy.pts[l]);
      if (r <= eps) continue;
      std::vector<V3> Y1 = {qy.pts[l]};
      evaluate_blocks(K, &qx.pts[kq], 1, Y1, kv, eps, true);
      const cplx g = (qx.w[kq] * kv[0]) * qy.w[l];
      for (int64_t p = bx.start[kq]; p < bx.start[kq + 1]; ++p)
        for (int64_t q = by.start[l]; q < by.start[l + 1]; ++q)
          A[by.dof[q] * nt + bx.dof[p]] += (bx.val[p] * g) * by.val[q];
    }
  return A;
}

std::vector<cplx> green_matvec(const Kernel& K, const std::vector<V3>& targets,
                               const std::vector<V3>& sources, const std::vector<cplx>& q, double eps,
                               const std::vector<int64_t>& target_ids, int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
  const int64_t nt = (int64_t)target_ids.size(), ns = (int64_t)sources.size();
  const double eps2 = eps * eps, k = K.k;
  std::vector<cplx> y(nt);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t t = 0; t < nt; ++t) {
    const V3 x = targets[target_ids[t]];
    cplx acc(0.0, 0.0);
    for (int64_t s = 0; s < ns; ++s) {
      const double dx = x.x - sources[s].x, dy = x.y - sources[s].y, dz = x.z - sources[s].z;
      const double r = std::sqrt(dx * dx + dy * dy + dz * dz);
      if (r * r <= eps2) continue;  // same distance mask as kernels.cpp:104
      const cplx eikr = (k != 0.0) ? cplx(std::cos(k * r), std::sin(k * r)) : cplx(1.0, 0.0);
      acc += cplx(eikr.real() / r, eikr.imag() / r) * q[s];
    }
    y[t] = acc;
  }
  return y;
}

std::vector<cplx> matvec(const cplx* A, int64_t rows, int64_t cols, int64_t lda, const cplx* x,
                         int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
  std::vector<cplx> y(rows, cplx(0.0, 0.0));
  const int64_t RB = 256;
#pragma omp parallel for schedule(static)
  for (int64_t r0 = 0; r0 < rows; r0 += RB) {
    const int64_t r1 = std::min(rows, r0 + RB);
    for (int64_t j = 0; j < cols; ++j) {
      const cplx xj = x[j];
      const cplx* col = A + j * lda;
      for (int64_t i = r0; i < r1; ++i) y[i] += col[i] * xj;
    }
  }
  return y;
}

// ---------------------------------------------------------------------------
// Near-field correction (assembly.cpp:358-697)
// ---------------------------------------------------------------------------
namespace {
double circumradius(const Mesh& m, int e) {  // assembly.cpp:358-366
  const V3 a = m.vertices[m.elements[e][0]];
  const V3 b = m.vertices[m.elements[e][1]];
  const V3 c = m.vertices[m.elements[e][2]];
  const double area = 0.5 * norm(cross(b - a, c - a));
  if (area <= 0.0) return m.element_radius(e);
  return norm(a - b) * norm(b - c) * norm(c - a) / (4.0 * area);
}

std::vector<std::pair<int, int>> close_pairs_impl(const std::vector<V3>& xc,
                                                  const std::vector<double>& xr,
                                                  const std::vector<V3>& yc,
                                                  const std::vector<double>& yr, NearRule rule,
                                                  double hbar) {  // assembly.cpp:370-401
  double rmax = 0.0;
  for (double r : xr) rmax = std::max(rmax, r);
  for (double r : yr) rmax = std::max(rmax, r);
  double cell = std::max(3.0 * rmax, 1e-300);
  if (rule == NearRule::TwoHbar) cell = std::max(cell, 2.0 * hbar);
  std::map<std::array<int64_t, 3>, std::vector<int>> grid;
  auto key = [cell](const V3& p) {
    return std::array<int64_t, 3>{(int64_t)std::floor(p.x / cell), (int64_t)std::floor(p.y / cell),
                                  (int64_t)std::floor(p.z / cell)};
  };
  for (int e = 0; e < (int)yc.size(); ++e) grid[key(yc[e])].push_back(e);
  std::vector<std::pair<int, int>> pairs;
  for (int i = 0; i < (int)xc.size(); ++i) {
    const V3 p = xc[i];
    auto k = key(p);
    for (int64_t dx = -1; dx <= 1; ++dx)
      for (int64_t dy = -1; dy <= 1; ++dy)
        for (int64_t dz = -1; dz <= 1; ++dz) {
          auto it = grid.find({k[0] + dx, k[1] + dy, k[2] + dz});
          if (it == grid.end()) continue;
          for (int e : it->second) {
            const double radius =
                rule == NearRule::Ref ? 3.0 * std::max(xr[i], yr[e]) : 2.0 * hbar;
            if (norm(yc[e] - p) <= radius) pairs.emplace_back(i, e);
          }
        }
  }
  return pairs;
}

struct TrialLocal {  // assembly.cpp:405-411 (scalar kinds only)
  int free_index;
  int kind;  // 0 P0, 1 P1 vertex
  int vertex;
};

struct YCtx {  // assembly.cpp:447-544, "[1/r]" scalar kernel
  V3 A, B, C;
  Family fam;
  std::vector<TrialLocal> tdofs;
  std::array<V3, 3> g_bary;

  std::array<double, 3> lam_at_rho(const TriangleNewton& tn) const {  // :455-466
    std::array<double, 3> lam{0, 0, 0};
    if (fam != P1) return lam;
    const V3 e0 = B - A, e1 = C - A, d = tn.rho - A;
    // (E^T E) uv = E^T d, LDLT with diagonal pivoting (Eigen LDLT)
    double m00 = dot(e0, e0), m01 = dot(e0, e1), m11 = dot(e1, e1);
    double r0 = dot(e0, d), r1 = dot(e1, d);
    const bool swap = std::abs(m11) > std::abs(m00);
    if (swap) {
      std::swap(m00, m11);
      std::swap(r0, r1);
    }
    const double d0 = m00, l10 = m01 / d0, d1 = m11 - l10 * l10 * d0;
    const double z0 = r0, z1 = r1 - l10 * z0;
    const double y1 = z1 / d1, y0 = z0 / d0;
    double u1 = y1, u0 = y0 - l10 * u1;
    if (swap) std::swap(u0, u1);
    lam = {1.0 - u0 - u1, u0, u1};
    return lam;
  }

  double exact(size_t j, const TriangleNewton& tn, const std::array<double, 3>& lam) const {
    const TrialLocal& td = tdofs[j];  // :469-500 (scalar kernel, kinds 0/1)
    if (td.kind == 0) return tn.newton;
    return lam[td.vertex] * tn.newton + dot(g_bary[td.vertex], tn.moment);
  }

  double gauss(const V3& x, size_t j, const Quad& yq, int ye, int yg, double eps,
               const Rule& yrule) const {  // :504-543
    const TrialLocal& td = tdofs[j];
    double d = 0.0;
    for (int l = 0; l < yg; ++l) {
      const int64_t idx = (int64_t)ye * yg + l;
      const V3 rv = x - yq.pts[idx];
      const double w = yq.w[idx];
      const double r = norm(rv);
      if (r <= eps) continue;
      const double psi = td.kind == 0 ? 1.0 : yrule.bary[l][td.vertex];
      const double kv = 1.0 / r;
      d += w * kv * psi;
    }
    return d;
  }
};

using Local = std::vector<double>;  // nt x ntr row-major

struct CellCtx {
  const Mesh* xmesh;
  Family xf;
  int ex;
  const YCtx* y;
  int nt;
  int64_t* calls;
};

Local accurate_cell(const CellCtx& c, const double corners[3][3], double measure_frac) {
  const Rule& rule = triangle_rule(7);  // assembly.cpp:548-577
  const int ntr = (int)c.y->tdofs.size();
  Local out(c.nt * ntr, 0.0);
  const double measure = c.xmesh->element_measure(c.ex) * measure_frac;
  const V3 v0 = c.xmesh->vertices[c.xmesh->elements[c.ex][0]];
  const V3 v1 = c.xmesh->vertices[c.xmesh->elements[c.ex][1]];
  const V3 v2 = c.xmesh->vertices[c.xmesh->elements[c.ex][2]];
  for (int q = 0; q < 7; ++q) {
    std::array<double, 3> bary;
    for (int col = 0; col < 3; ++col)
      bary[col] = rule.bary[q][0] * corners[0][col] + rule.bary[q][1] * corners[1][col] +
                  rule.bary[q][2] * corners[2][col];
    const V3 x = bary[0] * v0 + bary[1] * v1 + bary[2] * v2;
    const double w = rule.w[q] * measure;
    const TriangleNewton tn = analytic_triangle_integrals(c.y->A, c.y->B, c.y->C, x);
    ++*c.calls;
    const auto lam = c.y->lam_at_rho(tn);
    for (int j = 0; j < ntr; ++j) {
      const double d = c.y->exact(j, tn, lam);
      for (int i = 0; i < c.nt; ++i) {
        const double tv = basis_value(c.xf, bary, i);
        const double acc = tv * d;
        out[i * ntr + j] += w * acc;
      }
    }
  }
  return out;
}

void accurate_adaptive(const CellCtx& c, const double corners[3][3], double measure_frac,
                       double cell_tol, int depth, Local& acc,
                       std::array<int64_t, 8>* hist) {  // assembly.cpp:581-605
  const Local whole = accurate_cell(c, corners, measure_frac);
  double m01[3], m12[3], m20[3];
  for (int k = 0; k < 3; ++k) {
    m01[k] = 0.5 * (corners[0][k] + corners[1][k]);
    m12[k] = 0.5 * (corners[1][k] + corners[2][k]);
    m20[k] = 0.5 * (corners[2][k] + corners[0][k]);
  }
  double sub[4][3][3];
  for (int k = 0; k < 3; ++k) {
    sub[0][0][k] = corners[0][k]; sub[0][1][k] = m01[k];        sub[0][2][k] = m20[k];
    sub[1][0][k] = corners[1][k]; sub[1][1][k] = m12[k];        sub[1][2][k] = m01[k];
    sub[2][0][k] = corners[2][k]; sub[2][1][k] = m20[k];        sub[2][2][k] = m12[k];
    sub[3][0][k] = m01[k];        sub[3][1][k] = m12[k];        sub[3][2][k] = m20[k];
  }
  Local split(whole.size(), 0.0);
  for (int s = 0; s < 4; ++s) {
    const Local part = accurate_cell(c, sub[s], 0.25 * measure_frac);
    for (size_t t = 0; t < split.size(); ++t) split[t] += part[t];
  }
  double dmax = 0.0;
  for (size_t t = 0; t < split.size(); ++t) dmax = std::max(dmax, std::abs(split[t] - whole[t]));
  if (dmax <= cell_tol || depth >= 6) {
    for (size_t t = 0; t < split.size(); ++t) acc[t] += split[t];
    if (hist) (*hist)[std::min(depth, 7)]++;
    return;
  }
  for (int s = 0; s < 4; ++s)
    accurate_adaptive(c, sub[s], 0.25 * measure_frac, 0.5 * cell_tol, depth + 1, acc, hist);
}

struct PairResult {
  std::vector<int> rows, cols;
  Local local;
  int64_t calls = 0, gauss = 0;
  std::array<int64_t, 8> hist{};
};

PairResult one_pair(const Mesh& mx, int gx, Family fx, const Mesh& my, int gy, Family fy,
                    const Quad& xq, const Quad& yq, double eps, int ex, int ye) {
  PairResult pr;
  YCtx y;  // assembly.cpp:645-655
  y.A = my.vertices[my.elements[ye][0]];
  y.B = my.vertices[my.elements[ye][1]];
  y.C = my.vertices[my.elements[ye][2]];
  y.fam = fy;
  if (fy == P0) {
    y.tdofs.push_back({ye, 0, 0});
  } else {
    for (int l = 0; l < 3; ++l) y.tdofs.push_back({my.elements[ye][l], 1, l});
    y.g_bary = barycentric_gradients(my, ye);
  }
  const std::vector<int> test_dofs = element_dofs(mx, fx, ex);
  const int nt = (int)test_dofs.size(), ntr = (int)y.tdofs.size();
  const Rule& xrule = triangle_rule(gx);
  const Rule& yrule = triangle_rule(gy);
  Local local(nt * ntr, 0.0);
  for (int k = 0; k < gx; ++k) {  // Gauss x Gauss part, :659-674
    const int64_t xqi = (int64_t)ex * gx + k;
    const V3 x = xq.pts[xqi];
    const double w = xq.w[xqi];
    for (int j = 0; j < ntr; ++j) {
      const double d = y.gauss(x, j, yq, ye, gy, eps, yrule);
      pr.gauss += gy;
      for (int i = 0; i < nt; ++i) {
        const double acc = basis_value(fx, xrule.bary[k], i) * d;
        local[i * ntr + j] -= w * acc;
      }
    }
  }
  CellCtx c{&mx, fx, ex, &y, nt, &pr.calls};
  const double whole_bary[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  Local acc(nt * ntr, 0.0);
  const Local probe = accurate_cell(c, whole_bary, 1.0);  // :679-683
  double pmax = 0.0;
  for (double v : probe) pmax = std::max(pmax, std::abs(v));
  const double cell_tol = 1e-8 * std::max(pmax, 1e-300);
  accurate_adaptive(c, whole_bary, 1.0, cell_tol, 0, acc, &pr.hist);
  for (size_t t = 0; t < local.size(); ++t) local[t] += acc[t];
  pr.rows = test_dofs;
  for (auto& td : y.tdofs) pr.cols.push_back(td.free_index);
  pr.local = std::move(local);
  return pr;
}

void element_geometry(const Mesh& m, std::vector<V3>& c, std::vector<double>& r) {
  c.resize(m.ne());
  r.resize(m.ne());
  for (int e = 0; e < m.ne(); ++e) {
    c[e] = m.element_centroid(e);
    r[e] = circumradius(m, e);
  }
}
}  // namespace

std::vector<std::pair<int, int>> close_pairs(const std::vector<V3>& xc, const std::vector<double>& xr,
                                             const std::vector<V3>& yc,
                                             const std::vector<double>& yr) {
  return close_pairs_impl(xc, xr, yc, yr, NearRule::Ref, 0.0);
}

std::vector<std::pair<int, int>> near_pairs(const Mesh& mx, const Mesh& my, NearRule rule,
                                            double hbar) {
  std::vector<V3> xc, yc;
  std::vector<double> xr, yr;
  element_geometry(mx, xc, xr);
  element_geometry(my, yc, yr);
  return close_pairs_impl(xc, xr, yc, yr, rule, hbar);
}

std::vector<Triplet> regularize(const Mesh& mx, int gx, Family fx, const Mesh& my, int gy, Family fy,
                                const std::string& singular_name, RegStats* stats, NearRule rule,
                                double hbar, const std::vector<int>* only_x, int threads) {
  if (singular_name != "[1/r]") {  // assembly.cpp:611-614
    if (singular_name == "grady[1/r]")
      throw std::invalid_argument("regularize: grady[1/r] is outside this restatement (MFIE)");
    throw std::invalid_argument("regularize: unsupported singular kernel '" + singular_name + "'");
  }
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
  const Quad xq = quadrature(mx, gx), yq = quadrature(my, gy);
  const double eps = singular_guard_radius(xq.pts, yq.pts);
  auto pairs = near_pairs(mx, my, rule, hbar);
  if (only_x) {
    std::vector<char> keep(mx.ne(), 0);
    for (int e : *only_x) keep[e] = 1;
    std::vector<std::pair<int, int>> f;
    for (auto& p : pairs)
      if (keep[p.first]) f.push_back(p);
    pairs.swap(f);
  }
  std::vector<PairResult> res(pairs.size());
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t p = 0; p < (int64_t)pairs.size(); ++p)
    res[p] = one_pair(mx, gx, fx, my, gy, fy, xq, yq, eps, pairs[p].first, pairs[p].second);
  // setFromTriplets: duplicates summed in triplet order, output col-major sorted.
  std::map<std::pair<int, int>, double> acc;
  for (auto& r : res) {
    const int ntr = (int)r.cols.size();
    for (size_t i = 0; i < r.rows.size(); ++i)
      for (int j = 0; j < ntr; ++j) {
        auto key = std::make_pair(r.cols[j], r.rows[i]);
        auto it = acc.find(key);
        if (it == acc.end())
          acc.emplace(key, r.local[i * ntr + j]);
        else
          it->second += r.local[i * ntr + j];
      }
    if (stats) {
      stats->pairs++;
      stats->analytic_calls += r.calls;
      stats->gauss_evals += r.gauss;
      int64_t leaves = 0;
      for (int d = 0; d < 8; ++d) stats->depth_hist[d] += r.hist[d], leaves += r.hist[d];
      stats->pair_leaves.push_back((int32_t)leaves);
    }
  }
  if (stats)
    for (auto& pr : pairs) stats->pair_ex.push_back(pr.first), stats->pair_ey.push_back(pr.second);
  std::vector<Triplet> out;
  out.reserve(acc.size());
  for (auto& [k, v] : acc) out.push_back({k.second, k.first, v});
  return out;
}

std::vector<Triplet> regularize_radiation(const std::vector<V3>& points, const Mesh& my, int gy, Family fy,
                                          const std::string& singular_name) {  // assembly.cpp:699-750
  if (singular_name != "[1/r]") {
    if (singular_name == "grady[1/r]")
      throw std::invalid_argument("regularize: grady[1/r] is outside this restatement (MFIE)");
    throw std::invalid_argument("regularize: unsupported singular kernel '" + singular_name + "'");
  }
  const Quad yq = quadrature(my, gy);
  const Rule& yrule = triangle_rule(gy);
  const double eps = singular_guard_radius(points, yq.pts);
  std::vector<V3> yc;
  std::vector<double> yr;
  element_geometry(my, yc, yr);
  const std::vector<double> zero_radius(points.size(), 0.0);
  const auto pairs = close_pairs_impl(points, zero_radius, yc, yr, NearRule::Ref, 0.0);
  std::map<std::pair<int, int>, double> acc;  // setFromTriplets: (col, row) -> sum in triplet order
  for (const auto& [pt, ye] : pairs) {
    YCtx y;
    y.A = my.vertices[my.elements[ye][0]];
    y.B = my.vertices[my.elements[ye][1]];
    y.C = my.vertices[my.elements[ye][2]];
    y.fam = fy;
    if (fy == P0) {
      y.tdofs.push_back({ye, 0, 0});
    } else {
      for (int l = 0; l < 3; ++l) y.tdofs.push_back({my.elements[ye][l], 1, l});
      y.g_bary = barycentric_gradients(my, ye);
    }
    const V3 x = points[pt];
    const TriangleNewton tn = analytic_triangle_integrals(y.A, y.B, y.C, x);
    const auto lam = y.lam_at_rho(tn);
    for (size_t j = 0; j < y.tdofs.size(); ++j) {
      const double exact = y.exact(j, tn, lam);
      const double gauss = y.gauss(x, j, yq, ye, gy, eps, yrule);
      const auto key = std::make_pair(y.tdofs[j].free_index, pt);
      auto it = acc.find(key);
      if (it == acc.end())
        acc.emplace(key, exact - gauss);
      else
        it->second += exact - gauss;
    }
  }
  std::vector<Triplet> out;
  out.reserve(acc.size());
  for (auto& [k, v] : acc) out.push_back({k.second, k.first, v});
  return out;
}

std::vector<PairValue> regularize_pairs_p0(const Mesh& mx, int gx, const Mesh& my, int gy,
                                           NearRule rule, double hbar,
                                           const std::vector<int>* only_x, int threads,
                                           RegStats* stats) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
  const Quad xq = quadrature(mx, gx), yq = quadrature(my, gy);
  const double eps = singular_guard_radius(xq.pts, yq.pts);
  auto pairs = near_pairs(mx, my, rule, hbar);
  if (only_x) {
    std::vector<char> keep(mx.ne(), 0);
    for (int e : *only_x) keep[e] = 1;
    std::vector<std::pair<int, int>> f;
    for (auto& p : pairs)
      if (keep[p.first]) f.push_back(p);
    pairs.swap(f);
  }
  std::vector<PairResult> res(pairs.size());
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t p = 0; p < (int64_t)pairs.size(); ++p)
    res[p] = one_pair(mx, gx, P0, my, gy, P0, xq, yq, eps, pairs[p].first, pairs[p].second);
  std::vector<PairValue> out(pairs.size());
  for (size_t p = 0; p < pairs.size(); ++p) {
    out[p] = {pairs[p].first, pairs[p].second, res[p].local[0]};
    if (stats) {
      stats->pairs++;
      stats->analytic_calls += res[p].calls;
      stats->gauss_evals += res[p].gauss;
      for (int d = 0; d < 8; ++d) stats->depth_hist[d] += res[p].hist[d];
    }
  }
  return out;
}

// ---------------------------------------------------------------------------
// FEM helpers (assembly.cpp:59-111)
// ---------------------------------------------------------------------------
std::vector<double> linear_form_ones(const Mesh& m, Family f, int g) {
  const Quad q = quadrature(m, g);
  const PointRows b = eval_rows(m, f, g);
  std::vector<double> F(dof_count(m, f), 0.0);
  for (int64_t k = 0; k < (int64_t)q.pts.size(); ++k)
    for (int64_t p = b.start[k]; p < b.start[k + 1]; ++p) F[b.dof[p]] += b.val[p] * (q.w[k] * 1.0);
  return F;
}

std::vector<double> mass_dense(const Mesh& m, Family f, int g) {
  const Quad q = quadrature(m, g);
  const PointRows b = eval_rows(m, f, g);
  const int64_t n = dof_count(m, f);
  std::vector<double> M(n * n, 0.0);
  for (int64_t k = 0; k < (int64_t)q.pts.size(); ++k)
    for (int64_t p = b.start[k]; p < b.start[k + 1]; ++p)
      for (int64_t r = b.start[k]; r < b.start[k + 1]; ++r)
        M[b.dof[r] * n + b.dof[p]] += b.val[p] * q.w[k] * b.val[r];
  return M;
}

// ---------------------------------------------------------------------------
// Reference test-support oracles (tests/support/oracles.cpp:106-245)
// ---------------------------------------------------------------------------
namespace {
double factorial(int n) {
  double f = 1.0;
  for (int i = 2; i <= n; ++i) f *= i;
  return f;
}

struct GaussLegendre01 {  // n-point Gauss-Legendre on [0,1], nodes by Newton
  std::vector<double> x, w;
  explicit GaussLegendre01(int n) {
    for (int i = 1; i <= n; ++i) {
      double t = std::cos(M_PI * (i - 0.25) / (n + 0.5)), dp = 0.0;
      for (int it = 0; it < 100; ++it) {
        double p0 = 1.0, p1 = t;
        for (int k = 2; k <= n; ++k) {
          const double p2 = ((2.0 * k - 1.0) * t * p1 - (k - 1.0) * p0) / k;
          p0 = p1;
          p1 = p2;
        }
        dp = n * (t * p1 - p0) / (t * t - 1.0);
        const double dt = p1 / dp;
        t -= dt;
        if (std::abs(dt) < 1e-16) break;
      }
      x.push_back(0.5 * (t + 1.0));
      w.push_back(0.5 * 2.0 / ((1.0 - t * t) * dp * dp));
    }
  }
};

double adaptive_1d(const std::function<double(double)>& f, double lo, double hi, double tol,
                   int depth) {
  static const GaussLegendre01 gl(15);
  auto quad = [&](double a, double b) {
    double s = 0.0;
    for (int i = 0; i < 15; ++i) s += gl.w[i] * f(a + (b - a) * gl.x[i]);
    return s * (b - a);
  };
  const double whole = quad(lo, hi);
  const double mid = 0.5 * (lo + hi);
  const double split = quad(lo, mid) + quad(mid, hi);
  if (std::abs(split - whole) <= tol || depth >= 40) return split;
  return adaptive_1d(f, lo, mid, 0.5 * tol, depth + 1) + adaptive_1d(f, mid, hi, 0.5 * tol, depth + 1);
}

double tri7(const std::function<double(const V3&)>& f, const V3& a, const V3& b, const V3& c) {
  const Rule& r = triangle_rule(7);
  const double area = 0.5 * norm(cross(b - a, c - a));
  double s = 0.0;
  for (int i = 0; i < 7; ++i) s += r.w[i] * f(r.bary[i][0] * a + r.bary[i][1] * b + r.bary[i][2] * c);
  return s * area;
}

double adaptive_tri_rec(const std::function<double(const V3&)>& f, const V3& a, const V3& b,
                        const V3& c, double tol, int depth) {
  const double whole = tri7(f, a, b, c);
  const V3 ab = 0.5 * (a + b), bc = 0.5 * (b + c), ca = 0.5 * (c + a);
  const double split = tri7(f, a, ab, ca) + tri7(f, b, bc, ab) + tri7(f, c, ca, bc) + tri7(f, ab, bc, ca);
  if (std::abs(split - whole) <= tol || depth >= 24) return split;
  const double t = 0.5 * tol;
  return adaptive_tri_rec(f, a, ab, ca, t, depth + 1) + adaptive_tri_rec(f, b, bc, ab, t, depth + 1) +
         adaptive_tri_rec(f, c, ca, bc, t, depth + 1) + adaptive_tri_rec(f, ab, bc, ca, t, depth + 1);
}

struct Radial {
  V3 n, rho;
  double w0;
  V3 verts[3];
  double scale;
};
Radial radial_setup(const V3& a, const V3& b, const V3& c, const V3& x) {
  Radial s;
  const V3 cr = cross(b - a, c - a);
  s.n = cr / norm(cr);
  s.w0 = dot(x - a, s.n);
  s.rho = x - s.w0 * s.n;
  s.verts[0] = a;
  s.verts[1] = b;
  s.verts[2] = c;
  s.scale = std::max({norm(b - a), norm(c - b), norm(a - c)});
  return s;
}
double radial_sum(const Radial& s,
                  const std::function<double(const V3&, const V3&, double, double)>& edge_term,
                  double tol) {
  double total = 0.0;
  for (int i = 0; i < 3; ++i) {
    const V3 pa = s.verts[i] - s.rho;
    const V3 pb = s.verts[(i + 1) % 3] - s.rho;
    const double cr = dot(cross(pa, pb), s.n);
    if (std::abs(cr) <= 1e-15 * s.scale * s.scale) continue;
    total += edge_term(pa, pb, cr >= 0 ? 1.0 : -1.0, tol);
  }
  return total;
}
}  // namespace

double simplex_monomial(int dim, int a, int b, int c) {
  switch (dim) {
    case 1: return 1.0 / (a + 1);
    case 2: return factorial(a) * factorial(b) / factorial(a + b + 2);
    case 3: return factorial(a) * factorial(b) * factorial(c) / factorial(a + b + c + 3);
    default: throw std::invalid_argument("simplex_monomial: bad dimension");
  }
}

double newton_oracle(const V3& a, const V3& b, const V3& c, const V3& x, double tol) {
  Radial s = radial_setup(a, b, c, x);
  const double cc = std::abs(s.w0);
  auto edge = [&](const V3& pa, const V3& pb, double sign, double etol) {
    const double jac = norm(cross(pa, pb));
    auto fv = [&](double v) {
      const double g = norm((1.0 - v) * pa + v * pb);
      return (std::sqrt(cc * cc + g * g) - cc) / (g * g);
    };
    return sign * jac * adaptive_1d(fv, 0.0, 1.0, etol / jac, 0);
  };
  return radial_sum(s, edge, tol);
}

V3 newton_moment_oracle(const V3& a, const V3& b, const V3& c, const V3& x, double tol) {
  Radial s = radial_setup(a, b, c, x);
  const double cc = std::abs(s.w0);
  V3 out(0, 0, 0);
  for (int comp = 0; comp < 3; ++comp) {
    auto edge = [&](const V3& pa, const V3& pb, double sign, double etol) {
      const double jac = norm(cross(pa, pb));
      auto fv = [&](double v) {
        const V3 e = (1.0 - v) * pa + v * pb;
        const double g = norm(e);
        const double rt = std::sqrt(cc * cc + g * g);
        const double iu = cc <= 1e-300 ? 1.0 / (2.0 * g)
                                       : rt / (2.0 * g * g) -
                                             (cc * cc) / (2.0 * g * g * g) * std::log((g + rt) / cc);
        return e[comp] * iu;
      };
      return sign * jac * adaptive_1d(fv, 0.0, 1.0, etol / jac, 0);
    };
    out[comp] = radial_sum(s, edge, tol);
  }
  return out;
}

V3 newton_grad_oracle(const V3& a, const V3& b, const V3& c, const V3& x, double tol) {
  Radial s = radial_setup(a, b, c, x);
  const double cc = std::abs(s.w0);
  if (cc <= 1e-12 * s.scale) throw std::invalid_argument("newton_grad_oracle: x must lie off the plane");
  V3 out(0, 0, 0);
  for (int comp = 0; comp < 4; ++comp) {
    auto edge = [&](const V3& pa, const V3& pb, double sign, double etol) {
      const double jac = norm(cross(pa, pb));
      auto fv = [&](double v) {
        const V3 e = (1.0 - v) * pa + v * pb;
        const double g = norm(e);
        const double rt = std::sqrt(cc * cc + g * g);
        if (comp == 3) return (1.0 / cc - 1.0 / rt) / (g * g);
        const double iu = std::asinh(g / cc) / (g * g * g) - 1.0 / (g * g * rt);
        return -e[comp] * iu;
      };
      return sign * jac * adaptive_1d(fv, 0.0, 1.0, etol / jac, 0);
    };
    const double val = radial_sum(s, edge, tol);
    if (comp == 3)
      out = out + (s.w0 * val) * s.n;
    else
      out[comp] += val;
  }
  return out;
}

double double_newton_oracle(const V3& a, const V3& b, const V3& c, double tol) {
  auto outer = [&](const V3& x) { return newton_oracle(a, b, c, x, tol * 1e-3); };
  return adaptive_tri_rec(outer, a, b, c, tol, 0);
}

}  // namespace oracle
