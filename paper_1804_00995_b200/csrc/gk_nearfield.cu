// K3: near-field singular correction — regularize (assembly.cpp:609-697).
//
// For every near element pair (close_pairs, assembly.cpp:370-401) the
// correction is  local = semi-analytic(1/r) - Gauss x Gauss(1/r)  on the pair's
// local dofs; duplicates are summed in pair order (setFromTriplets).
//
// Device layout: one warp per near pair, pairs handed out by an atomic work
// counter (costs range from ~500 to ~50k analytic integrals per pair; the
// processing order does not change any result).  The recursion of
// accurate_adaptive (:581-605) runs on an explicit per-warp stack in shared
// memory, up to eight nodes per step with one lane per (node, sub-cell): each
// lane evaluates its sub-cell's 7 analytic_triangle_integrals calls
// (kernels.cpp:151-207) in registers, so a full step keeps all 32 lanes busy
// (see k_nearfield_b).  The parent's 'whole' value is the child's sub-cell
// value, so it is carried on the stack instead of being recomputed (the
// reference recomputes it: ~20% of its calls).  Per-triangle quantities of the
// y element (normal, edge frames) are computed once per pair.
#include <cuda_runtime.h>

#include <cstdlib>

#include <algorithm>
#include <array>
#include <cmath>
#include <map>
#include <memory>

#include "../../include/galerk_b200_diag.h"
#include "gk_internal.hpp"
#include "gk_math.cuh"

namespace gk {
namespace {

constexpr int kNfWarps = 4;       // warps per CTA
// Resident CTAs per SM the register budget is sized for, and rule points
// evaluated in lockstep per lane.  P0 x P0 (cfg 3), measured on cfg 3:
// (CTAs, unroll) = (4, 2) 48.9 ms, (5, 1) 47.7, (6, 1) 47.4, (7, 1) 47.8,
// (8, 1) 48.3, (3, 2) 54.1, (2, 4) 64.1: more resident warps beat more ILP per
// lane.  The P1 variants carry up to 9 local values and keep (4, 2).
template <int NL>
struct NfTune {
  static constexpr int minb = NL == 1 ? 6 : 4;
  static constexpr int qunroll = NL == 1 ? 1 : 2;
};
constexpr int kMaxLoc = 9;        // local matrix entries (P1 x P1)

struct V3 {
  double x, y, z;
};
__device__ __forceinline__ V3 mk(double a, double b, double c) { return {a, b, c}; }
__device__ __forceinline__ V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V3 operator*(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ V3 cross(V3 a, V3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ double nrm(V3 a) { return sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }
// |a| through the refined reciprocal square root (~1 ulp, no slow path); 0 at a = 0
__device__ __forceinline__ double nrm_fast(V3 a) {
  const double r2 = fma(a.z, a.z, fma(a.y, a.y, a.x * a.x));
  return r2 > 0.0 ? r2 * gk::rsqrt_refined(r2) : 0.0;
}

// div_fast, atan2_fast and log_ratio live in gk_math.cuh (shared with the
// device math accuracy probe, gk_diag_math).

// y-triangle frame shared by all analytic calls of a pair
struct YTri {
  V3 v[3];       // A, B, C
  V3 n;          // unit normal
  V3 s_hat[3], m_hat[3];
  double len[3];
  double r0min[3];  // 1e-28 len^2 (the log guard, kernels.cpp:184); +inf for an empty edge
  V3 g_bary[3];  // P1 tangential barycentric gradients (femspace.cpp:254-277)
  // in-plane frame for the batched kernel: origin v[0], axes e1 = s_hat[0],
  // e2 = n x e1, e3 = n; the triangle is P0 = 0, P1 = (len0, 0), P2
  V3 e1, e2;
  double p2x, p2y;
  double s2x[3], s2y[3];   // edge unit vectors in the plane; m_hat = (s2y, -s2x)
  double area2;            // |(B - A) x (C - A)|
  double g2x[3], g2y[3];   // in-plane barycentric gradients (P1)
};

struct V2 {
  double x, y;
};

// Fill the in-plane frame of T (after v, n, s_hat, len, g_bary).
__device__ __forceinline__ void frame2(YTri& T, double area2, bool p1) {
  T.e1 = T.s_hat[0];
  T.e2 = cross(T.n, T.e1);
  const V3 c = T.v[2] - T.v[0];
  T.p2x = dot(c, T.e1);
  T.p2y = dot(c, T.e2);
  T.area2 = area2;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    T.s2x[i] = dot(T.s_hat[i], T.e1);
    T.s2y[i] = dot(T.s_hat[i], T.e2);
    T.g2x[i] = p1 ? dot(T.g_bary[i], T.e1) : 0.0;
    T.g2y[i] = p1 ? dot(T.g_bary[i], T.e2) : 0.0;
  }
}

struct NfArgs {
  int64_t npairs;
  const int32_t* pair_ex;
  const int32_t* pair_ey;
  const double* xv;  // x mesh vertices [nv*3]
  const int32_t* xe; // x mesh elements [ne*3]
  const double* yv;
  const int32_t* ye;
  const double* xq;  // x quadrature per point: x,y,z,w  [nex*gx*4]
  const double* yq;  // y quadrature per point
  const double* xrule;  // [g*3] barycentric rule of the x domain (per plan)
  const double* yrule;
  int gx, gy;
  double eps;
  double* local;     // [npairs * kMaxLoc]
  unsigned long long* work;   // atomic pair counter
  unsigned long long* stats;  // [0] analytic calls, [1..7] leaves per depth, [8] degenerate flag
  int32_t* pair_leaves;       // [npairs] accepted leaves of accurate_adaptive per pair (diagnostics)
};

__constant__ double c_r7_bary[7][3];
__constant__ double c_r7_w[7];

// kernels.cpp:151-207 with the y-triangle frame precomputed, written for ILP:
// the three edges are independent chains (unrolled, branch-free selects for
// the cancellation-safe log argument).  The reference sums, per edge,
//   beta_i = atan(t sp / (r0^2 + |w| rp)) - atan(t sm / (r0^2 + |w| rm)),
// and uses only the sum (newton: -|w| sum beta; grad: sgn(w) n sum beta).
// That sum is the solid angle of the triangle seen from x:
//   sum_i beta_i = -sgn(w) Omega,
//   Omega = 2 atan2(A.(B x C), |A||B||C| + (A.B)|C| + (A.C)|B| + (B.C)|A|)
// (van Oosterom-Strackee, A,B,C = vertices - x; |A|,|B|,|C| are the edge
// end distances already at hand), so one atan2 replaces six atans:
//   newton = sum_i t_i f_i + w Omega.
// (Checked against the per-edge sum on 2e4 random configurations: max
// difference 3.4e-13 rad, i.e. rounding.)  At w = 0 the term vanishes, as it
// does in the reference (|w| = 0, sgn(w) = 0).
template <bool MOMENT>
__device__ __forceinline__ void analytic(const YTri& T, V3 x, double& newton, V3& moment, V3& rho) {
  // vertices relative to x, shared by the edge terms and the solid angle.  The
  // edge coordinates t = (v_i - rho).m_hat and s = (v - rho).s_hat equal
  // (v - x).m_hat and (v - x).s_hat because rho - x is along the normal,
  // which is orthogonal to both in-plane unit vectors; rho itself is only
  // needed for the P1 barycentric weights.
  const V3 Av[3] = {T.v[0] - x, T.v[1] - x, T.v[2] - x};
  const double w0 = -dot(Av[0], T.n);  // (x - v0).n
  rho = MOMENT ? x - w0 * T.n : x;
  const double rv[3] = {nrm_fast(Av[0]), nrm_fast(Av[1]), nrm_fast(Av[2])};  // rp of edge i == rm of edge i+1
  const double trip = dot(Av[0], cross(Av[1], Av[2]));
  const double vden = fma(rv[0] * rv[1], rv[2],
                          fma(dot(Av[0], Av[1]), rv[2], fma(dot(Av[0], Av[2]), rv[1], dot(Av[1], Av[2]) * rv[0])));
  const double omega = 2.0 * atan2_fast(trip, vden);
  double f[3], t[3], mo[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int ip = i == 2 ? 0 : i + 1;
    const double ti = dot(Av[i], T.m_hat[i]);
    const double sm = dot(Av[i], T.s_hat[i]);
    const double sp = dot(Av[ip], T.s_hat[i]);
    const double rm = rv[i], rp = rv[ip];
    const double r0sq = ti * ti + w0 * w0;
    const bool a = sm >= 0.0, b = sp <= 0.0;
    const double num = a ? rp + sp : (b ? rm - sm : (rp + sp) * (rm - sm));
    const double den = a ? rm + sm : (b ? rp - sp : r0sq);
    const bool ok = r0sq > T.r0min[i];  // same test as r0sq > 1e-28 len^2 && len > 1e-300
    f[i] = ok ? log_ratio(num, den) : 0.0;
    t[i] = T.len[i] > 1e-300 ? ti : 0.0;
    if (MOMENT) mo[i] = r0sq * f[i] + sp * rp - sm * rm;
  }
  newton = (t[0] * f[0] + t[1] * f[1] + t[2] * f[2]) + w0 * omega;
  if (MOMENT) {
    V3 mom = mk(0, 0, 0);
#pragma unroll
    for (int i = 0; i < 3; ++i)
      if (T.len[i] > 1e-300) mom = mom + mo[i] * (0.5 * T.m_hat[i]);
    moment = mom;
  }
}

// analytic() in the y triangle's in-plane frame: x = (u, v, w) local.  With
// A_i = v_i - x = (a_i, b_i, -w): every edge dot product is a 2D one, the
// normal offset w0 is w, and the triple product of the solid angle is the
// constant -w |(B-A) x (C-A)|.  The moment is returned in-plane.
template <bool MOMENT>
__device__ __forceinline__ void analytic2(const YTri& T, double u, double v, double w, double& newton, V2& moment) {
  const double a[3] = {-u, T.len[0] - u, T.p2x - u};
  const double b[3] = {-v, -v, T.p2y - v};
  const double w2 = w * w;
  double rv[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double r2 = fma(a[i], a[i], fma(b[i], b[i], w2));
    rv[i] = r2 > 0.0 ? r2 * gk::rsqrt_refined(r2) : 0.0;
  }
  const double d01 = fma(a[0], a[1], fma(b[0], b[1], w2));
  const double d02 = fma(a[0], a[2], fma(b[0], b[2], w2));
  const double d12 = fma(a[1], a[2], fma(b[1], b[2], w2));
  const double trip = -w * T.area2;
  const double vden = fma(rv[0] * rv[1], rv[2], fma(d01, rv[2], fma(d02, rv[1], d12 * rv[0])));
  const double omega = 2.0 * atan2_fast(trip, vden);
  double f[3], t[3], mo[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int ip = i == 2 ? 0 : i + 1;
    const double sx = T.s2x[i], sy = T.s2y[i];
    const double ti = fma(a[i], sy, -b[i] * sx);  // (a, b) . m, m = (sy, -sx)
    const double sm = fma(a[i], sx, b[i] * sy);
    const double sp = fma(a[ip], sx, b[ip] * sy);
    const double rm = rv[i], rp = rv[ip];
    const double r0sq = fma(ti, ti, w2);
    const bool ca = sm >= 0.0, cb = sp <= 0.0;
    const double num = ca ? rp + sp : (cb ? rm - sm : (rp + sp) * (rm - sm));
    const double den = ca ? rm + sm : (cb ? rp - sp : r0sq);
    const bool ok = r0sq > T.r0min[i];
    f[i] = ok ? log_ratio(num, den) : 0.0;
    t[i] = T.len[i] > 1e-300 ? ti : 0.0;
    if (MOMENT) mo[i] = r0sq * f[i] + sp * rp - sm * rm;
  }
  newton = (t[0] * f[0] + t[1] * f[1] + t[2] * f[2]) + w * omega;
  if (MOMENT) {
    V2 m = {0.0, 0.0};
#pragma unroll
    for (int i = 0; i < 3; ++i)
      if (T.len[i] > 1e-300) {
        const double h = 0.5 * mo[i];
        m.x = fma(h, T.s2y[i], m.x);
        m.y = fma(-h, T.s2x[i], m.y);
      }
    moment = m;
  }
}

// exact_values() from analytic2: lam at rho = (u, v) is affine in the plane
// (lam_0 = 1 + g_0.(u,v), lam_j = g_j.(u,v)), the moment term a 2D dot.
template <int NT, int NTR>
__device__ __forceinline__ void exact_values2(const YTri& T, double newton, V2 mom, double u, double v,
                                              double d[NTR]) {
  if (NTR == 1) {
    d[0] = newton;
  } else {
#pragma unroll
    for (int j = 0; j < NTR; ++j) {
      const double lam = (j == 0 ? 1.0 : 0.0) + fma(T.g2x[j], u, T.g2y[j] * v);
      d[j] = fma(lam, newton, fma(T.g2x[j], mom.x, T.g2y[j] * mom.y));
    }
  }
}

template <int NT, int NTR>
__device__ __forceinline__ void exact_values(const YTri& T, double newton, V3 moment, V3 rho, double d[NTR]) {
  if (NTR == 1) {
    d[0] = newton;
  } else {
    // lam_at_rho (assembly.cpp:455-466): (E^T E) uv = E^T (rho - A), pivoted LDLT
    const V3 e0 = T.v[1] - T.v[0], e1 = T.v[2] - T.v[0], dd = rho - T.v[0];
    double m00 = dot(e0, e0), m01 = dot(e0, e1), m11 = dot(e1, e1);
    double r0 = dot(e0, dd), r1 = dot(e1, dd);
    const bool sw = fabs(m11) > fabs(m00);
    if (sw) {
      double tt = m00;
      m00 = m11;
      m11 = tt;
      tt = r0;
      r0 = r1;
      r1 = tt;
    }
    const double d0 = m00, l10 = m01 / d0, d1 = m11 - l10 * l10 * d0;
    const double z0 = r0, z1 = r1 - l10 * z0;
    const double y1 = z1 / d1, y0 = z0 / d0;
    double u1 = y1, u0 = y0 - l10 * u1;
    if (sw) {
      const double tt = u0;
      u0 = u1;
      u1 = tt;
    }
    const double lam[3] = {1.0 - u0 - u1, u0, u1};
#pragma unroll
    for (int j = 0; j < 3; ++j) d[j] = lam[j] * newton + dot(T.g_bary[j], moment);
  }
}

// ---- batched traversal (B): lane = (node k of the batch, sub-cell) -------------
// Up to eight stack nodes are processed per iteration.  Lane 4k+s owns sub-cell
// s of node k and evaluates its seven 7-point-rule points in q order (the
// accurate_cell sum, assembly.cpp:562-575) in registers; the four sub values of
// a node meet in its leader lane by shuffles (split = 0 + s0 + s1 + s2 + s3),
// which applies the accept test (assembly.cpp:598-604) and accumulates the
// accepted split; refused nodes' children (sub-cell corners, sub value as
// their `whole`, depth + 1) are pushed by the four lanes that computed them.
// The set of accepted leaves is the reference's (each decision depends only on
// its own node); only the order in which leaves are summed differs.  Nodes are
// compact: barycentric corners are dyadic (midpoints of midpoints) and stored
// exactly as integers in units of 1/128; tol and frac follow from the depth.
constexpr int kStackB = 160;  // >= 8 + 24 * 5 + 32 for batch 8, branching 4, depth 6
constexpr int kUnit = 128;    // corner coordinates in units of 1/128 (depth <= 6)

template <int NL>
struct NodeB {
  double whole[NL];
  int16_t c[6];  // (b0, b1) of the three corners, units of 1/kUnit (b2 = 1 - b0 - b1)
  int16_t depth;
};

template <int NL>
struct WarpSmemB {
  NodeB<NL> stack[kStackB];
  double vals[8][kMaxLoc];  // Gauss part / probe scratch (<= 7 lanes)
  double acc[kMaxLoc];
  YTri tri;
  unsigned long long leaves[7];
};

template <int NT, int NTR>
__global__ void __launch_bounds__(32 * kNfWarps, NfTune<NT * NTR>::minb) k_nearfield_b(const NfArgs a) {
  constexpr int NL = NT * NTR;
  extern __shared__ unsigned char smem_raw[];
  WarpSmemB<NL>& S = reinterpret_cast<WarpSmemB<NL>*>(smem_raw)[threadIdx.x / 32];
  const int lane = threadIdx.x & 31;
  if (lane < 7) S.leaves[lane] = 0ull;
  unsigned long long calls = 0;
  while (true) {
    unsigned long long p = 0;
    if (lane == 0) p = atomicAdd(a.work, 1ull);
    p = __shfl_sync(0xffffffffu, p, 0);
    if (p >= (unsigned long long)a.npairs) break;
    const int ex = a.pair_ex[p], ey = a.pair_ey[p];
    // ---- y triangle frame (lane 0), kernels.cpp:153-175
    if (lane == 0) {
      YTri& T = S.tri;
      for (int c = 0; c < 3; ++c) {
        const int vi = a.ye[3 * ey + c];
        T.v[c] = mk(a.yv[3 * vi], a.yv[3 * vi + 1], a.yv[3 * vi + 2]);
      }
      const V3 cr = cross(T.v[1] - T.v[0], T.v[2] - T.v[0]);
      const double area2 = nrm(cr);
      const double diam = fmax(fmax(nrm(T.v[1] - T.v[0]), nrm(T.v[2] - T.v[1])), nrm(T.v[0] - T.v[2]));
      if (area2 <= 1e-14 * diam * diam) atomicExch(a.stats + 8, 1ull);
      T.n = mk(cr.x / area2, cr.y / area2, cr.z / area2);
      for (int i = 0; i < 3; ++i) {
        const V3 pm = T.v[i], pp = T.v[i == 2 ? 0 : i + 1];
        const double len = nrm(pp - pm);
        T.len[i] = len;
        T.r0min[i] = len > 1e-300 ? 1e-28 * len * len : __longlong_as_double(0x7ff0000000000000ll);
        const V3 d = pp - pm;
        T.s_hat[i] = mk(d.x / len, d.y / len, d.z / len);
        T.m_hat[i] = cross(T.s_hat[i], T.n);
      }
      if (NTR == 3) {
        const V3 e1 = T.v[1] - T.v[0], e2 = T.v[2] - T.v[0];
        const double g00 = dot(e1, e1), g01 = dot(e1, e2), g11 = dot(e2, e2);
        const double det = g00 * g11 - g01 * g01;
        const double i00 = g11 / det, i01 = -g01 / det, i11 = g00 / det;
        T.g_bary[1] = mk(e1.x * i00 + e2.x * i01, e1.y * i00 + e2.y * i01, e1.z * i00 + e2.z * i01);
        T.g_bary[2] = mk(e1.x * i01 + e2.x * i11, e1.y * i01 + e2.y * i11, e1.z * i01 + e2.z * i11);
        T.g_bary[0] = mk(0, 0, 0) - T.g_bary[1] - T.g_bary[2];
      }
      frame2(T, area2, NTR == 3);
    }
    __syncwarp();
    const YTri& T = S.tri;
    V3 xv[3];
    for (int c = 0; c < 3; ++c) {
      const int vi = a.xe[3 * ex + c];
      xv[c] = mk(a.xv[3 * vi], a.xv[3 * vi + 1], a.xv[3 * vi + 2]);
    }
    const double measure_x = 0.5 * nrm(cross(xv[1] - xv[0], xv[2] - xv[0]));
    // x-triangle vertices in the y triangle's frame: every rule point is then
    // (u, v, w) = sum b_c X_c and the analytic integral works in 2D
    double Xu[3], Xv[3], Xw[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const V3 d = xv[c] - T.v[0];
      Xu[c] = dot(d, T.e1);
      Xv[c] = dot(d, T.e2);
      Xw[c] = dot(d, T.n);
    }

    // ---- Gauss x Gauss part (assembly.cpp:659-674, YContext::gauss :504-543)
    if (lane < a.gx) {
      const double* xq = a.xq + ((int64_t)ex * a.gx + lane) * 4;
      const V3 x = mk(xq[0], xq[1], xq[2]);
      const double w = xq[3];
      double d[NTR];
#pragma unroll
      for (int j = 0; j < NTR; ++j) d[j] = 0.0;
      for (int l = 0; l < a.gy; ++l) {
        const double* yq = a.yq + ((int64_t)ey * a.gy + l) * 4;
        const double r = nrm(x - mk(yq[0], yq[1], yq[2]));
        if (r <= a.eps) continue;
        const double kv = 1.0 / r;
#pragma unroll
        for (int j = 0; j < NTR; ++j) {
          const double psi = NTR == 1 ? 1.0 : a.yrule[3 * l + j];
          d[j] += yq[3] * kv * psi;
        }
      }
#pragma unroll
      for (int i = 0; i < NT; ++i) {
        const double tv = NT == 1 ? 1.0 : a.xrule[3 * lane + i];
#pragma unroll
        for (int j = 0; j < NTR; ++j) S.vals[lane][i * NTR + j] = -(w * (tv * d[j]));
      }
    }
    __syncwarp();
    if (lane < NL) {  // local(i,j) -= w * acc, in x-point order
      double s = 0.0;
      for (int k = 0; k < a.gx; ++k) s += S.vals[k][lane];
      S.acc[lane] = s;
    }
    __syncwarp();

    // ---- probe = accurate_cell(whole) (lanes 0..6)
    double pv[NL];
    double tol0;
    {
      if (lane < 7) {
        const double* b = c_r7_bary[lane];
        const double u = b[0] * Xu[0] + b[1] * Xu[1] + b[2] * Xu[2];
        const double v = b[0] * Xv[0] + b[1] * Xv[1] + b[2] * Xv[2];
        const double wn = b[0] * Xw[0] + b[1] * Xw[1] + b[2] * Xw[2];
        const double w = c_r7_w[lane] * (measure_x * 1.0);
        double nw;
        V2 mo;
        analytic2<NTR == 3>(T, u, v, wn, nw, mo);
        double d[NTR];
        exact_values2<NT, NTR>(T, nw, mo, u, v, d);
#pragma unroll
        for (int i = 0; i < NT; ++i)
#pragma unroll
          for (int j = 0; j < NTR; ++j) S.vals[lane][i * NTR + j] = w * ((NT == 1 ? 1.0 : b[i]) * d[j]);
      }
      __syncwarp();
      double pmax = 0.0;
#pragma unroll
      for (int t = 0; t < NL; ++t) {
        double s = 0.0;
        for (int q = 0; q < 7; ++q) s += S.vals[q][t];
        pv[t] = s;
        pmax = fmax(pmax, fabs(s));
      }
      tol0 = 1e-8 * fmax(pmax, 1e-300);
      __syncwarp();
      if (lane == 0) {
        NodeB<NL>& r = S.stack[0];
        const int16_t I[6] = {kUnit, 0, 0, kUnit, 0, 0};
        for (int c = 0; c < 6; ++c) r.c[c] = I[c];
        for (int t = 0; t < NL; ++t) r.whole[t] = pv[t];
        r.depth = 0;
      }
    }
    calls += 7;  // the probe
    int pair_leaves = 0;
    double adapt[NL];  // leader lanes: accepted splits, in acceptance order
#pragma unroll
    for (int t = 0; t < NL; ++t) adapt[t] = 0.0;
    int sp = 1;
    const int k = lane >> 2, sub = lane & 3;
    __syncwarp();
    // ---- accurate_adaptive (assembly.cpp:581-605), batched
    while (sp > 0) {
      const int K = min(8, sp), base = sp - K;
      const bool active = k < K;
      double sv[NL], whole[NL];
#pragma unroll
      for (int t = 0; t < NL; ++t) sv[t] = whole[t] = 0.0;
      int depth = 0, cc[6] = {0, 0, 0, 0, 0, 0};
      if (active) {
        const NodeB<NL>& nd = S.stack[base + k];
        depth = nd.depth;
#pragma unroll
        for (int t = 0; t < NL; ++t) whole[t] = nd.whole[t];
        // sub-cell corners (assembly.cpp:587-594) in integer units, exact:
        // sub 0 = (c0, m01, m20), 1 = (c1, m12, m01), 2 = (c2, m20, m12), 3 = (m01, m12, m20)
        const int u0 = nd.c[0], v0 = nd.c[1], u1 = nd.c[2], v1 = nd.c[3], u2 = nd.c[4], v2 = nd.c[5];
        const int mu01 = (u0 + u1) >> 1, mv01 = (v0 + v1) >> 1, mu12 = (u1 + u2) >> 1, mv12 = (v1 + v2) >> 1;
        const int mu20 = (u2 + u0) >> 1, mv20 = (v2 + v0) >> 1;
        cc[0] = sub == 0 ? u0 : sub == 1 ? u1 : sub == 2 ? u2 : mu01;
        cc[1] = sub == 0 ? v0 : sub == 1 ? v1 : sub == 2 ? v2 : mv01;
        cc[2] = sub == 0 ? mu01 : sub == 1 ? mu12 : sub == 2 ? mu20 : mu12;
        cc[3] = sub == 0 ? mv01 : sub == 1 ? mv12 : sub == 2 ? mv20 : mv12;
        cc[4] = sub == 0 ? mu20 : sub == 1 ? mu01 : sub == 2 ? mu12 : mu20;
        cc[5] = sub == 0 ? mv20 : sub == 1 ? mv01 : sub == 2 ? mv12 : mv20;
        const double inv = 1.0 / kUnit;
        double cr[9];  // (b0, b1, b2) of the three corners, exact dyadics
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          cr[3 * i] = cc[2 * i] * inv;
          cr[3 * i + 1] = cc[2 * i + 1] * inv;
          cr[3 * i + 2] = (kUnit - cc[2 * i] - cc[2 * i + 1]) * inv;
        }
        const double frac = ldexp(1.0, -2 * (depth + 1));  // 0.25^(depth+1), as repeated quartering
        // the sub-cell's corners in the y frame: a rule point's frame
        // coordinates are affine in its barycentrics, so each point costs
        // three 3-term sums instead of barycentrics + frame sums
        double Cu[3], Cv[3], Cw[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          Cu[i] = cr[3 * i] * Xu[0] + cr[3 * i + 1] * Xu[1] + cr[3 * i + 2] * Xu[2];
          Cv[i] = cr[3 * i] * Xv[0] + cr[3 * i + 1] * Xv[1] + cr[3 * i + 2] * Xv[2];
          Cw[i] = cr[3 * i] * Xw[0] + cr[3 * i + 1] * Xw[1] + cr[3 * i + 2] * Xw[2];
        }
#pragma unroll NfTune<NL>::qunroll
        for (int q = 0; q < 7; ++q) {
          // re-read the y-triangle frame from shared memory every point instead
          // of keeping ~60 registers of it live across the loop
          asm volatile("" ::: "memory");
          const double r0 = c_r7_bary[q][0], r1 = c_r7_bary[q][1], r2 = c_r7_bary[q][2];
          double b[3];
          if (NT == 3) {
#pragma unroll
            for (int c = 0; c < 3; ++c) b[c] = r0 * cr[c] + r1 * cr[3 + c] + r2 * cr[6 + c];
          }
          const double u = r0 * Cu[0] + r1 * Cu[1] + r2 * Cu[2];
          const double v = r0 * Cv[0] + r1 * Cv[1] + r2 * Cv[2];
          const double wn = r0 * Cw[0] + r1 * Cw[1] + r2 * Cw[2];
          const double w = c_r7_w[q] * (measure_x * frac);
          double nw;
          V2 mo;
          analytic2<NTR == 3>(T, u, v, wn, nw, mo);
          double d[NTR];
          exact_values2<NT, NTR>(T, nw, mo, u, v, d);
#pragma unroll
          for (int i = 0; i < NT; ++i)
#pragma unroll
            for (int j = 0; j < NTR; ++j) sv[i * NTR + j] += w * ((NT == 1 ? 1.0 : b[i]) * d[j]);
        }
      }
      calls += 28 * K;
      // split = 0 + s0 + s1 + s2 + s3 at the node's leader lane (sub 0)
      double split[NL];
      double dmax = 0.0;
#pragma unroll
      for (int t = 0; t < NL; ++t) {
        const double s1 = __shfl_down_sync(0xffffffffu, sv[t], 1);
        const double s2 = __shfl_down_sync(0xffffffffu, sv[t], 2);
        const double s3 = __shfl_down_sync(0xffffffffu, sv[t], 3);
        split[t] = 0.0 + sv[t] + s1 + s2 + s3;
        dmax = fmax(dmax, fabs(split[t] - whole[t]));
      }
      const bool leader = active && sub == 0;
      const bool accept = dmax <= ldexp(tol0, -depth) || depth >= 6;
      if (leader && accept) {
#pragma unroll
        for (int t = 0; t < NL; ++t) adapt[t] += split[t];
      }
      {  // leaf histogram: one ballot per depth, lane 0 updates the warp's counters
        const bool leaf = leader && accept;
#pragma unroll
        for (int d = 0; d < 7; ++d) {
          const unsigned m = __ballot_sync(0xffffffffu, leaf && min(depth, 6) == d);
          if (lane == 0 && m) S.leaves[d] += (unsigned long long)__popc(m);
        }
        pair_leaves += __popc(__ballot_sync(0xffffffffu, leaf));
      }
      const unsigned refused = __ballot_sync(0xffffffffu, leader && !accept);
      const bool mine = (refused >> (lane & ~3)) & 1u;  // my node is refused: push my sub-cell
      __syncwarp();  // every lane has read its node before children overwrite the slots
      if (active && mine) {
        const int rank = __popc(refused & ((1u << (lane & ~3)) - 1u));
        NodeB<NL>& ch = S.stack[base + 4 * rank + sub];
#pragma unroll
        for (int c = 0; c < 6; ++c) ch.c[c] = (int16_t)cc[c];
#pragma unroll
        for (int t = 0; t < NL; ++t) ch.whole[t] = sv[t];
        ch.depth = (int16_t)(depth + 1);
      }
      sp = base + 4 * __popc(refused);
      __syncwarp();
    }
    // accepted leaves of the eight leader lanes, summed in lane order
#pragma unroll
    for (int t = 0; t < NL; ++t) {
      double tot = 0.0;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) tot += __shfl_sync(0xffffffffu, adapt[t], 4 * kk);
      adapt[t] = tot;
    }
    if (lane == 0) {
      for (int t = 0; t < NL; ++t) a.local[p * kMaxLoc + t] = S.acc[t] + adapt[t];
      a.pair_leaves[p] = pair_leaves;
    }
    __syncwarp();
  }
  __syncwarp();
  if (lane == 0) atomicAdd(a.stats, calls);
  if (lane < 7 && S.leaves[lane]) atomicAdd(a.stats + 1 + lane, S.leaves[lane]);
}

// regularize_radiation (assembly.cpp:725-745): one thread per (point, element)
// pair; local[j] = exact(j) - gauss(j) for the element's trial dofs.
template <int NTR>
__global__ void __launch_bounds__(128) k_nf_points(const NfArgs a) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= a.npairs) return;
  const int pt = a.pair_ex[p], ey = a.pair_ey[p];
  YTri T;
  for (int c = 0; c < 3; ++c) {
    const int vi = a.ye[3 * ey + c];
    T.v[c] = mk(a.yv[3 * vi], a.yv[3 * vi + 1], a.yv[3 * vi + 2]);
  }
  const V3 cr = cross(T.v[1] - T.v[0], T.v[2] - T.v[0]);
  const double area2 = nrm(cr);
  const double diam = fmax(fmax(nrm(T.v[1] - T.v[0]), nrm(T.v[2] - T.v[1])), nrm(T.v[0] - T.v[2]));
  if (area2 <= 1e-14 * diam * diam) atomicExch(a.stats + 8, 1ull);
  T.n = mk(cr.x / area2, cr.y / area2, cr.z / area2);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const V3 d = T.v[i == 2 ? 0 : i + 1] - T.v[i];
    const double len = nrm(d);
    T.len[i] = len;
    T.r0min[i] = len > 1e-300 ? 1e-28 * len * len : __longlong_as_double(0x7ff0000000000000ll);
    T.s_hat[i] = mk(d.x / len, d.y / len, d.z / len);
    T.m_hat[i] = cross(T.s_hat[i], T.n);
  }
  if (NTR == 3) {
    const V3 e1 = T.v[1] - T.v[0], e2 = T.v[2] - T.v[0];
    const double g00 = dot(e1, e1), g01 = dot(e1, e2), g11 = dot(e2, e2);
    const double det = g00 * g11 - g01 * g01;
    const double i00 = g11 / det, i01 = -g01 / det, i11 = g00 / det;
    T.g_bary[1] = mk(e1.x * i00 + e2.x * i01, e1.y * i00 + e2.y * i01, e1.z * i00 + e2.z * i01);
    T.g_bary[2] = mk(e1.x * i01 + e2.x * i11, e1.y * i01 + e2.y * i11, e1.z * i01 + e2.z * i11);
    T.g_bary[0] = mk(0, 0, 0) - T.g_bary[1] - T.g_bary[2];
  }
  const V3 x = mk(a.xv[3 * pt], a.xv[3 * pt + 1], a.xv[3 * pt + 2]);
  double nw;
  V3 mo, rho;
  analytic<NTR == 3>(T, x, nw, mo, rho);
  double d[NTR];
  exact_values<1, NTR>(T, nw, mo, rho, d);
  double gs[NTR];
#pragma unroll
  for (int j = 0; j < NTR; ++j) gs[j] = 0.0;
  for (int l = 0; l < a.gy; ++l) {  // YContext::gauss (assembly.cpp:504-543)
    const double* yq = a.yq + ((int64_t)ey * a.gy + l) * 4;
    const double r = nrm(x - mk(yq[0], yq[1], yq[2]));
    if (r <= a.eps) continue;
    const double kv = 1.0 / r;
#pragma unroll
    for (int j = 0; j < NTR; ++j) gs[j] += yq[3] * kv * (NTR == 1 ? 1.0 : a.yrule[3 * l + j]);
  }
#pragma unroll
  for (int j = 0; j < NTR; ++j) a.local[p * kMaxLoc + j] = d[j] - gs[j];
  atomicAdd(a.stats, 1ull);
}

// A[row + col*lda].re += sum of the entry's contributions in pair order
__global__ void k_nf_reduce(int64_t n, const int64_t* __restrict__ start, const int64_t* __restrict__ src,
                            const double* __restrict__ local, double* __restrict__ vals) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  double s = local[src[start[e]]];
  for (int64_t p = start[e] + 1; p < start[e + 1]; ++p) s += local[src[p]];
  vals[e] = s;
}

__global__ void k_nf_apply(int64_t n, const int32_t* __restrict__ row, const int32_t* __restrict__ col,
                           const double* __restrict__ vals, double2* __restrict__ A, long long lda) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  double2* a = A + row[e] + (long long)col[e] * lda;
  a->x += vals[e];
}

// ---- host helpers ---------------------------------------------------------------
struct HV3 {
  double x, y, z;
};
HV3 hsub(HV3 a, HV3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
double hnrm(HV3 a) { return std::sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }
HV3 hcross(HV3 a, HV3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }

struct HostMesh {
  const double* v;
  const int32_t* e;
  int64_t nv, ne;
  HV3 vert(int64_t e_, int c) const {
    const int i = e[3 * e_ + c];
    return {v[3 * i], v[3 * i + 1], v[3 * i + 2]};
  }
  HV3 centroid(int64_t k) const {  // mesh.cpp:73-78
    HV3 c{0, 0, 0};
    for (int i = 0; i < 3; ++i) {
      const HV3 p = vert(k, i);
      c = {c.x + p.x, c.y + p.y, c.z + p.z};
    }
    return {c.x / 3.0, c.y / 3.0, c.z / 3.0};
  }
  // kernels.cpp:151-157: analytic_triangle_integrals refuses a triangle with
  // |(b-a)x(c-a)| <= 1e-14 diam^2 (the regularize loop calls it for the y
  // triangle of every near pair).  Checked here, on the host, so that
  // compute / apply / triplets all raise the reference's exception before any
  // device work (the kernel's own flag stays as a second line of defence).
  bool degenerate(int64_t k) const {
    const HV3 a = vert(k, 0), b = vert(k, 1), c = vert(k, 2);
    const double area2 = hnrm(hcross(hsub(b, a), hsub(c, a)));
    const double diam = std::max({hnrm(hsub(b, a)), hnrm(hsub(c, b)), hnrm(hsub(a, c))});
    return area2 <= 1e-14 * diam * diam;
  }
  void check_pairs(const std::vector<int32_t>& pey) const {
    std::vector<char> seen((size_t)ne, 0);
    for (int32_t e : pey)
      if (!seen[e]) {
        seen[e] = 1;
        if (degenerate(e)) throw std::invalid_argument("analytic_triangle_integrals: degenerate triangle");
      }
  }
  double circumradius(int64_t k) const {  // assembly.cpp:358-366
    const HV3 a = vert(k, 0), b = vert(k, 1), c = vert(k, 2);
    const double area = 0.5 * hnrm(hcross(hsub(b, a), hsub(c, a)));
    if (area <= 0.0) {
      const HV3 cc = centroid(k);
      double r = 0.0;
      for (int i = 0; i < 3; ++i) r = std::max(r, hnrm(hsub(vert(k, i), cc)));
      return r;
    }
    return hnrm(hsub(a, b)) * hnrm(hsub(b, c)) * hnrm(hsub(c, a)) / (4.0 * area);
  }
};

std::vector<double> host_rule(int n, bool weights) {
  // triangle rules as in csrc/host/galerk.cpp (1/3/6/7 points)
  std::vector<double> b, w;
  auto orbit = [&](double a, double wt) {
    const double c = 1.0 - 2.0 * a;
    const double pts[3][3] = {{a, a, c}, {a, c, a}, {c, a, a}};
    for (auto& p : pts) b.insert(b.end(), p, p + 3), w.push_back(wt);
  };
  if (n == 1) {
    b = {1.0 / 3, 1.0 / 3, 1.0 / 3};
    w = {1.0};
  } else if (n == 3) {
    b = {0.5, 0.5, 0.0, 0.0, 0.5, 0.5, 0.5, 0.0, 0.5};
    w = {1.0 / 3, 1.0 / 3, 1.0 / 3};
  } else if (n == 6) {
    orbit(0.44594849091596488632, 0.22338158967801146570);
    orbit(0.091576213509770743460, 0.10995174365532186764);
  } else if (n == 7) {
    const double s15 = std::sqrt(15.0);
    b = {1.0 / 3, 1.0 / 3, 1.0 / 3};
    w = {9.0 / 40.0};
    orbit((6.0 - s15) / 21.0, (155.0 - s15) / 1200.0);
    orbit((6.0 + s15) / 21.0, (155.0 + s15) / 1200.0);
  } else {
    throw std::invalid_argument("regularize: unsupported quadrature rule");
  }
  return weights ? w : b;
}

std::vector<double> host_quadrature(const HostMesh& m, int g) {  // quadrature.cpp:167-189, x,y,z,w
  const std::vector<double> b = host_rule(g, false), w = host_rule(g, true);
  std::vector<double> out((size_t)m.ne * g * 4);
  for (int64_t e = 0; e < m.ne; ++e) {
    const HV3 a = m.vert(e, 0), bb = m.vert(e, 1), c = m.vert(e, 2);
    const double measure = 0.5 * hnrm(hcross(hsub(bb, a), hsub(c, a)));
    const HV3 vs[3] = {a, bb, c};
    for (int q = 0; q < g; ++q) {
      HV3 p{0, 0, 0};
      for (int k = 0; k < 3; ++k) {
        const double s = b[3 * q + k];
        p = {p.x + s * vs[k].x, p.y + s * vs[k].y, p.z + s * vs[k].z};
      }
      double* o = &out[((size_t)e * g + q) * 4];
      o[0] = p.x;
      o[1] = p.y;
      o[2] = p.z;
      o[3] = w[q] * measure;
    }
  }
  return out;
}

}  // namespace
}  // namespace gk

using namespace gk;

struct gk_nearfield {
  bool points = false;  // collocation form (regularize_radiation)
  int fx = 0, fy = 0, gx = 0, gy = 0, nt = 1, ntr = 1;
  int64_t npairs = 0, nentries = 0;
  double eps = 0.0;
  DevBuf pair_ex, pair_ey, xv, xe, yv, ye, xq, yq, local, work, stats, ent_row, ent_col, ent_start, ent_src, vals,
      xrule, yrule, leaves;
  std::vector<int32_t> h_row, h_col;
  bool computed = false;
};

extern "C" {

gk_status gk_nearfield_create(const gk_mesh_side* test, const gk_mesh_side* trial, const char* singular_name,
                              int32_t near_rule, double hbar, gk_nearfield** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("gk_nearfield_create: null output");
    *out = nullptr;
    const std::string name = singular_name ? singular_name : "";
    if (name != "[1/r]") {  // assembly.cpp:611-614
      if (name == "grady[1/r]")
        throw std::invalid_argument("regularize: grady[1/r] (MFIE/CFIE) is outside the B200 hot path");
      throw std::invalid_argument("regularize: unsupported singular kernel '" + name + "'");
    }
    if (!test || !trial) throw std::invalid_argument("regularize: null side");
    for (const gk_mesh_side* s : {test, trial}) {
      if (s->family != 0 && s->family != 1)
        throw std::invalid_argument("regularize: unsupported trial family/operator combination");
      if (s->ne <= 0 || !s->vertices || !s->elements) throw std::invalid_argument("regularize: empty mesh");
    }
    if (near_rule != GK_NEAR_REF && near_rule != GK_NEAR_2HBAR)
      throw std::invalid_argument("regularize: unknown near-field rule");
    require_device();
    auto N = std::make_unique<gk_nearfield>();
    N->fx = test->family;
    N->fy = trial->family;
    N->gx = test->g;
    N->gy = trial->g;
    N->nt = N->fx == 0 ? 1 : 3;
    N->ntr = N->fy == 0 ? 1 : 3;
    const HostMesh mx{test->vertices, test->elements, test->nv, test->ne};
    const HostMesh my{trial->vertices, trial->elements, trial->nv, trial->ne};
    const std::vector<double> xq = host_quadrature(mx, N->gx), yq = host_quadrature(my, N->gy);
    // eps over both point sets (kernels.cpp:14-19)
    {
      const int64_t na = mx.ne * N->gx, nb = my.ne * N->gy;
      std::vector<double> ax(na), ay(na), az(na), bx(nb), by(nb), bz(nb);
      for (int64_t i = 0; i < na; ++i) ax[i] = xq[4 * i], ay[i] = xq[4 * i + 1], az[i] = xq[4 * i + 2];
      for (int64_t i = 0; i < nb; ++i) bx[i] = yq[4 * i], by[i] = yq[4 * i + 1], bz[i] = yq[4 * i + 2];
      N->eps = guard_radius_pts(na, ax.data(), ay.data(), az.data(), nb, bx.data(), by.data(), bz.data());
    }
    // close_pairs (assembly.cpp:370-401): hash grid of y centroids, 27-cell probe
    std::vector<HV3> xc(mx.ne), yc(my.ne);
    std::vector<double> xr(mx.ne), yr(my.ne);
    double rmax = 0.0;
    for (int64_t e = 0; e < mx.ne; ++e) xc[e] = mx.centroid(e), xr[e] = mx.circumradius(e), rmax = std::max(rmax, xr[e]);
    for (int64_t e = 0; e < my.ne; ++e) yc[e] = my.centroid(e), yr[e] = my.circumradius(e), rmax = std::max(rmax, yr[e]);
    double cell = std::max(3.0 * rmax, 1e-300);
    if (near_rule == GK_NEAR_2HBAR) cell = std::max(cell, 2.0 * hbar);
    auto key = [cell](const HV3& p) {
      return std::array<int64_t, 3>{(int64_t)std::floor(p.x / cell), (int64_t)std::floor(p.y / cell),
                                    (int64_t)std::floor(p.z / cell)};
    };
    std::map<std::array<int64_t, 3>, std::vector<int>> grid;
    for (int64_t e = 0; e < my.ne; ++e) grid[key(yc[e])].push_back((int)e);
    std::vector<int32_t> pex, pey;
    for (int64_t i = 0; i < mx.ne; ++i) {
      const auto k = key(xc[i]);
      for (int64_t dx = -1; dx <= 1; ++dx)
        for (int64_t dy = -1; dy <= 1; ++dy)
          for (int64_t dz = -1; dz <= 1; ++dz) {
            const auto it = grid.find({k[0] + dx, k[1] + dy, k[2] + dz});
            if (it == grid.end()) continue;
            for (int e : it->second) {
              const double radius = near_rule == GK_NEAR_REF ? 3.0 * std::max(xr[i], yr[e]) : 2.0 * hbar;
              if (hnrm(hsub(yc[e], xc[i])) <= radius) {
                pex.push_back((int32_t)i);
                pey.push_back(e);
              }
            }
          }
    }
    N->npairs = (int64_t)pex.size();
    my.check_pairs(pey);
    // summed entries (setFromTriplets): col-major order, contributions in pair order
    std::map<std::pair<int32_t, int32_t>, std::vector<int64_t>> ent;
    for (int64_t p = 0; p < N->npairs; ++p)
      for (int i = 0; i < N->nt; ++i)
        for (int j = 0; j < N->ntr; ++j) {
          const int32_t r = N->fx == 0 ? pex[p] : test->elements[3 * pex[p] + i];
          const int32_t c = N->fy == 0 ? pey[p] : trial->elements[3 * pey[p] + j];
          if (r >= test->nfree || c >= trial->nfree) throw std::invalid_argument("regularize: dof out of range");
          ent[{c, r}].push_back(p * kMaxLoc + i * N->ntr + j);
        }
    N->nentries = (int64_t)ent.size();
    std::vector<int64_t> start{0}, src;
    for (auto& [k, v] : ent) {
      N->h_col.push_back(k.first);
      N->h_row.push_back(k.second);
      src.insert(src.end(), v.begin(), v.end());
      start.push_back((int64_t)src.size());
    }
    N->pair_ex.upload(pex);
    N->pair_ey.upload(pey);
    N->xv.upload(test->vertices, sizeof(double) * 3 * test->nv);
    N->xe.upload(test->elements, sizeof(int32_t) * 3 * test->ne);
    N->yv.upload(trial->vertices, sizeof(double) * 3 * trial->nv);
    N->ye.upload(trial->elements, sizeof(int32_t) * 3 * trial->ne);
    N->xq.upload(xq);
    N->yq.upload(yq);
    N->local.alloc(sizeof(double) * kMaxLoc * std::max<int64_t>(1, N->npairs));
    N->leaves.alloc(sizeof(int32_t) * std::max<int64_t>(1, N->npairs));
    N->work.alloc(sizeof(unsigned long long));
    N->stats.alloc(sizeof(unsigned long long) * 9);
    N->ent_row.upload(N->h_row);
    N->ent_col.upload(N->h_col);
    N->ent_start.upload(start);
    N->ent_src.upload(src);
    N->vals.alloc(sizeof(double) * std::max<int64_t>(1, N->nentries));
    // rule tables
    const std::vector<double> b7 = host_rule(7, false), w7 = host_rule(7, true);
    double bx[21] = {0}, by[21] = {0};
    const std::vector<double> rbx = host_rule(N->gx, false), rby = host_rule(N->gy, false);
    std::copy(rbx.begin(), rbx.end(), bx);
    std::copy(rby.begin(), rby.end(), by);
    cuda_check(cudaMemcpyToSymbol(c_r7_bary, b7.data(), sizeof(double) * 21), "rule7");
    cuda_check(cudaMemcpyToSymbol(c_r7_w, w7.data(), sizeof(double) * 7), "rule7w");
    N->xrule.upload(bx, sizeof(bx));
    N->yrule.upload(by, sizeof(by));
    *out = N.release();
  });
}

gk_status gk_nearfield_create_points(int64_t npts, const double* points, const gk_mesh_side* trial,
                                     const char* singular_name, gk_nearfield** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("gk_nearfield_create_points: null output");
    *out = nullptr;
    const std::string name = singular_name ? singular_name : "";
    if (name != "[1/r]") {  // assembly.cpp:701-704
      if (name == "grady[1/r]")
        throw std::invalid_argument("regularize: grady[1/r] (MFIE/CFIE) is outside the B200 hot path");
      throw std::invalid_argument("regularize: unsupported singular kernel '" + name + "'");
    }
    if (!trial || trial->ne <= 0 || !trial->vertices || !trial->elements)
      throw std::invalid_argument("regularize: dom_y must be a triangle mesh");
    if (trial->family != 0 && trial->family != 1)
      throw std::invalid_argument("regularize: unsupported trial family/operator combination");
    if (npts < 0 || (npts > 0 && !points)) throw std::invalid_argument("regularize_radiation: bad points");
    require_device();
    auto N = std::make_unique<gk_nearfield>();
    N->points = true;
    N->fx = 0;
    N->fy = trial->family;
    N->gx = 1;
    N->gy = trial->g;
    N->nt = 1;
    N->ntr = N->fy == 0 ? 1 : 3;
    const HostMesh my{trial->vertices, trial->elements, trial->nv, trial->ne};
    const std::vector<double> yq = host_quadrature(my, N->gy);
    {
      const int64_t nb = my.ne * N->gy;
      std::vector<double> ax(npts), ay(npts), az(npts), bx(nb), by(nb), bz(nb);
      for (int64_t i = 0; i < npts; ++i) ax[i] = points[3 * i], ay[i] = points[3 * i + 1], az[i] = points[3 * i + 2];
      for (int64_t i = 0; i < nb; ++i) bx[i] = yq[4 * i], by[i] = yq[4 * i + 1], bz[i] = yq[4 * i + 2];
      N->eps = guard_radius_pts(npts, ax.data(), ay.data(), az.data(), nb, bx.data(), by.data(), bz.data());
    }
    // close_pairs(points, zero radii, yc, yr) (assembly.cpp:721-722)
    std::vector<HV3> yc(my.ne);
    std::vector<double> yr(my.ne);
    double rmax = 0.0;
    for (int64_t e = 0; e < my.ne; ++e) yc[e] = my.centroid(e), yr[e] = my.circumradius(e), rmax = std::max(rmax, yr[e]);
    const double cell = std::max(3.0 * rmax, 1e-300);
    auto key = [cell](const HV3& p) {
      return std::array<int64_t, 3>{(int64_t)std::floor(p.x / cell), (int64_t)std::floor(p.y / cell),
                                    (int64_t)std::floor(p.z / cell)};
    };
    std::map<std::array<int64_t, 3>, std::vector<int>> grid;
    for (int64_t e = 0; e < my.ne; ++e) grid[key(yc[e])].push_back((int)e);
    std::vector<int32_t> ppt, pey;
    for (int64_t i = 0; i < npts; ++i) {
      const HV3 xi{points[3 * i], points[3 * i + 1], points[3 * i + 2]};
      const auto k = key(xi);
      for (int64_t dx = -1; dx <= 1; ++dx)
        for (int64_t dy = -1; dy <= 1; ++dy)
          for (int64_t dz = -1; dz <= 1; ++dz) {
            const auto it = grid.find({k[0] + dx, k[1] + dy, k[2] + dz});
            if (it == grid.end()) continue;
            for (int e : it->second)
              if (hnrm(hsub(yc[e], xi)) <= 3.0 * std::max(0.0, yr[e])) {
                ppt.push_back((int32_t)i);
                pey.push_back(e);
              }
          }
    }
    N->npairs = (int64_t)ppt.size();
    my.check_pairs(pey);
    std::map<std::pair<int32_t, int32_t>, std::vector<int64_t>> ent;  // (col,row) -> contributions
    for (int64_t p = 0; p < N->npairs; ++p)
      for (int j = 0; j < N->ntr; ++j) {
        const int32_t c = N->fy == 0 ? pey[p] : trial->elements[3 * pey[p] + j];
        if (c >= trial->nfree) throw std::invalid_argument("regularize: dof out of range");
        ent[{c, ppt[p]}].push_back(p * kMaxLoc + j);
      }
    N->nentries = (int64_t)ent.size();
    std::vector<int64_t> start{0}, src;
    for (auto& [k, v] : ent) {
      N->h_col.push_back(k.first);
      N->h_row.push_back(k.second);
      src.insert(src.end(), v.begin(), v.end());
      start.push_back((int64_t)src.size());
    }
    N->pair_ex.upload(ppt);
    N->pair_ey.upload(pey);
    N->xv.upload(points, sizeof(double) * 3 * std::max<int64_t>(npts, 0));
    N->yv.upload(trial->vertices, sizeof(double) * 3 * trial->nv);
    N->ye.upload(trial->elements, sizeof(int32_t) * 3 * trial->ne);
    N->yq.upload(yq);
    N->local.alloc(sizeof(double) * kMaxLoc * std::max<int64_t>(1, N->npairs));
    N->leaves.alloc(sizeof(int32_t) * std::max<int64_t>(1, N->npairs));
    N->work.alloc(sizeof(unsigned long long));
    N->stats.alloc(sizeof(unsigned long long) * 9);
    N->ent_row.upload(N->h_row);
    N->ent_col.upload(N->h_col);
    N->ent_start.upload(start);
    N->ent_src.upload(src);
    N->vals.alloc(sizeof(double) * std::max<int64_t>(1, N->nentries));
    const std::vector<double> rby = host_rule(N->gy, false);
    double by[21] = {0};
    std::copy(rby.begin(), rby.end(), by);
    N->yrule.upload(by, sizeof(by));
    *out = N.release();
  });
}

gk_status gk_nearfield_get_info(const gk_nearfield* N, int64_t* pairs, int64_t* entries) {
  return guard([&] {
    if (!N) throw std::invalid_argument("gk_nearfield_get_info: null handle");
    if (pairs) *pairs = N->npairs;
    if (entries) *entries = N->nentries;
  });
}

gk_status gk_nearfield_compute(gk_nearfield* N, gk_stream stream) {
  return guard([&] {
    if (!N) throw std::invalid_argument("gk_nearfield_compute: null handle");
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    cuda_check(cudaMemsetAsync(N->work.p, 0, N->work.bytes, s), "memset");
    cuda_check(cudaMemsetAsync(N->stats.p, 0, N->stats.bytes, s), "memset");
    if (N->npairs > 0) {
      NfArgs a;
      a.npairs = N->npairs;
      a.pair_ex = N->pair_ex.as<int32_t>();
      a.pair_ey = N->pair_ey.as<int32_t>();
      a.xv = N->xv.as<double>();
      a.xe = N->xe.as<int32_t>();
      a.yv = N->yv.as<double>();
      a.ye = N->ye.as<int32_t>();
      a.xq = N->xq.as<double>();
      a.yq = N->yq.as<double>();
      a.xrule = N->xrule.as<double>();
      a.yrule = N->yrule.as<double>();
      a.gx = N->gx;
      a.gy = N->gy;
      a.eps = N->eps;
      a.local = N->local.as<double>();
      a.work = N->work.as<unsigned long long>();
      a.stats = N->stats.as<unsigned long long>();
      a.pair_leaves = N->leaves.as<int32_t>();
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      auto launch = [&](auto kern, size_t warp_smem) {
        const size_t smem = warp_smem * kNfWarps;
        cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * kNfWarps, smem);
        const int64_t want = (N->npairs + kNfWarps - 1) / kNfWarps;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * std::max(1, per_sm)));
        kern<<<grid, 32 * kNfWarps, smem, s>>>(a);
      };
      if (N->points) {
        const unsigned grid = (unsigned)((N->npairs + 127) / 128);
        if (N->ntr == 1)
          k_nf_points<1><<<grid, 128, 0, s>>>(a);
        else
          k_nf_points<3><<<grid, 128, 0, s>>>(a);
      } else if (N->nt == 1 && N->ntr == 1)
        launch(k_nearfield_b<1, 1>, sizeof(WarpSmemB<1>));
      else if (N->nt == 3 && N->ntr == 3)
        launch(k_nearfield_b<3, 3>, sizeof(WarpSmemB<9>));
      else if (N->nt == 1)
        launch(k_nearfield_b<1, 3>, sizeof(WarpSmemB<3>));
      else
        launch(k_nearfield_b<3, 1>, sizeof(WarpSmemB<3>));
      cuda_check(cudaGetLastError(), "k_nearfield launch");
    }
    if (N->nentries > 0) {
      k_nf_reduce<<<(unsigned)((N->nentries + 255) / 256), 256, 0, s>>>(
          N->nentries, N->ent_start.as<int64_t>(), N->ent_src.as<int64_t>(), N->local.as<double>(),
          N->vals.as<double>());
      cuda_check(cudaGetLastError(), "k_nf_reduce launch");
    }
    N->computed = true;
  });
}

gk_status gk_nearfield_apply(gk_nearfield* N, gk_cplx* A, int64_t lda, gk_stream stream) {
  return guard([&] {
    if (!N || !A) throw std::invalid_argument("gk_nearfield_apply: null argument");
    if (!N->computed) throw std::invalid_argument("gk_nearfield_apply: call gk_nearfield_compute first");
    if (N->nentries == 0) return;
    k_nf_apply<<<(unsigned)((N->nentries + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        N->nentries, N->ent_row.as<int32_t>(), N->ent_col.as<int32_t>(), N->vals.as<double>(),
        reinterpret_cast<double2*>(A), lda);
    cuda_check(cudaGetLastError(), "k_nf_apply launch");
  });
}

gk_status gk_nearfield_triplets(gk_nearfield* N, int32_t* rows, int32_t* cols, double* vals) {
  return guard([&] {
    if (!N) throw std::invalid_argument("gk_nearfield_triplets: null handle");
    if (!N->computed) throw std::invalid_argument("gk_nearfield_triplets: call gk_nearfield_compute first");
    unsigned long long flag = 0;
    cuda_check(cudaMemcpy(&flag, N->stats.as<unsigned long long>() + 8, sizeof(flag), cudaMemcpyDeviceToHost),
               "stats");
    if (flag) throw std::invalid_argument("analytic_triangle_integrals: degenerate triangle");
    if (N->nentries == 0) return;
    if (rows) std::copy(N->h_row.begin(), N->h_row.end(), rows);
    if (cols) std::copy(N->h_col.begin(), N->h_col.end(), cols);
    if (vals) cuda_check(cudaMemcpy(vals, N->vals.p, sizeof(double) * N->nentries, cudaMemcpyDeviceToHost), "vals");
  });
}

gk_status gk_diag_nearfield_pairs(const gk_nearfield* N, int32_t* ex, int32_t* ey, int32_t* leaves) {
  return guard([&] {
    if (!N) throw std::invalid_argument("gk_diag_nearfield_pairs: null handle");
    if (N->npairs == 0) return;
    if (ex) cuda_check(cudaMemcpy(ex, N->pair_ex.p, sizeof(int32_t) * N->npairs, cudaMemcpyDeviceToHost), "pairs");
    if (ey) cuda_check(cudaMemcpy(ey, N->pair_ey.p, sizeof(int32_t) * N->npairs, cudaMemcpyDeviceToHost), "pairs");
    if (leaves) {
      if (!N->computed || N->points) throw std::invalid_argument("gk_diag_nearfield_pairs: no adaptive pass computed");
      cuda_check(cudaMemcpy(leaves, N->leaves.p, sizeof(int32_t) * N->npairs, cudaMemcpyDeviceToHost), "leaves");
    }
  });
}

gk_status gk_nearfield_stats(const gk_nearfield* N, int64_t* calls, int64_t* hist) {
  return guard([&] {
    if (!N) throw std::invalid_argument("gk_nearfield_stats: null handle");
    unsigned long long s[9];
    cuda_check(cudaMemcpy(s, N->stats.p, sizeof(s), cudaMemcpyDeviceToHost), "stats");
    if (calls) *calls = (int64_t)s[0];
    if (hist) {
      for (int d = 0; d < 7; ++d) hist[d] = (int64_t)s[1 + d];
      hist[7] = 0;
    }
  });
}

gk_status gk_nearfield_destroy(gk_nearfield* N) {
  return guard([&] { delete N; });
}

}  // extern "C"
