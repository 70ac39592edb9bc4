// K5: matrix-free Green-kernel matvec  y_i = sum_j [r_ij > eps] G(x_i, y_j) q_j.
//
// Semantics are Kernel::evaluate_blocks with mask=true (kernels.cpp:76-131)
// contracted with a weighted charge vector, i.e. bem_product with a point
// side (assembly.cpp:173-222).  "Self-interaction excluded" is the distance
// mask, which also drops the bit-identical twin of every edge-midpoint point.
//
// Twins are merged on both sides by the plan: charges of co-located sources
// are summed (fixed CSR order) and each unique target is evaluated once, then
// copied to all its original points.  Sources are staged through shared
// memory in tiles; every thread owns two targets (ILP, and each broadcast
// shared-memory read serves two pairs).  fp32 variant: fp32 pair math with a
// per-tile fp32 partial sum folded into an fp64 accumulator.
#include <cuda_runtime.h>

#include "gk_internal.hpp"
#include "gk_math.cuh"

namespace gk {

namespace {
constexpr int kGThreads = 128;
constexpr int kGTile = 256;

__global__ void k_merge_charges(const double2* __restrict__ q, const int64_t* __restrict__ start,
                                const int64_t* __restrict__ list, long long ns, double2* __restrict__ Q) {
  const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= ns) return;
  double re = 0.0, im = 0.0;
  for (int64_t p = start[v]; p < start[v + 1]; ++p) {
    const double2 c = q[list[p]];
    re += c.x;
    im += c.y;
  }
  Q[v] = make_double2(re, im);
}

__global__ void k_scatter_targets(const double2* __restrict__ Y, const int64_t* __restrict__ loc,
                                  long long n, double2* __restrict__ y) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = Y[loc[i]];
}

template <bool HELM>
__global__ void __launch_bounds__(kGThreads) k_green64(const GreenArgs a, const double2* __restrict__ Q,
                                                      double2* __restrict__ Y) {
  __shared__ double sx[kGTile], sy[kGTile], sz[kGTile];
  __shared__ double2 sq[kGTile];
  const long long t0 = ((long long)blockIdx.x * kGThreads + threadIdx.x) * 2;
  const bool v0 = t0 < a.nt, v1 = t0 + 1 < a.nt;
  const double x0 = v0 ? a.tx[t0] : 0.0, y0 = v0 ? a.ty[t0] : 0.0, z0 = v0 ? a.tz[t0] : 0.0;
  const double x1 = v1 ? a.tx[t0 + 1] : 0.0, y1 = v1 ? a.ty[t0 + 1] : 0.0, z1 = v1 ? a.tz[t0 + 1] : 0.0;
  double r0 = 0.0, i0 = 0.0, r1 = 0.0, i1 = 0.0;
  const double eps2 = a.eps2, kappa = a.kappa;
  for (long long b = 0; b < a.ns; b += kGTile) {
    const int n = (int)min((long long)kGTile, a.ns - b);
    __syncthreads();
    for (int s = threadIdx.x; s < n; s += kGThreads) {
      sx[s] = a.sx[b + s];
      sy[s] = a.sy[b + s];
      sz[s] = a.sz[b + s];
      sq[s] = Q[b + s];
    }
    __syncthreads();
    // two targets x two sources per step: four independent pair evaluations in
    // lockstep (green_parts_n), each folded as (cs + i sn) * (q / r) — the
    // charge times 1/r is formed once (two DMUL) and the complex product
    // accumulates with four DFMA; sources stay in ascending order per target
    double ra[2] = {r0, r1}, ia[2] = {i0, i1};
    const double tx[2] = {x0, x1}, ty[2] = {y0, y1}, tz[2] = {z0, z1};
    auto fold = [&](int k, double cs, double sn, double rinv, double2 q) {
      const double wr = q.x * rinv, wi = q.y * rinv;
      ra[k] = fma(cs, wr, fma(-sn, wi, ra[k]));
      ia[k] = fma(cs, wi, fma(sn, wr, ia[k]));
    };
    int s = 0;
    for (; s + 2 <= n; s += 2) {
      double dx[4], dy[4], dz[4];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          dx[2 * u + k] = tx[k] - sx[s + u];
          dy[2 * u + k] = ty[k] - sy[s + u];
          dz[2 * u + k] = tz[k] - sz[s + u];
        }
      double cs[4], sn[4], rinv[4];
      green_parts_n<HELM, 4, true>(dx, dy, dz, eps2, kappa, cs, sn, rinv);
      const double2 q0 = sq[s], q1 = sq[s + 1];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (HELM) {
          fold(k, cs[k], sn[k], rinv[k], q0);
          fold(k, cs[2 + k], sn[2 + k], rinv[2 + k], q1);
        } else {
          ra[k] = fma(rinv[k], q0.x, ra[k]);
          ia[k] = fma(rinv[k], q0.y, ia[k]);
          ra[k] = fma(rinv[2 + k], q1.x, ra[k]);
          ia[k] = fma(rinv[2 + k], q1.y, ia[k]);
        }
      }
    }
    for (; s < n; ++s) {
      double dx[2], dy[2], dz[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        dx[k] = tx[k] - sx[s];
        dy[k] = ty[k] - sy[s];
        dz[k] = tz[k] - sz[s];
      }
      double cs[2], sn[2], rinv[2];
      green_parts_n<HELM, 2, true>(dx, dy, dz, eps2, kappa, cs, sn, rinv);
      const double2 q = sq[s];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (HELM) {
          fold(k, cs[k], sn[k], rinv[k], q);
        } else {
          ra[k] = fma(rinv[k], q.x, ra[k]);
          ia[k] = fma(rinv[k], q.y, ia[k]);
        }
      }
    }
    r0 = ra[0];
    r1 = ra[1];
    i0 = ia[0];
    i1 = ia[1];
  }
  if (v0) Y[t0] = make_double2(r0, i0);
  if (v1) Y[t0 + 1] = make_double2(r1, i1);
}

template <bool HELM>
__device__ __forceinline__ float2 green_f(float dx, float dy, float dz, float eps2, float kappa) {
  const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
  const float rinv = rsqrtf(r2);
  float2 g;
  if (HELM) {
    const float r = r2 * rinv;
    float s, c;
    sincos_quarter_f(r * kappa, s, c);
    g.x = c * rinv;
    g.y = s * rinv;
  } else {
    g.x = rinv;
    g.y = 0.0f;
  }
  if (!(r2 > eps2)) g = make_float2(0.0f, 0.0f);
  return g;
}

template <bool HELM>
__global__ void __launch_bounds__(kGThreads) k_green32(const GreenArgs a, const double2* __restrict__ Q,
                                                      double2* __restrict__ Y) {
  __shared__ float sx[kGTile], sy[kGTile], sz[kGTile];
  __shared__ float2 sq[kGTile];
  const long long t0 = ((long long)blockIdx.x * kGThreads + threadIdx.x) * 2;
  const bool v0 = t0 < a.nt, v1 = t0 + 1 < a.nt;
  // target-relative source coordinates keep fp32 differences accurate
  const float x0 = v0 ? a.txf[t0] : 0.f, y0 = v0 ? a.tyf[t0] : 0.f, z0 = v0 ? a.tzf[t0] : 0.f;
  const float x1 = v1 ? a.txf[t0 + 1] : 0.f, y1 = v1 ? a.tyf[t0 + 1] : 0.f, z1 = v1 ? a.tzf[t0 + 1] : 0.f;
  double R0 = 0.0, I0 = 0.0, R1 = 0.0, I1 = 0.0;
  const float eps2 = a.eps2f, kappa = a.kappaf;
  for (long long b = 0; b < a.ns; b += kGTile) {
    const int n = (int)min((long long)kGTile, a.ns - b);
    __syncthreads();
    for (int s = threadIdx.x; s < n; s += kGThreads) {
      sx[s] = a.sxf[b + s];
      sy[s] = a.syf[b + s];
      sz[s] = a.szf[b + s];
      const double2 q = Q[b + s];
      sq[s] = make_float2((float)q.x, (float)q.y);
    }
    __syncthreads();
    float r0 = 0.f, i0 = 0.f, r1 = 0.f, i1 = 0.f;
    for (int s = 0; s < n; ++s) {
      const float px = sx[s], py = sy[s], pz = sz[s];
      const float2 q = sq[s];
      const float2 g0 = green_f<HELM>(x0 - px, y0 - py, z0 - pz, eps2, kappa);
      const float2 g1 = green_f<HELM>(x1 - px, y1 - py, z1 - pz, eps2, kappa);
      r0 = fmaf(g0.x, q.x, r0);
      r0 = fmaf(-g0.y, q.y, r0);
      i0 = fmaf(g0.x, q.y, i0);
      i0 = fmaf(g0.y, q.x, i0);
      r1 = fmaf(g1.x, q.x, r1);
      r1 = fmaf(-g1.y, q.y, r1);
      i1 = fmaf(g1.x, q.y, i1);
      i1 = fmaf(g1.y, q.x, i1);
    }
    R0 += r0;
    I0 += i0;
    R1 += r1;
    I1 += i1;
  }
  if (v0) Y[t0] = make_double2(R0, I0);
  if (v1) Y[t0 + 1] = make_double2(R1, I1);
}
}  // namespace

void launch_green(const GreenArgs& a, const void* q, void* Q, void* Yu, void* y, int precision, bool helmholtz,
                  void* stream) {
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (a.ntgt_orig <= 0) return;
  if (a.ns > 0) {
    k_merge_charges<<<(unsigned)((a.ns + 255) / 256), 256, 0, s>>>(
        static_cast<const double2*>(q), a.src_start, a.src_list, a.ns, static_cast<double2*>(Q));
    cuda_check(cudaGetLastError(), "k_merge_charges launch");
  }
  const unsigned grid = (unsigned)((a.nt + 2 * kGThreads - 1) / (2 * kGThreads));
  if (grid > 0) {
    const double2* Qc = static_cast<const double2*>(Q);
    double2* Yc = static_cast<double2*>(Yu);
    if (precision == GK_FP32) {
      if (helmholtz)
        k_green32<true><<<grid, kGThreads, 0, s>>>(a, Qc, Yc);
      else
        k_green32<false><<<grid, kGThreads, 0, s>>>(a, Qc, Yc);
    } else {
      if (helmholtz)
        k_green64<true><<<grid, kGThreads, 0, s>>>(a, Qc, Yc);
      else
        k_green64<false><<<grid, kGThreads, 0, s>>>(a, Qc, Yc);
    }
    cuda_check(cudaGetLastError(), "k_green launch");
  }
  k_scatter_targets<<<(unsigned)((a.ntgt_orig + 255) / 256), 256, 0, s>>>(
      static_cast<const double2*>(Yu), a.tgt_loc, a.ntgt_orig, static_cast<double2*>(y));
  cuda_check(cudaGetLastError(), "k_scatter_targets launch");
}

}  // namespace gk
