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

#include <algorithm>

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
  // Coordinates relative to the CTA's first target, formed in fp64 and then
  // rounded to fp32: a near pair's difference carries the fp32 error of the
  // local offsets (~ the block's extent) instead of that of the absolute
  // coordinates (~ the scene); far pairs keep ~ulp(scene) in r, which only
  // moves their phase (K5).
  const long long tc = min((long long)blockIdx.x * kGThreads * 2, (long long)a.nt - 1);
  const double cx = a.tx[tc], cy = a.ty[tc], cz = a.tz[tc];
  const float x0 = v0 ? (float)(a.tx[t0] - cx) : 0.f, y0 = v0 ? (float)(a.ty[t0] - cy) : 0.f,
              z0 = v0 ? (float)(a.tz[t0] - cz) : 0.f;
  const float x1 = v1 ? (float)(a.tx[t0 + 1] - cx) : 0.f, y1 = v1 ? (float)(a.ty[t0 + 1] - cy) : 0.f,
              z1 = v1 ? (float)(a.tz[t0 + 1] - cz) : 0.f;
  double R0 = 0.0, I0 = 0.0, R1 = 0.0, I1 = 0.0;
  const float eps2 = a.eps2f, kappa = a.kappaf;
  for (long long b = 0; b < a.ns; b += kGTile) {
    const int n = (int)min((long long)kGTile, a.ns - b);
    __syncthreads();
    for (int s = threadIdx.x; s < n; s += kGThreads) {
      sx[s] = (float)(a.sx[b + s] - cx);
      sy[s] = (float)(a.sy[b + s] - cy);
      sz[s] = (float)(a.sz[b + s] - cz);
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
// ---- symmetric fp64 matvec (targets == sources): each unordered block pair
// once.  G is symmetric, so tile (I, J), J > I, yields both the row sums
// y_I += G_IJ q_J and the column sums y_J += G_IJ^T q_I from one set of pair
// evaluations.  Inside a warp the column accumulators rotate through the
// lanes (one shuffle per pair and component pair): lane l evaluates its two
// targets against source (l + j) mod 32 at step j and passes the running
// column sum to lane l - 1, so after 32 steps every lane holds the complete
// warp sum for one source — no atomics, fixed order.  Tiles write row and
// column partials; a second kernel adds them into y in a fixed order.
constexpr int kSB = 256;  // locations per symmetric block (4 warps x 64 targets)

__device__ __forceinline__ void tile_of(int tile, int I0, int nb, int& I, int& J) {
  int off = 0;
  I = I0;
  while (off + (nb - I) <= tile) {
    off += nb - I;
    ++I;
  }
  J = I + (tile - off);
}

template <bool HELM>
__global__ void __launch_bounds__(128) k_green64_sym(const GreenArgs a, const double2* __restrict__ Q, int I0,
                                                    int nb, double2* __restrict__ R, double2* __restrict__ C) {
  __shared__ double sx[kSB], sy[kSB], sz[kSB];
  __shared__ double2 sq[kSB];
  __shared__ double2 colp[4][32];
  int I, J;
  tile_of(blockIdx.x, I0, nb, I, J);
  const long long U = a.nt;
  for (int e = threadIdx.x; e < kSB; e += 128) {
    const long long v = (long long)J * kSB + e;
    const bool ok = v < U;
    // padding (last block only): zero charge at a distant point; kr stays far
    // inside the quarter-turn reduction's range so every product is finite and
    // the zero charges contribute exactly 0 to real rows and columns
    sx[e] = ok ? a.tx[v] : 1e6;
    sy[e] = ok ? a.ty[v] : 0.0;
    sz[e] = ok ? a.tz[v] : 0.0;
    sq[e] = ok ? Q[v] : make_double2(0.0, 0.0);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double tx[2], ty[2], tz[2];
  double2 tq[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const long long v = (long long)I * kSB + w * 64 + 32 * k + lane;
    const bool ok = v < U;
    tx[k] = ok ? a.tx[v] : -1e6;
    ty[k] = ok ? a.ty[v] : 0.0;
    tz[k] = ok ? a.tz[v] : 0.0;
    tq[k] = ok ? Q[v] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  const double eps2 = a.eps2, kappa = a.kappa;
  double ra[2] = {0.0, 0.0}, ia[2] = {0.0, 0.0};
  const int src_lane = (lane + 1) & 31;
  for (int c = 0; c < kSB / 32; ++c) {
    double cr = 0.0, ci = 0.0;  // column sum of source c*32 + ((lane + j) & 31) at step j
    for (int j = 0; j < 32; j += 2) {
      // steps j and j+1 evaluated in lockstep (2 targets x 2 sources)
      int sidx[2];
      double dx[4], dy[4], dz[4];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        sidx[u] = c * 32 + ((lane + j + u) & 31);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          dx[2 * u + k] = tx[k] - sx[sidx[u]];
          dy[2 * u + k] = ty[k] - sy[sidx[u]];
          dz[2 * u + k] = tz[k] - sz[sidx[u]];
        }
      }
      double cs[4], sn[4], rinv[4];
      green_parts_n<HELM, 4, true>(dx, dy, dz, eps2, kappa, cs, sn, rinv);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const double2 q = sq[sidx[u]];
        double pr = 0.0, pi = 0.0;  // this step's column contribution (both targets)
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const double g = rinv[2 * u + k];
          if (HELM) {
            // G = (cs + i sn) / r formed once (two DMUL) and shared by the row
            // (G q_s) and column (G q_t) accumulations
            const double gr = cs[2 * u + k] * g, gi = sn[2 * u + k] * g;
            ra[k] = fma(gr, q.x, fma(-gi, q.y, ra[k]));
            ia[k] = fma(gr, q.y, fma(gi, q.x, ia[k]));
            pr = fma(gr, tq[k].x, fma(-gi, tq[k].y, pr));
            pi = fma(gr, tq[k].y, fma(gi, tq[k].x, pi));
          } else {
            ra[k] = fma(g, q.x, ra[k]);
            ia[k] = fma(g, q.y, ia[k]);
            pr = fma(g, tq[k].x, pr);
            pi = fma(g, tq[k].y, pi);
          }
        }
        cr += pr;
        ci += pi;
        cr = __shfl_sync(0xffffffffu, cr, src_lane);
        ci = __shfl_sync(0xffffffffu, ci, src_lane);
      }
    }
    // lane l now holds the warp's column sum of source c*32 + l
    colp[w][lane] = make_double2(cr, ci);
    __syncthreads();
    if (w == 0) {
      const double2 s0 = colp[0][lane], s1 = colp[1][lane], s2 = colp[2][lane], s3 = colp[3][lane];
      C[(long long)blockIdx.x * kSB + c * 32 + lane] =
          make_double2(((s0.x + s1.x) + s2.x) + s3.x, ((s0.y + s1.y) + s2.y) + s3.y);
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) R[(long long)blockIdx.x * kSB + w * 64 + 32 * k + lane] = make_double2(ra[k], ia[k]);
}

// fp32 variant of the symmetric tile: fp32 pair math and fp32 sums inside the
// tile (256 sources per row sum, 64 targets per rotating column sum), written
// as fp64 partials and added across tiles in fp64 by k_green_sym_reduce.
template <bool HELM>
__global__ void __launch_bounds__(128) k_green32_sym(const GreenArgs a, const double2* __restrict__ Q, int I0,
                                                    int nb, double2* __restrict__ R, double2* __restrict__ C) {
  __shared__ float sx[kSB], sy[kSB], sz[kSB];
  __shared__ float2 sq[kSB];
  __shared__ float2 colp[4][32];
  int I, J;
  tile_of(blockIdx.x, I0, nb, I, J);
  const long long U = a.nt;
  // coordinates relative to block I's first location (see k_green32)
  const long long tc = (long long)I * kSB;
  const double cx = a.tx[tc], cy = a.ty[tc], cz = a.tz[tc];
  for (int e = threadIdx.x; e < kSB; e += 128) {
    const long long v = (long long)J * kSB + e;
    const bool ok = v < U;
    sx[e] = ok ? (float)(a.tx[v] - cx) : 1e6f;  // padding as in the fp64 tile
    sy[e] = ok ? (float)(a.ty[v] - cy) : 0.f;
    sz[e] = ok ? (float)(a.tz[v] - cz) : 0.f;
    const double2 qq = ok ? Q[v] : make_double2(0.0, 0.0);
    sq[e] = make_float2((float)qq.x, (float)qq.y);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float tx[2], ty[2], tz[2];
  float2 tq[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const long long v = (long long)I * kSB + w * 64 + 32 * k + lane;
    const bool ok = v < U;
    tx[k] = ok ? (float)(a.tx[v] - cx) : -1e6f;
    ty[k] = ok ? (float)(a.ty[v] - cy) : 0.f;
    tz[k] = ok ? (float)(a.tz[v] - cz) : 0.f;
    const double2 qq = ok ? Q[v] : make_double2(0.0, 0.0);
    tq[k] = make_float2((float)qq.x, (float)qq.y);
  }
  __syncthreads();
  const float eps2 = a.eps2f, kappa = a.kappaf;
  float ra[2] = {0.f, 0.f}, ia[2] = {0.f, 0.f};
  const int src_lane = (lane + 1) & 31;
  for (int c = 0; c < kSB / 32; ++c) {
    float cr = 0.f, ci = 0.f;
    for (int j = 0; j < 32; j += 2) {
      float2 g[4];
      int sidx[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        sidx[u] = c * 32 + ((lane + j + u) & 31);
#pragma unroll
        for (int k = 0; k < 2; ++k)
          g[2 * u + k] = green_f<HELM>(tx[k] - sx[sidx[u]], ty[k] - sy[sidx[u]], tz[k] - sz[sidx[u]], eps2, kappa);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const float2 q = sq[sidx[u]];
        float pr = 0.f, pi = 0.f;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const float2 gg = g[2 * u + k];
          ra[k] = fmaf(gg.x, q.x, fmaf(-gg.y, q.y, ra[k]));
          ia[k] = fmaf(gg.x, q.y, fmaf(gg.y, q.x, ia[k]));
          pr = fmaf(gg.x, tq[k].x, fmaf(-gg.y, tq[k].y, pr));
          pi = fmaf(gg.x, tq[k].y, fmaf(gg.y, tq[k].x, pi));
        }
        cr += pr;
        ci += pi;
        cr = __shfl_sync(0xffffffffu, cr, src_lane);
        ci = __shfl_sync(0xffffffffu, ci, src_lane);
      }
    }
    colp[w][lane] = make_float2(cr, ci);
    __syncthreads();
    if (w == 0) {
      const float2 s0 = colp[0][lane], s1 = colp[1][lane], s2 = colp[2][lane], s3 = colp[3][lane];
      C[(long long)blockIdx.x * kSB + c * 32 + lane] =
          make_double2(((double)s0.x + s1.x) + s2.x + s3.x, ((double)s0.y + s1.y) + s2.y + s3.y);
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) R[(long long)blockIdx.x * kSB + w * 64 + 32 * k + lane] = make_double2(ra[k], ia[k]);
}

// y[v] += sum_{J >= I} R(I, J)[e]  (rows of the group)  +  sum_{I < J} C(I, J)[e]
// (columns from the group's rows), v = J*kSB + e; fixed order.
__global__ void k_green_sym_reduce(const double2* __restrict__ R, const double2* __restrict__ C, int I0, int I1,
                                   int nb, long long U, double2* __restrict__ Y, int first) {
  const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= U) return;
  const int b = (int)(v / kSB), e = (int)(v - (long long)b * kSB);
  double re = first ? 0.0 : Y[v].x, im = first ? 0.0 : Y[v].y;
  int off = 0;  // tile index of (I, I) within the group
  for (int I = I0; I < I1; ++I) {
    if (I == b) {
      for (int J = I; J < nb; ++J) {
        const double2 r = R[(long long)(off + J - I) * kSB + e];
        re += r.x;
        im += r.y;
      }
    } else if (I < b) {
      const double2 c = C[(long long)(off + b - I) * kSB + e];
      re += c.x;
      im += c.y;
    }
    off += nb - I;
  }
  Y[v] = make_double2(re, im);
}

}  // namespace

int green_sym_block() { return kSB; }

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
    if (a.sym_R) {
      const int nb = (int)((a.nt + kSB - 1) / kSB);
      const int G = a.sym_group;
      for (int I0 = 0; I0 < nb; I0 += G) {
        const int I1 = std::min(nb, I0 + G);
        const long long tiles = (long long)(I1 - I0) * nb - ((long long)I1 * (I1 - 1) / 2 - (long long)I0 * (I0 - 1) / 2);
        double2* Rb = static_cast<double2*>(a.sym_R);
        double2* Cb = static_cast<double2*>(a.sym_C);
        if (precision == GK_FP32) {
          if (helmholtz)
            k_green32_sym<true><<<(unsigned)tiles, 128, 0, s>>>(a, Qc, I0, nb, Rb, Cb);
          else
            k_green32_sym<false><<<(unsigned)tiles, 128, 0, s>>>(a, Qc, I0, nb, Rb, Cb);
        } else {
          if (helmholtz)
            k_green64_sym<true><<<(unsigned)tiles, 128, 0, s>>>(a, Qc, I0, nb, Rb, Cb);
          else
            k_green64_sym<false><<<(unsigned)tiles, 128, 0, s>>>(a, Qc, I0, nb, Rb, Cb);
        }
        k_green_sym_reduce<<<(unsigned)((a.nt + 255) / 256), 256, 0, s>>>(Rb, Cb, I0, I1, nb, a.nt, Yc, I0 == 0);
      }
    } else if (precision == GK_FP32) {
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
