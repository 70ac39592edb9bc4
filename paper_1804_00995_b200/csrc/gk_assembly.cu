// K1+K2: fused pair kernel + basis/quadrature contraction + scatter-to-DOF.
//
// Replaces, for one tile of the matrix, the x-chunk loop of bem_product
// (assembly.cpp:212-220): Kernel::evaluate_blocks (kernels.cpp:76-131), the
// y-side product kr = G (W_y Psi) (assembly.cpp:217) and the x-side update
// A += (W_x Phi)^T kr (assembly.cpp:218).
//
// Tile = (x block I, y block J).  Thread t owns x location u_t of the block
// (twins merged, <= 128 per block).  All threads walk the same list of y
// records (warp-uniform loads), evaluate G(u_t, v) once per unique location
// pair, and accumulate coef * G into H[slot][u_t] in shared memory — the
// y-side contraction, owner-computes per thread column, no atomics.  After a
// barrier each thread gathers whole entries A_ij = sum_u c_ui H[j][u] (the
// x-side contraction in a fixed order) and writes them; with identical sides
// only the upper triangle of tiles is computed and mirrored (G symmetric).
#include <cuda_runtime.h>

#include "gk_internal.hpp"
#include "gk_math.cuh"

namespace gk {

namespace {

__device__ __forceinline__ YRec load_rec(const YRec* p) {
  YRec r;
  const double2 a = __ldg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  const double2 c = __ldg(reinterpret_cast<const double2*>(p) + 2);
  r.x = a.x;
  r.y = a.y;
  r.z = b.x;
  r.c0 = b.y;
  r.c1 = c.x;
  const long long s = __double_as_longlong(c.y);
  r.s0 = (int32_t)(s & 0xffffffffll);
  r.s1 = (int32_t)(s >> 32);
  return r;
}

__device__ __forceinline__ void acc(double2* h, double c, const c64& g) {
  double2 v = *h;
  v.x = fma(c, g.re, v.x);
  v.y = fma(c, g.im, v.y);
  *h = v;
}

template <bool HELM>
__global__ void __launch_bounds__(kAsmThreads, 2) k_assemble(const AsmArgs a) {
  extern __shared__ double2 H[];  // [kJCap][kUCap]
  const int tile = blockIdx.x;
  const int bi = a.tile_i[tile], bj = a.tile_j[tile];
  const int t = threadIdx.x;
  const int i0 = a.xb_dof_start[bi], nI = a.xb_dof_start[bi + 1] - i0;
  const int j0 = a.yb_dof_start[bj], nJ = a.yb_dof_start[bj + 1] - j0;
  const int l0 = a.xb_loc_start[bi], nu = a.xb_loc_start[bi + 1] - l0;

  for (int e = t; e < nJ * kUCap; e += kAsmThreads) H[e] = make_double2(0.0, 0.0);
  double ux = 0.0, uy = 0.0, uz = 0.0;
  if (t < nu) {
    ux = a.xl_x[l0 + t];
    uy = a.xl_y[l0 + t];
    uz = a.xl_z[l0 + t];
  }
  __syncthreads();

  const double eps2 = a.eps2, kappa = a.kappa;
  const YRec* rec = a.yrec + a.yb_rec_start[bj];
  const int nrec = a.yb_rec_start[bj + 1] - a.yb_rec_start[bj];
  double2* Hc = H + t;
  int r = 0;
  for (; r + 1 < nrec; r += 2) {  // two independent pair evaluations in flight
    const YRec p = load_rec(rec + r);
    const YRec q = load_rec(rec + r + 1);
    const c64 gp = green<HELM>(ux - p.x, uy - p.y, uz - p.z, eps2, kappa);
    const c64 gq = green<HELM>(ux - q.x, uy - q.y, uz - q.z, eps2, kappa);
    acc(Hc + p.s0 * kUCap, p.c0, gp);
    if (p.s1 >= 0) acc(Hc + p.s1 * kUCap, p.c1, gp);
    acc(Hc + q.s0 * kUCap, q.c0, gq);
    if (q.s1 >= 0) acc(Hc + q.s1 * kUCap, q.c1, gq);
  }
  if (r < nrec) {
    const YRec p = load_rec(rec + r);
    const c64 gp = green<HELM>(ux - p.x, uy - p.y, uz - p.z, eps2, kappa);
    acc(Hc + p.s0 * kUCap, p.c0, gp);
    if (p.s1 >= 0) acc(Hc + p.s1 * kUCap, p.c1, gp);
  }
  __syncthreads();

  // x-side contraction + write (lanes along rows: coalesced columns)
  double2* A = reinterpret_cast<double2*>(a.A);
  const long long lda = a.lda;
  for (int e = t; e < nI * nJ; e += kAsmThreads) {
    const int ii = e % nI, jj = e / nI;
    const int pi = i0 + ii, pj = j0 + jj;
    if (a.symmetric && pi > pj) continue;
    double re = 0.0, im = 0.0;
    const double2* Hr = H + jj * kUCap;
    for (int s = a.xsup_start[pi]; s < a.xsup_start[pi + 1]; ++s) {
      const double2 h = Hr[a.xsup_u[s]];
      const double c = a.xsup_c[s];
      re = fma(c, h.x, re);
      im = fma(c, h.y, im);
    }
    const long long oi = a.xperm[pi], oj = a.yperm[pj];
    const double2 v = make_double2(re, im);
    A[oi + oj * lda] = v;
    if (a.symmetric && pi != pj) A[oj + oi * lda] = v;
  }
}

}  // namespace

void launch_assemble(const AsmArgs& a, int64_t ntiles, bool helmholtz, void* stream) {
  if (ntiles <= 0) return;
  const size_t smem = sizeof(double2) * kJCap * kUCap;
  static bool configured = false;
  if (!configured) {
    cuda_check(cudaFuncSetAttribute(k_assemble<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
               "cudaFuncSetAttribute");
    cuda_check(cudaFuncSetAttribute(k_assemble<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
               "cudaFuncSetAttribute");
    configured = true;
  }
  if (ntiles > INT32_MAX) throw std::invalid_argument("bem_dense: too many tiles");
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (helmholtz)
    k_assemble<true><<<(unsigned)ntiles, kAsmThreads, smem, s>>>(a);
  else
    k_assemble<false><<<(unsigned)ntiles, kAsmThreads, smem, s>>>(a);
  cuda_check(cudaGetLastError(), "k_assemble launch");
}

}  // namespace gk
