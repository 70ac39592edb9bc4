// K1+K2: fused pair kernel + basis/quadrature contraction + scatter-to-DOF.
//
// Replaces, for one tile of the matrix, the x-chunk loop of bem_product
// (assembly.cpp:212-220): Kernel::evaluate_blocks (kernels.cpp:76-131), the
// y-side product kr = G (W_y Psi) (assembly.cpp:217) and the x-side update
// A += (W_x Phi)^T kr (assembly.cpp:218).
//
// Tile = (x block I, y block J).  Thread t owns x location u_t of the block
// (twins merged, <= 128 per block).  The block's y records (unique y
// locations with their <= 2 (slot, coef) pairs, sorted by first slot) and the
// x support lists are staged in shared memory.  All threads walk the same
// record list (broadcast reads), evaluate G(u_t, v) once per unique location
// pair, keep a run accumulator for the current first slot in registers and
// add the second slot into H[slot][u_t] — the y-side contraction,
// owner-computes per thread column, no atomics.  After a barrier each thread
// gathers whole entries A_ij = sum_u c_ui H[j][u] (x-side contraction, fixed
// order) and writes them; with identical sides only tiles on or above the
// diagonal are computed and mirrored (G is symmetric).
#include <cuda_runtime.h>

#include "gk_internal.hpp"
#include "gk_math.cuh"

namespace gk {

namespace {

struct AsmSmem {
  double2 H[kJCap * kUCap];
  YRec rec[kRCap];
  double xs_c[kXsCap];
  int32_t xs_u[kXsCap];
  int32_t xs_start[kIMax + 1];
  int32_t orow[kIMax];  // original row index of each tile row
  int32_t ocol[kJCap];  // original column index of each tile column
};

__device__ __forceinline__ void rmw(char* Hb, int off, double c, double gr, double gi) {
  double2* h = reinterpret_cast<double2*>(Hb + off);
  double2 v = *h;
  v.x = fma(c, gr, v.x);
  v.y = fma(c, gi, v.y);
  *h = v;
}

template <bool HELM>
__global__ void __launch_bounds__(kAsmThreads, 2) k_assemble(const AsmArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  AsmSmem& S = *reinterpret_cast<AsmSmem*>(smem_raw);
  const int tile = blockIdx.x;
  const int bi = a.tile_i[tile], bj = a.tile_j[tile];
  const int t = threadIdx.x;
  const int i0 = a.xb_dof_start[bi], nI = a.xb_dof_start[bi + 1] - i0;
  const int j0 = a.yb_dof_start[bj], nJ = a.yb_dof_start[bj + 1] - j0;
  const int l0 = a.xb_loc_start[bi], nu = a.xb_loc_start[bi + 1] - l0;
  const int r0 = a.yb_rec_start[bj], nrec = a.yb_rec_start[bj + 1] - r0;
  const int xs0 = a.xsup_start[i0], nxs = a.xsup_start[i0 + nI] - xs0;

  // stage: zero H rows, copy records and x support lists
  for (int e = t; e < nJ * kUCap; e += kAsmThreads) S.H[e] = make_double2(0.0, 0.0);
  {
    const double2* src = reinterpret_cast<const double2*>(a.yrec + r0);
    double2* dst = reinterpret_cast<double2*>(S.rec);
    for (int e = t; e < nrec * 3; e += kAsmThreads) dst[e] = __ldg(src + e);
  }
  for (int e = t; e < nxs; e += kAsmThreads) {
    S.xs_c[e] = __ldg(a.xsup_c + xs0 + e);
    S.xs_u[e] = __ldg(a.xsup_u + xs0 + e);
  }
  for (int e = t; e <= nI; e += kAsmThreads) S.xs_start[e] = __ldg(a.xsup_start + i0 + e) - xs0;
  for (int e = t; e < nI; e += kAsmThreads) S.orow[e] = __ldg(a.xperm + i0 + e);
  for (int e = t; e < nJ; e += kAsmThreads) S.ocol[e] = __ldg(a.yperm + j0 + e);
  double ux = 0.0, uy = 0.0, uz = 0.0;
  if (t < nu) {
    ux = __ldg(a.xl_x + l0 + t);
    uy = __ldg(a.xl_y + l0 + t);
    uz = __ldg(a.xl_z + l0 + t);
  } else {
    ux = 1e100;  // idle columns: far away, finite, never gathered
  }
  __syncthreads();

  const double eps2 = a.eps2, kappa = a.kappa;
  char* Hb = reinterpret_cast<char*>(S.H) + t * 16;
  int cur = -1;  // byte offset of the run's slot row
  double ar = 0.0, ai = 0.0;
  // fold one evaluated pair into the run accumulator / second slot (uniform branches)
  auto fold = [&](const YRec& p, const c64& g) {
    if (p.off0 != cur) {
      if (cur >= 0) rmw(Hb, cur, 1.0, ar, ai);
      cur = p.off0;
      ar = 0.0;
      ai = 0.0;
    }
    ar = fma(p.c0, g.re, ar);
    ai = fma(p.c0, g.im, ai);
    if (p.off1 >= 0) rmw(Hb, p.off1, p.c1, g.re, g.im);
  };
  constexpr int kUnroll = 4;  // independent pair evaluations in flight per thread
  int r = 0;
  for (; r + kUnroll <= nrec; r += kUnroll) {
    double dx[kUnroll], dy[kUnroll], dz[kUnroll];
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) {
      const double2 a0 = *reinterpret_cast<const double2*>(&S.rec[r + k].x);
      const double2 a1 = *reinterpret_cast<const double2*>(&S.rec[r + k].z);
      dx[k] = ux - a0.x;
      dy[k] = uy - a0.y;
      dz[k] = uz - a1.x;
    }
    c64 g[kUnroll];
    green_n<HELM, kUnroll>(dx, dy, dz, eps2, kappa, g);
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) fold(S.rec[r + k], g[k]);
  }
  for (; r < nrec; ++r) {
    const YRec& p = S.rec[r];
    fold(p, green<HELM>(ux - p.x, uy - p.y, uz - p.z, eps2, kappa));
  }
  if (cur >= 0) rmw(Hb, cur, 1.0, ar, ai);
  __syncthreads();

  // x-side contraction + write (lanes along rows: coalesced columns for P0)
  double2* A = reinterpret_cast<double2*>(a.A);
  const long long lda = a.lda;
  const int total = nI * nJ;
  int ii = t % nI, jj = t / nI;
  const int di = kAsmThreads % nI, dj = kAsmThreads / nI;
  for (int e = t; e < total; e += kAsmThreads) {
    const int pi = i0 + ii, pj = j0 + jj;
    if (!(a.symmetric && pi > pj)) {
      double re = 0.0, im = 0.0;
      const double2* Hr = S.H + jj * kUCap;
      for (int s = S.xs_start[ii]; s < S.xs_start[ii + 1]; ++s) {
        const double2 h = Hr[S.xs_u[s]];
        const double c = S.xs_c[s];
        re = fma(c, h.x, re);
        im = fma(c, h.y, im);
      }
      const long long oi = S.orow[ii], oj = S.ocol[jj];
      const double2 v = make_double2(re, im);
      A[oi + oj * lda] = v;
      if (a.symmetric && pi != pj) A[oj + oi * lda] = v;
    }
    ii += di;
    jj += dj;
    if (ii >= nI) {
      ii -= nI;
      ++jj;
    }
  }
}

}  // namespace

void launch_assemble(const AsmArgs& a, int64_t ntiles, bool helmholtz, void* stream) {
  if (ntiles <= 0) return;
  const size_t smem = sizeof(AsmSmem);
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
