// K1+K2: fused pair kernel + basis/quadrature contraction + scatter-to-DOF.
//
// Replaces, for one tile of the matrix, the x-chunk loop of bem_product
// (assembly.cpp:212-220): Kernel::evaluate_blocks (kernels.cpp:76-131), the
// y-side product kr = G (W_y Psi) (assembly.cpp:217) and the x-side update
// A += (W_x Phi)^T kr (assembly.cpp:218).
//
// Tile = (x block I, y block J).  Thread t owns x locations t and t+128 of
// the block (twins merged, <= 256 per block).  The block's y records (unique
// y locations with their <= 2 (slot, coef) pairs, sorted by first slot) and
// the x support lists are staged in shared memory.  All threads walk the same
// record list (broadcast reads) and evaluate G(u, v) once per unique location
// pair — two x locations per record, so record loads and the uniform run /
// slot branches are shared by two pair evaluations and every thread carries
// 2 x kRecUnroll independent FP64 chains.  c0*G goes to a register run
// accumulator for the record's first slot (flushed when the slot changes),
// c1*G is added into H[slot][u] in shared memory: the y-side contraction,
// owner-computes per column, no atomics.  After a barrier each thread gathers
// whole entries A_ij = sum_u c_ui H[j][u] (x-side contraction, fixed order)
// and writes them; with identical sides only tiles on or above the diagonal
// are computed and mirrored (G is symmetric).
//
// Specialisations: MASK (tile may hold a coincident pair -> r^2 <= eps^2
// mask), S1 (some record has a second slot; P0 with twin-free rules has none).
#include <cuda_runtime.h>

#include "gk_internal.hpp"
#include "gk_math.cuh"

namespace gk {

namespace {

constexpr int kRecUnroll = 4 / kUPT;  // records per group (x kUPT locations = 4 independent evaluations)
constexpr int kGC = 4;                // gather: columns per work item
static_assert(kJCap % kGC == 0, "gather column groups must tile the H rows");

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

template <bool HELM, bool MASK, bool S1>
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

  // stage: records and x support lists.  Records run in descending first-slot
  // order, so each H row is first written by its own run flush (a plain store);
  // only rows without a run (host bitmask) are zero-filled.
  const uint32_t zero_rows = a.yb_zero[bj];
  if (zero_rows)
    for (int e = t; e < nJ * kUCap; e += kAsmThreads)
      if ((zero_rows >> (e / kUCap)) & 1u) S.H[e] = make_double2(0.0, 0.0);
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
  // my two x locations; idle columns are far away (finite, never gathered)
  double ux[kUPT], uy[kUPT], uz[kUPT];
#pragma unroll
  for (int h = 0; h < kUPT; ++h) {
    const int c = t + h * kAsmThreads;
    ux[h] = c < nu ? __ldg(a.xl_x + l0 + c) : 1e100;
    uy[h] = c < nu ? __ldg(a.xl_y + l0 + c) : 0.0;
    uz[h] = c < nu ? __ldg(a.xl_z + l0 + c) : 0.0;
  }
  __syncthreads();

  const double eps2 = a.eps2, kappa = a.kappa;
  char* Hb[kUPT];
#pragma unroll
  for (int h = 0; h < kUPT; ++h) Hb[h] = reinterpret_cast<char*>(S.H) + (t + h * kAsmThreads) * 16;
  // run accumulator of the current first slot; cur starts at the first
  // record's slot so that the fold below needs no "first run" case
  int cur = nrec > 0 ? S.rec[0].off0 : 0;  // byte offset of the run's slot row
  double ar[kUPT], ai[kUPT];
#pragma unroll
  for (int h = 0; h < kUPT; ++h) ar[h] = ai[h] = 0.0;
  auto flush = [&]() {
#pragma unroll
    for (int h = 0; h < kUPT; ++h) *reinterpret_cast<double2*>(Hb[h] + cur) = make_double2(ar[h], ai[h]);
  };
  // fold one record's evaluated pairs: a run change stores the finished run
  // (predicated) and restarts the accumulator with selects — no branches
  auto fold = [&](const YRec& p, const c64* g) {
    const bool fresh = p.off0 != cur;
    if (fresh) flush();
    cur = p.off0;
#pragma unroll
    for (int h = 0; h < kUPT; ++h) {
      ar[h] = fma(p.c0, g[h].re, fresh ? 0.0 : ar[h]);
      ai[h] = fma(p.c0, g[h].im, fresh ? 0.0 : ai[h]);
    }
    if (S1 && p.off1 >= 0)
#pragma unroll
      for (int h = 0; h < kUPT; ++h) rmw(Hb[h], p.off1, p.c1, g[h].re, g[h].im);
  };
  constexpr int N = kRecUnroll * kUPT;
  int r = 0;
  for (; r + kRecUnroll <= nrec; r += kRecUnroll) {
    // the whole group's records into registers first (3 LDS.128 each): the H
    // stores in fold() would otherwise force re-loads of every field
    YRec rr[kRecUnroll];
#pragma unroll
    for (int k = 0; k < kRecUnroll; ++k) {
      const double2* src = reinterpret_cast<const double2*>(&S.rec[r + k]);
      const double2 a0 = src[0], a1 = src[1], a2 = src[2];
      rr[k].x = a0.x;
      rr[k].y = a0.y;
      rr[k].z = a1.x;
      rr[k].c0 = a1.y;
      rr[k].c1 = a2.x;
      const long long s = __double_as_longlong(a2.y);
      rr[k].off0 = (int32_t)(s & 0xffffffffll);
      rr[k].off1 = (int32_t)(s >> 32);
    }
    double dx[N], dy[N], dz[N];
#pragma unroll
    for (int k = 0; k < kRecUnroll; ++k)
#pragma unroll
      for (int h = 0; h < kUPT; ++h) {
        dx[k * kUPT + h] = ux[h] - rr[k].x;
        dy[k * kUPT + h] = uy[h] - rr[k].y;
        dz[k * kUPT + h] = uz[h] - rr[k].z;
      }
    c64 g[N];
    green_n<HELM, N, MASK>(dx, dy, dz, eps2, kappa, g);
#pragma unroll
    for (int k = 0; k < kRecUnroll; ++k) fold(rr[k], g + k * kUPT);
  }
  for (; r < nrec; ++r) {
    const YRec& p = S.rec[r];
    double dx[kUPT], dy[kUPT], dz[kUPT];
#pragma unroll
    for (int h = 0; h < kUPT; ++h) {
      dx[h] = ux[h] - p.x;
      dy[h] = uy[h] - p.y;
      dz[h] = uz[h] - p.z;
    }
    c64 g[kUPT];
    green_n<HELM, kUPT, MASK>(dx, dy, dz, eps2, kappa, g);
    fold(p, g);
  }
  if (nrec > 0) flush();
  __syncthreads();

  // x-side contraction + write.  Work item = (row ii, kGC consecutive columns):
  // the row's support entries are read once per item and feed kGC independent
  // H loads; lanes run along rows (coalesced columns for the natural order).
  double2* A = reinterpret_cast<double2*>(a.A);
  const long long lda = a.lda;
  const int items = nI * ((nJ + kGC - 1) / kGC);
  for (int e = t; e < items; e += kAsmThreads) {
    const int ii = e % nI, jb = (e / nI) * kGC;
    const int pi = i0 + ii;
    if (a.symmetric && pi > j0 + min(jb + kGC, nJ) - 1) continue;  // whole group below the diagonal
    double re[kGC], im[kGC];
#pragma unroll
    for (int q = 0; q < kGC; ++q) re[q] = im[q] = 0.0;
    const double2* Hr = S.H + jb * kUCap;  // rows past nJ hold stale values that are never stored
    const int s1 = S.xs_start[ii + 1];
    for (int s = S.xs_start[ii]; s < s1; ++s) {
      const double c = S.xs_c[s];
      const int u = S.xs_u[s];
#pragma unroll
      for (int q = 0; q < kGC; ++q) {
        const double2 h = Hr[q * kUCap + u];
        re[q] = fma(c, h.x, re[q]);
        im[q] = fma(c, h.y, im[q]);
      }
    }
    const long long oi = S.orow[ii];
#pragma unroll
    for (int q = 0; q < kGC; ++q) {
      const int jj = jb + q, pj = j0 + jj;
      if (jj < nJ && !(a.symmetric && pi > pj)) {
        const long long oj = S.ocol[jj];
        const double2 v = make_double2(re[q], im[q]);
        A[oi + oj * lda] = v;
        if (a.symmetric && pi != pj) A[oj + oi * lda] = v;
      }
    }
  }
}

template <bool HELM, bool MASK, bool S1>
void launch_one(const AsmArgs& a, int64_t ntiles, cudaStream_t s) {
  const size_t smem = sizeof(AsmSmem);
  static bool configured = false;  // one flag per instantiation
  if (!configured) {
    cuda_check(cudaFuncSetAttribute(k_assemble<HELM, MASK, S1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem),
               "cudaFuncSetAttribute");
    configured = true;
  }
  k_assemble<HELM, MASK, S1><<<(unsigned)ntiles, kAsmThreads, smem, s>>>(a);
}

}  // namespace

void launch_assemble(const AsmArgs& a, int64_t ntiles, bool helmholtz, bool mask, bool second_slot,
                     void* stream) {
  if (ntiles <= 0) return;
  if (ntiles > INT32_MAX) throw std::invalid_argument("bem_dense: too many tiles");
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int sel = (helmholtz ? 4 : 0) | (mask ? 2 : 0) | (second_slot ? 1 : 0);
  switch (sel) {
    case 0: launch_one<false, false, false>(a, ntiles, s); break;
    case 1: launch_one<false, false, true>(a, ntiles, s); break;
    case 2: launch_one<false, true, false>(a, ntiles, s); break;
    case 3: launch_one<false, true, true>(a, ntiles, s); break;
    case 4: launch_one<true, false, false>(a, ntiles, s); break;
    case 5: launch_one<true, false, true>(a, ntiles, s); break;
    case 6: launch_one<true, true, false>(a, ntiles, s); break;
    default: launch_one<true, true, true>(a, ntiles, s); break;
  }
  cuda_check(cudaGetLastError(), "k_assemble launch");
}

}  // namespace gk
