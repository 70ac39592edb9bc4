// K1+K2: fused pair kernel + basis/quadrature contraction + scatter-to-DOF.
//
// Replaces, for one tile of the matrix, the x-chunk loop of bem_product
// (assembly.cpp:212-220): Kernel::evaluate_blocks (kernels.cpp:76-131), the
// y-side product kr = G (W_y Psi) (assembly.cpp:217) and the x-side update
// A += (W_x Phi)^T kr (assembly.cpp:218).
//
// Tile = (x block I, y block J), one CTA.  Thread t owns x location t of the
// block (twins merged, <= kUCap per block).  The block's y records (unique y
// locations with their <= 2 (slot, coef) pairs, in descending first-slot
// order) and the x support lists are staged in shared memory.  All threads
// walk the same record list (broadcast reads), kRecUnroll records at a time so
// that every thread carries kRecUnroll independent FP64 chains, and evaluate
// G(u, v) once per unique location pair.  c0*G goes to a register run
// accumulator for the record's first slot (stored to H[slot][u] when the slot
// changes), c1*G is added into H[slot][u] in shared memory: the y-side
// contraction, owner-computes per column, no atomics.  After a barrier the
// threads gather whole entries A_ij = sum_u c_ui H[j][u] (x-side contraction,
// fixed order) and write them; with identical sides only tiles on or above
// the diagonal are computed and mirrored (G is symmetric).
//
// Tiles that may hold a coincident pair (host-flagged) run the pair loop with
// the r^2 <= eps^2 mask, all others without it, in the same launch.
// Specialisation SLOTS = 0 (no record has a second slot: P0 with twin-free rules),
// 1 (second slots), 2 (second slots whose coefficient equals the first one in
// every record — the P1 edge-midpoint rule — so c*rinv is formed once).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <type_traits>

#include "gk_internal.hpp"
#include "gk_math.cuh"

namespace gk {

namespace {

#ifndef GK_GATHER_G
#define GK_GATHER_G 4  // tile columns per gather work unit of symmetric tiles (even)
#endif
// Two kernel shapes, chosen per launch by the plan's widest y block:
//  - JC = 22 (y blocks of up to 22 dofs; P1 vertex blocks, cfg 2): 4 CTAs per
//    SM, six records per lockstep group (cfg 2 / cfg 3 ms by records per
//    group: 2: 2.69 / 19.56, 4: 2.55 / 19.32, 6: 2.53 / 19.22, 8: 2.76 / 19.56);
//  - JC = 16 (every y block <= 16 dofs; P0 subtree blocks, cfg 4): H is 32 KB,
//    so 5 CTAs (20 warps) fit per SM, at <= 102 registers: three records per
//    group (96 registers, no spills).  cfg 4 by (CTAs, records per group):
//    (4, 6) 44.6, (4, 3) 46.1, (5, 2) 44.4, (5, 3) 43.3, (5, 4) 47.2,
//    (5, 5) 46.3 ms.
template <int JC>
struct AsmShape;
template <>
struct AsmShape<22> {
  static constexpr int ctas = 4, unroll = 6;
};
template <>
struct AsmShape<16> {
  static constexpr int ctas = 5, unroll = 3;
};
static_assert(kJCap == 22 && kJCapSmall == 16, "the kernel shapes cover the planner's two y-block caps");
// gather: columns per work item (divides JC).  Measured (cfg 2 P1 / cfg 3 P0
// ms): 1: 2.54 / 19.09, 2: 2.53 / 19.20, 11: 2.50 / 19.45 -> 11 for the P1
// edge-midpoint specialisation (SLOTS = 2), 2 otherwise.
template <int SLOTS, int JC>
constexpr int gather_cols() {
  return SLOTS == 2 && JC % 11 == 0 ? 11 : 2;
}
static_assert(22 % gather_cols<2, 22>() == 0 && 16 % gather_cols<2, 16>() == 0 && 22 % gather_cols<0, 22>() == 0 &&
                  16 % gather_cols<0, 16>() == 0,
              "gather column groups must tile the H rows");

template <int JC>
struct AsmSmem {
  double2 H[JC * kHS];  // y-side partial sums H[j][u]
  YRec rec[kRCap];
  double xs_c[kXsCap];
  int32_t xs_u[kXsCap];
  int32_t xs_start[kIMax + 1];
  int32_t orow[kIMax];  // original row index of each tile row
  int32_t ocol[JC];  // original column index of each tile column
  double ys[JC];      // per-column scale (SLOTS == 3)
  long long prof[3];     // diagnostics (GK_ASM_PROF): phase start clocks
  unsigned prof_done;    // threads finished (the last one records the end)
};

// Records in shared memory: 48-byte YRec, or 32-byte YRecU in the unit
// coefficient mode (SLOTS == 3: no coefficients; two LDS.128 per record).
template <int SLOTS>
constexpr int rec_words() {  // 16-byte words per record
  return SLOTS == 3 ? 2 : 3;
}
template <int SLOTS>
__device__ __forceinline__ YRec load_rec(const double2* src) {
  YRec r;
  if (SLOTS == 3) {
    const double2 a0 = src[0], a1 = src[1];
    r.x = a0.x;
    r.y = a0.y;
    r.z = a1.x;
    r.c0 = r.c1 = 1.0;
    const long long s = __double_as_longlong(a1.y);
    r.off0 = (int32_t)(s & 0xffffffffll);
    r.off1 = (int32_t)(s >> 32);
    return r;
  }
  const double2 a0 = src[0], a1 = src[1], a2 = src[2];
  r.x = a0.x;
  r.y = a0.y;
  r.z = a1.x;
  r.c0 = a1.y;
  r.c1 = a2.x;
  const long long s = __double_as_longlong(a2.y);
  r.off0 = (int32_t)(s & 0xffffffffll);
  r.off1 = (int32_t)(s >> 32);
  return r;
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// The pair loop of one tile for thread t (its x location u = (ux, uy, uz)):
// G(u, v) for every record v of the tile, folded into the thread's column Hb
// of the y-side accumulator H (see k_assemble).
template <bool HELM, int SLOTS, int kRecUnroll>
__device__ __forceinline__ void pair_phase(const AsmArgs& a, const double2* const recs, const int nrec, const int nu,
                                           const bool masked, const int t, const double ux, const double uy,
                                           const double uz, char* const Hb) {
  const double eps2 = a.eps2, kappa = a.kappa;
  constexpr int kRW = rec_words<SLOTS>();
  // run accumulator of the current first slot; cur starts at the first
  // record's slot so that the fold below needs no "first run" case
  int cur = nrec > 0 ? load_rec<SLOTS>(recs).off0 : 0;  // byte offset of the run's slot row
  double ar = 0.0, ai = 0.0;
  auto flush = [&]() { *reinterpret_cast<double2*>(Hb + cur) = make_double2(ar, ai); };
  // fold one record's evaluated pair G = (cs + i sn) rinv: a run change stores
  // the finished run (predicated) and restarts the accumulator with selects —
  // no branches.  The basis coefficient is folded into rinv (one DMUL).
  auto fold = [&](const YRec& p, double cs, double sn, double rinv) {
    const double w0 = SLOTS == 3 ? rinv : p.c0 * rinv;
    const bool fresh = p.off0 != cur;
    if (fresh) flush();
    cur = p.off0;
    if (HELM) {
      ar = fma(cs, w0, fresh ? 0.0 : ar);
      ai = fma(sn, w0, fresh ? 0.0 : ai);
    } else {
      ar = fresh ? w0 : ar + w0;
      ai = 0.0;
    }
    if (SLOTS > 0 && p.off1 >= 0 && !(a.dbg & 8)) {  // (dbg 8: timing experiment, no second slot)
      const double w1 = SLOTS >= 2 ? w0 : p.c1 * rinv;
      double2* h = reinterpret_cast<double2*>(Hb + p.off1);
      double2 v = *h;
      if (HELM) {
        v.x = fma(cs, w1, v.x);
        v.y = fma(sn, w1, v.y);
      } else {
        v.x += w1;
      }
      *h = v;
    }
  };
  auto pair_loop = [&](auto mask_tag) {
    constexpr bool MASK = decltype(mask_tag)::value;
    int r = 0;
    for (; r + kRecUnroll <= nrec; r += kRecUnroll) {
      // the whole group's records into registers first (3 LDS.128 each): the H
      // stores in fold() would otherwise force re-loads of every field
      YRec rr[kRecUnroll];
#pragma unroll
      for (int k = 0; k < kRecUnroll; ++k) rr[k] = load_rec<SLOTS>(recs + (r + k) * kRW);
      double dx[kRecUnroll], dy[kRecUnroll], dz[kRecUnroll];
#pragma unroll
      for (int k = 0; k < kRecUnroll; ++k) {
        dx[k] = ux - rr[k].x;
        dy[k] = uy - rr[k].y;
        dz[k] = uz - rr[k].z;
      }
      double cs[kRecUnroll], sn[kRecUnroll], rinv[kRecUnroll];
      green_parts_n<HELM, kRecUnroll, MASK>(dx, dy, dz, eps2, kappa, cs, sn, rinv);
#pragma unroll
      for (int k = 0; k < kRecUnroll; ++k) fold(rr[k], cs[k], sn[k], rinv[k]);
    }
    for (; r < nrec; ++r) {
      const YRec p = load_rec<SLOTS>(recs + r * kRW);
      double dx[1] = {ux - p.x}, dy[1] = {uy - p.y}, dz[1] = {uz - p.z};
      double cs[1], sn[1], rinv[1];
      green_parts_n<HELM, 1, MASK>(dx, dy, dz, eps2, kappa, cs, sn, rinv);
      fold(p, cs[0], sn[0], rinv[0]);
    }
  };
  // lanes without an x location (t >= nu: ~13% of the lanes of a cfg-4 x
  // block) skip the pair loop instead of evaluating a far dummy point: their
  // H column is never read, and predicated-off lanes draw no FP64 power
  // (the kernel runs under the board power cap)
  const bool active = t < nu;
  if ((a.dbg & 4) || !active) {  // (dbg 4: timing experiment, no pair loop)
  } else if (masked)  // uniform per CTA
    pair_loop(std::true_type{});
  else
    pair_loop(std::false_type{});
  if (nrec > 0 && active) flush();
}

// Shared-memory tables of one tile's x-side contraction.
struct GatherView {
  const double2* H;
  const double* xs_c;
  const int32_t* xs_u;
  const int32_t* xs_start;
  const int32_t* orow;
  const int32_t* ocol;
  const double* ys;
};

// The x-side contraction and matrix writes of one tile by the 128 threads
// t = 0..127 of a group (see k_assemble).
template <int SLOTS, int JC>
__device__ __forceinline__ void gather_phase(const AsmArgs& a, const GatherView& S, const int i0, const int nI,
                                             const int j0, const int nJ, const int xs0, const int t) {
  constexpr int kGC = gather_cols<SLOTS, JC>();
  // x-side contraction + write.  Work item = (row ii, kGC consecutive columns):
  // the row's support entries are read once per item and feed kGC independent
  // H loads; lanes run along rows (coalesced columns of the direct block).
  double2* A = reinterpret_cast<double2*>(a.A);
  const long long lda = a.lda;
  const int ngroups = (nJ + kGC - 1) / kGC;
  const int nIs = max(nI, 1);  // no items when nI = 0
  auto entries = [&](int ii, int jb, double (&re)[kGC], double (&im)[kGC]) {
#pragma unroll
    for (int q = 0; q < kGC; ++q) re[q] = im[q] = 0.0;
    const double2* Hr = S.H + jb * kHS;  // rows past nJ hold stale values that are never stored
    const int s1 = S.xs_start[ii + 1] - xs0;
    for (int s = S.xs_start[ii] - xs0; s < s1; ++s) {
      const double c = S.xs_c[s];
      const int u = S.xs_u[s];
#pragma unroll
      for (int q = 0; q < kGC; ++q) {
        const double2 h = Hr[q * kHS + u];
        re[q] = fma(c, h.x, re[q]);
        im[q] = fma(c, h.y, im[q]);
      }
    }
    if (SLOTS == 3)
#pragma unroll
      for (int q = 0; q < kGC; ++q) {
        const double f = S.ys[min(jb + q, JC - 1)];
        re[q] *= f;
        im[q] *= f;
      }
  };
  if (!a.symmetric) {
    // non-symmetric plans: direct stores straight from registers
    const int items = nI * ngroups;
    // item e = (row e % nI, column group e / nI), advanced incrementally
    const int di = kAsmThreads % nIs, dg = kAsmThreads / nIs;
    int ii = t % nIs, jb = (t / nIs) * kGC;
    for (int e = t; e < items; e += kAsmThreads, ii += di, jb += dg * kGC) {
      if (ii >= nI) ii -= nI, jb += kGC;
      const int pi = i0 + ii;
      if (a.symmetric && pi > j0 + min(jb + kGC, nJ) - 1) continue;  // whole group below the diagonal
      double re[kGC], im[kGC];
      entries(ii, jb, re, im);
      const long long oi = a.natural ? pi : S.orow[ii];
#pragma unroll
      for (int q = 0; q < kGC; ++q) {
        const int pj = j0 + jb + q;
        if (jb + q < nJ && !(a.symmetric && pi > pj)) {
          const long long oj = a.natural ? pj : S.ocol[jb + q];
          const double2 v = make_double2(re[q], im[q]);
          A[oi + oj * lda] = v;
          if (a.symmetric && pi != pj) A[oj + oi * lda] = v;
        }
      }
    }
    return;
  }
  // Symmetric tiles: work unit = (row ii, strip of kG consecutive tile
  // columns), units spread evenly over all threads (an x block of 128
  // locations holds ~73 P0 rows: one row per thread left 55 threads idle and
  // the others walking all 22 columns).  A unit loads its row's supports once,
  // then issues all 3 kG H loads before any multiply-add (independent chains:
  // the gather is latency-bound), and writes each entry to (i, j) — lanes
  // along rows: one column segment per warp store (natural order: contiguous;
  // RCB units of 4: 64-byte runs) — and to the mirror (j, i) — each lane down
  // its own column, two entries per 32-byte store (STG.256) where two
  // consecutive tile columns are adjacent, aligned rows of A (strips start on
  // even absolute columns).  Only entries with row <= column are written, the
  // diagonal once.
  constexpr int kSupCache = 3;  // supports in registers (P0 3-point rows have exactly three)
  constexpr int kG = GK_GATHER_G;
  if (a.dbg & 2) return;
  const int par = j0 & 1;  // strip s covers tile columns [s kG - par, (s + 1) kG - par)
  const int nstrips = (nJ + par + kG - 1) / kG;
  const int units = nI * nstrips;
  const int du_i = kAsmThreads % nIs, du_s = kAsmThreads / nIs;
  const bool nat = a.natural != 0;
  int ii = t % nIs, strip = t / nIs;
  for (int u = t; u < units; u += kAsmThreads, ii += du_i, strip += du_s) {
    if (ii >= nI) ii -= nI, ++strip;
    const int pi = i0 + ii;
    const int jb = strip * kG - par;  // tile column of slot q is jb + q
    if (j0 + min(jb + kG, nJ) - 1 < pi) continue;  // the whole strip lies below the diagonal
    const int sb = S.xs_start[ii] - xs0, ns = S.xs_start[ii + 1] - xs0 - sb;
    // supports padded with coefficient 0 on a real location (finite H); rows
    // without supports (constrained or oversized dofs) give entries 0
    int su[kSupCache];
    double sc[kSupCache];
    const int u0 = ns > 0 ? S.xs_u[sb] : 0;
#pragma unroll
    for (int k = 0; k < kSupCache; ++k) {
      su[k] = k < ns ? S.xs_u[sb + k] : u0;
      sc[k] = k < ns ? S.xs_c[sb + k] : 0.0;
    }
    int jq[kG];
#pragma unroll
    for (int q = 0; q < kG; ++q) jq[q] = min(max(jb + q, 0), JC - 1);  // in-bounds H row (stale rows unused)
    double2 h[kG][kSupCache];
#pragma unroll
    for (int q = 0; q < kG; ++q)
#pragma unroll
      for (int k = 0; k < kSupCache; ++k) h[q][k] = S.H[jq[q] * kHS + su[k]];
    double re[kG], im[kG];
#pragma unroll
    for (int q = 0; q < kG; ++q) {
      re[q] = sc[0] * h[q][0].x;
      im[q] = sc[0] * h[q][0].y;
#pragma unroll
      for (int k = 1; k < kSupCache; ++k) {
        re[q] = fma(sc[k], h[q][k].x, re[q]);
        im[q] = fma(sc[k], h[q][k].y, im[q]);
      }
    }
    if (ns > kSupCache)  // longer rows (6-point P0, P1 rows): the remaining supports in order
      for (int k = kSupCache; k < ns; ++k) {
        const double c = S.xs_c[sb + k];
        const int uk = S.xs_u[sb + k];
#pragma unroll
        for (int q = 0; q < kG; ++q) {
          const double2 hv = S.H[jq[q] * kHS + uk];
          re[q] = fma(c, hv.x, re[q]);
          im[q] = fma(c, hv.y, im[q]);
        }
      }
    if (SLOTS == 3)
#pragma unroll
      for (int q = 0; q < kG; ++q) {
        const double f = S.ys[jq[q]];
        re[q] *= f;
        im[q] *= f;
      }
    if (a.dbg & 1) {  // timing experiment: no stores (keep the values live)
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < kG; ++q) acc += re[q] + im[q];
      if (acc == 1234.5) A[0] = make_double2(acc, acc);
      continue;
    }
    const long long oi = nat ? (long long)pi : (long long)S.orow[ii];
    double2* const Arow = A + oi;        // direct (oi, oj) = Arow[oj * lda]
    double2* const Acol = A + oi * lda;  // mirror (oj, oi) = Acol[oj]
    long long oj[kG];
    bool ok[kG], off[kG];  // ok: entry in the tile and on/above the diagonal; off: strictly above
#pragma unroll
    for (int q = 0; q < kG; ++q) {
      const int j = jb + q;
      ok[q] = j >= 0 && j < nJ && j0 + j >= pi;
      off[q] = ok[q] && j0 + j != pi;
      oj[q] = nat ? (long long)(j0 + j) : (long long)S.ocol[jq[q]];
    }
#pragma unroll
    for (int q = 0; q < kG; ++q)
      if (ok[q] && !(a.dbg & 16)) Arow[oj[q] * lda] = make_double2(re[q], im[q]);  // (dbg 16: no direct stores)
    if (a.dbg & 32) continue;  // (dbg 32: no mirror stores)
#pragma unroll
    for (int q = 0; q < kG; q += 2) {
      double2* const m = Acol + oj[q];
      if (q + 1 < kG && off[q] && off[q + 1] && oj[q + 1] == oj[q] + 1 && (reinterpret_cast<uintptr_t>(m) & 31) == 0) {
        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(m), "d"(re[q]), "d"(im[q]), "d"(re[q + 1]),
                     "d"(im[q + 1]));
      } else {
        if (off[q]) *m = make_double2(re[q], im[q]);
        if (q + 1 < kG && off[q + 1]) Acol[oj[q + 1]] = make_double2(re[q + 1], im[q + 1]);
      }
    }
  }
}

template <bool HELM, int SLOTS, int JC>
__global__ void __launch_bounds__(kAsmThreads, AsmShape<JC>::ctas) k_assemble(const AsmArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  AsmSmem<JC>& S = *reinterpret_cast<AsmSmem<JC>*>(smem_raw);
  const int t = threadIdx.x;
  if (a.prof && t == 0) S.prof[0] = clock64(), S.prof_done = 0;
  const int4* dp = reinterpret_cast<const int4*>(a.tiles + blockIdx.x);
  const int4 d0 = __ldg(dp), d1 = __ldg(dp + 1), d2 = __ldg(dp + 2);
  const int i0 = d0.x, nI = d0.y, j0 = d0.z, nJ = d0.w;
  const int l0 = d1.x, nu = d1.y, r0 = d1.z, nrec = d1.w;
  const int xs0 = d2.x, nxs = d2.y;
  const uint32_t zero_rows = (uint32_t)d2.z;
  const bool masked = d2.w != 0;

  // stage with cp.async (no register staging): group 0 = the records the pair
  // loop needs now; group 1 = the x support lists and dof maps the gather
  // needs only after the pair loop, so their latency hides behind it.
  // Each H row is first written by its own run flush (a plain store; the
  // host orders the runs so that every read-modify-write of a row comes
  // after it); only rows without a run (host bitmask) are zero-filled.
  // each thread zero-fills its own column of the rows without a run (the
  // pair loop touches only that column; the gather comes after a barrier)
  for (uint32_t m = zero_rows; m; m &= m - 1) S.H[(__ffs(m) - 1) * kHS + t] = make_double2(0.0, 0.0);
  constexpr int kRW = rec_words<SLOTS>();
  // (records read straight from global memory by warp-uniform loads instead
  // of staged here measured 59.4 vs 44.6 ms on cfg 4)
  const double2* const recs = reinterpret_cast<const double2*>(S.rec);
  {
    const double2* src = reinterpret_cast<const double2*>(a.yrec) + (long long)r0 * kRW;
    double2* dst = reinterpret_cast<double2*>(S.rec);
    for (int e = t; e < nrec * kRW; e += kAsmThreads) cp_async16(dst + e, src + e);
  }
  cp_async_commit();
  for (int e = t; e < nxs; e += kAsmThreads) {
    cp_async8(S.xs_c + e, a.xsup_c + xs0 + e);
    cp_async4(S.xs_u + e, a.xsup_u + xs0 + e);
  }
  for (int e = t; e <= nI; e += kAsmThreads) cp_async4(S.xs_start + e, a.xsup_start + i0 + e);  // global offsets
  if (!a.natural) {  // natural order: A's row/column index is the permuted one (no maps)
    for (int e = t; e < nI; e += kAsmThreads) cp_async4(S.orow + e, a.xperm + i0 + e);
    for (int e = t; e < nJ; e += kAsmThreads) cp_async4(S.ocol + e, a.yperm + j0 + e);
  }
  if (SLOTS == 3)
    for (int e = t; e < nJ; e += kAsmThreads) cp_async8(S.ys + e, a.yscale + j0 + e);
  cp_async_commit();
  // my x location; idle columns are far away (finite, never gathered)
  const double ux = t < nu ? __ldg(a.xl_x + l0 + t) : 1e100;
  const double uy = t < nu ? __ldg(a.xl_y + l0 + t) : 0.0;
  const double uz = t < nu ? __ldg(a.xl_z + l0 + t) : 0.0;
  cp_async_wait<1>();
  __syncthreads();
  if (a.prof && t == 0) S.prof[1] = clock64();

  char* const Hb = reinterpret_cast<char*>(S.H) + t * 16;  // my column of H
  pair_phase<HELM, SLOTS, AsmShape<JC>::unroll>(a, recs, nrec, nu, masked, t, ux, uy, uz, Hb);
  cp_async_wait<0>();
  __syncthreads();
  // diagnostics (GK_ASM_PROF=1): per-tile cycles of staging / pair loop / gather
  struct PhaseProf {
    const AsmArgs& a;
    AsmSmem<JC>& S;
    __device__ ~PhaseProf() {
      if (!a.prof) return;
      // no barrier: threads leave the gather at different points; the last
      // one to finish records the end of the tile
      __threadfence_block();
      if (atomicAdd(&S.prof_done, 1u) == blockDim.x - 1) {
        unsigned long long* o = a.prof + 4ull * blockIdx.x;
        o[0] = (unsigned long long)(S.prof[1] - S.prof[0]);
        o[1] = (unsigned long long)(S.prof[2] - S.prof[1]);
        o[2] = (unsigned long long)(clock64() - S.prof[2]);
        unsigned smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        o[3] = smid;
      }
    }
  } prof_guard{a, S};
  if (a.prof && t == 0) S.prof[2] = clock64();

  gather_phase<SLOTS, JC>(a, GatherView{S.H, S.xs_c, S.xs_u, S.xs_start, S.orow, S.ocol, S.ys}, i0, nI, j0, nJ, xs0,
                          t);
}

template <bool HELM, int SLOTS, int JC>
void launch_shape(const AsmArgs& a, int64_t ntiles, cudaStream_t s) {
  const size_t smem = sizeof(AsmSmem<JC>);
  // the dynamic shared memory attribute is per device context: one flag per
  // device and instantiation
  static std::atomic<uint64_t> configured{0};
  const int dev = current_device();
  if (!((configured.load() >> dev) & 1u)) {
    cuda_check(cudaFuncSetAttribute(k_assemble<HELM, SLOTS, JC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem),
               "cudaFuncSetAttribute");
    configured |= 1ull << dev;
  }
  if (a.l2_window && a.l2_window_bytes) {
    // the plan tables in a persisting L2 window for this launch only (a launch
    // attribute: no stream state to set and clear)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)ntiles);
    cfg.blockDim = dim3(kAsmThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeAccessPolicyWindow;
    at[0].val.accessPolicyWindow.base_ptr = const_cast<void*>(a.l2_window);
    at[0].val.accessPolicyWindow.num_bytes = (size_t)a.l2_window_bytes;
    at[0].val.accessPolicyWindow.hitRatio = 1.0f;
    at[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cuda_check(cudaLaunchKernelEx(&cfg, k_assemble<HELM, SLOTS, JC>, a), "k_assemble launch");
    return;
  }
  k_assemble<HELM, SLOTS, JC><<<(unsigned)ntiles, kAsmThreads, smem, s>>>(a);
}

template <bool HELM, int SLOTS>
void launch_one(const AsmArgs& a, int64_t ntiles, cudaStream_t s) {
  if (a.jmax <= 16)
    launch_shape<HELM, SLOTS, 16>(a, ntiles, s);
  else
    launch_shape<HELM, SLOTS, 22>(a, ntiles, s);
}

template <bool HELM>
void launch_slots(const AsmArgs& a, int64_t ntiles, int slots, cudaStream_t s) {
  if (slots == 0)
    launch_one<HELM, 0>(a, ntiles, s);
  else if (slots == 1)
    launch_one<HELM, 1>(a, ntiles, s);
  else if (slots == 2)
    launch_one<HELM, 2>(a, ntiles, s);
  else
    launch_one<HELM, 3>(a, ntiles, s);
}

// Tile tables from mapped pinned host memory into device memory by SM loads:
// the copy engines stay free for the matrix slabs streaming the other way (a
// cudaMemcpyAsync of the tables would queue behind the previous slab's D2H).
__global__ void __launch_bounds__(256) k_fetch_tables(int4* __restrict__ dst, const int4* __restrict__ src,
                                                      int64_t n16) {
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < n16; i += (int64_t)gridDim.x * 256) dst[i] = src[i];
}

template <bool HELM>
__global__ void __launch_bounds__(256) k_big_entries(const BigArgs b) {
  const long long n_r = b.nbig_rows * b.ncols;  // big rows x all columns, then all rows x big columns
  const long long n = n_r + (b.symmetric ? 0 : b.nrows * b.nbig_cols);
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  long long i, j;
  if (e < n_r) {
    i = b.rows[e / b.ncols];
    j = e % b.ncols;
  } else {
    const long long f = e - n_r;
    i = f % b.nrows;
    j = b.cols[f / b.nrows];
  }
  double re = 0.0, im = 0.0;
  for (int64_t p = b.xs[i]; p < b.xs[i + 1]; ++p) {
    const int32_t u = b.xl[p];
    const double ux = b.xp[3 * u], uy = b.xp[3 * u + 1], uz = b.xp[3 * u + 2];
    double tr = 0.0, ti = 0.0;  // sum_v c_vj G(u, v)  (assembly.cpp:217, y side first)
    for (int64_t q = b.ys[j]; q < b.ys[j + 1]; ++q) {
      const int32_t v = b.yl[q];
      double dx[1] = {ux - b.yp[3 * v]}, dy[1] = {uy - b.yp[3 * v + 1]}, dz[1] = {uz - b.yp[3 * v + 2]};
      double cs[1], sn[1], rinv[1];
      green_parts_n<HELM, 1, true>(dx, dy, dz, b.eps2, b.kappa, cs, sn, rinv);
      const double w = b.yc[q] * rinv[0];
      if (HELM) {
        tr = fma(cs[0], w, tr);
        ti = fma(sn[0], w, ti);
      } else {
        tr += w;
      }
    }
    re = fma(b.xc[p], tr, re);
    im = fma(b.xc[p], ti, im);
  }
  double2* A = reinterpret_cast<double2*>(b.A);
  A[i + j * b.lda] = make_double2(re, im);
  if (b.symmetric) A[j + i * b.lda] = make_double2(re, im);
}

__global__ void __launch_bounds__(256) k_make_tiles(const TileBuildArgs b) {
  const int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (e >= b.ntiles) return;
  int lo = 0, hi = b.nIb;  // the last x block with tile_start <= e (empty blocks share starts)
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (b.tile_start[mid] <= e) lo = mid;
    else hi = mid;
  }
  const int bi = lo;
  const int bj = b.first_bj[bi] + (int)(e - b.tile_start[bi]);
  TileDesc D;
  D.i0 = b.xb_dof_start[bi];
  D.nI = b.xb_dof_start[bi + 1] - D.i0;
  D.j0 = b.yb_dof_start[bj];
  D.nJ = b.yb_dof_start[bj + 1] - D.j0;
  D.l0 = b.xb_loc_start[bi];
  D.nu = b.xb_loc_start[bi + 1] - D.l0;
  D.r0 = b.yb_rec_start[bj];
  D.nrec = b.yb_rec_start[bj + 1] - D.r0;
  D.xs0 = b.xsup_start[D.i0];
  D.nxs = b.xsup_start[D.i0 + D.nI] - D.xs0;
  D.zero_rows = b.yb_zero[bj];
  D.masked = (int32_t)((b.masked_bits[e >> 5] >> (e & 31)) & 1u);
  const int4* src = reinterpret_cast<const int4*>(&D);
  int4* dst = reinterpret_cast<int4*>(b.out + e);
  dst[0] = src[0];
  dst[1] = src[1];
  dst[2] = src[2];
}

}  // namespace

void launch_make_tiles(const TileBuildArgs& b, void* stream) {
  if (b.ntiles <= 0) return;
  k_make_tiles<<<(unsigned)((b.ntiles + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(b);
  cuda_check(cudaGetLastError(), "k_make_tiles launch");
}

void launch_big_entries(const BigArgs& b, bool helmholtz, void* stream) {
  const long long n = b.nbig_rows * b.ncols + (b.symmetric ? 0 : b.nrows * b.nbig_cols);
  if (n <= 0) return;
  const unsigned blocks = (unsigned)((n + 255) / 256);
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (helmholtz)
    k_big_entries<true><<<blocks, 256, 0, s>>>(b);
  else
    k_big_entries<false><<<blocks, 256, 0, s>>>(b);
  cuda_check(cudaGetLastError(), "k_big_entries launch");
}

void launch_fetch_tables(void* dst, const void* src_mapped, size_t bytes, void* stream) {
  const int64_t n16 = (int64_t)((bytes + 15) / 16);
  if (n16 == 0) return;
  const int blocks = (int)std::min<int64_t>(148, (n16 + 255) / 256);
  k_fetch_tables<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<int4*>(dst), static_cast<const int4*>(src_mapped), n16);
  cuda_check(cudaGetLastError(), "k_fetch_tables launch");
}

void launch_assemble(const AsmArgs& a, int64_t ntiles, bool helmholtz, int slots, void* stream) {
  if (ntiles <= 0) return;
  if (ntiles > INT32_MAX) throw std::invalid_argument("bem_dense: too many tiles");
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (helmholtz)
    launch_slots<true>(a, ntiles, slots, s);
  else
    launch_slots<false>(a, ntiles, slots, s);
  cuda_check(cudaGetLastError(), "k_assemble launch");
}

}  // namespace gk
