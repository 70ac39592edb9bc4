// K4: stored-matrix matvec y = A x (complex128, column-major), the product the
// reference performs with Eigen::MatrixXcd * VectorXcd (test_assembly.cpp:233,
// :277; LinearOperator::from_matrix, linsolve.hpp:20-23).
//
// HBM-bound: 16 bytes of A per complex MAC.  Each thread owns one row and a
// contiguous column range (split-K); a warp reads 32 consecutive rows of a
// column (512 contiguous bytes) with 8 independent 16-byte streaming loads in
// flight per thread.  Partial sums land in a [splits x rows] scratch and a
// second kernel adds them in split order: deterministic, no atomics.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <mutex>
#include <utility>

#include "gk_internal.hpp"

namespace gk {

namespace {
constexpr int kMvThreads = 256;
constexpr int kMvUnroll = 8;

__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 v;
  asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

__global__ void __launch_bounds__(kMvThreads) k_matvec_partial(const double2* __restrict__ A, long long rows,
                                                               long long cols, long long lda,
                                                               const double2* __restrict__ x,
                                                               double2* __restrict__ P, long long cps) {
  const long long i = (long long)blockIdx.x * kMvThreads + threadIdx.x;
  const long long c0 = (long long)blockIdx.y * cps;
  const long long c1 = min(cols, c0 + cps);
  if (i >= rows) return;
  const double2* a = A + i + c0 * lda;
  double re0 = 0.0, im0 = 0.0, re1 = 0.0, im1 = 0.0;
  long long j = c0;
  for (; j + kMvUnroll <= c1; j += kMvUnroll) {
    double2 v[kMvUnroll];
#pragma unroll
    for (int u = 0; u < kMvUnroll; ++u) v[u] = ld_stream(a + (long long)u * lda);
#pragma unroll
    for (int u = 0; u < kMvUnroll; ++u) {
      const double2 xj = __ldg(x + j + u);
      if (u & 1) {
        re1 = fma(v[u].x, xj.x, re1);
        re1 = fma(-v[u].y, xj.y, re1);
        im1 = fma(v[u].x, xj.y, im1);
        im1 = fma(v[u].y, xj.x, im1);
      } else {
        re0 = fma(v[u].x, xj.x, re0);
        re0 = fma(-v[u].y, xj.y, re0);
        im0 = fma(v[u].x, xj.y, im0);
        im0 = fma(v[u].y, xj.x, im0);
      }
    }
    a += kMvUnroll * lda;
  }
  for (; j < c1; ++j) {
    const double2 v = ld_stream(a);
    const double2 xj = __ldg(x + j);
    re0 = fma(v.x, xj.x, re0);
    re0 = fma(-v.y, xj.y, re0);
    im0 = fma(v.x, xj.y, im0);
    im0 = fma(v.y, xj.x, im0);
    a += lda;
  }
  P[(long long)blockIdx.y * rows + i] = make_double2(re0 + re1, im0 + im1);
}

__global__ void k_matvec_reduce(const double2* __restrict__ P, long long rows, int splits,
                                double2* __restrict__ y) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  double re = 0.0, im = 0.0;
  for (int s = 0; s < splits; ++s) {
    const double2 v = P[(long long)s * rows + i];
    re += v.x;
    im += v.y;
  }
  y[i] = make_double2(re, im);
}

void plan(int64_t rows, int64_t cols, int64_t& splits, int64_t& cps) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t row_blocks = (rows + kMvThreads - 1) / kMvThreads;
  const int64_t target = (int64_t)sms * 48;  // CTAs of 256 threads in flight (measured: x8 -> x48 moved cfg 2 from 5660 to 5820 GB/s)
  splits = std::max<int64_t>(1, std::min<int64_t>((target + row_blocks - 1) / row_blocks,
                                                  std::max<int64_t>(1, cols / 64)));
  splits = std::min<int64_t>(splits, 65535);
  cps = (cols + splits - 1) / splits;
  splits = (cols + cps - 1) / cps;
}

// ---- several right-hand sides in one pass over A: Y = A X -------------------
// (Eigen::MatrixXcd * MatrixXcd with a few columns; the stored-matrix step of
// BASELINE cfg 4 multiplies A by 10 independent vectors.)  Per 16-byte element
// of A, R right-hand sides cost 4 R DFMAs: for R = 10 the FP64 pipe and HBM
// bound the pass about equally, so the A stream must never wait on the FP64
// work.  A register-prefetch version stalled on its loads (long_scoreboard 66%,
// FP64 pipe 44%), so the stream is asynchronous: one elected thread per CTA
// issues bulk copies (cp.async.bulk, the TMA engine; one contiguous
// column segment of the CTA's rows per column, L2 evict-first) into a
// ring of shared-memory stages completed on mbarriers, while all threads
// multiply the stage that has landed (thread = row; A from shared memory,
// conflict-free; x values broadcast from the stage's copy of X).  Each
// (row, right-hand side) sums its columns in order in one chain; the same
// split-K + fixed-order reduce as above: deterministic, and column r of Y does
// not depend on the other columns.
#ifndef GK_MM_STAGES
#define GK_MM_STAGES 2
#endif
#ifndef GK_MM_MINB
#define GK_MM_MINB 3
#endif
#ifndef GK_MM_STAGE_KB
#define GK_MM_STAGE_KB 28
#endif
#ifndef GK_MM_THREADS
#define GK_MM_THREADS 128
#endif
// CTA shape (sweep on cfg 4, 10 vectors; threads / stages / KB of A per stage
// / min CTAs per SM -> ms): 256/3/32/2 24.0, 128/3/32/2 25.3, 128/2/32/2 22.7,
// 128/2/24/2 22.3, 128/2/24/4 23.5, 128/2/48/2 24.6, 64/2/32/2 28.3,
// 128/3/16/2 31.2, 128/2/28/3 21.9 (kept: three CTAs of four warps per SM,
// each with one stage landing while the other is multiplied)
constexpr int kBkStages = GK_MM_STAGES;
constexpr int kMmThreads = GK_MM_THREADS;
constexpr int kMmMaxR = 10;   // right-hand sides per pass (larger counts: several passes)
// Rows per thread: 2 for many right-hand sides (each broadcast x value then
// feeds two rows: 9 instead of 14 shared-memory wavefronts per 32 rows and
// column at R = 10), 1 otherwise.  A stage holds kMmThreads RPT rows x as
// many columns as fit in GK_MM_STAGE_KB.
template <int R>
constexpr int mm_rpt() {
  return R >= 6 ? 2 : 1;
}
template <int RPT>
struct MmSmem {
  static constexpr int kRows = kMmThreads * RPT, kCols = GK_MM_STAGE_KB * 64 / kRows;  // KB of A per stage
  double2 a[kBkStages][kCols][kRows];
  double2 x[kBkStages][kMmMaxR][kCols];
  unsigned long long full[kBkStages];
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                         unsigned long long policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

template <int R>
__global__ void __launch_bounds__(kMmThreads, GK_MM_MINB)
    k_matvec_multi_partial(const double2* __restrict__ A, long long rows, long long cols, long long lda,
                           const double2* __restrict__ X, long long ldx, double2* __restrict__ P, long long cps,
                           int splits) {
  constexpr int RPT = mm_rpt<R>();
  using Smem = MmSmem<RPT>;
  constexpr int kRows = Smem::kRows, kCols = Smem::kCols;
  extern __shared__ __align__(128) unsigned char mm_raw[];
  Smem& S = *reinterpret_cast<Smem*>(mm_raw);
  const int t = threadIdx.x;
  const long long ib = (long long)blockIdx.x * kRows;
  const int nr = (int)min((long long)kRows, rows - ib);
  const long long c0 = (long long)blockIdx.y * cps;
  const long long c1 = min(cols, c0 + cps);
  const long long ngroups = (c1 - c0 + kCols - 1) / kCols;
  unsigned long long policy = 0;
  if (t == 0) {
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    for (int q = 0; q < kBkStages; ++q) mbar_init(&S.full[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](long long g) {  // thread 0 only
    const int buf = (int)(g % kBkStages);
    const long long j = c0 + g * kCols;
    const int nc = (int)min((long long)kCols, c1 - j);
    mbar_expect_tx(&S.full[buf], (unsigned)(16 * nc * (nr + R)));
    for (int c = 0; c < nc; ++c) bulk_g2s(&S.a[buf][c][0], A + ib + (j + c) * lda, 16u * nr, &S.full[buf], policy);
    for (int r = 0; r < R; ++r) bulk_g2s(&S.x[buf][r][0], X + r * ldx + j, 16u * nc, &S.full[buf], policy);
  };
  if (t == 0)
    for (long long g = 0; g < min((long long)kBkStages, ngroups); ++g) issue(g);
  // rows t and t + 256 (RPT = 2): both conflict-free in the stage
  double re[RPT][R], im[RPT][R];
#pragma unroll
  for (int k = 0; k < RPT; ++k)
#pragma unroll
    for (int r = 0; r < R; ++r) re[k][r] = im[k][r] = 0.0;
  bool act[RPT];
#pragma unroll
  for (int k = 0; k < RPT; ++k) act[k] = t + k * kMmThreads < nr;
  auto column = [&](int buf, int c) {
    double2 v[RPT];
#pragma unroll
    for (int k = 0; k < RPT; ++k) v[k] = S.a[buf][c][t + k * kMmThreads];  // rows past nr: stale, never stored
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double2 xj = S.x[buf][r][c];
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        re[k][r] = fma(v[k].x, xj.x, re[k][r]);
        re[k][r] = fma(-v[k].y, xj.y, re[k][r]);
        im[k][r] = fma(v[k].x, xj.y, im[k][r]);
        im[k][r] = fma(v[k].y, xj.x, im[k][r]);
      }
    }
  };
  for (long long g = 0; g < ngroups; ++g) {
    const int buf = (int)(g % kBkStages);
    const int nc = (int)min((long long)kCols, c1 - (c0 + g * kCols));
    mbar_wait(&S.full[buf], (unsigned)((g / kBkStages) & 1));
    if (act[0]) {
      if (nc == kCols) {
#pragma unroll
        for (int c = 0; c < kCols; ++c) column(buf, c);
      } else {
        for (int c = 0; c < nc; ++c) column(buf, c);
      }
    }
    __syncthreads();  // every thread is done with this stage
    if (t == 0 && g + kBkStages < ngroups) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the async refill
      issue(g + kBkStages);
    }
  }
#pragma unroll
  for (int k = 0; k < RPT; ++k)
    if (act[k])
#pragma unroll
      for (int r = 0; r < R; ++r)
        P[((long long)r * splits + blockIdx.y) * rows + ib + t + k * kMmThreads] = make_double2(re[k][r], im[k][r]);
}

__global__ void k_matvec_multi_reduce(const double2* __restrict__ P, long long rows, int splits, int nr,
                                      double2* __restrict__ Y, long long ldy) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * nr) return;
  const long long r = e / rows, i = e - r * rows;
  const double2* p = P + r * splits * rows + i;
  double re = 0.0, im = 0.0;
  for (int s = 0; s < splits; ++s) {
    const double2 v = p[(long long)s * rows];
    re += v.x;
    im += v.y;
  }
  Y[r * ldy + i] = make_double2(re, im);
}

template <int R>
void launch_multi_r(const double2* A, int64_t rows, int64_t cols, int64_t lda, const double2* X, int64_t ldx,
                    double2* P, int64_t cps, int64_t splits, cudaStream_t s) {
  constexpr int kRows = MmSmem<mm_rpt<R>()>::kRows;
  const dim3 grid((unsigned)((rows + kRows - 1) / kRows), (unsigned)splits);
  const size_t smem = sizeof(MmSmem<mm_rpt<R>()>);
  static std::atomic<uint64_t> configured{0};  // the attribute is per device context
  const int dev = current_device();
  if (!((configured.load() >> dev) & 1u)) {
    cuda_check(cudaFuncSetAttribute(k_matvec_multi_partial<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
               "cudaFuncSetAttribute");
    configured |= 1ull << dev;
  }
  k_matvec_multi_partial<R><<<grid, kMmThreads, smem, s>>>(A, rows, cols, lda, X, ldx, P, cps, (int)splits);
}

using MultiFn = void (*)(const double2*, int64_t, int64_t, int64_t, const double2*, int64_t, double2*, int64_t,
                         int64_t, cudaStream_t);
template <int... Rs>
constexpr auto multi_table(std::integer_sequence<int, Rs...>) {
  return std::array<MultiFn, sizeof...(Rs)>{&launch_multi_r<Rs + 1>...};
}

void plan_multi(int64_t rows, int64_t cols, int64_t& splits, int64_t& cps) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // FP64-bound: two resident CTAs per SM, about eight waves (short tail)
  const int64_t row_blocks = (rows + kMvThreads - 1) / kMvThreads;
  const int64_t target = (int64_t)sms * 2 * 8;
  splits = std::max<int64_t>(1, std::min<int64_t>((target + row_blocks / 2) / row_blocks,
                                                  std::max<int64_t>(1, cols / 64)));
  splits = std::min<int64_t>(splits, 65535);
  cps = (cols + splits - 1) / splits;
  splits = (cols + cps - 1) / cps;
}

// The partial sums live in stream-ordered memory (cudaMallocAsync from the
// device's default pool, see ensure_pool), so matvecs on different streams
// never share a scratch buffer.
}  // namespace

int matvec_launch_count(int64_t rows, int64_t cols) { return (rows > 0 && cols > 0) ? 2 : 1; }

void launch_matvec(const void* A, int64_t rows, int64_t cols, int64_t lda, const void* x, void* y, void* stream) {
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (rows <= 0) return;
  if (cols <= 0) {
    cuda_check(cudaMemsetAsync(y, 0, sizeof(double2) * rows, s), "cudaMemsetAsync");
    return;
  }
  int64_t splits, cps;
  plan(rows, cols, splits, cps);
  const size_t need = sizeof(double2) * (size_t)rows * (size_t)splits;
  ensure_pool();
  void* P = nullptr;
  if (cudaMallocAsync(&P, need, s) != cudaSuccess) {
    cudaGetLastError();
    throw NoMemError("gk_matvec: scratch allocation failed");
  }
  const dim3 grid((unsigned)((rows + kMvThreads - 1) / kMvThreads), (unsigned)splits);
  k_matvec_partial<<<grid, kMvThreads, 0, s>>>(static_cast<const double2*>(A), rows, cols, lda,
                                               static_cast<const double2*>(x),
                                               static_cast<double2*>(P), cps);
  const cudaError_t e1 = cudaGetLastError();
  k_matvec_reduce<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(static_cast<const double2*>(P), rows,
                                                                (int)splits, static_cast<double2*>(y));
  const cudaError_t e2 = cudaGetLastError();
  cudaFreeAsync(P, s);
  cuda_check(e1, "k_matvec_partial launch");
  cuda_check(e2, "k_matvec_reduce launch");
}

int matvec_multi_launch_count(int64_t rows, int64_t cols, int32_t nrhs) {
  if (rows <= 0 || nrhs <= 0) return 0;
  if (cols <= 0) return nrhs;
  return 2 * (int)((nrhs + kMmMaxR - 1) / kMmMaxR);
}

void launch_matvec_multi(const void* A, int64_t rows, int64_t cols, int64_t lda, const void* X, int64_t ldx, void* Y,
                         int64_t ldy, int32_t nrhs, void* stream) {
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (rows <= 0 || nrhs <= 0) return;
  if (cols <= 0) {
    for (int32_t r = 0; r < nrhs; ++r)
      cuda_check(cudaMemsetAsync(static_cast<double2*>(Y) + r * ldy, 0, sizeof(double2) * rows, s),
                 "cudaMemsetAsync");
    return;
  }
  int64_t splits, cps;
  plan_multi(rows, cols, splits, cps);
  const int32_t rpass = std::min<int32_t>(nrhs, kMmMaxR);
  const size_t need = sizeof(double2) * (size_t)rows * (size_t)splits * (size_t)rpass;
  ensure_pool();
  void* P = nullptr;
  if (cudaMallocAsync(&P, need, s) != cudaSuccess) {
    cudaGetLastError();
    throw NoMemError("gk_matvec_multi: scratch allocation failed");
  }
  static constexpr auto table = multi_table(std::make_integer_sequence<int, kMmMaxR>{});
  cudaError_t e = cudaSuccess;
  for (int32_t r0 = 0; r0 < nrhs && e == cudaSuccess; r0 += kMmMaxR) {
    const int32_t nr = std::min<int32_t>(kMmMaxR, nrhs - r0);
    table[nr - 1](static_cast<const double2*>(A), rows, cols, lda, static_cast<const double2*>(X) + r0 * ldx, ldx,
                  static_cast<double2*>(P), cps, splits, s);
    e = cudaGetLastError();
    if (e != cudaSuccess) break;
    k_matvec_multi_reduce<<<(unsigned)((rows * nr + 255) / 256), 256, 0, s>>>(
        static_cast<const double2*>(P), rows, (int)splits, nr, static_cast<double2*>(Y) + r0 * ldy, ldy);
    e = cudaGetLastError();
  }
  cudaFreeAsync(P, s);
  cuda_check(e, "k_matvec_multi launch");
}

}  // namespace gk
