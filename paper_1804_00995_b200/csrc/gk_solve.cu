// Solve step on the device-resident dense matrix.
//
//  * gk_lu_factor / gk_lu_solve: partial-pivot LU, the reference's
//    Eigen::PartialPivLU solve (test_assembly.cpp:227), through cuSOLVER's
//    64-bit getrf/getrs (a library factorisation, loaded on first use).
//  * gk_gmres: restarted GMRES of linsolve.cpp:19-121 with the stored matrix
//    as the operator (LinearOperator::from_matrix, linsolve.hpp:20-23).  The
//    Krylov basis stays in HBM; each iteration is one K4 matvec, the
//    reference's modified Gram-Schmidt (linsolve.cpp:59-63: j + 1 dependent
//    dot / axpy pairs, each dot a two-stage fixed-order reduction left on the
//    device for the axpy that follows) and a norm.  The tiny
//    Hessenberg least-squares problem (Givens rotations, back substitution)
//    runs on the host exactly as in the reference.  All reductions are
//    two-stage with a fixed order: results are deterministic.
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <dlfcn.h>

#include <cmath>
#include <complex>
#include <mutex>
#include <vector>

#include "gk_internal.hpp"

using namespace gk;

namespace gk {
namespace {

// ---- cuSOLVER (dlopen'ed: the library has no link-time dependency on it) ------
struct Cusolver {
  bool ok = false;
  std::string why;
  cusolverStatus_t (*create)(cusolverDnHandle_t*) = nullptr;
  cusolverStatus_t (*destroy)(cusolverDnHandle_t) = nullptr;
  cusolverStatus_t (*set_stream)(cusolverDnHandle_t, cudaStream_t) = nullptr;
  cusolverStatus_t (*create_params)(cusolverDnParams_t*) = nullptr;
  cusolverStatus_t (*destroy_params)(cusolverDnParams_t) = nullptr;
  cusolverStatus_t (*getrf_bs)(cusolverDnHandle_t, cusolverDnParams_t, int64_t, int64_t, cudaDataType, const void*,
                               int64_t, cudaDataType, size_t*, size_t*) = nullptr;
  cusolverStatus_t (*getrf)(cusolverDnHandle_t, cusolverDnParams_t, int64_t, int64_t, cudaDataType, void*, int64_t,
                            int64_t*, cudaDataType, void*, size_t, void*, size_t, int*) = nullptr;
  cusolverStatus_t (*getrs)(cusolverDnHandle_t, cusolverDnParams_t, cublasOperation_t, int64_t, int64_t,
                            cudaDataType, const void*, int64_t, const int64_t*, cudaDataType, void*, int64_t,
                            int*) = nullptr;
};

const Cusolver& cusolver() {
  static Cusolver C;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libcusolver.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      C.why = std::string("cuSOLVER not loadable: ") + (e ? e : "unknown");
      return;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) C.why = std::string("cuSOLVER symbol missing: ") + name;
      return fn != nullptr;
    };
    C.ok = sym(C.create, "cusolverDnCreate") && sym(C.destroy, "cusolverDnDestroy") &&
           sym(C.set_stream, "cusolverDnSetStream") && sym(C.create_params, "cusolverDnCreateParams") &&
           sym(C.destroy_params, "cusolverDnDestroyParams") && sym(C.getrf_bs, "cusolverDnXgetrf_bufferSize") &&
           sym(C.getrf, "cusolverDnXgetrf") && sym(C.getrs, "cusolverDnXgetrs");
  });
  if (!C.ok) throw CudaError(C.why);
  return C;
}

void solver_check(cusolverStatus_t s, const char* what) {
  if (s != CUSOLVER_STATUS_SUCCESS) throw CudaError(std::string(what) + ": cuSOLVER status " + std::to_string((int)s));
}

struct Session {  // handle + params bound to one stream for one call
  const Cusolver& C;
  cusolverDnHandle_t h = nullptr;
  cusolverDnParams_t p = nullptr;
  explicit Session(cudaStream_t s) : C(cusolver()) {
    solver_check(C.create(&h), "cusolverDnCreate");
    solver_check(C.set_stream(h, s), "cusolverDnSetStream");
    solver_check(C.create_params(&p), "cusolverDnCreateParams");
  }
  ~Session() {
    if (p) C.destroy_params(p);
    if (h) C.destroy(h);
  }
};

// ---- GMRES vector kernels -----------------------------------------------------------
constexpr int kVThreads = 256;
constexpr int kVRows = 1024;  // rows per block of the multi-dot (4 per thread)
constexpr int kMaxDot = 64;   // columns per multi-dot pass

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// part[b][i] = sum over the block's rows of conj(V[r, i]) * w[r], i < k
__global__ void __launch_bounds__(kVThreads) k_multidot(const double2* __restrict__ V, long long ldv, int k,
                                                        const double2* __restrict__ w, long long n,
                                                        double2* __restrict__ part) {
  __shared__ double sre[kVThreads / 32], sim[kVThreads / 32];
  const long long r0 = (long long)blockIdx.x * kVRows;
  for (int i = 0; i < k; ++i) {
    double re = 0.0, im = 0.0;
    for (long long r = r0 + threadIdx.x; r < min(n, r0 + kVRows); r += kVThreads) {
      const double2 v = V[r + i * ldv], x = w[r];
      re = fma(v.x, x.x, fma(v.y, x.y, re));   // conj(v) * x
      im = fma(v.x, x.y, fma(-v.y, x.x, im));
    }
    re = warp_sum(re);
    im = warp_sum(im);
    if ((threadIdx.x & 31) == 0) {
      sre[threadIdx.x >> 5] = re;
      sim[threadIdx.x >> 5] = im;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double a = 0.0, b = 0.0;
      for (int q = 0; q < kVThreads / 32; ++q) {
        a += sre[q];
        b += sim[q];
      }
      part[(long long)blockIdx.x * k + i] = make_double2(a, b);
    }
    __syncthreads();
  }
}

// h[i] (+)= sum_b part[b][i], fixed block order
__global__ void k_dot_reduce(const double2* __restrict__ part, int nb, int k, double2* __restrict__ h, int accumulate) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  double re = 0.0, im = 0.0;
  for (int b = 0; b < nb; ++b) {
    const double2 p = part[(long long)b * k + i];
    re += p.x;
    im += p.y;
  }
  if (accumulate) {
    h[i].x += re;
    h[i].y += im;
  } else {
    h[i] = make_double2(re, im);
  }
}

// w[r] += sign * sum_i V[r, i] h[i]
__global__ void __launch_bounds__(kVThreads) k_multiaxpy(const double2* __restrict__ V, long long ldv, int k,
                                                         const double2* __restrict__ h, double sign,
                                                         double2* __restrict__ w, long long n) {
  const long long r = (long long)blockIdx.x * kVThreads + threadIdx.x;
  if (r >= n) return;
  double re = 0.0, im = 0.0;
  for (int i = 0; i < k; ++i) {
    const double2 v = V[r + i * ldv], c = h[i];
    re = fma(v.x, c.x, fma(-v.y, c.y, re));
    im = fma(v.x, c.y, fma(v.y, c.x, im));
  }
  w[r].x = fma(sign, re, w[r].x);
  w[r].y = fma(sign, im, w[r].y);
}

// out = in / s (s = sqrt(h[0].x), the reduced squared norm)
__global__ void k_normalize(const double2* __restrict__ in, const double2* __restrict__ nrm2,
                            double2* __restrict__ out, long long n) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const double s = sqrt(nrm2[0].x);
  out[r] = make_double2(in[r].x / s, in[r].y / s);
}


// r = b - r
__global__ void k_bminus(const double2* __restrict__ b, double2* __restrict__ r, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) r[i] = make_double2(b[i].x - r[i].x, b[i].y - r[i].y);
}

struct Krylov {
  long long n;
  cudaStream_t s;
  DevBuf part;
  int nb;
  Krylov(long long n_, cudaStream_t s_) : n(n_), s(s_) {
    nb = (int)((n + kVRows - 1) / kVRows);
    part.alloc(sizeof(double2) * (size_t)nb * kMaxDot);
  }
  // h[0..k) (+)= V[:, :k]^H w
  void dots(const double2* V, long long ldv, int k, const double2* w, double2* h, bool accumulate) {
    for (int i0 = 0; i0 < k; i0 += kMaxDot) {
      const int kk = std::min(kMaxDot, k - i0);
      k_multidot<<<nb, kVThreads, 0, s>>>(V + i0 * ldv, ldv, kk, w, n, part.as<double2>());
      k_dot_reduce<<<(kk + 63) / 64, 64, 0, s>>>(part.as<double2>(), nb, kk, h + i0, accumulate ? 1 : 0);
    }
  }
  void axpys(const double2* V, long long ldv, int k, const double2* h, double sign, double2* w) {
    k_multiaxpy<<<(unsigned)((n + kVThreads - 1) / kVThreads), kVThreads, 0, s>>>(V, ldv, k, h, sign, w, n);
  }
  unsigned grid(int t = 256) const { return (unsigned)((n + t - 1) / t); }
};

using cd = std::complex<double>;

}  // namespace
}  // namespace gk

extern "C" {

gk_status gk_lu_factor(gk_cplx* A, int64_t n, int64_t lda, int64_t* ipiv, int64_t* singular_at, gk_stream stream) {
  return guard([&] {
    if (n < 0) throw std::invalid_argument("gk_lu_factor: negative size");
    if (n > 0 && (!A || !ipiv)) throw std::invalid_argument("gk_lu_factor: null matrix or pivots");
    if (lda < std::max<int64_t>(1, n)) throw std::invalid_argument("gk_lu_factor: lda < n");
    if (singular_at) *singular_at = 0;
    if (n == 0) return;
    require_device();
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    Session S(s);
    size_t dbytes = 0, hbytes = 0;
    solver_check(S.C.getrf_bs(S.h, S.p, n, n, CUDA_C_64F, A, lda, CUDA_C_64F, &dbytes, &hbytes),
                 "cusolverDnXgetrf_bufferSize");
    DevBuf work, dinfo;
    work.alloc(std::max<size_t>(dbytes, 16));
    dinfo.alloc(sizeof(int));
    std::vector<char> hwork(std::max<size_t>(hbytes, 1));
    solver_check(S.C.getrf(S.h, S.p, n, n, CUDA_C_64F, A, lda, ipiv, CUDA_C_64F, work.p, dbytes, hwork.data(),
                           hbytes, dinfo.as<int>()),
                 "cusolverDnXgetrf");
    int info = 0;
    cuda_check(cudaMemcpyAsync(&info, dinfo.p, sizeof(int), cudaMemcpyDeviceToHost, s), "getrf info");
    cuda_check(cudaStreamSynchronize(s), "getrf sync");
    if (info < 0) throw std::invalid_argument("gk_lu_factor: cuSOLVER rejected argument " + std::to_string(-info));
    if (singular_at) *singular_at = info;  // > 0: U(info, info) is exactly zero (1-based)
  });
}

gk_status gk_lu_solve(const gk_cplx* LU, int64_t n, int64_t lda, const int64_t* ipiv, gk_cplx* B, int64_t ldb,
                      int64_t nrhs, gk_stream stream) {
  return guard([&] {
    if (n < 0 || nrhs < 0) throw std::invalid_argument("gk_lu_solve: negative size");
    if (n > 0 && nrhs > 0 && (!LU || !ipiv || !B)) throw std::invalid_argument("gk_lu_solve: null argument");
    if (lda < std::max<int64_t>(1, n) || ldb < std::max<int64_t>(1, n))
      throw std::invalid_argument("gk_lu_solve: leading dimension < n");
    if (n == 0 || nrhs == 0) return;
    require_device();
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    Session S(s);
    DevBuf dinfo;
    dinfo.alloc(sizeof(int));
    solver_check(S.C.getrs(S.h, S.p, CUBLAS_OP_N, n, nrhs, CUDA_C_64F, LU, lda, ipiv, CUDA_C_64F, B, ldb,
                           dinfo.as<int>()),
                 "cusolverDnXgetrs");
    int info = 0;
    cuda_check(cudaMemcpyAsync(&info, dinfo.p, sizeof(int), cudaMemcpyDeviceToHost, s), "getrs info");
    cuda_check(cudaStreamSynchronize(s), "getrs sync");
    if (info != 0) throw std::invalid_argument("gk_lu_solve: cuSOLVER rejected argument " + std::to_string(-info));
  });
}

gk_status gk_gmres(const gk_cplx* A, int64_t n, int64_t lda, const gk_cplx* b, gk_cplx* x, double tol,
                   int32_t restart, int32_t maxit, gk_solve_info* info, double* history, gk_stream stream) {
  return guard([&] {
    if (!(tol > 0)) throw std::invalid_argument("gmres: tol must be positive");  // linsolve.cpp:24
    if (restart <= 0 || maxit < 0) throw std::invalid_argument("gmres: restart must be positive");
    if (n < 0) throw std::invalid_argument("gmres: negative size");
    if (n > 0 && (!A || !b || !x)) throw std::invalid_argument("gmres: null argument");
    if (lda < std::max<int64_t>(1, n)) throw std::invalid_argument("gmres: lda < n");
    gk_solve_info I{0, 0, 0.0, 0};
    auto finish = [&] {
      if (info) *info = I;
    };
    if (n == 0) {
      I.converged = 1;
      finish();
      return;
    }
    require_device();
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int m = restart;
    Krylov K(n, s);
    DevBuf Vb, wb, rb, hb;
    Vb.alloc(sizeof(double2) * (size_t)n * (m + 1));
    wb.alloc(sizeof(double2) * (size_t)n);
    rb.alloc(sizeof(double2) * (size_t)n);
    hb.alloc(sizeof(double2) * (size_t)(m + 2));
    double2* V = Vb.as<double2>();
    double2* w = wb.as<double2>();
    double2* r = rb.as<double2>();
    double2* h = hb.as<double2>();     // [0..j]: projections, [m+1]: squared norm
    double2* X = reinterpret_cast<double2*>(x);
    const double2* B = reinterpret_cast<const double2*>(b);
    const double2* Ad = reinterpret_cast<const double2*>(A);
    std::vector<double2> hh(m + 2);
    auto fetch = [&](int count) {  // h[0..count) and the norm slot to the host
      cuda_check(cudaMemcpyAsync(hh.data(), h, sizeof(double2) * count, cudaMemcpyDeviceToHost, s), "gmres D2H");
      cuda_check(cudaMemcpyAsync(&hh[m + 1], h + m + 1, sizeof(double2), cudaMemcpyDeviceToHost, s), "gmres D2H");
      cuda_check(cudaStreamSynchronize(s), "gmres sync");
    };
    auto norm_of = [&](const double2* v) {  // ||v|| (also leaves ||v||^2 in h[m+1])
      K.dots(v, n, 1, v, h + m + 1, false);
      fetch(0);
      return std::sqrt(hh[m + 1].x);
    };
    auto residual = [&]() {  // r = b - A x, returns ||r||
      launch_matvec(Ad, n, n, lda, X, r, s);
      k_bminus<<<K.grid(), 256, 0, s>>>(B, r, n);
      return norm_of(r);
    };
    cuda_check(cudaMemsetAsync(X, 0, sizeof(double2) * n, s), "gmres x = 0");
    const double bnorm = norm_of(B);
    if (bnorm == 0.0) {
      I.converged = 1;
      finish();
      return;
    }
    std::vector<cd> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1);
    auto Hij = [&](int i, int j) -> cd& { return H[(size_t)i + (size_t)(m + 1) * j]; };
    int total = 0, hist_n = 0;
    bool done = false;
    while (total < maxit && !done) {
      const double beta = residual();
      if (beta / bnorm <= tol) {
        I.converged = 1;
        break;
      }
      k_normalize<<<K.grid(), 256, 0, s>>>(r, h + m + 1, V, n);
      std::fill(g.begin(), g.end(), cd(0.0));
      std::fill(H.begin(), H.end(), cd(0.0));
      g[0] = beta;
      int j = 0;
      for (; j < m && total < maxit; ++j, ++total) {
        launch_matvec(Ad, n, n, lda, V + (size_t)j * n, w, s);
        // modified Gram-Schmidt as linsolve.cpp:59-63: h_i = V_i^H w, w -= h_i V_i
        for (int i = 0; i <= j; ++i) {
          K.dots(V + (size_t)i * n, n, 1, w, h + i, false);
          K.axpys(V + (size_t)i * n, n, 1, h + i, -1.0, w);
        }
        K.dots(w, n, 1, w, h + m + 1, false);
        fetch(j + 1);
        for (int i = 0; i <= j; ++i) Hij(i, j) = cd(hh[i].x, hh[i].y);
        const double hn = std::sqrt(hh[m + 1].x);
        Hij(j + 1, j) = hn;
        if (hn > 0) k_normalize<<<K.grid(), 256, 0, s>>>(w, h + m + 1, V + (size_t)(j + 1) * n, n);
        // Givens rotations exactly as linsolve.cpp:66-85
        for (int i = 0; i < j; ++i) {
          const cd tmp1 = cs[i] * Hij(i, j) + sn[i] * Hij(i + 1, j);
          Hij(i + 1, j) = -std::conj(sn[i]) * Hij(i, j) + std::conj(cs[i]) * Hij(i + 1, j);
          Hij(i, j) = tmp1;
        }
        const double h0 = std::abs(Hij(j, j)), h1 = std::abs(Hij(j + 1, j));
        if (h1 == 0.0) {
          cs[j] = 1.0;
          sn[j] = 0.0;
        } else {
          const double d = std::hypot(h0, h1);
          cs[j] = cd(h0 / d);
          const cd phase = (h0 == 0.0) ? cd(1) : Hij(j, j) / cd(h0);
          sn[j] = phase * std::conj(Hij(j + 1, j)) / cd(d);
        }
        const cd tmp2 = cs[j] * Hij(j, j) + sn[j] * Hij(j + 1, j);
        Hij(j + 1, j) = 0;
        Hij(j, j) = tmp2;
        const cd g1 = -std::conj(sn[j]) * g[j];
        g[j] = cs[j] * g[j];
        g[j + 1] = g1;
        const double rel = std::abs(g[j + 1]) / bnorm;
        if (history && hist_n < maxit) history[hist_n] = rel;
        I.history_len = ++hist_n;
        if (rel <= tol) {  // as the reference: the converging iteration is not counted in total
          ++j;
          break;
        }
      }
      // back substitution (linsolve.cpp:95-103), then x += V[:, :j] y
      std::vector<double2> y(std::max(j, 1));
      for (int i = j - 1; i >= 0; --i) {
        cd acc = g[i];
        for (int k2 = i + 1; k2 < j; ++k2) acc -= Hij(i, k2) * cd(y[k2].x, y[k2].y);
        if (std::abs(Hij(i, i)) == 0.0) throw std::runtime_error("gmres: breakdown (zero diagonal in Hessenberg)");
        const cd yi = acc / Hij(i, i);
        y[i] = make_double2(yi.real(), yi.imag());
      }
      if (j > 0) {
        cuda_check(cudaMemcpyAsync(h, y.data(), sizeof(double2) * j, cudaMemcpyHostToDevice, s), "gmres H2D");
        K.axpys(V, n, j, h, 1.0, X);
      }
      const double rel = residual() / bnorm;
      I.residual = rel;
      if (rel <= tol) {
        I.converged = 1;
        done = true;
      }
    }
    I.iterations = total;
    I.residual = residual() / bnorm;  // linsolve.cpp:115-118
    if (I.residual <= tol) I.converged = 1;
    finish();
  });
}

}  // extern "C"
