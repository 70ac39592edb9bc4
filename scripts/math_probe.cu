// Probe: is one Newton step on MUFU.RCP64H enough for div_fast (K3)?
// Prints the max ulp error of a/b (b > 0) for the production div_fast and for
// a variant with one Newton step + the residual correction, against host long
// double, plus the raw relative error of rcp.approx.ftz.f64.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1804_00995_b200/csrc scripts/math_probe.cu -o /tmp/mp
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "gk_math.cuh"

__device__ __forceinline__ double div_one_newton(double d, double sg) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(sg));
  y = fma(y, fma(-sg, y, 1.0), y);
  const double q0 = d * y;
  return fma(fma(-sg, q0, d), y, q0);
}

__global__ void k(int n, const double* a, const double* b, double* o0, double* o1, double* o2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  o0[i] = gk::div_fast(a[i], b[i]);
  o1[i] = div_one_newton(a[i], b[i]);
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(b[i]));
  o2[i] = y;
}

int main() {
  const int n = 1 << 22;
  std::mt19937_64 g(7);
  std::uniform_real_distribution<double> u(-1, 1), e(-20, 20);
  std::vector<double> a(n), b(n), r0(n), r1(n), r2(n);
  for (int i = 0; i < n; ++i) {
    a[i] = u(g) * std::exp(e(g));
    b[i] = std::exp(e(g)) * (1.0 + 0.5 * u(g));
  }
  double *da, *db, *d0, *d1, *d2;
  cudaMalloc(&da, n * 8);
  cudaMalloc(&db, n * 8);
  cudaMalloc(&d0, n * 8);
  cudaMalloc(&d1, n * 8);
  cudaMalloc(&d2, n * 8);
  cudaMemcpy(da, a.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), n * 8, cudaMemcpyHostToDevice);
  k<<<(n + 255) / 256, 256>>>(n, da, db, d0, d1, d2);
  cudaMemcpy(r0.data(), d0, n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(r1.data(), d1, n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(r2.data(), d2, n * 8, cudaMemcpyDeviceToHost);
  double m0 = 0, m1 = 0, mr = 0;
  for (int i = 0; i < n; ++i) {
    const long double ex = (long double)a[i] / (long double)b[i];
    const double ulp = std::nextafter(std::fabs((double)ex), INFINITY) - std::fabs((double)ex);
    m0 = std::max(m0, (double)(std::fabs((long double)r0[i] - ex) / ulp));
    m1 = std::max(m1, (double)(std::fabs((long double)r1[i] - ex) / ulp));
    mr = std::max(mr, (double)std::fabs((long double)r2[i] * (long double)b[i] - 1.0L));
  }
  printf("div_fast (2 Newton) max %.3f ulp; 1 Newton max %.3f ulp; rcp.approx.f64 max rel err %.3e (2^%.1f)\n", m0, m1,
         mr, std::log2(mr));
  return 0;
}
