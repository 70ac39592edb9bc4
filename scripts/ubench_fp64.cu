// Microbenchmarks: FP64 dependent latency and throughput vs warps/SM on B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat_dfma(double* out, long long* cyc, int n) {
  double a = out[0], b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  out[1] = a; cyc[0] = t1 - t0;
}
__global__ void lat_dmul(double* out, long long* cyc, int n) {
  double a = out[0], b = 1.0000001;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = a * b;
  long long t1 = clock64();
  out[1] = a; cyc[0] = t1 - t0;
}
__global__ void lat_rsq(double* out, long long* cyc, int n) {
  double a = out[0] + 2.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a)); a = y + 2.0; }
  long long t1 = clock64();
  out[1] = a; cyc[0] = t1 - t0;
}
template <int CH>
__global__ void thr_dfma(double* out, int n) {
  double a[CH];
  for (int k = 0; k < CH; ++k) a[k] = threadIdx.x + k;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < CH; ++k) a[k] = fma(a[k], 0.999999, 1e-9);
  double s = 0; for (int k = 0; k < CH; ++k) s += a[k];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 64); cudaMalloc(&c, 64);
  double h[2] = {1.0, 0}; cudaMemcpy(d, h, 16, cudaMemcpyHostToDevice);
  long long cy; const int n = 4096;
  lat_dfma<<<1,1>>>(d, c, n); lat_dfma<<<1,1>>>(d, c, n); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); printf("DFMA dependent latency: %.2f cyc\n", (double)cy / n);
  lat_dmul<<<1,1>>>(d, c, n); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); printf("DMUL dependent latency: %.2f cyc\n", (double)cy / n);
  lat_rsq<<<1,1>>>(d, c, n); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); printf("MUFU.RSQ64H+DADD dependent latency: %.2f cyc\n", (double)cy / n);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps = 1; warps <= 16; warps *= 2) {
    for (int ch : {1, 2, 4, 8}) {
      int iters = 20000;
      cudaEventRecord(e0);
      if (ch == 1) thr_dfma<1><<<sms, 32 * warps>>>(d, iters);
      if (ch == 2) thr_dfma<2><<<sms, 32 * warps>>>(d, iters);
      if (ch == 4) thr_dfma<4><<<sms, 32 * warps>>>(d, iters);
      if (ch == 8) thr_dfma<8><<<sms, 32 * warps>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)sms * 32 * warps * iters * ch;
      printf("warps/SM %2d chains %d: %.2f Tinstr/s (peak at 1.965GHz = %.2f)\n", warps, ch, ops / ms / 1e9, sms * 64 * 1.965e9 / 1e12);
    }
  }
  return 0;
}
