// Host probe: can the CPU mirror the lower triangle of a column-major complex128
// matrix fast enough to halve the PCIe bytes of the one-shot symmetric path?
// Times a blocked transpose of the strictly-lower triangle from the upper one
// (N = 10242, cfg 2) with 1..T threads, next to a plain memcpy of the same bytes.
// build: g++ -O3 -march=native -fopenmp scripts/transpose_probe.cpp -o /tmp/tp
#include <omp.h>

#include <chrono>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

using cd = std::complex<double>;

int main(int argc, char** argv) {
  const long n = argc > 1 ? atol(argv[1]) : 10242;
  const int B = argc > 2 ? atoi(argv[2]) : 64;
  cd* A = static_cast<cd*>(aligned_alloc(64, n * n * sizeof(cd)));
  cd* C = static_cast<cd*>(aligned_alloc(64, n * n * sizeof(cd)));
#pragma omp parallel for schedule(static)
  for (long j = 0; j < n; ++j)
    for (long i = 0; i < n; ++i) {
      A[i + j * n] = i <= j ? cd(i, j) : cd(0, 0);
      C[i + j * n] = cd(1, 1);
    }
  printf("nproc %d\n", omp_get_num_procs());
  const double half = 0.5 * n * n * sizeof(cd);
  for (int nt : {1, 4, 8, 16, 32}) {
    if (nt > omp_get_num_procs()) break;
    double best = 1e9, bestc = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      auto t0 = std::chrono::steady_clock::now();
      // lower(i > j) = upper(j, i): tile (I, J) with I > J, each tile by one thread
      const long nb = (n + B - 1) / B;
#pragma omp parallel for num_threads(nt) schedule(dynamic, 4)
      for (long I = 0; I < nb; ++I)
        for (long J = 0; J <= I; ++J) {
          const long i1 = std::min(n, (I + 1) * B), j1 = std::min(n, (J + 1) * B);
          cd buf[128 * 128];  // tile through a local buffer: contiguous reads, contiguous writes
          const long bi = I * B, bj = J * B;
          for (long i = bi; i < i1; ++i)
            for (long j = bj; j < j1; ++j) buf[(j - bj) * B + (i - bi)] = A[j + i * n];
          for (long j = bj; j < j1; ++j)
            for (long i = std::max(bi, j + 1); i < i1; ++i) A[i + j * n] = buf[(j - bj) * B + (i - bi)];
        }
      auto t1 = std::chrono::steady_clock::now();
#pragma omp parallel for num_threads(nt) schedule(static)
      for (long j = 0; j < n / 2; ++j) memcpy(C + j * n, A + j * n, n * sizeof(cd));
      auto t2 = std::chrono::steady_clock::now();
      best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
      bestc = std::min(bestc, std::chrono::duration<double>(t2 - t1).count());
    }
    printf("threads %2d: mirror %.1f ms (%.1f GB/s of written bytes), memcpy of the same bytes %.1f ms\n", nt, 1e3 * best,
           half / best / 1e9, 1e3 * bestc);
  }
  long bad = 0;
  for (long j = 0; j < n; j += 97)
    for (long i = 0; i < n; i += 89)
      if (A[i + j * n] != cd(std::min(i, j), std::max(i, j))) ++bad;
  printf("check bad=%ld\n", bad);
  return 0;
}
