/*
 * galerk_b200 diagnostics — measurement helpers used by bench.py and the
 * profiling notes.  Not part of the reference-facing interface.
 */
#ifndef GALERK_B200_DIAG_H
#define GALERK_B200_DIAG_H

#include <stdint.h>

#include "galerk_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* FP64 pipe peak: a DFMA-only kernel (8 independent chains per thread, all
 * SMs).  Returns achieved GFLOP/s (2 flops per DFMA) over `iters` iterations,
 * timed with CUDA events on `stream`. */
gk_status gk_diag_fp64_peak(int64_t iters, double* gflops, gk_stream stream);

/* Sustained FP64 peak: the DFMA chains of gk_diag_fp64_peak plus a streaming
 * 16-byte store per 64 flops into `scratch` (device, >= 1 MB; sized above L2
 * so the stores reach HBM), launched back to back for about `seconds`.  This
 * is the clock the power cap allows under a DFMA + HBM-write load such as the
 * 107 GB cfg-4 assembly; gflops = DFMA flops / elapsed. */
gk_status gk_diag_fp64_sustained(double seconds, void* scratch, uint64_t scratch_bytes, double* gflops,
                                 double* elapsed_ms, gk_stream stream);

/* The canonical F_pair probe: the reference formula of
 * kernels.cpp:94-114 compiled with libdevice (sqrt, sin, cos, complex / real
 * division, r*r <= eps^2 mask) plus one complex x real accumulate, evaluated
 * for every (target, source) pair of n x n points (device SoA arrays).
 * ncu's FP64 instruction counters over this launch divided by n*n give F_pair.
 * out: device [n] complex accumulators. */
gk_status gk_diag_probe_pairs(int64_t n, const double* x, const double* y, const double* z, double k,
                              double eps, gk_cplx* out, gk_stream stream);

/* The same pair count through the production pair function (gk_math.cuh). */
gk_status gk_diag_fast_pairs(int64_t n, const double* x, const double* y, const double* z, double k,
                             double eps, gk_cplx* out, gk_stream stream);

/* The canonical F_analytic probe: the reference formula of
 * analytic_triangle_integrals (kernels.cpp:151-207, libdevice log / atan /
 * sqrt / division) for n calls, call i = triangle i % ntri (device [ntri*9]
 * vertex coordinates) against point i (device [n*3]); out: device [n*4].
 * ncu's FP64 instruction counters over the launch / n give F_analytic. */
gk_status gk_diag_probe_analytic(int64_t n, const double* tri, const double* pts, int64_t ntri, double* out,
                                 gk_stream stream);

/* Device math accuracy probe: out[i] = f(a[i], b[i]) for one scalar helper of
 * the kernels (gk_math.cuh), on device arrays; b may be NULL for unary f.
 *   GK_MATH_LOG_RATIO   log(a / b)            (near-field edge logs, K3)
 *   GK_MATH_ATAN2       atan2(a, b)           (solid angle, K3)
 *   GK_MATH_DIV         a / b, b > 0          (K3 reductions)
 *   GK_MATH_SIN_QUARTER sin(pi a / 2)         (phase of the pair kernel)
 *   GK_MATH_COS_QUARTER cos(pi a / 2)
 *   GK_MATH_RSQRT       1 / sqrt(a)           (1/r of every kernel) */
enum { GK_MATH_LOG_RATIO = 0, GK_MATH_ATAN2, GK_MATH_DIV, GK_MATH_SIN_QUARTER, GK_MATH_COS_QUARTER, GK_MATH_RSQRT };
gk_status gk_diag_math(int32_t fn, int64_t n, const double* a, const double* b, double* out, gk_stream stream);

/* Near-field pair list (element pairs in close_pairs order) and, after
 * gk_nearfield_compute (element-pair form), the number of accepted leaves of
 * the adaptive recursion per pair (accurate_adaptive, assembly.cpp:581-605):
 * compared pair by pair with the oracle it counts accept/split decision flips.
 * Host arrays of gk_nearfield_get_info's `pairs` entries; any may be NULL. */
typedef struct gk_nearfield gk_nearfield;
gk_status gk_diag_nearfield_pairs(const gk_nearfield* nf, int32_t* ex, int32_t* ey, int32_t* leaves);

/* Host-only dry run of gk_plan_create (no device needed): fills the plan
 * statistics (locations, tiles, evaluated vs unique pairs) so the tiling can
 * be inspected and tested on a CPU-only machine. */
gk_status gk_diag_plan_info(const gk_side* test, const gk_side* trial, const gk_kernel* kernel,
                            const gk_options* opts, gk_plan_info* info);

/* Host-only: the planner's location numbering of one side (twins merged, ids
 * in first-seen point order).  point_loc[npts] receives each point's location
 * id, xyz[3 * n_locations] (may be NULL) the location coordinates.  serial != 0
 * forces the one-thread path; the threaded, hash-sharded path used for large
 * sides must give the same ids (tests/test_host_cpu.py). */
gk_status gk_diag_location_ids(const gk_side* side, int32_t serial, int64_t* point_loc, int64_t* n_locations,
                               double* xyz);

#ifdef __cplusplus
}
#endif
#endif
