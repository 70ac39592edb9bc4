/*
 * galerk_b200 — C-ABI of the B200 (sm_100a) dense BEM hot path.
 *
 * This is the drop-in boundary under the reference's operator API
 * (/root/reference/proj/include/galerk/assembly.hpp).  Plain C types only: no
 * Eigen, no torch, no C++ in the signatures.  Each entry point names the
 * reference routine whose body it replaces:
 *
 *   gk_plan_create + gk_plan_assemble
 *       replace the x-chunk loop of bem_product (assembly.cpp:192-222):
 *       Kernel::evaluate_blocks (kernels.cpp:76-131) + the two sparse
 *       contractions (assembly.cpp:217-218) + scatter-to-DOF.
 *   gk_bem_dense
 *       one-shot host-in/host-out form of bem_product, as called by bem_dense
 *       (assembly.cpp:313-320) and radiation_dense (assembly.cpp:334-341).
 *   gk_matvec
 *       replaces Eigen::MatrixXcd * VectorXcd at the matvec call sites
 *       (tests/test_assembly.cpp:233,277; linsolve.hpp:20-23 from_matrix).
 *   gk_green_plan_* / gk_green_matvec
 *       matrix-free Green-kernel matvec with the evaluate_blocks semantics
 *       (distance mask, kernels.cpp:104-111) contracted with a weighted charge
 *       vector (make_point_side + bem_product, assembly.cpp:173-222).
 *   gk_evaluator_*
 *       replace GalerkinEvaluator::eval (assembly.cpp:240-291), the entry
 *       generator HMatrix::assemble / aca call (hmatrix.hpp:45-52), batched.
 *   gk_nearfield_*
 *       replace regularize (assembly.cpp:609-697) including close_pairs
 *       (:370-401), YContext gauss/exact (:447-544), accurate_cell /
 *       accurate_adaptive (:548-605) and analytic_triangle_integrals
 *       (kernels.cpp:151-207).
 *
 * Conventions
 *   - Matrices are column-major interleaved complex128 (gk_cplx), i.e. the
 *     storage of Eigen::MatrixXcd; `lda` is the leading dimension in elements.
 *   - Pointers documented "device" must be CUDA device (or managed) memory;
 *     "host" pointers may be pageable or pinned.
 *   - Every function returns gk_status; on failure gk_last_error() returns a
 *     thread-local message.  GK_EINVAL maps to std::invalid_argument and
 *     GK_ERUNTIME to std::runtime_error in the C++ wrapper, with the
 *     reference's messages (e.g. the memory cap message contains "tol").
 *   - There is no CPU fallback: without a usable CUDA device every compute
 *     entry point fails with GK_ECUDA.
 *   - Results are deterministic: no atomics whose ordering changes results.
 */
#ifndef GALERK_B200_H
#define GALERK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t gk_status;
#define GK_OK 0
#define GK_EINVAL 1   /* std::invalid_argument */
#define GK_ERUNTIME 2 /* std::runtime_error    */
#define GK_ECUDA 3    /* CUDA failure / no device */
#define GK_ENOMEM 4   /* device allocation failed */

typedef struct gk_cplx {
  double re, im;
} gk_cplx;

typedef void* gk_stream; /* cudaStream_t; NULL = legacy default stream */

/* One side of the double integral (reference BemSide, assembly.cpp:135-171):
 * quadrature points of a triangle mesh (quadrature.cpp:167-189), their weights
 * (rule weight x element measure), and the element -> dof map with the basis
 * values at the rule's barycentric points (femspace.cpp:460-494).
 * Point e*g+q belongs to element e (pinned by test_quadrature.cpp:160-166).
 * All pointers are host memory. */
typedef struct gk_side {
  int64_t npts;              /* M = nelem * g                                   */
  const double* x;           /* [M] point coordinates, SoA                      */
  const double* y;           /* [M]                                             */
  const double* z;           /* [M]                                             */
  const double* w;           /* [M] quadrature weights                          */
  int32_t g;                 /* points per element                              */
  int64_t nelem;             /* elements                                        */
  int32_t nloc;              /* local dofs per element (P0: 1, P1: 3)           */
  const int32_t* elem_dofs;  /* [nelem*nloc] free-dof index, -1 = constrained   */
  const double* basis;       /* [g*nloc] basis value of local dof l at point q  */
  int64_t nfree;             /* number of free dofs (matrix dimension)          */
} gk_side;

#define GK_LAPLACE 0   /* "[1/r]"          : 1/r            (k forced to 0)  */
#define GK_HELMHOLTZ 1 /* "[exp(ikr)/r]"   : e^{ikr}/r                       */
typedef struct gk_kernel {
  int32_t kind;       /* GK_LAPLACE / GK_HELMHOLTZ; no 1/(4 pi) (kernels.hpp:17) */
  int32_t components; /* must be 1 (scalar); 3 = grady kernels -> GK_EINVAL      */
  double k;           /* wavenumber                                             */
} gk_kernel;

typedef struct gk_options {
  uint64_t memory_cap_bytes; /* BemOptions::memory_cap_bytes (assembly.hpp:28)   */
  int64_t chunk;             /* BemOptions::chunk (enters the cap formula only)  */
  int32_t symmetric;         /* -1 auto-detect identical sides, 0 off, 1 force   */
  int32_t reserved;
} gk_options;

/* Default options: cap 8e9 bytes, chunk 1024, symmetric auto. */
void gk_options_default(gk_options* opts);

/* ---- dense assembly ------------------------------------------------------ */
typedef struct gk_plan gk_plan;

typedef struct gk_plan_info {
  int64_t rows, cols;           /* N_test, N_trial                               */
  int64_t x_locations;          /* unique x quadrature locations (twins merged)  */
  int64_t y_locations;
  int64_t pairs_reference;      /* M_x * M_y (reference pair evaluations)        */
  int64_t pairs_unique;         /* unique location pairs (symmetry-halved if on) */
  int64_t pairs_evaluated;      /* location pairs the kernel evaluates (halo)    */
  int64_t tiles;                /* CTA tiles launched (after symmetric skip)     */
  int64_t masked_tiles;         /* of which apply the r^2 <= eps^2 mask          */
  int32_t symmetric;
  double eps;                   /* singular_guard_radius (kernels.cpp:14-19)     */
  uint64_t device_bytes;        /* plan tables resident on the device            */
  double x_halo;                /* sum over x blocks of their locations / U_x    */
  double y_halo;                /* sum over y blocks of their records / U_y      */
  int32_t natural_order;        /* 1 if the dof order kept the input numbering   */
  int64_t x_blocks, y_blocks;   /* tile rows / columns of blocks                 */
} gk_plan_info;

/* Builds the location/dof tables (host) and uploads them (device).  Applies
 * the reference's memory-cap check and raises its "tol" message. */
gk_status gk_plan_create(const gk_side* test, const gk_side* trial, const gk_kernel* kernel,
                         const gk_options* opts, gk_plan** out);
gk_status gk_plan_get_info(const gk_plan* plan, gk_plan_info* info);
/* A: device, N_test x N_trial, column-major, lda >= N_test.  Overwrites A. */
gk_status gk_plan_assemble(gk_plan* plan, gk_cplx* A, int64_t lda, gk_stream stream);
/* Re-targets a plan to another wavenumber: the tables depend only on the
 * geometry, so one plan serves a frequency sweep (gk_plan_set_wavenumber, then
 * gk_plan_assemble, per k).  The kernel kind is kept: a "[1/r]" plan stays
 * k = 0 (kernels.cpp:47-49); k must be finite. */
gk_status gk_plan_set_wavenumber(gk_plan* plan, double k);
/* Number of kernel launches gk_plan_assemble issues (for launch accounting). */
int32_t gk_plan_launches(const gk_plan* plan);
gk_status gk_plan_destroy(gk_plan* plan);

/* One-shot drop-in for bem_product: host sides in, host matrix out. */
gk_status gk_bem_dense(const gk_side* test, const gk_side* trial, const gk_kernel* kernel,
                       const gk_options* opts, gk_cplx* A_host, int64_t lda);

/* ---- stored-matrix matvec ------------------------------------------------ */
/* y = A x; A, x, y device.  Deterministic split-K with a fixed-order reduce. */
gk_status gk_matvec(const gk_cplx* A, int64_t rows, int64_t cols, int64_t lda, const gk_cplx* x,
                    gk_cplx* y, gk_stream stream);
int32_t gk_matvec_launches(int64_t rows, int64_t cols);
/* Y = A X for nrhs right-hand sides in one pass over A (X, Y column-major with
   leading dimensions ldx, ldy >= rows/cols; device).  Replaces nrhs
   MatrixXcd * VectorXcd products with independent vectors (the matvec sites
   test_assembly.cpp:233,277 repeated; Eigen's MatrixXcd * MatrixXcd).  Column r
   of Y is computed in a fixed order that does not depend on the other columns. */
gk_status gk_matvec_multi(const gk_cplx* A, int64_t rows, int64_t cols, int64_t lda, const gk_cplx* X,
                          int64_t ldx, gk_cplx* Y, int64_t ldy, int32_t nrhs, gk_stream stream);
int32_t gk_matvec_multi_launches(int64_t rows, int64_t cols, int32_t nrhs);

/* ---- matrix-free Green matvec -------------------------------------------- */
typedef struct gk_green_plan gk_green_plan;
#define GK_FP64 0
#define GK_FP32 1
/* targets/sources: host SoA point arrays.  y_i = sum_j [r_ij > eps] G(x_i,y_j) q_j
 * with eps = singular_guard_radius(targets, sources); twins (bit-identical
 * points) are merged on both sides. */
gk_status gk_green_plan_create(int64_t ntargets, const double* tx, const double* ty,
                               const double* tz, int64_t nsources, const double* sx,
                               const double* sy, const double* sz, const gk_kernel* kernel,
                               gk_green_plan** out);
/* q: device [nsources] charges (already weighted), y: device [ntargets]. */
gk_status gk_green_matvec(gk_green_plan* plan, const gk_cplx* q, gk_cplx* y, int32_t precision,
                          gk_stream stream);
gk_status gk_green_plan_get_info(const gk_green_plan* plan, int64_t* unique_targets,
                                 int64_t* unique_sources, double* eps);
/* 1 if targets == sources and the symmetric path (each unordered pair once) is used. */
int32_t gk_green_plan_is_symmetric(const gk_green_plan* plan);
/* Kernel launches one gk_green_matvec issues (for launch accounting). */
int32_t gk_green_plan_launches(const gk_green_plan* plan, int32_t precision);
gk_status gk_green_plan_destroy(gk_green_plan* plan);

/* ---- near-field singular correction (regularize) -------------------------- */
typedef struct gk_nearfield gk_nearfield;
#define GK_NEAR_REF 0    /* |c_x - c_y| <= 3 max(R_x, R_y)  (assembly.cpp:394-396) */
#define GK_NEAR_2HBAR 1  /* |c_x - c_y| <= 2 hbar           (BASELINE cfg 3 text)  */
/* Mesh-level description (the correction integrates over the triangles, not
 * only at quadrature points).  vertices: host [nv*3] row-major xyz;
 * elements: host [ne*3]; family: 0 = P0, 1 = P1; g = domain rule points. */
typedef struct gk_mesh_side {
  int64_t nv;
  const double* vertices;
  int64_t ne;
  const int32_t* elements;
  int32_t family;
  int32_t g;
  int64_t nfree;
} gk_mesh_side;
gk_status gk_nearfield_create(const gk_mesh_side* test, const gk_mesh_side* trial,
                              const char* singular_name, int32_t near_rule, double hbar,
                              gk_nearfield** out);
/* Collocation form, replacing regularize_radiation (assembly.cpp:699-750):
 * rows are the given points (host [npts*3] xyz), pairs are (point, element)
 * with |c_y - x| <= 3 R_y.  Same compute/apply/triplets calls. */
gk_status gk_nearfield_create_points(int64_t npts, const double* points, const gk_mesh_side* trial,
                                     const char* singular_name, gk_nearfield** out);
/* Number of near element pairs and of summed (row, col) entries. */
gk_status gk_nearfield_get_info(const gk_nearfield* nf, int64_t* pairs, int64_t* entries);
/* Evaluate the correction on the device (one warp per near pair). */
gk_status gk_nearfield_compute(gk_nearfield* nf, gk_stream stream);
/* A += correction, in place on a device matrix (deterministic, fixed order). */
gk_status gk_nearfield_apply(gk_nearfield* nf, gk_cplx* A, int64_t lda, gk_stream stream);
/* Copy the summed correction to host triplets (setFromTriplets semantics,
 * col-major sorted); arrays sized by gk_nearfield_get_info's `entries`. */
gk_status gk_nearfield_triplets(gk_nearfield* nf, int32_t* rows, int32_t* cols, double* vals);
/* Analytic-integral calls the adaptive recursion made in the last compute. */
gk_status gk_nearfield_stats(const gk_nearfield* nf, int64_t* analytic_calls,
                             int64_t depth_hist[8]);
gk_status gk_nearfield_destroy(gk_nearfield* nf);

/* ---- block evaluation (entry generator of the compressed / H-matrix path) --- */
/* Replaces GalerkinEvaluator (assembly.cpp:225-299), the BlockEvaluator
 * plugin that HMatrix::assemble (hmatrix.hpp:45-52, hmatrix.cpp:811-866)
 * calls for ACA row/column panels and dense leaves.  eps is taken from the
 * full sides (assembly.cpp:231) and the distance mask is always on. */
typedef struct gk_evaluator gk_evaluator;
gk_status gk_evaluator_create(const gk_side* test, const gk_side* trial, const gk_kernel* kernel,
                              gk_evaluator** out);
gk_status gk_evaluator_dims(const gk_evaluator* ev, int64_t* rows, int64_t* cols);
/* One BlockEvaluator::eval(row_ids, col_ids, out) request.  All host memory:
 * ids are free-dof indices (duplicates allowed), out is nrows x ncols
 * column-major with leading dimension ldo >= nrows. */
typedef struct gk_block {
  int32_t nrows, ncols;
  const int32_t* row_ids;
  const int32_t* col_ids;
  gk_cplx* out;
  int64_t ldo;
} gk_block;
/* Evaluates a batch of blocks with one copy in, one launch and one copy out
 * (returns after the results are in the callers' buffers). */
gk_status gk_evaluator_eval(gk_evaluator* ev, int32_t nblocks, const gk_block* blocks, gk_stream stream);
gk_status gk_evaluator_destroy(gk_evaluator* ev);

/* Kernel::evaluate_blocks (kernels.hpp:37-39, kernels.cpp:76-131) as one
 * device panel: out(i, j) = G(x_i, y_j) for the built-in scalar kernels, no
 * 1/(4 pi), column-major nx x ny (ldo >= nx), HOST arrays (X: nx x 3 and
 * Y: ny x 3 row-major xyz, out).  mask = 1: pairs with r^2 <= eps_r^2 give 0.
 * mask = 0: a pair with r^2 <= eps_r^2 fails with GK_ERUNTIME and the
 * reference's message "kernel evaluation at singular point pair (i,j), r=..."
 * naming the first such pair in the reference's loop order. */
gk_status gk_evaluate_blocks(int64_t nx, const double* X, int64_t ny, const double* Y, const gk_kernel* kernel,
                             double eps_r, int32_t mask, gk_cplx* out, int64_t ldo, gk_stream stream);

/* ---- solve step on the device-resident matrix ------------------------------ */
/* Partial-pivot LU in place, replacing Eigen's partialPivLu()
 * (test_assembly.cpp:227).  A: device n x n column-major; ipiv: device
 * int64[n]; singular_at (host, optional): 0, or the 1-based index of an
 * exactly zero pivot (the factorisation still completes, as Eigen's does). */
gk_status gk_lu_factor(gk_cplx* A, int64_t n, int64_t lda, int64_t* ipiv, int64_t* singular_at, gk_stream stream);
/* B <- A^{-1} B with the factors of gk_lu_factor; B: device n x nrhs. */
gk_status gk_lu_solve(const gk_cplx* LU, int64_t n, int64_t lda, const int64_t* ipiv, gk_cplx* B, int64_t ldb,
                      int64_t nrhs, gk_stream stream);
/* SolveInfo (linsolve.hpp:26-31); history_len entries of the relative
 * residual history were written if a history array was given. */
typedef struct gk_solve_info {
  int32_t converged;
  int32_t iterations;
  double residual;
  int32_t history_len;
  int32_t reserved;
} gk_solve_info;
/* Restarted GMRES (linsolve.cpp:19-121) with the stored matrix as operator
 * (LinearOperator::from_matrix, linsolve.hpp:20-23), no preconditioner.
 * A, b, x: device; x is overwritten with the solution (start 0).
 * history: host double[maxit] or NULL.  tol <= 0 -> GK_EINVAL "gmres: tol
 * must be positive" (linsolve.cpp:24). */
gk_status gk_gmres(const gk_cplx* A, int64_t n, int64_t lda, const gk_cplx* b, gk_cplx* x, double tol,
                   int32_t restart, int32_t maxit, gk_solve_info* info, double* history, gk_stream stream);

/* ---- device memory helpers for callers without a CUDA allocator ----------- */
gk_status gk_device_alloc(uint64_t bytes, void** ptr);
gk_status gk_device_free(void* ptr);
gk_status gk_copy_to_device(void* dst, const void* src, uint64_t bytes, gk_stream stream);
gk_status gk_copy_to_host(void* dst, const void* src, uint64_t bytes, gk_stream stream);
gk_status gk_stream_synchronize(gk_stream stream);

const char* gk_last_error(void);
const char* gk_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GALERK_B200_H */
