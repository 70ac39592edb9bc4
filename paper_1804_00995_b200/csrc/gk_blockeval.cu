// K6: batched block evaluation — the entry generator of the compressed
// (H-matrix / ACA) path.
//
// Replaces GalerkinEvaluator::eval (assembly.cpp:240-291), the
// BlockEvaluator plugin of HMatrix::assemble (hmatrix.hpp:45-52,
// hmatrix.cpp:811-866): out(a, b) = sum_x lt(a, x) sum_y K(x, y) ru(y, b)
// over the quadrature points supporting row dof a and column dof b, with the
// distance mask on (mask=true, eps from the FULL sides as in the evaluator's
// constructor, assembly.cpp:227-233).
//
// A batch of blocks (ACA row/column panels, dense leaves) becomes one
// host->device copy of the index lists, one kernel launch over all entries
// and one device->host copy.  One thread per entry: it walks the twin-merged
// x locations of its row dof (outer) and y locations of its column dof
// (inner), the reference's lt * (K * ru) nesting; twins give bit-identical
// kernel values, so merging them only reorders additions.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "gk_internal.hpp"
#include "gk_math.cuh"

using namespace gk;

namespace gk {
namespace {

struct BlkMeta {
  long long e0;    // first entry of the block in the packed output
  int32_t r0, c0;  // offsets into the packed row / column id lists
  int32_t nr, nc;
};
static_assert(sizeof(BlkMeta) == 24, "BlkMeta layout");

struct SideDev {  // per dof: twin-merged support locations with summed w*phi
  DevBuf start, loc, coef, x, y, z;
  int64_t nfree = 0;
};

struct EvalArgs {
  const BlkMeta* meta;
  int32_t nblocks;
  long long entries;
  const int32_t* ids;  // row ids then column ids
  const int64_t* xs;
  const int32_t* xl;
  const double* xc;
  const double *xx, *xy, *xz;
  const int64_t* ys;
  const int32_t* yl;
  const double* yc;
  const double *yx, *yy, *yz;
  double eps2, kappa;
  double2* out;
};

template <bool HELM>
__global__ void __launch_bounds__(256) k_block_eval(const EvalArgs a) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= a.entries) return;
  int lo = 0, hi = a.nblocks - 1;  // last block with e0 <= e
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.meta[mid].e0 <= e)
      lo = mid;
    else
      hi = mid - 1;
  }
  const BlkMeta m = a.meta[lo];
  const long long le = e - m.e0;
  const int i = (int)(le % m.nr), j = (int)(le / m.nr);  // column-major: lanes along rows
  const int row = a.ids[m.r0 + i], col = a.ids[m.c0 + j];
  const int64_t y0 = a.ys[col], y1 = a.ys[col + 1];
  double re = 0.0, im = 0.0;
  for (int64_t p = a.xs[row]; p < a.xs[row + 1]; ++p) {
    const int32_t u = a.xl[p];
    const double ux = a.xx[u], uy = a.xy[u], uz = a.xz[u];
    double sr = 0.0, si = 0.0;
    for (int64_t q = y0; q < y1; ++q) {
      const int32_t v = a.yl[q];
      const c64 g = green<HELM>(ux - a.yx[v], uy - a.yy[v], uz - a.yz[v], a.eps2, a.kappa);
      sr = fma(a.yc[q], g.re, sr);
      si = fma(a.yc[q], g.im, si);
    }
    re = fma(a.xc[p], sr, re);
    im = fma(a.xc[p], si, im);
  }
  a.out[e] = make_double2(re, im);
}

// Kernel::evaluate_blocks (kernels.cpp:76-131) as a panel: out(i, j) =
// G(x_i, y_j), column-major nx x ny, one thread per entry (lanes along i).
// mask = 1: pairs with r^2 <= eps^2 are 0.  mask = 0: the reference raises for
// the first such pair in its loop order (j outer, i inner = column-major), so
// the smallest linear index i + j*nx of a singular pair is kept (atomicMin).
template <bool HELM>
__global__ void __launch_bounds__(256) k_panel(long long nx, long long ny, const double* __restrict__ X,
                                               const double* __restrict__ Y, double eps2, double kappa, int mask,
                                               double2* __restrict__ out, unsigned long long* first_singular) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nx * ny) return;
  const long long i = e % nx, j = e / nx;
  const double dx = X[i] - Y[j], dy = X[nx + i] - Y[ny + j], dz = X[2 * nx + i] - Y[2 * ny + j];
  double cs[1], sn[1], rinv[1], ddx[1] = {dx}, ddy[1] = {dy}, ddz[1] = {dz};
  green_parts_n<HELM, 1, true>(ddx, ddy, ddz, eps2, kappa, cs, sn, rinv);
  if (!mask && rinv[0] == 0.0) atomicMin(first_singular, (unsigned long long)e);
  out[e] = HELM ? make_double2(cs[0] * rinv[0], sn[0] * rinv[0]) : make_double2(rinv[0], 0.0);
}

void upload_side(SideDev& D, const Locations& L) {
  // per ORIGINAL dof d: the permuted dof's (location, coef) list
  const int64_t n = L.nfree;
  std::vector<int64_t> start(n + 1, 0);
  for (int64_t d = 0; d < n; ++d) {
    const int32_t p = L.iperm[d];
    start[d + 1] = start[d] + (L.dstart[p + 1] - L.dstart[p]);
  }
  std::vector<int32_t> loc(start[n]);
  std::vector<double> coef(start[n]);
  for (int64_t d = 0; d < n; ++d) {
    const int32_t p = L.iperm[d];
    for (int64_t s = L.dstart[p], k = start[d]; s < L.dstart[p + 1]; ++s, ++k) {
      loc[k] = L.dloc[s];
      coef[k] = L.dcoef[s];
    }
  }
  D.start.upload(start);
  D.loc.upload(loc);
  D.coef.upload(coef);
  D.x.upload(L.x);
  D.y.upload(L.y);
  D.z.upload(L.z);
  D.nfree = n;
}

}  // namespace
}  // namespace gk

struct gk_evaluator {
  SideDev X, Y;
  bool helmholtz = false;
  double eps = 0.0, k = 0.0;
  // batch staging (grown on demand): pinned host + device
  void* h_in = nullptr;
  size_t h_in_bytes = 0;
  void* h_out = nullptr;
  size_t h_out_bytes = 0;
  DevBuf d_in, d_out;
  ~gk_evaluator() {
    if (h_in) cudaFreeHost(h_in);
    if (h_out) cudaFreeHost(h_out);
  }
};

namespace {
void grow_pinned(void*& p, size_t& have, size_t need) {
  if (need <= have) return;
  if (p) cudaFreeHost(p);
  p = nullptr;
  have = 0;
  const size_t n = std::max<size_t>(need, 2 * have);
  if (cudaMallocHost(&p, n) != cudaSuccess) {
    cudaGetLastError();
    throw NoMemError("pinned host allocation of " + std::to_string(n) + " bytes failed");
  }
  have = n;
}
void grow_dev(DevBuf& b, size_t need) {
  if (need > b.bytes) b.alloc(std::max<size_t>(need, 2 * b.bytes));
}
}  // namespace

extern "C" {

gk_status gk_evaluator_create(const gk_side* test, const gk_side* trial, const gk_kernel* kernel,
                              gk_evaluator** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("gk_evaluator_create: null output");
    *out = nullptr;
    if (!test || !trial) throw std::invalid_argument("gk_evaluator_create: null side");
    if (!kernel) throw std::invalid_argument("gk_evaluator_create: null kernel");
    if (kernel->components != 1)
      throw std::invalid_argument("assembly: incompatible operand components (1," +
                                  std::to_string(kernel->components) + ",1)");
    if (kernel->kind != GK_LAPLACE && kernel->kind != GK_HELMHOLTZ)
      throw std::invalid_argument("gk_evaluator_create: only the built-in scalar Green kernels run on the GPU path");
    require_device();
    auto E = std::make_unique<gk_evaluator>();
    E->helmholtz = kernel->kind == GK_HELMHOLTZ && kernel->k != 0.0;
    E->k = kernel->kind == GK_LAPLACE ? 0.0 : kernel->k;  // kernels.cpp:47-49
    E->eps = guard_radius(*test, *trial);                // assembly.cpp:231
    const Locations X = build_locations(*test, "evaluator(test)");
    const Locations Y = build_locations(*trial, "evaluator(trial)");
    upload_side(E->X, X);
    upload_side(E->Y, Y);
    *out = E.release();
  });
}

gk_status gk_evaluator_dims(const gk_evaluator* E, int64_t* rows, int64_t* cols) {
  return guard([&] {
    if (!E) throw std::invalid_argument("gk_evaluator_dims: null handle");
    if (rows) *rows = E->X.nfree;
    if (cols) *cols = E->Y.nfree;
  });
}

gk_status gk_evaluator_eval(gk_evaluator* E, int32_t nblocks, const gk_block* blocks, gk_stream stream) {
  return guard([&] {
    if (!E) throw std::invalid_argument("gk_evaluator_eval: null handle");
    if (nblocks < 0 || (nblocks > 0 && !blocks)) throw std::invalid_argument("gk_evaluator_eval: bad block list");
    // pack: metadata, then row ids and column ids of every block
    std::vector<BlkMeta> meta;
    meta.reserve(nblocks);
    long long entries = 0;
    int64_t nids = 0;
    for (int32_t b = 0; b < nblocks; ++b) {
      const gk_block& B = blocks[b];
      if (B.nrows < 0 || B.ncols < 0) throw std::invalid_argument("gk_evaluator_eval: negative block size");
      if ((B.nrows > 0 && !B.row_ids) || (B.ncols > 0 && !B.col_ids))
        throw std::invalid_argument("gk_evaluator_eval: null index list");
      if (B.nrows > 0 && B.ncols > 0 && (!B.out || B.ldo < B.nrows))
        throw std::invalid_argument("gk_evaluator_eval: bad output (null or ldo < nrows)");
      for (int32_t i = 0; i < B.nrows; ++i)
        if (B.row_ids[i] < 0 || B.row_ids[i] >= E->X.nfree)
          throw std::invalid_argument("gk_evaluator_eval: row index out of range");
      for (int32_t j = 0; j < B.ncols; ++j)
        if (B.col_ids[j] < 0 || B.col_ids[j] >= E->Y.nfree)
          throw std::invalid_argument("gk_evaluator_eval: column index out of range");
      if ((long long)B.nrows * B.ncols == 0) continue;
      BlkMeta m;
      m.e0 = entries;
      m.r0 = (int32_t)nids;
      m.c0 = (int32_t)(nids + B.nrows);
      m.nr = B.nrows;
      m.nc = B.ncols;
      meta.push_back(m);
      entries += (long long)B.nrows * B.ncols;
      nids += B.nrows + B.ncols;
      if (nids > INT32_MAX) throw std::invalid_argument("gk_evaluator_eval: batch too large");
    }
    if (meta.empty()) return;
    const size_t meta_bytes = meta.size() * sizeof(BlkMeta);
    const size_t in_bytes = meta_bytes + (size_t)nids * sizeof(int32_t);
    const size_t out_bytes = (size_t)entries * sizeof(double2);
    grow_pinned(E->h_in, E->h_in_bytes, in_bytes);
    grow_pinned(E->h_out, E->h_out_bytes, out_bytes);
    grow_dev(E->d_in, in_bytes);
    grow_dev(E->d_out, out_bytes);
    char* hin = static_cast<char*>(E->h_in);
    std::memcpy(hin, meta.data(), meta_bytes);
    int32_t* ids = reinterpret_cast<int32_t*>(hin + meta_bytes);
    for (int32_t b = 0, k = 0; b < nblocks; ++b) {
      const gk_block& B = blocks[b];
      if ((long long)B.nrows * B.ncols == 0) continue;
      std::memcpy(ids + meta[k].r0, B.row_ids, sizeof(int32_t) * B.nrows);
      std::memcpy(ids + meta[k].c0, B.col_ids, sizeof(int32_t) * B.ncols);
      ++k;
    }
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    cuda_check(cudaMemcpyAsync(E->d_in.p, E->h_in, in_bytes, cudaMemcpyHostToDevice, s), "evaluator H2D");
    EvalArgs a;
    a.meta = E->d_in.as<BlkMeta>();
    a.nblocks = (int32_t)meta.size();
    a.entries = entries;
    a.ids = reinterpret_cast<const int32_t*>(static_cast<const char*>(E->d_in.p) + meta_bytes);
    a.xs = E->X.start.as<int64_t>();
    a.xl = E->X.loc.as<int32_t>();
    a.xc = E->X.coef.as<double>();
    a.xx = E->X.x.as<double>();
    a.xy = E->X.y.as<double>();
    a.xz = E->X.z.as<double>();
    a.ys = E->Y.start.as<int64_t>();
    a.yl = E->Y.loc.as<int32_t>();
    a.yc = E->Y.coef.as<double>();
    a.yx = E->Y.x.as<double>();
    a.yy = E->Y.y.as<double>();
    a.yz = E->Y.z.as<double>();
    a.eps2 = E->eps * E->eps;
    a.kappa = 2.0 * E->k / M_PI;
    a.out = E->d_out.as<double2>();
    const unsigned grid = (unsigned)((entries + 255) / 256);
    if (E->helmholtz)
      k_block_eval<true><<<grid, 256, 0, s>>>(a);
    else
      k_block_eval<false><<<grid, 256, 0, s>>>(a);
    cuda_check(cudaGetLastError(), "k_block_eval launch");
    cuda_check(cudaMemcpyAsync(E->h_out, E->d_out.p, out_bytes, cudaMemcpyDeviceToHost, s), "evaluator D2H");
    cuda_check(cudaStreamSynchronize(s), "evaluator sync");
    const double2* ho = static_cast<const double2*>(E->h_out);
    for (int32_t b = 0, k = 0; b < nblocks; ++b) {
      const gk_block& B = blocks[b];
      if ((long long)B.nrows * B.ncols == 0) continue;
      const double2* src = ho + meta[k].e0;
      for (int32_t j = 0; j < B.ncols; ++j)
        std::memcpy(B.out + (int64_t)j * B.ldo, src + (int64_t)j * B.nrows, sizeof(double2) * B.nrows);
      ++k;
    }
  });
}

gk_status gk_evaluate_blocks(int64_t nx, const double* X, int64_t ny, const double* Y, const gk_kernel* kernel,
                             double eps_r, int32_t mask, gk_cplx* out, int64_t ldo, gk_stream stream) {
  return guard([&] {
    if (!kernel) throw std::invalid_argument("evaluate_blocks: null kernel");
    if (kernel->components != 1)
      throw std::invalid_argument("assembly: incompatible operand components (1," + std::to_string(kernel->components) +
                                  ",1)");
    if (kernel->kind != GK_LAPLACE && kernel->kind != GK_HELMHOLTZ)
      throw std::invalid_argument("evaluate_blocks: only the built-in scalar Green kernels run on the GPU path");
    if (nx < 0 || ny < 0 || (nx > 0 && !X) || (ny > 0 && !Y)) throw std::invalid_argument("evaluate_blocks: bad points");
    if (nx == 0 || ny == 0) return;
    if (!out || ldo < nx) throw std::invalid_argument("evaluate_blocks: bad output (null or ldo < nx)");
    require_device();
    const double k = kernel->kind == GK_LAPLACE ? 0.0 : kernel->k;  // kernels.cpp:47-49
    const bool helm = k != 0.0;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    // SoA point tables (host xyz rows -> device x | y | z)
    std::vector<double> soa(3 * (size_t)(nx + ny));
    for (int64_t i = 0; i < nx; ++i)
      for (int c = 0; c < 3; ++c) soa[c * nx + i] = X[3 * i + c];
    for (int64_t j = 0; j < ny; ++j)
      for (int c = 0; c < 3; ++c) soa[3 * nx + c * ny + j] = Y[3 * j + c];
    DevBuf pts, dout, flag;
    pts.upload(soa.data(), soa.size() * sizeof(double));
    dout.alloc(sizeof(double2) * (size_t)(nx * ny));
    const unsigned long long none = ~0ull;
    flag.upload(&none, sizeof(none));
    const long long n = nx * ny;
    const unsigned grid = (unsigned)((n + 255) / 256);
    auto launch = [&](auto kern) {
      kern<<<grid, 256, 0, s>>>(nx, ny, pts.as<double>(), pts.as<double>() + 3 * nx, eps_r * eps_r, 2.0 * k / M_PI,
                                mask ? 1 : 0, dout.as<double2>(), flag.as<unsigned long long>());
    };
    if (helm)
      launch(k_panel<true>);
    else
      launch(k_panel<false>);
    cuda_check(cudaGetLastError(), "k_panel launch");
    unsigned long long first = none;
    cuda_check(cudaMemcpyAsync(&first, flag.p, sizeof(first), cudaMemcpyDeviceToHost, s), "panel flag");
    cuda_check(cudaStreamSynchronize(s), "panel");
    if (!mask && first != none) {
      // kernels.cpp:104-108: the message names the first singular pair and its r
      const int64_t i = (int64_t)(first % (unsigned long long)nx), j = (int64_t)(first / (unsigned long long)nx);
      const double dx = X[3 * i] - Y[3 * j], dy = X[3 * i + 1] - Y[3 * j + 1], dz = X[3 * i + 2] - Y[3 * j + 2];
      const double r = std::sqrt(dx * dx + dy * dy + dz * dz);
      throw std::runtime_error("kernel evaluation at singular point pair (" + std::to_string(i) + "," +
                               std::to_string(j) + "), r=" + std::to_string(r));
    }
    cuda_check(cudaMemcpy2D(out, sizeof(gk_cplx) * ldo, dout.p, sizeof(gk_cplx) * nx, sizeof(gk_cplx) * nx, ny,
                            cudaMemcpyDeviceToHost),
               "panel D2H");
  });
}

gk_status gk_evaluator_destroy(gk_evaluator* E) {
  return guard([&] { delete E; });
}

}  // extern "C"
