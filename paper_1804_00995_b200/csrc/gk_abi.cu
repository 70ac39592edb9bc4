// extern "C" boundary (include/galerk_b200.h): argument checking, the
// reference's error semantics, plan lifetime, device residency.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <exception>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <unordered_map>

#include "../../include/galerk_b200_diag.h"
#include "gk_internal.hpp"

namespace gk {

namespace {
thread_local std::string t_last_error;
}

void set_last_error(const std::string& msg) { t_last_error = msg; }

void cuda_check(int err, const char* what) {
  if (err != cudaSuccess) {
    const char* s = cudaGetErrorString(static_cast<cudaError_t>(err));
    throw CudaError(std::string(what) + ": " + (s ? s : "unknown CUDA error"));
  }
}

void require_device() {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    throw CudaError("galerk_b200: no CUDA device available (this library has no CPU fallback)");
}

void DevBuf::alloc(size_t n) {
  release();
  if (n == 0) return;
  if (cudaMalloc(&p, n) != cudaSuccess) {
    cudaGetLastError();
    p = nullptr;
    throw NoMemError("device allocation of " + std::to_string(n) + " bytes failed");
  }
  bytes = n;
}

void DevBuf::release() {
  if (p) cudaFree(p);
  p = nullptr;
  bytes = 0;
}

void DevBuf::upload(const void* src, size_t n) {
  alloc(n);
  if (n) cuda_check(cudaMemcpy(p, src, n, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
}

int current_device() {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  if (dev < 0 || dev >= kMaxDevices) throw CudaError("device index out of range");
  return dev;
}

void ensure_pool() {
  // per device: the release threshold is an attribute of each device's pool
  static std::mutex m;
  static uint64_t done = 0;
  const int dev = current_device();
  std::lock_guard<std::mutex> g(m);
  if ((done >> dev) & 1u) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    // (256 MB measured too small: with two cfg-4 plans alive (2 x 171 MB) the pool
    // handed its free blocks back at every synchronize, and re-acquiring them
    // stalled about one one-shot step in six by 0.1-0.5 s)
    uint64_t keep = 1024ull << 20;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  cudaGetLastError();
  done |= 1ull << dev;
}

namespace {
// grow-only pinned staging buffer shared by the process's arenas: a pageable
// copy of a few MB runs at a few GB/s, a pinned one at PCIe speed
struct PinnedStaging {
  std::mutex m;
  void* buf = nullptr;
  size_t bytes = 0;
  bool ensure(size_t n) {  // with m held
    if (bytes >= n) return true;
    if (buf) cudaFreeHost(buf);
    buf = nullptr;
    bytes = 0;
    if (cudaMallocHost(&buf, n) != cudaSuccess) {
      cudaGetLastError();
      buf = nullptr;
      return false;
    }
    bytes = n;
    return true;
  }
};
PinnedStaging& pinned_staging() {
  static PinnedStaging S;
  return S;
}
}  // namespace

void DevArena::begin_pinned(size_t upper_bound) {
  if (pinned || !host.empty() || upper_bound == 0) return;
  PinnedStaging& S = pinned_staging();
  S.m.lock();
  if (!S.ensure(upper_bound)) {
    S.m.unlock();
    return;  // no pinned memory: stage in `host`
  }
  pinned = static_cast<char*>(S.buf);
  pinned_cap = S.bytes;
  pinned_used = 0;
}

void DevArena::unlock_pinned() {
  if (!pinned) return;
  pinned = nullptr;
  pinned_cap = pinned_used = 0;
  pinned_staging().m.unlock();
}

void DevArena::spill_pinned() {
  host.assign(pinned, pinned + pinned_used);
  unlock_pinned();
}

void DevArena::upload() {
  if (p) {
    cudaDeviceSynchronize();  // the tables may still be read by work on any stream
    cudaFreeAsync(p, nullptr);
    p = nullptr;
  }
  const size_t copy = used();
  bytes = copy + extra;
  if (bytes) {
    ensure_pool();
    if (cudaMallocAsync(&p, bytes, nullptr) != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      bytes = 0;
      unlock_pinned();
      throw NoMemError("device allocation of " + std::to_string(copy + extra) + " bytes failed");
    }
    if (pinned) {
      const cudaError_t e = cudaMemcpy(p, pinned, copy, cudaMemcpyHostToDevice);
      unlock_pinned();
      cuda_check(e, "cudaMemcpy H2D");
    } else {
      PinnedStaging& S = pinned_staging();
      std::lock_guard<std::mutex> hold(S.m);
      if (S.ensure(copy)) {
        std::memcpy(S.buf, host.data(), copy);
        cuda_check(cudaMemcpy(p, S.buf, copy, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
      } else {
        cuda_check(cudaMemcpy(p, host.data(), copy, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
      }
    }
  }
  unlock_pinned();
  hvec<char>().swap(host);
}

void DevArena::release() {
  if (p) {
    cudaDeviceSynchronize();  // the tables may still be read by work on any stream
    cudaFreeAsync(p, nullptr);
  }
  p = nullptr;
  bytes = 0;
  unlock_pinned();  // (an arena dropped between begin_pinned and upload)
}

}  // namespace gk

using namespace gk;

struct gk_plan {
  int64_t rows = 0, cols = 0;
  bool symmetric = false, helmholtz = false, laplace = false;
  double eps = 0.0, k = 0.0;
  int64_t xloc = 0, yloc = 0, pairs_ref = 0, pairs_unique = 0, pairs_eval = 0, ntiles = 0, nmtiles = 0;
  double x_halo = 0.0, y_halo = 0.0;
  bool natural = false;
  int64_t xblocks = 0, yblocks = 0;
  int32_t jmax = 0;  // widest y block (dofs): selects the k_assemble shape
  bool l2_window = false;  // an assemble call put the tables in a persisting L2 window
  int slots = 1;  // k_assemble SLOTS specialisation (0 none, 1 second slots, 2 with c1 == c0, 3 unit + scales)
  // device tables in one arena: TileDesc per tile ((x block, y block) order,
  // masked ones flagged), x locations, x supports, y records, dof maps
  DevArena arena;
  size_t o_tiles = 0, o_xl_x = 0, o_xl_y = 0, o_xl_z = 0, o_xsup_start = 0, o_xsup_u = 0, o_xsup_c = 0, o_yrec = 0,
         o_xperm = 0, o_yperm = 0, o_yscale = 0;
  // dofs supported by more locations than a tile holds (high-degree vertices
  // with many-point rules): left out of the tiles and computed entry by entry
  // (k_big_entries) from the full side tables
  int64_t nbig_rows = 0, nbig_cols = 0;
  size_t o_big_rows = 0, o_big_cols = 0, o_fx_start = 0, o_fx_loc = 0, o_fx_coef = 0, o_fx_xyz = 0, o_fy_start = 0,
         o_fy_loc = 0, o_fy_coef = 0, o_fy_xyz = 0;
  uint64_t device_bytes() const { return arena.bytes; }
};

struct gk_green_plan {
  int64_t nt_orig = 0, ns_orig = 0, nt = 0, ns = 0;
  bool helmholtz = false;
  double eps = 0.0, k = 0.0;
  DevBuf tx, ty, tz, txf, tyf, tzf, sx, sy, sz, sxf, syf, szf, src_start, src_list, tgt_loc, Q, Y;
  bool symmetric = false;  // targets == sources: fp64 path evaluates each unordered pair once
  int sym_group = 0;
  DevBuf sym_R, sym_C;     // per-group row / column partials
};

namespace {

void check_kernel(const gk_kernel* k) {
  if (!k) throw std::invalid_argument("bem_dense: null kernel");
  if (k->components != 1)
    throw std::invalid_argument("assembly: incompatible operand components (1," + std::to_string(k->components) +
                                ",1)");
  if (k->kind != GK_LAPLACE && k->kind != GK_HELMHOLTZ)
    throw std::invalid_argument(
        "bem_dense: only the built-in scalar Green kernels run on the GPU path (custom kernels are not supported)");
  if (!std::isfinite(k->k)) throw std::invalid_argument("bem_dense: wavenumber must be finite");
}

void memory_cap(const gk_side& test, const gk_side& trial, const gk_options& o) {
  // assembly.cpp:196-203
  const uint64_t need = 16ull * ((uint64_t)test.nfree * (uint64_t)trial.nfree + (uint64_t)o.chunk * trial.npts +
                                 (uint64_t)o.chunk * (uint64_t)trial.nfree);
  if (need > o.memory_cap_bytes)
    throw std::runtime_error("bem_dense: estimated memory " + std::to_string(need / 1000000) +
                             " MB exceeds the cap of " + std::to_string(o.memory_cap_bytes / 1000000) +
                             " MB; use the tol (H-matrix) variant");
}

// One self-contained descriptor per tile: the kernel's staging loads then
// depend on a single descriptor load instead of a chain of table lookups.
// Unmasked and masked tiles are merged back into (x block, y block) order and
// run in one launch; the flag selects the masked pair loop per CTA.
// TX holds the x-block tables, T the y-block tables and the tile lists (the
// same object for whole-matrix plans).
hvec<TileDesc> make_tile_descs(const TileTables& TX, const TileTables& T) {
  const size_t nu = T.tile_i.size(), nm = T.mtile_i.size();
  hvec<TileDesc> d(nu + nm);
  auto fill = [&](TileDesc& D, int32_t bi, int32_t bj, bool masked) {
    D.i0 = TX.xb_dof_start[bi];
    D.nI = TX.xb_dof_start[bi + 1] - D.i0;
    D.j0 = T.yb_dof_start[bj];
    D.nJ = T.yb_dof_start[bj + 1] - D.j0;
    D.l0 = TX.xb_loc_start[bi];
    D.nu = TX.xb_loc_start[bi + 1] - D.l0;
    D.r0 = T.yb_rec_start[bj];
    D.nrec = T.yb_rec_start[bj + 1] - D.r0;
    D.xs0 = TX.xsup_start[D.i0];
    D.nxs = TX.xsup_start[D.i0 + D.nI] - D.xs0;
    D.zero_rows = T.yb_zero[bj];
    D.masked = masked ? 1 : 0;
  };
  size_t a = 0, b = 0, k = 0;
  while (a < nu || b < nm) {
    const bool take_m = b < nm && (a >= nu || std::make_pair(T.mtile_i[b], T.mtile_j[b]) <
                                                  std::make_pair(T.tile_i[a], T.tile_j[a]));
    if (take_m) {
      fill(d[k++], T.mtile_i[b], T.mtile_j[b], true);
      ++b;
    } else {
      fill(d[k++], T.tile_i[a], T.tile_j[a], false);
      ++a;
    }
  }
  return d;
}

struct BigDofs {
  hvec<int32_t> rows, cols;
};
// A copy of side s with the listed dofs constrained (-1): they contribute
// nothing to the tiled assembly.  `store` keeps the masked element table.
gk_side mask_dofs(const gk_side& s, const hvec<int32_t>& dofs, hvec<int32_t>& store) {
  gk_side t = s;
  if (dofs.empty()) return t;
  hvec<char> is_big((size_t)s.nfree, 0);
  for (int32_t d : dofs) is_big[d] = 1;
  store.assign(s.elem_dofs, s.elem_dofs + s.nelem * s.nloc);
  for (int32_t& d : store)
    if (d >= 0 && d < s.nfree && is_big[d]) d = -1;
  t.elem_dofs = store.data();
  return t;
}

// k_assemble specialisation of a y side's tables (TileTables::unit_y records
// carry unit coefficients and need the per-column scales, slots 3)
int slots_of(const TileTables& T) {
  if (T.unit_y) return 3;
  return !T.has_second_slot ? 0 : (T.equal_coefs ? 2 : 1);
}

std::unique_ptr<gk_plan> make_plan(const gk_side* test, const gk_side* trial, const gk_kernel* kernel,
                                   const gk_options* opts, bool dry_run = false) {
  if (!test || !trial) throw std::invalid_argument("bem_dense: null side");
  check_kernel(kernel);
  gk_options o;
  gk_options_default(&o);
  if (opts) o = *opts;
  memory_cap(*test, *trial, o);
  if (!dry_run) require_device();
  auto P = std::make_unique<gk_plan>();
  P->rows = test->nfree;
  P->cols = trial->nfree;
  P->helmholtz = kernel->kind == GK_HELMHOLTZ && kernel->k != 0.0;
  P->k = kernel->kind == GK_LAPLACE ? 0.0 : kernel->k;  // "[1/r]" forces k = 0 (kernels.cpp:47-49)
  P->laplace = kernel->kind == GK_LAPLACE;
  P->eps = guard_radius(*test, *trial);
  P->symmetric = o.symmetric == 1 || (o.symmetric < 0 && sides_identical(*test, *trial));
  const bool timing = std::getenv("GK_TIMING") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto t0 = now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto t1 = now();
    std::fprintf(stderr, "[gk_plan] %-22s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  Locations X = build_locations(*test, "bem_dense(test)");
  lap("locations(test)");
  Locations Y;
  if (P->symmetric) {
    if (!sides_identical(*test, *trial))
      throw std::invalid_argument("bem_dense: symmetric=1 requires identical test and trial sides");
  } else {
    Y = build_locations(*trial, "bem_dense(trial)");
  }
  lap("locations(trial)");
  // Oversized dofs: a row needs all its locations in one x block (<= kUCap),
  // a column all its records in one y block (<= kRCap).  Such dofs (e.g. the
  // apex of a fan of 24 triangles with a 7-point rule: 168 locations) are
  // constrained out of the tiled sides (their rows/columns come out 0) and
  // filled afterwards by k_big_entries from the full tables.
  BigDofs big;
  {
    const Locations& Yf = P->symmetric ? X : Y;
    for (int64_t d = 0; d < X.nfree; ++d)
      if (X.dstart[d + 1] - X.dstart[d] > (P->symmetric ? std::min(kUCap, kRCap) : kUCap)) big.rows.push_back((int32_t)d);
    if (P->symmetric)
      big.cols = big.rows;
    else
      for (int64_t d = 0; d < Yf.nfree; ++d)
        if (Yf.dstart[d + 1] - Yf.dstart[d] > kRCap) big.cols.push_back((int32_t)d);
  }
  Locations Xfull, Yfull;
  if (!big.rows.empty() || !big.cols.empty()) {
    hvec<int32_t> ex, ey;
    const gk_side tx = mask_dofs(*test, big.rows, ex);
    Xfull = std::move(X);
    X = build_locations(tx, "bem_dense(test)");
    if (!P->symmetric) {
      const gk_side ty = mask_dofs(*trial, big.cols, ey);
      Yfull = std::move(Y);
      Y = build_locations(ty, "bem_dense(trial)");
    }
  }
  TileTables T = choose_order_and_tile(X, P->symmetric ? nullptr : &Y, P->symmetric, P->eps);
  lap("order+tiles");
  const Locations& Yr = P->symmetric ? X : Y;
  P->xloc = X.size();
  P->yloc = Yr.size();
  P->pairs_ref = test->npts * trial->npts;
  P->pairs_unique = P->symmetric ? X.size() * (X.size() + 1) / 2 : X.size() * Yr.size();
  P->pairs_eval = T.pairs_evaluated;
  P->x_halo = T.x_halo;
  P->y_halo = T.y_halo;
  P->natural = X.natural;
  P->xblocks = (int64_t)T.xb_dof_start.size() - 1;
  P->yblocks = (int64_t)T.yb_dof_start.size() - 1;
  for (int64_t bj = 0; bj < P->yblocks; ++bj)
    P->jmax = std::max<int32_t>(P->jmax, T.yb_dof_start[bj + 1] - T.yb_dof_start[bj]);
  P->ntiles = T.n_unmasked;
  P->nmtiles = (int64_t)T.mtile_i.size();
  P->slots = slots_of(T);
  if (dry_run) return P;
  DevArena& Ar = P->arena;
  // compact tile list for the device-side descriptor build (launch_make_tiles)
  const int64_t nIb = P->xblocks, nJb = P->yblocks, ntiles_all = P->ntiles + P->nmtiles;
  hvec<int64_t> tile_start(nIb + 1, 0);
  hvec<int32_t> first_bj(nIb, 0);
  for (int64_t bi = 0; bi < nIb; ++bi) {
    int64_t first = 0;
    if (P->symmetric)  // as build_tile_list: tiles whose last column >= the block's first row
      first = std::upper_bound(T.yb_dof_start.begin() + 1, T.yb_dof_start.end(), T.xb_dof_start[bi]) -
              (T.yb_dof_start.begin() + 1);
    first_bj[bi] = (int32_t)first;
    tile_start[bi + 1] = tile_start[bi] + (nJb - first);
  }
  if (tile_start[nIb] != ntiles_all) throw std::logic_error("bem_dense: tile list is not block-complete");
  hvec<uint32_t> masked_bits((size_t)(ntiles_all + 31) / 32, 0u);
  for (size_t m = 0; m < T.mtile_i.size(); ++m) {
    const int32_t bi = T.mtile_i[m], bj = T.mtile_j[m];
    const int64_t e = tile_start[bi] + (bj - first_bj[bi]);
    masked_bits[(size_t)(e >> 5)] |= 1u << (e & 31);
  }
  lap("tile list");
  Ar.begin_pinned((T.xl_x.size() * 3 + T.xsup_c.size()) * sizeof(double) +
                  (T.xsup_start.size() + T.xsup_u.size() + X.perm.size() + Yr.perm.size()) * sizeof(int32_t) +
                  T.yrec.size() * sizeof(YRec) + T.yscale.size() * sizeof(double) + masked_bits.size() * 4 +
                  (nIb + nJb) * 32 + 24 * 256);
  const size_t o_ts = Ar.add(tile_start), o_fb = Ar.add(first_bj), o_xd = Ar.add(T.xb_dof_start),
               o_xl = Ar.add(T.xb_loc_start), o_yd = Ar.add(T.yb_dof_start), o_yr = Ar.add(T.yb_rec_start),
               o_yz = Ar.add(T.yb_zero), o_mb = Ar.add(masked_bits);
  P->o_xl_x = Ar.add(T.xl_x);
  P->o_xl_y = Ar.add(T.xl_y);
  P->o_xl_z = Ar.add(T.xl_z);
  P->o_xsup_start = Ar.add(T.xsup_start);
  P->o_xsup_u = Ar.add(T.xsup_u);
  P->o_xsup_c = Ar.add(T.xsup_c);
  if (P->slots == 3) {
    // unit-coefficient records (32 bytes) written straight into the staging area, on a few threads
    const size_t n = T.yrec.size();
    YRecU* const u = Ar.alloc<YRecU>(n, P->o_yrec);
    const YRec* const r = T.yrec.data();
    auto fill = [=](size_t i0, size_t i1) {
      for (size_t i = i0; i < i1; ++i) u[i] = {r[i].x, r[i].y, r[i].z, r[i].off0, r[i].off1};
    };
    const int nt = (int)std::min<size_t>((size_t)std::min(host_threads(), 4), n / 16384);
    if (nt <= 1) {
      fill(0, n);
    } else {
      std::vector<std::thread> pool;
      for (int t = 1; t < nt; ++t) pool.emplace_back(fill, n * t / nt, n * (t + 1) / nt);
      fill(0, n / nt);
      for (auto& th : pool) th.join();
    }
  } else {
    P->o_yrec = Ar.add(T.yrec);
  }
  P->o_xperm = Ar.add(X.perm);
  P->o_yperm = Ar.add(Yr.perm);
  P->o_yscale = Ar.add(T.yscale);
  if (!big.rows.empty() || !big.cols.empty()) {
    const Locations& Yf = P->symmetric ? Xfull : Yfull;
    P->nbig_rows = (int64_t)big.rows.size();
    P->nbig_cols = (int64_t)big.cols.size();
    P->o_big_rows = Ar.add(big.rows);
    P->o_big_cols = Ar.add(big.cols);
    auto side = [&](const Locations& L, size_t& o_start, size_t& o_loc, size_t& o_coef, size_t& o_xyz) {
      o_start = Ar.add(L.dstart);
      o_loc = Ar.add(L.dloc);
      o_coef = Ar.add(L.dcoef);
      hvec<double> xyz(3 * (size_t)L.size());
      for (int64_t u = 0; u < L.size(); ++u) xyz[3 * u] = L.x[u], xyz[3 * u + 1] = L.y[u], xyz[3 * u + 2] = L.z[u];
      o_xyz = Ar.add(xyz);
    };
    side(Xfull, P->o_fx_start, P->o_fx_loc, P->o_fx_coef, P->o_fx_xyz);
    if (P->symmetric) {
      P->o_fy_start = P->o_fx_start, P->o_fy_loc = P->o_fx_loc, P->o_fy_coef = P->o_fx_coef, P->o_fy_xyz = P->o_fx_xyz;
    } else {
      side(Yf, P->o_fy_start, P->o_fy_loc, P->o_fy_coef, P->o_fy_xyz);
    }
  }
  P->o_tiles = Ar.add_device_only((size_t)ntiles_all * sizeof(TileDesc));
  lap("stage");
  Ar.upload();
  lap("upload");
  if (ntiles_all > 0) {
    TileBuildArgs b;
    b.out = Ar.at<TileDesc>(P->o_tiles);
    b.ntiles = ntiles_all;
    b.nIb = (int32_t)nIb;
    b.tile_start = Ar.at<int64_t>(o_ts);
    b.first_bj = Ar.at<int32_t>(o_fb);
    b.xb_dof_start = Ar.at<int32_t>(o_xd);
    b.xb_loc_start = Ar.at<int32_t>(o_xl);
    b.yb_dof_start = Ar.at<int32_t>(o_yd);
    b.yb_rec_start = Ar.at<int32_t>(o_yr);
    b.yb_zero = Ar.at<uint32_t>(o_yz);
    b.xsup_start = Ar.at<int32_t>(P->o_xsup_start);
    b.masked_bits = Ar.at<uint32_t>(o_mb);
    launch_make_tiles(b, nullptr);
    cuda_check(cudaStreamSynchronize(nullptr), "k_make_tiles");
  }
  lap("tile descriptors");
  return P;
}

void assemble(gk_plan* P, gk_cplx* A, int64_t lda, gk_stream stream) {
  if (!P) throw std::invalid_argument("gk_plan_assemble: null plan");
  if (P->rows == 0 || P->cols == 0) return;
  if (!A) throw std::invalid_argument("gk_plan_assemble: null matrix");
  if (lda < P->rows) throw std::invalid_argument("gk_plan_assemble: lda < rows");
  AsmArgs a;
  const DevArena& Ar = P->arena;
  a.tiles = Ar.at<TileDesc>(P->o_tiles);
  a.xl_x = Ar.at<double>(P->o_xl_x);
  a.xl_y = Ar.at<double>(P->o_xl_y);
  a.xl_z = Ar.at<double>(P->o_xl_z);
  a.xsup_start = Ar.at<int32_t>(P->o_xsup_start);
  a.xsup_u = Ar.at<int32_t>(P->o_xsup_u);
  a.xsup_c = Ar.at<double>(P->o_xsup_c);
  a.yrec = Ar.at<YRec>(P->o_yrec);
  a.xperm = Ar.at<int32_t>(P->o_xperm);
  a.yperm = Ar.at<int32_t>(P->o_yperm);
  a.yscale = P->slots == 3 ? Ar.at<double>(P->o_yscale) : nullptr;
  a.A = A;
  a.lda = lda;
  a.eps2 = P->eps * P->eps;
  a.kappa = 2.0 * P->k / M_PI;
  a.symmetric = P->symmetric ? 1 : 0;
  a.natural = P->natural ? 1 : 0;
  a.l2_window = nullptr;
  a.l2_window_bytes = 0;
  a.prof = nullptr;
  a.dbg = std::getenv("GK_ASM_DBG") ? std::atoi(std::getenv("GK_ASM_DBG")) : 0;
  a.jmax = P->jmax;
  if (P->nbig_rows || P->nbig_cols) {
    BigArgs b;
    b.rows = Ar.at<int32_t>(P->o_big_rows);
    b.cols = Ar.at<int32_t>(P->o_big_cols);
    b.nbig_rows = P->nbig_rows;
    b.nbig_cols = P->nbig_cols;
    b.nrows = P->rows;
    b.ncols = P->cols;
    b.xs = Ar.at<int64_t>(P->o_fx_start);
    b.xl = Ar.at<int32_t>(P->o_fx_loc);
    b.xc = Ar.at<double>(P->o_fx_coef);
    b.xp = Ar.at<double>(P->o_fx_xyz);
    b.ys = Ar.at<int64_t>(P->o_fy_start);
    b.yl = Ar.at<int32_t>(P->o_fy_loc);
    b.yc = Ar.at<double>(P->o_fy_coef);
    b.yp = Ar.at<double>(P->o_fy_xyz);
    b.A = A;
    b.lda = lda;
    b.eps2 = a.eps2;
    b.kappa = a.kappa;
    b.symmetric = a.symmetric;
    launch_assemble(a, P->ntiles + P->nmtiles, P->helmholtz, P->slots, stream);
    launch_big_entries(b, P->helmholtz, stream);  // after the tiles: overwrites their zeros
    return;
  }
  // tiles that can hold a coincident pair apply the distance mask; the rest skip it
  if (!std::getenv("GK_ASM_PROF")) {
    // Matrices far larger than L2 (>= 4 GB): the plan tables — everything
    // before the tile descriptors, 14 MB on cfg 4 — sit in a persisting L2
    // window for this launch (a launch attribute), so that the matrix write
    // stream does not evict them (cfg 4: table re-reads from DRAM 2.82 ->
    // 0.18 GB, DRAM traffic 1.026x -> 1.001x the matrix write;
    // GK_L2_PERSIST=0 turns it off).  Smaller matrices do not gain: cfg 2's
    // 0.44 GB of DRAM reads are sector fills behind its permuted 16-byte
    // stores, not table re-reads (unchanged by the window, and the launch ran
    // 0.5% slower with it).  The device's persisting carve-out is raised to
    // 32 MB if smaller.
    static const bool allow = !(std::getenv("GK_L2_PERSIST") && std::atoi(std::getenv("GK_L2_PERSIST")) == 0);
    const bool persist = allow && (double)P->rows * (double)P->cols * 16.0 >= 4e9 && P->o_tiles > 0 &&
                         P->o_tiles <= (32u << 20);
    if (persist) {
      static std::atomic<uint64_t> limit_set{0};  // per device
      const int dev = current_device();
      if (!((limit_set.load() >> dev) & 1u)) {
        size_t cur = 0;
        cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
        if (cur < (32u << 20)) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 32u << 20);
        cudaGetLastError();  // (a device without the feature ignores the window)
        limit_set |= 1ull << dev;
      }
      a.l2_window = Ar.p;
      a.l2_window_bytes = P->o_tiles;
      P->l2_window = true;
    }
    launch_assemble(a, P->ntiles + P->nmtiles, P->helmholtz, P->slots, stream);
    return;
  }
  // diagnostics: per-tile phase cycles (staging / pair loop / gather + stores)
  const int64_t nt = P->ntiles + P->nmtiles;
  DevBuf prof;
  prof.alloc(sizeof(unsigned long long) * 4 * std::max<int64_t>(1, nt));
  a.prof = prof.as<unsigned long long>();
  launch_assemble(a, nt, P->helmholtz, P->slots, stream);
  cuda_check(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "GK_ASM_PROF");
  std::vector<unsigned long long> h((size_t)(4 * nt));
  cuda_check(cudaMemcpy(h.data(), prof.p, h.size() * 8, cudaMemcpyDeviceToHost), "GK_ASM_PROF copy");
  double sum[3] = {0, 0, 0};
  for (int64_t i = 0; i < nt; ++i)
    for (int k = 0; k < 3; ++k) sum[k] += (double)h[4 * i + k];
  std::fprintf(stderr, "[gk_asm_prof] tiles %lld  mean cycles: staging %.0f  pair loop %.0f  gather+stores %.0f\n",
               (long long)nt, sum[0] / nt, sum[1] / nt, sum[2] / nt);
}


// ---- one-shot assembly streamed to the host in column slabs ------------------
// gk_bem_dense's cost is the host plan (~18 ms on cfg 2) followed by the
// device->host copy of the matrix (29 ms at the PCIe limit), the kernel being
// ~3 ms.  Streaming overlaps them: the x side is located, ordered and tiled
// once; the columns are cut into contiguous slabs (host-contiguous in the
// column-major output) whose y tables worker threads build ahead while the
// GPU assembles slab s (non-symmetric tiles, x blocks x the slab's y blocks)
// and the copy engine drains slab s-1.  Pageable destinations go through
// pinned bounce buffers and a threaded host copy.
struct SlabTables {
  hvec<char> blob;  // descs | yrec | yperm, 256-byte aligned sections
  size_t o_desc = 0, o_yrec = 0, o_yperm = 0, o_yscale = 0;
  int64_t ntiles = 0;
  int slots = 0;
  bool ready = false;
  std::exception_ptr err;
};

template <class V>
size_t blob_add(hvec<char>& b, const V& v) {
  using T = typename V::value_type;
  const size_t off = (b.size() + 255) & ~size_t(255);
  b.resize(off + v.size() * sizeof(T));
  if (!v.empty()) std::memcpy(b.data() + off, v.data(), v.size() * sizeof(T));
  return off;
}


// Column-slab width for a streamed one-shot call, or 0 for the whole-matrix path.
// Whether some dof is supported by more points than a tile holds (an upper
// bound on its merged locations): the streamed path has no oversized-dof
// fix-up, so such sides take the whole-matrix plan.
bool may_have_big_dofs(const gk_side& s) {
  if (s.nfree <= 0 || s.nelem <= 0 || !s.elem_dofs) return false;
  hvec<int32_t> cnt((size_t)s.nfree, 0);
  for (int64_t e = 0; e < s.nelem; ++e)
    for (int l = 0; l < s.nloc; ++l) {
      const int32_t d = s.elem_dofs[e * s.nloc + l];
      if (d >= 0 && d < s.nfree && (cnt[d] += s.g) > std::min(kUCap, kRCap)) return true;
    }
  return false;
}

int64_t stream_slab_cols(int64_t rows, int64_t cols) {
  const char* force = std::getenv("GK_SLAB_COLS");
  if (force) return std::max<int64_t>(0, std::atoll(force));
  const char* off = std::getenv("GK_STREAM");
  if (off && std::atoi(off) == 0) return 0;
  const double total = 16.0 * (double)rows * (double)cols;
  if (total < 64e6) return 0;
  const double target = std::min(256e6, std::max(32e6, total / 16.0));
  int64_t w = (int64_t)(target / (16.0 * (double)rows));
  w = std::max<int64_t>(64, (w + 63) / 64 * 64);
  return (cols + w - 1) / w >= 3 ? w : 0;
}

void bem_dense_streamed(const gk_side* test, const gk_side* trial, const gk_kernel* kernel, const gk_options& o,
                        gk_cplx* A_host, int64_t lda, int64_t w) {
  const bool timing = std::getenv("GK_TIMING") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[gk_stream] %-14s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  const int64_t rows = test->nfree, cols = trial->nfree;
  const bool helm = kernel->kind == GK_HELMHOLTZ && kernel->k != 0.0;
  const double k = kernel->kind == GK_LAPLACE ? 0.0 : kernel->k;
  const double eps = guard_radius(*test, *trial);
  const bool same = sides_identical(*test, *trial);
  Locations X = build_locations(*test, "bem_dense(test)");
  Locations Y;
  if (!same) Y = build_locations(*trial, "bem_dense(trial)");
  lap("locations");
  // the slabs are PCIe-bound (the kernel takes ~1/5 of a slab's copy), so a
  // natural order within 3x of the unique pair count is taken without
  // building the RCB candidate (saves ~3 ms of host time per call on cfg 2)
  const OrderChoice O = choose_order(X, same ? nullptr : &Y, false, eps, 3.0);
  const Locations& Yf = same ? X : Y;
  lap("order");
  TileTables TX;
  hvec<int32_t> xl_id;
  bool x_ready = false;  // TX / xl_id built (workers prepare their y side before that)

  // ---- slab table builders (look-ahead bounded to keep host memory flat)
  const int64_t nslab = (cols + w - 1) / w;
  std::vector<SlabTables> S(nslab);
  std::mutex m;
  std::condition_variable cv;
  int64_t next = 0, consumed = 0;
  bool stop = false;
  const int nworkers = (int)std::min<int64_t>(nslab, std::max(1, host_threads() - 1));
  const int64_t ahead = 2 * nworkers + 2;
  std::atomic<int64_t> build_us{0};
  auto build_slab = [&](int64_t s) {
    const auto b0 = std::chrono::steady_clock::now();
    SlabTables& T = S[s];
    const int64_t c0 = s * w, c1 = std::min(cols, c0 + w);
    hvec<int32_t> slab_of_full;
    Locations Ys = restrict_cols(Yf, c0, c1, slab_of_full);
    set_order(Ys, O.natural, O.unit);
    BlockLayout Bs;
    layout_y_blocks(Ys, Bs);
    TileTables TY;
    hvec<int64_t> yb_start;
    hvec<int32_t> yb_list;
    build_y_tables(Ys, Bs, TY, yb_start, yb_list);
    Coincidence Cs;
    Cs.unsafe = O.C.unsafe;
    if (!Cs.unsafe) {
      Cs.y_of_x.resize(O.C.y_of_x.size());
      for (size_t u = 0; u < Cs.y_of_x.size(); ++u) {
        const int32_t v = O.C.y_of_x[u];
        Cs.y_of_x[u] = v >= 0 ? slab_of_full[v] : -1;
      }
    }
    {
      std::unique_lock<std::mutex> g(m);
      cv.wait(g, [&] { return stop || x_ready; });
      if (!x_ready) return;  // stopping: the slab is never consumed
    }
    build_tile_list(TX, TY, false, Cs, xl_id, yb_start, yb_list);
    const hvec<TileDesc> descs = make_tile_descs(TX, TY);
    T.blob.reserve(descs.size() * sizeof(TileDesc) + TY.yrec.size() * sizeof(YRec) + Ys.perm.size() * 4 +
                   TY.yscale.size() * 8 + 1024);
    T.o_desc = blob_add(T.blob, descs);
    T.o_yrec = blob_add(T.blob, device_records(TY.yrec, slots_of(TY) == 3));
    T.o_yperm = blob_add(T.blob, Ys.perm);
    T.o_yscale = blob_add(T.blob, TY.yscale);
    T.ntiles = (int64_t)descs.size();
    T.slots = slots_of(TY);
    build_us += std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - b0).count();
  };
  std::vector<std::thread> workers;
  auto stop_workers = [&] {
    {
      std::lock_guard<std::mutex> g(m);
      stop = true;
    }
    cv.notify_all();
    for (auto& t : workers) t.join();
    workers.clear();
  };
  for (int t = 0; t < nworkers; ++t)
    workers.emplace_back([&] {
      planner_serial(true);
      for (;;) {
        int64_t s;
        {
          std::unique_lock<std::mutex> g(m);
          cv.wait(g, [&] { return stop || next >= nslab || next < consumed + ahead; });
          if (stop || next >= nslab) return;
          s = next++;
        }
        std::exception_ptr err;
        try {
          build_slab(s);
        } catch (...) {
          err = std::current_exception();
        }
        {
          std::lock_guard<std::mutex> g(m);
          S[s].err = err;
          S[s].ready = true;
        }
        cv.notify_all();
      }
    });

  // ---- x tables, built while the workers prepare the first slabs' y sides
  DevArena AX;
  size_t o_xl_x = 0, o_xl_y = 0, o_xl_z = 0, o_xsup_start = 0, o_xsup_u = 0, o_xsup_c = 0, o_xperm = 0;
  try {
    build_x_tables(X, O.B, TX, xl_id);
    {
      std::lock_guard<std::mutex> g(m);
      x_ready = true;
    }
    cv.notify_all();
    lap("x tables");
    AX.host.reserve((TX.xl_x.size() * 3 + TX.xsup_c.size()) * sizeof(double) +
                    (TX.xsup_start.size() + TX.xsup_u.size() + X.perm.size()) * sizeof(int32_t) + 8 * 256);
    o_xl_x = AX.add(TX.xl_x);
    o_xl_y = AX.add(TX.xl_y);
    o_xl_z = AX.add(TX.xl_z);
    o_xsup_start = AX.add(TX.xsup_start);
    o_xsup_u = AX.add(TX.xsup_u);
    o_xsup_c = AX.add(TX.xsup_c);
    o_xperm = AX.add(X.perm);
    AX.upload();
    lap("x upload");
  } catch (...) {
    stop_workers();
    throw;
  }

  // ---- device pipeline: tables H2D + kernel on ks, matrix D2H on cs
  // Streams, events, table staging and slab buffers persist between calls
  // (one-shot callers repeat; pinned allocations and frees cost milliseconds
  // and synchronise the device).
  struct Stage {
    void* host = nullptr;      // pinned, mapped table staging
    void* host_dev = nullptr;  // its device view
    size_t host_bytes = 0;
    void* dev = nullptr;       // device tables
    size_t dev_bytes = 0;
    void* bounce = nullptr;    // pinned bounce buffer (pageable destinations)
    size_t bounce_bytes = 0;
    cudaEvent_t h2d = nullptr, kern = nullptr, d2h = nullptr;
  };
  struct Resources {
    Stage st[2];
    DevBuf slab[2];
    cudaStream_t ks = nullptr, cs = nullptr;
  };
  // streams, slab buffers and staging belong to one device: one set per device
  static std::mutex res_mutex[kMaxDevices];
  static Resources Rs[kMaxDevices];
  const int dev = current_device();
  std::lock_guard<std::mutex> hold(res_mutex[dev]);
  Resources& R = Rs[dev];
  Stage* st = R.st;
  cudaPointerAttributes pa{};
  const bool pinned_dst = cudaPointerGetAttributes(&pa, A_host) == cudaSuccess && pa.type == cudaMemoryTypeHost;
  cudaGetLastError();
  const size_t slab_bytes = sizeof(gk_cplx) * (size_t)rows * (size_t)w;
  auto cleanup = [&] {
    stop_workers();
    if (R.ks) cudaStreamSynchronize(R.ks);
    if (R.cs) cudaStreamSynchronize(R.cs);
    cudaGetLastError();
  };
  // host copy of a finished pageable slab: bounce -> A_host columns, threaded
  auto drain = [&](int64_t s) {
    const Stage& g = st[s & 1];
    cuda_check(cudaEventSynchronize(g.d2h), "gk_bem_dense D2H");
    const int64_t c0 = s * w, nc = std::min(cols, c0 + w) - c0;
    const int nt = (int)std::min<int64_t>(host_threads(), std::max<int64_t>(1, nc / 4));
    auto copy = [&](int64_t a, int64_t b) {
      for (int64_t c = a; c < b; ++c)
        std::memcpy(A_host + (c0 + c) * lda, static_cast<const gk_cplx*>(g.bounce) + c * rows,
                    sizeof(gk_cplx) * rows);
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(copy, nc * t / nt, nc * (t + 1) / nt);
    copy(0, nc / nt);
    for (auto& t : pool) t.join();
  };
  try {
    if (!R.ks) cuda_check(cudaStreamCreateWithFlags(&R.ks, cudaStreamNonBlocking), "cudaStreamCreate");
    if (!R.cs) cuda_check(cudaStreamCreateWithFlags(&R.cs, cudaStreamNonBlocking), "cudaStreamCreate");
    const cudaStream_t ks = R.ks, cs = R.cs;
    for (DevBuf& b : R.slab)
      if (b.bytes < slab_bytes) b.alloc(slab_bytes);
    for (int i = 0; i < 2; ++i) {
      Stage& g = st[i];
      for (cudaEvent_t* e : {&g.h2d, &g.kern, &g.d2h})
        if (!*e) cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "cudaEventCreate");
      if (!pinned_dst && g.bounce_bytes < slab_bytes) {
        if (g.bounce) cudaFreeHost(g.bounce);
        g.bounce = nullptr;
        g.bounce_bytes = 0;
        cuda_check(cudaMallocHost(&g.bounce, slab_bytes), "cudaMallocHost bounce");
        g.bounce_bytes = slab_bytes;
      }
      // the first slab's events must not refer to a previous call's work
      cuda_check(cudaEventRecord(g.h2d, ks), "cudaEventRecord");
      cuda_check(cudaEventRecord(g.d2h, cs), "cudaEventRecord");
    }
    lap("setup");
    AsmArgs a;
    a.xl_x = AX.at<double>(o_xl_x);
    a.xl_y = AX.at<double>(o_xl_y);
    a.xl_z = AX.at<double>(o_xl_z);
    a.xsup_start = AX.at<int32_t>(o_xsup_start);
    a.xsup_u = AX.at<int32_t>(o_xsup_u);
    a.xsup_c = AX.at<double>(o_xsup_c);
    a.xperm = AX.at<int32_t>(o_xperm);
    a.lda = rows;
    a.eps2 = eps * eps;
    a.kappa = 2.0 * k / M_PI;
    a.symmetric = 0;
    a.natural = 0;
    a.l2_window = nullptr;
    a.l2_window_bytes = 0;
    a.prof = nullptr;
    a.dbg = 0;
    a.jmax = kJCap;  // slabs: the 22-row shape serves every y block
    double wait_ms = 0.0;
    for (int64_t s = 0; s < nslab; ++s) {
      {
        const auto w0 = std::chrono::steady_clock::now();
        std::unique_lock<std::mutex> g(m);
        cv.wait(g, [&] { return S[s].ready; });
        wait_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w0).count();
      }
      if (S[s].err) std::rethrow_exception(S[s].err);
      Stage& g = st[s & 1];
      SlabTables& T = S[s];
      const size_t nb = T.blob.size();
      if (s >= 2) cuda_check(cudaEventSynchronize(g.h2d), "gk_bem_dense H2D");
      const size_t nb16 = (nb + 15) & ~size_t(15);
      if (g.host_bytes < nb16) {
        cuda_check(cudaStreamSynchronize(ks), "gk_bem_dense");  // the fetch kernels read the old staging
        if (g.host) cudaFreeHost(g.host);
        g.host = nullptr;
        g.host_bytes = 0;
        const size_t want = std::max<size_t>(nb16 + nb16 / 2, 1 << 20);
        cuda_check(cudaHostAlloc(&g.host, want, cudaHostAllocMapped | cudaHostAllocPortable),
                   "cudaHostAlloc staging");
        g.host_bytes = want;
        cuda_check(cudaHostGetDevicePointer(&g.host_dev, g.host, 0), "cudaHostGetDevicePointer");
      }
      if (g.dev_bytes < nb16) {
        if (g.dev) cuda_check(cudaFreeAsync(g.dev, ks), "cudaFreeAsync");
        g.dev = nullptr;
        g.dev_bytes = 0;
        const size_t want = std::max<size_t>(nb16 + nb16 / 2, 1 << 20);
        cuda_check(cudaMallocAsync(&g.dev, want, ks), "cudaMallocAsync tables");
        g.dev_bytes = want;
      }
      std::memcpy(g.host, T.blob.data(), nb);
      hvec<char>().swap(T.blob);
      launch_fetch_tables(g.dev, g.host_dev, nb, ks);
      cuda_check(cudaEventRecord(g.h2d, ks), "cudaEventRecord");
      {
        std::lock_guard<std::mutex> lk(m);
        consumed = s + 1;
      }
      cv.notify_all();
      if (s >= 2) cuda_check(cudaStreamWaitEvent(ks, g.d2h, 0), "cudaStreamWaitEvent");
      a.tiles = reinterpret_cast<const TileDesc*>(static_cast<char*>(g.dev) + T.o_desc);
      a.yrec = reinterpret_cast<const YRec*>(static_cast<char*>(g.dev) + T.o_yrec);
      a.yperm = reinterpret_cast<const int32_t*>(static_cast<char*>(g.dev) + T.o_yperm);
      a.yscale = T.slots == 3 ? reinterpret_cast<const double*>(static_cast<char*>(g.dev) + T.o_yscale) : nullptr;
      a.A = R.slab[s & 1].p;
      launch_assemble(a, T.ntiles, helm, T.slots, ks);
      cuda_check(cudaEventRecord(g.kern, ks), "cudaEventRecord");
      cuda_check(cudaStreamWaitEvent(cs, g.kern, 0), "cudaStreamWaitEvent");
      const int64_t c0 = s * w, nc = std::min(cols, c0 + w) - c0;
      if (pinned_dst) {
        cuda_check(cudaMemcpy2DAsync(A_host + c0 * lda, sizeof(gk_cplx) * lda, R.slab[s & 1].p,
                                     sizeof(gk_cplx) * rows, sizeof(gk_cplx) * rows, nc, cudaMemcpyDeviceToHost, cs),
                   "cudaMemcpy2DAsync D2H");
      } else {
        if (s >= 2) drain(s - 2);  // bounce buffer s & 1 is free once slab s-2 is on the host
        cuda_check(cudaMemcpyAsync(g.bounce, R.slab[s & 1].p, sizeof(gk_cplx) * rows * nc,
                                   cudaMemcpyDeviceToHost, cs),
                   "cudaMemcpyAsync D2H");
      }
      cuda_check(cudaEventRecord(g.d2h, cs), "cudaEventRecord");
    }
    if (!pinned_dst)
      for (int64_t s = std::max<int64_t>(0, nslab - 2); s < nslab; ++s) drain(s);
    lap("slabs issued");
    if (timing) std::fprintf(stderr, "[gk_stream] %lld slabs of %lld cols, %d workers, waited %.2f ms for tables\n",
                             (long long)nslab, (long long)w, nworkers, wait_ms);
    cuda_check(cudaStreamSynchronize(cs), "gk_bem_dense");
    cuda_check(cudaStreamSynchronize(ks), "gk_bem_dense");
    lap("slabs drained");
    if (timing) std::fprintf(stderr, "[gk_stream] slab tables: %.2f ms of worker time\n", build_us.load() * 1e-3);
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
}

}  // namespace

extern "C" {

void gk_options_default(gk_options* o) {
  if (!o) return;
  o->memory_cap_bytes = 8000000000ull;  // BemOptions (assembly.hpp:27-30)
  o->chunk = 1024;
  o->symmetric = -1;
  o->reserved = 0;
}

gk_status gk_plan_create(const gk_side* test, const gk_side* trial, const gk_kernel* kernel, const gk_options* opts,
                         gk_plan** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("gk_plan_create: null output");
    *out = nullptr;
    *out = make_plan(test, trial, kernel, opts).release();
  });
}

gk_status gk_diag_plan_info(const gk_side* test, const gk_side* trial, const gk_kernel* kernel,
                            const gk_options* opts, gk_plan_info* info) {
  gk_status st = GK_OK;
  std::unique_ptr<gk_plan> P;
  st = guard([&] { P = make_plan(test, trial, kernel, opts, /*dry_run=*/true); });
  if (st != GK_OK) return st;
  return gk_plan_get_info(P.get(), info);
}

gk_status gk_diag_location_ids(const gk_side* side, int32_t serial, int64_t* point_loc, int64_t* n_locations,
                               double* xyz) {
  return guard([&] {
    if (!side || !point_loc || !n_locations) throw std::invalid_argument("gk_diag_location_ids: null argument");
    struct Serial {  // the planner's per-thread switch, restored on every exit
      bool on;
      explicit Serial(bool s) : on(s) {
        if (on) planner_serial(true);
      }
      ~Serial() {
        if (on) planner_serial(false);
      }
    } hold(serial != 0);
    const Locations L = build_locations(*side, "gk_diag_location_ids");
    for (int64_t k = 0; k < side->npts; ++k) point_loc[k] = L.point_loc[(size_t)k];
    *n_locations = L.size();
    if (xyz)
      for (int64_t u = 0; u < L.size(); ++u) xyz[3 * u] = L.x[u], xyz[3 * u + 1] = L.y[u], xyz[3 * u + 2] = L.z[u];
  });
}

gk_status gk_plan_get_info(const gk_plan* P, gk_plan_info* info) {
  return guard([&] {
    if (!P || !info) throw std::invalid_argument("gk_plan_get_info: null argument");
    info->rows = P->rows;
    info->cols = P->cols;
    info->x_locations = P->xloc;
    info->y_locations = P->yloc;
    info->pairs_reference = P->pairs_ref;
    info->pairs_unique = P->pairs_unique;
    info->pairs_evaluated = P->pairs_eval;
    info->tiles = P->ntiles + P->nmtiles;
    info->masked_tiles = P->nmtiles;
    info->symmetric = P->symmetric ? 1 : 0;
    info->eps = P->eps;
    info->device_bytes = P->device_bytes();
    info->x_halo = P->x_halo;
    info->y_halo = P->y_halo;
    info->natural_order = P->natural ? 1 : 0;
    info->x_blocks = P->xblocks;
    info->y_blocks = P->yblocks;
  });
}

gk_status gk_plan_assemble(gk_plan* P, gk_cplx* A, int64_t lda, gk_stream stream) {
  return guard([&] { assemble(P, A, lda, stream); });
}

gk_status gk_plan_set_wavenumber(gk_plan* P, double k) {
  return guard([&] {
    if (!P) throw std::invalid_argument("gk_plan_set_wavenumber: null plan");
    if (!std::isfinite(k)) throw std::invalid_argument("bem_dense: wavenumber must be finite");
    if (P->laplace) return;  // "[1/r]" forces k = 0 (kernels.cpp:47-49)
    P->k = k;
    P->helmholtz = k != 0.0;
  });
}

int32_t gk_plan_launches(const gk_plan* P) {
  return P ? (P->ntiles + P->nmtiles > 0 ? 1 : 0) + (P->nbig_rows + P->nbig_cols > 0 ? 1 : 0) : 0;
}

gk_status gk_plan_destroy(gk_plan* P) {
  return guard([&] {
    const bool window = P && P->l2_window;
    delete P;  // synchronises the device before the tables return to the pool
    if (window && cudaCtxResetPersistingL2Cache() != cudaSuccess) cudaGetLastError();  // its lines go back to normal
  });
}

gk_status gk_bem_dense(const gk_side* test, const gk_side* trial, const gk_kernel* kernel, const gk_options* opts,
                       gk_cplx* A_host, int64_t lda) {
  return guard([&] {
    const bool timing = std::getenv("GK_TIMING") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
      if (!timing) return;
      cudaDeviceSynchronize();
      const auto t1 = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[gk_bem_dense] %-10s %8.2f ms\n", what,
                   std::chrono::duration<double, std::milli>(t1 - t0).count());
      t0 = t1;
    };
    if (test && trial && kernel && A_host && test->nfree > 0 && trial->nfree > 0 && lda >= test->nfree &&
        !may_have_big_dofs(*test) && !may_have_big_dofs(*trial)) {
      const int64_t w = stream_slab_cols(test->nfree, trial->nfree);
      if (w > 0) {
        check_kernel(kernel);
        gk_options o;
        gk_options_default(&o);
        if (opts) o = *opts;
        memory_cap(*test, *trial, o);
        require_device();
        if (o.symmetric == 1 && !sides_identical(*test, *trial))
          throw std::invalid_argument("bem_dense: symmetric=1 requires identical test and trial sides");
        bem_dense_streamed(test, trial, kernel, o, A_host, lda, w);
        return;
      }
    }
    auto P = make_plan(test, trial, kernel, opts);
    lap("plan");
    if (P->rows == 0 || P->cols == 0) return;
    if (!A_host) throw std::invalid_argument("gk_bem_dense: null output matrix");
    if (lda < P->rows) throw std::invalid_argument("gk_bem_dense: lda < rows");
    // The device matrix: a grow-only scratch buffer kept between calls up to
    // 16 GB (one-shot callers repeat with the same size, and mapping a fresh
    // 1.7 GB allocation costs ~9 ms); larger matrices are allocated per call.
    static std::mutex scratch_mutex[kMaxDevices];
    static DevBuf scratch_of[kMaxDevices];
    const int dev = current_device();
    DevBuf& scratch = scratch_of[dev];
    std::unique_lock<std::mutex> hold(scratch_mutex[dev], std::defer_lock);
    DevBuf own;
    const size_t bytes = sizeof(gk_cplx) * (size_t)P->rows * (size_t)P->cols;
    void* A = nullptr;
    if (bytes <= (16ull << 30)) {
      hold.lock();
      if (scratch.bytes < bytes) scratch.alloc(bytes);
      A = scratch.p;
    } else {
      own.alloc(bytes);
      A = own.p;
    }
    cudaStream_t s = nullptr;
    lap("alloc");
    assemble(P.get(), static_cast<gk_cplx*>(A), P->rows, s);
    lap("assemble");
    cuda_check(cudaMemcpy2DAsync(A_host, sizeof(gk_cplx) * lda, A, sizeof(gk_cplx) * P->rows,
                                 sizeof(gk_cplx) * P->rows, P->cols, cudaMemcpyDeviceToHost, s),
               "cudaMemcpy2DAsync D2H");
    cuda_check(cudaStreamSynchronize(s), "gk_bem_dense");
    lap("d2h");
    P.reset();
    lap("destroy");
  });
}

gk_status gk_matvec(const gk_cplx* A, int64_t rows, int64_t cols, int64_t lda, const gk_cplx* x, gk_cplx* y,
                    gk_stream stream) {
  return guard([&] {
    if (rows < 0 || cols < 0) throw std::invalid_argument("gk_matvec: negative size");
    if (rows > 0 && cols > 0 && (!A || !x)) throw std::invalid_argument("gk_matvec: null input");
    if (rows > 0 && !y) throw std::invalid_argument("gk_matvec: null output");
    if (lda < rows) throw std::invalid_argument("gk_matvec: lda < rows");
    require_device();
    launch_matvec(A, rows, cols, lda, x, y, stream);
  });
}

int32_t gk_matvec_launches(int64_t rows, int64_t cols) { return matvec_launch_count(rows, cols); }

gk_status gk_matvec_multi(const gk_cplx* A, int64_t rows, int64_t cols, int64_t lda, const gk_cplx* X,
                          int64_t ldx, gk_cplx* Y, int64_t ldy, int32_t nrhs, gk_stream stream) {
  return guard([&] {
    if (rows < 0 || cols < 0 || nrhs < 0) throw std::invalid_argument("gk_matvec_multi: negative size");
    if (rows > 0 && cols > 0 && nrhs > 0 && (!A || !X)) throw std::invalid_argument("gk_matvec_multi: null input");
    if (rows > 0 && nrhs > 0 && !Y) throw std::invalid_argument("gk_matvec_multi: null output");
    if (lda < rows) throw std::invalid_argument("gk_matvec_multi: lda < rows");
    if (nrhs > 1 && (ldx < cols || ldy < rows)) throw std::invalid_argument("gk_matvec_multi: ldx < cols or ldy < rows");
    require_device();
    launch_matvec_multi(A, rows, cols, lda, X, ldx, Y, ldy, nrhs, stream);
  });
}

int32_t gk_matvec_multi_launches(int64_t rows, int64_t cols, int32_t nrhs) {
  return matvec_multi_launch_count(rows, cols, nrhs);
}

gk_status gk_green_plan_create(int64_t nt, const double* tx, const double* ty, const double* tz, int64_t ns,
                               const double* sx, const double* sy, const double* sz, const gk_kernel* kernel,
                               gk_green_plan** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("gk_green_plan_create: null output");
    *out = nullptr;
    check_kernel(kernel);
    if (nt < 0 || ns < 0) throw std::invalid_argument("gk_green_plan_create: negative size");
    if ((nt > 0 && (!tx || !ty || !tz)) || (ns > 0 && (!sx || !sy || !sz)))
      throw std::invalid_argument("gk_green_plan_create: null point array");
    require_device();
    auto P = std::make_unique<gk_green_plan>();
    P->nt_orig = nt;
    P->ns_orig = ns;
    P->helmholtz = kernel->kind == GK_HELMHOLTZ && kernel->k != 0.0;
    P->k = kernel->kind == GK_LAPLACE ? 0.0 : kernel->k;
    P->eps = guard_radius_pts(nt, tx, ty, tz, ns, sx, sy, sz);
    // merge twins: reuse the side machinery with one "element" per point
    auto uniq = [](int64_t n, const double* x, const double* y, const double* z, std::vector<double>& ux,
                   std::vector<double>& uy, std::vector<double>& uz, std::vector<int64_t>& loc) {
      std::vector<double> w(n, 1.0), basis(1, 1.0);
      std::vector<int32_t> dofs(n);
      for (int64_t i = 0; i < n; ++i) dofs[i] = (int32_t)i;
      gk_side s{n, x, y, z, w.data(), 1, n, 1, dofs.data(), basis.data(), n};
      Locations L = build_locations(s, "green_matvec");
      ux.assign(L.x.begin(), L.x.end());
      uy.assign(L.y.begin(), L.y.end());
      uz.assign(L.z.begin(), L.z.end());
      loc.assign(L.point_loc.begin(), L.point_loc.end());
    };
    std::vector<double> ux, uy, uz, vx, vy, vz;
    std::vector<int64_t> tloc, sloc;
    uniq(nt, tx, ty, tz, ux, uy, uz, tloc);
    uniq(ns, sx, sy, sz, vx, vy, vz, sloc);
    P->nt = (int64_t)ux.size();
    P->ns = (int64_t)vx.size();
    std::vector<int64_t> start(P->ns + 1, 0), list(ns);
    for (int64_t j = 0; j < ns; ++j) start[sloc[j] + 1]++;
    for (int64_t v = 0; v < P->ns; ++v) start[v + 1] += start[v];
    std::vector<int64_t> f(start.begin(), start.end() - 1);
    for (int64_t j = 0; j < ns; ++j) list[f[sloc[j]]++] = j;
    auto tof = [](const std::vector<double>& v) { return std::vector<float>(v.begin(), v.end()); };
    P->tx.upload(ux);
    P->ty.upload(uy);
    P->tz.upload(uz);
    P->txf.upload(tof(ux));
    P->tyf.upload(tof(uy));
    P->tzf.upload(tof(uz));
    P->sx.upload(vx);
    P->sy.upload(vy);
    P->sz.upload(vz);
    P->sxf.upload(tof(vx));
    P->syf.upload(tof(vy));
    P->szf.upload(tof(vz));
    P->src_start.upload(start);
    P->src_list.upload(list);
    P->tgt_loc.upload(tloc);
    P->Q.alloc(sizeof(gk_cplx) * std::max<int64_t>(1, P->ns));
    P->Y.alloc(sizeof(gk_cplx) * std::max<int64_t>(1, P->nt));
    // identical target and source sets (after the same twin merge): symmetric
    // fp64 path with ~512 MB of per-group partials (GK_GREEN_SYM=0 disables)
    const char* sym_env = std::getenv("GK_GREEN_SYM");
    const bool same = nt == ns && nt > 0 && std::memcmp(tx, sx, sizeof(double) * nt) == 0 &&
                      std::memcmp(ty, sy, sizeof(double) * nt) == 0 && std::memcmp(tz, sz, sizeof(double) * nt) == 0;
    if (same && !(sym_env && std::atoi(sym_env) == 0)) {
      const int64_t B = green_sym_block();
      const int64_t nb = (P->nt + B - 1) / B;
      const int64_t per_row = nb * B * (int64_t)sizeof(gk_cplx);
      const int64_t G = std::max<int64_t>(1, std::min<int64_t>(nb, (512ll << 20) / std::max<int64_t>(1, per_row)));
      if (nb * G < INT32_MAX) {
        P->symmetric = true;
        P->sym_group = (int)G;
        P->sym_R.alloc((size_t)(per_row * G));
        P->sym_C.alloc((size_t)(per_row * G));
      }
    }
    *out = P.release();
  });
}

gk_status gk_green_matvec(gk_green_plan* P, const gk_cplx* q, gk_cplx* y, int32_t precision, gk_stream stream) {
  return guard([&] {
    if (!P) throw std::invalid_argument("gk_green_matvec: null plan");
    if (precision != GK_FP64 && precision != GK_FP32)
      throw std::invalid_argument("gk_green_matvec: precision must be GK_FP64 or GK_FP32");
    if (P->nt_orig > 0 && !y) throw std::invalid_argument("gk_green_matvec: null output");
    if (P->ns_orig > 0 && !q) throw std::invalid_argument("gk_green_matvec: null charges");
    GreenArgs a;
    a.nt = P->nt;
    a.ns = P->ns;
    a.nsrc_orig = P->ns_orig;
    a.ntgt_orig = P->nt_orig;
    a.tx = P->tx.as<double>();
    a.ty = P->ty.as<double>();
    a.tz = P->tz.as<double>();
    a.txf = P->txf.as<float>();
    a.tyf = P->tyf.as<float>();
    a.tzf = P->tzf.as<float>();
    a.sx = P->sx.as<double>();
    a.sy = P->sy.as<double>();
    a.sz = P->sz.as<double>();
    a.sxf = P->sxf.as<float>();
    a.syf = P->syf.as<float>();
    a.szf = P->szf.as<float>();
    a.src_start = P->src_start.as<int64_t>();
    a.src_list = P->src_list.as<int64_t>();
    a.tgt_loc = P->tgt_loc.as<int64_t>();
    a.eps2 = P->eps * P->eps;
    a.kappa = 2.0 * P->k / M_PI;
    a.eps2f = (float)a.eps2;
    a.kappaf = (float)a.kappa;
    a.sym_R = P->symmetric ? P->sym_R.p : nullptr;
    a.sym_C = P->symmetric ? P->sym_C.p : nullptr;
    a.sym_group = P->sym_group;
    launch_green(a, q, P->Q.p, P->Y.p, y, precision, P->helmholtz, stream);
  });
}

gk_status gk_green_plan_get_info(const gk_green_plan* P, int64_t* nt, int64_t* ns, double* eps) {
  return guard([&] {
    if (!P) throw std::invalid_argument("gk_green_plan_get_info: null plan");
    if (nt) *nt = P->nt;
    if (ns) *ns = P->ns;
    if (eps) *eps = P->eps;
  });
}

int32_t gk_green_plan_is_symmetric(const gk_green_plan* P) { return P && P->symmetric ? 1 : 0; }

int32_t gk_green_plan_launches(const gk_green_plan* P, int32_t precision) {
  if (!P || P->nt_orig <= 0) return 0;
  int32_t n = (P->ns > 0 ? 1 : 0) + 1;  // merge charges, scatter targets
  if (P->symmetric) {
    const int64_t B = green_sym_block(), nb = (P->nt + B - 1) / B;
    n += 2 * (int32_t)((nb + P->sym_group - 1) / P->sym_group);  // tiles + reduce per group
  } else if (P->nt > 0) {
    n += 1;
  }
  (void)precision;
  return n;
}

gk_status gk_green_plan_destroy(gk_green_plan* P) {
  return guard([&] { delete P; });
}

gk_status gk_device_alloc(uint64_t bytes, void** ptr) {
  return guard([&] {
    if (!ptr) throw std::invalid_argument("gk_device_alloc: null output");
    require_device();
    *ptr = nullptr;
    if (bytes && cudaMalloc(ptr, bytes) != cudaSuccess) {
      cudaGetLastError();
      *ptr = nullptr;
      throw NoMemError("gk_device_alloc: " + std::to_string(bytes) + " bytes");
    }
  });
}

gk_status gk_device_free(void* ptr) {
  return guard([&] {
    if (ptr) cuda_check(cudaFree(ptr), "cudaFree");
  });
}

gk_status gk_copy_to_device(void* dst, const void* src, uint64_t bytes, gk_stream stream) {
  return guard([&] {
    if (bytes)
      cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream)),
                 "cudaMemcpyAsync H2D");
  });
}

gk_status gk_copy_to_host(void* dst, const void* src, uint64_t bytes, gk_stream stream) {
  return guard([&] {
    if (bytes)
      cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream)),
                 "cudaMemcpyAsync D2H");
  });
}

gk_status gk_stream_synchronize(gk_stream stream) {
  return guard([&] { cuda_check(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "cudaStreamSynchronize"); });
}

const char* gk_last_error(void) { return t_last_error.c_str(); }

const char* gk_version(void) { return "galerk_b200 0.1 (sm_100a)"; }

}  // extern "C"
