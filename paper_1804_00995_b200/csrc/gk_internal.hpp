// Internal (non-ABI) declarations shared by the galerk_b200 translation units.
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/galerk_b200.h"

namespace gk {

// ---- errors: exceptions inside, status codes + gk_last_error() at the ABI ----
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NoMemError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
void set_last_error(const std::string& msg);

template <class F>
gk_status guard(F&& f) {
  try {
    f();
    return GK_OK;
  } catch (const CudaError& e) {
    set_last_error(e.what());
    return GK_ECUDA;
  } catch (const NoMemError& e) {
    set_last_error(e.what());
    return GK_ENOMEM;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return GK_EINVAL;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return GK_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return GK_ERUNTIME;
  }
}

// ---- host allocator of the planner ------------------------------------------------
// The one-shot path plans on every call, and its large temporaries (hash
// tables, location and tile tables: tens of MB per cfg-2 plan) would otherwise
// come fresh from mmap each time and be page-faulted in again (~30% of the
// plan time measured).  Blocks of >= 64 KB are kept in a process-wide cache
// of size classes (up to 512 MB retained) and reused by later plans; smaller
// ones go straight to malloc.  Thread-safe.
void* plan_alloc(size_t bytes);
void plan_free(void* p, size_t bytes) noexcept;
size_t plan_cache_bytes();  // bytes currently retained by the cache
template <class T>
struct PlanAlloc {
  using value_type = T;
  PlanAlloc() = default;
  template <class U>
  PlanAlloc(const PlanAlloc<U>&) noexcept {}
  T* allocate(size_t n) { return static_cast<T*>(plan_alloc(n * sizeof(T))); }
  void deallocate(T* p, size_t n) noexcept { plan_free(p, n * sizeof(T)); }
  template <class U>
  bool operator==(const PlanAlloc<U>&) const noexcept { return true; }
  template <class U>
  bool operator!=(const PlanAlloc<U>&) const noexcept { return false; }
};
template <class T>
using hvec = std::vector<T, PlanAlloc<T>>;

void cuda_check(int err, const char* what);  // err is a cudaError_t
void require_device();

// ---- device buffers -----------------------------------------------------------
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    release();
    p = o.p;
    bytes = o.bytes;
    o.p = nullptr;
    o.bytes = 0;
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t n);
  void release();
  void upload(const void* src, size_t n);
  template <class T, class A>
  void upload(const std::vector<T, A>& v) {
    upload(v.data(), v.size() * sizeof(T));
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// One device allocation for many read-only tables: staged on the host at
// 256-byte aligned offsets, then one stream-ordered allocation from the
// device's default pool (cached between plans) and one copy.  Replaces a
// cudaMalloc/cudaMemcpy/cudaFree per table (~10 ms per one-shot plan).
struct DevArena {
  void* p = nullptr;
  size_t bytes = 0;
  hvec<char> host;
  DevArena() = default;
  DevArena(const DevArena&) = delete;
  DevArena& operator=(const DevArena&) = delete;
  ~DevArena() { release(); }
  // Optional: stage straight into the process-wide pinned buffer (held, with
  // its lock, until upload() or release()), so that each table is copied once
  // instead of into `host` (zero-filled first) and from there into the pinned
  // buffer.  `upper_bound` covers every later add(); a larger total falls back
  // to `host`.  Without this call add() stages in `host`.
  void begin_pinned(size_t upper_bound);
  template <class T>
  size_t add(const T* data, size_t n) {
    const size_t off = (used() + 255) & ~size_t(255);
    const size_t end = off + n * sizeof(T);
    if (pinned && end > pinned_cap) spill_pinned();
    if (pinned) {
      if (n) std::memcpy(pinned + off, data, n * sizeof(T));
      pinned_used = end;
    } else {
      host.resize(end);
      if (n) std::memcpy(host.data() + off, data, n * sizeof(T));
    }
    return off;
  }
  template <class V>
  size_t add(const V& v) {
    return add(v.data(), v.size());
  }
  // n uninitialised elements to be written in place before the next add()
  // (which may move the staging area)
  template <class T>
  T* alloc(size_t n, size_t& off) {
    off = (used() + 255) & ~size_t(255);
    const size_t end = off + n * sizeof(T);
    if (pinned && end > pinned_cap) spill_pinned();
    if (pinned) {
      pinned_used = end;
      return reinterpret_cast<T*>(pinned + off);
    }
    host.resize(end);
    return reinterpret_cast<T*>(host.data() + off);
  }
  // device-only bytes after the uploaded tables (filled on the device);
  // call after the last add()
  size_t add_device_only(size_t n) {
    const size_t off = (used() + 255) & ~size_t(255);
    extra = off + n - used();
    return off;
  }
  size_t extra = 0;
  void upload();  // allocate + copy; releases the host staging
  void release();
  template <class T>
  T* at(size_t off) const {
    return reinterpret_cast<T*>(static_cast<char*>(p) + off);
  }

 private:
  char* pinned = nullptr;  // the shared pinned staging buffer while this arena holds its lock
  size_t pinned_cap = 0, pinned_used = 0;
  size_t used() const { return pinned ? pinned_used : host.size(); }
  void spill_pinned();   // move what is staged into `host` and give the pinned buffer back
  void unlock_pinned();
};
void ensure_pool();  // default memory pool keeps up to 1 GB cached (per device)
constexpr int kMaxDevices = 64;  // process-wide device caches are per device index
int current_device();            // cudaGetDevice, checked against kMaxDevices

// ---- unique quadrature locations of one side (host) -----------------------------
// Points that are bit-identical (the edge-midpoint rule's twins, SURVEY trap 1)
// are merged into one location carrying the summed (dof, w*phi) contributions.
// The reference evaluates each twin separately and gets bit-identical kernel
// values, so merging only reorders the additions.
struct Locations {
  int64_t npts = 0, nfree = 0;
  hvec<double> x, y, z;           // [U]
  hvec<int64_t> cstart;           // [U+1]
  hvec<int32_t> cdof;             // contributing dof (original index)
  hvec<double> ccoef;             // sum over twins of w_k * phi_dof(x_k)
  hvec<int32_t> perm, iperm;      // locality order: perm[p] = dof
  bool natural = false;                  // perm is the identity
  int unit = 1;                          // RCB over aligned groups of `unit` consecutive dofs
  double xcut = 0.8;                     // x blocks cut back to a strong boundary in their last (1 - xcut)
  hvec<int8_t> strength;          // [nfree+1] boundary strength of each cut position
  hvec<int64_t> dstart;           // [nfree+1] by permuted dof
  hvec<int32_t> dloc;             // location id
  hvec<double> dcoef;
  hvec<int64_t> point_loc;        // [npts] location of each point
  int64_t size() const { return (int64_t)x.size(); }
};
Locations build_locations(const gk_side& s, const char* who);
bool sides_identical(const gk_side& a, const gk_side& b);
double guard_radius(const gk_side& a, const gk_side& b);  // kernels.cpp:14-19
double guard_radius_pts(int64_t na, const double* ax, const double* ay, const double* az,
                        int64_t nb, const double* bx, const double* by, const double* bz);

// ---- assembly tiling ----------------------------------------------------------------
// Tile shape.  A CTA alternates an FP64-bound pair loop with a latency-bound
// staging + gather phase, so the SM needs several independent CTAs at random
// phases to keep the FP64 pipe fed: four 128-thread CTAs per SM (16 warps;
// 121 registers x 512 threads fits the register file), shared memory per CTA
// = H (kJCap x kUCap x 16 B = 44 KB) + staged records and x supports (~10 KB).
// Measured on cfg 2: 2 x 256-thread CTAs (24-dof y blocks) 2.81 ms; 4 x
// 128-thread CTAs (22-dof y blocks) 2.57 ms although the smaller blocks
// evaluate 7% more pairs (halo 1.71 vs 1.61).
constexpr int kUCap = 128;   // x locations per tile, one per thread
constexpr int kJCap = 22;       // y dofs per tile (H accumulator rows)
constexpr int kJCapSmall = 16;  // alternative y-block cap the planner tries (layout_y_blocks)
constexpr int kIMax = 128;   // x dofs per tile
constexpr int kRCap = 112;   // y records per tile (staged in shared memory)
constexpr int kXsCap = 320;  // x support entries per tile (staged in shared memory)
constexpr int kAsmThreads = kUCap;
constexpr int kAlign = 16;   // natural-order block alignment (4^2 subdivision subtrees)
constexpr int kHS = kUCap;  // H row stride in 16-byte entries

struct YRec {  // one y location restricted to one tile's dofs (<= 2 slots)
  double x, y, z, c0, c1;
  int32_t off0, off1;  // byte offsets slot * kHS * 16 into H (off0: run slot, off1: read-modify-write slot or -1)
};
static_assert(sizeof(YRec) == 48, "YRec layout");
struct YRecU {  // the 32-byte record of the unit-coefficient mode (k_assemble SLOTS 3)
  double x, y, z;
  int32_t off0, off1;
};
static_assert(sizeof(YRecU) == 32, "YRecU layout");
// The device record table of a y side: YRecU for unit coefficients, else YRec.
hvec<char> device_records(const hvec<YRec>& recs, bool unit);
static_assert(kJCap <= 32, "per-block zero-fill mask is 32 bits");

// Dof order used for tiling: natural (input numbering; blocks cut at 4^k
// boundaries of subdivided meshes, rows of A stay contiguous) or recursive
// coordinate bisection of the dof locations (blocks cut at bisection splits).
void set_order(Locations& L, bool natural, int unit = 1, double xcut = 0.8);

struct TileTables {
  // x blocks
  hvec<int32_t> xb_dof_start;  // [nIb+1] permuted row ranges
  hvec<int32_t> xb_loc_start;  // [nIb+1]
  hvec<double> xl_x, xl_y, xl_z;
  hvec<int32_t> xsup_start;    // [nrows+1] by permuted row (global offsets)
  hvec<int32_t> xsup_u;        // local location index in its block
  hvec<double> xsup_c;
  // y blocks
  hvec<int32_t> yb_dof_start;  // [nJb+1]
  hvec<int32_t> yb_rec_start;  // [nJb+1]
  hvec<YRec> yrec;
  hvec<uint32_t> yb_zero;      // [nJb] bitmask of H rows with no run (need zero fill)
  // tiles: `masked` tiles may contain coincident location pairs and apply the
  // r^2 <= eps^2 mask; the others provably cannot (exact coincidences only,
  // checked on the host) and skip it.
  hvec<int32_t> tile_i, tile_j;          // unmasked tiles (listed only for the streamed path)
  int64_t n_unmasked = 0;
  hvec<int32_t> mtile_i, mtile_j;        // masked tiles
  bool has_second_slot = false;                 // any record with off1 >= 0
  bool equal_coefs = true;                      // every such record has c1 == c0 (bitwise)
  // unit_y: every y dof's contributions share one coefficient (P0 with an
  // equal-weight rule: w = area/g at every point), so records carry unit
  // coefficients and the dof's factor yscale[permuted dof] is applied once
  // per matrix entry in the gather instead of once per pair.
  bool unit_y = false;
  hvec<double> yscale;
  int64_t pairs_evaluated = 0;
  double x_halo = 0.0, y_halo = 0.0;
};
// Exact x/y location coincidences (the only pairs the r^2 <= eps^2 mask can
// hit when `unsafe` is false: no two points closer than 8 eps are distinct).
struct Coincidence {
  hvec<int32_t> y_of_x;  // y location with the same coordinates, or -1
  bool unsafe = false;          // some near-coincidence is not exact: mask every tile
};
Coincidence find_coincidences(const Locations& X, const Locations& Y, bool same, double eps);
// Block boundaries for the current dof orders and the pairs they evaluate
// (count-only: cheap enough to compare orders).
struct BlockLayout {
  hvec<int32_t> xb, xloc;  // x block dof starts [nIb+1], locations per block
  hvec<int32_t> yb, yrec;  // y block dof starts [nJb+1], records per block
  int64_t pairs = 0;       // location pairs the tiles evaluate
  int64_t lane_pairs = 0;  // the same with every x block rounded up to whole warps (issued work)
};
BlockLayout layout_blocks(const Locations& X, const Locations& Y, bool symmetric);
TileTables build_tiles(const Locations& X, const Locations& Y, bool symmetric, const Coincidence& C,
                       const BlockLayout& B);
// Picks natural vs RCB order by the evaluated pair count of the resulting
// tiles (natural preferred within 10%: coalesced writes); GK_ORDER=natural|rcb
// overrides.  Y may be null (symmetric: Y = X).
TileTables choose_order_and_tile(Locations& X, Locations* Y, bool symmetric, double eps);
// The pieces, for planners that tile one side once and the other in slabs.
struct OrderChoice {
  bool natural = true;
  int unit = 1;
  BlockLayout B;
  Coincidence C;
};
OrderChoice choose_order(Locations& X, Locations* Y, bool symmetric, double eps, double accept_natural = 0.0);
void layout_x_blocks(const Locations& X, BlockLayout& B);
void layout_y_blocks(const Locations& Y, BlockLayout& B);
void build_x_tables(const Locations& X, const BlockLayout& B, TileTables& T, hvec<int32_t>& xl_id);
void build_y_tables(const Locations& Y, const BlockLayout& B, TileTables& T, hvec<int64_t>& yb_start,
                    hvec<int32_t>& yb_list);
void build_tile_list(const TileTables& TX, TileTables& T, bool symmetric, const Coincidence& C,
                     const hvec<int32_t>& xl_id, const hvec<int64_t>& yb_start,
                     const hvec<int32_t>& yb_list, bool list_unmasked = true);
// Trial locations restricted to dofs [c0, c1) (renumbered from 0, natural
// order not yet set); slab_of_full maps full location ids to slab ids or -1.
Locations restrict_cols(const Locations& Y, int64_t c0, int64_t c1, hvec<int32_t>& slab_of_full);
// Run this thread's planner loops serially (slab workers run one slab per thread).
void planner_serial(bool on);
// Host threads the planner and the streamed path use: GK_THREADS, else the
// hardware threads divided among the node's ranks (LOCAL_WORLD_SIZE), <= 16.
int host_threads();

struct TileDesc {  // everything a k_assemble CTA needs to stage its tile
  int32_t i0, nI;      // x block: first permuted row, rows
  int32_t j0, nJ;      // y block: first permuted column, columns
  int32_t l0, nu;      // x locations
  int32_t r0, nrec;    // y records
  int32_t xs0, nxs;    // x support entries
  uint32_t zero_rows;  // H rows without a run (zero-filled)
  int32_t masked;      // 1: the tile may hold a coincident pair (distance mask on)
};
static_assert(sizeof(TileDesc) == 48, "TileDesc is loaded as three 16-byte vectors");

struct AsmArgs {
  const TileDesc* tiles;
  const double* xl_x;
  const double* xl_y;
  const double* xl_z;
  const int32_t* xsup_start;
  const int32_t* xsup_u;
  const double* xsup_c;
  const YRec* yrec;
  const int32_t* xperm;
  const int32_t* yperm;
  const double* yscale;  // [permuted y dof] (slots == 3 only)
  void* A;
  int64_t lda;
  double eps2;
  double kappa;  // 2k/pi
  int32_t symmetric;
  int32_t natural;  // dof orders are the identity: A's indices are the permuted ones (no perm lookups)
  unsigned long long* prof;  // diagnostics: [tile][4] phase cycles + SM id, or null
  int32_t jmax;              // widest y block of the launch (dofs): selects the kernel shape (16 or 22)
  const void* l2_window;     // host side only: tables to keep in a persisting L2 window for the launch (or null)
  uint64_t l2_window_bytes;
  int32_t dbg;               // timing experiments only (GK_ASM_DBG; results invalid when set): 1 no stores, 2 no gather, 4 no pair loop, 8 no second-slot read-modify-write, 16 no direct stores, 32 no mirror stores
};
// Entries of oversized dofs (rows `rows` x all columns, all rows x columns
// `cols`; symmetric: rows == cols and both orientations are written), one
// thread per entry from the full per-dof tables: A_ij = sum_u c_ui sum_v c_vj
// G(u, v) with the distance mask, in bem_product's nesting.
struct BigArgs {
  const int32_t* rows;
  const int32_t* cols;
  int64_t nbig_rows, nbig_cols, nrows, ncols;
  const int64_t* xs;
  const int32_t* xl;
  const double* xc;
  const double* xp;  // [U][3]
  const int64_t* ys;
  const int32_t* yl;
  const double* yc;
  const double* yp;
  void* A;
  int64_t lda;
  double eps2, kappa;
  int32_t symmetric;
};
void launch_big_entries(const BigArgs& b, bool helmholtz, void* stream);
// slots: 0 = no second slots, 1 = second slots, 2 = second slots with c1 == c0,
// 3 = unit coefficients with per-column scales (TileTables::unit_y)
void launch_assemble(const AsmArgs& a, int64_t ntiles, bool helmholtz, int slots, void* stream);
// Tile descriptors built on the device from the block tables: every x block
// bi owns the tiles (bi, bj) for bj in [first_bj[bi], nJb), numbered in
// (bi, bj) order from tile_start[bi]; `masked_bits` flags the masked ones.
// (The descriptors are 48 B per tile — 157 MB for cfg 4 — and building and
// uploading them on the host cost ~70 ms per plan.)
struct TileBuildArgs {
  TileDesc* out;
  int64_t ntiles;
  int32_t nIb;
  const int64_t* tile_start;    // [nIb + 1]
  const int32_t* first_bj;      // [nIb]
  const int32_t* xb_dof_start;  // [nIb + 1]
  const int32_t* xb_loc_start;  // [nIb + 1]
  const int32_t* yb_dof_start;  // [nJb + 1]
  const int32_t* yb_rec_start;  // [nJb + 1]
  const uint32_t* yb_zero;      // [nJb]
  const int32_t* xsup_start;    // [rows + 1]
  const uint32_t* masked_bits;  // [ceil(ntiles / 32)]
};
void launch_make_tiles(const TileBuildArgs& b, void* stream);
// Copy ceil(bytes/16) 16-byte words from mapped pinned host memory (device
// view) to device memory with SM loads (both 16-byte aligned and padded).
void launch_fetch_tables(void* dst, const void* src_mapped, size_t bytes, void* stream);

// ---- matvec ---------------------------------------------------------------------------
void launch_matvec(const void* A, int64_t rows, int64_t cols, int64_t lda, const void* x, void* y,
                   void* stream);
int matvec_launch_count(int64_t rows, int64_t cols);
void launch_matvec_multi(const void* A, int64_t rows, int64_t cols, int64_t lda, const void* X, int64_t ldx, void* Y,
                         int64_t ldy, int32_t nrhs, void* stream);
int matvec_multi_launch_count(int64_t rows, int64_t cols, int32_t nrhs);

// ---- green matvec ------------------------------------------------------------------------
struct GreenArgs {
  int64_t nt, ns, nsrc_orig, ntgt_orig;
  const double* tx;
  const double* ty;
  const double* tz;
  const float* txf;
  const float* tyf;
  const float* tzf;
  const double* sx;
  const double* sy;
  const double* sz;
  const float* sxf;
  const float* syf;
  const float* szf;
  const int64_t* src_start;  // [ns+1] CSR: unique source -> original sources
  const int64_t* src_list;
  const int64_t* tgt_loc;    // [ntgt_orig] original target -> unique target
  double eps2;
  double kappa;
  float eps2f;
  float kappaf;
  void* sym_R;    // targets == sources: per-group row / column partials (null: general path)
  void* sym_C;
  int32_t sym_group;  // target blocks per group
};
int green_sym_block();  // locations per block of the symmetric path
void launch_green(const GreenArgs& a, const void* q, void* Q, void* Y, void* y, int precision,
                  bool helmholtz, void* stream);

}  // namespace gk
