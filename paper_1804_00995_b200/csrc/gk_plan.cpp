// Host-side plan construction for the dense assembly (runs once per operator;
// the timed device work is gk_plan_assemble).  Replaces the host part of
// make_side (assembly.cpp:144-171): the reference builds complex CSC
// matrices (W B)^T and per-dof std::map lists; here the same information is
// laid out for the device as unique locations + per-tile tables.
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <numeric>
#include <cstdlib>
#include <exception>
#include <future>
#include <mutex>
#include <thread>
#include <unordered_map>

#include "gk_internal.hpp"

namespace gk {

// ---- planner allocator (gk_internal.hpp) ----------------------------------------
namespace {
constexpr size_t kPoolMin = size_t(64) << 10;       // smaller blocks: plain malloc
constexpr size_t kPoolCap = size_t(512) << 20;      // retained bytes at most
// size class: the request rounded up to 1/8 of its power-of-two range (<= 12.5% waste)
size_t pool_class_bytes(size_t bytes) {
  size_t p = 1;
  while (p < bytes) p <<= 1;
  const size_t step = std::max<size_t>(p >> 3, 4096);
  return (bytes + step - 1) / step * step;
}
struct PlanPool {
  std::mutex m;
  std::unordered_map<size_t, std::vector<void*>> free;  // class bytes -> cached blocks
  size_t retained = 0;
  ~PlanPool() {
    for (auto& kv : free)
      for (void* p : kv.second) std::free(p);
  }
};
PlanPool& plan_pool() {
  static PlanPool* pool = new PlanPool();  // never destroyed: deallocations may run at exit
  return *pool;
}
}  // namespace

void* plan_alloc(size_t bytes) {
  if (bytes < kPoolMin) {
    void* p = std::malloc(bytes ? bytes : 1);
    if (!p) throw std::bad_alloc();
    return p;
  }
  const size_t c = pool_class_bytes(bytes);
  PlanPool& P = plan_pool();
  {
    std::lock_guard<std::mutex> g(P.m);
    auto it = P.free.find(c);
    if (it != P.free.end() && !it->second.empty()) {
      void* p = it->second.back();
      it->second.pop_back();
      P.retained -= c;
      return p;
    }
  }
  void* p = std::malloc(c);
  if (!p) throw std::bad_alloc();
  return p;
}

void plan_free(void* p, size_t bytes) noexcept {
  if (!p) return;
  if (bytes < kPoolMin) {
    std::free(p);
    return;
  }
  const size_t c = pool_class_bytes(bytes);
  PlanPool& P = plan_pool();
  {
    std::lock_guard<std::mutex> g(P.m);
    if (P.retained + c <= kPoolCap) {
      try {
        P.free[c].push_back(p);
        P.retained += c;
        return;
      } catch (...) {  // bookkeeping allocation failed: release the block instead
      }
    }
  }
  std::free(p);
}

size_t plan_cache_bytes() {
  PlanPool& P = plan_pool();
  std::lock_guard<std::mutex> g(P.m);
  return P.retained;
}

namespace {
thread_local bool t_serial = false;  // set by callers that already run one task per thread
struct Key {
  uint64_t a, b, c;
  bool operator==(const Key& o) const { return a == o.a && b == o.b && c == o.c; }
};
struct KeyHash {  // splitmix64-style mixing of the three coordinate bit patterns
  static uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  size_t operator()(const Key& k) const {
    return (size_t)mix(k.a ^ mix(k.b ^ mix(k.c + 0x9E3779B97F4A7C15ULL)));
  }
};
uint64_t bits(double v) {
  v += 0.0;  // -0.0 -> +0.0 (same location)
  uint64_t u;
  std::memcpy(&u, &v, 8);
  return u;
}
}  // namespace

double guard_radius_pts(int64_t na, const double* ax, const double* ay, const double* az,
                        int64_t nb, const double* bx, const double* by, const double* bz) {
  if (na == 0 || nb == 0) return 0.0;  // kernels.cpp:14-19
  double lo[3] = {ax[0], ay[0], az[0]}, hi[3] = {ax[0], ay[0], az[0]};
  auto upd = [&](double x, double y, double z) {
    const double p[3] = {x, y, z};
    for (int c = 0; c < 3; ++c) {
      lo[c] = std::min(lo[c], p[c]);
      hi[c] = std::max(hi[c], p[c]);
    }
  };
  for (int64_t i = 0; i < na; ++i) upd(ax[i], ay[i], az[i]);
  for (int64_t i = 0; i < nb; ++i) upd(bx[i], by[i], bz[i]);
  const double d0 = hi[0] - lo[0], d1 = hi[1] - lo[1], d2 = hi[2] - lo[2];
  return 1e-12 * std::sqrt(d0 * d0 + d1 * d1 + d2 * d2);
}

double guard_radius(const gk_side& a, const gk_side& b) {
  return guard_radius_pts(a.npts, a.x, a.y, a.z, b.npts, b.x, b.y, b.z);
}

static void validate(const gk_side& s, const char* who) {
  if (s.npts < 0 || s.nelem < 0 || s.nfree < 0)
    throw std::invalid_argument(std::string(who) + ": negative size");
  if (s.g <= 0 || s.nloc <= 0) throw std::invalid_argument(std::string(who) + ": g and nloc must be positive");
  if (s.npts != s.nelem * (int64_t)s.g)
    throw std::invalid_argument(std::string(who) + ": npts must equal nelem * g (point e*g+q belongs to element e)");
  if (s.npts > 0 && (!s.x || !s.y || !s.z || !s.w || !s.elem_dofs || !s.basis))
    throw std::invalid_argument(std::string(who) + ": null array");
  if (s.nfree > INT32_MAX) throw std::invalid_argument(std::string(who) + ": too many dofs");
  if (s.npts > INT32_MAX) throw std::invalid_argument(std::string(who) + ": too many quadrature points");
}

bool sides_identical(const gk_side& a, const gk_side& b) {
  if (&a == &b) return true;
  if (a.npts != b.npts || a.g != b.g || a.nelem != b.nelem || a.nloc != b.nloc || a.nfree != b.nfree)
    return false;
  auto same = [](const void* p, const void* q, size_t n) { return p == q || std::memcmp(p, q, n) == 0; };
  const size_t m = (size_t)a.npts * sizeof(double);
  return same(a.x, b.x, m) && same(a.y, b.y, m) && same(a.z, b.z, m) && same(a.w, b.w, m) &&
         same(a.elem_dofs, b.elem_dofs, (size_t)a.nelem * a.nloc * sizeof(int32_t)) &&
         same(a.basis, b.basis, (size_t)a.g * a.nloc * sizeof(double));
}

Locations build_locations(const gk_side& s, const char* who) {
  const bool timing = std::getenv("GK_TIMING") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[gk_plan]   %-20s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  validate(s, who);
  lap("validate");
  Locations L;
  L.npts = s.npts;
  L.nfree = s.nfree;
  L.point_loc.resize(s.npts);
  // Location ids in first-seen point order.  Large sides: hash-sharded on the
  // planner's threads — thread q owns the keys whose hash falls in its slice,
  // scans all points in order and records for each of its points the first
  // point with the same key (its own small table stays in cache); the ids are
  // then the ranks of the first occurrences, exactly the serial numbering.
  const int nth = t_serial ? 1 : (int)std::min<int64_t>(host_threads(), s.npts / 16384);
  if (nth > 1) {
    const size_t n = (size_t)s.npts;
    hvec<uint64_t> hs(n);
    hvec<int32_t> rep(n);  // first point with the same coordinates
    auto fan = [&](auto&& fn) {
      std::vector<std::thread> pool;
      for (int q = 1; q < nth; ++q) pool.emplace_back([&fn, q] { fn(q); });
      fn(0);
      for (auto& th : pool) th.join();
    };
    const KeyHash hasher;
    fan([&](int q) {
      for (size_t k = n * q / nth; k < n * (q + 1) / nth; ++k)
        hs[k] = hasher(Key{bits(s.x[k]), bits(s.y[k]), bits(s.z[k])});
    });
    fan([&](int q) {
      // slice of the hash space by the top bits; table of >= 2x the expected keys
      size_t cap = 16;
      while (cap < 3 * n / (size_t)nth) cap <<= 1;
      hvec<int32_t> slot(cap, -1);
      for (size_t k = 0; k < n; ++k) {
        const uint64_t hv = hs[k];
        if ((int)(((hv >> 40) * (uint64_t)nth) >> 24) != q) continue;
        const Key key{bits(s.x[k]), bits(s.y[k]), bits(s.z[k])};
        size_t h = hv & (cap - 1);
        for (;;) {
          const int32_t f = slot[h];
          if (f < 0) {
            slot[h] = (int32_t)k;
            rep[k] = (int32_t)k;
            break;
          }
          if (hs[(size_t)f] == hv && bits(s.x[f]) == key.a && bits(s.y[f]) == key.b && bits(s.z[f]) == key.c) {
            rep[k] = f;
            break;
          }
          h = (h + 1) & (cap - 1);
        }
      }
    });
    int64_t U = 0;
    for (size_t k = 0; k < n; ++k)
      if (rep[k] == (int32_t)k) L.point_loc[k] = U++;
    L.x.resize((size_t)U);
    L.y.resize((size_t)U);
    L.z.resize((size_t)U);
    fan([&](int q) {
      for (size_t k = n * q / nth; k < n * (q + 1) / nth; ++k) {
        const int32_t f = rep[k];
        if (f == (int32_t)k) {
          const int64_t u = L.point_loc[k];
          L.x[(size_t)u] = s.x[k];
          L.y[(size_t)u] = s.y[k];
          L.z[(size_t)u] = s.z[k];
        } else {
          L.point_loc[k] = L.point_loc[(size_t)f];  // f < k: a first occurrence, numbered by the serial pass
        }
      }
    });
  } else {
    // open-addressing table of location ids keyed by the coordinate bit
    // patterns (linear probing, load <= 1/2); ids in first-seen point order.
    // The table is far larger than the host caches (cfg 4: 4 MB for 245,760
    // points), so the hashes are formed in a first pass and each probe's slot is
    // prefetched a few points ahead; a slot holds the id and 32 hash bits that
    // filter out nearly every foreign key without touching the key array.
    size_t cap = 16;
    while (cap < 2 * (size_t)s.npts) cap <<= 1;
    struct Slot {
      int32_t id;
      uint32_t tag;
    };
    hvec<Slot> slot(cap, Slot{-1, 0u});
    hvec<Key> keys;
    keys.reserve((size_t)s.npts);
    L.x.reserve((size_t)s.npts);
    L.y.reserve((size_t)s.npts);
    L.z.reserve((size_t)s.npts);
    const KeyHash hasher;
    hvec<uint64_t> hs((size_t)s.npts);
    for (int64_t k = 0; k < s.npts; ++k) hs[(size_t)k] = hasher(Key{bits(s.x[k]), bits(s.y[k]), bits(s.z[k])});
    constexpr int64_t kAhead = 16;
    for (int64_t k = 0; k < s.npts; ++k) {
      if (k + kAhead < s.npts) __builtin_prefetch(&slot[hs[(size_t)(k + kAhead)] & (cap - 1)], 1);
      const Key key{bits(s.x[k]), bits(s.y[k]), bits(s.z[k])};
      const uint64_t hv = hs[(size_t)k];
      const uint32_t tag = (uint32_t)(hv >> 32);
      size_t h = hv & (cap - 1);
      while (slot[h].id >= 0 && !(slot[h].tag == tag && keys[(size_t)slot[h].id] == key)) h = (h + 1) & (cap - 1);
      if (slot[h].id < 0) {
        const int64_t u = (int64_t)L.x.size();
        slot[h] = Slot{(int32_t)u, tag};
        keys.push_back(key);
        L.x.push_back(s.x[k]);
        L.y.push_back(s.y[k]);
        L.z.push_back(s.z[k]);
        L.point_loc[k] = u;
      } else {
        L.point_loc[k] = slot[h].id;
      }
    }
  }
  lap("location ids");
  const int64_t U = L.size();
  // contributions: (dof, w_k * phi) for nonzero basis values of free dofs
  // (femspace.cpp:476-484 skips exact zeros and constrained dofs), merged per
  // (location, dof) in point order.
  hvec<int64_t> cnt(U + 1, 0);
  for (int64_t k = 0; k < s.npts; ++k) cnt[L.point_loc[k] + 1] += s.nloc;
  for (int64_t u = 0; u < U; ++u) cnt[u + 1] += cnt[u];
  hvec<int32_t> tdof(cnt[U]);
  hvec<double> tcoef(cnt[U]);
  hvec<int64_t> fill(cnt.begin(), cnt.end() - 1), used(U, 0);
  for (int64_t k = 0; k < s.npts; ++k) {
    const int64_t e = k / s.g;
    const int q = (int)(k % s.g);
    const int64_t u = L.point_loc[k];
    for (int l = 0; l < s.nloc; ++l) {
      const int32_t dof = s.elem_dofs[e * s.nloc + l];
      const double b = s.basis[(int64_t)q * s.nloc + l];
      if (dof < 0 || b == 0.0) continue;
      if (dof >= s.nfree) throw std::invalid_argument(std::string(who) + ": dof index out of range");
      const double c = s.w[k] * b;
      int64_t base = cnt[u], n = used[u], p = base;
      for (; p < base + n; ++p)
        if (tdof[p] == dof) break;
      if (p < base + n) {
        tcoef[p] += c;
      } else {
        tdof[p] = dof;
        tcoef[p] = c;
        used[u]++;
      }
    }
  }
  (void)fill;
  L.cstart.assign(U + 1, 0);
  for (int64_t u = 0; u < U; ++u) L.cstart[u + 1] = L.cstart[u] + used[u];
  L.cdof.resize(L.cstart[U]);
  L.ccoef.resize(L.cstart[U]);
  for (int64_t u = 0; u < U; ++u)
    for (int64_t i = 0; i < used[u]; ++i) {
      L.cdof[L.cstart[u] + i] = tdof[cnt[u] + i];
      L.ccoef[L.cstart[u] + i] = tcoef[cnt[u] + i];
    }
  lap("contributions");
  set_order(L, true);
  lap("natural order");
  return L;
}

namespace {
// per permuted dof: (location, coef) in location order
void finalize_perm(Locations& L) {
  const int64_t U = L.size(), n = L.nfree;
  L.iperm.assign(n, -1);
  for (int64_t p = 0; p < n; ++p) L.iperm[L.perm[p]] = (int32_t)p;
  L.dstart.assign(n + 1, 0);
  for (int64_t p = 0; p < L.cstart[U]; ++p) L.dstart[L.iperm[L.cdof[p]] + 1]++;
  for (int64_t d = 0; d < n; ++d) L.dstart[d + 1] += L.dstart[d];
  L.dloc.resize(L.cstart[U]);
  L.dcoef.resize(L.cstart[U]);
  hvec<int64_t> f(L.dstart.begin(), L.dstart.end() - 1);
  for (int64_t u = 0; u < U; ++u)
    for (int64_t p = L.cstart[u]; p < L.cstart[u + 1]; ++p) {
      const int32_t pd = L.iperm[L.cdof[p]];
      L.dloc[f[pd]] = (int32_t)u;
      L.dcoef[f[pd]] = L.ccoef[p];
      f[pd]++;
    }
}

double env_frac(const char* name, double dflt) {
  const char* e = std::getenv(name);
  return e ? std::atof(e) : dflt;
}

struct RcbPoint {
  double c[3];
  int32_t dof;
};

void rcb(hvec<RcbPoint>& pts, int64_t lo, int64_t hi, int64_t leaf, int depth, hvec<int8_t>& strength) {
  if (hi - lo <= leaf) return;
  double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
  for (int64_t i = lo; i < hi; ++i)
    for (int c = 0; c < 3; ++c) {
      mn[c] = std::min(mn[c], pts[i].c[c]);
      mx[c] = std::max(mx[c], pts[i].c[c]);
    }
  int ax = 0;
  for (int c = 1; c < 3; ++c)
    if (mx[c] - mn[c] > mx[ax] - mn[ax]) ax = c;
  const int64_t mid = lo + (hi - lo) / 2;
  std::nth_element(pts.begin() + lo, pts.begin() + mid, pts.begin() + hi, [ax](const RcbPoint& a, const RcbPoint& b) {
    return a.c[ax] < b.c[ax] || (a.c[ax] == b.c[ax] && a.dof < b.dof);
  });
  strength[mid] = (int8_t)std::max<int>(strength[mid], 60 - depth);
  rcb(pts, lo, mid, leaf, depth + 1, strength);
  rcb(pts, mid, hi, leaf, depth + 1, strength);
}
}  // namespace

void set_order(Locations& L, bool natural, int unit_req, double xcut) {
  const int64_t n = L.nfree, U = L.size();
  L.natural = natural;
  L.unit = natural ? 1 : std::max(1, (int)env_frac("GK_UNIT", unit_req));
  L.xcut = env_frac("GK_XCUT", xcut);
  L.strength.assign(n + 1, 0);
  if (natural) {
    // subdivided meshes number children 4-by-4: boundaries at multiples of 4^k
    L.perm.resize(n);
    std::iota(L.perm.begin(), L.perm.end(), 0);
    for (int64_t p = 0; p <= n; ++p) {
      int s = 0;
      for (int64_t q = p; q > 0 && q % 4 == 0 && s < 30; q /= 4) ++s;
      L.strength[p] = (int8_t)s;
    }
  } else {
    // recursive coordinate bisection of the dof locations (mean of their
    // supporting quadrature locations); unsupported dofs go last.
    hvec<double> sx(n, 0.0), sy(n, 0.0), sz(n, 0.0);
    hvec<int64_t> cnt(n, 0);
    for (int64_t u = 0; u < U; ++u)
      for (int64_t p = L.cstart[u]; p < L.cstart[u + 1]; ++p) {
        const int32_t d = L.cdof[p];
        sx[d] += L.x[u];
        sy[d] += L.y[u];
        sz[d] += L.z[u];
        cnt[d]++;
      }
    // RCB over units of `unit` consecutive dofs (aligned groups): the rows
    // of a unit stay adjacent in every block, so matrix writes come in whole
    // 32-byte sectors (unit 2) instead of scattered 16-byte halves.
    const int64_t unit = L.unit;
    hvec<RcbPoint> pts;
    pts.reserve(n / unit + 1);
    for (int64_t d0 = 0; d0 < n; d0 += unit) {
      double c[3] = {0, 0, 0};
      int64_t m = 0;
      for (int64_t d = d0; d < std::min(n, d0 + unit); ++d) {
        if (!cnt[d]) continue;
        c[0] += sx[d] / cnt[d];
        c[1] += sy[d] / cnt[d];
        c[2] += sz[d] / cnt[d];
        ++m;
      }
      if (m) pts.push_back({{c[0] / m, c[1] / m, c[2] / m}, (int32_t)d0});
    }
    hvec<int8_t> ustrength(pts.size() + 1, 0);
    rcb(pts, 0, (int64_t)pts.size(), std::max<int64_t>(1, 4 / unit), 0, ustrength);
    L.perm.clear();
    L.perm.reserve(n);
    hvec<char> placed(n, 0);
    for (size_t u = 0; u < pts.size(); ++u) {
      const int64_t pos = (int64_t)L.perm.size();
      L.strength[pos] = ustrength[u];
      for (int64_t d = pts[u].dof; d < std::min(n, (int64_t)pts[u].dof + unit); ++d)
        if (cnt[d]) {
          if (L.perm.size() > (size_t)pos) L.strength[L.perm.size()] = -1;  // inside a unit: never cut
          L.perm.push_back((int32_t)d);
          placed[d] = 1;
        }
    }
    for (int64_t d = 0; d < n; ++d)
      if (!placed[d]) L.perm.push_back((int32_t)d);
  }
  L.strength[0] = L.strength[n] = 127;
  finalize_perm(L);
}

namespace {
// Cut a greedy block [start, end_max) back to the strongest order boundary in
// its last 20% so blocks are unions of whole spatial clusters.
int64_t cut(const Locations& L, int64_t start, int64_t end_max, double frac = 0.8) {
  if (end_max >= L.nfree) return end_max;
  if (frac >= 1.0) {  // no preference: the last position that is not inside a unit
    int64_t e = end_max;
    while (e > start + 1 && L.strength[e] < 0) --e;
    return e;
  }
  const int64_t lo = start + std::max<int64_t>(1, (int64_t)std::ceil(frac * (double)(end_max - start)));
  int64_t best = end_max;
  for (int64_t e = end_max; e >= lo; --e)
    if (L.strength[e] > L.strength[best]) best = e;
  return best;
}
}  // namespace

void layout_x_blocks(const Locations& X, BlockLayout& B) {
  const int64_t nrows = X.nfree;
  B.xb.clear();
  B.xloc.clear();
  // ---- x blocks: consecutive permuted rows while their locations fit kUCap,
  // cut back to the strongest order boundary
  hvec<int64_t> owner(X.size(), -1);
  int64_t p = 0, trial_id = 0;
  B.xb.push_back(0);
  while (p < nrows) {
    const int64_t start = p;
    int64_t end = start, nl = 0, ns = 0;
    ++trial_id;
    while (end < nrows && end - start < kIMax) {
      int fresh = 0;  // a row lists each location once (merged per (location, dof))
      for (int64_t s = X.dstart[end]; s < X.dstart[end + 1]; ++s) fresh += owner[X.dloc[s]] != trial_id;
      const int64_t nsup = X.dstart[end + 1] - X.dstart[end];
      if (nl + fresh > kUCap || ns + nsup > kXsCap) break;
      for (int64_t s = X.dstart[end]; s < X.dstart[end + 1]; ++s) owner[X.dloc[s]] = trial_id;
      nl += fresh;
      ns += nsup;
      ++end;
    }
    if (end == start)
      throw std::invalid_argument("bem_dense: a test dof is supported by more than " + std::to_string(kUCap) +
                                  " quadrature locations");
    end = cut(X, start, end, X.xcut);
    ++trial_id;  // count the locations of the final block
    int64_t nloc = 0;
    for (int64_t q = start; q < end; ++q)
      for (int64_t s = X.dstart[q]; s < X.dstart[q + 1]; ++s)
        if (owner[X.dloc[s]] != trial_id) {
          owner[X.dloc[s]] = trial_id;
          ++nloc;
        }
    B.xb.push_back((int32_t)end);
    B.xloc.push_back((int32_t)nloc);
    p = end;
  }
}

namespace {
void layout_y_blocks_cap(const Locations& Y, BlockLayout& B, int64_t cap) {
  const int64_t ncols = Y.nfree;
  B.yb.clear();
  B.yrec.clear();
  // ---- y blocks: up to kJCap consecutive permuted cols (fewer if their
  // records would exceed kRCap), cut back to the strongest order boundary
  hvec<int64_t> ystamp(Y.size(), -1);
  int64_t sid = 0;
  auto count_records = [&](int64_t q0, int64_t q1) {
    ++sid;
    int64_t n = 0;
    for (int64_t q = q0; q < q1; ++q)
      for (int64_t s = Y.dstart[q]; s < Y.dstart[q + 1]; ++s) {
        const int32_t v = Y.dloc[s];
        if (ystamp[v] == sid) continue;
        ystamp[v] = sid;
        int slots = 0;
        for (int64_t c = Y.cstart[v]; c < Y.cstart[v + 1]; ++c) {
          const int32_t pq = Y.iperm[Y.cdof[c]];
          slots += pq >= q0 && pq < q1;
        }
        n += (slots + 1) / 2;
      }
    return n;
  };
  B.yb.push_back(0);
  for (int64_t q0 = 0; q0 < ncols;) {
    int64_t q1 = std::min<int64_t>(ncols, q0 + cap);
    int64_t nrec = count_records(q0, q1);
    while (nrec > kRCap && q1 - q0 > 1) {
      q1 = q0 + std::max<int64_t>(1, (q1 - q0) * 7 / 8);
      nrec = count_records(q0, q1);
    }
    const int64_t qc = cut(Y, q0, q1, env_frac("GK_YCUT", 0.8));
    if (qc != q1) {
      q1 = qc;
      nrec = count_records(q0, q1);
    }
    if (nrec > kRCap)
      throw std::invalid_argument("bem_dense: a trial dof is supported by more than " + std::to_string(kRCap) +
                                  " quadrature locations");
    B.yb.push_back((int32_t)q1);
    B.yrec.push_back((int32_t)nrec);
    q0 = q1;
  }
}

}  // namespace

// y blocks of at most kJCap dofs, or of at most kJCapSmall when that needs
// fewer records in total (records x x locations = evaluated pairs): on a
// subdivided mesh in natural order, 16 dofs are one 4^2 subtree (P0 L6, cfg 4:
// y halo 1.25 instead of 1.34, 7% fewer evaluated pairs, measured 46.2 ->
// 44.6 ms), while P1 vertex blocks (cfg 2) keep 22.
void layout_y_blocks(const Locations& Y, BlockLayout& B) {
  if (std::getenv("GK_JCAP")) {  // diagnostics: a fixed cap
    layout_y_blocks_cap(Y, B, std::max<int64_t>(1, std::min<int64_t>(kJCap, (int64_t)env_frac("GK_JCAP", kJCap))));
    return;
  }
  layout_y_blocks_cap(Y, B, kJCap);
  if (kJCapSmall >= kJCap) return;
  BlockLayout S;
  layout_y_blocks_cap(Y, S, kJCapSmall);
  int64_t rb = 0, rs = 0;
  for (int32_t r : B.yrec) rb += r;
  for (int32_t r : S.yrec) rs += r;
  if (rs < rb) {
    B.yb = std::move(S.yb);
    B.yrec = std::move(S.yrec);
  }
}

int64_t layout_pairs(const BlockLayout& B, bool symmetric, bool lanes = false) {
  int64_t pairs = 0;
  // ---- evaluated pairs: symmetric plans keep tiles whose last column >= first row
  const int64_t nJb = (int64_t)B.yrec.size();
  hvec<int64_t> suffix(nJb + 1, 0);
  for (int64_t bj = nJb - 1; bj >= 0; --bj) suffix[bj] = suffix[bj + 1] + B.yrec[bj];
  for (size_t bi = 0; bi < B.xloc.size(); ++bi) {
    int64_t first = 0;
    if (symmetric)  // first y block with yb[bj+1] - 1 >= xb[bi]
      first = std::upper_bound(B.yb.begin() + 1, B.yb.end(), B.xb[bi]) - (B.yb.begin() + 1);
    pairs += (int64_t)(lanes ? (B.xloc[bi] + 31) / 32 * 32 : B.xloc[bi]) * suffix[first];
  }
  return pairs;
}

BlockLayout layout_blocks(const Locations& X, const Locations& Y, bool symmetric) {
  BlockLayout B;
  layout_x_blocks(X, B);
  layout_y_blocks(Y, B);
  B.pairs = layout_pairs(B, symmetric);
  B.lane_pairs = layout_pairs(B, symmetric, true);
  return B;
}

int host_threads() {
  static const int n = [] {
    const char* e = std::getenv("GK_THREADS");
    if (e) return std::max(1, std::atoi(e));
    int hw = (int)std::max(1u, std::thread::hardware_concurrency());
    // one process per GPU (torchrun exports LOCAL_WORLD_SIZE): share the node's cores
    const char* lw = std::getenv("LOCAL_WORLD_SIZE");
    if (lw && std::atoi(lw) > 1) hw = std::max(1, hw / std::atoi(lw));
    return std::min(hw, 16);
  }();
  return n;
}

namespace {
// Static-partition parallel loop over [0, n) on up to host_threads() threads;
// fn(begin, end) per chunk.
template <class F>
void parallel_for(int64_t n, F&& fn) {
  const int nthreads = host_threads();
  const int nt = t_serial ? 1 : (int)std::min<int64_t>(nthreads, std::max<int64_t>(1, n / 8));
  if (nt <= 1) {
    fn((int64_t)0, n);
    return;
  }
  hvec<std::thread> pool;
  std::exception_ptr err;
  std::mutex m;
  for (int t = 0; t < nt; ++t)
    pool.emplace_back([&, t] {
      try {
        fn(n * t / nt, n * (t + 1) / nt);
      } catch (...) {
        std::lock_guard<std::mutex> g(m);
        if (!err) err = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}

struct XBlock {  // one x block's tables (block-local location indices)
  hvec<int32_t> locs, sup_u, sup_n;  // locations; per-entry local index; entries per row
  hvec<double> sup_c;
};
struct YBlock {  // one y block's records, in descending first-slot order
  hvec<YRec> recs;
  hvec<int32_t> loc;
  uint32_t zero = 0;
  bool second = false, equal = true;
};
}  // namespace

namespace {
// Location slots of one x block, chosen so that the gather's shared-memory
// reads are free of bank conflicts.  The gather thread of row ii reads
// H[j][u_k(ii)] for its k-th support; a 16-byte LDS is served in four phases
// of eight consecutive lanes (rows), each conflict-free iff its eight slots
// lie in distinct 16-byte bank groups (slot mod 8).  First-appearance slots
// put the supports of neighbouring rows at slot ~1.5 ii, two per bank group.
// Here locations are greedily coloured with residues mod 8 such that no two
// different locations at the same support position k of rows in the same
// phase share a residue (capacity kUCap/8 locations per residue), and the
// slot of a location is its residue + 8 x its rank within the residue.
// The slot is also the pair-loop thread that owns the location, so nothing
// else changes.  Falls back to first-appearance slots if the colouring fails.
void bank_balance(XBlock& XB) {
  const int nl = (int)XB.locs.size();
  if (nl == 0 || nl > kUCap) return;
  const int nrows = (int)XB.sup_n.size();
  hvec<int32_t> start(nrows + 1, 0);
  for (int r = 0; r < nrows; ++r) start[r + 1] = start[r] + XB.sup_n[r];
  // conflict graph: bitsets over locations (<= 128) per location
  std::vector<std::array<uint64_t, 2>> adj(nl, {0ull, 0ull});
  auto link = [&](int a, int b) {
    if (a == b) return;
    adj[a][b >> 6] |= 1ull << (b & 63);
    adj[b][a >> 6] |= 1ull << (a & 63);
  };
  for (int p0 = 0; p0 < nrows; p0 += 8)
    for (int k = 0; k < 8; ++k)
      for (int r1 = p0; r1 < std::min(nrows, p0 + 8); ++r1)
        for (int r2 = r1 + 1; r2 < std::min(nrows, p0 + 8); ++r2)
          if (k < XB.sup_n[r1] && k < XB.sup_n[r2]) link(XB.sup_u[start[r1] + k], XB.sup_u[start[r2] + k]);
  hvec<int8_t> color(nl, -1);
  int load[8] = {0};
  const int cap = kUCap / 8;
  // most constrained first (degree), ties by first appearance
  hvec<int32_t> order(nl);
  std::iota(order.begin(), order.end(), 0);
  auto deg = [&](int a) { return __builtin_popcountll(adj[a][0]) + __builtin_popcountll(adj[a][1]); };
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return deg(a) > deg(b); });
  for (int a : order) {
    int clash[8] = {0};  // coloured neighbours per residue
    for (int w = 0; w < 2; ++w)
      for (uint64_t m = adj[a][w]; m; m &= m - 1) {
        const int b = w * 64 + __builtin_ctzll(m);
        if (color[b] >= 0) ++clash[color[b]];
      }
    int best = -1;  // fewest clashes (a clash costs one extra wavefront), then lightest residue
    for (int c = 0; c < 8; ++c)
      if (load[c] < cap && (best < 0 || clash[c] < clash[best] || (clash[c] == clash[best] && load[c] < load[best])))
        best = c;
    if (best < 0) return;  // keep first-appearance slots
    color[a] = (int8_t)best;
    ++load[best];
  }
  hvec<int32_t> slot(nl), rank(8, 0);
  for (int a = 0; a < nl; ++a) slot[a] = color[a] + 8 * rank[color[a]]++;
  hvec<int32_t> locs(kUCap, -1);
  for (int a = 0; a < nl; ++a) locs[slot[a]] = XB.locs[a];
  for (int32_t& u : XB.sup_u) u = slot[u];
  // slots are sparse now: unused ones hold no location (the pair loop's
  // padding threads), so the block's location list keeps kUCap-granular holes
  int top = 0;
  for (int i = 0; i < kUCap; ++i)
    if (locs[i] >= 0) top = i + 1;
  XB.locs.assign(locs.begin(), locs.begin() + top);
}
}  // namespace

void build_x_tables(const Locations& X, const BlockLayout& B, TileTables& T, hvec<int32_t>& xl_id) {
  const int64_t nrows = X.nfree;
  const int64_t nIb = (int64_t)B.xb.size() - 1;
  // ---- x blocks (boundaries from the layout), built in parallel
  hvec<XBlock> xb(nIb);
  parallel_for(nIb, [&](int64_t b0, int64_t b1) {
    hvec<int64_t> owner(X.size(), -1);
    hvec<int32_t> local(X.size(), 0);
    for (int64_t blk = b0; blk < b1; ++blk) {
      XBlock& XB = xb[blk];
      for (int64_t p = B.xb[blk]; p < B.xb[blk + 1]; ++p) {
        for (int64_t s = X.dstart[p]; s < X.dstart[p + 1]; ++s) {
          const int32_t u = X.dloc[s];
          if (owner[u] != blk) {
            owner[u] = blk;
            local[u] = (int32_t)XB.locs.size();
            XB.locs.push_back(u);
          }
          XB.sup_u.push_back(local[u]);
          XB.sup_c.push_back(X.dcoef[s]);
        }
        XB.sup_n.push_back((int32_t)(X.dstart[p + 1] - X.dstart[p]));
      }
      bank_balance(XB);
    }
  });
  xl_id.clear();  // global x location id of every block entry (parallel to xl_x)
  {
    size_t nl = 0, ns = 0;
    for (const XBlock& XB : xb) {
      nl += XB.locs.size();
      ns += XB.sup_u.size();
    }
    xl_id.reserve(nl);
    T.xl_x.reserve(nl);
    T.xl_y.reserve(nl);
    T.xl_z.reserve(nl);
    T.xsup_u.reserve(ns);
    T.xsup_c.reserve(ns);
  }
  T.xb_dof_start.push_back(0);
  T.xb_loc_start.push_back(0);
  T.xsup_start.assign(nrows + 1, 0);
  {
    int64_t p = 0;
    for (int64_t blk = 0; blk < nIb; ++blk) {
      const XBlock& XB = xb[blk];
      for (int32_t n : XB.sup_n) {
        T.xsup_start[p + 1] = T.xsup_start[p] + n;
        ++p;
      }
      T.xsup_u.insert(T.xsup_u.end(), XB.sup_u.begin(), XB.sup_u.end());
      T.xsup_c.insert(T.xsup_c.end(), XB.sup_c.begin(), XB.sup_c.end());
      for (int32_t u : XB.locs) {
        // bank_balance holes: an unused slot is a far point (finite pair
        // values in a column no row reads), like the kernel's idle lanes
        T.xl_x.push_back(u >= 0 ? X.x[u] : 1e100);
        T.xl_y.push_back(u >= 0 ? X.y[u] : 0.0);
        T.xl_z.push_back(u >= 0 ? X.z[u] : 0.0);
        xl_id.push_back(u);
      }
      T.xb_dof_start.push_back((int32_t)p);
      T.xb_loc_start.push_back((int32_t)T.xl_x.size());
    }
  }
}

hvec<char> device_records(const hvec<YRec>& recs, bool unit) {
  hvec<char> out;
  if (!unit) {
    out.resize(recs.size() * sizeof(YRec));
    if (!recs.empty()) std::memcpy(out.data(), recs.data(), out.size());
    return out;
  }
  out.resize(recs.size() * sizeof(YRecU));
  YRecU* u = reinterpret_cast<YRecU*>(out.data());
  for (size_t i = 0; i < recs.size(); ++i) u[i] = {recs[i].x, recs[i].y, recs[i].z, recs[i].off0, recs[i].off1};
  return out;
}

void build_y_tables(const Locations& Y, const BlockLayout& B, TileTables& T, hvec<int64_t>& yb_start,
                    hvec<int32_t>& yb_list) {
  const int64_t nJb = (int64_t)B.yb.size() - 1;
  // ---- y blocks (boundaries from the layout): records = incident locations,
  // each carrying <= 2 (slot, coef) pairs: a run slot (accumulated in a
  // register run, flushed to its H row with a plain store when the run ends)
  // and a read-modify-write slot.  Run order: breadth-first over the block's
  // slot graph (slots joined by two-slot records) from a slot that has a
  // single-slot record; every two-slot record runs on its later slot, so each
  // row's run flush precedes all read-modify-writes of that row, and every
  // slot reached from such a root has a run of its own.  Rows without a run
  // (a component with no single-slot record) are zero-filled (bitmask).
  // unit_y: every dof's contributions share one coefficient -> unit records,
  // the factor goes to yscale (applied per entry in the gather).
  bool unit = Y.nfree > 0;
  T.yscale.assign(Y.nfree, 0.0);
  for (int64_t q = 0; q < Y.nfree && unit; ++q)
    for (int64_t s = Y.dstart[q]; s < Y.dstart[q + 1]; ++s) {
      if (s == Y.dstart[q]) {
        T.yscale[q] = Y.dcoef[s];
      } else if (std::memcmp(&Y.dcoef[s], &T.yscale[q], sizeof(double)) != 0) {
        unit = false;
        break;
      }
    }
  if (!unit) T.yscale.clear();
  T.unit_y = unit;
  hvec<YBlock> yb(nJb);
  parallel_for(nJb, [&](int64_t b0, int64_t b1) {
    hvec<int64_t> ystamp(Y.size(), -1);
    hvec<std::pair<int32_t, double>> sl;  // slots of one location inside the block
    hvec<YRec> recs;
    hvec<int32_t> rec_loc, order;
    int32_t pos[kJCap], queue[kJCap];
    uint32_t adj[kJCap];
    for (int64_t b = b0; b < b1; ++b) {
      const int64_t q0 = B.yb[b], q1 = B.yb[b + 1];
      const int nJ = (int)(q1 - q0);
      recs.clear();
      rec_loc.clear();
      uint32_t single = 0;  // slots with a single-slot record
      for (int j = 0; j < nJ; ++j) adj[j] = 0;
      for (int64_t q = q0; q < q1; ++q)
        for (int64_t s = Y.dstart[q]; s < Y.dstart[q + 1]; ++s) {
          const int32_t v = Y.dloc[s];
          if (ystamp[v] == b) continue;
          ystamp[v] = b;
          sl.clear();
          for (int64_t c = Y.cstart[v]; c < Y.cstart[v + 1]; ++c) {
            const int32_t pq = Y.iperm[Y.cdof[c]];
            if (pq >= q0 && pq < q1) sl.push_back({(int32_t)(pq - q0), unit ? 1.0 : Y.ccoef[c]});
          }
          std::stable_sort(sl.begin(), sl.end(), [](const auto& a, const auto& c) { return a.first < c.first; });
          for (size_t a = 0; a < sl.size(); a += 2) {
            YRec r;
            r.x = Y.x[v];
            r.y = Y.y[v];
            r.z = Y.z[v];
            r.off0 = sl[a].first;  // slot indices for now, byte offsets below
            r.c0 = sl[a].second;
            if (a + 1 < sl.size()) {
              r.off1 = sl[a + 1].first;
              r.c1 = sl[a + 1].second;
              adj[r.off0] |= 1u << r.off1;
              adj[r.off1] |= 1u << r.off0;
            } else {
              r.off1 = -1;
              r.c1 = 0.0;
              single |= 1u << r.off0;
            }
            recs.push_back(r);
            rec_loc.push_back(v);
          }
        }
      // breadth-first slot positions, roots with single-slot records first
      for (int j = 0; j < nJ; ++j) pos[j] = -1;
      int npos = 0;
      for (int pass = 0; pass < 2; ++pass)
        for (int root = 0; root < nJ; ++root) {
          if (pos[root] >= 0 || (pass == 0 && !((single >> root) & 1u))) continue;
          int head = npos;
          pos[root] = npos;
          queue[npos++] = root;
          while (head < npos) {
            const int u = queue[head++];
            for (uint32_t m = adj[u]; m; m &= m - 1) {
              const int w = __builtin_ctz(m);
              if (pos[w] < 0) {
                pos[w] = npos;
                queue[npos++] = w;
              }
            }
          }
        }
      for (YRec& r : recs)
        if (r.off1 >= 0 && pos[r.off1] > pos[r.off0]) {
          std::swap(r.off0, r.off1);
          std::swap(r.c0, r.c1);
        }
      order.resize(recs.size());
      std::iota(order.begin(), order.end(), 0);
      std::stable_sort(order.begin(), order.end(),
                       [&](int32_t a, int32_t c) { return pos[recs[a].off0] < pos[recs[c].off0]; });
      YBlock& YB = yb[b];
      YB.recs.resize(recs.size());
      YB.loc.resize(recs.size());
      uint32_t has_run = 0;
      for (size_t i = 0; i < order.size(); ++i) {
        YRec r = recs[order[i]];
        has_run |= 1u << r.off0;
        r.off0 *= kHS * 16;
        if (r.off1 >= 0) r.off1 *= kHS * 16;
        YB.recs[i] = r;
        YB.loc[i] = rec_loc[order[i]];
        YB.second |= r.off1 >= 0;
        if (r.off1 >= 0 && std::memcmp(&r.c0, &r.c1, sizeof(double)) != 0) YB.equal = false;
      }
      const uint32_t all = nJ >= 32 ? 0xffffffffu : ((1u << nJ) - 1u);
      YB.zero = all & ~has_run;
    }
  });
  // y location -> y blocks holding it (CSR; a location is listed once per block)
  yb_start.assign(Y.size() + 1, 0);
  yb_list.clear();
  hvec<int32_t> last(Y.size(), -1);
  for (int64_t b = 0; b < nJb; ++b)
    for (int32_t v : yb[b].loc)
      if (last[v] != (int32_t)b) {
        last[v] = (int32_t)b;
        yb_start[v + 1]++;
      }
  for (int64_t v = 0; v < Y.size(); ++v) yb_start[v + 1] += yb_start[v];
  yb_list.resize(yb_start[Y.size()]);
  {
    hvec<int64_t> fill(yb_start.begin(), yb_start.end() - 1);
    std::fill(last.begin(), last.end(), -1);
    for (int64_t b = 0; b < nJb; ++b)
      for (int32_t v : yb[b].loc)
        if (last[v] != (int32_t)b) {
          last[v] = (int32_t)b;
          yb_list[fill[v]++] = (int32_t)b;
        }
  }
  size_t nrec_total = 0;
  for (const YBlock& YB : yb) nrec_total += YB.recs.size();
  T.yrec.reserve(nrec_total);
  T.yb_zero.reserve(nJb);
  T.yb_dof_start.reserve(nJb + 1);
  T.yb_rec_start.reserve(nJb + 1);
  T.yb_dof_start.push_back(0);
  T.yb_rec_start.push_back(0);
  for (int64_t b = 0; b < nJb; ++b) {
    const YBlock& YB = yb[b];
    T.has_second_slot |= YB.second;
    if (YB.second && !YB.equal) T.equal_coefs = false;
    T.yb_zero.push_back(YB.zero);
    T.yrec.insert(T.yrec.end(), YB.recs.begin(), YB.recs.end());
    T.yb_dof_start.push_back((int32_t)B.yb[b + 1]);
    T.yb_rec_start.push_back((int32_t)T.yrec.size());
  }
}

void build_tile_list(const TileTables& TX, TileTables& T, bool symmetric, const Coincidence& C,
                     const hvec<int32_t>& xl_id, const hvec<int64_t>& yb_start,
                     const hvec<int32_t>& yb_list, bool list_unmasked) {
  const int64_t nIb = (int64_t)TX.xb_dof_start.size() - 1, nJb = (int64_t)T.yb_dof_start.size() - 1;
  T.tile_i.clear();
  T.tile_j.clear();
  T.mtile_i.clear();
  T.mtile_j.clear();
  T.pairs_evaluated = 0;
  T.n_unmasked = 0;
  // ---- which tiles can hold a coincident (masked) pair?  With only exact
  // coincidences (find_coincidences), a tile needs the mask iff one of its x
  // locations coincides with one of its y records' locations.
  const bool unsafe = C.unsafe;
  hvec<hvec<int32_t>> masked_j(nIb);
  if (!unsafe)
    parallel_for(nIb, [&](int64_t b0, int64_t b1) {
      for (int64_t bi = b0; bi < b1; ++bi) {
        for (int32_t e = TX.xb_loc_start[bi]; e < TX.xb_loc_start[bi + 1]; ++e) {
          if (xl_id[e] < 0) continue;  // a bank_balance hole
          const int32_t v = C.y_of_x[xl_id[e]];
          if (v >= 0)
            masked_j[bi].insert(masked_j[bi].end(), yb_list.begin() + yb_start[v], yb_list.begin() + yb_start[v + 1]);
        }
        std::sort(masked_j[bi].begin(), masked_j[bi].end());
        masked_j[bi].erase(std::unique(masked_j[bi].begin(), masked_j[bi].end()), masked_j[bi].end());
      }
    });
  // ---- tiles (symmetric: skip tiles strictly below the diagonal)
  for (int64_t bi = 0; bi < nIb; ++bi) {
    int64_t first = 0;
    if (symmetric)
      first = std::upper_bound(T.yb_dof_start.begin() + 1, T.yb_dof_start.end(), TX.xb_dof_start[bi]) -
              (T.yb_dof_start.begin() + 1);
    if (list_unmasked || unsafe) {
      for (int64_t bj = first; bj < nJb; ++bj) {
        const bool m = unsafe || std::binary_search(masked_j[bi].begin(), masked_j[bi].end(), (int32_t)bj);
        if (m) {
          T.mtile_i.push_back((int32_t)bi);
          T.mtile_j.push_back((int32_t)bj);
        } else {
          ++T.n_unmasked;
          if (list_unmasked) {
            T.tile_i.push_back((int32_t)bi);
            T.tile_j.push_back((int32_t)bj);
          }
        }
      }
    } else {  // count the unmasked tiles, list only the masked ones (sorted, unique)
      const auto lo = std::lower_bound(masked_j[bi].begin(), masked_j[bi].end(), (int32_t)first);
      for (auto it = lo; it != masked_j[bi].end(); ++it) {
        T.mtile_i.push_back((int32_t)bi);
        T.mtile_j.push_back(*it);
      }
      T.n_unmasked += (nJb - first) - (int64_t)(masked_j[bi].end() - lo);
    }
    T.pairs_evaluated += (int64_t)(TX.xb_loc_start[bi + 1] - TX.xb_loc_start[bi]) *
                         (T.yb_rec_start[nJb] - T.yb_rec_start[first]);
  }
}

TileTables build_tiles(const Locations& X, const Locations& Y, bool symmetric, const Coincidence& C,
                       const BlockLayout& B) {
  TileTables T;
  hvec<int32_t> xl_id;
  hvec<int64_t> yb_start;
  hvec<int32_t> yb_list;
  const bool timing = std::getenv("GK_TIMING") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[gk_plan]     %-18s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  // the x and y tables are independent (disjoint members of T): built concurrently
  auto ytab = std::async(std::launch::async, [&] { build_y_tables(Y, B, T, yb_start, yb_list); });
  build_x_tables(X, B, T, xl_id);
  ytab.get();
  lap("x + y tables");
  T.x_halo = X.size() ? (double)T.xl_x.size() / (double)X.size() : 0.0;
  T.y_halo = Y.size() ? (double)T.yrec.size() / (double)Y.size() : 0.0;
  // the plan path builds its descriptors on the device from the block tables
  // (launch_make_tiles): only the masked tiles are listed
  build_tile_list(T, T, symmetric, C, xl_id, yb_start, yb_list, false);
  lap("tile list");
  return T;
}

Coincidence find_coincidences(const Locations& X, const Locations& Y, bool same, double eps) {
  // Sweep over x-coordinate-sorted points of both sides with a window of
  // 8 eps: every pair closer than that must be an exact coincidence, or the
  // plan keeps the distance mask everywhere.
  Coincidence C;
  C.y_of_x.assign(X.size(), -1);
  if (!(eps > 0.0)) {
    C.unsafe = true;
    return C;
  }
  const double win = 8.0 * eps, win2 = win * win;
  struct P {
    double x;
    int32_t id;
    int8_t side;
  };
  hvec<P> pts;
  pts.reserve(X.size() + (same ? 0 : Y.size()));
  for (int64_t u = 0; u < X.size(); ++u) pts.push_back({X.x[u], (int32_t)u, 0});
  if (!same)
    for (int64_t v = 0; v < Y.size(); ++v) pts.push_back({Y.x[v], (int32_t)v, 1});
  // sorted by x: chunks sorted on the planner's threads, then merged pairwise
  // (the order among equal keys is immaterial: every pair inside the window
  // is examined whatever it is)
  auto before = [](const P& a, const P& b) { return a.x < b.x || (a.x == b.x && a.side < b.side); };
  {
    const size_t n = pts.size();
    const int nt = t_serial ? 1 : (int)std::min<size_t>((size_t)host_threads(), n / 8192);
    if (nt <= 1) {
      std::sort(pts.begin(), pts.end(), before);
    } else {
      auto bound = [&](int c) { return n * (size_t)std::min(c, nt) / (size_t)nt; };
      auto fan = [&](int tasks, auto&& fn) {
        std::vector<std::thread> pool;
        for (int t = 1; t < tasks; ++t) pool.emplace_back([&fn, t] { fn(t); });
        fn(0);
        for (auto& th : pool) th.join();
      };
      fan(nt, [&](int c) { std::sort(pts.begin() + bound(c), pts.begin() + bound(c + 1), before); });
      hvec<P> tmp(n);
      for (int w = 1; w < nt; w *= 2) {
        const int pairs = (nt + 2 * w - 1) / (2 * w);
        fan(pairs, [&](int q) {
          const size_t a = bound(2 * w * q), m = bound(2 * w * q + w), e = bound(2 * w * q + 2 * w);
          std::merge(pts.begin() + a, pts.begin() + m, pts.begin() + m, pts.begin() + e, tmp.begin() + a, before);
        });
        pts.swap(tmp);
      }
    }
  }
  auto coord = [&](const P& p, double& x, double& y, double& z) {
    const Locations& L = p.side ? Y : X;
    x = L.x[p.id];
    y = L.y[p.id];
    z = L.z[p.id];
  };
  for (size_t i = 0; i < pts.size() && !C.unsafe; ++i)
    for (size_t j = i + 1; j < pts.size() && pts[j].x - pts[i].x <= win; ++j) {
      double ax, ay, az, bx, by, bz;
      coord(pts[i], ax, ay, az);
      coord(pts[j], bx, by, bz);
      const double dx = ax - bx, dy = ay - by, dz = az - bz;
      if (dx * dx + dy * dy + dz * dz > win2) continue;
      // within 8 eps: allowed only as an exact x/y coincidence
      const bool exact = bits(ax) == bits(bx) && bits(ay) == bits(by) && bits(az) == bits(bz);
      if (same || pts[i].side == pts[j].side || !exact) {
        C.unsafe = true;  // distinct locations of one side within 8 eps, or a near miss
        break;
      }
      const P& px = pts[i].side == 0 ? pts[i] : pts[j];
      const P& py = pts[i].side == 0 ? pts[j] : pts[i];
      C.y_of_x[px.id] = py.id;
    }
  if (same && !C.unsafe)
    for (int64_t u = 0; u < X.size(); ++u) C.y_of_x[u] = (int32_t)u;
  return C;
}

void planner_serial(bool on) { t_serial = on; }

OrderChoice choose_order(Locations& X, Locations* Y, bool symmetric, double eps, double accept_natural) {
  const char* force = std::getenv("GK_ORDER");
  const std::string f = force ? force : "";
  const bool timing = std::getenv("GK_TIMING") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[gk_plan]   %-20s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  // The coincidence sweep and the candidate orders are independent (the
  // sweep reads coordinates only; the candidates work on copies), so they run
  // concurrently; build_locations left X and Y in natural order.
  auto sweep = std::async(std::launch::async, [&] {
    const auto s0 = std::chrono::steady_clock::now();
    Coincidence C = find_coincidences(X, Y ? *Y : X, Y == nullptr, eps);
    if (timing)
      std::fprintf(stderr, "[gk_plan]     %-18s %8.2f ms (concurrent)\n", "coincidence sweep",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - s0).count());
    return C;
  });
  auto layout_of = [&](Locations& Lx, Locations* Ly) { return layout_blocks(Lx, Ly ? *Ly : Lx, symmetric); };
  OrderChoice O;
  O.natural = true;
  O.unit = 1;
  // Candidates (natural, RCB unit, x cut):
  //  - natural: the input numbering (subdivided meshes number children 4 by
  //    4), blocks cut back to 4^k subtree boundaries; rows of a tile are
  //    contiguous in A;
  //  - RCB over aligned units of 4 consecutive dofs (P0 on a subdivided mesh:
  //    the 4 children of one parent triangle), x blocks filled to 128
  //    locations: compact blocks with whole warps busy, but matrix writes in
  //    64-byte runs only;
  //  - RCB over single dofs, x blocks filled: the most compact blocks for
  //    unstructured numberings (P1 vertices), but every matrix write is a
  //    scattered 16-byte half sector (a DRAM read-modify-write).
  // Cost = location pairs issued by whole warps; both RCB candidates are
  // charged 1.25x for their writes.  Measured on the cfg-4 P0 tile structure:
  // natural 47.1 ms vs RCB units of 4 48.6-49.2 ms (17% fewer issued pairs,
  // but a 1.6x longer gather + store phase) vs RCB single dofs 5.0 vs 3.0 ms
  // on L5; on P1 (cfg 2) natural issues 1.65x the pairs and RCB wins.
  struct Cand {
    bool natural;
    int unit;
    double xcut, penalty;
  };
  std::vector<Cand> cands;
  if (f == "natural")
    cands = {{true, 1, 0.8, 1.0}};
  else if (f == "rcb")
    cands = {{false, 1, 1.0, 1.0}};
  else if (f == "rcb4")
    cands = {{false, 4, 1.0, 1.0}};
  else
    cands = {{true, 1, 0.8, 1.0}, {false, 4, 1.0, 1.25}, {false, 1, 1.0, 1.25}};
  if (accept_natural > 0.0 && cands.size() > 1) {
    // take natural order without building the others when it evaluates at
    // most accept_natural pairs per unique pair (callers whose kernel time
    // hides under a larger cost, like the PCIe-bound streamed path)
    BlockLayout B = layout_of(X, Y);
    lap("  natural layout");
    const double unique = (double)X.size() * (double)(Y ? Y->size() : X.size()) * (symmetric ? 0.5 : 1.0);
    if ((double)B.pairs <= accept_natural * unique) {
      O.C = sweep.get();
      O.B = std::move(B);
      lap("coincidences+orders (natural accepted)");
      return O;
    }
  }
  struct Result {
    Locations X, Y;
    BlockLayout B;
    double cost = 0.0;
  };
  std::vector<std::future<Result>> futs;
  for (size_t c = 1; c < cands.size(); ++c)
    futs.push_back(std::async(std::launch::async, [&, c] {
      Result R;
      R.X = X;
      if (Y) R.Y = *Y;
      set_order(R.X, cands[c].natural, cands[c].unit, cands[c].xcut);
      if (Y) set_order(R.Y, cands[c].natural, cands[c].unit, cands[c].xcut);
      R.B = layout_of(R.X, Y ? &R.Y : nullptr);
      R.cost = (double)R.B.lane_pairs * cands[c].penalty;
      return R;
    }));
  if (!cands[0].natural) {
    set_order(X, false, cands[0].unit, cands[0].xcut);
    if (Y) set_order(*Y, false, cands[0].unit, cands[0].xcut);
  }
  BlockLayout B = layout_of(X, Y);
  double best = (double)B.lane_pairs * cands[0].penalty;
  O.natural = cands[0].natural;
  O.unit = cands[0].unit;
  for (size_t c = 1; c < cands.size(); ++c) {
    Result R = futs[c - 1].get();
    if (R.cost < best) {
      best = R.cost;
      X = std::move(R.X);
      if (Y) *Y = std::move(R.Y);
      B = std::move(R.B);
      O.natural = cands[c].natural;
      O.unit = cands[c].unit;
    }
  }
  O.C = sweep.get();
  O.B = std::move(B);
  lap(O.natural ? "coincidences+orders (natural)" : (O.unit > 1 ? "coincidences+orders (rcb units)"
                                                                 : "coincidences+orders (rcb)"));
  return O;
}

TileTables choose_order_and_tile(Locations& X, Locations* Y, bool symmetric, double eps) {
  // symmetric plans take natural order without building the RCB candidates
  // when it evaluates at most 1.6 pairs per unique pair (P0 on subdivided
  // meshes: cfg 4 1.45, cfg 3 1.00 — measured faster than RCB there, and the
  // two RCB candidates cost ~20 ms of every plan); P1 vertex numberings
  // (cfg 2: natural ~2.9) and row-slab plans still compare all three
  const OrderChoice O = choose_order(X, Y, symmetric, eps, symmetric ? 1.6 : 0.0);
  const auto t0 = std::chrono::steady_clock::now();
  TileTables T = build_tiles(X, Y ? *Y : X, symmetric, O.C, O.B);
  if (std::getenv("GK_TIMING"))
    std::fprintf(stderr, "[gk_plan]   %-20s %8.2f ms\n", "tiles",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  return T;
}

Locations restrict_cols(const Locations& Y, int64_t c0, int64_t c1, hvec<int32_t>& slab_of_full) {
  // the trial locations supporting dofs [c0, c1), in increasing location id,
  // with only those dofs' contributions (renumbered from 0)
  Locations S;
  S.nfree = c1 - c0;
  slab_of_full.assign(Y.size(), -1);
  hvec<int32_t> locs;
  for (int64_t d = c0; d < c1; ++d) {
    const int64_t q = Y.iperm[d];
    for (int64_t s = Y.dstart[q]; s < Y.dstart[q + 1]; ++s) {
      const int32_t v = Y.dloc[s];
      if (slab_of_full[v] < 0) {
        slab_of_full[v] = 0;
        locs.push_back(v);
      }
    }
  }
  std::sort(locs.begin(), locs.end());
  const size_t n = locs.size();
  S.x.resize(n);
  S.y.resize(n);
  S.z.resize(n);
  S.cstart.assign(n + 1, 0);
  for (size_t i = 0; i < n; ++i) {
    const int32_t v = locs[i];
    slab_of_full[v] = (int32_t)i;
    S.x[i] = Y.x[v];
    S.y[i] = Y.y[v];
    S.z[i] = Y.z[v];
    for (int64_t c = Y.cstart[v]; c < Y.cstart[v + 1]; ++c) {
      const int64_t d = Y.cdof[c];
      if (d >= c0 && d < c1) {
        S.cdof.push_back((int32_t)(d - c0));
        S.ccoef.push_back(Y.ccoef[c]);
      }
    }
    S.cstart[i + 1] = (int64_t)S.cdof.size();
  }
  return S;
}

}  // namespace gk
