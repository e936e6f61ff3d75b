// hull.cpp -- the host hull stage that runs on the filter's survivors.
//
// The north star keeps this stage on the host with the reference's own
// semantics (reference hull.cpp:18-150, 205-232): per-quadrant sweep sort +
// strict-left-turn chain, then cycle clean-up (de-duplication, collinear
// collapse, strict_cycle peeling, rotation to the east-most vertex).
// Outputs are coordinate-identical to the reference for every input; the
// implementation differs where that cannot change the result:
//  * large survivor sets arrive already sorted from the device
//    (hullsort.cu); smaller ones use the libstdc++ (parallel) sort -- equal
//    points are indistinguishable, so any order of ties yields the same
//    chain;
//  * the four quadrant chains run concurrently (each chain is the
//    reference's sequential stack loop: its decisions are the reference's
//    predicate sequence, which a parallel hull would not reproduce on
//    near-degenerate inputs);
//  * the clean-up's linear passes (de-duplication, collinearity test,
//    compaction, rotation) run in parallel, and the peel replays the
//    reference's LIFO worklist exactly while skipping the vertices whose
//    test cannot change (see peel).
#include <omp.h>
#include <pthread.h>
#include <sys/mman.h>
#include <unistd.h>

#include <parallel/algorithm>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <exception>
#include <functional>
#include <memory>
#include <condition_variable>
#include <mutex>
#include <new>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "internal.hpp"

namespace ohx {

namespace {
struct BigCache {
  std::mutex mu;
  struct Block {
    void* p;
    std::size_t bytes;
  };
  std::vector<Block> blocks;  // freed blocks kept mapped (pages faulted)
  std::size_t held = 0;
  static constexpr std::size_t kMaxHeld = std::size_t(8) << 30;
  static constexpr std::size_t kMaxBlocks = 8;
};
BigCache& big_cache() {
  static BigCache* c = new BigCache;  // never destroyed: freeing at exit is moot
  return *c;
}
std::size_t round_2m(std::size_t b) { return (b + (std::size_t(2) << 20) - 1) & ~((std::size_t(2) << 20) - 1); }
}  // namespace

void* big_alloc(std::size_t bytes) {
  bytes = round_2m(bytes);
  BigCache& c = big_cache();
  {
    std::lock_guard<std::mutex> g(c.mu);
    std::size_t best = c.blocks.size();
    for (std::size_t i = 0; i < c.blocks.size(); ++i)  // smallest block that fits (<= 2x)
      if (c.blocks[i].bytes >= bytes && c.blocks[i].bytes <= 2 * bytes &&
          (best == c.blocks.size() || c.blocks[i].bytes < c.blocks[best].bytes))
        best = i;
    if (best != c.blocks.size()) {
      void* p = c.blocks[best].p;
      c.held -= c.blocks[best].bytes;
      c.blocks.erase(c.blocks.begin() + static_cast<std::ptrdiff_t>(best));
      return p;
    }
  }
  void* p = nullptr;
  if (posix_memalign(&p, std::size_t(2) << 20, bytes) != 0) throw std::bad_alloc();
  madvise(p, bytes, MADV_HUGEPAGE);
  return p;
}

void big_cache_trim() noexcept {
  BigCache& c = big_cache();
  std::lock_guard<std::mutex> g(c.mu);
  for (const auto& b : c.blocks) std::free(b.p);
  c.blocks.clear();
  c.held = 0;
}

void big_free(void* p, std::size_t bytes) noexcept {
  bytes = round_2m(bytes);
  BigCache& c = big_cache();
  std::lock_guard<std::mutex> g(c.mu);
  // a recycled block may be larger than the size its last owner knew: the
  // recorded size is then a lower bound, which is all big_alloc relies on
  if (c.held + bytes <= BigCache::kMaxHeld && c.blocks.size() < BigCache::kMaxBlocks) {
    c.blocks.push_back({p, bytes});
    c.held += bytes;
    return;
  }
  std::free(p);
}

namespace {
bool g_forked = false;
void on_fork_child() {
  g_forked = true;
  omp_set_num_threads(1);
}
[[maybe_unused]] const int g_atfork = pthread_atfork(nullptr, nullptr, on_fork_child);
}  // namespace

int team(int want) { return g_forked || want < 1 ? 1 : want; }

int orient(const P2& a, const P2& b, const P2& c) {
  // reference geometry.hpp:27-32
  const double det = (b.x - a.x) * (c.y - a.y) - (b.y - a.y) * (c.x - a.x);
  return det > 0.0 ? 1 : (det < 0.0 ? -1 : 0);
}

namespace {

// OHX_TRACE=1: wall time of the hull phases on stderr
bool trace_on() {
  static const bool on = [] {
    const char* e = std::getenv("OHX_TRACE");
    return e && *e && std::string(e) != "0";
  }();
  return on;
}
double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

bool same(const P2& a, const P2& b) { return a.x == b.x && a.y == b.y; }

// CCW sweep keys of the four quadrant arcs (reference hull.cpp:18-30),
// one comparator type per quadrant so the sort inlines a branch-light key
template <int Q>
struct SweepLess {
  bool operator()(const P2& a, const P2& b) const {
    if constexpr (Q == 1) return a.x != b.x ? a.x > b.x : a.y < b.y;
    else if constexpr (Q == 2) return a.y != b.y ? a.y > b.y : a.x > b.x;
    else if constexpr (Q == 3) return a.x != b.x ? a.x < b.x : a.y > b.y;
    else return a.y != b.y ? a.y < b.y : a.x < b.x;
  }
};

bool lex(const P2& a, const P2& b) { return a.x != b.x ? a.x < b.x : a.y < b.y; }

// the reference's preferred first vertex: max x, ties to the smaller y
bool starts_before(const P2& a, const P2& b) { return a.x != b.x ? a.x > b.x : a.y < b.y; }

template <class V, class Cmp>
void big_sort(V& v, Cmp cmp) {
  if (v.size() >= (1u << 17)) __gnu_parallel::sort(v.begin(), v.end(), cmp);
  else std::sort(v.begin(), v.end(), cmp);
}

constexpr std::size_t kParMin = 1u << 16;  // below: serial loops

// Order-preserving u64 of a coordinate (-0.0 folded onto +0.0: the
// reference's comparator sees them equal); hullsort.cu uses the same map.
inline std::uint64_t asc_key(double v) {
  if (v == 0.0) v = 0.0;
  std::uint64_t u;
  std::memcpy(&u, &v, 8);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// Sweep sort of a mid-sized arc: LSD radix sort (8-bit digits, one
// histogram pass for all four, digits all keys share skipped) of a 32-bit
// key -- the primary key relative to the arc's smallest, shifted so that
// the arc's key range fills 32 bits (survivors cluster: a fixed top-32-bit
// slice of the key left long runs of equal keys) -- then runs of equal
// 32-bit keys sorted by the comparator (rare).  A few linear passes over
// per-thread scratch instead of ~n log n mispredicted comparisons (~50 ns
// per point on the box's host for random arcs).  Equal points may come
// out in any order, as with std::sort.
template <int Q>
void radix_sweep_sort(std::vector<P2>& pts) {
  struct E {
    std::uint32_t k, i;
  };
  const std::size_t n = pts.size();
  thread_local std::vector<E> a, b;
  thread_local std::vector<std::uint64_t> k64;
  thread_local std::vector<P2> out;
  if (a.size() < n) {
    a.resize(n);
    b.resize(n);
    k64.resize(n);
    out.resize(n);
  }
  std::uint64_t lo = ~0ull, hi = 0;
  for (std::size_t i = 0; i < n; ++i) {
    const P2& p = pts[i];
    const std::uint64_t k = Q == 1 ? ~asc_key(p.x) : Q == 2 ? ~asc_key(p.y)
                          : Q == 3 ? asc_key(p.x) : asc_key(p.y);
    k64[i] = k;
    lo = std::min(lo, k);
    hi = std::max(hi, k);
  }
  const std::uint64_t span = hi - lo;
  const int shift = span >> 32 ? 64 - __builtin_clzll(span) - 32 : 0;
  constexpr int kDigits = 4;
  std::uint32_t cnt[kDigits][257] = {};
  for (std::size_t i = 0; i < n; ++i) {
    const auto k = static_cast<std::uint32_t>((k64[i] - lo) >> shift);
    a[i] = {k, static_cast<std::uint32_t>(i)};
    for (int d = 0; d < kDigits; ++d) ++cnt[d][((k >> (8 * d)) & 255u) + 1];
  }
  E* src = a.data();
  E* dst = b.data();
  for (int d = 0; d < kDigits; ++d) {
    std::uint32_t* c = cnt[d];
    if (c[((src[0].k >> (8 * d)) & 255u) + 1] == n) continue;  // every key has this digit
    for (int v = 0; v < 256; ++v) c[v + 1] += c[v];
    for (std::size_t i = 0; i < n; ++i) dst[c[(src[i].k >> (8 * d)) & 255u]++] = src[i];
    std::swap(src, dst);
  }
  for (std::size_t i = 0; i < n; ++i) out[i] = pts[src[i].i];
  for (std::size_t r = 0; r < n;) {  // equal 32-bit keys: the comparator's order
    std::size_t e = r + 1;
    while (e < n && src[e].k == src[r].k) ++e;
    if (e - r > 1) std::sort(out.begin() + r, out.begin() + e, SweepLess<Q>{});
    r = e;
  }
  std::copy(out.begin(), out.begin() + n, pts.begin());
}

template <int Q>
void sweep_sort(std::vector<P2>& pts) {
  if (pts.size() >= 512 && pts.size() < (1u << 17)) radix_sweep_sort<Q>(pts);
  else big_sort(pts, SweepLess<Q>{});
}

// Parallel stream compaction: the elements i of `in` with keep(i), in order.
template <class Keep>
PVec compact(const P2* in, std::size_t n, Keep keep) {
  PVec out;
  if (n < kParMin) {
    out.reserve(n);
    for (std::size_t i = 0; i < n; ++i)
      if (keep(i)) out.push_back(in[i]);
    return out;
  }
  const int T = omp_get_max_threads();
  std::vector<std::size_t> cnt(T + 1, 0);
#pragma omp parallel num_threads(T)
  {
    const int t = omp_get_thread_num(), nt = omp_get_num_threads();
    const std::size_t b = n * t / nt, e = n * (t + 1) / nt;
    std::size_t c = 0;
    for (std::size_t i = b; i < e; ++i) c += keep(i) ? 1 : 0;
    cnt[t + 1] = c;
#pragma omp barrier
#pragma omp single
    {
      for (int k = 0; k < nt; ++k) cnt[k + 1] += cnt[k];
      out.resize(cnt[nt]);
    }
    std::size_t o = cnt[t];
    for (std::size_t i = b; i < e; ++i)
      if (keep(i)) out[o++] = in[i];
  }
  return out;
}

// Peel every vertex that does not turn strictly left, re-examining the
// neighbours of each removal: the reference's LIFO worklist
// (hull.cpp:54-92) replayed exactly, so degenerate cycles reduce
// identically.  The worklist initially holds every vertex (m-1 on top);
// popping a vertex that turns strictly left and whose neighbours never
// changed is a no-op (its only effect, clearing its pending flag, is
// implicit here: "pending" = below the scan pointer or on the explicit
// stack), so the scan jumps from one vertex that needs a test -- a
// non-strict turn (all found in parallel up front) or a pending vertex
// whose neighbour was removed -- to the next.  Links of the cyclic list
// are stored only where they changed (few removals: hash maps; many:
// arrays).  Returns false when nothing is removed (`cyc` is the answer).
template <class Links>
bool peel_with(PVec& cyc, std::vector<std::size_t> todo, Links& L) {
  const std::size_t m = cyc.size();
  std::make_heap(todo.begin(), todo.end());  // pending tests, max first
  std::vector<std::size_t> stack;            // explicit pushes (above the scan)
  std::size_t ptr = m;                       // scan entries [0, ptr) still pending
  std::size_t live = m;
  bool removed = false;
  while (live > 2) {
    std::size_t i;
    if (!stack.empty()) {
      i = stack.back();
      stack.pop_back();
      L.set_on_stack(i, false);
    } else {
      if (todo.empty()) break;  // the rest of the scan is no-ops
      std::pop_heap(todo.begin(), todo.end());
      i = todo.back();
      todo.pop_back();
      L.set_queued(i, false);
      ptr = i;  // every scan entry above i was popped as a no-op
    }
    const std::size_t a = L.prv(i), c = L.nxt(i);
    if (!L.alive(i) || orient(cyc[a], cyc[i], cyc[c]) > 0) continue;
    L.kill(i);
    removed = true;
    --live;
    L.set_nxt(a, c);
    L.set_prv(c, a);
    for (std::size_t nb : {a, c}) {
      if (!L.alive(nb)) continue;
      if (nb < ptr) {  // still pending in the scan: test it when reached
        if (!L.queued(nb)) {
          L.set_queued(nb, true);
          todo.push_back(nb);
          std::push_heap(todo.begin(), todo.end());
        }
      } else if (!L.on_stack(nb)) {
        stack.push_back(nb);
        L.set_on_stack(nb, true);
      }
    }
  }
  if (removed) {
    // unlinking keeps the cyclic index order: the survivors in index order
    // (the reference walks the list from the first alive vertex)
    PVec out = compact(cyc.data(), m, [&](std::size_t k) { return L.alive(k); });
    cyc.swap(out);
  }
  return removed;
}

struct SparseLinks {
  std::size_t m;
  std::unordered_map<std::size_t, std::size_t> p, n;
  std::unordered_set<std::size_t> dead, stacked, que;
  std::size_t prv(std::size_t i) const {
    const auto it = p.find(i);
    return it != p.end() ? it->second : (i == 0 ? m - 1 : i - 1);
  }
  std::size_t nxt(std::size_t i) const {
    const auto it = n.find(i);
    return it != n.end() ? it->second : (i + 1 == m ? 0 : i + 1);
  }
  void set_prv(std::size_t i, std::size_t v) { p[i] = v; }
  void set_nxt(std::size_t i, std::size_t v) { n[i] = v; }
  bool alive(std::size_t i) const { return !dead.count(i); }
  void kill(std::size_t i) { dead.insert(i); }
  bool on_stack(std::size_t i) const { return stacked.count(i); }
  void set_on_stack(std::size_t i, bool v) { v ? (void)stacked.insert(i) : (void)stacked.erase(i); }
  bool queued(std::size_t i) const { return que.count(i); }
  void set_queued(std::size_t i, bool v) { v ? (void)que.insert(i) : (void)que.erase(i); }
};

struct DenseLinks {
  std::vector<std::size_t> p, n;
  std::vector<std::uint8_t> flags;  // 1 dead, 2 on stack, 4 queued
  explicit DenseLinks(std::size_t m) : p(m), n(m), flags(m, 0) {
#pragma omp parallel for schedule(static) if (m >= kParMin)
    for (std::int64_t i = 0; i < static_cast<std::int64_t>(m); ++i) {
      p[i] = i == 0 ? m - 1 : i - 1;
      n[i] = i + 1 == static_cast<std::int64_t>(m) ? 0 : i + 1;
    }
  }
  std::size_t prv(std::size_t i) const { return p[i]; }
  std::size_t nxt(std::size_t i) const { return n[i]; }
  void set_prv(std::size_t i, std::size_t v) { p[i] = v; }
  void set_nxt(std::size_t i, std::size_t v) { n[i] = v; }
  bool alive(std::size_t i) const { return !(flags[i] & 1); }
  void kill(std::size_t i) { flags[i] |= 1; }
  bool on_stack(std::size_t i) const { return flags[i] & 2; }
  void set_on_stack(std::size_t i, bool v) { flags[i] = v ? (flags[i] | 2) : (flags[i] & ~2); }
  bool queued(std::size_t i) const { return flags[i] & 4; }
  void set_queued(std::size_t i, bool v) { flags[i] = v ? (flags[i] | 4) : (flags[i] & ~4); }
};

// the non-strict turns of the cyclic sequence, ascending
std::vector<std::size_t> non_strict_turns(const PVec& cyc) {
  const std::size_t m = cyc.size();
  const int T = omp_get_max_threads();
  std::vector<std::vector<std::size_t>> part(m >= kParMin ? T : 1);
#pragma omp parallel num_threads(static_cast<int>(part.size())) if (m >= kParMin)
  {
    const int t = omp_get_thread_num(), nt = omp_get_num_threads();
    const std::size_t b = m * t / nt, e = m * (t + 1) / nt;
    for (std::size_t i = b; i < e; ++i) {
      const std::size_t a = i == 0 ? m - 1 : i - 1, c = i + 1 == m ? 0 : i + 1;
      if (orient(cyc[a], cyc[i], cyc[c]) <= 0) part[t].push_back(i);
    }
  }
  std::vector<std::size_t> todo;
  for (auto& v : part) todo.insert(todo.end(), v.begin(), v.end());
  return todo;
}

// returns whether anything was removed
bool peel(PVec& cyc, std::vector<std::size_t> todo) {
  const std::size_t m = cyc.size();
  if (todo.empty()) return false;
  if (todo.size() * 64 < m) {
    SparseLinks L{m, {}, {}, {}, {}, {}};
    for (std::size_t i : todo) L.que.insert(i);
    return peel_with(cyc, std::move(todo), L);
  }
  DenseLinks L(m);
  for (std::size_t i : todo) L.flags[i] |= 4;
  return peel_with(cyc, std::move(todo), L);
}

// the first vertex with max x, ties to the smaller y (reference
// hull.cpp:35-49)
std::size_t start_vertex(const PVec& d) {
  const std::size_t sz = d.size();
  std::size_t best = 0;
  if (sz < kParMin) {
    for (std::size_t i = 1; i < sz; ++i)
      if (starts_before(d[i], d[best])) best = i;
    return best;
  }
  const int T = omp_get_max_threads();
  std::vector<std::size_t> pb(T, sz);
#pragma omp parallel num_threads(T)
  {
    const int t = omp_get_thread_num(), nt = omp_get_num_threads();
    const std::size_t b = sz * t / nt, e = sz * (t + 1) / nt;
    std::size_t bi = b;
    for (std::size_t i = b + 1; i < e; ++i)
      if (starts_before(d[i], d[bi])) bi = i;
    if (b < e) pb[t] = bi;
  }
  best = pb[0];
  for (int t = 1; t < T; ++t)
    if (pb[t] < sz && starts_before(d[pb[t]], d[best])) best = pb[t];
  return best;
}

// One parallel pass over a cycle that the fast path of finalize_cycle
// needs: consecutive duplicates?  all collinear with (c0, c1)?  its
// non-strict turns, and its start vertex.
struct CycleScan {
  bool dups = false, flat = true;
  std::vector<std::size_t> bad;
  std::size_t best = 0;
};

CycleScan scan_cycle(const PVec& c) {
  CycleScan r;
  const std::size_t m = c.size();
  const int T = m >= kParMin ? omp_get_max_threads() : 1;
  std::vector<std::vector<std::size_t>> part(T);
  std::vector<std::size_t> pb(T, m);
  std::vector<unsigned char> dups(T, 0), flat(T, 1);
#pragma omp parallel num_threads(T)
  {
    const int t = omp_get_thread_num(), nt = omp_get_num_threads();
    const std::size_t b = m * t / nt, e = m * (t + 1) / nt;
    bool du = false, fl = true;
    std::size_t bi = b;
    for (std::size_t i = b; i < e; ++i) {
      const std::size_t a = i == 0 ? m - 1 : i - 1, n = i + 1 == m ? 0 : i + 1;
      if (i > 0) du = du || same(c[a], c[i]);
      if (i >= 2) fl = fl && orient(c[0], c[1], c[i]) == 0;
      if (orient(c[a], c[i], c[n]) <= 0) part[t].push_back(i);
      if (i > b && starts_before(c[i], c[bi])) bi = i;
    }
    dups[t] = du;
    flat[t] = fl;
    if (b < e) pb[t] = bi;
  }
  for (int t = 0; t < T; ++t) {
    r.dups = r.dups || dups[t];
    r.flat = r.flat && flat[t];
    r.bad.insert(r.bad.end(), part[t].begin(), part[t].end());
    if (pb[t] < m && (t == 0 || starts_before(c[pb[t]], c[r.best]))) r.best = pb[t];
  }
  return r;
}

void rotate_to(PVec& d, std::size_t best) {
  if (best == 0) return;
  const std::size_t sz = d.size();
  PVec r(sz);
  copy_points(r.data(), d.data() + best, sz - best);
  copy_points(r.data() + (sz - best), d.data(), best);
  d.swap(r);
}

}  // namespace

void copy_points(P2* dst, const P2* src, std::size_t n) {
  if (n < kParMin) {
    std::memcpy(static_cast<void*>(dst), src, n * sizeof(P2));
    return;
  }
#pragma omp parallel
  {
    const int t = omp_get_thread_num(), nt = omp_get_num_threads();
    const std::size_t b = n * t / nt, e = n * (t + 1) / nt;
    std::memcpy(static_cast<void*>(dst + b), src + b, (e - b) * sizeof(P2));
  }
}

namespace {

inline bool strict_left(const P2& a, const P2& b, const P2& p) {
  // orientation(a, b, p) > 0 with the reference's operations (geometry.hpp:27-32)
  return (b.x - a.x) * (p.y - a.y) - (b.y - a.y) * (p.x - a.x) > 0.0;
}

// OHX_CHAIN_PAR_MIN / OHX_CHAIN_CHUNKS: size from which an arc's chain runs
// in parallel, and its number of chunks (test hooks; defaults 2^22, 16).
// Smaller arcs (and arcs whose chunks rarely coincide, like a disk's) are
// cheaper with the plain loop.
std::size_t env_size(const char* name, std::size_t dflt) {
  const char* e = std::getenv(name);
  return e && *e ? static_cast<std::size_t>(std::atoll(e)) : dflt;
}
std::size_t chain_par_min() {
  static const std::size_t v = env_size("OHX_CHAIN_PAR_MIN", std::size_t(1) << 22);
  return v;
}

// Chains computed in parallel with IDENTICAL decisions.  Every chunk of an
// arc first runs the loop on its own (empty stack); then, chunk by chunk,
// the true loop resumes from the true stack G and replays the chunk's first
// points until it provably coincides with the chunk's own run: the part of
// G pushed in this chunk (C) equals the top |C| >= 2 entries of the local
// stack after the same point, and the local run never again drops below
// those entries' base + 2 (so every later test and pop touches only entries
// both runs share).  From there the chunk's local final stack above that
// base is the true result.  A chunk that does not coincide within
// kSyncWindow points is finished by the plain loop on a flattened copy of G.
constexpr std::size_t kSyncWindow = 64;

struct ChunkRun {
  std::size_t b, e, height;          // points [b, e) of the arc, local stack height
  std::uint32_t low[kSyncWindow];    // stack height after point k's pops (k < window)
  std::uint32_t low_rest;            // min of that height over the later points
};

struct ArcChain {
  const P2* pts = nullptr;
  std::size_t n = 0;
  PVec loc;                          // the chunks' local stacks, each in place
  std::vector<ChunkRun> runs;
  struct Slice {
    const P2* base;
    std::size_t from, to;
  };
  std::vector<Slice> G;              // the true stack, as slices
  std::size_t gsize = 0;
  PVec extra;                        // entries pushed by replayed points

  void local_run(std::size_t j) {  // phase A, one chunk (any thread)
    ChunkRun& r = runs[j];
    const P2* in = pts + r.b;
    P2* ch = loc.data() + r.b;
    const std::size_t len = r.e - r.b;
    std::size_t top = 0;
    std::uint32_t rest = ~0u;
    for (std::size_t k = 0; k < len; ++k) {
      const P2 p = in[k];
      while (top >= 2 && !strict_left(ch[top - 2], ch[top - 1], p)) --top;
      if (k < kSyncWindow) r.low[k] = static_cast<std::uint32_t>(top);
      else rest = std::min(rest, static_cast<std::uint32_t>(top));
      ch[top++] = p;
    }
    r.height = top;
    r.low_rest = rest;
  }

  const P2& at(std::size_t d) const {  // d-th entry from the top of G
    for (std::size_t s = G.size(); s-- > 0;) {
      const std::size_t len = G[s].to - G[s].from;
      if (d < len) return G[s].base[G[s].to - 1 - d];
      d -= len;
    }
    return G[0].base[0];  // unreachable: callers keep d < gsize
  }
  void pop() {
    if (--G.back().to == G.back().from) G.pop_back();
    --gsize;
  }
  void push_extra(const P2& p) {
    extra.push_back(p);  // reserved: never moves
    const std::size_t i = extra.size() - 1;
    if (!G.empty() && G.back().base == extra.data() && G.back().to == i) ++G.back().to;
    else G.push_back({extra.data(), i, i + 1});
    ++gsize;
  }

  void resolve() {  // phase B (sequential per arc)
    extra.reserve(n + 1);
    G.push_back({loc.data() + runs[0].b, 0, runs[0].height});  // chunk 0 is the true run
    gsize = runs[0].height;
    for (std::size_t j = 1; j < runs.size(); ++j) {
      const ChunkRun& r = runs[j];
      const std::size_t len = r.e - r.b;
      std::vector<std::size_t> C;  // chunk-local indices of G's chunk part
      std::size_t t = 0;
      bool synced = false;
      for (; t < std::min(len, kSyncWindow) && !synced; ++t) {
        const P2 p = pts[r.b + t];
        while (gsize >= 2 && !strict_left(at(1), at(0), p)) {
          pop();  // the chunk's own entries sit on top of the earlier ones
          if (!C.empty()) C.pop_back();
        }
        push_extra(p);
        C.push_back(t);
        const std::size_t h = r.low[t] + 1, c = C.size();
        std::uint32_t later = r.low_rest;  // min height after pops, later points
        for (std::size_t k = t + 1; k < std::min(len, kSyncWindow); ++k) later = std::min(later, r.low[k]);
        if (c < 2 || c > h || std::size_t(later) < h - c + 2) continue;
        bool same_top = true;  // local entry at level l = last point k <= t pushed at l
        for (std::size_t i = 0; i < c && same_top; ++i) {
          const std::size_t level = h - c + i;
          std::size_t k = t;
          while (r.low[k] != level) --k;
          same_top = k == C[i];
        }
        if (!same_top) continue;
        for (std::size_t i = 0; i < c; ++i) pop();
        G.push_back({loc.data() + r.b, h - c, r.height});
        gsize += r.height - (h - c);
        synced = true;
      }
      if (synced || t == len) continue;
      // no coincidence within the window: flatten G and run the plain loop
      PVec flat(gsize + (len - t));
      std::size_t top = 0;
      for (const Slice& sl : G) {
        std::memcpy(static_cast<void*>(flat.data() + top), sl.base + sl.from,
                    (sl.to - sl.from) * sizeof(P2));
        top += sl.to - sl.from;
      }
      for (std::size_t k = t; k < len; ++k) {
        const P2 p = pts[r.b + k];
        while (top >= 2 && !strict_left(flat[top - 2], flat[top - 1], p)) --top;
        flat[top++] = p;
      }
      flat.resize(top);
      extra.clear();  // nothing in G refers to it any more
      G.clear();
      gsize = top;
      flats.push_back(std::move(flat));
      G.push_back({flats.back().data(), 0, top});
    }
  }
  std::vector<PVec> flats;
};

}  // namespace

namespace {

// A cycle held as pieces of other buffers (the arcs' chain stacks), read as
// one virtual sequence.
struct PieceCycle {
  std::vector<const P2*> ptr;
  std::vector<std::size_t> off{0};  // piece k = [off[k], off[k+1])
  std::size_t n = 0;
  void add(const P2* p, std::size_t len) {
    if (!len) return;
    ptr.push_back(p);
    n += len;
    off.push_back(n);
  }
  std::size_t piece_of(std::size_t i) const {
    return static_cast<std::size_t>(std::upper_bound(off.begin(), off.end(), i) - off.begin()) - 1;
  }
  const P2& at(std::size_t i) const {
    const std::size_t k = piece_of(i);
    return ptr[k][i - off[k]];
  }
  // f(i, p) for i in [b, e), in order
  template <class F>
  void walk(std::size_t b, std::size_t e, F&& f) const {
    if (b >= e) return;
    std::size_t k = piece_of(b), j = b - off[k];
    for (std::size_t i = b; i < e; ++i, ++j) {
      while (j >= off[k + 1] - off[k]) {
        ++k;
        j = 0;
      }
      f(i, ptr[k][j]);
    }
  }
  // dst[0, e - b) = sequence[b, e)
  void copy_out(P2* dst, std::size_t b, std::size_t e) const {
    const std::size_t k0 = b < e ? piece_of(b) : 0;
    for (std::size_t k = k0; k + 1 < off.size() && off[k] < e; ++k) {
      const std::size_t s0 = std::max(b, off[k]), s1 = std::min(e, off[k + 1]);
      if (s0 < s1)
        std::memcpy(static_cast<void*>(dst + (s0 - b)), ptr[k] + (s0 - off[k]), (s1 - s0) * sizeof(P2));
    }
  }
  void copy_out_parallel(P2* dst, std::size_t b, std::size_t e) const {
    const std::size_t len = e - b;
    if (len < kParMin) {
      copy_out(dst, b, e);
      return;
    }
#pragma omp parallel
    {
      const int t = omp_get_thread_num(), nt = omp_get_num_threads();
      const std::size_t s0 = b + len * t / nt, s1 = b + len * (t + 1) / nt;
      copy_out(dst + (s0 - b), s0, s1);
    }
  }
};

struct ChainedArcs {
  ArcChain A[4];
  PieceCycle cycle;  // every arc's chain minus its last entry, in arc order
};

// The chains of the four arcs (already in sweep order); arcs of >= par_min
// points run in parallel chunks (all arcs' chunks in one parallel loop);
// wait_arc(q) is called before arc q is read.
std::unique_ptr<ChainedArcs> run_chains(const P2* const arcs[4], const std::uint64_t len[4],
                                        const ArcWait& wait_arc) {
  const std::size_t par_min = chain_par_min();
  static const std::size_t chunks = std::max<std::size_t>(2, env_size("OHX_CHAIN_CHUNKS", 16));
  auto R = std::make_unique<ChainedArcs>();
  ArcChain* A = R->A;
  struct Task {
    int q;
    std::size_t j;
  };
  std::vector<Task> tasks;
  for (int q = 0; q < 4; ++q) {
    A[q].pts = arcs[q];
    A[q].n = len[q];
    const std::size_t n = len[q];
    const std::size_t K = n >= par_min && n >= 2 * chunks ? chunks : 1;
    const std::size_t step = n ? (n + K - 1) / K : 0;
    for (std::size_t b = 0; b < n; b += step) A[q].runs.push_back({b, std::min(n, b + step), 0, {}, 0});
    A[q].loc.resize(n);
    for (std::size_t j = 0; j < A[q].runs.size(); ++j) tasks.push_back({q, j});
  }
  std::sort(tasks.begin(), tasks.end(), [&](const Task& x, const Task& y) {  // long runs first
    return A[x.q].runs[x.j].e - A[x.q].runs[x.j].b > A[y.q].runs[y.j].e - A[y.q].runs[y.j].b;
  });
  const std::uint64_t total = len[0] + len[1] + len[2] + len[3];
  const double t0 = now_ms();
  // an arc whose input never arrived (wait_arc false) is not chained: the
  // caller learns of the failure at once instead of after chaining garbage
  std::atomic<bool> lost[4] = {false, false, false, false};
#pragma omp parallel for schedule(dynamic, 1) if (total >= (1u << 12))
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(tasks.size()); ++i) {
    const int q = tasks[i].q;
    if (lost[q] || (wait_arc && !wait_arc(q))) {
      lost[q] = true;
      continue;
    }
    A[q].local_run(tasks[i].j);
  }
  for (int q = 0; q < 4; ++q)
    if (lost[q]) throw std::runtime_error("hull stage: the input of arc " + std::to_string(q + 1) +
                                          " did not arrive");
  const double t1 = now_ms();
#pragma omp parallel for schedule(dynamic, 1) if (total >= (1u << 12))
  for (int q = 0; q < 4; ++q)
    if (A[q].n) A[q].resolve();
  for (int q = 0; q < 4; ++q) {
    if (A[q].gsize == 0) continue;
    std::size_t keep = A[q].gsize - 1;  // the arc's last point is the next arc's entry
    for (const auto& sl : A[q].G) {
      const std::size_t l = std::min(keep, sl.to - sl.from);
      R->cycle.add(sl.base + sl.from, l);
      keep -= l;
    }
  }
  if (trace_on())
    std::fprintf(stderr, "[ohx]   chains: local runs %.3f ms, resolve %.3f ms (%zu tasks)\n",
                 t1 - t0, now_ms() - t1, tasks.size());
  return R;
}

// One parallel pass over a piece cycle: duplicates?  all collinear with
// (c0, c1)?  any non-strict turn?  the start vertex.
struct PieceScan {
  bool dups = false, flat = true, bad = false;
  std::size_t best = 0;
};

// (dst set: element i is also copied to dst[i] -- the unrotated cycle -- in
// the same pass)
PieceScan scan_pieces(const PieceCycle& c, P2* dst = nullptr) {
  PieceScan r;
  const std::size_t m = c.n;
  const P2 c0 = c.at(0), c1 = c.at(1);
  const int T = m >= kParMin ? omp_get_max_threads() : 1;
  std::vector<std::size_t> pb(T, m);
  std::vector<unsigned char> dups(T, 0), flat(T, 1), bad(T, 0);
#pragma omp parallel num_threads(T)
  {
    const int t = omp_get_thread_num(), nt = omp_get_num_threads();
    const std::size_t b = m * t / nt, e = m * (t + 1) / nt;
    if (b < e) {
      bool du = false, fl = true, ba = false;
      std::size_t bi = b;
      P2 bp = c.at(b);
      P2 prev = c.at(b == 0 ? m - 1 : b - 1), cur = bp;
      // cur = element i; the walk delivers i + 1 as `nx`
      auto step = [&](std::size_t i, const P2& nx) {
        if (dst) dst[i] = cur;
        if (i > 0) du = du || same(prev, cur);
        if (i >= 2) fl = fl && orient(c0, c1, cur) == 0;
        ba = ba || orient(prev, cur, nx) <= 0;
        if (i > b && starts_before(cur, bp)) {
          bi = i;
          bp = cur;
        }
        prev = cur;
        cur = nx;
      };
      c.walk(b + 1, e, [&](std::size_t i, const P2& nx) { step(i - 1, nx); });
      step(e - 1, c.at(e == m ? 0 : e));
      dups[t] = du;
      flat[t] = fl;
      bad[t] = ba;
      pb[t] = bi;
    }
  }
  for (int t = 0; t < T; ++t) {
    r.dups = r.dups || dups[t];
    r.flat = r.flat && flat[t];
    r.bad = r.bad || bad[t];
    if (pb[t] < m && (t == 0 || starts_before(c.at(pb[t]), c.at(r.best)))) r.best = pb[t];
  }
  return r;
}

}  // namespace

PVec chain_arcs(const P2* const arcs[4], const std::uint64_t len[4],
                const ArcWait& wait_arc) {
  auto R = run_chains(arcs, len, wait_arc);
  PVec cycle(R->cycle.n);
  R->cycle.copy_out_parallel(cycle.data(), 0, R->cycle.n);
  return cycle;
}

// The strict-left-turn chain of one arc already in sweep order (reference
// hull.cpp:140-149); the sweep's last point is dropped (it is the next
// arc's entry).  Long arcs run in parallel chunks with the same decisions.
PVec chain_sorted(const P2* pts, std::size_t n) {
  if (n == 0) return {};
  if (n >= chain_par_min()) {
    const P2* arcs[4] = {pts, pts, pts, pts};
    const std::uint64_t len[4] = {n, 0, 0, 0};
    return chain_arcs(arcs, len, {});
  }
  PVec chain(n);  // the plain loop
  P2* ch = chain.data();
  std::size_t top = 0;
  for (std::size_t k = 0; k < n; ++k) {
    const P2 p = pts[k];
    while (top >= 2 && !strict_left(ch[top - 2], ch[top - 1], p)) --top;
    ch[top++] = p;
  }
  chain.resize(top - 1);
  return chain;
}

PVec quadrant_chain(std::vector<P2> pts, int quadrant) {
  // reference hull.cpp:133-150
  if (pts.empty()) return {};
  const double t0 = now_ms();
  switch (quadrant) {
    case 1: sweep_sort<1>(pts); break;
    case 2: sweep_sort<2>(pts); break;
    case 3: sweep_sort<3>(pts); break;
    default: sweep_sort<4>(pts); break;
  }
  const double t1 = now_ms();
  PVec chain = chain_sorted(pts.data(), pts.size());
  if (trace_on())
    std::fprintf(stderr, "[ohx] hull q%d: %zu pts sort %.3f ms chain %.3f ms\n", quadrant,
                 pts.size(), t1 - t0, now_ms() - t1);
  return chain;
}

PVec finalize_cycle(PVec cycle) {
  // reference hull.cpp:94-120.  Consecutive duplicates collapse first (a
  // point is dropped iff it equals its predecessor: the last kept point
  // always equals the predecessor), then equal front/back pairs; a fully
  // collinear cycle reduces to its two extreme points, any other is peeled
  // to strict left turns; the result starts at the east-most vertex.
  double tt = now_ms();
  auto tmark = [&](const char* w) {
    if (trace_on()) std::fprintf(stderr, "[ohx]   finalize %-8s %.3f ms\n", w, now_ms() - tt);
    tt = now_ms();
  };
  const std::size_t n0 = cycle.size();
  if (n0 > 2 && !same(cycle.front(), cycle.back())) {
    // fast path: one fused parallel scan; valid as is when the cycle has no
    // duplicates (the usual case: chains of strict turns)
    CycleScan sc = scan_cycle(cycle);
    tmark("scan");
    if (!sc.dups) {
      if (sc.flat) {
        const auto mm = std::minmax_element(cycle.begin(), cycle.end(), lex);
        PVec d = {*mm.first, *mm.second};
        rotate_to(d, start_vertex(d));
        return d;
      }
      const bool removed = peel(cycle, std::move(sc.bad));
      tmark("peel");
      rotate_to(cycle, removed ? start_vertex(cycle) : sc.best);
      tmark("rotate");
      return cycle;
    }
  }
  PVec d;
  {
    const P2* c = cycle.data();
    d = compact(c, n0, [&](std::size_t k) { return k == 0 || !same(c[k - 1], c[k]); });
    PVec().swap(cycle);
  }
  tmark("dedup");
  while (d.size() > 1 && same(d.front(), d.back())) d.pop_back();
  const std::size_t m = d.size();
  if (m > 2) {
    bool flat = true;
#pragma omp parallel for schedule(static) reduction(&& : flat) if (m >= kParMin)
    for (std::int64_t k = 2; k < static_cast<std::int64_t>(m); ++k)
      flat = flat && orient(d[0], d[1], d[k]) == 0;
    if (flat) {
      const auto mm = std::minmax_element(d.begin(), d.end(), lex);
      d = {*mm.first, *mm.second};
    } else {
      peel(d, non_strict_turns(d));
    }
    tmark("peel");
  }
  if (d.size() >= 2) rotate_to(d, start_vertex(d));
  tmark("rotate");
  return d;
}

std::size_t hull_from_sorted_arcs(const P2* const arcs[4], const std::uint64_t len[4],
                                  const ArcWait& wait_arc, const HullSink& sink) {
  const std::uint64_t total = len[0] + len[1] + len[2] + len[3];
  const double t0 = now_ms();
  auto R = run_chains(arcs, len, wait_arc);
  const PieceCycle& pc = R->cycle;
  const double t1 = now_ms();
  std::size_t h = 0;
  // fast path: no duplicates, no non-strict turn, not flat (the clean-up
  // keeps every vertex): the hull is the cycle rotated to its start vertex.
  // The checking scan also copies the cycle to the output (one pass over
  // the chain stacks instead of two); the start is nearly always the first
  // vertex (the east anchor), else the rotated copy is redone.
  bool done = false;
  if (pc.n > 2 && !same(pc.at(0), pc.at(pc.n - 1))) {
    P2* out = nullptr;
    try {
      out = sink(pc.n);
    } catch (...) {  // no room for the whole cycle: check first, the hull may be smaller
      out = nullptr;
    }
    const PieceScan sc = scan_pieces(pc, out);
    if (trace_on()) std::fprintf(stderr, "[ohx]   piece scan + copy %.3f ms\n", now_ms() - t1);
    if (!sc.dups && !sc.flat && !sc.bad) {
      h = pc.n;
      if (!out || sc.best != 0) {
        if (!out) out = sink(h);
        pc.copy_out_parallel(out, sc.best, pc.n);
        pc.copy_out_parallel(out + (pc.n - sc.best), 0, sc.best);
      }
      done = true;
    }
  }
  if (!done) {  // the general clean-up on a contiguous copy
    PVec cycle(pc.n);
    pc.copy_out_parallel(cycle.data(), 0, pc.n);
    PVec d = finalize_cycle(std::move(cycle));
    h = d.size();
    copy_points(sink(h), d.data(), h);
  }
  if (trace_on())
    std::fprintf(stderr,
                 "[ohx] hull chains (sorted arcs, %llu pts) %.3f ms, clean-up + output %zu vertices %.3f ms%s\n",
                 static_cast<unsigned long long>(total), t1 - t0, h, now_ms() - t1,
                 done ? " (fast path)" : "");
  return h;
}

PVec hull_from_sorted_arcs(const P2* const arcs[4], const std::uint64_t len[4],
                           const ArcWait& wait_arc) {
  PVec out;
  hull_from_sorted_arcs(arcs, len, wait_arc, [&](std::size_t h) {
    out.resize(h);
    return out.data();
  });
  return out;
}

// Three persistent workers for the arcs 1..3 of hull_from_queue_points
// (the caller runs arc 0): starting threads per call cost more than the
// sorts of a few thousand points, and the workers keep warm heaps.  One
// job at a time (calls from several host threads queue on the mutex).
class ArcWorkers {
 public:
  static ArcWorkers& get() {
    // never destroyed: the workers wait until process exit ends them (no
    // join at exit; a forked child's copy holds threads it does not have)
    static ArcWorkers* w = new ArcWorkers;
    return *w;
  }
  void run4(const std::function<void(int)>& f) {
    if (getpid() != pid_) {  // a forked child: the workers did not survive the fork
      for (int q = 0; q < 4; ++q) f(q);
      return;
    }
    std::lock_guard<std::mutex> call(call_);
    {
      std::lock_guard<std::mutex> lk(m_);
      job_ = &f;
      left_ = 3;
      ++gen_;
    }
    cv_.notify_all();
    std::exception_ptr mine;
    try {
      f(0);
    } catch (...) {
      mine = std::current_exception();
    }
    std::unique_lock<std::mutex> lk(m_);
    done_.wait(lk, [&] { return left_ == 0; });  // the workers hold f: always wait
    job_ = nullptr;
    std::exception_ptr e = mine ? mine : err_;
    err_ = nullptr;
    if (e) std::rethrow_exception(e);
  }

 private:
  ArcWorkers() : pid_(getpid()) {
    for (int k = 1; k <= 3; ++k) th_.emplace_back([this, k] { loop(k); });
  }
  void loop(int k) {
    std::uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* f;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        f = job_;
      }
      std::exception_ptr e;
      try {
        (*f)(k);
      } catch (...) {
        e = std::current_exception();
      }
      std::lock_guard<std::mutex> lk(m_);
      if (e && !err_) err_ = e;
      if (--left_ == 0) done_.notify_one();
    }
  }
  const pid_t pid_;
  std::mutex call_, m_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  std::exception_ptr err_;
  int left_ = 0;
  std::uint64_t gen_ = 0;
  std::vector<std::thread> th_;
};

PVec hull_from_queue_points(const P2 anchors[4], const P2* const q_pts[4],
                            const std::uint64_t q_len[4]) {
  // reference hull.cpp:164-183: arc q runs from anchor q-1 (entry) to
  // anchor q (exit) over the queue's members, in queue order
  PVec chains[4];
  auto arc = [&](int q) {
    std::vector<P2> cand;
    cand.reserve(q_len[q] + 2);
    cand.push_back(anchors[q]);
    cand.insert(cand.end(), q_pts[q], q_pts[q] + q_len[q]);
    cand.push_back(anchors[(q + 1) % 4]);
    chains[q] = quadrant_chain(std::move(cand), q + 1);
  };
  const std::uint64_t total = q_len[0] + q_len[1] + q_len[2] + q_len[3];
  if (total >= (1u << 12)) {  // one thread per arc
    const std::function<void(int)> job = arc;
    ArcWorkers::get().run4(job);
  } else {
    for (int q = 0; q < 4; ++q) arc(q);
  }
  PVec cycle;
  for (int q = 0; q < 4; ++q) cycle.insert(cycle.end(), chains[q].begin(), chains[q].end());
  const double t0 = now_ms();
  PVec out = finalize_cycle(std::move(cycle));
  if (trace_on())
    std::fprintf(stderr, "[ohx] hull finalize: %zu vertices %.3f ms\n", out.size(), now_ms() - t0);
  return out;
}

PVec monotone_chain(const P2* pts, std::uint64_t n) {
  // reference hull.cpp:205-232
  std::vector<P2> s(pts, pts + n);
  big_sort(s, lex);
  s.erase(std::unique(s.begin(), s.end(), same), s.end());
  if (s.size() <= 2) return PVec(s.begin(), s.end());
  PVec lo, hi;
  for (const P2& p : s) {
    while (lo.size() >= 2 && orient(lo[lo.size() - 2], lo.back(), p) <= 0) lo.pop_back();
    lo.push_back(p);
  }
  for (auto it = s.rbegin(); it != s.rend(); ++it) {
    while (hi.size() >= 2 && orient(hi[hi.size() - 2], hi.back(), *it) <= 0) hi.pop_back();
    hi.push_back(*it);
  }
  PVec cyc(lo.begin(), lo.end() - 1);
  cyc.insert(cyc.end(), hi.begin(), hi.end() - 1);
  return cyc;
}

}  // namespace ohx
