// hullchain.cu -- the hull stage's chains and cycle scan on the device
// (SURVEY §8f item 3), for survivor sets that arrive sorted from
// hullsort.cu.
//
// Reference semantics (hull.cpp:133-150): per quadrant arc, in sweep order,
//   while (|chain| >= 2 && orientation(chain[-2], chain[-1], p) <= 0) pop;
//   push p;   ... and finally drop the arc's last point.
// The chain must take the reference loop's exact decisions (a generic
// parallel hull evaluates other orientation triples, which on
// near-degenerate inputs -- 1e8 points on a circle -- need not agree), so
// the parallel form is the same "replay until coincidence" as the host
// chains (hull.cpp ArcChain), arranged for thousands of chunks:
//
//  1. chain_local: one thread per chunk of ~kChunk points runs the loop
//     from an empty stack, in place (its stack overwrites its own slice of
//     the chunk buffer), recording the stack height after each of the
//     first kWin points' pops and the minimum height after that.
//  2. chain_replay: one thread per chunk j >= 1 replays the TRUE loop over
//     its first points, starting from chunk j-1's final local stack, until
//     it provably coincides with its own local run (the part of the true
//     stack pushed in chunk j equals the local stack's top c >= 2 entries,
//     and the local run never again drops below their base + 2: every later
//     test and pop sees the same entries).  Chunk j-1's final local stack
//     above ITS sync base is the true stack's top when chunk j starts --
//     provided chunk j-1 synced and chunk j's replay never reads below that
//     base, which is checked next; the replay records the lowest level of
//     chunk j-1's stack it read and where it left chunk j-1's top.
//  3. chain_check: every chunk synced and every replay stayed above its
//     predecessor's base => by induction over the chunks, the arc's true
//     final stack is the concatenation of the chunks' slices
//     [base_j, top_j) (top_j = where chunk j+1's replay left it, the last
//     chunk's own height); otherwise the call reports failure and the host
//     chains run (the sorted arcs are still on the device).
//  4. an exclusive scan of the slice lengths and a copy give the cycle
//     (the four arcs' chains, each without its last point).
//  5. cycle_stats: one reduction over the cycle -- consecutive duplicates,
//     all collinear with (c0, c1), non-strict turns, and the start vertex
//     (max x, ties to the smaller y, first occurrence; hull.cpp:35-49) --
//     decides whether finalize_cycle (hull.cpp:94-120) keeps every vertex,
//     in which case the hull is the cycle rotated to its start.
//
// Orientation is the reference's binary64 determinant with explicit _rn
// intrinsics (no contraction; the TU is also built with -fmad=false).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstring>
#include <cstdlib>
#include <string>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "internal.hpp"

namespace ohx {
namespace {

constexpr int kChunk = 1024;  // points per chunk (chunks hold kChunk .. 2 kChunk - 1)
constexpr int kWin = 64;      // replay window (points)

__device__ __forceinline__ bool strict_left(double2 a, double2 b, double2 p) {
  // orientation(a, b, p) > 0 (reference geometry.hpp:27-32)
  const double l = __dmul_rn(__dsub_rn(b.x, a.x), __dsub_rn(p.y, a.y));
  const double r = __dmul_rn(__dsub_rn(b.y, a.y), __dsub_rn(p.x, a.x));
  return __dsub_rn(l, r) > 0.0;
}

struct ArcGeom {
  std::uint64_t aoff[4], len[4];
  std::uint32_t nch[4], choff[5];  // chunks per arc, first chunk of each arc
  std::uint32_t c_lo, c_hi;        // the chunks a launch works on (all, or one arc's)
};

struct ChunkPos {
  int q;
  std::uint32_t j;
  std::uint64_t b, e;
};

__device__ __forceinline__ ChunkPos chunk_pos(const ArcGeom& g, std::uint32_t c) {
  ChunkPos p;
  p.q = (c >= g.choff[1]) + (c >= g.choff[2]) + (c >= g.choff[3]);
  p.j = c - g.choff[p.q];
  const std::uint64_t n = g.len[p.q], k = g.nch[p.q];
  p.b = g.aoff[p.q] + n * p.j / k;
  p.e = g.aoff[p.q] + n * (p.j + 1) / k;
  return p;
}

// per-chunk state (structure of arrays in one work area)
struct ChunkState {
  std::uint32_t* height;    // final local stack height
  std::uint32_t* low_rest;  // min height after pops over the points >= kWin
  std::uint16_t* low;       // [chunk][kWin] height after point k's pops
  std::uint32_t* base;      // sync base (chunk 0 of an arc: 0)
  std::uint32_t* keep;      // chunk j-1's top as left by chunk j's replay
  std::int32_t* deep;       // lowest level of chunk j-1's stack the replay read
  std::uint8_t* synced;
  std::uint64_t* slice;     // slice length, then (scan) its offset in the cycle
  std::uint64_t* offs;
};

// One thread per chunk: the lanes of a warp walk 32 different chunks, so
// the points are staged through shared memory kCT at a time with coalesced
// loads (two chunks' kCT-point runs per load instruction) -- direct
// per-lane loads fetched 32 separate lines per warp load.
constexpr int kCT = 16;  // points per chunk per staging round
__global__ void __launch_bounds__(128) chain_local(const double2* __restrict__ in, double2* loc,
                                                   ArcGeom g, ChunkState st) {
  __shared__ double2 tile[4][32][kCT + 1];  // per warp: 32 chunks x kCT (+1: 4-way banks)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const std::uint32_t c = g.c_lo + blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = c < g.c_hi;
  std::uint64_t b0 = 0;
  std::uint32_t len = 0;
  if (live) {
    const ChunkPos p = chunk_pos(g, c);
    b0 = p.b;
    len = static_cast<std::uint32_t>(p.e - p.b);
  }
  double2* s = loc + b0;
  std::uint32_t top = 0, rest = 0xffffffffu;
  double2 s0 = make_double2(0, 0), s1 = make_double2(0, 0);  // s[top-2], s[top-1]
  std::uint16_t* low = st.low + std::uint64_t(c) * kWin;
  const std::uint32_t maxlen = __reduce_max_sync(0xffffffffu, len);
  const int half = lane >> 4, hl = lane & 15;
  for (std::uint32_t t0 = 0; t0 < maxlen; t0 += kCT) {
#pragma unroll 4
    for (int j = 0; j < 32; j += 2) {  // chunks j (lanes 0-15) and j+1 (lanes 16-31)
      const std::uint64_t bj = __shfl_sync(0xffffffffu, b0, j + half);
      const std::uint32_t lj = __shfl_sync(0xffffffffu, len, j + half);
      if (t0 + hl < lj) tile[warp][j + half][hl] = __ldg(in + bj + t0 + hl);
    }
    __syncwarp();
    const std::uint32_t kend = min(len, t0 + kCT);
    for (std::uint32_t k = t0; k < kend; ++k) {
      const double2 pt = tile[warp][lane][k - t0];
      while (top >= 2 && !strict_left(s0, s1, pt)) {
        --top;
        s1 = s0;
        if (top >= 2) s0 = s[top - 2];
      }
      if (k < kWin) low[k] = static_cast<std::uint16_t>(top);
      else rest = min(rest, top);
      s[top] = pt;
      s0 = s1;
      s1 = pt;
      ++top;
    }
    __syncwarp();
  }
  if (!live) return;
  st.height[c] = top;
  st.low_rest[c] = rest;
}

__global__ void __launch_bounds__(128) chain_replay(const double2* __restrict__ in,
                                                    const double2* __restrict__ loc, ArcGeom g,
                                                    ChunkState st) {
  const std::uint32_t c = g.c_lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= g.c_hi) return;
  const ChunkPos p = chunk_pos(g, c);
  if (p.j == 0) {  // the arc's first chunk: its local run is the true run
    st.base[c] = 0;
    st.synced[c] = 1;
    st.deep[c] = INT_MAX;
    st.keep[c] = 0;
    return;
  }
  const ChunkPos pp = chunk_pos(g, c - 1);
  const double2* P = loc + pp.b;               // chunk j-1's final local stack
  const bool exact_below = pp.j == 0;          // nothing under chunk j-1's stack
  std::int64_t k = st.height[c - 1];           // its top as this replay leaves it
  const double2* src = in + p.b;
  const std::uint16_t* low = st.low + std::uint64_t(c) * kWin;
  const std::uint32_t len = static_cast<std::uint32_t>(p.e - p.b);
  const std::uint32_t W = len < kWin ? len : kWin;
  std::uint16_t C[kWin];  // chunk-local indices of the true stack's chunk part
  int cn = 0;
  std::int64_t deep = INT_MAX;
  bool ok = false;
  for (std::uint32_t t = 0; t < W && !ok; ++t) {
    const double2 pt = src[t];
    for (;;) {
      if (k + cn < 2) {
        if (!exact_below) deep = -1;  // would read under chunk j-1's stack
        break;
      }
      double2 a1, a0;
      if (cn >= 2) {
        a1 = src[C[cn - 2]];
        a0 = src[C[cn - 1]];
      } else if (cn == 1) {
        a1 = P[k - 1];
        a0 = src[C[0]];
        deep = min(deep, k - 1);
      } else {
        a1 = P[k - 2];
        a0 = P[k - 1];
        deep = min(deep, k - 2);
      }
      if (strict_left(a1, a0, pt)) break;
      if (cn > 0) --cn;
      else --k;
    }
    if (deep < 0) break;
    C[cn++] = static_cast<std::uint16_t>(t);
    // coincidence with the local run after point t (hull.cpp ArcChain::resolve)
    const std::uint32_t h = low[t] + 1u;
    const std::uint32_t cc = static_cast<std::uint32_t>(cn);
    std::uint32_t later = st.low_rest[c];
    for (std::uint32_t q = t + 1; q < W; ++q) later = min(later, static_cast<std::uint32_t>(low[q]));
    if (cc < 2 || cc > h || later < h - cc + 2) continue;
    bool same = true;  // local entry at level l = the last point <= t pushed at l
    for (std::uint32_t i = 0; i < cc && same; ++i) {
      const std::uint32_t level = h - cc + i;
      std::uint32_t q = t;
      while (low[q] != level) --q;
      same = q == C[i];
    }
    if (!same) continue;
    ok = true;
    st.base[c] = h - cc;
  }
  st.synced[c] = ok ? 1 : 0;
  st.deep[c] = deep < 0 ? -1 : static_cast<std::int32_t>(deep > INT_MAX ? INT_MAX : deep);
  st.keep[c] = static_cast<std::uint32_t>(k < 0 ? 0 : k);
}

// slice lengths; *fail set when the chunk decomposition does not hold
__global__ void chain_check(ArcGeom g, ChunkState st, int* fail) {
  const std::uint32_t c = g.c_lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= g.c_hi) return;
  const ChunkPos p = chunk_pos(g, c);
  const bool last = p.j + 1 == g.nch[p.q];
  bool ok = st.synced[c] != 0;
  const std::uint32_t base = st.base[c];
  std::uint64_t top = st.height[c];
  if (!last) {
    ok = ok && st.deep[c + 1] >= 0 && static_cast<std::uint32_t>(st.deep[c + 1]) >= base;
    top = st.keep[c + 1];
  }
  if (!ok || top < base) {
    atomicExch(fail, 1);
    st.slice[c] = 0;
    return;
  }
  std::uint64_t L = top - base;
  if (last) L = L > 0 ? L - 1 : 0;  // the arc's last point is the next arc's entry
  st.slice[c] = L;
}

__global__ void __launch_bounds__(128) chain_copy(const double2* __restrict__ loc, ArcGeom g,
                                                  ChunkState st, double2* __restrict__ cycle) {
  const std::uint32_t c = g.c_lo + blockIdx.x;
  const ChunkPos p = chunk_pos(g, c);
  const double2* s = loc + p.b + st.base[c];
  double2* d = cycle + st.offs[c];
  const std::uint64_t L = st.slice[c];
  // four independent loads in flight per thread (one at a time left the
  // copy latency-bound: 0.65 -> 0.55 ms for the circle's 1.55 GB)
  std::uint64_t i = threadIdx.x;
  for (; i + 3 * blockDim.x < L; i += 4 * blockDim.x) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = s[i + u * blockDim.x];
#pragma unroll
    for (int u = 0; u < 4; ++u) d[i + u * blockDim.x] = v[u];
  }
  for (; i < L; i += blockDim.x) d[i] = s[i];
}

// ---- cycle statistics (finalize_cycle's fast-path test)
struct CycStat {
  double bx, by;
  std::uint64_t bi;
  std::uint32_t dups, notflat;
  std::uint64_t bad;
};

__device__ __forceinline__ int orient_sign(double2 a, double2 b, double2 c) {
  const double l = __dmul_rn(__dsub_rn(b.x, a.x), __dsub_rn(c.y, a.y));
  const double r = __dmul_rn(__dsub_rn(b.y, a.y), __dsub_rn(c.x, a.x));
  const double det = __dsub_rn(l, r);
  return det > 0.0 ? 1 : (det < 0.0 ? -1 : 0);
}

struct StatOf {
  const double2* c;
  std::uint64_t m;
  __device__ CycStat operator()(std::uint64_t i) const {
    const double2 a = c[i == 0 ? m - 1 : i - 1], b = c[i], n = c[i + 1 == m ? 0 : i + 1];
    CycStat s;
    s.bx = b.x;
    s.by = b.y;
    s.bi = i;
    s.dups = i > 0 && a.x == b.x && a.y == b.y;
    s.notflat = i >= 2 && orient_sign(c[0], c[1], b) != 0;
    s.bad = orient_sign(a, b, n) <= 0 ? 1 : 0;
    return s;
  }
};

struct StatCombine {
  __device__ CycStat operator()(const CycStat& u, const CycStat& v) const {
    CycStat r;
    r.dups = u.dups | v.dups;
    r.notflat = u.notflat | v.notflat;
    r.bad = u.bad + v.bad;
    // starts_before (hull.cpp:35-38), ties to the smaller index: a total
    // order, so the combine is commutative as well as associative
    bool take_v;
    if (u.bx != v.bx) take_v = v.bx > u.bx;
    else if (u.by != v.by) take_v = v.by < u.by;
    else take_v = v.bi < u.bi;
    r.bx = take_v ? v.bx : u.bx;
    r.by = take_v ? v.by : u.by;
    r.bi = take_v ? v.bi : u.bi;
    return r;
  }
};

__device__ __forceinline__ CycStat stat_identity() {
  CycStat s;
  s.bx = -INFINITY;
  s.by = INFINITY;
  s.bi = ~0ull;
  s.dups = 0;
  s.notflat = 0;
  s.bad = 0;
  return s;
}

// one CycStat per 128-thread block (thread 0 holds it)
__device__ __forceinline__ CycStat block_stat(CycStat v) {
  __shared__ CycStat part[4];
  const StatCombine comb;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    CycStat o;
    o.bx = __shfl_down_sync(0xffffffffu, v.bx, off);
    o.by = __shfl_down_sync(0xffffffffu, v.by, off);
    o.bi = __shfl_down_sync(0xffffffffu, v.bi, off);
    o.dups = __shfl_down_sync(0xffffffffu, v.dups, off);
    o.notflat = 0;
    o.bad = __shfl_down_sync(0xffffffffu, v.bad, off);
    v = comb(v, o);
  }
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0)
    for (int w = 1; w < 4; ++w) v = comb(v, part[w]);
  return v;
}

// chain_copy + the cycle statistics of the slice's own positions (all four
// arcs): every position's best-start candidacy, the duplicate test of every
// pair inside the slice and the turn test of every position with both
// neighbours inside it; the slice ends' tests need the neighbouring slices
// and are done by chain_stat_ends once the cycle is written.  Saves the
// reduction's second read of the whole cycle (1.55 GB on the circle).
__global__ void __launch_bounds__(128) chain_copy_stats(const double2* __restrict__ loc,
                                                        ArcGeom g, ChunkState st,
                                                        double2* __restrict__ cycle,
                                                        CycStat* __restrict__ part) {
  const std::uint32_t c = g.c_lo + blockIdx.x;
  const ChunkPos p = chunk_pos(g, c);
  const double2* s = loc + p.b + st.base[c];
  const std::uint64_t o = st.offs[c];
  double2* d = cycle + o;
  const std::uint64_t L = st.slice[c];
  CycStat acc = stat_identity();
  auto visit = [&](std::uint64_t i, double2 b) {
    bool take;  // starts_before (hull.cpp:35-38), ties to the smaller index
    if (b.x != acc.bx) take = b.x > acc.bx;
    else if (b.y != acc.by) take = b.y < acc.by;
    else take = o + i < acc.bi;
    if (take) {
      acc.bx = b.x;
      acc.by = b.y;
      acc.bi = o + i;
    }
    if (i >= 1) {
      const double2 a = __ldg(s + i - 1);
      acc.dups |= a.x == b.x && a.y == b.y;
      if (i + 1 < L) acc.bad += orient_sign(a, b, __ldg(s + i + 1)) <= 0 ? 1 : 0;
    }
  };
  std::uint64_t i = threadIdx.x;
  for (; i + 3 * blockDim.x < L; i += 4 * blockDim.x) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = s[i + u * blockDim.x];
#pragma unroll
    for (int u = 0; u < 4; ++u) d[i + u * blockDim.x] = v[u];
#pragma unroll
    for (int u = 0; u < 4; ++u) visit(i + u * blockDim.x, v[u]);
  }
  for (; i < L; i += blockDim.x) {
    const double2 v = s[i];
    d[i] = v;
    visit(i, v);
  }
  acc = block_stat(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

struct CycMeta {
  double2 tail;            // cycle[m - 1]
  std::uint64_t m;
  std::uint32_t notflat3;  // orientation(c[0], c[1], c[2]) != 0
  std::uint32_t pad;
};

// the slice ends' statistics (first and last position of every non-empty
// slice, with their neighbours in the written cycle) into part[G + k]; the
// cycle length, its last point and the first three points' turn into meta
__global__ void chain_stat_ends(ArcGeom g, ChunkState st, const double2* __restrict__ cycle,
                                CycStat* __restrict__ part, CycMeta* meta) {
  const std::uint32_t G = g.c_hi - g.c_lo;
  const std::uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= G) return;
  const std::uint32_t c = g.c_lo + k, last = g.c_hi - 1;
  const std::uint64_t m = st.offs[last] + st.slice[last];
  CycStat acc = stat_identity();
  const std::uint64_t L = st.slice[c];
  if (L && m) {
    const std::uint64_t p0 = st.offs[c], p1 = p0 + L - 1;
    const double2 a0 = cycle[p0 ? p0 - 1 : m - 1], b0 = cycle[p0],
                  n0 = cycle[p0 + 1 == m ? 0 : p0 + 1];
    acc.dups = p0 > 0 && a0.x == b0.x && a0.y == b0.y;
    acc.bad = orient_sign(a0, b0, n0) <= 0 ? 1 : 0;
    if (L >= 2)
      acc.bad += orient_sign(cycle[p1 - 1], cycle[p1], cycle[p1 + 1 == m ? 0 : p1 + 1]) <= 0 ? 1 : 0;
  }
  part[G + k] = acc;
  if (k == 0) {
    CycMeta mt{};
    mt.m = m;
    if (m) mt.tail = cycle[m - 1];
    mt.notflat3 = m >= 3 && orient_sign(cycle[0], cycle[1], cycle[2]) != 0;
    *meta = mt;
  }
}

// OHX_CYCLE_STATS=reduce: the statistics as a separate reduction over the
// whole cycle (A/B and test hook)
bool fused_cycle_stats() {
  static const bool v = [] {
    const char* e = std::getenv("OHX_CYCLE_STATS");
    return !(e && std::string(e) == "reduce");
  }();
  return v;
}

std::size_t align256(std::size_t b) { return (b + 255) & ~std::size_t(255); }

ArcGeom arc_geom(const std::uint64_t len[4]) {
  ArcGeom g{};
  std::uint64_t a = 0;
  std::uint32_t ch = 0;
  for (int q = 0; q < 4; ++q) {
    g.aoff[q] = a;
    g.len[q] = len[q];
    a += len[q];
    g.nch[q] = static_cast<std::uint32_t>(len[q] >= 2 * kChunk ? len[q] / kChunk : 1);
    g.choff[q] = ch;
    ch += g.nch[q];
  }
  g.choff[4] = ch;
  g.c_lo = 0;
  g.c_hi = ch;
  return g;
}

std::size_t scan_tmp_bytes(std::uint32_t chunks) {
  std::size_t b = 0;
  check_cuda(cub::DeviceScan::ExclusiveSum(nullptr, b, static_cast<std::uint64_t*>(nullptr),
                                           static_cast<std::uint64_t*>(nullptr),
                                           static_cast<int>(chunks)),
             "cub scan temp size");
  return b;
}

std::size_t stat_tmp_bytes(std::uint64_t m) {
  std::size_t b = 0;
  thrust::counting_iterator<std::uint64_t> it(0);
  thrust::transform_iterator<StatOf, thrust::counting_iterator<std::uint64_t>, CycStat> tin(
      it, StatOf{nullptr, 1});
  check_cuda(cub::DeviceReduce::Reduce(nullptr, b, tin, static_cast<CycStat*>(nullptr),
                                       static_cast<std::int64_t>(m), StatCombine{}, CycStat{}),
             "cub reduce temp size");
  return b;
}

std::size_t part_tmp_bytes(std::uint64_t k) {
  std::size_t b = 0;
  check_cuda(cub::DeviceReduce::Reduce(nullptr, b, static_cast<const CycStat*>(nullptr),
                                       static_cast<CycStat*>(nullptr),
                                       static_cast<std::int64_t>(k), StatCombine{}, CycStat{}),
             "cub reduce temp size");
  return b;
}

struct ChainLayout {
  ArcGeom g;
  std::uint64_t total;
  std::size_t bytes;
  std::size_t o_loc, o_cycle, o_h, o_lr, o_low, o_base, o_keep, o_deep, o_sync, o_slice, o_offs,
      o_stat, o_part, o_flag, o_tmp;
  std::size_t tmp_bytes;
};

ChainLayout chain_layout(const std::uint64_t len[4]) {
  ChainLayout L{};
  L.g = arc_geom(len);
  L.total = len[0] + len[1] + len[2] + len[3];
  const std::uint32_t G = L.g.choff[4];
  std::size_t o = 0;
  auto take = [&](std::size_t b) {
    const std::size_t r = o;
    o += align256(b);
    return r;
  };
  L.o_loc = take(L.total * 16);
  L.o_cycle = take(L.total * 16);
  L.o_h = take(G * 4ull);
  L.o_lr = take(G * 4ull);
  L.o_low = take(G * 2ull * kWin);
  L.o_base = take(G * 4ull);
  L.o_keep = take(G * 4ull);
  L.o_deep = take(G * 4ull);
  L.o_sync = take(G);
  L.o_slice = take(G * 8ull);
  L.o_offs = take(G * 8ull);
  L.o_stat = take(sizeof(CycStat));
  L.o_part = take(2ull * G * sizeof(CycStat) + sizeof(CycMeta));
  L.o_flag = take(16);
  const std::size_t a = scan_tmp_bytes(G), b = stat_tmp_bytes(L.total),
                    c = part_tmp_bytes(2ull * G);
  L.tmp_bytes = std::max(a, std::max(b, c));
  L.o_tmp = take(L.tmp_bytes);
  L.bytes = o;
  return L;
}

}  // namespace

static void cycle_stats_into(const double2* cycle, std::uint64_t m, CycStat* stat, void* tmp,
                             std::size_t tmp_bytes, cudaStream_t s, DeviceCycle* out);

std::size_t device_chain_work_bytes(const std::uint64_t len[4]) { return chain_layout(len).bytes; }

bool device_chains(const double* d_sorted, const std::uint64_t len[4], void* d_work,
                   cudaStream_t s, DeviceCycle* out, double* direct, std::uint64_t direct_cap,
                   int only_q) {
  ChainLayout L = chain_layout(len);
  if (only_q >= 0) {  // one arc's chain, alone, at the start of the cycle buffer
    L.g.c_lo = L.g.choff[only_q];
    L.g.c_hi = L.g.choff[only_q + 1];
  }
  const std::uint64_t need = only_q >= 0 ? len[only_q] : L.total;
  auto* w = static_cast<unsigned char*>(d_work);
  auto* loc = reinterpret_cast<double2*>(w + L.o_loc);
  // the cycle straight into the caller's device buffer when it can hold
  // every arc point (the hull is usually the cycle as is)
  auto* cycle = direct != nullptr && direct_cap >= need ? reinterpret_cast<double2*>(direct)
                                                        : reinterpret_cast<double2*>(w + L.o_cycle);
  ChunkState st;
  st.height = reinterpret_cast<std::uint32_t*>(w + L.o_h);
  st.low_rest = reinterpret_cast<std::uint32_t*>(w + L.o_lr);
  st.low = reinterpret_cast<std::uint16_t*>(w + L.o_low);
  st.base = reinterpret_cast<std::uint32_t*>(w + L.o_base);
  st.keep = reinterpret_cast<std::uint32_t*>(w + L.o_keep);
  st.deep = reinterpret_cast<std::int32_t*>(w + L.o_deep);
  st.synced = w + L.o_sync;
  st.slice = reinterpret_cast<std::uint64_t*>(w + L.o_slice);
  st.offs = reinterpret_cast<std::uint64_t*>(w + L.o_offs);
  auto* stat = reinterpret_cast<CycStat*>(w + L.o_stat);
  int* flag = reinterpret_cast<int*>(w + L.o_flag);
  void* tmp = w + L.o_tmp;
  const auto* in = reinterpret_cast<const double2*>(d_sorted);
  const std::uint32_t G = L.g.c_hi - L.g.c_lo;
  const unsigned blocks = (G + 127) / 128;

  check_cuda(cudaMemsetAsync(flag, 0, sizeof(int), s), "cudaMemsetAsync(chain flag)");
  chain_local<<<blocks, 128, 0, s>>>(in, loc, L.g, st);
  check_cuda(cudaGetLastError(), "chain_local launch");
  chain_replay<<<blocks, 128, 0, s>>>(in, loc, L.g, st);
  check_cuda(cudaGetLastError(), "chain_replay launch");
  chain_check<<<blocks, 128, 0, s>>>(L.g, st, flag);
  check_cuda(cudaGetLastError(), "chain_check launch");
  std::size_t tb = L.tmp_bytes;
  check_cuda(cub::DeviceScan::ExclusiveSum(tmp, tb, st.slice + L.g.c_lo, st.offs + L.g.c_lo,
                                           static_cast<int>(G), s),
             "cub::DeviceScan::ExclusiveSum(slices)");
  struct Head {
    int fail;
    std::uint32_t pad;
    std::uint64_t last_off, last_len;
  };
  Head hd{};
  // all four arcs: the cycle statistics with the copy (chain_copy_stats +
  // the slice ends + a reduction over 2 G partials), read with the head in
  // the same sync; one arc (the pipelined stage) needs none
  const bool fused = only_q < 0 && fused_cycle_stats();
  auto* part = reinterpret_cast<CycStat*>(w + L.o_part);
  auto* meta = reinterpret_cast<CycMeta*>(part + 2ull * G);
  // the copy runs regardless (harmless on failure: every slice length is
  // then whatever chain_check wrote, bounded by the chunk)
  if (fused) {
    chain_copy_stats<<<G, 128, 0, s>>>(loc, L.g, st, cycle, part);
    check_cuda(cudaGetLastError(), "chain_copy_stats launch");
    chain_stat_ends<<<(G + 127) / 128, 128, 0, s>>>(L.g, st, cycle, part, meta);
    check_cuda(cudaGetLastError(), "chain_stat_ends launch");
    CycStat init{};
    init.bx = -INFINITY;
    init.by = INFINITY;
    init.bi = ~0ull;
    tb = L.tmp_bytes;
    check_cuda(cub::DeviceReduce::Reduce(tmp, tb, part, stat, static_cast<std::int64_t>(2ull * G),
                                         StatCombine{}, init, s),
               "cub::DeviceReduce::Reduce(cycle stat partials)");
  } else {
    chain_copy<<<G, 128, 0, s>>>(loc, L.g, st, cycle);
    check_cuda(cudaGetLastError(), "chain_copy launch");
  }
  static_assert(sizeof(CycStat) <= 64 && sizeof(CycMeta) <= 64, "small_reads slots");
  const SmallRead rd[6] = {{flag, sizeof(int)},
                           {st.offs + (L.g.c_hi - 1), 8},
                           {st.slice + (L.g.c_hi - 1), 8},
                           {stat, sizeof(CycStat)},
                           {meta, sizeof(CycMeta)},
                           {cycle, 16}};
  const unsigned char* hv = small_reads(rd, fused ? 6 : 3, s);
  check_cuda(cudaStreamSynchronize(s), "device chains");
  std::memcpy(&hd.fail, hv, sizeof(int));
  std::memcpy(&hd.last_off, hv + 8, 8);
  std::memcpy(&hd.last_len, hv + 16, 8);
  out->launches = fused ? 8 : 5;
  if (hd.fail) return false;
  const std::uint64_t m = hd.last_off + hd.last_len;
  out->d_cycle = reinterpret_cast<double*>(cycle);
  out->d_scratch = reinterpret_cast<double*>(w + L.o_cycle);
  out->m = m;
  out->chunks = G;
  if (m == 0 || only_q >= 0) return true;  // (one arc: no cycle statistics)
  if (fused) {
    CycStat hs;
    CycMeta mt;
    double2 c0;
    std::memcpy(&hs, hv + 24, sizeof(hs));
    std::memcpy(&mt, hv + 24 + sizeof(CycStat), sizeof(mt));
    std::memcpy(&c0, hv + 24 + sizeof(CycStat) + sizeof(CycMeta), 16);
    // notflat is decided by the first three points when they turn (every
    // non-degenerate cycle); a cycle starting with three collinear points
    // takes the full reduction below
    if (mt.m == m && mt.notflat3) {
      out->front_eq_back = c0.x == mt.tail.x && c0.y == mt.tail.y;
      out->dups = hs.dups != 0;
      out->flat = false;
      out->bad = hs.bad;
      out->best = hs.bi;
      return true;
    }
  }
  cycle_stats_into(cycle, m, stat, tmp, L.tmp_bytes, s, out);
  return true;
}

// finalize_cycle's fast-path statistics of a cycle of m points (m >= 1)
static void cycle_stats_into(const double2* cycle, std::uint64_t m, CycStat* stat, void* tmp,
                             std::size_t tmp_bytes, cudaStream_t s, DeviceCycle* out) {
  std::size_t tb;
  thrust::counting_iterator<std::uint64_t> it(0);
  thrust::transform_iterator<StatOf, thrust::counting_iterator<std::uint64_t>, CycStat> tin(
      it, StatOf{cycle, m});
  CycStat init{};
  init.bx = -INFINITY;
  init.by = INFINITY;
  init.bi = ~0ull;
  tb = tmp_bytes;
  check_cuda(cub::DeviceReduce::Reduce(tmp, tb, tin, stat, static_cast<std::int64_t>(m),
                                       StatCombine{}, init, s),
             "cub::DeviceReduce::Reduce(cycle stats)");
  CycStat hs;
  double2 ends[2];
  static_assert(sizeof(CycStat) <= 64 && sizeof(CycStat) % 8 == 0, "small_reads slots");
  const SmallRead rd[3] = {{stat, sizeof(CycStat)}, {cycle, 16}, {cycle + (m - 1), 16}};
  const unsigned char* hv = small_reads(rd, 3, s);
  check_cuda(cudaStreamSynchronize(s), "cycle stats");
  std::memcpy(&hs, hv, sizeof(hs));
  std::memcpy(&ends[0], hv + sizeof(CycStat), 16);
  std::memcpy(&ends[1], hv + sizeof(CycStat) + 16, 16);
  out->launches += 2;
  out->front_eq_back = ends[0].x == ends[1].x && ends[0].y == ends[1].y;
  out->dups = hs.dups != 0;
  out->flat = hs.notflat == 0;
  out->bad = hs.bad;
  out->best = hs.bi;
}

void device_cycle_stats(const double* d_cycle, std::uint64_t m, const std::uint64_t len[4],
                        void* d_work, cudaStream_t s, DeviceCycle* out) {
  const ChainLayout L = chain_layout(len);
  auto* w = static_cast<unsigned char*>(d_work);
  out->d_cycle = const_cast<double*>(d_cycle);
  out->m = m;
  if (m == 0) return;
  cycle_stats_into(reinterpret_cast<const double2*>(d_cycle), m,
                   reinterpret_cast<CycStat*>(w + L.o_stat), w + L.o_tmp, L.tmp_bytes, s, out);
}

}  // namespace ohx
