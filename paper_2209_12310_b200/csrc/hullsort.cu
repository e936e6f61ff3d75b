// hullsort.cu -- the hull stage's sweep sort on the device (SURVEY §8f
// item 3: "a segmented sort by quadrant key").
//
// The host hull (reference hull.cpp:133-150) sorts each quadrant arc
// [anchor q, queue q..., anchor q+1] by its CCW sweep order, then runs the
// strict-left-turn chain.  For large survivor sets the sort dominates
// (circle 1e8: 4 x 25M points, ~0.85 s each on 16 host cores), so the arcs
// are sorted here, in three tiers (the first that holds):
//   1. a 32-bit key monotone in the primary coordinate (its position in the
//      input's bounding box, square-rooted; see linear_keys), 4 radix
//      passes, the points gathered in key order straight from the packed
//      survivors, runs of equal keys put in the full comparator order;
//   2. the 64-bit primary key (half the radix passes of the full 128-bit
//      key), runs of equal primary key ordered by the secondary key
//      (repair_ties, runs up to 64);
//   3. the full 128-bit (primary, secondary) key.
// One arc can be sorted alone (the pipelined hull stage).  The chains and
// the cycle statistics follow in hullchain.cu.
//
// Keys of tiers 2-3: each coordinate maps to an order-preserving u64
// (negative values bit-complemented, others with the sign bit set); a
// descending component is complemented once more.  -0.0 is folded onto
// +0.0 first, because the reference's comparator treats them as equal
// (a.x != b.x is false).  LSD radix sorts with a u32 payload (the element's
// position), then the points are gathered.  Points equal under the
// comparator may come out in any order -- the reference's std::sort is not
// stable either, and such points only differ in the sign of a zero
// coordinate.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <cub/block/block_merge_sort.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cuda/std/tuple>
#include <cstdlib>
#include <string>

#include "internal.hpp"

namespace ohx {
namespace {

struct SweepKey {
  std::uint64_t hi, lo;
};

struct SweepDecomposer {
  __host__ __device__ ::cuda::std::tuple<std::uint64_t&, std::uint64_t&> operator()(
      SweepKey& k) const {
    return {k.hi, k.lo};
  }
};

__device__ __forceinline__ std::uint64_t asc_key(double v) {
  const std::uint64_t u = static_cast<std::uint64_t>(__double_as_longlong(v == 0.0 ? 0.0 : v));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// Builds arc q = [anchor q, queue q (packed[qoff[q] ...]), anchor q+1] at
// aoff[q] and its sweep keys (reference hull.cpp:18-30):
//   q1 (x desc, y asc), q2 (y desc, x desc), q3 (x asc, y desc), q4 (y asc, x asc)
__global__ void build_arc_keys(const double2* __restrict__ packed, ulonglong4 qoff,
                               ulonglong4 aoff, std::uint64_t total, const double2* anchors,
                               double2* __restrict__ arcs, SweepKey* __restrict__ keys,
                               std::uint32_t* __restrict__ vals) {
  for (std::uint64_t k = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += std::uint64_t(gridDim.x) * blockDim.x) {
    const int q = (k >= aoff.y) + (k >= aoff.z) + (k >= aoff.w);
    const std::uint64_t a0 = q == 0 ? aoff.x : (q == 1 ? aoff.y : (q == 2 ? aoff.z : aoff.w));
    const std::uint64_t a1 = q == 0 ? aoff.y : (q == 1 ? aoff.z : (q == 2 ? aoff.w : total));
    const std::uint64_t p0 = q == 0 ? qoff.x : (q == 1 ? qoff.y : (q == 2 ? qoff.z : qoff.w));
    double2 p;
    if (k == a0) p = anchors[q];
    else if (k == a1 - 1) p = anchors[(q + 1) & 3];
    else p = packed[p0 + (k - a0 - 1)];
    arcs[k] = p;
    if (keys == nullptr) continue;  // the fast path computes its own keys
    const std::uint64_t ax = asc_key(p.x), ay = asc_key(p.y);
    SweepKey key;
    switch (q) {
      case 0: key = {~ax, ay}; break;
      case 1: key = {~ay, ~ax}; break;
      case 2: key = {ax, ~ay}; break;
      default: key = {ay, ax}; break;
    }
    keys[k] = key;
    vals[k] = static_cast<std::uint32_t>(k - a0);
  }
}

// Primary sweep key only (u64), for the fast sort: arc q ascending by
//   q1 ~x, q2 ~y, q3 x, q4 y; ties are repaired afterwards by the secondary
// key (repair_ties).
__device__ __forceinline__ std::uint64_t primary_key(int q, double2 p) {
  switch (q) {
    case 0: return ~asc_key(p.x);
    case 1: return ~asc_key(p.y);
    case 2: return asc_key(p.x);
    default: return asc_key(p.y);
  }
}
__device__ __forceinline__ std::uint64_t secondary_key(int q, double2 p) {
  switch (q) {
    case 0: return asc_key(p.y);
    case 1: return ~asc_key(p.x);
    case 2: return ~asc_key(p.y);
    default: return asc_key(p.x);
  }
}

__global__ void primary_keys(const double2* __restrict__ arcs, ulonglong4 aoff, std::uint64_t total,
                             std::uint64_t* __restrict__ keys, std::uint32_t* __restrict__ vals) {
  for (std::uint64_t k = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += std::uint64_t(gridDim.x) * blockDim.x) {
    const int q = (k >= aoff.y) + (k >= aoff.z) + (k >= aoff.w);
    const std::uint64_t a0 = q == 0 ? aoff.x : (q == 1 ? aoff.y : (q == 2 ? aoff.z : aoff.w));
    keys[k] = primary_key(q, arcs[k]);
    vals[k] = static_cast<std::uint32_t>(k - a0);
  }
}

// Runs of equal primary key (equal coordinate) ordered by the secondary
// key: one thread per run, insertion sort; runs longer than 64 (degenerate
// inputs: many equal coordinates) raise *long_run and the arcs are sorted
// again by the full 128-bit key.
constexpr int kMaxRun = 64;
__global__ void repair_ties(const std::uint64_t* __restrict__ keys, std::uint32_t* vals,
                            const double2* __restrict__ arcs, ulonglong4 aoff, std::uint64_t total,
                            int* long_run) {
  for (std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += std::uint64_t(gridDim.x) * blockDim.x) {
    const int q = (i >= aoff.y) + (i >= aoff.z) + (i >= aoff.w);
    const std::uint64_t a0 = q == 0 ? aoff.x : (q == 1 ? aoff.y : (q == 2 ? aoff.z : aoff.w));
    const std::uint64_t a1 = q == 0 ? aoff.y : (q == 1 ? aoff.z : (q == 2 ? aoff.w : total));
    const std::uint64_t key = keys[i];
    if (i + 1 >= a1 || keys[i + 1] != key || (i > a0 && keys[i - 1] == key)) continue;
    std::uint64_t j = i + 1;
    while (j < a1 && keys[j] == key && j - i <= kMaxRun) ++j;
    if (j - i > kMaxRun) {
      atomicExch(long_run, 1);
      continue;
    }
    for (std::uint64_t k = i + 1; k < j; ++k) {  // insertion sort by the secondary key
      const std::uint32_t v = vals[k];
      const std::uint64_t sk = secondary_key(q, arcs[a0 + v]);
      std::uint64_t m = k;
      while (m > i && secondary_key(q, arcs[a0 + vals[m - 1]]) > sk) {
        vals[m] = vals[m - 1];
        --m;
      }
      vals[m] = v;
    }
  }
}

__global__ void gather_sorted(const double2* __restrict__ arcs, const std::uint32_t* __restrict__ vals,
                              ulonglong4 aoff, std::uint64_t total, double2* __restrict__ out) {
  for (std::uint64_t k = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += std::uint64_t(gridDim.x) * blockDim.x) {
    const int q = (k >= aoff.y) + (k >= aoff.z) + (k >= aoff.w);
    const std::uint64_t a0 = q == 0 ? aoff.x : (q == 1 ? aoff.y : (q == 2 ? aoff.z : aoff.w));
    out[k] = arcs[a0 + vals[k]];
  }
}

// ---- first tier: 32-bit keys linear in the primary coordinate ----------
// The primary coordinate mapped onto 32 bits over the input's bounding box
// (the anchors: east / west / north / south extremes), t =
// sqrt(fl(fl(X - x) / fl(X - W))) * 2^32 truncated: every step is monotone
// (IEEE rounding is), so the key never decreases along the sweep order and
// ties in it only group points; 4 radix passes over (u32, u32) pairs
// instead of 8 over (u64, u32).  Runs of equal keys (equal or nearly equal
// primary coordinates -- a few hundred points where an arc's coordinate is
// stationary, e.g. a circle's tangent points) are then put in the full
// sweep order: up to 32 points by one thread, up to kRunMax by one block
// (cub::BlockMergeSort over the comparator); a longer run sends the call to
// the 64-bit tier below.  This tier reads the arcs' points where they are
// (the packed survivors + the anchors): no materialised copy of the arcs.
constexpr std::uint32_t kRunSmall = 32;
constexpr int kRunThreads = 256, kRunItems = 8;
constexpr std::uint32_t kRunMax = kRunThreads * kRunItems;  // 2048
constexpr std::uint32_t kRunCap = 8192;  // large runs handled per call

// the four arcs [anchor q, packed[qoff[q] ...], anchor q+1] at aoff[q]
struct ArcSrc {
  const double2* packed;
  const double2* anchors;
  ulonglong4 qoff, aoff;
  std::uint64_t total;
  __device__ __forceinline__ int arc_of(std::uint64_t k) const {
    return (k >= aoff.y) + (k >= aoff.z) + (k >= aoff.w);
  }
  __device__ __forceinline__ std::uint64_t begin(int q) const {
    return q == 0 ? aoff.x : (q == 1 ? aoff.y : (q == 2 ? aoff.z : aoff.w));
  }
  __device__ __forceinline__ std::uint64_t end(int q) const {
    return q == 0 ? aoff.y : (q == 1 ? aoff.z : (q == 2 ? aoff.w : total));
  }
  // point j of arc q
  __device__ __forceinline__ double2 point(int q, std::uint64_t j) const {
    const std::uint64_t p0 = q == 0 ? qoff.x : (q == 1 ? qoff.y : (q == 2 ? qoff.z : qoff.w));
    if (j == 0) return anchors[q];
    if (j == end(q) - begin(q) - 1) return anchors[(q + 1) & 3];
    return packed[p0 + j - 1];
  }
};

// (kernels of this tier work on the elements [lo, hi): all four arcs, or one)
__global__ void linear_keys(const ArcSrc A, std::uint32_t* __restrict__ keys,
                            std::uint32_t* __restrict__ vals, std::uint64_t lo, std::uint64_t hi) {
  const double xE = A.anchors[0].x, yN = A.anchors[1].y, xW = A.anchors[2].x, yS = A.anchors[3].y;
  const double sx = __dsub_rn(xE, xW), sy = __dsub_rn(yN, yS);
  for (std::uint64_t k = lo + std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < hi;
       k += std::uint64_t(gridDim.x) * blockDim.x) {
    const int q = A.arc_of(k);
    const std::uint64_t j = k - A.begin(q);
    const double2 p = A.point(q, j);
    double t;
    switch (q) {
      case 0: t = __ddiv_rn(__dsub_rn(xE, p.x), sx); break;  // x descending
      case 1: t = __ddiv_rn(__dsub_rn(yN, p.y), sy); break;  // y descending
      case 2: t = __ddiv_rn(__dsub_rn(p.x, xW), sx); break;  // x ascending
      default: t = __ddiv_rn(__dsub_rn(p.y, yS), sy); break;  // y ascending
    }
    // sqrt: the arc's anchor end is where survivors crowd (an arc leaves
    // its anchor tangent to the anchor's axis: on a circle x = cos(theta),
    // so sqrt(1 - x) is linear in the angle there); correctly rounded,
    // hence monotone like the steps before it
    t = __dmul_rn(__dsqrt_rn(t), 4294967296.0);
    keys[k] = t >= 4294967295.0 ? 0xffffffffu : (t > 0.0 ? static_cast<std::uint32_t>(t) : 0u);
    vals[k] = static_cast<std::uint32_t>(j);
  }
}

__device__ __forceinline__ bool sweep_less(int q, double2 a, double2 b) {  // hull.cpp:18-30
  switch (q) {
    case 0: return a.x != b.x ? a.x > b.x : a.y < b.y;
    case 1: return a.y != b.y ? a.y > b.y : a.x > b.x;
    case 2: return a.x != b.x ? a.x < b.x : a.y > b.y;
    default: return a.y != b.y ? a.y < b.y : a.x < b.x;
  }
}
struct SweepLessOp {
  int q;
  __device__ __forceinline__ bool operator()(const double2& a, const double2& b) const {
    return sweep_less(q, a, b);
  }
};

// Runs of equal keys, fixed on the gathered points (contiguous, in key
// order): short ones sorted here by the comparator, the others listed for
// sort_runs; flag = a run past kRunMax points or more than kRunCap runs.
// Warp-cooperative scan: lane l looks at key w0 + l (coalesced) and its
// neighbours by shuffle; only run starts do any work.
__device__ __forceinline__ void fix_run_at(const std::uint32_t* __restrict__ keys, double2* out,
                                           const ArcSrc& A, std::uint64_t i, std::uint32_t key,
                                           std::uint32_t prev, std::uint32_t next, uint2* runs,
                                           unsigned* nruns, int* flag) {
  if (next != key) return;  // (nearly every element: no arc arithmetic)
  const int q = A.arc_of(i);
  const std::uint64_t a0 = A.begin(q), a1 = A.end(q);
  if (i + 1 >= a1 || (i > a0 && prev == key)) return;  // not a run start
  std::uint64_t j = i + 2;
  while (j < a1 && keys[j] == key && j - i <= kRunMax) ++j;
  const std::uint64_t len = j - i;
  if (len > kRunMax) {
    atomicExch(flag, 1);
    return;
  }
  if (len > kRunSmall) {
    const unsigned r = atomicAdd(nruns, 1u);
    if (r < kRunCap) runs[r] = make_uint2(static_cast<unsigned>(i), static_cast<unsigned>(len));
    else atomicExch(flag, 1);
    return;
  }
  for (std::uint64_t k = i + 1; k < j; ++k) {  // insertion sort by the comparator
    const double2 pv = out[k];
    std::uint64_t m = k;
    while (m > i && sweep_less(q, pv, out[m - 1])) {
      out[m] = out[m - 1];
      --m;
    }
    out[m] = pv;
  }
}

// Warp-cooperative scan: lane l reads keys w0 + 4l .. w0 + 4l + 3 (one
// 16-byte load; keys 16-byte aligned), the neighbours across lanes by
// shuffle; only run starts do any work.
__global__ void fix_runs(const std::uint32_t* __restrict__ keys, double2* out, const ArcSrc A,
                         uint2* runs, unsigned* nruns, int* flag, std::uint64_t lo,
                         std::uint64_t hi) {
  const int lane = threadIdx.x & 31;
  const std::uint64_t nwarps = std::uint64_t(gridDim.x) * (blockDim.x / 32);
  const std::uint64_t n = A.total;
  for (std::uint64_t w0 = lo / 128 * 128 +
                          (std::uint64_t(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5)) * 128;
       w0 < hi; w0 += nwarps * 128) {
    const std::uint64_t i0 = w0 + 4 * lane;
    std::uint32_t k[4];
    if (i0 + 3 < n) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(keys + i0));
      k[0] = v.x;
      k[1] = v.y;
      k[2] = v.z;
      k[3] = v.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) k[e] = i0 + e < n ? keys[i0 + e] : 0u;
    }
    std::uint32_t prev = __shfl_up_sync(0xffffffffu, k[3], 1);
    std::uint32_t next = __shfl_down_sync(0xffffffffu, k[0], 1);
    if (lane == 0 && i0 > 0 && i0 < n) prev = keys[i0 - 1];
    if (lane == 31 && i0 + 4 < n) next = keys[i0 + 4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const std::uint64_t i = i0 + e;
      if (i >= hi) break;
      if (i < lo) continue;
      fix_run_at(keys, out, A, i, k[e], e == 0 ? prev : k[e - 1], e == 3 ? next : k[e + 1], runs,
                 nruns, flag);
    }
  }
}

__global__ void __launch_bounds__(kRunThreads)
    sort_runs(const uint2* __restrict__ runs, const unsigned* __restrict__ nruns, double2* out,
              const ArcSrc A) {
  using Sort = cub::BlockMergeSort<double2, kRunThreads, kRunItems>;
  __shared__ typename Sort::TempStorage tmp;
  if (blockIdx.x >= min(*nruns, kRunCap)) return;
  const uint2 run = runs[blockIdx.x];
  const std::uint64_t i = run.x;
  const int n = static_cast<int>(run.y);
  const int q = A.arc_of(i);
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  double2 pad;  // after every finite point in this quadrant's order
  switch (q) {
    case 0: pad = make_double2(-inf, inf); break;
    case 1: pad = make_double2(-inf, -inf); break;
    case 2: pad = make_double2(inf, -inf); break;
    default: pad = make_double2(inf, inf); break;
  }
  double2 key[kRunItems];
#pragma unroll
  for (int u = 0; u < kRunItems; ++u) {
    const int t = threadIdx.x * kRunItems + u;
    key[u] = t < n ? out[i + t] : pad;
  }
  Sort(tmp).Sort(key, SweepLessOp{q}, n, pad);
#pragma unroll
  for (int u = 0; u < kRunItems; ++u) {
    const int t = threadIdx.x * kRunItems + u;
    if (t < n) out[i + t] = key[u];
  }
}

// The points in key order: random 16-byte reads.  Every read costs ~4 L2
// sectors / ~116 B of DRAM whatever the path (ld default, .cg, .cs,
// .nc.L1::no_allocate, cp.async .cg / .ca: ncu, circle 1e8, 11.6-12.9 GB
// read for 1.6 GB of points); four reads in flight per thread through
// cp.async.ca into the thread's shared-memory slots measured fastest
// (2.37 vs 2.46 ms).  kAsync = false: one plain load at a time (A/B hook
// OHX_GATHER_LD=0).
template <bool kAsync>
__global__ void gather_arcs(const ArcSrc A, const std::uint32_t* __restrict__ vals,
                            double2* __restrict__ out, std::uint64_t lo, std::uint64_t hi) {
  auto src_of = [&](std::uint64_t k) -> const double2* {
    const int q = A.arc_of(k);
    const std::uint64_t j = vals[k];
    if (j == 0) return A.anchors + q;
    if (j == A.end(q) - A.begin(q) - 1) return A.anchors + ((q + 1) & 3);
    const std::uint64_t p0 =
        q == 0 ? A.qoff.x : (q == 1 ? A.qoff.y : (q == 2 ? A.qoff.z : A.qoff.w));
    return A.packed + p0 + j - 1;
  };
  const std::uint64_t stride = std::uint64_t(gridDim.x) * blockDim.x;
  const std::uint64_t first = lo + std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if constexpr (kAsync) {
    __shared__ double2 slot[4][256];
    for (std::uint64_t k0 = first; k0 < hi; k0 += 4 * stride) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const std::uint64_t k = k0 + u * stride;
        if (k >= hi) break;
        const unsigned dst =
            static_cast<unsigned>(__cvta_generic_to_shared(&slot[u][threadIdx.x]));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src_of(k)));
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const std::uint64_t k = k0 + u * stride;
        if (k < hi) out[k] = slot[u][threadIdx.x];
      }
    }
  } else {
    for (std::uint64_t k = first; k < hi; k += stride) out[k] = *src_of(k);
  }
}

bool gather_async() {
  static const bool v = [] {
    const char* e = std::getenv("OHX_GATHER_LD");
    return !(e && std::string(e) == "0");
  }();
  return v;
}

struct ArcLayout {
  std::uint64_t total;
  ulonglong4 qoff, aoff;
  std::uint64_t len[4];
};

ArcLayout arc_layout(const std::uint64_t counts[4]) {
  ArcLayout L{};
  std::uint64_t q = 0, a = 0;
  std::uint64_t qo[4], ao[4];
  for (int k = 0; k < 4; ++k) {
    qo[k] = q;
    ao[k] = a;
    L.len[k] = counts[k] + 2;
    q += counts[k];
    a += L.len[k];
  }
  L.total = a;
  L.qoff = make_ulonglong4(qo[0], qo[1], qo[2], qo[3]);
  L.aoff = make_ulonglong4(ao[0], ao[1], ao[2], ao[3]);
  return L;
}

std::size_t cub_tmp_bytes(std::uint64_t max_len) {  // for either sort
  std::size_t b128 = 0, b64 = 0;
  cub::DoubleBuffer<SweepKey> kb(nullptr, nullptr);
  cub::DoubleBuffer<std::uint64_t> kb64(nullptr, nullptr);
  cub::DoubleBuffer<std::uint32_t> vb(nullptr, nullptr);
  check_cuda(cub::DeviceRadixSort::SortPairs(nullptr, b128, kb, vb,
                                             static_cast<std::int64_t>(max_len),
                                             SweepDecomposer{}),
             "cub temp size");
  check_cuda(cub::DeviceRadixSort::SortPairs(nullptr, b64, kb64, vb,
                                             static_cast<std::int64_t>(max_len)),
             "cub temp size");
  return b128 > b64 ? b128 : b64;
}

std::size_t align256(std::size_t b) { return (b + 255) & ~std::size_t(255); }

// OHX_HULL_SORT=u64: skip the 32-bit linear-key tier (A/B and test hook)
bool linear_tier() {
  static const bool v = [] {
    const char* e = std::getenv("OHX_HULL_SORT");
    return !(e && std::string(e) == "u64");
  }();
  return v;
}

}  // namespace

std::size_t sort_arcs_work_bytes(const std::uint64_t counts[4]) {
  const ArcLayout L = arc_layout(counts);
  std::uint64_t mx = 0;
  for (std::uint64_t l : L.len) mx = l > mx ? l : mx;
  // arcs (16) + 2 x keys (32) + 2 x vals (8) per element, anchors, cub temp
  return align256(L.total * 16) + 2 * align256(L.total * 16) + 2 * align256(L.total * 4) + 256 +
         align256(cub_tmp_bytes(mx));
}

void sort_arcs(const double* d_packed, const std::uint64_t counts[4], const double anchors[8],
               void* d_work, double* d_sorted, cudaStream_t s, int only_q) {
  const ArcLayout L = arc_layout(counts);
  if (L.total >= (1ull << 32)) throw Error(OHX_E_INVALID, "sort_arcs: > 2^32 survivors");
  std::uint64_t mx = 0;
  for (std::uint64_t l : L.len) mx = l > mx ? l : mx;
  auto* b = static_cast<unsigned char*>(d_work);
  auto take = [&](std::size_t bytes) {
    unsigned char* p = b;
    b += align256(bytes);
    return p;
  };
  auto* arcs = reinterpret_cast<double2*>(take(L.total * 16));
  auto* k0 = reinterpret_cast<SweepKey*>(take(L.total * 16));
  auto* k1 = reinterpret_cast<SweepKey*>(take(L.total * 16));
  auto* v0 = reinterpret_cast<std::uint32_t*>(take(L.total * 4));
  auto* v1 = reinterpret_cast<std::uint32_t*>(take(L.total * 4));
  auto* d_anchors = reinterpret_cast<double2*>(take(256));
  const std::size_t tmp_bytes = cub_tmp_bytes(mx);
  void* tmp = take(tmp_bytes);
  check_cuda(cudaMemcpyAsync(d_anchors, anchors, 64, cudaMemcpyHostToDevice, s),
             "cudaMemcpyAsync(anchors)");
  const unsigned grid = static_cast<unsigned>(L.total < 148ull * 2048 ? (L.total + 255) / 256 : 148 * 8);
  const std::uint64_t ao[4] = {L.aoff.x, L.aoff.y, L.aoff.z, L.aoff.w};
  int* d_flag = reinterpret_cast<int*>(d_anchors + 8);  // 4 bytes after the 4 anchors
  // first tier: 32-bit linear keys (needs a bounding box of positive extent)
  if (linear_tier() && anchors[0] > anchors[4] && anchors[3] > anchors[7]) {
    auto* q0 = reinterpret_cast<std::uint32_t*>(k1);
    auto* q1 = q0 + (L.total + 3) / 4 * 4;  // 16-byte aligned (fix_runs' vector loads)
    auto* runs = reinterpret_cast<uint2*>(k0);
    auto* nruns = reinterpret_cast<unsigned*>(d_flag + 1);
    const ArcSrc A{reinterpret_cast<const double2*>(d_packed), d_anchors, L.qoff, L.aoff, L.total};
    // one arc (only_q) or all four
    const std::uint64_t lo = only_q >= 0 ? ao[only_q] : 0;
    const std::uint64_t hi = only_q >= 0 ? lo + L.len[only_q] : L.total;
    const unsigned g1 = static_cast<unsigned>(
        hi - lo < 148ull * 2048 ? (hi - lo + 255) / 256 : 148 * 8);
    linear_keys<<<g1, 256, 0, s>>>(A, q0, v1, lo, hi);
    check_cuda(cudaGetLastError(), "linear_keys launch");
    int lsel[4] = {0, 0, 0, 0};
    for (int q = 0; q < 4; ++q) {
      if (only_q >= 0 && q != only_q) continue;
      cub::DoubleBuffer<std::uint32_t> kb(q0 + ao[q], q1 + ao[q]);
      cub::DoubleBuffer<std::uint32_t> vb(v1 + ao[q], v0 + ao[q]);
      std::size_t tb = tmp_bytes;
      check_cuda(cub::DeviceRadixSort::SortPairs(tmp, tb, kb, vb,
                                                 static_cast<std::int64_t>(L.len[q]), 0, 32, s),
                 "cub::DeviceRadixSort::SortPairs(u32)");
      lsel[q] = kb.selector;
    }
    const int q_ref = only_q >= 0 ? only_q : 0;
    std::uint32_t* lkeys = lsel[q_ref] ? q1 : q0;
    std::uint32_t* lvals = lsel[q_ref] ? v0 : v1;
    for (int q = 1; q < 4 && only_q < 0; ++q)
      if (lsel[q] != lsel[0]) {
        check_cuda(cudaMemcpyAsync(lkeys + ao[q], (lsel[q] ? q1 : q0) + ao[q], L.len[q] * 4,
                                   cudaMemcpyDeviceToDevice, s), "cudaMemcpyAsync(sorted keys)");
        check_cuda(cudaMemcpyAsync(lvals + ao[q], (lsel[q] ? v0 : v1) + ao[q], L.len[q] * 4,
                                   cudaMemcpyDeviceToDevice, s), "cudaMemcpyAsync(sorted positions)");
      }
    // the points in key order, then the runs of equal keys in full order
    auto* out = reinterpret_cast<double2*>(d_sorted);
    if (gather_async()) gather_arcs<true><<<g1, 256, 0, s>>>(A, lvals, out, lo, hi);
    else gather_arcs<false><<<g1, 256, 0, s>>>(A, lvals, out, lo, hi);
    check_cuda(cudaGetLastError(), "gather_arcs launch");
    check_cuda(cudaMemsetAsync(d_flag, 0, 2 * sizeof(int), s), "cudaMemsetAsync(flag)");
    fix_runs<<<g1, 256, 0, s>>>(lkeys, out, A, runs, nruns, d_flag, lo, hi);
    check_cuda(cudaGetLastError(), "fix_runs launch");
    sort_runs<<<kRunCap, kRunThreads, 0, s>>>(runs, nruns, out, A);
    check_cuda(cudaGetLastError(), "sort_runs launch");
    int too_long = 0;
    const SmallRead rd{d_flag, sizeof(int)};
    const unsigned char* hv = small_reads(&rd, 1, s);
    check_cuda(cudaStreamSynchronize(s), "hull sort runs");
    std::memcpy(&too_long, hv, sizeof(int));
    if (!too_long) return;
  }
  // the arcs materialised for the tiers below
  build_arc_keys<<<grid, 256, 0, s>>>(reinterpret_cast<const double2*>(d_packed), L.qoff, L.aoff,
                                      L.total, d_anchors, arcs, nullptr, nullptr);
  check_cuda(cudaGetLastError(), "build_arc_keys launch");
  // second tier: 64-bit primary keys (half the passes of the full key), ties repaired
  auto* p0 = reinterpret_cast<std::uint64_t*>(k1);  // k1 is free until the fallback
  auto* p1 = p0 + L.total;
  primary_keys<<<grid, 256, 0, s>>>(arcs, L.aoff, L.total, p0, v1);
  check_cuda(cudaGetLastError(), "primary_keys launch");
  int sel[4];
  for (int q = 0; q < 4; ++q) {
    cub::DoubleBuffer<std::uint64_t> kb(p0 + ao[q], p1 + ao[q]);
    cub::DoubleBuffer<std::uint32_t> vb(v1 + ao[q], v0 + ao[q]);
    std::size_t tb = tmp_bytes;
    check_cuda(cub::DeviceRadixSort::SortPairs(tmp, tb, kb, vb, static_cast<std::int64_t>(L.len[q]),
                                               0, 64, s),
               "cub::DeviceRadixSort::SortPairs(u64)");
    sel[q] = kb.selector;
  }
  // bring every arc's sorted keys / positions into the same pair of buffers
  std::uint64_t* keys = sel[0] ? p1 : p0;
  std::uint32_t* vals = sel[0] ? v0 : v1;
  for (int q = 1; q < 4; ++q)
    if (sel[q] != sel[0]) {
      check_cuda(cudaMemcpyAsync(keys + ao[q], (sel[q] ? p1 : p0) + ao[q], L.len[q] * 8,
                                 cudaMemcpyDeviceToDevice, s), "cudaMemcpyAsync(sorted keys)");
      check_cuda(cudaMemcpyAsync(vals + ao[q], (sel[q] ? v0 : v1) + ao[q], L.len[q] * 4,
                                 cudaMemcpyDeviceToDevice, s), "cudaMemcpyAsync(sorted positions)");
    }
  check_cuda(cudaMemsetAsync(d_flag, 0, sizeof(int), s), "cudaMemsetAsync(flag)");
  repair_ties<<<grid, 256, 0, s>>>(keys, vals, arcs, L.aoff, L.total, d_flag);
  check_cuda(cudaGetLastError(), "repair_ties launch");
  int long_run = 0;
  const SmallRead rd{d_flag, sizeof(int)};
  const unsigned char* hv = small_reads(&rd, 1, s);
  check_cuda(cudaStreamSynchronize(s), "hull sort ties");
  std::memcpy(&long_run, hv, sizeof(int));
  if (long_run) {  // degenerate arcs: the full 128-bit key sort
    build_arc_keys<<<grid, 256, 0, s>>>(reinterpret_cast<const double2*>(d_packed), L.qoff,
                                        L.aoff, L.total, d_anchors, arcs, k0, v0);
    check_cuda(cudaGetLastError(), "build_arc_keys launch");
    for (int q = 0; q < 4; ++q) {
      cub::DoubleBuffer<SweepKey> kb(k0 + ao[q], k1 + ao[q]);
      cub::DoubleBuffer<std::uint32_t> vb(v0 + ao[q], v1 + ao[q]);
      std::size_t tb = tmp_bytes;
      check_cuda(cub::DeviceRadixSort::SortPairs(tmp, tb, kb, vb,
                                                 static_cast<std::int64_t>(L.len[q]),
                                                 SweepDecomposer{}, 0, 128, s),
                 "cub::DeviceRadixSort::SortPairs");
      sel[q] = vb.selector;
    }
    vals = sel[0] ? v1 : v0;
    for (int q = 1; q < 4; ++q)
      if (sel[q] != sel[0])
        check_cuda(cudaMemcpyAsync(vals + ao[q], (sel[q] ? v1 : v0) + ao[q], L.len[q] * 4,
                                   cudaMemcpyDeviceToDevice, s),
                   "cudaMemcpyAsync(sorted positions)");
  }
  gather_sorted<<<grid, 256, 0, s>>>(arcs, vals, L.aoff, L.total,
                                     reinterpret_cast<double2*>(d_sorted));
  check_cuda(cudaGetLastError(), "gather_sorted launch");
}

}  // namespace ohx
