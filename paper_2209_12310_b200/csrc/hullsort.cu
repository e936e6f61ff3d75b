// hullsort.cu -- the hull stage's sweep sort on the device (SURVEY §8f
// item 3: "a segmented sort by quadrant key").
//
// The host hull (reference hull.cpp:133-150) sorts each quadrant arc
// [anchor q, queue q..., anchor q+1] by its CCW sweep order, then runs the
// strict-left-turn chain.  For large survivor sets the sort dominates
// (circle 1e8: 4 x 25M points, ~0.85 s each on 16 host cores), so the arcs
// are built and sorted here and come back to the host already in sweep
// order; the chain and the cycle clean-up stay on the host (their
// decisions are the reference's predicate sequence).  The sort runs on the
// 64-bit primary key (half the radix passes of the full 128-bit key); runs
// of equal primary key are then ordered by the secondary key (repair_ties),
// and arcs with runs longer than 64 fall back to the 128-bit sort.
//
// Keys: each coordinate maps to an order-preserving u64 (negative values
// bit-complemented, others with the sign bit set); a descending component
// is complemented once more.  -0.0 is folded onto +0.0 first, because the
// reference's comparator treats them as equal (a.x != b.x is false).  The
// sort is an LSD radix sort over the 128-bit (primary, secondary) key with a
// u32 payload (the element's position), then the points are gathered.
// Points equal under the comparator may come out in any order -- the
// reference's std::sort is not stable either, and such points only differ
// in the sign of a zero coordinate.
#include <cuda_runtime.h>

#include <cstdint>
#include <cub/device/device_radix_sort.cuh>
#include <cuda/std/tuple>

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
               void* d_work, double* d_sorted, cudaStream_t s) {
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
  build_arc_keys<<<grid, 256, 0, s>>>(reinterpret_cast<const double2*>(d_packed), L.qoff, L.aoff,
                                      L.total, d_anchors, arcs, nullptr, nullptr);
  check_cuda(cudaGetLastError(), "build_arc_keys launch");
  const std::uint64_t ao[4] = {L.aoff.x, L.aoff.y, L.aoff.z, L.aoff.w};
  // fast path: 64-bit primary keys (half the radix passes), ties repaired
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
  int* d_flag = reinterpret_cast<int*>(d_anchors + 8);  // 4 bytes after the 4 anchors
  check_cuda(cudaMemsetAsync(d_flag, 0, sizeof(int), s), "cudaMemsetAsync(flag)");
  repair_ties<<<grid, 256, 0, s>>>(keys, vals, arcs, L.aoff, L.total, d_flag);
  check_cuda(cudaGetLastError(), "repair_ties launch");
  int long_run = 0;
  check_cuda(cudaMemcpyAsync(&long_run, d_flag, sizeof(int), cudaMemcpyDeviceToHost, s),
             "cudaMemcpyAsync(flag)");
  check_cuda(cudaStreamSynchronize(s), "hull sort ties");
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
