// kernels.cu -- the sm_100a kernels of the heaphull filter.
//
//   K1  k1_extremes    one streaming pass: 4 axis argmax/argmin + 4 diagonal
//                      argmax with second-best keys (corner certificate).
//                      Replaces the 8 passes of find_axis_extremes and
//                      find_corner_extremes (reference filter.cpp:8-45).
//   K1b k1b_corners    exact Manhattan corner argmins (filter.cpp:25-45),
//                      run only when the certificate fails.
//   K2  k2_filter      octagon classify (filter.cpp:104-131, geometry.cpp:8-25,
//                      filter.cpp:88-102) fused with the ordered per-quadrant
//                      compaction of build_queues (hull.cpp:124-131):
//                      warp ballot/popc, block scan, decoupled look-back.
//   gather_xy          survivor coordinates for a queue (index order).
//
// All arithmetic on point data reproduces the reference's binary64
// operations exactly: explicit __dadd_rn/__dsub_rn/__dmul_rn (no FMA
// contraction; the TU is also built with -fmad=false).
//
// HBM is the roofline: every kernel streams AoS double2 points with 16-byte
// non-allocating loads, several loads in flight per thread, grids sized from
// the SM count and the occupancy of the kernel.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "internal.hpp"

namespace ohx {
namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}

__device__ __forceinline__ std::uint64_t ld_relaxed(const std::uint64_t* p) {
  std::uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed(std::uint64_t* p, std::uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}


// ---- TMA bulk copies (cp.async.bulk) + mbarrier, for the streaming kernels
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// one arrival that also announces `bytes` of incoming async-proxy writes
__device__ __forceinline__ void mbar_arrive_expect(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

// ===================================================================== K1 ==
// Every slot is an argmax of a maximised key; ties keep the smaller index
// (combine_max / combine_min, reference parallel.hpp:34-43; argmin of a key
// is argmax of its exact negation).  Within a thread indices only grow, so
// a strict '>' keeps the earliest index.

template <int NK, int NS, typename I = std::uint64_t>
struct ArgState {
  double k[NK];
  I i[NK];
  double s[NS > 0 ? NS : 1];

  __device__ __forceinline__ void init() {
#pragma unroll
    for (int a = 0; a < NK; ++a) {
      k[a] = __longlong_as_double(0xfff0000000000000ll);  // -inf
      i[a] = ~I(0);
    }
#pragma unroll
    for (int a = 0; a < (NS > 0 ? NS : 1); ++a) s[a] = __longlong_as_double(0xfff0000000000000ll);
  }
};

// in-thread update: strict improvement only
template <typename I>
__device__ __forceinline__ void upd(double& bk, I& bi, double key, I j) {
  const bool take = key > bk;
  bk = take ? key : bk;
  bi = take ? j : bi;
}

// in-thread update tracking the second-largest key of the multiset
template <typename I>
__device__ __forceinline__ void upd2(double& bk, I& bi, double& s2, double key, I j) {
  const bool take = key > bk;
  const double lo = take ? bk : key;  // the value that does not become best
  s2 = lo > s2 ? lo : s2;
  bk = take ? key : bk;
  bi = take ? j : bi;
}

// cross-thread merge of (ak,ai) with (bk,bi): argmax, ties -> smaller index
template <typename I>
__device__ __forceinline__ void merge(double& ak, I& ai, double bk, I bi) {
  const bool take = bk > ak || (bk == ak && bi < ai);
  ak = take ? bk : ak;
  ai = take ? bi : ai;
}

template <typename I>
__device__ __forceinline__ void merge2(double& ak, I& ai, double& as, double bk, I bi,
                                       double bs) {
  // second of the union = max(both seconds, the smaller of the two bests)
  const double lo = ak < bk ? ak : bk;
  double s = as > bs ? as : bs;
  s = lo > s ? lo : s;
  as = s;
  merge(ak, ai, bk, bi);
}

template <int NK, int NS>
__device__ __forceinline__ void warp_reduce(ArgState<NK, NS>& st) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int a = 0; a < NK; ++a) {
      const double ok = __shfl_xor_sync(kFull, st.k[a], off);
      const std::uint64_t oi = __shfl_xor_sync(kFull, st.i[a], off);
      if (a >= NK - NS) {
        const double os = __shfl_xor_sync(kFull, st.s[a - (NK - NS)], off);
        merge2(st.k[a], st.i[a], st.s[a - (NK - NS)], ok, oi, os);
      } else {
        merge(st.k[a], st.i[a], ok, oi);
      }
    }
  }
}

// Block-wide reduction; the result is valid in warp 0.  kUniform: every
// warp's lanes already hold one identical (warp-reduced) state -- reducing
// those copies again would count each diagonal winner twice in its
// second-best key.
template <int NK, int NS, int BLOCK, bool kUniform = false>
__device__ __forceinline__ void block_reduce(ArgState<NK, NS>& st) {
  constexpr int W = BLOCK / 32;
  __shared__ double sk[W][NK];
  __shared__ std::uint64_t si[W][NK];
  __shared__ double ss[W][NS > 0 ? NS : 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (!kUniform) warp_reduce(st);
  __syncthreads();  // smem may be reused by a previous call
  if (lane == 0) {
#pragma unroll
    for (int a = 0; a < NK; ++a) {
      sk[warp][a] = st.k[a];
      si[warp][a] = st.i[a];
    }
#pragma unroll
    for (int a = 0; a < NS; ++a) ss[warp][a] = st.s[a];
  }
  __syncthreads();
  if (warp == 0) {
    st.init();
    if (lane < W) {
#pragma unroll
      for (int a = 0; a < NK; ++a) {
        st.k[a] = sk[lane][a];
        st.i[a] = si[lane][a];
      }
#pragma unroll
      for (int a = 0; a < NS; ++a) st.s[a] = ss[lane][a];
    }
    warp_reduce(st);
  }
}

// Final grid combine: the last block to finish (atomic ticket) merges all
// per-block partials.  Returns true in the block that holds the result
// (valid in warp 0).
template <int NK, int NS, int BLOCK>
__device__ __forceinline__ bool grid_combine(ArgState<NK, NS>& st,
                                             K1Partial* partials,
                                             unsigned* ticket) {
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
    K1Partial& p = partials[blockIdx.x];
#pragma unroll
    for (int a = 0; a < NK; ++a) {
      p.key[a] = st.k[a];
      p.idx[a] = st.i[a];
    }
#pragma unroll
    for (int a = 0; a < NS; ++a) p.second[a] = st.s[a];
    __threadfence();
    s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  st.init();
  for (unsigned b = threadIdx.x; b < gridDim.x; b += BLOCK) {
    const K1Partial* p = partials + b;
#pragma unroll
    for (int a = 0; a < NK; ++a) {
      const double k = __ldcg(&p->key[a]);
      const std::uint64_t i = __ldcg(reinterpret_cast<const unsigned long long*>(&p->idx[a]));
      if (a >= NK - NS) {
        merge2(st.k[a], st.i[a], st.s[a - (NK - NS)], k, i,
               __ldcg(&p->second[a - (NK - NS)]));
      } else {
        merge(st.k[a], st.i[a], k, i);
      }
    }
  }
  block_reduce<NK, NS, BLOCK>(st);
  if (threadIdx.x == 0) *ticket = 0u;  // re-arm for the next launch
  return true;
}

constexpr int kK1Block = 256;
constexpr int kK1Unroll = 8;
constexpr int kK1MinBlocks = 3;

// widen a streaming-phase state (32- or 64-bit indices) for the reductions
template <int NK, int NS, typename I>
__device__ __forceinline__ ArgState<NK, NS> widen(const ArgState<NK, NS, I>& t) {
  ArgState<NK, NS> st;
#pragma unroll
  for (int a = 0; a < NK; ++a) {
    st.k[a] = t.k[a];
    st.i[a] = t.i[a] == ~I(0) ? ~0ull : static_cast<std::uint64_t>(t.i[a]);
  }
#pragma unroll
  for (int a = 0; a < (NS > 0 ? NS : 1); ++a) st.s[a] = t.s[a];
  return st;
}

// Slots (ohx.h): 0 east x, 1 north y, 2 west -x, 3 south -y,
//                4 ne fl(x+y), 5 nw fl(y-x), 6 sw -fl(x+y), 7 se fl(x-y);
// slots 4..7 also keep their second-best key.
//
// The state is warp-uniform: all 32 lanes hold the warp's best (and second)
// of every slot.  Fast path: a point can change the state only if one of its
// keys beats the warp's best (axis slots) or second (diagonal slots), which
// after a warp has seen m points happens with probability ~1/m per key; the
// common path is therefore 2 DADD + 8 DSETP + one vote per point.  On a hit
// the slots that some lane improves are reduced across the warp (argmax
// with ties to the smaller index; multiset top-2 for the diagonals) and
// merged.  A per-lane state would take its divergent update path 32x more
// often (every lane's own record breaks stall the whole warp).
// The warp-uniform extremes state, one per warp in shared memory (only the
// eight thresholds live in registers).
struct WarpExt {
  double k[8];
  double s[4];
  std::uint64_t i[8];
};

struct K1Visit {
  template <typename I>
  __device__ __forceinline__ static void reduce1(double& bk, I& bi, double key, I j) {
    double k = key;
    I i = j;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ok = __shfl_xor_sync(kFull, k, off);
      const I oi = __shfl_xor_sync(kFull, i, off);
      merge(k, i, ok, oi);
    }
    merge(bk, bi, k, i);
  }
  template <typename I>
  __device__ __forceinline__ static void reduce2(double& bk, I& bi, double& bs, double key, I j) {
    double k = key, s2 = __longlong_as_double(0xfff0000000000000ll);
    I i = j;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ok = __shfl_xor_sync(kFull, k, off);
      const I oi = __shfl_xor_sync(kFull, i, off);
      const double os = __shfl_xor_sync(kFull, s2, off);
      merge2(k, i, s2, ok, oi, os);
    }
    merge2(bk, bi, bs, k, i, s2);
  }
  // Can point p change the warp's state?  th[a] is the value a key must beat:
  // the best for the axis slots, the second for the diagonal ones.
  __device__ __forceinline__ static bool hits(const double (&th)[8], double2 p) {
    const double t = __dadd_rn(p.x, p.y);
    const double d = __dsub_rn(p.x, p.y);
    return (p.x > th[0]) | (p.y > th[1]) | (-p.x > th[2]) | (-p.y > th[3]) | (t > th[4]) |
           (-d > th[5]) | (-t > th[6]) | (d > th[7]);
  }
  // Called by all 32 lanes of the warp; `valid` lanes contribute point j.
  __device__ __forceinline__ static void update(WarpExt& w, double (&th)[8], double2 p,
                                                std::uint64_t j, bool valid) {
    const int lane = threadIdx.x & 31;
    const double t = __dadd_rn(p.x, p.y);
    const double d = __dsub_rn(p.x, p.y);
    double key[8] = {p.x, p.y, -p.x, -p.y, t, -d, -t, d};
    if (!valid) {
#pragma unroll
      for (int a = 0; a < 8; ++a) key[a] = __longlong_as_double(0xfff0000000000000ll);
    }
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      if (!__any_sync(kFull, key[a] > th[a])) continue;
      double bk = w.k[a];
      std::uint64_t bi = w.i[a];
      if (a < 4) {
        reduce1(bk, bi, key[a], j);
        th[a] = bk;
      } else {
        double bs = w.s[a - 4];
        reduce2(bk, bi, bs, key[a], j);
        th[a] = bs;
        __syncwarp();
        if (lane == 0) w.s[a - 4] = bs;
      }
      __syncwarp();
      if (lane == 0) {
        w.k[a] = bk;
        w.i[a] = bi;
      }
      __syncwarp();
    }
  }
};

__device__ __forceinline__ void warp_ext_init(WarpExt& w, double (&th)[8]) {
  const double ninf = __longlong_as_double(0xfff0000000000000ll);
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      w.k[a] = ninf;
      w.i[a] = ~0ull;
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) w.s[a] = ninf;
  }
#pragma unroll
  for (int a = 0; a < 8; ++a) th[a] = ninf;
  __syncwarp();
}

__device__ __forceinline__ ArgState<8, 4> warp_ext_state(const WarpExt& w) {
  ArgState<8, 4> st;
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    st.k[a] = w.k[a];
    st.i[a] = w.i[a];
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) st.s[a] = w.s[a];
  return st;
}

// Visit the 8 points v[u] (index j0 + u * step) of every lane of a warp.
// Fast path: no lane's point can change the state -> one vote for all 8.
// Otherwise the points go through a per-warp shared-memory stage so that the
// update path is instantiated once (a rolled loop), not per item.
template <bool all_valid, typename I>
__device__ __forceinline__ void visit8(WarpExt& w, double (&th)[8], const double2 (&v)[8], I j0,
                                       I step, std::uint64_t n, double2* stage) {
  bool any = false;
#pragma unroll
  for (int u = 0; u < 8; ++u)
    any |= (all_valid || std::uint64_t(j0) + u * std::uint64_t(step) < n) && K1Visit::hits(th, v[u]);
  if (!__any_sync(kFull, any)) return;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int u = 0; u < 8; ++u) stage[u * 32 + lane] = v[u];
  __syncwarp();
#pragma unroll 1
  for (int u = 0; u < 8; ++u) {
    const std::uint64_t j = std::uint64_t(j0) + std::uint64_t(u) * std::uint64_t(step);
    K1Visit::update(w, th, stage[u * 32 + lane], j, all_valid || j < n);
  }
  __syncwarp();
}

template <typename IdxT>
__global__ void __launch_bounds__(kK1Block, kK1MinBlocks)
    k1_extremes(const double2* __restrict__ pts, std::uint64_t n,
                std::uint64_t base, K1Partial* partials, unsigned* ticket,
                ohx_extremes_rec* out) {
  static_assert(kK1Unroll == 8, "visit8 takes 8 points per lane");
  __shared__ double2 k1_stage[kK1Block / 32][8 * 32];
  __shared__ WarpExt k1_ext[kK1Block / 32];
  WarpExt& we = k1_ext[threadIdx.x >> 5];
  double th[8];
  warp_ext_init(we, th);
  // each block streams one contiguous range of 2048-point chunks (32 KB of
  // consecutive addresses per block step, 8 loads in flight per thread)
  constexpr std::uint64_t kChunk = std::uint64_t(kK1Block) * kK1Unroll;
  const std::uint64_t nchunks = (n + kChunk - 1) / kChunk;
  const std::uint64_t per = (nchunks + gridDim.x - 1) / gridDim.x;
  const std::uint64_t c_end = min(nchunks, (blockIdx.x + 1) * per);
  for (std::uint64_t c = blockIdx.x * per; c < c_end; ++c) {
    const IdxT j0 = static_cast<IdxT>(c * kChunk + threadIdx.x);
    if ((c + 1) * kChunk <= n) {
      double2 v[kK1Unroll];
#pragma unroll
      for (int u = 0; u < kK1Unroll; ++u) v[u] = ld_stream(pts + j0 + u * kK1Block);
      visit8<true>(we, th, v, j0, IdxT(kK1Block), n, k1_stage[threadIdx.x >> 5]);
    } else {
      double2 v[kK1Unroll];
#pragma unroll
      for (int u = 0; u < kK1Unroll; ++u)
        v[u] = std::uint64_t(j0) + u * kK1Block < n ? ld_stream(pts + j0 + u * kK1Block)
                                                    : make_double2(0.0, 0.0);
      visit8<false>(we, th, v, j0, IdxT(kK1Block), n, k1_stage[threadIdx.x >> 5]);
    }
  }

  __syncwarp();
  ArgState<8, 4> st = warp_ext_state(we);
  block_reduce<8, 4, kK1Block, true>(st);
  if (!grid_combine<8, 4, kK1Block>(st, partials, ticket)) return;
  if (threadIdx.x < 8) {
    // lane a of warp 0 publishes slot a with its winner's coordinates
    const int a = threadIdx.x;
    double k = 0, s = 0;
    std::uint64_t i = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b)
      if (b == a) {
        k = st.k[b];
        i = st.i[b];
        if (b >= 4) s = st.s[b - 4];
      }
    const double2 p = pts[i];
    out->key[a] = k;
    out->idx[a] = base + i;
    out->x[a] = p.x;
    out->y[a] = p.y;
    if (a >= 4) out->second[a - 4] = s;
    if (a == 0) out->n = n;
  }
}

// ============================================================ K1 (small) ==
// K1 for small inputs -- the provisional region's sample and the fused
// pass's candidate list.  With few points per warp nearly every point would
// take the warp-uniform update path of k1_extremes, so here every thread
// keeps its own state (register compare-and-select per point) and the
// states are reduced once per warp / block / grid.  blockIdx.y selects an
// independent input (a sub-sample), each with its own partials, ticket and
// record.
//   sampled: input g is the sample runs b = s * subs + g (s = 0..segs/subs-1)
//            of `len` consecutive points starting at (n - len) * b /
//            (segs - 1); reported indices are global.
//   list:    input 0 is pts[0, n).
// list mode: the published indices are map[i] + base (the fused pass's
// candidate list maps gathered positions back to point indices)
struct ListMap {
  const void* idx;
  int bytes;  // 4 or 8
  std::uint64_t base;
};
struct SampleMap {
  std::uint64_t n;
  int segs, len, subs;
  __device__ __forceinline__ std::uint64_t run_start(std::uint64_t b) const {
    return (n - std::uint64_t(len)) * b / std::uint64_t(segs > 1 ? segs - 1 : 1);
  }
};

template <typename LI>
__device__ __forceinline__ void k1_visit(ArgState<8, 4, LI>& st, double2 p, LI j) {
  const double t = __dadd_rn(p.x, p.y);
  const double d = __dsub_rn(p.x, p.y);
  upd(st.k[0], st.i[0], p.x, j);
  upd(st.k[1], st.i[1], p.y, j);
  upd(st.k[2], st.i[2], -p.x, j);
  upd(st.k[3], st.i[3], -p.y, j);
  upd2(st.k[4], st.i[4], st.s[0], t, j);
  upd2(st.k[5], st.i[5], st.s[1], -d, j);
  upd2(st.k[6], st.i[6], st.s[2], -t, j);
  upd2(st.k[7], st.i[7], st.s[3], d, j);
}

// List mode: threads track 32-bit indices whenever the list fits (one
// select per slot update instead of two), widened before the block / grid
// reduction.
template <bool kSampled, typename LI>
__global__ void __launch_bounds__(256)
    k1_small(const double2* __restrict__ pts, std::uint64_t n, const unsigned long long* d_n,
             const SampleMap sm, const ListMap lm, K1Partial* partials, unsigned* ticket,
             ohx_extremes_rec* out, unsigned long long* zero = nullptr) {
  // (sample mode: zero the coverage counter count_in_region adds to next)
  if (zero != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *zero = 0;
  if (d_n != nullptr && *d_n < n) n = *d_n;  // list length counted on the device
  const int g = blockIdx.y;
  partials += std::uint64_t(g) * gridDim.x;
  ticket += g;
  out += g;
  ArgState<8, 4, LI> lst;
  lst.init();
  if constexpr (kSampled) {
    // global indices (LI = u64: a 32-bit run-local index measured slower
    // here) only grow along a thread's runs (run b increases with r); 8
    // loads in flight per thread (runs are multiples of 2048 points)
    static_assert(!kSampled || sizeof(LI) == 8, "sampled indices are global");
    const int nrun = sm.segs / sm.subs;
    for (int r = blockIdx.x; r < nrun; r += gridDim.x) {
      const std::uint64_t start = sm.run_start(std::uint64_t(r) * sm.subs + g);
      for (int k0 = threadIdx.x; k0 < sm.len; k0 += 256 * 8) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = ld_stream(pts + start + k0 + u * 256);
#pragma unroll
        for (int u = 0; u < 8; ++u) k1_visit(lst, v[u], LI(start + k0 + u * 256));
      }
    }
  } else {
    const std::uint64_t stride = std::uint64_t(gridDim.x) * 256;
    std::uint64_t j = std::uint64_t(blockIdx.x) * 256 + threadIdx.x;
    for (; j + 3 * stride < n; j += 4 * stride) {
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = ld_stream(pts + j + u * stride);
#pragma unroll
      for (int u = 0; u < 4; ++u) k1_visit(lst, v[u], LI(j + u * stride));
    }
    for (; j < n; j += stride) k1_visit(lst, ld_stream(pts + j), LI(j));
  }
  ArgState<8, 4> st;
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    st.k[a] = lst.k[a];
    std::uint64_t i = ~std::uint64_t(0);  // untouched slot
    if (lst.i[a] != ~LI(0)) i = lst.i[a];
    st.i[a] = i;
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) st.s[a] = lst.s[a];
  block_reduce<8, 4, 256>(st);
  if (!grid_combine<8, 4, 256>(st, partials, ticket)) return;
  if (threadIdx.x < 8) {
    const int a = threadIdx.x;
    double k = 0, s2 = 0;
    std::uint64_t i = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b)
      if (b == a) {
        k = st.k[b];
        i = st.i[b];
        if (b >= 4) s2 = st.s[b - 4];
      }
    const std::uint64_t cnt = kSampled ? std::uint64_t(sm.segs / sm.subs) * sm.len : n;
    const double2 p = cnt ? pts[i] : make_double2(0.0, 0.0);  // an empty list has no winner
    if (cnt && lm.idx)
      i = lm.base + (lm.bytes == 4 ? std::uint64_t(static_cast<const std::uint32_t*>(lm.idx)[i])
                                   : static_cast<const std::uint64_t*>(lm.idx)[i]);
    out->key[a] = k;
    out->idx[a] = i;
    out->x[a] = p.x;
    out->y[a] = p.y;
    if (a >= 4) out->second[a - 4] = s2;
    if (a == 0) out->n = cnt;
  }
}

// ==================================================================== K1b ==
// slot k: argmax of -(|x - cx| + |y - cy|) = the reference argmin of
// manhattan(p, corner) (geometry.hpp:35-37), corners ne, nw, sw, se.
__global__ void __launch_bounds__(kK1Block, kK1MinBlocks)
    k1b_corners(const double2* __restrict__ pts, std::uint64_t n,
                std::uint64_t base, double xmax, double ymax, double xmin,
                double ymin, K1Partial* partials, unsigned* ticket,
                ohx_corner_rec* out) {
  ArgState<4, 0> st;
  st.init();
  const double cx[4] = {xmax, xmin, xmin, xmax};
  const double cy[4] = {ymax, ymax, ymin, ymin};
  const std::uint64_t stride = std::uint64_t(gridDim.x) * kK1Block;
  std::uint64_t j = std::uint64_t(blockIdx.x) * kK1Block + threadIdx.x;
  auto visit = [&](double2 p, std::uint64_t jj) {
    double m[4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
      m[a] = __dadd_rn(fabs(__dsub_rn(p.x, cx[a])), fabs(__dsub_rn(p.y, cy[a])));
    // fast path as in K1: only a strictly closer point touches the state
    const bool hit = (-m[0] > st.k[0]) | (-m[1] > st.k[1]) | (-m[2] > st.k[2]) |
                     (-m[3] > st.k[3]);
    if (hit) {
#pragma unroll
      for (int a = 0; a < 4; ++a) upd(st.k[a], st.i[a], -m[a], jj);
    }
  };
  for (; j + (kK1Unroll - 1) * stride < n; j += kK1Unroll * stride) {
    double2 v[kK1Unroll];
#pragma unroll
    for (int u = 0; u < kK1Unroll; ++u) v[u] = ld_stream(pts + j + u * stride);
#pragma unroll
    for (int u = 0; u < kK1Unroll; ++u) visit(v[u], j + u * stride);
  }
  for (; j < n; j += stride) visit(ld_stream(pts + j), j);

  block_reduce<4, 0, kK1Block>(st);
  if (!grid_combine<4, 0, kK1Block>(st, partials, ticket)) return;
  if (threadIdx.x < 4) {
    const int a = threadIdx.x;
    double k = 0;
    std::uint64_t i = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if (b == a) {
        k = st.k[b];
        i = st.i[b];
      }
    const double2 p = pts[i];
    out->key[a] = -k;
    out->idx[a] = base + i;
    out->x[a] = p.x;
    out->y[a] = p.y;
    if (a == 0) out->n = n;
  }
}

// ===================================================================== K2 ==
// Two launches:
//   k2_filter   labels every point of a 2048-point tile and writes the tile's
//               survivors, ordered (quadrant, index), as 16-bit tile offsets
//               into the tile's own slice of a scratch buffer, plus the
//               tile's four queue counts.  No cross-tile dependency, one
//               block barrier per tile.
//   k2_compact  one thread per tile: scans the tile counts (block scan +
//               decoupled look-back over groups of 256 tiles) and copies each
//               tile's survivors into the four queues as global indices.
// Survivors cost 2 B (scratch write) + 2 B (read) + the index write, which is
// negligible for filtered inputs and keeps the fully-surviving circle case
// free of per-tile serialisation.
constexpr std::uint64_t kFlagA = 1ull << 62;  // aggregate published
constexpr std::uint64_t kFlagP = 2ull << 62;  // inclusive prefix published
constexpr std::uint64_t kValMask = (1ull << 62) - 1;
constexpr int kK2Warps = kK2Block / 32;
constexpr int kK2Seg = kK2Items * kK2Warps;  // (item, warp) segments of a tile
constexpr int kK2Stage = 256;  // staged hard points per warp (all its items)

// orientation(a, b, p) < 0 with the edge constants A = fl(b.x-a.x),
// C = fl(b.y-a.y): det = fl(fl(A*fl(p.y-a.y)) - fl(C*fl(p.x-a.x))) is
// negative exactly when the first rounded product is below the second
// (geometry.hpp:27-32).
__device__ __forceinline__ bool right_of(double px, double py, double4 e) {
  return __dmul_rn(e.z, __dsub_rn(py, e.y)) < __dmul_rn(e.w, __dsub_rn(px, e.x));
}

struct K2Shared {
  double4 edge[12];  // octagon edges 0..7, then find_queue edges E->N, N->W, W->S, S->E
  std::uint32_t tile;
  std::uint32_t has_kept;
  std::uint32_t off[4][kK2Seg];
  std::uint32_t qbase[4];
  // per warp: up to kK2Stage of the warp's points outside the certified
  // box, densely packed, then their labels
  double2 stage[kK2Warps][kK2Stage];
  std::uint8_t lab[kK2Warps][kK2Stage];
};

// Edge constants are re-read from shared memory at every use (volatile):
// hoisting all twelve edges into registers would spill.
__device__ __forceinline__ double4 edge_at(const double4* e) {
  double4 r;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y)
               : "r"(static_cast<unsigned>(__cvta_generic_to_shared(e))));
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+16];" : "=d"(r.z), "=d"(r.w)
               : "r"(static_cast<unsigned>(__cvta_generic_to_shared(e))));
  return r;
}


// One warp walks back over predecessor status words of one quadrant and
// returns the exclusive prefix (decoupled look-back).
__device__ __forceinline__ std::uint64_t look_back(const std::uint64_t* st,
                                                   std::uint64_t unit) {
  const int lane = threadIdx.x & 31;
  std::uint64_t excl = 0;
  long long pos = static_cast<long long>(unit) - 1;
  for (;;) {
    const long long at = pos - lane;
    std::uint64_t w = kFlagP;  // before unit 0: a virtual zero prefix
    if (at >= 0) {
      do {
        w = ld_relaxed(st + at);
      } while ((w >> 62) == 0);
    }
    const unsigned pmask = __ballot_sync(kFull, (w & kFlagP) != 0);
    std::uint64_t v = w & kValMask;
    if (pmask) {
      const int first = __ffs(pmask) - 1;  // nearest inclusive prefix
      if (lane > first) v = 0;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
    excl += v;
    if (pmask) return excl;
    pos -= 32;
  }
}

// Gather mode (GIdx != void): the tile's items are the points gidx[t0 + jl]
// of a candidate list rather than consecutive points.
template <typename GIdx>
__device__ __forceinline__ std::uint64_t item_index(const GIdx* gidx, std::uint64_t k) {
  if constexpr (std::is_void_v<GIdx>) return k;
  else return static_cast<std::uint64_t>(__ldg(gidx + k));
}

// In gather mode `cpts` (when set) holds the candidates' coordinates already
// gathered, cpts[k] = pts[gidx[k]]: contiguous loads instead of a gather.
template <bool kFull_, typename GIdx>
__device__ __forceinline__ std::uint32_t k2_label_tile(const KPlan& plan, const double2* pts,
                                                       const GIdx* gidx, const double2* cpts,
                                                       std::uint64_t n, std::uint64_t t0,
                                                       bool has_kept, K2Shared& S) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  double2 v[kK2Items];
#pragma unroll
  for (int it = 0; it < kK2Items; ++it) {
    const std::uint32_t jl = it * kK2Block + threadIdx.x;
    v[it] = (kFull_ || t0 + jl < n)
                ? ld_stream(cpts != nullptr ? cpts + t0 + jl : pts + item_index(gidx, t0 + jl))
                : make_double2(0.0, 0.0);
  }
  // 1) kept overrides and the certified box; everything else is "hard".
  //    Labels live packed in one register, 4 bits per item.
  std::uint32_t labs = 0;
  std::uint32_t hard = 0;  // bit it: item it needs the full test
#pragma unroll
  for (int it = 0; it < kK2Items; ++it) {
    const bool inbox = v[it].x >= plan.box[0] && v[it].x <= plan.box[1] &&
                       v[it].y >= plan.box[2] && v[it].y <= plan.box[3];
    const std::uint32_t jl = it * kK2Block + threadIdx.x;
    bool h = !inbox && (kFull_ || t0 + jl < n);
    if (has_kept && (kFull_ || t0 + jl < n)) {
      const std::uint64_t j = item_index(gidx, t0 + jl);
      std::uint32_t kl = 0;
#pragma unroll
      for (int k = 7; k >= 0; --k)  // first match wins (filter.cpp:122-124)
        if (j == plan.kept[k]) kl = plan.kept_label[k];
      if (kl) {
        labs |= kl << (4 * it);
        h = false;
      }
    }
    hard |= std::uint32_t(h) << it;
  }
  // 2) the warp's hard points are packed into shared memory and classified
  //    there: a few out-of-box lanes do not make every item of the warp pay
  //    for the full test, and each lane tests up to four staged points per
  //    read of an edge's constants (warp-uniform shared loads: with one
  //    point per read they were the shared-memory pipe's whole budget on
  //    inputs where every point is hard -- ncu, circle 1e8: L1/shared 93 %
  //    busy, FP64 pipe 40 %)
  if (__any_sync(kFull, hard != 0)) {
    std::uint32_t H = 0;
#pragma unroll
    for (int it = 0; it < kK2Items; ++it) {
      const unsigned hb = __ballot_sync(kFull, hard >> it & 1u);
      if (hard >> it & 1u) S.stage[warp][H + __popc(hb & lt)] = v[it];
      H += __popc(hb);
    }
    __syncwarp();
    // (gather mode holds more live state: two points per read there)
    constexpr int U = std::is_void_v<GIdx> ? 4 : 2;
    for (std::uint32_t s0 = lane; s0 < H; s0 += U * 32) {
      double2 p[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        p[u] = s0 + 32 * u < H ? S.stage[warp][s0 + 32 * u] : make_double2(0.0, 0.0);
      bool out[U];
      std::uint32_t q[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        out[u] = plan.m < 3;  // degenerate octagon filters nothing (filter.cpp:125)
        q[u] = 1;             // default queue (filter.cpp:101)
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {  // "some edge < 0", in any order
        const double4 E = edge_at(S.edge + e);
#pragma unroll
        for (int u = 0; u < U; ++u) out[u] |= right_of(p[u].x, p[u].y, E);
      }
#pragma unroll
      for (int k = 3; k >= 0; --k) {  // find_queue: the lowest matching edge wins
        const double4 E = edge_at(S.edge + 8 + k);
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (right_of(p[u].x, p[u].y, E)) q[u] = k + 1;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (s0 + 32 * u < H) S.lab[warp][s0 + 32 * u] = static_cast<std::uint8_t>(out[u] ? q[u] : 0);
    }
    __syncwarp();
    H = 0;
#pragma unroll
    for (int it = 0; it < kK2Items; ++it) {
      const unsigned hb = __ballot_sync(kFull, hard >> it & 1u);
      if (hard >> it & 1u) labs |= std::uint32_t(S.lab[warp][H + __popc(hb & lt)]) << (4 * it);
      H += __popc(hb);
    }
  }
  return labs;
}

// One-pass mode (gather mode over a candidate list of at most
// kK2OnePassMaxTiles tiles): each tile publishes its four quadrant counts
// and sums the counts of ALL the tiles before it (one load per lane per 32
// tiles, in parallel: a chained look-back advances one L2 round trip per
// 32 tiles, and with every tile resident at once that chain was the
// kernel's critical path); then it writes its survivors' indices and
// coordinates straight into the four queues -- no scratch slice, no
// k2_compact, no separate coordinate gather.  Tile ids are taken in launch
// order, so the tiles before a tile are resident or done.
// The work words are left zeroed by the kernel itself (the last tile to
// finish clears them and re-arms the counters): no memset per launch.
// The first spec_q survivors of each quadrant also go to `spec` ([q][spec_q]
// coordinates, then the four counts): one small copy brings the host both.
struct K2OnePass {
  std::uint64_t* status;  // 4 x ntiles count words (kFlagA | count)
  unsigned* tile_counter;
  unsigned* done;         // finished tiles
  void* queues;           // 4 queues of cap entries (the list's index type)
  double2* qxy;           // 4 x cap survivor coordinates, same positions
  std::uint64_t cap;
  double2* spec;          // 4 x spec_q coordinates + 4 counts (u64)
  std::uint32_t spec_q;
};
__host__ __device__ inline unsigned long long* k2_spec_counts(double2* spec, std::uint32_t spec_q) {
  return reinterpret_cast<unsigned long long*>(spec + 4ull * spec_q);
}

// One-pass tail (see K2OnePass): the tile's quadrant totals are in
// S.qbase, the per-(item, warp) exclusive offsets in S.off.
template <typename GIdx>
__device__ __forceinline__ void k2_one_pass_tail(const GIdx* __restrict__ gidx,
                                                 const double2* __restrict__ cpts,
                                                 std::uint64_t t0, std::uint64_t tile,
                                                 std::uint64_t ntiles, std::uint32_t labs,
                                                 K2Shared& S, const K2OnePass& op) {
  constexpr int W = kK2Warps;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  __shared__ std::uint64_t s_excl[4];
  if (warp < 4) {
    const int q = warp;
    const std::uint64_t agg = S.qbase[q];
    std::uint64_t* st = op.status + std::uint64_t(q) * ntiles;
    if (lane == 0) st_relaxed(st + tile, kFlagA | agg);
    std::uint64_t excl = 0;
    for (std::uint64_t k = lane; k < tile; k += 32) {
      std::uint64_t w;
      do {
        w = ld_relaxed(st + k);
      } while ((w >> 62) == 0);
      excl += w & kValMask;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) excl += __shfl_xor_sync(kFull, excl, off);
    if (lane == 0) {
      s_excl[q] = excl;
      if (tile == ntiles - 1) k2_spec_counts(op.spec, op.spec_q)[q] = excl + agg;
    }
  }
  __syncthreads();
  GIdx* queues = static_cast<GIdx*>(op.queues);
#define LAB(it) ((labs >> (4 * (it))) & 0xFu)
#pragma unroll
  for (int it = 0; it < kK2Items; ++it) {
    const std::uint32_t q = LAB(it) - 1u;
    const unsigned live = __ballot_sync(kFull, LAB(it) != 0);
    if (!live) continue;
    const unsigned b0 = __ballot_sync(kFull, q & 1u);
    const unsigned b1 = __ballot_sync(kFull, q & 2u);
    if (LAB(it) == 0) continue;
    const unsigned mine = live & ((q & 1u) ? b0 : ~b0) & ((q & 2u) ? b1 : ~b1);
    const std::uint64_t pos = s_excl[q] + S.off[q][it * W + warp] + __popc(mine & lt);
    if (pos < op.cap) {
      const std::uint64_t k = t0 + std::uint64_t(it) * kK2Block + threadIdx.x;
      const double2 p = cpts[k];
      queues[q * op.cap + pos] = gidx[k];
      op.qxy[q * op.cap + pos] = p;
      if (pos < op.spec_q) op.spec[q * op.spec_q + pos] = p;
    }
  }
#undef LAB
  // the last tile to finish leaves the work words zeroed for the next launch
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(op.done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  for (std::uint64_t i = threadIdx.x; i < 4 * ntiles; i += kK2Block) op.status[i] = 0;
  if (threadIdx.x == 0) {
    *op.tile_counter = 0;
    *op.done = 0;
  }
}

template <typename GIdx, bool kOnePass = false>
__global__ void __launch_bounds__(kK2Block, 4)
    k2_filter(const double2* __restrict__ pts, const GIdx* __restrict__ gidx,
              const double2* __restrict__ cpts, std::uint64_t n,
              const __grid_constant__ KPlan plan, unsigned* tile_counter,
              std::uint32_t* tile_counts, std::uint64_t ntiles,
              std::uint16_t* scratch, std::uint8_t* labels, const K2OnePass op) {
  static_assert(!kOnePass || !std::is_void_v<GIdx>, "one-pass mode is gather mode");
  constexpr int W = kK2Warps;
  extern __shared__ __align__(16) unsigned char k2_smem[];
  K2Shared& S = *reinterpret_cast<K2Shared*>(k2_smem);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;

  if (threadIdx.x < 8)
    S.edge[threadIdx.x] = make_double4(plan.ax[threadIdx.x], plan.ay[threadIdx.x],
                                       plan.ea[threadIdx.x], plan.ec[threadIdx.x]);
  else if (threadIdx.x < 12)
    S.edge[threadIdx.x] = make_double4(plan.qax[threadIdx.x - 8], plan.qay[threadIdx.x - 8],
                                       plan.qa[threadIdx.x - 8], plan.qc[threadIdx.x - 8]);
  if (threadIdx.x == 32) {
    const std::uint32_t t = atomicAdd(tile_counter, 1u);
    S.tile = t;
    bool hk = !std::is_void_v<GIdx>;  // gather mode: a candidate may be any point
    for (int k = 0; k < 8; ++k) hk |= (plan.kept[k] - std::uint64_t(t) * kK2Tile) < kK2Tile;
    S.has_kept = hk;
  }
  __syncthreads();
  const std::uint64_t tile = S.tile;
  const std::uint64_t t0 = tile * kK2Tile;
  const bool has_kept = S.has_kept;
  const std::uint32_t labs = (t0 + kK2Tile <= n)
                                 ? k2_label_tile<true>(plan, pts, gidx, cpts, n, t0, has_kept, S)
                                 : k2_label_tile<false>(plan, pts, gidx, cpts, n, t0, has_kept, S);
#define LAB(it) ((labs >> (4 * (it))) & 0xFu)
  if (labels != nullptr) {
#pragma unroll
    for (int it = 0; it < kK2Items; ++it) {
      const std::uint64_t j = t0 + std::uint64_t(it) * kK2Block + threadIdx.x;
      if (j < n) labels[item_index(gidx, j)] = static_cast<std::uint8_t>(LAB(it));
    }
  }
  if (!__syncthreads_or(labs != 0) && !kOnePass) {
    if (threadIdx.x < 4) tile_counts[threadIdx.x * ntiles + tile] = 0;
    return;
  }
  // 3) per (item, warp, quadrant) survivor counts; a lane's own quadrant
  //    mask comes from two ballots of the label bits
#pragma unroll
  for (int it = 0; it < kK2Items; ++it) {
    const std::uint32_t code = LAB(it) - 1u;  // 0..3 for survivors
    const unsigned live = __ballot_sync(kFull, LAB(it) != 0);
    const unsigned b0 = __ballot_sync(kFull, code & 1u);
    const unsigned b1 = __ballot_sync(kFull, code & 2u);
    if (lane < 4) {
      const unsigned m0 = (lane & 1) ? b0 : ~b0;
      const unsigned m1 = (lane & 2) ? b1 : ~b1;
      S.off[lane][it * W + warp] = __popc(live & m0 & m1);
    }
  }
  __syncthreads();
  // exclusive scan of each quadrant's segment counts (warp q), then the
  // quadrant bases inside the tile's scratch slice (q-major order)
  if (warp < 4) {
    constexpr int PER = kK2Seg / 32;
    std::uint32_t c[PER];
    std::uint32_t sum = 0;
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      c[r] = S.off[warp][lane * PER + r];
      sum += c[r];
    }
    std::uint32_t incl = sum;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const std::uint32_t o = __shfl_up_sync(kFull, incl, off);
      if (lane >= off) incl += o;
    }
    std::uint32_t run = incl - sum;
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      S.off[warp][lane * PER + r] = run;
      run += c[r];
    }
    if (lane == 31) {
      if (!kOnePass) tile_counts[warp * ntiles + tile] = incl;
      S.qbase[warp] = incl;  // the quadrant total, turned into a base below
    }
  }
  __syncthreads();
  if constexpr (kOnePass) {
    k2_one_pass_tail<GIdx>(gidx, cpts, t0, tile, ntiles, labs, S, op);
    return;
  }
  const std::uint32_t tot0 = S.qbase[0], tot1 = S.qbase[1], tot2 = S.qbase[2];
  const std::uint32_t tot01 = tot0 + tot1, tot012 = tot01 + tot2;
  std::uint16_t* slice = scratch + t0;
  // 4) scatter survivors in (quadrant, index) order: one 16-bit store each
#pragma unroll
  for (int it = 0; it < kK2Items; ++it) {
    const std::uint32_t q = LAB(it) - 1u;
    const unsigned live = __ballot_sync(kFull, LAB(it) != 0);
    if (!live) continue;
    const unsigned b0 = __ballot_sync(kFull, q & 1u);
    const unsigned b1 = __ballot_sync(kFull, q & 2u);
    if (LAB(it) == 0) continue;
    const unsigned mine = live & ((q & 1u) ? b0 : ~b0) & ((q & 2u) ? b1 : ~b1);
    const std::uint32_t qb = q == 0 ? 0u : (q == 1 ? tot0 : (q == 2 ? tot01 : tot012));
    const std::uint32_t pos = qb + S.off[q][it * W + warp] + __popc(mine & lt);
    slice[pos] = static_cast<std::uint16_t>(it * kK2Block + threadIdx.x);
  }
#undef LAB
}

constexpr int kK2cBlock = 256;  // threads per compaction block
constexpr int kK2cTiles = static_cast<int>(kK2GroupTiles);  // tiles per compaction group

template <typename IdxT, bool kGather>
__global__ void __launch_bounds__(kK2cBlock)
    k2_compact(const std::uint32_t* __restrict__ tile_counts, std::uint64_t ntiles,
               const std::uint16_t* __restrict__ scratch, std::uint64_t* status,
               unsigned* group_counter, IdxT* queues, std::uint64_t cap,
               unsigned long long* counts, const IdxT* __restrict__ gidx) {
  constexpr int G = kK2cTiles;  // tiles per group: threads [0, G) hold one tile each
  static_assert(G == 64 && kK2cBlock >= 128, "scan below assumes two warps of tiles");
  __shared__ std::uint32_t s_group;
  __shared__ std::uint64_t s_excl[4];
  __shared__ std::uint32_t s_tot[4];
  __shared__ std::uint32_t s_pre[4][G];  // group-level exclusive prefix per tile
  __shared__ std::uint16_t s_src[4][G];  // quadrant offset inside each tile slice
  __shared__ std::uint16_t s_cnt[4][G];  // survivors of each quadrant in each tile
  __shared__ std::uint32_t s_w0[4];      // warp 0's totals
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const std::uint64_t ngroups = (ntiles + G - 1) / G;
  if (threadIdx.x == 0) s_group = atomicAdd(group_counter, 1u);
  __syncthreads();
  const std::uint64_t g = s_group;
  if (threadIdx.x < G) {
    const std::uint64_t tile = g * G + threadIdx.x;
    std::uint32_t c[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) c[q] = tile < ntiles ? tile_counts[q * ntiles + tile] : 0u;
    s_src[0][threadIdx.x] = 0;
    s_src[1][threadIdx.x] = static_cast<std::uint16_t>(c[0]);
    s_src[2][threadIdx.x] = static_cast<std::uint16_t>(c[0] + c[1]);
    s_src[3][threadIdx.x] = static_cast<std::uint16_t>(c[0] + c[1] + c[2]);
#pragma unroll
    for (int q = 0; q < 4; ++q) s_cnt[q][threadIdx.x] = static_cast<std::uint16_t>(c[q]);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      std::uint32_t incl = c[q];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const std::uint32_t o = __shfl_up_sync(kFull, incl, off);
        if (lane >= off) incl += o;
      }
      s_pre[q][threadIdx.x] = incl - c[q];  // warp-local for now
      if (warp == 0 && lane == 31) s_w0[q] = incl;
      if (warp == 1 && lane == 31) s_tot[q] = incl;  // warp 1's total, fixed up below
    }
  }
  __syncthreads();
  if (warp < 4) {
    const int q = warp;
    const std::uint32_t agg = s_w0[q] + s_tot[q];
    std::uint64_t excl = 0;
    if (g == 0) {
      if (lane == 0) st_relaxed(status + q * ngroups, kFlagP | agg);
    } else {
      if (lane == 0) st_relaxed(status + q * ngroups + g, kFlagA | agg);
      excl = look_back(status + q * ngroups, g);
      if (lane == 0) st_relaxed(status + q * ngroups + g, kFlagP | (excl + agg));
    }
    // the second warp's tiles come after the first warp's
    s_pre[q][32 + lane] += s_w0[q];
    __syncwarp();
    if (lane == 0) {
      s_excl[q] = excl;
      s_tot[q] = agg;
      if (g == ngroups - 1) counts[q] = excl + agg;
    }
  }
  __syncthreads();
  // copy: one warp per (quadrant, tile) run -- a run is contiguous in the
  // tile's scratch slice and in the queue, so loads and stores coalesce;
  // four independent loads in flight per lane (survivor-heavy inputs: with
  // a per-survivor binary search over the group prefix this kernel was
  // latency-bound, 0.39 ms for the circle's 1e8 survivors)
  constexpr int kWarps = kK2cBlock / 32;
#pragma unroll 1
  for (int r = warp; r < 4 * G; r += kWarps) {
    const int q = r / G, ti = r % G;
    const std::uint32_t cnt = s_cnt[q][ti];
    if (cnt == 0) continue;
    const std::uint64_t t = g * G + ti;
    const std::uint64_t dst = s_excl[q] + s_pre[q][ti];
    IdxT* out = queues + std::uint64_t(q) * cap;
    const std::uint16_t* src = scratch + t * kK2Tile + s_src[q][ti];
    for (std::uint32_t e0 = lane; e0 < cnt; e0 += 4 * 32) {
      std::uint16_t v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = e0 + 32 * u < cnt ? src[e0 + 32 * u] : std::uint16_t(0);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const std::uint32_t e = e0 + 32 * u;
        if (e < cnt && dst + e < cap) {
          const std::uint64_t item = t * kK2Tile + v[u];
          out[dst + e] = kGather ? gidx[item] : static_cast<IdxT>(item);
        }
      }
    }
  }
}

// ===================================================================== KF ==
// Fused single pass.  Before the pass the host fits a provisional region Q
// (an octagon with the slot directions as edge normals) from a sample, with
// every bound of Q strictly below the sample's value of the matching
// extremes key (the best for the axis slots, the second for the diagonal
// ones).  The whole input's best / second can only be larger, so a point
// inside Q can be neither an extreme, nor tied with one, nor a second-best:
// the eight extremes and the second-best keys are exactly those of the
// points OUTSIDE Q (the candidates).  KF therefore only streams the points
// once, tests Q (2 DADD + 8 DSETP per point, the same rounded keys as K1)
// and appends the candidates' indices to per-warp regions; kf_gather turns
// those into one ordered candidate list with the candidates' coordinates
// gathered next to it, K1 runs on the gathered candidates, and after the
// octagon is known the host checks that Q lies inside it (exact error bounds) and holds no kept point; then every
// dropped point has the reference label 0 and only the candidates need K2
// (gather mode).  Otherwise the regular K2 pass runs over all points.
constexpr int kKFBlock = 256;
constexpr int kKFMinBlocks = 4;
constexpr int kWT = 256;  // points per warp tile (8 items x 32 lanes)

// Is p inside the provisional region Q?  (a predicate chain: 2 DADD +
// 8 DSETP, no integer select per comparison)
__device__ __forceinline__ bool in_region(const KFRegion& q, double2 p) {
  std::uint32_t r;
  asm("{\n\t.reg .pred p;\n\t.reg .f64 t, d;\n\t"
      "add.rn.f64 t, %1, %2;\n\t"
      "sub.rn.f64 d, %1, %2;\n\t"
      "setp.ge.f64 p, %1, %3;\n\t"
      "setp.le.and.f64 p, %1, %4, p;\n\t"
      "setp.ge.and.f64 p, %2, %5, p;\n\t"
      "setp.le.and.f64 p, %2, %6, p;\n\t"
      "setp.ge.and.f64 p, t, %7, p;\n\t"
      "setp.le.and.f64 p, t, %8, p;\n\t"
      "setp.ge.and.f64 p, d, %9, p;\n\t"
      "setp.le.and.f64 p, d, %10, p;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(r)
      : "d"(p.x), "d"(p.y), "d"(q.x0), "d"(q.x1), "d"(q.y0), "d"(q.y1), "d"(q.t0), "d"(q.t1),
        "d"(q.d0), "d"(q.d1));
  return r != 0;
}

__device__ __forceinline__ std::uint64_t l2_evict_last_policy() {
  std::uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// candidate stores stay in L2 (they are read back right after the pass)
__device__ __forceinline__ void st_keep(std::uint32_t* p, std::uint32_t v, std::uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_keep(std::uint64_t* p, std::uint64_t v, std::uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}

// Every warp streams its own contiguous range of 256-point tiles (point
// t0 + it * 32 + lane in item it) and appends its candidates' indices, in
// index order, to a private region of cap_w entries: the only stores of the
// pass are the candidates themselves, written densely (the measured cost of
// any per-tile record -- counts, slots or bit masks -- is 10x its share of
// the bytes: writes interleaved with the read stream).  The exact count is
// kept even past cap_w (the host then falls back to two passes).
template <bool kFullTile, typename IdxT>
__device__ __forceinline__ void kf_tile(const double2* __restrict__ pts, std::uint64_t n,
                                        std::uint64_t t0, const KFRegion& q, IdxT* reg,
                                        std::uint64_t cap_w, std::uint64_t pol,
                                        std::uint32_t& c) {
  const int lane = threadIdx.x & 31;
  double2 v[8];
#pragma unroll
  for (int it = 0; it < 8; ++it)
    v[it] = (kFullTile || t0 + it * 32 + lane < n) ? ld_stream(pts + t0 + it * 32 + lane)
                                                   : make_double2(0.0, 0.0);
  std::uint32_t cand = 0;
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    if (!in_region(q, v[it]) && (kFullTile || t0 + it * 32 + lane < n)) cand |= 1u << it;
  }
  std::uint32_t items = __reduce_or_sync(kFull, cand);
  if (items == 0) return;
  const unsigned lt = (1u << lane) - 1u;
  do {
    const int it = __ffs(items) - 1;
    items &= items - 1;
    const bool mine = cand >> it & 1u;
    const unsigned b = __ballot_sync(kFull, mine);
    if (mine) {
      const std::uint32_t pos = c + __popc(b & lt);
      if (pos < cap_w) st_keep(reg + pos, static_cast<IdxT>(t0 + it * 32 + lane), pol);
    }
    c += __popc(b);
  } while (items);
}

template <typename IdxT>
__global__ void __launch_bounds__(kKFBlock, kKFMinBlocks)
    kf_filter(const double2* __restrict__ pts, std::uint64_t n, const KFRegion q,
              IdxT* __restrict__ regions, std::uint64_t cap_w,
              std::uint32_t* __restrict__ warp_counts, const unsigned long long* __restrict__ gate,
              unsigned long long gate_min) {
  const std::uint64_t nt = (n + kWT - 1) / kWT;
  const std::uint64_t nw = std::uint64_t(gridDim.x) * (kKFBlock / 32);
  const std::uint64_t gw = std::uint64_t(blockIdx.x) * (kKFBlock / 32) + (threadIdx.x >> 5);
  if (*gate < gate_min) {  // the sample's coverage of Q is too low: no pass
    if ((threadIdx.x & 31) == 0) warp_counts[gw] = 0;
    return;
  }
  const std::uint64_t per = (nt + nw - 1) / nw;
  const std::uint64_t b0 = min(nt, gw * per), b1 = min(nt, b0 + per);
  const std::uint64_t bf = max(b0, min(b1, n / kWT));  // tiles [b0, bf) are full
  IdxT* reg = regions + gw * cap_w;
  const std::uint64_t pol = l2_evict_last_policy();
  std::uint32_t c = 0;  // a warp range holds < 2^32 points
  for (std::uint64_t t = b0; t < bf; ++t) kf_tile<true>(pts, n, t * kWT, q, reg, cap_w, pol, c);
  if (bf < b1) kf_tile<false>(pts, n, bf * kWT, q, reg, cap_w, pol, c);
  if ((threadIdx.x & 31) == 0) warp_counts[gw] = c;
}

// One warp per KF warp region: copies its candidates to the ordered list
// and gathers their coordinates (cpts[k] = pts[cand[k]]) for the candidate
// K1 and the gather-mode K2.  The list offsets need no scan launch: block b
// sums the counts of warps [0, 8b) itself (<= 19 KB of L2 reads), and the
// last block publishes counts[0] = total, counts[1] = whether a region
// overflowed, counts[2] = the coverage count KF was gated on.
template <typename IdxT>
__global__ void __launch_bounds__(256)
    kf_gather(const double2* __restrict__ pts, const IdxT* __restrict__ regions,
              std::uint64_t cap_w, std::uint64_t nw, const std::uint32_t* __restrict__ warp_counts,
              const unsigned long long* __restrict__ gate, unsigned long long* __restrict__ counts,
              IdxT* __restrict__ cand, double2* __restrict__ cpts, std::uint64_t cap_c) {
  __shared__ std::uint64_t s_sum[8];
  __shared__ std::uint32_t s_max[8], s_own[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const std::uint64_t w0 = std::uint64_t(blockIdx.x) * 8;  // a multiple of 4: uint4 reads
  std::uint64_t acc = 0;
  std::uint32_t mx = 0;
  const auto* c4 = reinterpret_cast<const uint4*>(warp_counts);
  const std::uint64_t n4 = w0 / 4;
  for (std::uint64_t i = threadIdx.x; i < n4; i += 256 * 4) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      v[u] = i + u * 256 < n4 ? c4[i + u * 256] : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      acc += std::uint64_t(v[u].x) + v[u].y + v[u].z + v[u].w;
      mx = max(mx, max(max(v[u].x, v[u].y), max(v[u].z, v[u].w)));
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    acc += __shfl_xor_sync(kFull, acc, off);
    mx = max(mx, __shfl_xor_sync(kFull, mx, off));
  }
  if (lane == 0) {
    s_sum[warp] = acc;
    s_max[warp] = mx;
    s_own[warp] = w0 + warp < nw ? warp_counts[w0 + warp] : 0;
  }
  __syncthreads();
  std::uint64_t o = 0, total = 0;
  std::uint32_t over = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    o += s_sum[k] + (k < warp ? s_own[k] : 0);
    total += s_sum[k] + s_own[k];
    over = max(over, max(s_max[k], s_own[k]));
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
    counts[0] = total;
    counts[1] = over > cap_w;
    counts[2] = *gate;
  }
  const std::uint64_t w = w0 + warp;
  if (w >= nw || o >= cap_c) return;
  const std::uint64_t cnt = min(std::uint64_t(s_own[warp]), cap_c - o);
  const IdxT* r = regions + w * cap_w;
  for (std::uint64_t k = lane; k < cnt; k += 32) {
    const IdxT j = r[k];
    cand[o + k] = j;
    cpts[o + k] = ld_stream(pts + j);
  }
}

// ====================================================== K1 (TMA variant) ==
// K1's streaming pass fed by TMA bulk copies (OHX_STREAM=tma; the register-
// staged k1_extremes is the default -- it measured faster on B200): each
// block owns a contiguous range of 2048-point (32 KB) chunks and keeps
// kSStages of them in flight in shared memory (cp.async.bulk + mbarrier).
// Warp w processes the chunk's w-th 256-point tile straight from shared
// memory; the warp-uniform extremes update reads its points from the same
// buffer.
constexpr int kSBlock = 256;
constexpr int kSChunk = 2048;
constexpr int kSStages = 3;

struct StreamSmem {
  double2 buf[kSStages][kSChunk];
  unsigned long long bar[kSStages];
  WarpExt ext[kSBlock / 32];
};

__global__ void __launch_bounds__(kSBlock, 2)
    k1_stream_tma(const double2* __restrict__ pts, std::uint64_t n, std::uint64_t base,
                  K1Partial* partials, unsigned* ticket, ohx_extremes_rec* out) {
  extern __shared__ __align__(128) unsigned char k_stream_smem[];
  StreamSmem& S = *reinterpret_cast<StreamSmem*>(k_stream_smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpExt& we = S.ext[warp];
  double th[8];
  warp_ext_init(we, th);
  const std::uint64_t nchunks = (n + kSChunk - 1) / kSChunk;
  const std::uint64_t per = (nchunks + gridDim.x - 1) / gridDim.x;
  const std::uint64_t c0 = min(nchunks, std::uint64_t(blockIdx.x) * per);
  const std::uint64_t c1 = min(nchunks, c0 + per);
  auto issue = [&](std::uint64_t c, int st) {
    const std::uint64_t p0 = c * kSChunk;
    const unsigned bytes = static_cast<unsigned>((min(n, p0 + kSChunk) - p0) * sizeof(double2));
    mbar_arrive_expect(&S.bar[st], bytes);
    bulk_g2s(S.buf[st], pts + p0, bytes, &S.bar[st]);
  };
  if (threadIdx.x == 0) {
    for (int st = 0; st < kSStages; ++st) mbar_init(&S.bar[st], 1);
    mbar_fence_init();
    for (int st = 0; st < kSStages && c0 + st < c1; ++st) issue(c0 + st, st);
  }
  __syncthreads();
  for (std::uint64_t c = c0, k = 0; c < c1; ++c, ++k) {
    const int st = static_cast<int>(k % kSStages);
    mbar_wait(&S.bar[st], static_cast<unsigned>((k / kSStages) & 1));
    const std::uint64_t t0 = c * kSChunk + std::uint64_t(warp) * 256;  // this warp's tile
    double2* tile = S.buf[st] + warp * 256;
    if (t0 < n) {
      double2 v[8];
#pragma unroll
      for (int it = 0; it < 8; ++it) v[it] = tile[it * 32 + lane];
      if (t0 + 256 <= n) visit8<true>(we, th, v, t0 + lane, std::uint64_t(32), n, tile);
      else visit8<false>(we, th, v, t0 + lane, std::uint64_t(32), n, tile);
    }
    __syncthreads();  // every warp is done with stage st
    if (threadIdx.x == 0 && c + kSStages < c1) {
      fence_proxy_async_smem();  // order the generic reads before the async refill
      issue(c + kSStages, st);
    }
  }
  __syncwarp();
  ArgState<8, 4> res = warp_ext_state(we);
  block_reduce<8, 4, kSBlock, true>(res);
  if (!grid_combine<8, 4, kSBlock>(res, partials, ticket)) return;
  if (threadIdx.x < 8) {
    const int a = threadIdx.x;
    double kk = 0, s2 = 0;
    std::uint64_t i = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b)
      if (b == a) {
        kk = res.k[b];
        i = res.i[b];
        if (b >= 4) s2 = res.s[b - 4];
      }
    const double2 p = pts[i];
    out->key[a] = kk;
    out->idx[a] = base + i;
    out->x[a] = p.x;
    out->y[a] = p.y;
    if (a >= 4) out->second[a - 4] = s2;
    if (a == 0) out->n = n;
  }
}

// Number of the sample's points inside the region Q (sample coverage
// estimate): runs 0, step, 2 step, ... of the sample, each split over
// kCountSplit blocks (1024 points per block, 4 loads in flight per thread:
// one block per run left most SMs idle, 9 us for 8 MB).
constexpr int kCountSplit = 8;
__global__ void __launch_bounds__(256)
    count_in_region(const double2* __restrict__ pts, const SampleMap sm, int step,
                    const KFRegion q, unsigned long long* count) {
  __shared__ unsigned s_c[8];
  const int part = blockIdx.x % kCountSplit;
  const std::uint64_t start = sm.run_start(std::uint64_t(blockIdx.x / kCountSplit) * step);
  const int span = sm.len / kCountSplit;  // a multiple of 1024
  unsigned c = 0;
  for (int k0 = part * span + threadIdx.x; k0 < (part + 1) * span; k0 += 256 * 4) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = ld_stream(pts + start + k0 + u * 256);
#pragma unroll
    for (int u = 0; u < 4; ++u) c += in_region(q, v[u]);
  }
  c = __reduce_add_sync(kFull, c);
  if ((threadIdx.x & 31) == 0) s_c[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int w = 0; w < 8; ++w) t += s_c[w];
    atomicAdd(count, static_cast<unsigned long long>(t));
  }
}

// The smallest index of a point with a non-finite coordinate (the PTS2
// loader's validation, reference io.cpp:117-120), or leaves *first as is.
__global__ void first_nonfinite(const double2* __restrict__ pts, std::uint64_t n,
                                unsigned long long* first) {
  unsigned long long mine = ~0ull;
  for (std::uint64_t k = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
       k += std::uint64_t(gridDim.x) * blockDim.x) {
    const double2 p = ld_stream(pts + k);
    if (!isfinite(p.x) || !isfinite(p.y)) {
      mine = k;
      break;  // a thread's later indices are larger
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(kFull, mine, off);
    mine = o < mine ? o : mine;
  }
  if ((threadIdx.x & 31) == 0 && mine != ~0ull) atomicMin(first, mine);
}

// classify_points with a caller's polygon of more than 8 vertices
// (filter.cpp:104-131 accepts any vertex list; build_octagon never makes
// one): kept overrides first, then "some edge has orientation < 0" over all
// m edges (geometry.cpp:16-22, edges read through the read-only cache: every
// thread of a warp reads the same edge), then find_queue.  Labels only --
// the queues of a heaphull always come from K2 on a <= 8-vertex octagon.
__global__ void __launch_bounds__(256)
    k3_polygon_labels(const double2* __restrict__ pts, std::uint64_t n,
                      const double4* __restrict__ edges, int m, const KPlan plan,
                      std::uint8_t* __restrict__ labels) {
  for (std::uint64_t j = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
       j += std::uint64_t(gridDim.x) * blockDim.x) {
    std::uint32_t lab = 0xff;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (lab == 0xff && j == plan.kept[k]) lab = plan.kept_label[k];
    if (lab == 0xff) {
      const double2 p = ld_stream(pts + j);
      bool out = false;
      for (int e = 0; e < m && !out; ++e) {
        const double2 lo = __ldg(reinterpret_cast<const double2*>(edges + e));
        const double2 hi = __ldg(reinterpret_cast<const double2*>(edges + e) + 1);
        out = right_of(p.x, p.y, make_double4(lo.x, lo.y, hi.x, hi.y));
      }
      lab = 0;
      if (out) {
        lab = 1;
#pragma unroll
        for (int k = 3; k >= 0; --k)
          if (right_of(p.x, p.y, make_double4(plan.qax[k], plan.qay[k], plan.qa[k], plan.qc[k])))
            lab = k + 1;
      }
    }
    labels[j] = static_cast<std::uint8_t>(lab);
  }
}

template <typename IdxT>
__global__ void gather_xy(const double2* __restrict__ pts,
                          const IdxT* __restrict__ idx, std::uint64_t count,
                          double2* __restrict__ out) {
  for (std::uint64_t k = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
       k < count; k += std::uint64_t(gridDim.x) * blockDim.x)
    out[k] = pts[idx[k]];
}

// All four queues in one launch, packed back to back: out = [q1|q2|q3|q4].
template <typename IdxT>
__global__ void gather_xy4(const double2* __restrict__ pts, const IdxT* __restrict__ queues,
                           std::uint64_t cap, ulonglong4 ends, double2* __restrict__ out) {
  const std::uint64_t total = ends.w;
  for (std::uint64_t k = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += std::uint64_t(gridDim.x) * blockDim.x) {
    const int q = (k >= ends.x) + (k >= ends.y) + (k >= ends.z);
    const std::uint64_t start = q == 0 ? 0 : (q == 1 ? ends.x : (q == 2 ? ends.y : ends.z));
    out[k] = pts[queues[std::uint64_t(q) * cap + (k - start)]];
  }
}

// The same for large survivor sets, block b over the points [b S, (b+1) S):
// each queue's entries in that index range (two binary searches per queue)
// copied one queue after the other.  The four queues interleave in the
// index order (a circle's survivors: every line holds all four), so a
// grid-stride pass over the packed output reads every line once per queue,
// far apart in time; here the four reads of a line fall inside one block.
constexpr std::uint64_t kGatherRange = 4096;  // blocks in flight x 64 KB stay in L2
template <typename IdxT>
__device__ __forceinline__ std::uint64_t lower_bound_idx(const IdxT* q, std::uint64_t n,
                                                         std::uint64_t v) {
  std::uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const std::uint64_t mid = (lo + hi) >> 1;
    if (static_cast<std::uint64_t>(q[mid]) < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
template <typename IdxT>
__global__ void __launch_bounds__(256)
    gather_xy4_ranged(const double2* __restrict__ pts, std::uint64_t n,
                      const IdxT* __restrict__ queues, std::uint64_t cap, ulonglong4 ends,
                      double2* __restrict__ out) {
  __shared__ std::uint64_t s_lo[4], s_hi[4];
  const std::uint64_t a = std::uint64_t(blockIdx.x) * kGatherRange;
  const std::uint64_t b = min(n, a + kGatherRange);
  const std::uint64_t cnt[4] = {ends.x, ends.y - ends.x, ends.z - ends.y, ends.w - ends.z};
  if (threadIdx.x < 8) {
    const int q = threadIdx.x >> 1;
    const std::uint64_t v = lower_bound_idx(queues + std::uint64_t(q) * cap, cnt[q],
                                            (threadIdx.x & 1) ? b : a);
    if (threadIdx.x & 1) s_hi[q] = v;
    else s_lo[q] = v;
  }
  __syncthreads();
#pragma unroll 1
  for (int q = 0; q < 4; ++q) {
    const std::uint64_t start = q == 0 ? 0 : (q == 1 ? ends.x : (q == 2 ? ends.y : ends.z));
    const IdxT* qq = queues + std::uint64_t(q) * cap;
    for (std::uint64_t k = s_lo[q] + threadIdx.x; k < s_hi[q]; k += 256)
      out[start + k] = pts[qq[k]];
  }
}

// The same with the counts read on the device, for the first `limit`
// survivors: launched right behind K2 so that a small survivor set comes
// back with the counts, in the same round trip.  Nothing is written when a
// queue overflowed its capacity (the host re-runs K2 then).
template <typename IdxT>
__global__ void gather_xy4_dev(const double2* __restrict__ pts, const IdxT* __restrict__ queues,
                               std::uint64_t cap, const unsigned long long* __restrict__ counts,
                               std::uint64_t limit, double2* __restrict__ out) {
  const std::uint64_t c0 = counts[0], c1 = counts[1], c2 = counts[2], c3 = counts[3];
  if (c0 > cap || c1 > cap || c2 > cap || c3 > cap) return;
  const ulonglong4 ends = make_ulonglong4(c0, c0 + c1, c0 + c1 + c2, c0 + c1 + c2 + c3);
  const std::uint64_t total = ends.w < limit ? ends.w : limit;
  for (std::uint64_t k = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += std::uint64_t(gridDim.x) * blockDim.x) {
    const int q = (k >= ends.x) + (k >= ends.y) + (k >= ends.z);
    const std::uint64_t start = q == 0 ? 0 : (q == 1 ? ends.x : (q == 2 ? ends.y : ends.z));
    out[k] = pts[queues[std::uint64_t(q) * cap + (k - start)]];
  }
}

// ------------------------------------------------- hull vertex indices ----
// Each hull vertex -> the smallest input index with equal coordinates.
// Every hull vertex is a survivor (the extremes carry their queue label),
// and duplicates of a vertex share its label except duplicates of a kept
// extreme -- whose index is already the smallest with that key -- so the
// survivors are the only points to probe: the vertices go into an
// open-addressing table (distinct coordinates: the clean-up leaves strict
// turns), the survivors probe it and atomicMin their index.  -0.0 and
// +0.0 are the same coordinate (the reference's == comparisons).
__device__ __forceinline__ std::uint64_t coord_bits(double v) {
  return static_cast<std::uint64_t>(__double_as_longlong(v == 0.0 ? 0.0 : v));
}
__device__ __forceinline__ std::uint64_t coord_hash(double2 p) {
  std::uint64_t z = coord_bits(p.x) * 0x9E3779B97F4A7C15ull ^ coord_bits(p.y);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void hidx_insert(const double2* __restrict__ hull, std::uint64_t h,
                            std::uint32_t* __restrict__ slots, std::uint64_t mask) {
  const std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= h) return;
  for (std::uint64_t s = coord_hash(hull[i]) & mask;; s = (s + 1) & mask)
    if (atomicCAS(slots + s, 0xffffffffu, static_cast<std::uint32_t>(i)) == 0xffffffffu) return;
}

template <typename IdxT>
__global__ void hidx_probe(const double2* __restrict__ pts, const IdxT* __restrict__ queues,
                           std::uint64_t cap, ulonglong4 ends, std::uint64_t base,
                           const double2* __restrict__ hull, const std::uint32_t* __restrict__ slots,
                           std::uint64_t mask, unsigned long long* __restrict__ res) {
  for (std::uint64_t k = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < ends.w;
       k += std::uint64_t(gridDim.x) * blockDim.x) {
    const int q = (k >= ends.x) + (k >= ends.y) + (k >= ends.z);
    const std::uint64_t start = q == 0 ? 0 : (q == 1 ? ends.x : (q == 2 ? ends.y : ends.z));
    const std::uint64_t j = queues[std::uint64_t(q) * cap + (k - start)];
    const double2 p = pts[j];
    for (std::uint64_t s = coord_hash(p) & mask;; s = (s + 1) & mask) {
      const std::uint32_t v = slots[s];
      if (v == 0xffffffffu) break;  // not a hull vertex
      const double2 c = hull[v];
      if (c.x == p.x && c.y == p.y) {
        atomicMin(res + v, static_cast<unsigned long long>(base + j));
        break;
      }
    }
  }
}

}  // namespace

// ============================================================ launchers ==
static int tma_grid(int device, std::uint64_t n) {
  int sms = 0;
  check_cuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device),
             "cudaDeviceGetAttribute");
  const std::uint64_t nchunks = (n + kSChunk - 1) / kSChunk;
  const std::uint64_t full = std::uint64_t(sms) * 2;  // two 98 KB blocks per SM
  return static_cast<int>(nchunks < full ? (nchunks > 0 ? nchunks : 1) : full);
}

static void k1_tma_launch(const double* d_xy, std::uint64_t n, std::uint64_t base,
                          K1Partial* partials, int grid, unsigned* ticket,
                          ohx_extremes_rec* d_out, cudaStream_t stream) {
  constexpr int smem = sizeof(StreamSmem);
  static bool configured = false;
  if (!configured) {
    check_cuda(cudaFuncSetAttribute(k1_stream_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    smem),
               "cudaFuncSetAttribute(k1_stream_tma)");
    configured = true;
  }
  k1_stream_tma<<<grid, kSBlock, smem, stream>>>(reinterpret_cast<const double2*>(d_xy), n, base,
                                                 partials, ticket, d_out);
  check_cuda(cudaGetLastError(), "k1_stream_tma launch");
}

// OHX_STREAM selects K1's streaming implementation: unset/"reg" = the
// register-staged loads (default), "tma" = the cp.async.bulk pipeline.
static bool stream_tma() {
  static const bool tma = [] {
    const char* e = std::getenv("OHX_STREAM");
    return e && std::string(e) == "tma";
  }();
  return tma;
}

template <typename K>
static int occupancy_grid(int device, K kernel, int block, std::uint64_t need) {
  int sms = 0, per_sm = 0;
  check_cuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device),
             "cudaDeviceGetAttribute");
  check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, 0),
             "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
  if (per_sm < 1) per_sm = 1;
  const std::uint64_t full = std::uint64_t(sms) * per_sm;
  return static_cast<int>(need < full ? (need > 0 ? need : 1) : full);
}

int k1_grid(int device, std::uint64_t n) {
  if (stream_tma()) return tma_grid(device, n);
  return occupancy_grid(device, k1_extremes<std::uint32_t>, kK1Block,
                        (n + kK1Block * kK1Unroll - 1) / (kK1Block * kK1Unroll));
}

void launch_k1(const double* d_xy, std::uint64_t n, std::uint64_t base,
               K1Partial* partials, int grid, unsigned* ticket,
               ohx_extremes_rec* d_out, cudaStream_t stream) {
  if (stream_tma()) {
    k1_tma_launch(d_xy, n, base, partials, grid, ticket, d_out, stream);
    return;
  }
  const auto* pts = reinterpret_cast<const double2*>(d_xy);
  // 32-bit in-loop indices whenever the shard (plus a full grid stride of
  // overshoot) fits
  if (n + std::uint64_t(kK1Block) * kK1Unroll < 0xffffffffull)
    k1_extremes<std::uint32_t><<<grid, kK1Block, 0, stream>>>(pts, n, base, partials, ticket, d_out);
  else
    k1_extremes<std::uint64_t><<<grid, kK1Block, 0, stream>>>(pts, n, base, partials, ticket, d_out);
  check_cuda(cudaGetLastError(), "k1_extremes launch");
}

void launch_k1b(const double* d_xy, std::uint64_t n, std::uint64_t base,
                const double bbox[4], K1Partial* partials, int grid,
                unsigned* ticket, ohx_corner_rec* d_out, cudaStream_t stream) {
  k1b_corners<<<grid, kK1Block, 0, stream>>>(
      reinterpret_cast<const double2*>(d_xy), n, base, bbox[0], bbox[1], bbox[2],
      bbox[3], partials, ticket, d_out);
  check_cuda(cudaGetLastError(), "k1b_corners launch");
}

template <typename GIdx, bool kOnePass = false>
static void k2_filter_launch(const double2* pts, const GIdx* gidx, const double2* cpts,
                             std::uint64_t n,
                             const KPlan& plan, const K2Work& w, std::uint64_t ntiles,
                             std::uint8_t* d_labels, cudaStream_t stream,
                             const K2OnePass& op = K2OnePass{}) {
  constexpr int smem = sizeof(K2Shared);
  static bool configured = false;  // opt in to > 48 KB dynamic smem once per instantiation
  if (!configured) {
    check_cuda(cudaFuncSetAttribute(k2_filter<GIdx, kOnePass>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
               "cudaFuncSetAttribute");
    configured = true;
  }
  k2_filter<GIdx, kOnePass><<<static_cast<unsigned>(ntiles), kK2Block, smem, stream>>>(
      pts, gidx, cpts, n, plan, w.tile_counter, w.tile_counts, ntiles, w.scratch, d_labels, op);
  check_cuda(cudaGetLastError(), "k2_filter launch");
}

template <typename IdxT, bool kGather>
static void k2_compact_launch(const K2Work& w, std::uint64_t ntiles, IdxT* queues,
                              std::uint64_t cap, unsigned long long* d_counts,
                              const IdxT* gidx, cudaStream_t stream) {
  const unsigned ngroups = static_cast<unsigned>((ntiles + kK2cTiles - 1) / kK2cTiles);
  k2_compact<IdxT, kGather><<<ngroups, kK2cBlock, 0, stream>>>(
      w.tile_counts, ntiles, w.scratch, w.status, w.group_counter, queues, cap, d_counts, gidx);
  check_cuda(cudaGetLastError(), "k2_compact launch");
}

template <typename IdxT>
static void k2_launch(const double2* pts, std::uint64_t n, const KPlan& plan, void* d_work,
                      std::uint64_t ntiles, IdxT* q, std::uint64_t cap, std::uint8_t* d_labels,
                      unsigned long long* d_counts, cudaStream_t stream, const IdxT* g,
                      const double2* cp, const K2OnePassBufs* op_bufs) {
  if (op_bufs) {
    if (g == nullptr || cp == nullptr || ntiles > kK2OnePassMaxTiles)
      throw Error(OHX_E_INTERNAL, "k2 one-pass mode: a candidate list of <= kK2OnePassMaxTiles tiles");
    // the work area [tile counter | done | 4 x ntiles words] is zero on entry
    // (cleared once when allocated, then by the kernel's last tile)
    auto* w = static_cast<unsigned char*>(op_bufs->work);
    K2Work kw{};
    kw.tile_counter = reinterpret_cast<unsigned*>(w);
    const K2OnePass op{reinterpret_cast<std::uint64_t*>(w + 256), reinterpret_cast<unsigned*>(w),
                       reinterpret_cast<unsigned*>(w + 4), q,
                       reinterpret_cast<double2*>(op_bufs->qxy), cap,
                       reinterpret_cast<double2*>(op_bufs->spec), op_bufs->spec_q};
    k2_filter_launch<IdxT, true>(pts, g, cp, n, plan, kw, ntiles, d_labels, stream, op);
    return;
  }
  const K2Work w = k2_work_layout(d_work, ntiles);
  // re-arm the work counters and the look-back words
  check_cuda(cudaMemsetAsync(d_work, 0, w.clear_bytes, stream), "cudaMemsetAsync(k2 work)");
  if (g) {
    k2_filter_launch(pts, g, cp, n, plan, w, ntiles, d_labels, stream);
    k2_compact_launch<IdxT, true>(w, ntiles, q, cap, d_counts, g, stream);
  } else {
    k2_filter_launch<void>(pts, nullptr, nullptr, n, plan, w, ntiles, d_labels, stream);
    k2_compact_launch<IdxT, false>(w, ntiles, q, cap, d_counts, nullptr, stream);
  }
}

void launch_k2(const double* d_xy, std::uint64_t n, const KPlan& plan, void* d_work,
               std::uint64_t ntiles, void* d_queues, int idx_bytes, std::uint64_t cap,
               std::uint8_t* d_labels, unsigned long long* d_counts, cudaStream_t stream,
               const void* d_gather, const double* d_gather_xy, const K2OnePassBufs* op) {
  const auto* pts = reinterpret_cast<const double2*>(d_xy);
  const auto* cp = reinterpret_cast<const double2*>(d_gather_xy);
  if (idx_bytes == 4)
    k2_launch(pts, n, plan, d_work, ntiles, static_cast<std::uint32_t*>(d_queues), cap, d_labels,
              d_counts, stream, static_cast<const std::uint32_t*>(d_gather), cp, op);
  else
    k2_launch(pts, n, plan, d_work, ntiles, static_cast<std::uint64_t*>(d_queues), cap, d_labels,
              d_counts, stream, static_cast<const std::uint64_t*>(d_gather), cp, op);
}

int kf_grid(int device) {
  return occupancy_grid(device, kf_filter<std::uint32_t>, kKFBlock, ~0ull);
}

void launch_kf(const double* d_xy, std::uint64_t n, const KFRegion& q, int grid, void* d_regions,
               int idx_bytes, std::uint64_t cap_w, std::uint32_t* d_warp_counts,
               const unsigned long long* d_gate, std::uint64_t gate_min, cudaStream_t stream) {
  const auto* pts = reinterpret_cast<const double2*>(d_xy);
  if (idx_bytes == 4)
    kf_filter<std::uint32_t><<<grid, kKFBlock, 0, stream>>>(
        pts, n, q, static_cast<std::uint32_t*>(d_regions), cap_w, d_warp_counts, d_gate, gate_min);
  else
    kf_filter<std::uint64_t><<<grid, kKFBlock, 0, stream>>>(
        pts, n, q, static_cast<std::uint64_t*>(d_regions), cap_w, d_warp_counts, d_gate, gate_min);
  check_cuda(cudaGetLastError(), "kf_filter launch");
}

void launch_kf_gather(const double* d_xy, const void* d_regions, int idx_bytes,
                      std::uint64_t cap_w, const std::uint32_t* d_warp_counts, std::uint64_t nw,
                      const unsigned long long* d_gate, unsigned long long* d_counts,
                      void* d_cand, double* d_cpts, std::uint64_t cap_c, cudaStream_t stream) {
  const auto* pts = reinterpret_cast<const double2*>(d_xy);
  auto* cp = reinterpret_cast<double2*>(d_cpts);
  const unsigned grid = static_cast<unsigned>((nw + 7) / 8);
  if (idx_bytes == 4)
    kf_gather<<<grid, 256, 0, stream>>>(pts, static_cast<const std::uint32_t*>(d_regions), cap_w,
                                        nw, d_warp_counts, d_gate, d_counts,
                                        static_cast<std::uint32_t*>(d_cand), cp, cap_c);
  else
    kf_gather<<<grid, 256, 0, stream>>>(pts, static_cast<const std::uint64_t*>(d_regions), cap_w,
                                        nw, d_warp_counts, d_gate, d_counts,
                                        static_cast<std::uint64_t*>(d_cand), cp, cap_c);
  check_cuda(cudaGetLastError(), "kf_gather launch");
}

void launch_k1_sample(const double* d_xy, std::uint64_t n, int segs, int len, int subs,
                      K1Partial* partials, unsigned* ticket, ohx_extremes_rec* d_recs,
                      unsigned long long* d_count, cudaStream_t stream) {
  const SampleMap sm{n, segs, len, subs};
  // 2 runs per block (4 sub-samples x 128 runs at 1e9: 256 blocks; 1 run:
  // 36 us, 2: 33 us, 4: 37 us -- fewer partials vs. fewer blocks in flight);
  // OHX_SAMPLE_RPB overrides (tuning hook)
  static const int runs_per_block = [] {
    const char* e = std::getenv("OHX_SAMPLE_RPB");
    const int k = e ? std::atoi(e) : 0;
    return k >= 1 ? k : 2;
  }();
  const int bx = std::max(1, segs / subs / runs_per_block);
  k1_small<true, std::uint64_t><<<dim3(bx, subs), 256, 0, stream>>>(
      reinterpret_cast<const double2*>(d_xy), 0, nullptr, sm, ListMap{nullptr, 0, 0}, partials,
      ticket, d_recs, d_count);
  check_cuda(cudaGetLastError(), "k1_small<sample> launch");
}

int k1_list_grid(std::uint64_t n) {
  // at most one wave (the reduction's cost grows with the grid); the list
  // length is often counted on the device, n is then its capacity
  static const int wave = [] {
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    return occupancy_grid(dev, k1_small<false, std::uint32_t>, 256, ~0ull);
  }();
  // points per thread aimed at (OHX_K1LIST_PER overrides; tuning hook)
  static const std::uint64_t per = [] {
    const char* e = std::getenv("OHX_K1LIST_PER");
    const int k = e ? std::atoi(e) : 0;
    return static_cast<std::uint64_t>(k >= 1 ? k : 16);
  }();
  const std::uint64_t b = (n + 256 * per - 1) / (256 * per);
  return static_cast<int>(b < 1 ? 1 : (b > std::uint64_t(wave) ? wave : b));
}

void launch_k1_list(const double* d_xy, std::uint64_t n, const unsigned long long* d_n,
                    const void* d_map, int map_bytes, std::uint64_t map_base,
                    K1Partial* partials, int grid, unsigned* ticket, ohx_extremes_rec* d_rec,
                    cudaStream_t stream) {
  const auto* pts = reinterpret_cast<const double2*>(d_xy);
  const ListMap lm{d_map, map_bytes, map_base};
  if (n < 0xffffffffull)
    k1_small<false, std::uint32_t><<<dim3(grid, 1), 256, 0, stream>>>(
        pts, n, d_n, SampleMap{0, 1, 1, 1}, lm, partials, ticket, d_rec);
  else
    k1_small<false, std::uint64_t><<<dim3(grid, 1), 256, 0, stream>>>(
        pts, n, d_n, SampleMap{0, 1, 1, 1}, lm, partials, ticket, d_rec);
  check_cuda(cudaGetLastError(), "k1_small<list> launch");
}

void launch_count_in_region(const double* d_xy, std::uint64_t n, int segs, int len, int step,
                            const KFRegion& q, unsigned long long* d_count, cudaStream_t stream) {
  // (*d_count was zeroed by the sample kernel, earlier on this stream)
  if (len % (kCountSplit * 1024) != 0) throw Error(OHX_E_INTERNAL, "count_in_region: run length");
  count_in_region<<<(segs + step - 1) / step * kCountSplit, 256, 0, stream>>>(
      reinterpret_cast<const double2*>(d_xy), SampleMap{n, segs, len, 1}, step, q, d_count);
  check_cuda(cudaGetLastError(), "count_in_region launch");
}

void launch_polygon_labels(const double* d_xy, std::uint64_t n, const double* d_edges, int m,
                           const KPlan& plan, std::uint8_t* d_labels, cudaStream_t stream) {
  const std::uint64_t blocks = (n + 255) / 256;
  const unsigned grid = static_cast<unsigned>(blocks < 148ull * 16 ? blocks : 148ull * 16);
  k3_polygon_labels<<<grid, 256, 0, stream>>>(reinterpret_cast<const double2*>(d_xy), n,
                                              reinterpret_cast<const double4*>(d_edges), m, plan,
                                              d_labels);
  check_cuda(cudaGetLastError(), "k3_polygon_labels launch");
}

void launch_first_nonfinite(const double* d_xy, std::uint64_t n, unsigned long long* d_first,
                            cudaStream_t stream) {
  check_cuda(cudaMemsetAsync(d_first, 0xFF, sizeof(unsigned long long), stream), "cudaMemsetAsync");
  const unsigned grid = static_cast<unsigned>(n / (256 * 16) + 1 < 148 * 8 ? n / (256 * 16) + 1 : 148 * 8);
  first_nonfinite<<<grid, 256, 0, stream>>>(reinterpret_cast<const double2*>(d_xy), n, d_first);
  check_cuda(cudaGetLastError(), "first_nonfinite launch");
}

void launch_gather4(const double* d_xy, const void* d_queues, int idx_bytes,
                    std::uint64_t cap, const std::uint64_t counts[4], double* d_out,
                    cudaStream_t stream, std::uint64_t n) {
  const ulonglong4 ends = make_ulonglong4(counts[0], counts[0] + counts[1],
                                          counts[0] + counts[1] + counts[2],
                                          counts[0] + counts[1] + counts[2] + counts[3]);
  if (ends.w == 0) return;
  const auto* pts = reinterpret_cast<const double2*>(d_xy);
  // many survivors (at least one per 64 points on average): by index range
  if (n && ends.w >= (1u << 20) && ends.w * 64 >= n) {
    const unsigned g = static_cast<unsigned>((n + kGatherRange - 1) / kGatherRange);
    if (idx_bytes == 4)
      gather_xy4_ranged<<<g, 256, 0, stream>>>(pts, n, static_cast<const std::uint32_t*>(d_queues),
                                               cap, ends, reinterpret_cast<double2*>(d_out));
    else
      gather_xy4_ranged<<<g, 256, 0, stream>>>(pts, n, static_cast<const std::uint64_t*>(d_queues),
                                               cap, ends, reinterpret_cast<double2*>(d_out));
    check_cuda(cudaGetLastError(), "gather_xy4_ranged launch");
    return;
  }
  const unsigned grid = static_cast<unsigned>(ends.w < 148ull * 2048 ? (ends.w + 255) / 256 : 148 * 8);
  if (idx_bytes == 4)
    gather_xy4<<<grid, 256, 0, stream>>>(pts, static_cast<const std::uint32_t*>(d_queues), cap,
                                         ends, reinterpret_cast<double2*>(d_out));
  else
    gather_xy4<<<grid, 256, 0, stream>>>(pts, static_cast<const std::uint64_t*>(d_queues), cap,
                                         ends, reinterpret_cast<double2*>(d_out));
  check_cuda(cudaGetLastError(), "gather_xy4 launch");
}

void launch_gather4_dev(const double* d_xy, const void* d_queues, int idx_bytes,
                        std::uint64_t cap, const unsigned long long* d_counts,
                        std::uint64_t limit, double* d_out, cudaStream_t stream) {
  const auto* pts = reinterpret_cast<const double2*>(d_xy);
  const unsigned grid = static_cast<unsigned>((limit + 255) / 256);
  if (idx_bytes == 4)
    gather_xy4_dev<<<grid, 256, 0, stream>>>(pts, static_cast<const std::uint32_t*>(d_queues),
                                             cap, d_counts, limit,
                                             reinterpret_cast<double2*>(d_out));
  else
    gather_xy4_dev<<<grid, 256, 0, stream>>>(pts, static_cast<const std::uint64_t*>(d_queues),
                                             cap, d_counts, limit,
                                             reinterpret_cast<double2*>(d_out));
  check_cuda(cudaGetLastError(), "gather_xy4_dev launch");
}

void launch_hull_indices(const double* d_xy, const void* d_queues, int idx_bytes,
                         std::uint64_t cap, const std::uint64_t counts[4], std::uint64_t base,
                         const double* d_hull, std::uint64_t h, std::uint32_t* d_slots,
                         std::uint64_t nslots, unsigned long long* d_res, cudaStream_t stream) {
  const auto* hull = reinterpret_cast<const double2*>(d_hull);
  check_cuda(cudaMemsetAsync(d_slots, 0xff, nslots * 4, stream), "cudaMemsetAsync(slots)");
  check_cuda(cudaMemsetAsync(d_res, 0xff, h * 8, stream), "cudaMemsetAsync(hull indices)");
  hidx_insert<<<static_cast<unsigned>((h + 255) / 256), 256, 0, stream>>>(hull, h, d_slots,
                                                                         nslots - 1);
  check_cuda(cudaGetLastError(), "hidx_insert launch");
  const ulonglong4 ends = make_ulonglong4(counts[0], counts[0] + counts[1],
                                          counts[0] + counts[1] + counts[2],
                                          counts[0] + counts[1] + counts[2] + counts[3]);
  if (ends.w == 0) return;
  const unsigned grid = static_cast<unsigned>(ends.w < 148ull * 2048 ? (ends.w + 255) / 256 : 148 * 8);
  const auto* pts = reinterpret_cast<const double2*>(d_xy);
  if (idx_bytes == 4)
    hidx_probe<<<grid, 256, 0, stream>>>(pts, static_cast<const std::uint32_t*>(d_queues), cap,
                                         ends, base, hull, d_slots, nslots - 1, d_res);
  else
    hidx_probe<<<grid, 256, 0, stream>>>(pts, static_cast<const std::uint64_t*>(d_queues), cap,
                                         ends, base, hull, d_slots, nslots - 1, d_res);
  check_cuda(cudaGetLastError(), "hidx_probe launch");
}

void launch_gather(const double* d_xy, const void* d_idx, int idx_bytes,
                   std::uint64_t count, double* d_out, cudaStream_t stream) {
  if (count == 0) return;
  const unsigned grid = static_cast<unsigned>(count < 148ull * 2048 ? (count + 255) / 256 : 148 * 8);
  const auto* pts = reinterpret_cast<const double2*>(d_xy);
  if (idx_bytes == 4)
    gather_xy<<<grid, 256, 0, stream>>>(pts, static_cast<const std::uint32_t*>(d_idx), count,
                                        reinterpret_cast<double2*>(d_out));
  else
    gather_xy<<<grid, 256, 0, stream>>>(pts, static_cast<const std::uint64_t*>(d_idx), count,
                                        reinterpret_cast<double2*>(d_out));
  check_cuda(cudaGetLastError(), "gather_xy launch");
}

// ---- small reads through mapped memory (see internal.hpp)
namespace {
struct SmallReadArgs {
  const unsigned char* src[8];
  std::uint32_t bytes[8], off[8];
  int k;
};
__global__ void small_reads_k(SmallReadArgs a, unsigned char* dst) {
  const int i = threadIdx.x;
  if (i >= a.k) return;
  for (std::uint32_t b = 0; b < a.bytes[i]; ++b) dst[a.off[i] + b] = a.src[i][b];
}
}  // namespace

const unsigned char* small_reads(const SmallRead* r, int k, cudaStream_t s) {
  if (k < 1 || k > 8) throw Error(OHX_E_INTERNAL, "small_reads: 1..8 values");
  struct Buf {
    unsigned char* h = nullptr;
    unsigned char* d = nullptr;
    ~Buf() {
      if (h) cudaFreeHost(h);
    }
  };
  thread_local Buf buf;
  if (!buf.h) {
    void* p = nullptr;
    check_cuda(cudaHostAlloc(&p, 1024, cudaHostAllocMapped | cudaHostAllocPortable),
               "cudaHostAlloc(small reads)");
    buf.h = static_cast<unsigned char*>(p);
    void* d = nullptr;
    check_cuda(cudaHostGetDevicePointer(&d, p, 0), "cudaHostGetDevicePointer");
    buf.d = static_cast<unsigned char*>(d);
  }
  SmallReadArgs a{};
  std::uint32_t off = 0;
  for (int i = 0; i < k; ++i) {
    if (r[i].bytes > 64) throw Error(OHX_E_INTERNAL, "small_reads: a value over 64 bytes");
    a.src[i] = static_cast<const unsigned char*>(r[i].src);
    a.bytes[i] = r[i].bytes;
    a.off[i] = off;
    off += (r[i].bytes + 7) / 8 * 8;
  }
  a.k = k;
  small_reads_k<<<1, 32, 0, s>>>(a, buf.d);
  check_cuda(cudaGetLastError(), "small_reads launch");
  return buf.h;
}

}  // namespace ohx

