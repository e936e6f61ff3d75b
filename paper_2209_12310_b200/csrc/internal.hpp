// internal.hpp -- declarations shared by the CUDA kernels (kernels.cu), the
// C ABI (capi.cpp), the host hull (hull.cpp) and the C++ API
// (octohull_api.cpp).  Not installed; the public surfaces are
// include/ohx.h and include/octohull/*.hpp.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <new>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ohx.h"

namespace ohx {

// Host worker teams for OpenMP regions: `want` threads, 1 in a forked child
// (the parent's OpenMP pool does not survive a fork; a child that used it
// would hang).  A fork handler also sets the child's default team to 1.
int team(int want);

// ---- kernel-side plan (K2): the C-ABI plan with shard-local kept indices
struct KPlan {
  double ax[8], ay[8], ea[8], ec[8];
  double qax[4], qay[4], qa[4], qc[4];
  double box[4];
  std::uint64_t kept[8];  // shard-local, ~0 when not in this shard
  std::uint32_t kept_label[8];
  std::int32_t m;
};

// per-block K1 partial (device scratch)
struct K1Partial {
  double key[8];
  std::uint64_t idx[8];
  double second[4];
};

// geometry of the K2 tiles (kernels.cu)
constexpr int kK2Block = 256;
constexpr int kK2Items = 8;
constexpr std::uint64_t kK2Tile = std::uint64_t(kK2Block) * kK2Items;

// Launchers (kernels.cu).  All asynchronous on `stream`.
int k1_grid(int device, std::uint64_t n);
void launch_k1(const double* d_xy, std::uint64_t n, std::uint64_t base,
               K1Partial* partials, int grid, unsigned* ticket,
               ohx_extremes_rec* d_out, cudaStream_t stream);
void launch_k1b(const double* d_xy, std::uint64_t n, std::uint64_t base,
                const double bbox[4], K1Partial* partials, int grid,
                unsigned* ticket, ohx_corner_rec* d_out, cudaStream_t stream);
// K2 work area: [2 counters | k2_compact look-back words (4 per group of 64
// tiles) | per-tile queue counts (4 x u32 per tile) | survivor scratch
// (one 16-bit slot per point)].  Only the first part is cleared per launch.
constexpr std::uint64_t kK2GroupTiles = 64;
struct K2Work {
  unsigned* tile_counter;
  unsigned* group_counter;
  std::uint64_t* status;
  std::uint32_t* tile_counts;
  std::uint16_t* scratch;
  std::uint64_t clear_bytes;
  std::uint64_t total_bytes;
};
inline K2Work k2_work_layout(void* base, std::uint64_t ntiles) {
  const std::uint64_t ngroups = (ntiles + kK2GroupTiles - 1) / kK2GroupTiles;
  auto* b = static_cast<unsigned char*>(base);
  K2Work w{};
  std::uint64_t off = 0;
  w.tile_counter = reinterpret_cast<unsigned*>(b + off);
  w.group_counter = reinterpret_cast<unsigned*>(b + off + 4);
  off += 256;
  w.status = reinterpret_cast<std::uint64_t*>(b + off);
  off += 4 * ngroups * 8;
  w.clear_bytes = off;
  off = (off + 255) & ~std::uint64_t(255);
  w.tile_counts = reinterpret_cast<std::uint32_t*>(b + off);
  off += 4 * ntiles * 4;
  off = (off + 255) & ~std::uint64_t(255);
  w.scratch = reinterpret_cast<std::uint16_t*>(b + off);
  off += ntiles * kK2Tile * 2;
  w.total_bytes = off;
  return w;
}
inline std::uint64_t k2_work_bytes(std::uint64_t ntiles) {
  return k2_work_layout(nullptr, ntiles).total_bytes;
}
// K2 (k2_filter + k2_compact; re-arms its work area first).  d_queues holds
// 4 queues of `cap` shard-local indices of idx_bytes each.
// d_gather (nullable): gather mode over a candidate list of n shard-local
// indices (same width as the queues); labels are then scattered.
// op (gather mode with d_gather_xy, at most kK2OnePassMaxTiles tiles): one
// launch that writes the queues, the survivors' coordinates (qxy[q * cap +
// i] for queue entry i of quadrant q) and, for the first spec_q of each
// quadrant, spec[q * spec_q + i], then the four counts after them
// (k2_one_pass_spec_bytes); d_counts is not written.  op->work
// (k2_one_pass_work_bytes) must be zero the first time -- the kernel leaves
// it zeroed.  Null: k2_filter + k2_compact.
constexpr std::uint64_t kK2OnePassMaxTiles = 2048;
struct K2OnePassBufs {
  void* work;
  double* qxy;
  double* spec;
  std::uint32_t spec_q;
};
inline std::uint64_t k2_one_pass_work_bytes() { return 256 + 4 * kK2OnePassMaxTiles * 8; }
inline std::uint64_t k2_one_pass_spec_bytes(std::uint32_t spec_q) { return 4ull * spec_q * 16 + 64; }
void launch_k2(const double* d_xy, std::uint64_t n, const KPlan& plan, void* d_work,
               std::uint64_t ntiles, void* d_queues, int idx_bytes, std::uint64_t cap,
               std::uint8_t* d_labels, unsigned long long* d_counts, cudaStream_t stream,
               const void* d_gather = nullptr, const double* d_gather_xy = nullptr,
               const K2OnePassBufs* op = nullptr);
// The fused pass's provisional region Q (heuristic; certified inside the
// true octagon after the pass): x0 <= x <= x1, y0 <= y <= y1,
// t0 <= fl(x+y) <= t1, d0 <= fl(x-y) <= d1.
struct KFRegion {
  double x0, x1, y0, y1, t0, t1, d0, d1;
};

// KF: blocks of the fused filter pass (occupancy-sized, one warp per range)
int kf_grid(int device);
constexpr int kKFWarpsPerBlock = 8;
// KF runs only if *d_gate >= gate_min (the sample's coverage count)
void launch_kf(const double* d_xy, std::uint64_t n, const KFRegion& q, int grid, void* d_regions,
               int idx_bytes, std::uint64_t cap_w, std::uint32_t* d_warp_counts,
               const unsigned long long* d_gate, std::uint64_t gate_min, cudaStream_t stream);
// the first cap_c candidates (ordered) and their coordinates; d_counts[0] =
// candidates, [1] = 1 if some warp region overflowed, [2] = *d_gate
void launch_kf_gather(const double* d_xy, const void* d_regions, int idx_bytes,
                      std::uint64_t cap_w, const std::uint32_t* d_warp_counts, std::uint64_t nw,
                      const unsigned long long* d_gate, unsigned long long* d_counts,
                      void* d_cand, double* d_cpts, std::uint64_t cap_c, cudaStream_t stream);
// K1 over the provisional region's sample, read in place: `segs` runs of
// `len` points at evenly spaced offsets, run b belonging to sub-sample
// b % subs; one record per sub-sample (global indices).  Partials: subs x
// (segs / subs) entries, tickets: subs.
// *d_count (the coverage counter of launch_count_in_region) is zeroed.
void launch_k1_sample(const double* d_xy, std::uint64_t n, int segs, int len, int subs,
                      K1Partial* partials, unsigned* ticket, ohx_extremes_rec* d_recs,
                      unsigned long long* d_count, cudaStream_t stream);
// K1 over a short contiguous list (the fused pass's candidates)
int k1_list_grid(std::uint64_t n);
// (n capped by *d_n when d_n is set: a length counted on the device; the
// record's indices are d_map[i] + map_base when d_map is set -- map_bytes 4
// or 8 -- else positions in the list)
void launch_k1_list(const double* d_xy, std::uint64_t n, const unsigned long long* d_n,
                    const void* d_map, int map_bytes, std::uint64_t map_base,
                    K1Partial* partials, int grid, unsigned* ticket, ohx_extremes_rec* d_rec,
                    cudaStream_t stream);
// points of the sample runs 0, step, 2 step, ... inside Q, added to
// *d_count (zeroed by launch_k1_sample)
void launch_count_in_region(const double* d_xy, std::uint64_t n, int segs, int len, int step,
                            const KFRegion& q, unsigned long long* d_count, cudaStream_t stream);
// labels of classify_points against a polygon of m > 8 vertices: d_edges =
// m x {a.x, a.y, fl(b.x-a.x), fl(b.y-a.y)}; kept overrides and find_queue
// edges from plan (its own octagon part unused)
void launch_polygon_labels(const double* d_xy, std::uint64_t n, const double* d_edges, int m,
                           const KPlan& plan, std::uint8_t* d_labels, cudaStream_t stream);
// *d_first = the smallest index with a non-finite coordinate, else ~0
void launch_first_nonfinite(const double* d_xy, std::uint64_t n, unsigned long long* d_first,
                            cudaStream_t stream);
// n (the shard's points, optional): large, dense survivor sets are
// gathered by index range (one read of each line)
void launch_gather4(const double* d_xy, const void* d_queues, int idx_bytes,
                    std::uint64_t cap, const std::uint64_t counts[4], double* d_out,
                    cudaStream_t stream, std::uint64_t n = 0);
void launch_gather(const double* d_xy, const void* d_idx, int idx_bytes,
                   std::uint64_t count, double* d_out, cudaStream_t stream);
// hull vertices -> smallest survivor index (+ base) with equal coordinates
// (d_res, ~0 where none; nslots a power of two >= 2h)
void launch_hull_indices(const double* d_xy, const void* d_queues, int idx_bytes,
                         std::uint64_t cap, const std::uint64_t counts[4], std::uint64_t base,
                         const double* d_hull, std::uint64_t h, std::uint32_t* d_slots,
                         std::uint64_t nslots, unsigned long long* d_res, cudaStream_t stream);
// the first `limit` survivors' coordinates with the counts read on the device
void launch_gather4_dev(const double* d_xy, const void* d_queues, int idx_bytes,
                        std::uint64_t cap, const unsigned long long* d_counts,
                        std::uint64_t limit, double* d_out, cudaStream_t stream);

// ---- host helpers (capi.cpp)
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
void check_cuda(cudaError_t e, const char* what);
// thread-local message returned by ohx_last_error()
void set_last_error(const char* msg);

// Runs f() and maps exceptions to the C ABI's status codes; nothing ever
// propagates across the extern "C" boundary.
template <typename F>
int guard(F&& f) {
  try {
    f();
    return OHX_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return OHX_E_INVALID;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return OHX_E_NOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return OHX_E_INTERNAL;
  } catch (...) {
    set_last_error("unknown exception");
    return OHX_E_INTERNAL;
  }
}

// ---- host hull (hull.cpp), semantics of hull.cpp:18-150 of the reference
struct P2 {
  double x, y;
};
// A std::vector whose resize leaves new elements default-initialised: the
// hull stage's buffers (up to ~1.6 GB) are written once, in parallel, with
// no zero-fill pass over freshly mapped pages first.
// Blocks of >= kBigBlock bytes come from big_alloc: 2 MB aligned, marked
// for transparent huge pages (the box runs THP in madvise mode: 4 KB pages
// would fault ~400K times per GB) and recycled through a small cache, so
// the hull stage's GB-sized buffers are not re-faulted on every call.
constexpr std::size_t kBigBlock = std::size_t(64) << 20;
void* big_alloc(std::size_t bytes);
void big_free(void* p, std::size_t bytes) noexcept;
void big_cache_trim() noexcept;  // frees the recycled blocks

template <class T>
struct DefaultInitAlloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = DefaultInitAlloc<U>;
  };
  DefaultInitAlloc() noexcept = default;
  template <class U>
  DefaultInitAlloc(const DefaultInitAlloc<U>&) noexcept {}
  T* allocate(std::size_t n) {
    if (n * sizeof(T) >= kBigBlock) return static_cast<T*>(big_alloc(n * sizeof(T)));
    return std::allocator<T>::allocate(n);
  }
  void deallocate(T* p, std::size_t n) noexcept {
    if (n * sizeof(T) >= kBigBlock) big_free(p, n * sizeof(T));
    else std::allocator<T>::deallocate(p, n);
  }
  template <class U>
  void construct(U* p) noexcept {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
  }
};
using PVec = std::vector<P2, DefaultInitAlloc<P2>>;
// Parallel copy of n points (OpenMP above a size threshold)
void copy_points(P2* dst, const P2* src, std::size_t n);

PVec quadrant_chain(std::vector<P2> pts, int quadrant);
// wait_arc(q): called before arc q is read (the arcs may still be arriving
// from the device); false = its input will never arrive (the stage throws)
using ArcWait = std::function<bool(int)>;
// chain of an arc already in sweep order (the arc's last point dropped)
PVec chain_sorted(const P2* pts, std::size_t n);
// the four arcs' chains concatenated (the cycle of hull.cpp:164-183)
PVec chain_arcs(const P2* const arcs[4], const std::uint64_t len[4],
                const ArcWait& wait_arc);
// The hull stage's sweep sort on the device (hullsort.cu): the four arcs
// [anchor q, queue q (packed [q1|q2|q3|q4] coordinates), anchor q+1], each
// sorted in its quadrant's sweep order, written back to back to d_sorted
// (sum(counts) + 8 points).
std::size_t sort_arcs_work_bytes(const std::uint64_t counts[4]);
// only_q >= 0: arc only_q is the one that must come out sorted (the others
// may or may not be; the layout is the same).
void sort_arcs(const double* d_packed, const std::uint64_t counts[4], const double anchors[8],
               void* d_work, double* d_sorted, cudaStream_t s, int only_q = -1);
// The chains and the cycle scan on the device (hullchain.cu) over the sorted
// arcs (the layout sort_arcs writes; len[q] = counts[q] + 2).  false: the
// chunked replay could not prove every chunk (the host chains must run);
// true: the cycle (the four chains, each without its last point) is in
// d_cycle, with the statistics finalize_cycle's fast path needs.
struct DeviceCycle {
  double* d_cycle = nullptr;
  double* d_scratch = nullptr;  // room for a copy of the cycle (when d_cycle is the caller's)
  std::uint64_t m = 0, best = 0, bad = 0;
  std::uint32_t chunks = 0;
  bool front_eq_back = false, dups = false, flat = false;
  int launches = 0;
};
std::size_t device_chain_work_bytes(const std::uint64_t len[4]);
// direct (nullable): the caller's device output; the cycle is written there
// when direct_cap covers every arc point.
// Small device -> host reads that must not queue behind a bulk copy on the
// copy engine (the pipelined hull stage streams the hull to the host while
// the next arc is sorted and chained): one kernel stores up to 8 values
// (<= 64 bytes each) into mapped pinned memory; the returned host view, the
// values at 8-byte aligned offsets in order, is valid once s is
// synchronised (until the calling thread's next small_reads).
struct SmallRead {
  const void* src;
  std::uint32_t bytes;
};
const unsigned char* small_reads(const SmallRead* r, int k, cudaStream_t s);
// The cycle statistics alone, for a cycle of m points assembled elsewhere
// (d_work: a device_chain_work_bytes(len) area; out->d_cycle / m set too).
void device_cycle_stats(const double* d_cycle, std::uint64_t m, const std::uint64_t len[4],
                        void* d_work, cudaStream_t s, DeviceCycle* out);
// only_q >= 0: arc only_q's chain alone (its chunks only; no statistics).
bool device_chains(const double* d_sorted, const std::uint64_t len[4], void* d_work,
                   cudaStream_t s, DeviceCycle* out, double* direct = nullptr,
                   std::uint64_t direct_cap = 0, int only_q = -1);
// hull stage from the four arcs [anchor q, queue q, anchor q+1] already in
// sweep order (device-sorted)
// (wait_arc(q), when set, is called by arc q's thread before it reads the
// arc: the arcs may still be arriving from the device)
PVec hull_from_sorted_arcs(const P2* const arcs[4], const std::uint64_t len[4],
                           const ArcWait& wait_arc = {});
// Same, the hull written to sink(h) (it returns where h vertices go and may
// throw; it may first be called with a larger size -- the chained cycle
// before its clean-up -- the last call's size is the hull's); returns h.
using HullSink = std::function<P2*(std::size_t)>;
std::size_t hull_from_sorted_arcs(const P2* const arcs[4], const std::uint64_t len[4],
                                  const ArcWait& wait_arc, const HullSink& sink);
PVec finalize_cycle(PVec cycle);
PVec hull_from_queue_points(const P2 anchors[4], const P2* const q_pts[4],
                            const std::uint64_t q_len[4]);
PVec monotone_chain(const P2* pts, std::uint64_t n);
int orient(const P2& a, const P2& b, const P2& c);

// ---- point files (io.cpp)
[[noreturn]] void io_fail(const std::string& path, const std::string& what);
// validated PTS2 header -> point count (reference io.cpp:87-107 messages)
std::uint64_t pts2_count(const std::string& path);
std::string nonfinite_message(std::uint64_t i);

// ---- host generator (pointgen.cpp)
void generate_points(int dist, std::uint64_t n, std::uint64_t seed,
                     double distort_pct, double* xy, int threads);
// points [lo, lo + cnt) of the same n-point corpus (a shard's slice)
void generate_points_range(int dist, std::uint64_t n, std::uint64_t seed, double distort_pct,
                           std::uint64_t lo, std::uint64_t cnt, double* xy, int threads);

}  // namespace ohx
