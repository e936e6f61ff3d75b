// host.hpp -- shared by the host-side translation units of the library
// (context.cpp, plan.cpp, device.cpp, capi.cpp): the device context and its
// workspaces, the plan geometry, and the fused pass's two halves.
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "internal.hpp"
#include "ohx.h"
#include "pipeline.hpp"

// ====================================================================== ctx
// d_rec / h_rec blocks: the extremes record, then 8 count words
constexpr std::size_t kRecCountsOff = (sizeof(ohx_extremes_rec) + 63) / 64 * 64;
constexpr std::size_t kRecBlock = kRecCountsOff + 64;
inline unsigned long long* rec_counts(ohx_extremes_rec* r) {
  return reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(r) + kRecCountsOff);
}

struct ohx_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  std::uint64_t launches = 0;

  // K1 / K1b scratch
  int partial_cap = 0;
  ohx::K1Partial* d_partials = nullptr;
  unsigned* d_ticket = nullptr;
  ohx_extremes_rec* d_rec = nullptr;
  ohx_corner_rec* d_crec = nullptr;
  ohx_extremes_rec* h_rec = nullptr;  // pinned
  ohx_extremes_rec* h_srec = nullptr;  // pinned: the fused pass's sub-sample records
  ohx_corner_rec* h_crec = nullptr;   // pinned
  unsigned long long* d_counts = nullptr;  // 8 words right after d_rec (kRecBlock)
  unsigned long long* h_counts = nullptr;  // pinned, right after h_rec

  // K2 scratch and queues
  std::uint64_t* d_status = nullptr;
  std::uint64_t status_bytes = 0;
  void* d_queues = nullptr;
  std::uint64_t queue_bytes = 0;

  // result of the last ohx_filter
  const double* last_xy = nullptr;
  std::uint64_t last_n = 0, last_base = 0, last_cap = 0;
  int last_idx_bytes = 4;
  std::uint64_t last_counts[4] = {0, 0, 0, 0};

  // host threads the current call may use for staging copies (0 = all):
  // the C++ API sets it to the caller's ReduceEngine workers -- the host
  // lanes the reference grants a call (parallel.hpp:18-21)
  int host_lanes = 0;
  bool spec_zeroed = false;  // d_gather's speculative survivor slots are cleared
  // d_gather holds the last filter's survivor coordinates per quadrant
  // (one-pass K2: entry i of quadrant q at q * last_cap + i)
  bool qxy_valid = false;
  // ohx_heaphull_device_out's buffer, for the duration of that call: the
  // device hull stage writes its cycle there directly
  double* dev_out = nullptr;
  std::uint64_t dev_out_cap = 0;
  // ... and a C-ABI call's host output buffer: the pipelined hull stage
  // streams the hull into it when it is page-locked
  double* host_out = nullptr;
  std::uint64_t host_out_cap = 0;
  // one-pass K2: its self-clearing work words and the small block it
  // returns (the first survivors' coordinates + the counts)
  void* d_k2op = nullptr;
  std::uint64_t k2op_bytes = 0;
  double* d_spec = nullptr;
  std::uint64_t dspec_bytes = 0;
  void* d_poly = nullptr;    // classify_points' edges of a polygon with > 8 vertices
  std::uint64_t poly_bytes = 0;
  // staging for host-API calls
  double* d_pts = nullptr;
  std::uint64_t pts_bytes = 0;
  std::uint8_t* d_labels = nullptr;
  std::uint64_t labels_bytes = 0;
  double* d_gather = nullptr;
  std::uint64_t gather_bytes = 0;
  // the first survivors' coordinates, fetched with the K2 counts (pinned):
  // valid for the last filter when spec_n != ~0 (how many are there)
  static constexpr std::uint64_t kSpecSurvivors = 4096;
  double* h_spec = nullptr;
  std::uint64_t spec_bytes = 0;
  std::uint64_t spec_n = ~0ull;

  // fused single-pass mode: sample, candidate list, coverage counter
  double* d_sample = nullptr;
  std::uint64_t sample_bytes = 0;
  void* d_cand = nullptr;
  std::uint64_t cand_bytes = 0;
  void* d_regions = nullptr;  // KF per-warp candidate regions
  std::uint64_t regions_bytes = 0;
  double* d_cpts = nullptr;  // gathered candidate coordinates
  std::uint64_t cpts_bytes = 0;
  void* d_hsort = nullptr;  // hull stage: device sweep sort work + sorted arcs
  std::uint64_t hsort_bytes = 0;
  void* d_hchain = nullptr;  // hull stage: device chains work + cycle
  std::uint64_t hchain_bytes = 0;
  void* h_sorted = nullptr;  // pinned: the sorted arcs on the host
  std::uint64_t h_sorted_bytes = 0;
  void* h_packed = nullptr;  // pinned: a small survivor set's coordinates for the host hull
  std::uint64_t h_packed_bytes = 0;
  cudaEvent_t arc_ev[4] = {};  // their per-arc copies
  // the pipelined hull stage: the whole cycle on the device, a copy stream
  // and one event per arc
  double* d_cycfull = nullptr;
  std::uint64_t cycfull_bytes = 0;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t pipe_ev[4] = {};
  unsigned long long* d_cnt = nullptr;
  unsigned long long* h_cnt = nullptr;  // pinned

  ohx_run_info last_run = {};

  // the last fused pass (fused_begin) awaiting its fused_finish
  struct {
    bool active = false;
    ohx::KFRegion q{};
    const double* d_xy = nullptr;
    std::uint64_t n = 0, base = 0, n_cand = 0;
  } fz;
  std::uint64_t cand_hint = 0;  // candidates of the last fused pass (sizes the next K1 grid)

  // pinned staging ring for host copies of pageable user buffers
  static constexpr int kStageBufs = 4;
  void* h_stage[kStageBufs] = {};
  cudaEvent_t stage_ev[kStageBufs] = {};

  // CUDA events bracketing the last launch of each stage: K1 (or KF), K1b,
  // K2, and the fused path's candidate stage (compaction + candidate K1)
  cudaEvent_t ev[4][2] = {};
  bool timed[4] = {false, false, false, false};
  // running sums of those stage times over calls (folded once per call when
  // its events have completed; read and reset by ohx_ctx_kernel_ms_sum)
  bool folded[4] = {true, true, true, true};
  double ksum[4] = {0, 0, 0, 0};
  std::uint64_t kcnt[4] = {0, 0, 0, 0};
};

namespace ohx {

// OHX_TRACE=1: host wall time of each pipeline phase on stderr
// OHX_TRACE=1: stage marks on stderr; OHX_TRACE=2: sub-stage marks too
inline int trace_level() {
  static const int v = [] {
    const char* e = std::getenv("OHX_TRACE");
    return e && *e ? std::atoi(e) : 0;
  }();
  return v;
}
struct Trace {
  bool on = trace_level() >= 1;
  void fine(const char* what) {
    if (trace_level() >= 2) mark(what);
  }
  // one timeline per thread: a mark measures from the previous mark of any
  // Trace (OHX_TRACE=2), or of this one (OHX_TRACE=1)
  static std::chrono::steady_clock::time_point& last() {
    thread_local std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    return t;
  }
  std::chrono::steady_clock::time_point t =
      trace_level() >= 2 ? last() : std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    const auto from = trace_level() >= 2 ? last() : t;
    std::fprintf(stderr, "[ohx] %-14s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - from).count());
    t = last() = std::chrono::steady_clock::now();  // the print itself not counted
  }
};

// ---- stage timing (device.cpp)
void mark_timed(ohx_ctx* c, int k);
void fold_stage_times(ohx_ctx* c, bool wait);

// ---- context workspaces (context.cpp)
const char* last_error();  // this thread's last error message
// grow-only device buffer; true when (re)allocated
bool dev_grow(void** p, std::uint64_t* have, std::uint64_t need, const char* what);
// the survivor gather buffer (ohx_ctx::d_gather); a new allocation is not
// yet cleared for the fixed-size speculative survivor copy
inline void grow_gather(ohx_ctx* c, std::uint64_t bytes) {
  if (dev_grow(reinterpret_cast<void**>(&c->d_gather), &c->gather_bytes, bytes, "gather")) {
    c->spec_zeroed = false;
    c->qxy_valid = false;
  }
}
void host_grow(void** p, std::uint64_t* have, std::uint64_t need, const char* what);
// page-locked (or registered) host memory: copies to / from it are direct DMA
bool is_pinned(const void* h);
// device -> host copy of a user buffer (pageable: through the pinned ring);
// returns when the bytes have landed
void copy_d2h(ohx_ctx* c, void* h, const void* d, std::uint64_t bytes, cudaStream_t s);
cudaStream_t pick(ohx_ctx* c, void* s);
void bind(ohx_ctx* c);
void ensure_partials(ohx_ctx* c, int grid);
std::uint64_t load_pts2_device(ohx_ctx* c, const std::string& path, double* d_xy,
                               std::uint64_t cap, cudaStream_t s);

// ---- hull stage on the device (device.cpp)
bool device_chain_mode();
bool hull_device_chains(ohx_ctx* c, const double* d_sorted, const std::uint64_t len[4],
                        cudaStream_t s, const HullSink& sink, std::size_t* h,
                        bool raw = false, bool dev = false);

// ---- plan geometry (plan.cpp)
bool certify_corner(const ohx_extremes_rec& r, int k);
void fit_box(const double* oct, int m, const double* ea, const double* ec, double box[4]);
bool region_certified(const ohx_filter_plan& plan, const KFRegion& q);
bool in_region_host(const KFRegion& q, double x, double y);
void clip_left(const std::vector<P2>& poly, P2 a, P2 b, std::vector<P2>& out);
bool fit_region(const std::vector<P2>& R, const double lim[8], KFRegion* q);

// ---- the fused pass (device.cpp)
bool fused_begin(ohx_ctx* c, const double* d_xy, std::uint64_t n, std::uint64_t base,
                 FilterOut& f, ohx_extremes_rec* rec, cudaStream_t s, Trace& tr);
void fused_finish(ohx_ctx* c, const double* d_xy, std::uint64_t n, std::uint64_t base,
                  const ohx_extreme_set& ext, const ohx_filter_plan& plan,
                  std::uint8_t* d_labels, std::uint64_t counts[4], FilterOut& f,
                  cudaStream_t s);

}  // namespace ohx
