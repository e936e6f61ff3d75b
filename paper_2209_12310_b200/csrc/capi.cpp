// capi.cpp -- the C ABI of include/ohx.h: device contexts and workspaces,
// kernel orchestration, and the small host-side steps between the kernels
// (extremes combine + corner certificate, build_octagon, the K2 plan with
// its certified interior box).
//
// Host arithmetic that must match the reference (orientation, manhattan,
// edge constants) is plain binary64 in a TU built with -ffp-contract=off
// and no -march, like the reference objects.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <unistd.h>

#include <omp.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "internal.hpp"
#include "ohx.h"
#include "pipeline.hpp"

// ====================================================================== ctx
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
  ohx_corner_rec* h_crec = nullptr;   // pinned
  unsigned long long* d_counts = nullptr;
  unsigned long long* h_counts = nullptr;  // pinned

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

  // staging for host-API calls
  double* d_pts = nullptr;
  std::uint64_t pts_bytes = 0;
  std::uint8_t* d_labels = nullptr;
  std::uint64_t labels_bytes = 0;
  double* d_gather = nullptr;
  std::uint64_t gather_bytes = 0;

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
  void* h_sorted = nullptr;  // pinned: the sorted arcs on the host
  std::uint64_t h_sorted_bytes = 0;
  cudaEvent_t arc_ev[4] = {};  // their per-arc copies
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

  // pinned staging ring for host copies of pageable user buffers
  static constexpr int kStageBufs = 4;
  void* h_stage[kStageBufs] = {};
  cudaEvent_t stage_ev[kStageBufs] = {};

  // CUDA events bracketing the last launch of each stage: K1 (or KF), K1b,
  // K2, and the fused path's candidate stage (compaction + candidate K1)
  cudaEvent_t ev[4][2] = {};
  bool timed[4] = {false, false, false, false};
};

namespace ohx {
namespace {

void dev_grow(void** p, std::uint64_t* have, std::uint64_t need, const char* what) {
  if (*have >= need && *p) return;
  if (*p) check_cuda(cudaFree(*p), "cudaFree");
  *p = nullptr;
  *have = 0;
  cudaError_t e = cudaMalloc(p, need);
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(OHX_E_NOMEM, std::string("cudaMalloc(") + what + ", " +
                                 std::to_string(need) + " bytes) failed: " +
                                 cudaGetErrorString(e));
  }
  *have = need;
}

cudaStream_t pick(ohx_ctx* c, void* s) {
  return s ? static_cast<cudaStream_t>(s) : c->stream;
}

void bind(ohx_ctx* c) { check_cuda(cudaSetDevice(c->device), "cudaSetDevice"); }

void ensure_partials(ohx_ctx* c, int grid) {
  if (grid <= c->partial_cap) return;
  if (c->d_partials) check_cuda(cudaFree(c->d_partials), "cudaFree");
  c->d_partials = nullptr;
  check_cuda(cudaMalloc(&c->d_partials, sizeof(K1Partial) * grid), "cudaMalloc(partials)");
  c->partial_cap = grid;
}

// Corner certificate (SURVEY §7 hard part 1).  For corner slot k with
// signs (sx, sy) every point of the bounding box satisfies
//   manhattan(p, corner) = C - s_p,  C = sx*cx + sy*cy,  s_p = sx*x + sy*y
// exactly in the reals; K1 maximised t_p = fl(s_p).  With u = 2^-53 and
// t2 the second-largest t, every p other than the winner has
//   s_p <= t2 + u/(1-u)|t2|   and   fl-manhattan(p) >= (C - s_p)(1-u)^2,
// so the winner is the unique reference argmin whenever its exact
// reference key is below (C - t2 - u'|t2|)(1 - 2u).  Evaluated in long
// double with an extra 2^-60 relative slack.
bool certify_corner(const ohx_extremes_rec& r, int k) {
  static const int sx[4] = {1, -1, -1, 1};
  static const int sy[4] = {1, 1, -1, -1};
  const double cx = sx[k] > 0 ? r.x[OHX_EAST] : r.x[OHX_WEST];
  const double cy = sy[k] > 0 ? r.y[OHX_NORTH] : r.y[OHX_SOUTH];
  const double t2 = r.second[k];
  if (std::isinf(t2) && t2 < 0) return true;  // a single point: nothing to beat
  const double m1 = std::abs(r.x[4 + k] - cx) + std::abs(r.y[4 + k] - cy);
  const long double u = 0x1p-53L;
  const long double C = static_cast<long double>(sx[k]) * cx +
                        static_cast<long double>(sy[k]) * cy;
  const long double g = C - static_cast<long double>(t2) -
                        (u / (1.0L - u)) * std::fabs(static_cast<long double>(t2));
  const long double scale = std::fabs(static_cast<long double>(cx)) +
                            std::fabs(static_cast<long double>(cy)) +
                            std::fabs(static_cast<long double>(t2));
  const long double bound = g * (1.0L - 2.0000001L * u) - 0x1p-60L * scale;
  return static_cast<long double>(m1) < bound;
}

// ------------------------------------------------ certified interior box --
// Each edge i (origin a, constants A = fl(b.x-a.x), C = fl(b.y-a.y)) has
// computed det = fl(fl(A*fl(p.y-a.y)) - fl(C*fl(p.x-a.x))) whose sign is that
// of P1 - P2 with |P1 - A(p.y-a.y)| <= g2|A||p.y-a.y| (g2 = 2u+u^2), same for
// P2.  det(p) >= E(p) - g2(|A||p.y-a.y| + |C||p.x-a.x|) with the exact affine
// E(p) = A(p.y-a.y) - C(p.x-a.x).  That lower bound is concave in p, so its
// minimum over a box sits at a corner: the box is certified when every
// corner c of it has E(c) > 8u(|A||c.y-a.y| + |C||c.x-a.x|) (8u > g2 leaves
// room for the long double evaluation), and then every point of the box has
// det > 0 on every edge.
// The search runs in double with a 16u margin (double evaluation of E is
// within ~4u of exact, so 16u in double implies > 8u exactly); the final
// box is re-verified in long double at 8u before it is used.
template <typename R>
struct EdgeT {
  R ax, ay, A, C;
};

template <typename R>
bool box_ok(const std::vector<EdgeT<R>>& edges, R x0, R x1, R y0, R y1, R factor) {
  if (!(x0 <= x1) || !(y0 <= y1)) return false;
  const R uf = factor * R(0x1p-53);
  const R xs[2] = {x0, x1}, ys[2] = {y0, y1};
  for (const EdgeT<R>& e : edges) {
    for (R cx : xs)
      for (R cy : ys) {
        const R dy = cy - e.ay, dx = cx - e.ax;
        const R E = e.A * dy - e.C * dx;
        const R margin = uf * (std::fabs(e.A) * std::fabs(dy) + std::fabs(e.C) * std::fabs(dx)) +
                         R(0x1p-1000);
        if (!(E > margin)) return false;
      }
  }
  return true;
}

// Fallback search: centred box, then the sides grown together.
void fit_box_ascent(const double* oct, int m, const double* ea, const double* ec,
                    double box[4]) {
  box[0] = 1.0;
  box[1] = 0.0;
  box[2] = 1.0;
  box[3] = 0.0;  // empty
  if (m < 3) return;
  std::vector<EdgeT<double>> edges;
  std::vector<EdgeT<long double>> edges_l;
  double vx0 = oct[0], vx1 = oct[0], vy0 = oct[1], vy1 = oct[1];
  double cx = 0, cy = 0;
  for (int i = 0; i < m; ++i) {
    edges.push_back({oct[2 * i], oct[2 * i + 1], ea[i], ec[i]});
    edges_l.push_back({oct[2 * i], oct[2 * i + 1], ea[i], ec[i]});
    vx0 = std::min(vx0, oct[2 * i]);
    vx1 = std::max(vx1, oct[2 * i]);
    vy0 = std::min(vy0, oct[2 * i + 1]);
    vy1 = std::max(vy1, oct[2 * i + 1]);
    cx += oct[2 * i];
    cy += oct[2 * i + 1];
  }
  cx /= m;
  cy /= m;
  const double hx = (vx1 - vx0) / 2, hy = (vy1 - vy0) / 2;
  auto ok = [&](const double* t) { return box_ok(edges, t[0], t[1], t[2], t[3], 16.0); };
  // 1) the largest centred box with the octagon's aspect ratio
  double b[4] = {cx - 1e-9 * hx, cx + 1e-9 * hx, cy - 1e-9 * hy, cy + 1e-9 * hy};
  if (!ok(b)) return;  // sliver octagon: no certified box, every point takes the full test
  double lo = 0, hi = 1;
  for (int it = 0; it < 24; ++it) {
    const double s = (lo + hi) / 2;
    const double t[4] = {cx - s * hx, cx + s * hx, cy - s * hy, cy + s * hy};
    if (ok(t)) lo = s;
    else hi = s;
  }
  b[0] = cx - lo * hx;
  b[1] = cx + lo * hx;
  b[2] = cy - lo * hy;
  b[3] = cy + lo * hy;
  // 2) grow the sides together: each round moves every side part of the
  //    way to the furthest position it could reach alone, so no side pins a
  //    corner early (a greedy one-side-at-a-time push gets stuck on
  //    near-flat octagon edges); the last round takes the full step
  const double lim[4] = {vx0, vx1, vy0, vy1};
  constexpr int kRounds = 6;
  for (int round = 0; round < kRounds; ++round) {
    const double step = round == kRounds - 1 ? 1.0 : 0.6;
    for (int side = 0; side < 4; ++side) {
      double good = b[side], bad = lim[side];
      for (int it = 0; it < 20; ++it) {
        double t[4] = {b[0], b[1], b[2], b[3]};
        t[side] = (good + bad) / 2;
        if (ok(t)) good = t[side];
        else bad = t[side];
      }
      b[side] += step * (good - b[side]);
    }
  }
  // certify the exact double box in long double before using it
  if (box_ok<long double>(edges_l, b[0], b[1], b[2], b[3], 8.0L)) std::memcpy(box, b, sizeof(b));
}

// Horizontal chord [left, right] of the convex polygon at height y.
bool chord(const double* oct, int m, double y, double& left, double& right) {
  left = INFINITY;
  right = -INFINITY;
  for (int i = 0; i < m; ++i) {
    const int j = i + 1 == m ? 0 : i + 1;
    const double ax = oct[2 * i], ay = oct[2 * i + 1], bx = oct[2 * j], by = oct[2 * j + 1];
    if (ay == by) {
      if (y == ay) {
        left = std::min(left, std::min(ax, bx));
        right = std::max(right, std::max(ax, bx));
      }
      continue;
    }
    if (y < std::min(ay, by) || y > std::max(ay, by)) continue;
    const double x = ax + (y - ay) * (bx - ax) / (by - ay);
    left = std::min(left, x);
    right = std::max(right, x);
  }
  return left <= right;
}

// The certified interior box: the largest-area axis-aligned rectangle in the
// (convex) octagon -- for heights y0 < y1 the widest rectangle spans the
// intersection of the two chords -- found by a grid search over (y0, y1)
// and a local refinement, then pulled inwards until box_ok certifies it.
// Area is the coverage proxy (exact for uniform data, near-centred boxes for
// normal data).  Falls back to fit_box_ascent.
void fit_box(const double* oct, int m, const double* ea, const double* ec, double box[4]) {
  box[0] = 1.0;
  box[1] = 0.0;
  box[2] = 1.0;
  box[3] = 0.0;  // empty
  if (m < 3) return;
  double vy0 = oct[1], vy1 = oct[1], vx0 = oct[0], vx1 = oct[0];
  for (int i = 1; i < m; ++i) {
    vy0 = std::min(vy0, oct[2 * i + 1]);
    vy1 = std::max(vy1, oct[2 * i + 1]);
    vx0 = std::min(vx0, oct[2 * i]);
    vx1 = std::max(vx1, oct[2 * i]);
  }
  if (!(vy1 > vy0) || !(vx1 > vx0)) return;
  auto area = [&](double y0, double y1, double* b) {
    double l0, r0, l1, r1;
    if (!(y1 > y0) || !chord(oct, m, y0, l0, r0) || !chord(oct, m, y1, l1, r1)) return -1.0;
    b[0] = std::max(l0, l1);
    b[1] = std::min(r0, r1);
    b[2] = y0;
    b[3] = y1;
    return b[1] > b[0] ? (b[1] - b[0]) * (y1 - y0) : -1.0;
  };
  constexpr int G = 40;
  const double dy = (vy1 - vy0) / G;
  double gy[G + 1], gl[G + 1], gr[G + 1];
  for (int i = 0; i <= G; ++i) {
    gy[i] = i == G ? vy1 : vy0 + i * dy;
    if (!chord(oct, m, gy[i], gl[i], gr[i])) gl[i] = INFINITY, gr[i] = -INFINITY;
  }
  double best = -1, by0 = 0, by1 = 0, tmp[4];
  for (int i = 0; i <= G; ++i)
    for (int k = i + 1; k <= G; ++k) {
      const double w = std::min(gr[i], gr[k]) - std::max(gl[i], gl[k]);
      const double a = w > 0 ? w * (gy[k] - gy[i]) : -1.0;
      if (a > best) {
        best = a;
        by0 = gy[i];
        by1 = gy[k];
      }
    }
  // local refinement: shrinking pattern search on (y0, y1)
  for (double step = dy; step > (vy1 - vy0) * 1e-9; step *= 0.5) {
    for (bool moved = true; moved;) {
      moved = false;
      const double cand[4][2] = {{by0 - step, by1}, {by0 + step, by1}, {by0, by1 - step},
                                 {by0, by1 + step}};
      for (const auto& c : cand) {
        if (c[0] < vy0 || c[1] > vy1) continue;
        const double a = area(c[0], c[1], tmp);
        if (a > best) {
          best = a;
          by0 = c[0];
          by1 = c[1];
          moved = true;
        }
      }
    }
  }
  double b[4];
  if (best > 0 && area(by0, by1, b) > 0) {
    std::vector<EdgeT<double>> edges;
    std::vector<EdgeT<long double>> edges_l;
    for (int i = 0; i < m; ++i) {
      edges.push_back({oct[2 * i], oct[2 * i + 1], ea[i], ec[i]});
      edges_l.push_back({oct[2 * i], oct[2 * i + 1], ea[i], ec[i]});
    }
    const double ex = vx1 - vx0, ey = vy1 - vy0;
    for (double eps = 1e-12; eps < 1e-3; eps *= 8) {
      const double t[4] = {b[0] + eps * ex, b[1] - eps * ex, b[2] + eps * ey, b[3] - eps * ey};
      if (box_ok(edges, t[0], t[1], t[2], t[3], 16.0) &&
          box_ok<long double>(edges_l, t[0], t[1], t[2], t[3], 8.0L)) {
        std::memcpy(box, t, sizeof(t));
        return;
      }
    }
  }
  fit_box_ascent(oct, m, ea, ec, box);
}

}  // namespace

namespace {
thread_local std::string g_last_error;
}
void set_last_error(const char* msg) { g_last_error = msg; }

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    const int code = (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
                         ? OHX_E_NODEVICE
                         : (e == cudaErrorMemoryAllocation ? OHX_E_NOMEM : OHX_E_CUDA);
    throw Error(code, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

// =================================================== internal pipeline API
cudaStream_t ctx_stream(ohx_ctx* c) { return c->stream; }
std::mutex& ctx_mutex(ohx_ctx* c) { return c->mu; }
void ctx_bind(ohx_ctx* c) { bind(c); }

// ---- host <-> device copies of user buffers.  Page-locked memory is
// copied directly; pageable memory (std::vector, numpy: what the reference's
// API and bindings pass) would go through the driver's staging at ~11 GB/s,
// so it goes through the context's ring of pinned chunks instead: host
// threads copy chunk k into a pinned buffer while the copy engine moves
// chunk k-1 (PCIe-bound, ~55 GB/s).
constexpr std::uint64_t kStageChunk = 64ull << 20;  // bytes per pinned chunk
constexpr std::uint64_t kStageMin = 1ull << 20;     // smaller copies go direct

bool is_pinned(const void* h) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void ensure_stage(ohx_ctx* c) {
  if (c->h_stage[0]) return;
  for (int b = 0; b < ohx_ctx::kStageBufs; ++b) {
    check_cuda(cudaMallocHost(&c->h_stage[b], kStageChunk), "cudaMallocHost(staging)");
    check_cuda(cudaEventCreateWithFlags(&c->stage_ev[b], cudaEventDisableTiming),
               "cudaEventCreate(staging)");
  }
}

void host_memcpy(void* dst, const void* src, std::uint64_t bytes) {
  if (bytes < (8ull << 20)) {
    std::memcpy(dst, src, bytes);
    return;
  }
#pragma omp parallel
  {
    const int t = omp_get_thread_num(), nt = omp_get_num_threads();
    const std::uint64_t b = bytes * t / nt, e = bytes * (t + 1) / nt;
    std::memcpy(static_cast<char*>(dst) + b, static_cast<const char*>(src) + b, e - b);
  }
}

void copy_h2d(ohx_ctx* c, void* d, const void* h, std::uint64_t bytes, cudaStream_t s) {
  if (bytes < kStageMin || is_pinned(h)) {
    check_cuda(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s), "cudaMemcpyAsync(H2D)");
    return;
  }
  ensure_stage(c);
  const std::uint64_t chunks = (bytes + kStageChunk - 1) / kStageChunk;
  for (std::uint64_t k = 0; k < chunks; ++k) {
    const int b = static_cast<int>(k % ohx_ctx::kStageBufs);
    const std::uint64_t off = k * kStageChunk, len = std::min(kStageChunk, bytes - off);
    if (k >= ohx_ctx::kStageBufs)
      check_cuda(cudaEventSynchronize(c->stage_ev[b]), "cudaEventSynchronize(staging)");
    host_memcpy(c->h_stage[b], static_cast<const char*>(h) + off, len);
    check_cuda(cudaMemcpyAsync(static_cast<char*>(d) + off, c->h_stage[b], len,
                               cudaMemcpyHostToDevice, s), "cudaMemcpyAsync(H2D chunk)");
    check_cuda(cudaEventRecord(c->stage_ev[b], s), "cudaEventRecord(staging)");
  }
}

void copy_d2h(ohx_ctx* c, void* h, const void* d, std::uint64_t bytes, cudaStream_t s) {
  if (bytes < kStageMin || is_pinned(h)) {
    check_cuda(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync(D2H)");
    check_cuda(cudaStreamSynchronize(s), "D2H");
    return;
  }
  ensure_stage(c);
  const std::uint64_t chunks = (bytes + kStageChunk - 1) / kStageChunk;
  auto drain = [&](std::uint64_t k) {  // chunk k has been issued: copy it out
    const int b = static_cast<int>(k % ohx_ctx::kStageBufs);
    const std::uint64_t off = k * kStageChunk, len = std::min(kStageChunk, bytes - off);
    check_cuda(cudaEventSynchronize(c->stage_ev[b]), "cudaEventSynchronize(staging)");
    host_memcpy(static_cast<char*>(h) + off, c->h_stage[b], len);
  };
  for (std::uint64_t k = 0; k < chunks; ++k) {
    const int b = static_cast<int>(k % ohx_ctx::kStageBufs);
    if (k >= ohx_ctx::kStageBufs) drain(k - ohx_ctx::kStageBufs);
    const std::uint64_t off = k * kStageChunk, len = std::min(kStageChunk, bytes - off);
    check_cuda(cudaMemcpyAsync(c->h_stage[b], static_cast<const char*>(d) + off, len,
                               cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync(D2H chunk)");
    check_cuda(cudaEventRecord(c->stage_ev[b], s), "cudaEventRecord(staging)");
  }
  for (std::uint64_t k = chunks > ohx_ctx::kStageBufs ? chunks - ohx_ctx::kStageBufs : 0;
       k < chunks; ++k)
    drain(k);
}

// A PTS2 file straight into device memory: the payload
// streams through the pinned staging ring -- host threads pread chunk k
// while the copy engine moves chunk k-1 -- and a device scan finds the
// first non-finite point (reference io.cpp:87-124 semantics and messages).
std::uint64_t load_pts2_device(ohx_ctx* c, const std::string& path, double* d_xy,
                               std::uint64_t cap, cudaStream_t s) {
  const std::uint64_t n = pts2_count(path);
  if (n > cap) throw std::invalid_argument(path + ": " + std::to_string(n) +
                                           " points exceed the device buffer (" +
                                           std::to_string(cap) + ")");
  const int fd = ::open(path.c_str(), O_RDONLY);
  if (fd < 0) io_fail(path, "cannot open for reading");
  ensure_stage(c);
  const std::uint64_t bytes = 16 * n;
  const std::uint64_t chunks = (bytes + kStageChunk - 1) / kStageChunk;
  bool ok = true;
  for (std::uint64_t k = 0; k < chunks && ok; ++k) {
    const int b = static_cast<int>(k % ohx_ctx::kStageBufs);
    const std::uint64_t off = k * kStageChunk, len = std::min(kStageChunk, bytes - off);
    if (k >= ohx_ctx::kStageBufs)
      check_cuda(cudaEventSynchronize(c->stage_ev[b]), "cudaEventSynchronize(staging)");
    char* dst = static_cast<char*>(c->h_stage[b]);
#pragma omp parallel num_threads(len >= (16u << 20) ? 8 : 1) reduction(&& : ok)
    {
      const int t = omp_get_thread_num(), nt = omp_get_num_threads();
      std::uint64_t p = len * t / nt, e = len * (t + 1) / nt;
      while (p < e && ok) {
        const ssize_t r = ::pread(fd, dst + p, static_cast<std::size_t>(e - p),
                                  static_cast<off_t>(12 + off + p));
        if (r <= 0) ok = false;
        else p += static_cast<std::uint64_t>(r);
      }
    }
    if (!ok) break;
    check_cuda(cudaMemcpyAsync(reinterpret_cast<char*>(d_xy) + off, dst, len,
                               cudaMemcpyHostToDevice, s), "cudaMemcpyAsync(PTS2 chunk)");
    check_cuda(cudaEventRecord(c->stage_ev[b], s), "cudaEventRecord(staging)");
  }
  ::close(fd);
  if (!ok) {
    check_cuda(cudaStreamSynchronize(s), "PTS2 load");
    io_fail(path, "read error");
  }
  launch_first_nonfinite(d_xy, n, c->d_cnt, s);
  ++c->launches;
  check_cuda(cudaMemcpyAsync(c->h_cnt, c->d_cnt, 8, cudaMemcpyDeviceToHost, s),
             "cudaMemcpyAsync(non-finite)");
  check_cuda(cudaStreamSynchronize(s), "PTS2 load");
  if (*c->h_cnt < n) io_fail(path, nonfinite_message(*c->h_cnt));
  return n;
}

const double* stage_pts2(ohx_ctx* c, const std::string& path, std::uint64_t* n, cudaStream_t s) {
  const std::uint64_t count = pts2_count(path);
  dev_grow(reinterpret_cast<void**>(&c->d_pts), &c->pts_bytes, count * 16, "points");
  *n = load_pts2_device(c, path, c->d_pts, count, s);
  return c->d_pts;
}

const double* stage_points(ohx_ctx* c, const double* h_xy, std::uint64_t n,
                           cudaStream_t s) {
  const std::uint64_t bytes = n * 16;
  dev_grow(reinterpret_cast<void**>(&c->d_pts), &c->pts_bytes, bytes, "points");
  copy_h2d(c, c->d_pts, h_xy, bytes, s);
  return c->d_pts;
}

void fetch_labels(ohx_ctx* c, std::uint8_t* h_labels, const std::uint8_t* d_labels,
                  std::uint64_t n, cudaStream_t s) {
  copy_d2h(c, h_labels, d_labels, n, s);
}

std::uint8_t* stage_labels(ohx_ctx* c, std::uint64_t n) {
  dev_grow(reinterpret_cast<void**>(&c->d_labels), &c->labels_bytes, n, "labels");
  return c->d_labels;
}

void extremes(ohx_ctx* c, const double* d_xy, std::uint64_t n, std::uint64_t base,
              ohx_extremes_rec* out, cudaStream_t s) {
  if (n == 0) throw std::invalid_argument("find_axis_extremes: empty point set");
  const int grid = k1_grid(c->device, n);
  ensure_partials(c, grid);
  check_cuda(cudaEventRecord(c->ev[0][0], s), "cudaEventRecord");
  launch_k1(d_xy, n, base, c->d_partials, grid, c->d_ticket, c->d_rec, s);
  check_cuda(cudaEventRecord(c->ev[0][1], s), "cudaEventRecord");
  c->timed[0] = true;
  ++c->launches;
  check_cuda(cudaMemcpyAsync(c->h_rec, c->d_rec, sizeof(ohx_extremes_rec),
                             cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync(rec)");
  check_cuda(cudaStreamSynchronize(s), "k1_extremes");
  *out = *c->h_rec;
}

void corners_exact(ohx_ctx* c, const double* d_xy, std::uint64_t n,
                   std::uint64_t base, const double bbox[4], ohx_corner_rec* out,
                   cudaStream_t s) {
  if (n == 0) throw std::invalid_argument("find_corner_extremes: empty point set");
  const int grid = k1_grid(c->device, n);
  ensure_partials(c, grid);
  check_cuda(cudaEventRecord(c->ev[1][0], s), "cudaEventRecord");
  launch_k1b(d_xy, n, base, bbox, c->d_partials, grid, c->d_ticket, c->d_crec, s);
  check_cuda(cudaEventRecord(c->ev[1][1], s), "cudaEventRecord");
  c->timed[1] = true;
  ++c->launches;
  check_cuda(cudaMemcpyAsync(c->h_crec, c->d_crec, sizeof(ohx_corner_rec),
                             cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync(crec)");
  check_cuda(cudaStreamSynchronize(s), "k1b_corners");
  *out = *c->h_crec;
}

void combine_extremes(const ohx_extremes_rec* recs, int k, ohx_extremes_rec* out) {
  if (k < 1) throw std::invalid_argument("ohx_extremes_combine: no records");
  ohx_extremes_rec r = recs[0];
  for (int j = 1; j < k; ++j) {
    const ohx_extremes_rec& b = recs[j];
    for (int a = 0; a < 8; ++a) {
      if (a >= 4) {
        const double lo = std::min(r.key[a], b.key[a]);
        r.second[a - 4] = std::max(std::max(r.second[a - 4], b.second[a - 4]), lo);
      }
      if (b.key[a] > r.key[a] || (b.key[a] == r.key[a] && b.idx[a] < r.idx[a])) {
        r.key[a] = b.key[a];
        r.idx[a] = b.idx[a];
        r.x[a] = b.x[a];
        r.y[a] = b.y[a];
      }
    }
    r.n += b.n;
  }
  *out = r;
}

void combine_corners(const ohx_corner_rec* recs, int k, ohx_corner_rec* out) {
  if (k < 1) throw std::invalid_argument("ohx_corners_combine: no records");
  ohx_corner_rec r = recs[0];
  for (int j = 1; j < k; ++j) {
    const ohx_corner_rec& b = recs[j];
    for (int a = 0; a < 4; ++a) {
      if (b.key[a] < r.key[a] || (b.key[a] == r.key[a] && b.idx[a] < r.idx[a])) {
        r.key[a] = b.key[a];
        r.idx[a] = b.idx[a];
        r.x[a] = b.x[a];
        r.y[a] = b.y[a];
      }
    }
    r.n += b.n;
  }
  *out = r;
}

std::uint32_t resolve_extremes(const ohx_extremes_rec& r, ohx_extreme_set* out) {
  std::uint32_t mask = 0;
  for (int a = 0; a < 8; ++a) {
    out->ext[a] = r.idx[a];
    out->x[a] = r.x[a];
    out->y[a] = r.y[a];
  }
  for (int k = 0; k < 4; ++k)
    if (!certify_corner(r, k)) mask |= 1u << k;
  return mask;
}

void apply_corners(const ohx_corner_rec& c, ohx_extreme_set* ext) {
  for (int k = 0; k < 4; ++k) {
    ext->ext[4 + k] = c.idx[k];
    ext->x[4 + k] = c.x[k];
    ext->y[4 + k] = c.y[k];
  }
}

int build_octagon(const double cand[16], double oct[16]) {
  // reference filter.cpp:54-86: cyclic de-duplication, then repeatedly erase
  // the first vertex that does not turn strictly left
  std::vector<P2> cyc;
  for (int k = 0; k < 8; ++k) {
    const P2 p{cand[2 * k], cand[2 * k + 1]};
    if (cyc.empty() || cyc.back().x != p.x || cyc.back().y != p.y) cyc.push_back(p);
  }
  while (cyc.size() > 1 && cyc.front().x == cyc.back().x && cyc.front().y == cyc.back().y)
    cyc.pop_back();
  for (bool again = true; again && cyc.size() > 2;) {
    again = false;
    const std::size_t m = cyc.size();
    for (std::size_t i = 0; i < m; ++i) {
      const P2& a = cyc[(i + m - 1) % m];
      const P2& c = cyc[(i + 1) % m];
      if (orient(a, cyc[i], c) <= 0) {
        cyc.erase(cyc.begin() + static_cast<std::ptrdiff_t>(i));
        again = true;
        break;
      }
    }
  }
  for (std::size_t i = 0; i < cyc.size(); ++i) {
    oct[2 * i] = cyc[i].x;
    oct[2 * i + 1] = cyc[i].y;
  }
  return static_cast<int>(cyc.size());
}

void make_plan(const ohx_extreme_set& e, const double* oct, int m,
               ohx_filter_plan* p) {
  std::memset(p, 0, sizeof(*p));
  if (m < 0 || m > 8) throw std::invalid_argument("octagon must have 0..8 vertices");
  p->m = m;
  if (m >= 3) {
    for (int i = 0; i < m; ++i) {
      const int j = (i + 1 == m) ? 0 : i + 1;
      p->ax[i] = oct[2 * i];
      p->ay[i] = oct[2 * i + 1];
      p->ea[i] = oct[2 * j] - oct[2 * i];          // (b.x - a.x)
      p->ec[i] = oct[2 * j + 1] - oct[2 * i + 1];  // (b.y - a.y)
    }
  }
  // find_queue edges E->N, N->W, W->S, S->E (filter.cpp:94-97)
  const int from[4] = {OHX_EAST, OHX_NORTH, OHX_WEST, OHX_SOUTH};
  const int to[4] = {OHX_NORTH, OHX_WEST, OHX_SOUTH, OHX_EAST};
  for (int q = 0; q < 4; ++q) {
    p->qax[q] = e.x[from[q]];
    p->qay[q] = e.y[from[q]];
    p->qa[q] = e.x[to[q]] - e.x[from[q]];
    p->qc[q] = e.y[to[q]] - e.y[from[q]];
  }
  // kept overrides in the reference's first-match order (filter.cpp:108-117)
  const int slot[8] = {OHX_EAST, OHX_NE, OHX_NORTH, OHX_NW,
                       OHX_WEST, OHX_SW, OHX_SOUTH, OHX_SE};
  for (int k = 0; k < 8; ++k) {
    p->kept[k] = e.ext[slot[k]];
    p->kept_label[k] = static_cast<std::uint8_t>(1 + k / 2);
  }
  fit_box(oct, m, p->ea, p->ec, p->box);
}

namespace {

KPlan make_kplan(const ohx_filter_plan& plan, std::uint64_t base, std::uint64_t n) {
  KPlan kp;
  std::memcpy(kp.ax, plan.ax, sizeof(kp.ax));
  std::memcpy(kp.ay, plan.ay, sizeof(kp.ay));
  std::memcpy(kp.ea, plan.ea, sizeof(kp.ea));
  std::memcpy(kp.ec, plan.ec, sizeof(kp.ec));
  std::memcpy(kp.qax, plan.qax, sizeof(kp.qax));
  std::memcpy(kp.qay, plan.qay, sizeof(kp.qay));
  std::memcpy(kp.qa, plan.qa, sizeof(kp.qa));
  std::memcpy(kp.qc, plan.qc, sizeof(kp.qc));
  std::memcpy(kp.box, plan.box, sizeof(kp.box));
  for (int k = 0; k < 8; ++k) {
    const std::uint64_t g = plan.kept[k];
    kp.kept[k] = (g >= base && g - base < n) ? g - base : ~0ull;
    kp.kept_label[k] = plan.kept_label[k];
  }
  kp.m = plan.m;
  return kp;
}

// K2 over the n points of a shard, or (d_cand != null) over the n_cand
// candidates listed there (shard-local indices, same width as the queues).
void filter_core(ohx_ctx* c, const double* d_xy, std::uint64_t n, std::uint64_t base,
                 const ohx_filter_plan& plan, std::uint8_t* d_labels, std::uint64_t counts[4],
                 cudaStream_t s, const void* d_cand, std::uint64_t n_cand,
                 const double* d_cpts) {
  const KPlan kp = make_kplan(plan, base, n);
  const std::uint64_t items = d_cand ? n_cand : n;
  const int idx_bytes = n <= 0xffffffffull ? 4 : 8;
  if (items == 0) {  // no candidates at all
    for (int q = 0; q < 4; ++q) counts[q] = 0;
  } else {
    const std::uint64_t ntiles = (items + kK2Tile - 1) / kK2Tile;
    dev_grow(reinterpret_cast<void**>(&c->d_status), &c->status_bytes,
             k2_work_bytes(ntiles), "k2 work area");
    // queue capacity: 1/16 of the items (at least 1M); grown to the exact
    // counts and re-run on overflow (counts are exact even when stores are
    // dropped)
    std::uint64_t cap =
        std::min<std::uint64_t>(items, std::max<std::uint64_t>(1u << 20, items / 16));
    if (c->queue_bytes / (4ull * idx_bytes) > cap)
      cap = std::min<std::uint64_t>(items, c->queue_bytes / (4ull * idx_bytes));
    for (int attempt = 0; attempt < 2; ++attempt) {
      dev_grow(&c->d_queues, &c->queue_bytes, 4ull * idx_bytes * cap, "queues");
      check_cuda(cudaEventRecord(c->ev[2][0], s), "cudaEventRecord");
      launch_k2(d_xy, items, kp, c->d_status, ntiles, c->d_queues, idx_bytes, cap, d_labels,
                c->d_counts, s, d_cand, d_cpts);  // k2_filter + k2_compact
      check_cuda(cudaEventRecord(c->ev[2][1], s), "cudaEventRecord");
      c->timed[2] = true;
      c->launches += 2;
      check_cuda(cudaMemcpyAsync(c->h_counts, c->d_counts, 4 * sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync(counts)");
      check_cuda(cudaStreamSynchronize(s), "k2_filter");
      std::uint64_t mx = 0;
      for (int q = 0; q < 4; ++q) {
        counts[q] = c->h_counts[q];
        mx = std::max<std::uint64_t>(mx, counts[q]);
      }
      if (mx <= cap) break;
      if (attempt == 1) throw Error(OHX_E_INTERNAL, "k2_filter: queue overflow after regrow");
      cap = std::min<std::uint64_t>(items, mx + mx / 8 + 1024);
    }
    c->last_cap = cap;
  }
  c->last_xy = d_xy;
  c->last_n = n;
  c->last_base = base;
  c->last_idx_bytes = idx_bytes;
  for (int q = 0; q < 4; ++q) c->last_counts[q] = counts[q];
}

}  // namespace

void filter(ohx_ctx* c, const double* d_xy, std::uint64_t n, std::uint64_t base,
            const ohx_filter_plan& plan, std::uint8_t* d_labels, std::uint64_t counts[4],
            cudaStream_t s) {
  if (n == 0) throw std::invalid_argument("classify_points: empty point set");
  filter_core(c, d_xy, n, base, plan, d_labels, counts, s, nullptr, 0, nullptr);
}

// Vertices of the convex polygon {p : key_a(p) <= b[a], a = 0..7} (the slot
// keys x, y, -x, -y, x+y, y-x, -(x+y), x-y), in long double: the axis box
// clipped by the four diagonal half-planes.
std::vector<std::pair<long double, long double>> region_vertices(const long double b[8]) {
  using V = std::pair<long double, long double>;
  std::vector<V> poly = {{-b[2], -b[3]}, {b[0], -b[3]}, {b[0], b[1]}, {-b[2], b[1]}};
  static const int dx[4] = {1, -1, -1, 1}, dy[4] = {1, 1, -1, -1};
  for (int k = 0; k < 4 && poly.size() >= 3; ++k) {
    std::vector<V> out;
    auto val = [&](const V& p) { return dx[k] * p.first + dy[k] * p.second - b[4 + k]; };
    for (std::size_t i = 0; i < poly.size(); ++i) {
      const V p = poly[i], q = poly[(i + 1) % poly.size()];
      const long double vp = val(p), vq = val(q);
      if (vp <= 0) out.push_back(p);
      if ((vp <= 0) != (vq <= 0)) {
        const long double t = vp / (vp - vq);
        out.push_back({p.first + t * (q.first - p.first), p.second + t * (q.second - p.second)});
      }
    }
    poly = out;
  }
  return poly;
}

// Is every point the fused pass dropped (in_region true) strictly inside the
// true octagon, i.e. reference label 0?  The accepted set is within Q with
// its diagonal bounds widened by the rounding of fl(x+y), fl(x-y)
// (|fl(s) - s| <= u(|x| + |y|)); every vertex of that widened polygon must
// clear every octagon edge by the determinant's error bound (the bound is
// concave, see box_ok, so vertices suffice).
bool region_certified(const ohx_filter_plan& plan, const KFRegion& q) {
  if (plan.m < 3) return false;
  if (!(q.x0 <= q.x1) || !(q.y0 <= q.y1) || !(q.t0 <= q.t1) || !(q.d0 <= q.d1)) return false;
  const long double X = std::max(std::fabs((long double)q.x0), std::fabs((long double)q.x1));
  const long double Y = std::max(std::fabs((long double)q.y0), std::fabs((long double)q.y1));
  const long double w = 4.0L * 0x1p-53L * (X + Y) + 0x1p-1000L;
  const long double b[8] = {q.x1, q.y1, -(long double)q.x0, -(long double)q.y0,
                            q.t1 + w, -(long double)q.d0 + w, -(long double)q.t0 + w, q.d1 + w};
  const auto verts = region_vertices(b);
  if (verts.size() < 3) return false;
  const long double uf = 8.0L * 0x1p-53L;
  for (int i = 0; i < plan.m; ++i) {
    const long double ax = plan.ax[i], ay = plan.ay[i], A = plan.ea[i], C = plan.ec[i];
    for (const auto& v : verts) {
      const long double dy = v.second - ay, dx = v.first - ax;
      const long double E = A * dy - C * dx;
      const long double margin = uf * (std::fabs(A) * std::fabs(dy) + std::fabs(C) * std::fabs(dx)) +
                                 0x1p-1000L;
      if (!(E > margin)) return false;
    }
  }
  return true;
}

// The fused pass's own test, on the host (same binary64 operations).
bool in_region_host(const KFRegion& q, double x, double y) {
  const double t = x + y, d = x - y;
  return x >= q.x0 && x <= q.x1 && y >= q.y0 && y <= q.y1 && t >= q.t0 && t <= q.t1 &&
         d >= q.d0 && d <= q.d1;
}

void queue_fetch(ohx_ctx* c, int q, std::uint64_t* h_idx, double* h_xy,
                 std::uint64_t cap, cudaStream_t s) {
  if (q < 1 || q > 4) throw std::invalid_argument("queue must be 1..4");
  if (c->last_n == 0) throw std::invalid_argument("no filter result in this context");
  const std::uint64_t cnt = c->last_counts[q - 1];
  if (cnt > cap) throw std::invalid_argument("queue larger than the output capacity");
  if (cnt == 0) return;
  const auto* qbase = static_cast<const char*>(c->d_queues) +
                      std::uint64_t(q - 1) * c->last_cap * c->last_idx_bytes;
  if (h_xy) {
    dev_grow(reinterpret_cast<void**>(&c->d_gather), &c->gather_bytes, cnt * 16, "gather");
    launch_gather(c->last_xy, qbase, c->last_idx_bytes, cnt, c->d_gather, s);
    ++c->launches;
    check_cuda(cudaMemcpyAsync(h_xy, c->d_gather, cnt * 16, cudaMemcpyDeviceToHost, s),
               "cudaMemcpyAsync(queue xy)");
  }
  if (h_idx) {
    if (c->last_idx_bytes == 8) {
      check_cuda(cudaMemcpyAsync(h_idx, qbase, cnt * 8, cudaMemcpyDeviceToHost, s),
                 "cudaMemcpyAsync(queue idx)");
      check_cuda(cudaStreamSynchronize(s), "queue fetch");
    } else {
      std::vector<std::uint32_t> tmp(cnt);
      check_cuda(cudaMemcpyAsync(tmp.data(), qbase, cnt * 4, cudaMemcpyDeviceToHost, s),
                 "cudaMemcpyAsync(queue idx)");
      check_cuda(cudaStreamSynchronize(s), "queue fetch");
      for (std::uint64_t k = 0; k < cnt; ++k) h_idx[k] = c->last_base + tmp[k];
    }
    if (c->last_idx_bytes == 8 && c->last_base)
      for (std::uint64_t k = 0; k < cnt; ++k) h_idx[k] += c->last_base;
  }
  check_cuda(cudaStreamSynchronize(s), "queue fetch");
}

void queues_fetch_xy(ohx_ctx* c, double* h_xy, cudaStream_t s) {
  if (c->last_n == 0) throw std::invalid_argument("no filter result in this context");
  const std::uint64_t total =
      c->last_counts[0] + c->last_counts[1] + c->last_counts[2] + c->last_counts[3];
  if (total == 0) return;
  dev_grow(reinterpret_cast<void**>(&c->d_gather), &c->gather_bytes, total * 16, "gather");
  launch_gather4(c->last_xy, c->d_queues, c->last_idx_bytes, c->last_cap, c->last_counts,
                 c->d_gather, s);
  ++c->launches;
  check_cuda(cudaMemcpyAsync(h_xy, c->d_gather, total * 16, cudaMemcpyDeviceToHost, s),
             "cudaMemcpyAsync(queues xy)");
  check_cuda(cudaStreamSynchronize(s), "queues fetch");
}

namespace {
// OHX_TRACE=1: host wall time of each pipeline phase on stderr
struct Trace {
  bool on = [] {
    const char* e = std::getenv("OHX_TRACE");
    return e && *e && std::string(e) != "0";
  }();
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[ohx] %-14s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};
}  // namespace

// Survivor counts from which the hull stage's sweep sort runs on the device
constexpr std::uint64_t kDeviceSortMin = 1u << 17;

void host_grow(void** p, std::uint64_t* have, std::uint64_t need, const char* what) {
  if (*have >= need && *p) return;
  if (*p) check_cuda(cudaFreeHost(*p), "cudaFreeHost");
  *p = nullptr;
  *have = 0;
  check_cuda(cudaMallocHost(p, need), what);
  *have = need;
}

PVec device_queues_hull(ohx_ctx* c, const FilterOut& f, cudaStream_t s) {
  // reference hull.cpp:164-183 on the device queues
  const std::uint64_t total = f.counts[0] + f.counts[1] + f.counts[2] + f.counts[3];
  const P2 anchors[4] = {{f.ext.x[OHX_EAST], f.ext.y[OHX_EAST]},
                         {f.ext.x[OHX_NORTH], f.ext.y[OHX_NORTH]},
                         {f.ext.x[OHX_WEST], f.ext.y[OHX_WEST]},
                         {f.ext.x[OHX_SOUTH], f.ext.y[OHX_SOUTH]}};
  if (total >= kDeviceSortMin) {
    // large survivor sets: the arcs are built and sorted on the device and
    // come back in sweep order; the chains and the clean-up run on the host
    dev_grow(reinterpret_cast<void**>(&c->d_gather), &c->gather_bytes, total * 16, "gather");
    launch_gather4(c->last_xy, c->d_queues, c->last_idx_bytes, c->last_cap, c->last_counts,
                   c->d_gather, s);
    ++c->launches;
    const std::uint64_t arcs_n = total + 8;
    dev_grow(&c->d_hsort, &c->hsort_bytes, sort_arcs_work_bytes(f.counts) + arcs_n * 16,
             "hull sort work");
    auto* d_sorted = reinterpret_cast<double*>(static_cast<unsigned char*>(c->d_hsort) +
                                               sort_arcs_work_bytes(f.counts));
    Trace tr;
    sort_arcs(c->d_gather, f.counts, reinterpret_cast<const double*>(anchors), c->d_hsort,
              d_sorted, s);
    c->launches += 2 + 4 * 4;  // build/gather + four radix sorts
    if (tr.on) {
      check_cuda(cudaStreamSynchronize(s), "hull sort");
      tr.mark("hull dev sort");
    }
    host_grow(&c->h_sorted, &c->h_sorted_bytes, arcs_n * 16, "cudaMallocHost(sorted arcs)");
    // one copy per arc: arc q's chain starts as soon as its copy lands
    if (!c->arc_ev[0])
      for (auto& e : c->arc_ev)
        check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate(arc)");
    const P2* arcs[4];
    std::uint64_t len[4], off = 0;
    for (int q = 0; q < 4; ++q) {
      arcs[q] = static_cast<const P2*>(c->h_sorted) + off;
      len[q] = f.counts[q] + 2;
      check_cuda(cudaMemcpyAsync(static_cast<P2*>(c->h_sorted) + off,
                                 reinterpret_cast<const P2*>(d_sorted) + off, len[q] * 16,
                                 cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync(sorted arc)");
      check_cuda(cudaEventRecord(c->arc_ev[q], s), "cudaEventRecord(arc)");
      off += len[q];
    }
    std::atomic<int> failed{cudaSuccess};  // set by the arc threads (no throwing there)
    PVec cyc = hull_from_sorted_arcs(arcs, len, [&](int q) {
      const cudaError_t e = cudaEventSynchronize(c->arc_ev[q]);
      if (e != cudaSuccess) failed = e;
    });
    check_cuda(static_cast<cudaError_t>(failed.load()), "cudaEventSynchronize(sorted arc)");
    tr.mark("hull D2H + host");
    return cyc;
  }
  // one gather launch and one D2H of the survivors' coordinates, then the
  // host hull stage
  std::vector<P2> packed(total);
  queues_fetch_xy(c, reinterpret_cast<double*>(packed.data()), s);
  const P2* qp[4];
  std::uint64_t off = 0;
  for (int k = 0; k < 4; ++k) {
    qp[k] = packed.data() + off;
    off += f.counts[k];
  }
  return hull_from_queue_points(anchors, qp, f.counts);
}

namespace {

void finish_extremes(ohx_ctx* c, const double* d_xy, std::uint64_t n,
                     const ohx_extremes_rec& rec, FilterOut& f, cudaStream_t s) {
  const std::uint32_t mask = resolve_extremes(rec, &f.ext);
  f.corner_pass = mask != 0;
  if (mask) {
    const double bbox[4] = {rec.x[OHX_EAST], rec.y[OHX_NORTH], rec.x[OHX_WEST],
                            rec.y[OHX_SOUTH]};
    ohx_corner_rec cr;
    corners_exact(c, d_xy, n, 0, bbox, &cr, s);
    apply_corners(cr, &f.ext);
  }
  const int slot[8] = {OHX_EAST, OHX_NE, OHX_NORTH, OHX_NW,
                       OHX_WEST, OHX_SW, OHX_SOUTH, OHX_SE};
  double cand[16];
  for (int k = 0; k < 8; ++k) {
    cand[2 * k] = f.ext.x[slot[k]];
    cand[2 * k + 1] = f.ext.y[slot[k]];
  }
  f.m = build_octagon(cand, f.oct);
  make_plan(f.ext, f.oct, f.m, &f.plan);
}

constexpr std::uint64_t kFuseMinPoints = 1ull << 23;  // below: both passes are cheap

// OHX_FUSE: unset/"auto" = fused pass when it pays, "0" = always two passes,
// "fallback" = run the fused pass but reject its region (exercises the
// verification-failure path), "force" = fuse whatever the sample coverage
// (exercises heavy candidate lists).  The last two are for tests.
int fuse_mode() {
  static const int mode = [] {
    const char* e = std::getenv("OHX_FUSE");
    if (!e || !*e || std::string(e) == "auto") return 1;
    if (std::string(e) == "0") return 0;
    if (std::string(e) == "fallback") return 2;
    if (std::string(e) == "force") return 3;
    return 1;
  }();
  return mode;
}
constexpr int kSampleLen = 8192;     // points per sample run
static_assert(kSampleLen % 2048 == 0, "k1_small reads sample runs 2048 points at a time");
constexpr int kCoverageStep = 4;      // coverage counted on every 4th run
constexpr int kSampleMaxSegs = 1024;  // runs (8M points, 128 MB) for n >= 2^27
// OHX_SAMPLE_SEGS overrides the cap (experiment switch)
int sample_max_segs() {
  static const int v = [] {
    const char* e = std::getenv("OHX_SAMPLE_SEGS");
    const int k = e ? std::atoi(e) : 0;
    return k >= 64 ? k : kSampleMaxSegs;
  }();
  return v;
}
constexpr int kSubSamples = 8;  // disjoint sub-samples of kSampleSegs / 8 runs each
constexpr double kFuseMinCoverage = 0.8;

// Part of the convex polygon `poly` on the left of a -> b (Sutherland-Hodgman
// step; heuristic geometry, the box is certified exactly after the pass).
std::vector<P2> clip_left(const std::vector<P2>& poly, P2 a, P2 b) {
  std::vector<P2> out;
  const std::size_t m = poly.size();
  auto side = [&](P2 p) { return (b.x - a.x) * (p.y - a.y) - (b.y - a.y) * (p.x - a.x); };
  for (std::size_t i = 0; i < m; ++i) {
    const P2 p = poly[i], q = poly[(i + 1) % m];
    const double sp = side(p), sq = side(q);
    if (sp >= 0) out.push_back(p);
    if ((sp >= 0) != (sq >= 0)) {
      const double t = sp / (sp - sq);
      out.push_back({p.x + t * (q.x - p.x), p.y + t * (q.y - p.y)});
    }
  }
  return out;
}


// key of slot a (ohx.h slot order: x, y, -x, -y, x+y, y-x, -(x+y), x-y)
double slot_key(int a, double x, double y) {
  switch (a) {
    case 0: return x;
    case 1: return y;
    case 2: return -x;
    case 3: return -y;
    case 4: return x + y;
    case 5: return y - x;
    case 6: return -(x + y);
    default: return x - y;
  }
}

// Is the region {key_a <= b[a]} inside the convex CCW polygon R?  (R is
// convex, so the region's vertices decide.)  Heuristic geometry in double,
// no allocation: it runs a few hundred times per fit.
bool region_inside(const double b[8], const std::vector<P2>& R) {
  P2 poly[16], out[16];
  int m = 4;
  poly[0] = {-b[2], -b[3]};
  poly[1] = {b[0], -b[3]};
  poly[2] = {b[0], b[1]};
  poly[3] = {-b[2], b[1]};
  static const int dx[4] = {1, -1, -1, 1}, dy[4] = {1, 1, -1, -1};
  for (int k = 0; k < 4 && m >= 3; ++k) {
    int o = 0;
    for (int i = 0; i < m; ++i) {
      const P2 p = poly[i], q = poly[i + 1 == m ? 0 : i + 1];
      const double vp = dx[k] * p.x + dy[k] * p.y - b[4 + k];
      const double vq = dx[k] * q.x + dy[k] * q.y - b[4 + k];
      if (vp <= 0) out[o++] = p;
      if ((vp <= 0) != (vq <= 0)) {
        const double t = vp / (vp - vq);
        out[o++] = {p.x + t * (q.x - p.x), p.y + t * (q.y - p.y)};
      }
    }
    m = o;
    for (int i = 0; i < m; ++i) poly[i] = out[i];
  }
  if (m < 3) return false;
  const std::size_t r = R.size();
  for (int v = 0; v < m; ++v)
    for (std::size_t i = 0; i < r; ++i) {
      const P2 a = R[i], c = R[i + 1 == r ? 0 : i + 1];
      if ((c.x - a.x) * (poly[v].y - a.y) - (c.y - a.y) * (poly[v].x - a.x) < 0) return false;
    }
  return true;
}

// The fused pass's region Q: an octagon with the slot directions as edge
// normals, fitted inside the convex polygon R.  Start from R's own slot
// support values scaled towards R's centroid until the octagon fits, then
// push each bound out on its own (a few rounds), then pull everything 0.2 %
// back towards the centre.  Finally every bound is clamped strictly below
// lim[a] (the sample's best / second key of the slot).
bool fit_region(const std::vector<P2>& R, const double lim[8], KFRegion* q) {
  if (R.size() < 3) return false;
  double cx = 0, cy = 0;
  for (const P2& p : R) {
    cx += p.x;
    cy += p.y;
  }
  cx /= double(R.size());
  cy /= double(R.size());
  double h[8], c0[8], b[8];
  for (int a = 0; a < 8; ++a) {
    h[a] = -INFINITY;
    for (const P2& p : R) h[a] = std::max(h[a], slot_key(a, p.x, p.y));
    c0[a] = slot_key(a, cx, cy);
    if (!(h[a] > c0[a])) return false;
  }
  auto at = [&](double sc, double* out) {
    for (int a = 0; a < 8; ++a) out[a] = c0[a] + sc * (h[a] - c0[a]);
  };
  double lo = 0, hi = 1;
  at(1e-6, b);
  if (!region_inside(b, R)) return false;
  // bisections to ~1e-4 of the span: Q is pulled 0.2 % inwards afterwards
  for (int it = 0; it < 14; ++it) {
    const double mid = (lo + hi) / 2;
    at(mid, b);
    if (region_inside(b, R)) lo = mid;
    else hi = mid;
  }
  at(lo, b);
  for (int round = 0; round < 2; ++round)
    for (int a = 0; a < 8; ++a) {
      double good = b[a], bad = h[a];
      for (int it = 0; it < 10; ++it) {
        double t[8];
        std::memcpy(t, b, sizeof(t));
        t[a] = (good + bad) / 2;
        if (region_inside(t, R)) good = t[a];
        else bad = t[a];
      }
      b[a] = good;
    }
  double r[8];
  for (int a = 0; a < 8; ++a) {
    r[a] = c0[a] + 0.998 * (b[a] - c0[a]);
    const double below = std::nextafter(lim[a], -INFINITY);
    if (r[a] > below) r[a] = below;
  }
  *q = KFRegion{-r[2], r[0], -r[3], r[1], -r[6], r[4], -r[5], r[7]};
  return q->x0 < q->x1 && q->y0 < q->y1 && q->t0 < q->t1 && q->d0 < q->d1;
}

// The provisional region of the fused pass.  A sample of about n/16 points
// (up to 8M: runs of kSampleLen consecutive points at evenly spaced offsets,
// read in place) is split into kSubSamples disjoint sub-samples (run b goes
// to sub-sample b % kSubSamples, so each spans the whole index range); each
// one's eight extremes (one batched launch) give an octagon, and Q is fitted
// inside the INTERSECTION of those octagons.  The sub-sample octagons
// scatter the way the true octagon may sit relative to any one sample's, so
// a region inside all of them rarely leaves the true octagon (checked
// exactly after the pass; a miss costs the regular second pass).  Q's bounds
// are also kept strictly below the whole sample's extremes keys, which is
// what lets the fused pass skip the extremes test for points inside Q.
// Returns false when fusing does not pay (small input, no region, sample
// coverage below kFuseMinCoverage).
bool provisional_region(ohx_ctx* c, const double* d_xy, std::uint64_t n, KFRegion* q,
                        std::uint64_t* sampled, cudaStream_t s, FilterOut& f, Trace& tr) {
  if (n < kFuseMinPoints || fuse_mode() == 0) return false;
  f.fuse_state = 2;
  // about n/16 sampled points, 64..1024 runs, a multiple of kSubSamples
  const int segs = static_cast<int>(std::clamp<std::uint64_t>(
                       n / (16ull * kSampleLen), 64, sample_max_segs())) / kSubSamples * kSubSamples;
  dev_grow(reinterpret_cast<void**>(&c->d_sample), &c->sample_bytes,
           kSubSamples * sizeof(ohx_extremes_rec), "sample records");
  auto* d_recs = reinterpret_cast<ohx_extremes_rec*>(c->d_sample);
  ensure_partials(c, segs);
  launch_k1_sample(d_xy, n, segs, kSampleLen, kSubSamples, c->d_partials, c->d_ticket, d_recs, s);
  ++c->launches;
  ohx_extremes_rec rs[kSubSamples];
  check_cuda(cudaMemcpyAsync(rs, d_recs, sizeof(rs), cudaMemcpyDeviceToHost, s),
             "cudaMemcpyAsync(sample recs)");
  check_cuda(cudaStreamSynchronize(s), "sample extremes");
  tr.mark("sample k1");
  const int slot[8] = {OHX_EAST, OHX_NE, OHX_NORTH, OHX_NW,
                       OHX_WEST, OHX_SW, OHX_SOUTH, OHX_SE};
  std::vector<P2> region;
  for (int g = 0; g < kSubSamples; ++g) {
    ohx_extreme_set es;
    resolve_extremes(rs[g], &es);  // heuristic octagons: diagonal winners need no certificate
    double cand[16], oct[16];
    for (int k = 0; k < 8; ++k) {
      cand[2 * k] = es.x[slot[k]];
      cand[2 * k + 1] = es.y[slot[k]];
    }
    const int m = build_octagon(cand, oct);
    if (m < 3) return false;
    if (g == 0) {
      for (int i = 0; i < m; ++i) region.push_back({oct[2 * i], oct[2 * i + 1]});
      continue;
    }
    for (int i = 0; i < m && region.size() >= 3; ++i) {
      const int j = i + 1 == m ? 0 : i + 1;
      region = clip_left(region, {oct[2 * i], oct[2 * i + 1]}, {oct[2 * j], oct[2 * j + 1]});
    }
    if (region.size() < 3) return false;
  }
  // the whole sample's best (axis) / second (diagonal) keys
  ohx_extremes_rec all;
  combine_extremes(rs, kSubSamples, &all);
  double lim[8];
  for (int a = 0; a < 8; ++a) lim[a] = a < 4 ? all.key[a] : all.second[a - 4];
  if (!fit_region(region, lim, q)) return false;
  tr.mark("region fit");
  // the coverage count stays on the device: KF reads it and runs only when
  // enough of the sample falls inside Q (no host round trip here)
  launch_count_in_region(d_xy, n, segs, kSampleLen, kCoverageStep, *q, c->d_cnt, s);
  ++c->launches;
  *sampled = std::uint64_t((segs + kCoverageStep - 1) / kCoverageStep) * kSampleLen;
  f.fuse_state = 3;
  return true;
}

}  // namespace

namespace {
FilterOut device_filter_impl(ohx_ctx* c, const double* d_xy, std::uint64_t n,
                             std::uint8_t* d_labels, cudaStream_t s);
}

FilterOut device_filter(ohx_ctx* c, const double* d_xy, std::uint64_t n,
                        std::uint8_t* d_labels, cudaStream_t s) {
  const FilterOut f = device_filter_impl(c, d_xy, n, d_labels, s);
  c->last_run.fused = f.fused;
  c->last_run.corner_pass = f.corner_pass;
  c->last_run.candidates = f.candidates;
  c->last_run.fuse_state = f.fuse_state;
  c->last_run.sample_coverage = f.sample_coverage;
  for (int q = 0; q < 4; ++q) c->last_run.counts[q] = f.counts[q];
  return f;
}

namespace {

// Fused pass, first half, over the n points of one shard (global indices
// base + j): provisional region -> KF -> ordered candidate list -> K1 over
// the candidates.  Returns true with the shard's extremes record in *rec
// (what K1 over all points would have produced) when the fused pass ran;
// false (f.fuse_state says why) when the caller must run K1 instead.
bool fused_begin(ohx_ctx* c, const double* d_xy, std::uint64_t n, std::uint64_t base,
                 FilterOut& f, ohx_extremes_rec* rec, cudaStream_t s, Trace& tr) {
  c->fz.active = false;
  KFRegion q;
  std::uint64_t sampled = 0;
  if (!provisional_region(c, d_xy, n, &q, &sampled, s, f, tr)) return false;
  const int idx_bytes = n <= 0xffffffffull ? 4 : 8;
  const int grid = kf_grid(c->device);
  const std::uint64_t nw = std::uint64_t(grid) * kKFWarpsPerBlock;
  const std::uint64_t per = ((n + 255) / 256 + nw - 1) / nw * 256;  // points per warp
  // KF runs (device-side gate) when >= kFuseMinCoverage of the sample is in
  // Q; each warp region has room for 1.5x the miss rate that allows (+256).
  // A region that overflows sends the call down the two-pass path.
  const double min_cov = fuse_mode() == 3 ? 0.0 : kFuseMinCoverage;
  const auto gate_min = static_cast<std::uint64_t>(std::ceil(min_cov * double(sampled)));
  const std::uint64_t cap_w = std::min<std::uint64_t>(
      per, 256 + static_cast<std::uint64_t>(1.5 * (1.0 - min_cov) * double(per)));
  dev_grow(&c->d_regions, &c->regions_bytes, nw * cap_w * idx_bytes, "kf regions");
  dev_grow(reinterpret_cast<void**>(&c->d_status), &c->status_bytes, nw * 12 + 16, "kf counts");
  auto* d_wcounts = reinterpret_cast<std::uint32_t*>(c->d_status);
  auto* d_offsets = c->d_status + (nw + 1) / 2;  // 8-byte aligned after the u32 counts
  check_cuda(cudaEventRecord(c->ev[0][0], s), "cudaEventRecord");
  launch_kf(d_xy, n, q, grid, c->d_regions, idx_bytes, cap_w, d_wcounts, c->d_cnt, gate_min, s);
  check_cuda(cudaEventRecord(c->ev[0][1], s), "cudaEventRecord");
  c->timed[0] = true;
  ++c->launches;
  // candidate list + coordinates and K1 over them, sized on the device: the
  // list buffers hold cap_c candidates (more: regrown and redone below)
  check_cuda(cudaEventRecord(c->ev[3][0], s), "cudaEventRecord");
  launch_kf_scan(d_wcounts, nw, cap_w, d_offsets, c->d_cnt, c->d_counts, s);
  std::uint64_t cap_c = std::max<std::uint64_t>(c->cpts_bytes / 16,
                                                std::max<std::uint64_t>(1u << 20, n / 32));
  auto candidates = [&](std::uint64_t cap) {
    dev_grow(&c->d_cand, &c->cand_bytes, cap * idx_bytes, "candidates");
    dev_grow(reinterpret_cast<void**>(&c->d_cpts), &c->cpts_bytes, cap * 16, "candidate points");
    launch_kf_gather(d_xy, c->d_regions, idx_bytes, cap_w, d_wcounts, d_offsets, nw, c->d_cand,
                     c->d_cpts, cap, s);
    const int k1g = k1_list_grid(cap);
    ensure_partials(c, k1g);
    launch_k1_list(c->d_cpts, cap, c->d_counts, c->d_partials, k1g, c->d_ticket, c->d_rec, s);
    launch_map_rec(c->d_rec, c->d_cand, idx_bytes, base, s);
    c->launches += 3;
    check_cuda(cudaMemcpyAsync(c->h_counts, c->d_counts, 4 * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync(counts)");
    check_cuda(cudaMemcpyAsync(c->h_rec, c->d_rec, sizeof(ohx_extremes_rec),
                               cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync(rec)");
    check_cuda(cudaStreamSynchronize(s), "kf + candidate extremes");
  };
  candidates(cap_c);
  ++c->launches;  // kf_scan
  tr.mark("kf+cand-k1");
  f.sample_coverage = double(c->h_counts[2]) / double(sampled);
  const std::uint64_t n_cand = c->h_counts[0];
  f.candidates = n_cand;
  if (c->h_counts[2] < gate_min) return false;  // KF did not run: low coverage
  if (n_cand == 0 || c->h_counts[1] != 0) {
    f.fuse_state = 5;  // a warp region overflowed: the two-pass path
    return false;
  }
  if (n_cand > cap_c) {  // more candidates than the list buffers held
    cap_c = n_cand;
    candidates(cap_c);
  }
  check_cuda(cudaEventRecord(c->ev[3][1], s), "cudaEventRecord");
  c->timed[3] = true;
  *rec = *c->h_rec;
  rec->n = n;
  c->fz = {true, q, d_xy, n, base, n_cand};
  return true;
}

// Fused pass, second half: with the (global) ExtremeSet and plan, the
// points KF dropped have the reference label 0 iff Q lies inside the
// octagon (exact error bounds) and holds none of the eight kept points;
// then K2 runs over the candidates only, otherwise over all n points.
void fused_finish(ohx_ctx* c, const double* d_xy, std::uint64_t n, std::uint64_t base,
                  const ohx_extreme_set& ext, const ohx_filter_plan& plan,
                  std::uint8_t* d_labels, std::uint64_t counts[4], FilterOut& f,
                  cudaStream_t s) {
  if (!c->fz.active || c->fz.d_xy != d_xy || c->fz.n != n || c->fz.base != base)
    throw std::invalid_argument("filter_fused: no fused pass over these points in this context");
  c->fz.active = false;
  const KFRegion& q = c->fz.q;
  bool ok = region_certified(plan, q) && fuse_mode() != 2;
  f.fuse_state = 4;
  for (int a = 0; a < 8 && ok; ++a) ok = !in_region_host(q, ext.x[a], ext.y[a]);
  if (!ok) {  // not certified: the regular K2 pass over all points
    filter(c, d_xy, n, base, plan, d_labels, counts, s);
    return;
  }
  f.fuse_state = 1;
  f.fused = true;
  if (d_labels) check_cuda(cudaMemsetAsync(d_labels, 0, n, s), "cudaMemsetAsync(labels)");
  filter_core(c, d_xy, n, base, plan, d_labels, counts, s, c->d_cand, c->fz.n_cand, c->d_cpts);
}

FilterOut device_filter_impl(ohx_ctx* c, const double* d_xy, std::uint64_t n,
                             std::uint8_t* d_labels, cudaStream_t s) {
  if (n == 0) throw std::invalid_argument("heaphull: empty point set");
  FilterOut f{};
  for (bool& t : c->timed) t = false;  // kernel_ms reports this pipeline's stages
  Trace tr;
  ohx_extremes_rec rec;
  if (fused_begin(c, d_xy, n, 0, f, &rec, s, tr)) {
    finish_extremes(c, d_xy, n, rec, f, s);
    tr.mark("octagon+plan");
    fused_finish(c, d_xy, n, 0, f.ext, f.plan, d_labels, f.counts, f, s);
    tr.mark("k2");
    return f;
  }
  // ---- two passes: K1, then K2
  extremes(c, d_xy, n, 0, &rec, s);
  finish_extremes(c, d_xy, n, rec, f, s);
  filter(c, d_xy, n, 0, f.plan, d_labels, f.counts, s);
  return f;
}
}  // namespace

ohx_ctx* create_ctx(int device) {
  int ndev = 0;
  check_cuda(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (device < 0 || device >= ndev)
    throw Error(OHX_E_NODEVICE, "device " + std::to_string(device) + " not visible (" +
                                    std::to_string(ndev) + " devices)");
  cudaDeviceProp prop;
  check_cuda(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (prop.major != 10)
    throw Error(OHX_E_NODEVICE, std::string("device ") + prop.name +
                                    " is not sm_100 (this library is built for sm_100a only)");
  auto c = std::make_unique<ohx_ctx>();
  c->device = device;
  bind(c.get());
  check_cuda(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
  check_cuda(cudaMalloc(&c->d_ticket, 256), "cudaMalloc(ticket)");
  check_cuda(cudaMemset(c->d_ticket, 0, 256), "cudaMemset(ticket)");
  check_cuda(cudaMalloc(&c->d_rec, sizeof(ohx_extremes_rec)), "cudaMalloc(rec)");
  check_cuda(cudaMalloc(&c->d_crec, sizeof(ohx_corner_rec)), "cudaMalloc(crec)");
  check_cuda(cudaMalloc(&c->d_counts, 64), "cudaMalloc(counts)");
  check_cuda(cudaMallocHost(&c->h_rec, sizeof(ohx_extremes_rec)), "cudaMallocHost");
  check_cuda(cudaMallocHost(&c->h_crec, sizeof(ohx_corner_rec)), "cudaMallocHost");
  check_cuda(cudaMallocHost(&c->h_counts, 64), "cudaMallocHost");
  check_cuda(cudaMalloc(&c->d_cnt, 64), "cudaMalloc(cnt)");
  check_cuda(cudaMallocHost(&c->h_cnt, 64), "cudaMallocHost");
  for (auto& pair : c->ev)
    for (auto& e : pair) check_cuda(cudaEventCreate(&e), "cudaEventCreate");
  return c.release();
}

void destroy_ctx(ohx_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (void* p : {static_cast<void*>(c->d_partials), static_cast<void*>(c->d_ticket),
                  static_cast<void*>(c->d_rec), static_cast<void*>(c->d_crec),
                  static_cast<void*>(c->d_counts), static_cast<void*>(c->d_status),
                  c->d_queues, static_cast<void*>(c->d_pts),
                  static_cast<void*>(c->d_labels), static_cast<void*>(c->d_gather),
                  static_cast<void*>(c->d_sample), c->d_cand, static_cast<void*>(c->d_cnt),
                  c->d_regions, static_cast<void*>(c->d_cpts), c->d_hsort})
    if (p) cudaFree(p);
  for (void* p : {static_cast<void*>(c->h_rec), static_cast<void*>(c->h_crec),
                  static_cast<void*>(c->h_counts), static_cast<void*>(c->h_cnt), c->h_sorted})
    if (p) cudaFreeHost(p);
  for (int b = 0; b < ohx_ctx::kStageBufs; ++b) {
    if (c->h_stage[b]) cudaFreeHost(c->h_stage[b]);
    if (c->stage_ev[b]) cudaEventDestroy(c->stage_ev[b]);
  }
  for (auto& e : c->arc_ev)
    if (e) cudaEventDestroy(e);
  for (auto& pair : c->ev)
    for (auto& e : pair)
      if (e) cudaEventDestroy(e);
  cudaStreamDestroy(c->stream);
  delete c;
}

ohx_ctx* default_ctx(int device) {
  static std::mutex mu;
  static std::vector<ohx_ctx*> ctxs;  // intentionally leaked at exit
  std::lock_guard<std::mutex> g(mu);
  if (device < 0) {
    const char* env = std::getenv("OHX_DEVICE");
    device = env ? std::atoi(env) : 0;
  }
  if (static_cast<int>(ctxs.size()) <= device) ctxs.resize(device + 1, nullptr);
  if (!ctxs[device]) ctxs[device] = create_ctx(device);
  return ctxs[device];
}

}  // namespace ohx

// =================================================================== C ABI
using namespace ohx;

extern "C" {

int ohx_abi_version(void) { return OHX_ABI_VERSION; }

const char* ohx_last_error(void) { return g_last_error.c_str(); }

int ohx_device_count(int* n) {
  return guard([&] {
    int k = 0;
    check_cuda(cudaGetDeviceCount(&k), "cudaGetDeviceCount");
    *n = k;
  });
}

int ohx_ctx_create(int device, ohx_ctx** out) {
  return guard([&] { *out = create_ctx(device); });
}

int ohx_ctx_destroy(ohx_ctx* ctx) {
  return guard([&] { destroy_ctx(ctx); });
}

int ohx_ctx_default(int device, ohx_ctx** out) {
  return guard([&] { *out = default_ctx(device); });
}

int ohx_ctx_device(const ohx_ctx* ctx) { return ctx ? ctx->device : -1; }

uint64_t ohx_ctx_launches(const ohx_ctx* ctx) { return ctx ? ctx->launches : 0; }

int ohx_ctx_last_run(const ohx_ctx* ctx, ohx_run_info* info) {
  return guard([&] { *info = ctx->last_run; });
}

int ohx_ctx_kernel_ms(ohx_ctx* ctx, double ms[4]) {
  return guard([&] {
    std::lock_guard<std::mutex> g(ctx->mu);
    bind(ctx);
    for (int k = 0; k < 4; ++k) {
      ms[k] = -1.0;
      if (!ctx->timed[k]) continue;
      float v = 0.f;
      check_cuda(cudaEventSynchronize(ctx->ev[k][1]), "cudaEventSynchronize");
      check_cuda(cudaEventElapsedTime(&v, ctx->ev[k][0], ctx->ev[k][1]), "cudaEventElapsedTime");
      ms[k] = v;
    }
  });
}

int ohx_extremes(ohx_ctx* ctx, const double* d_xy, uint64_t n, uint64_t index_base,
                 ohx_extremes_rec* h_rec, void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> g(ctx->mu);
    bind(ctx);
    extremes(ctx, d_xy, n, index_base, h_rec, pick(ctx, stream));
  });
}

int ohx_pts2_count(const char* path, uint64_t* n) {
  return guard([&] { *n = pts2_count(path); });
}

int ohx_pts2_load_device(ohx_ctx* ctx, const char* path, double* d_xy, uint64_t cap, uint64_t* n,
                         void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> g(ctx->mu);
    bind(ctx);
    *n = load_pts2_device(ctx, path, d_xy, cap, pick(ctx, stream));
  });
}

int ohx_fused_extremes(ohx_ctx* ctx, const double* d_xy, uint64_t n, uint64_t index_base,
                       ohx_extremes_rec* h_rec, int* fused, void* stream) {
  return guard([&] {
    if (n == 0) throw std::invalid_argument("find_extremes: empty point set");
    std::lock_guard<std::mutex> g(ctx->mu);
    bind(ctx);
    for (bool& t : ctx->timed) t = false;
    FilterOut f{};
    Trace tr;
    *fused = fused_begin(ctx, d_xy, n, index_base, f, h_rec, pick(ctx, stream), tr) ? 1 : 0;
    ctx->last_run = {};
    ctx->last_run.candidates = f.candidates;
    ctx->last_run.fuse_state = f.fuse_state;
    ctx->last_run.sample_coverage = f.sample_coverage;
  });
}

int ohx_filter_fused(ohx_ctx* ctx, const double* d_xy, uint64_t n, uint64_t index_base,
                     const ohx_extreme_set* ext, const ohx_filter_plan* plan, uint8_t* d_labels,
                     uint64_t h_counts[4], int* fused, void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> g(ctx->mu);
    bind(ctx);
    FilterOut f{};
    fused_finish(ctx, d_xy, n, index_base, *ext, *plan, d_labels, h_counts, f, pick(ctx, stream));
    *fused = f.fused ? 1 : 0;
    ctx->last_run.fused = f.fused;
    ctx->last_run.fuse_state = f.fuse_state;
    for (int q = 0; q < 4; ++q) ctx->last_run.counts[q] = h_counts[q];
  });
}

int ohx_extremes_combine(const ohx_extremes_rec* recs, int k, ohx_extremes_rec* out) {
  return guard([&] { combine_extremes(recs, k, out); });
}

int ohx_extremes_resolve(const ohx_extremes_rec* rec, ohx_extreme_set* out,
                         uint32_t* uncertified_mask) {
  return guard([&] {
    const std::uint32_t m = resolve_extremes(*rec, out);
    if (uncertified_mask) *uncertified_mask = m;
  });
}

int ohx_corners_exact(ohx_ctx* ctx, const double* d_xy, uint64_t n,
                      uint64_t index_base, const double bbox[4],
                      ohx_corner_rec* h_rec, void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> g(ctx->mu);
    bind(ctx);
    corners_exact(ctx, d_xy, n, index_base, bbox, h_rec, pick(ctx, stream));
  });
}

int ohx_corners_combine(const ohx_corner_rec* recs, int k, ohx_corner_rec* out) {
  return guard([&] { combine_corners(recs, k, out); });
}

int ohx_build_octagon(const double cand_xy[16], double oct_xy[16], int* m) {
  return guard([&] { *m = build_octagon(cand_xy, oct_xy); });
}

int ohx_filter_plan_build(const ohx_extreme_set* ext, const double* oct_xy, int m,
                          ohx_filter_plan* plan) {
  return guard([&] { make_plan(*ext, oct_xy, m, plan); });
}

int ohx_filter(ohx_ctx* ctx, const double* d_xy, uint64_t n, uint64_t index_base,
               const ohx_filter_plan* plan, uint8_t* d_labels, uint64_t h_counts[4],
               void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> g(ctx->mu);
    bind(ctx);
    filter(ctx, d_xy, n, index_base, *plan, d_labels, h_counts, pick(ctx, stream));
  });
}

int ohx_queue_fetch(ohx_ctx* ctx, int q, uint64_t* h_idx, double* h_xy, uint64_t cap,
                    void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> g(ctx->mu);
    bind(ctx);
    queue_fetch(ctx, q, h_idx, h_xy, cap, pick(ctx, stream));
  });
}

int ohx_queue_device(ohx_ctx* ctx, int q, const void** d_idx, int* idx_bytes,
                     uint64_t* count) {
  return guard([&] {
    if (q < 1 || q > 4) throw std::invalid_argument("queue must be 1..4");
    *d_idx = static_cast<const char*>(ctx->d_queues) +
             std::uint64_t(q - 1) * ctx->last_cap * ctx->last_idx_bytes;
    *idx_bytes = ctx->last_idx_bytes;
    *count = ctx->last_counts[q - 1];
  });
}

}  // extern "C"
