// pipeline.cpp -- pipeline-level C ABI (include/ohx.h): the entry points the
// reference binds to Python (python/module.cpp:40-108), each a thin
// exception-safe wrapper over the C++ API of octohull_api.cpp, plus the
// device-resident variant used for the kernel-level throughput numbers.
#include <chrono>
#include <cstring>
#include <span>
#include <string>

#include "internal.hpp"
#include "host.hpp"
#include "octohull/filter.hpp"
#include "octohull/hull.hpp"
#include "octohull/pointgen.hpp"
#include "ohx.h"
#include "pipeline.hpp"

namespace {

using Clock = std::chrono::steady_clock;

double ms(Clock::time_point a, Clock::time_point b) {
  return std::chrono::duration<double, std::milli>(b - a).count();
}

std::span<const octohull::Point2D> pts_of(const double* xy, std::uint64_t n) {
  return {reinterpret_cast<const octohull::Point2D*>(xy), static_cast<std::size_t>(n)};
}

void copy_hull(const std::vector<octohull::Point2D>& v, double* out, std::uint64_t cap,
               std::uint64_t* h) {
  *h = v.size();
  if (v.size() > cap) throw std::invalid_argument("hull output capacity too small");
  ohx::copy_points(reinterpret_cast<ohx::P2*>(out), reinterpret_cast<const ohx::P2*>(v.data()),
                   v.size());
}

// The caller's output buffer, visible to the hull stage for one call: a
// device buffer (the cycle is chained straight into it) or a host buffer
// (page-locked: the pipelined stage streams the hull into it).
struct OutScope {
  ohx_ctx* c;
  OutScope(ohx_ctx* c_, double* p, std::uint64_t cap, bool device) : c(c_) {
    if (device) {
      c->dev_out = p;
      c->dev_out_cap = cap;
    } else {  // (whether it is page-locked is asked only when it matters)
      c->host_out = p;
      c->host_out_cap = cap;
    }
  }
  ~OutScope() {
    c->dev_out = c->host_out = nullptr;
    c->dev_out_cap = c->host_out_cap = 0;
  }
};

// the caller's hull buffer as the hull stage's sink (capacity checked, the
// size reported either way)
ohx::HullSink hull_sink(double* h_hull, std::uint64_t cap, std::uint64_t* h) {
  return [=](std::size_t hh) {
    *h = hh;
    if (hh > cap) throw std::invalid_argument("hull output capacity too small");
    return reinterpret_cast<ohx::P2*>(h_hull);
  };
}

}  // namespace

namespace ohx {
namespace {
thread_local int tl_api_lanes = -1;
}
int api_lanes_override() { return tl_api_lanes; }
ApiLanes::ApiLanes(int lanes) : saved(tl_api_lanes) { tl_api_lanes = lanes; }
ApiLanes::~ApiLanes() { tl_api_lanes = saved; }
}  // namespace ohx

using ohx::guard;

extern "C" {

int ohx_heaphull(const double* h_xy, uint64_t n, double* h_hull, uint64_t cap, uint64_t* h,
                 double* timings) {
  // octohull::heaphull (hull.cpp:196-198) without the intermediate
  // std::vector<Point2D>: the hull goes straight into the caller's buffer
  return guard([&] {
    if (n == 0) throw std::invalid_argument("heaphull: empty point set");
    const auto t0 = Clock::now();
    ohx_ctx* ctx = ohx::default_ctx();
    std::lock_guard<std::mutex> g(ohx::ctx_mutex(ctx));
    ohx::ctx_bind(ctx);
    cudaStream_t s = ohx::ctx_stream(ctx);
    const double* d_xy = ohx::stage_points(ctx, h_xy, n, s);
    const ohx::FilterOut f = ohx::device_filter(ctx, d_xy, n, nullptr, s);
    const auto t1 = Clock::now();
    const OutScope os(ctx, h_hull, cap, false);
    ohx::device_queues_hull(ctx, f, s, hull_sink(h_hull, cap, h));
    if (timings) {
      timings[0] = ms(t0, t1);
      timings[1] = ms(t1, Clock::now());
      timings[2] = ms(t0, Clock::now());
      timings[3] = 0.0;
    }
  });
}

int ohx_heaphull_device(ohx_ctx* ctx, const double* d_xy, uint64_t n, double* h_hull,
                        uint64_t cap, uint64_t* h, double* timings) {
  return guard([&] {
    if (n == 0) throw std::invalid_argument("heaphull: empty point set");
    std::lock_guard<std::mutex> g(ohx::ctx_mutex(ctx));
    ohx::ctx_bind(ctx);
    cudaStream_t s = ohx::ctx_stream(ctx);
    const auto t0 = Clock::now();
    const ohx::FilterOut f = ohx::device_filter(ctx, d_xy, n, nullptr, s);
    const auto t1 = Clock::now();
    const OutScope os(ctx, h_hull, cap, false);
    ohx::device_queues_hull(ctx, f, s, hull_sink(h_hull, cap, h));
    const auto t2 = Clock::now();
    if (timings) {
      timings[0] = ms(t0, t1);
      timings[1] = ms(t1, t2);
      timings[2] = ms(t0, t2);
      timings[3] = 0.0;
    }
  });
}

int ohx_heaphull_device_out(ohx_ctx* ctx, const double* d_xy, uint64_t n, double* d_hull,
                            uint64_t cap, uint64_t* h, double* timings) {
  return guard([&] {
    if (n == 0) throw std::invalid_argument("heaphull: empty point set");
    std::lock_guard<std::mutex> g(ohx::ctx_mutex(ctx));
    ohx::ctx_bind(ctx);
    cudaStream_t s = ohx::ctx_stream(ctx);
    const auto t0 = Clock::now();
    const ohx::FilterOut f = ohx::device_filter(ctx, d_xy, n, nullptr, s);
    const auto t1 = Clock::now();
    const OutScope os(ctx, d_hull, cap, true);
    ohx::device_queues_hull(ctx, f, s, hull_sink(d_hull, cap, h), true);
    const auto t2 = Clock::now();
    if (timings) {
      timings[0] = ms(t0, t1);
      timings[1] = ms(t1, t2);
      timings[2] = ms(t0, t2);
      timings[3] = 0.0;
    }
  });
}

int ohx_heaphull_pts2(const char* path, double* h_hull, uint64_t cap, uint64_t* h,
                      double* timings) {
  // the reference CLI's read_points(Binary) + heaphull (tools/octohull_main
  // .cpp), with the file streamed straight into device memory
  return guard([&] {
    const auto t0 = Clock::now();
    ohx_ctx* ctx = ohx::default_ctx();
    std::lock_guard<std::mutex> g(ohx::ctx_mutex(ctx));
    ohx::ctx_bind(ctx);
    cudaStream_t s = ohx::ctx_stream(ctx);
    std::uint64_t n = 0;
    const double* d_xy = ohx::stage_pts2(ctx, path, &n, s);
    const auto tl = Clock::now();
    const ohx::FilterOut f = ohx::device_filter(ctx, d_xy, n, nullptr, s);
    const auto t1 = Clock::now();
    const OutScope os(ctx, h_hull, cap, false);
    ohx::device_queues_hull(ctx, f, s, hull_sink(h_hull, cap, h));
    if (timings) {
      timings[0] = ms(tl, t1);
      timings[1] = ms(t1, Clock::now());
      timings[2] = ms(t0, Clock::now());
      timings[3] = ms(t0, tl);  // file -> device
    }
  });
}

int ohx_classify(const double* h_xy, uint64_t n, uint8_t* h_labels) {
  return guard([&] {
    octohull::ReduceEngine engine;
    const ohx::ApiLanes all_cores(0);
    const auto pts = pts_of(h_xy, n);
    const octohull::ExtremeSet ext = octohull::find_extremes(pts, engine);
    const octohull::Octagon oct = octohull::build_octagon(pts, ext);
    const octohull::LabelArray l = octohull::classify_points(pts, oct, ext, engine);
    std::memcpy(h_labels, l.data(), l.size());
  });
}

int ohx_classify_points(const double* h_xy, uint64_t n, const double* poly_xy, uint64_t m,
                        const uint64_t ext[8], uint8_t* h_labels) {
  // octohull::classify_points (filter.cpp:104-131; python/module.cpp binds
  // it) with the caller's polygon and extremes
  return guard([&] {
    octohull::ReduceEngine engine;
    const ohx::ApiLanes all_cores(0);
    const auto pts = pts_of(h_xy, n);
    octohull::Octagon oct;
    oct.vertices.assign(reinterpret_cast<const octohull::Point2D*>(poly_xy),
                        reinterpret_cast<const octohull::Point2D*>(poly_xy) + m);
    octohull::ExtremeSet e;
    e.axis = {ext[0], ext[1], ext[2], ext[3]};
    e.corner = {ext[4], ext[5], ext[6], ext[7]};
    const octohull::LabelArray l = octohull::classify_points(pts, oct, e, engine);
    std::memcpy(h_labels, l.data(), l.size());
  });
}

int ohx_heaphull_run(const double* h_xy, uint64_t n, double* h_hull, uint64_t cap,
                     uint64_t* h, uint8_t* h_labels, double* timings) {
  return guard([&] {
    octohull::ReduceEngine engine;
    const ohx::ApiLanes all_cores(0);
    const octohull::HeaphullRun run = octohull::heaphull_run(pts_of(h_xy, n), engine);
    copy_hull(run.hull.vertices, h_hull, cap, h);
    if (h_labels) std::memcpy(h_labels, run.labels.data(), run.labels.size());
    if (timings) {
      timings[0] = run.filter_ms;
      timings[1] = run.hull_ms;
      timings[2] = run.total_ms;
      timings[3] = 0.0;
    }
  });
}

int ohx_find_extremes(const double* h_xy, uint64_t n, uint64_t ext[8]) {
  return guard([&] {
    octohull::ReduceEngine engine;
    const ohx::ApiLanes all_cores(0);
    const octohull::ExtremeSet e = octohull::find_extremes(pts_of(h_xy, n), engine);
    const uint64_t v[8] = {e.axis.east, e.axis.north, e.axis.west, e.axis.south,
                           e.corner.ne, e.corner.nw,  e.corner.sw, e.corner.se};
    std::memcpy(ext, v, sizeof(v));
  });
}

int ohx_hull_from_sorted_arcs(const double* const arcs_xy[4], const uint64_t len[4],
                              double* h_hull, uint64_t cap, uint64_t* h) {
  return guard([&] {
    const ohx::P2* arcs[4];
    for (int q = 0; q < 4; ++q) arcs[q] = reinterpret_cast<const ohx::P2*>(arcs_xy[q]);
    ohx::hull_from_sorted_arcs(arcs, len, {}, hull_sink(h_hull, cap, h));
  });
}

int ohx_hull_from_sorted_arcs_device(ohx_ctx* ctx, const double* d_arcs, const uint64_t len[4],
                                     double* h_hull, uint64_t cap, uint64_t* h, int* proven,
                                     int flags, void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> g(ohx::ctx_mutex(ctx));
    ohx::ctx_bind(ctx);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ohx::ctx_stream(ctx);
    for (int q = 0; q < 4; ++q)
      if (len[q] < 2) throw std::invalid_argument("every arc holds at least its two anchors");
    const bool raw = flags & OHX_ARCS_RAW_CYCLE;
    std::size_t hh = 0;
    const bool ok = ohx::hull_device_chains(ctx, d_arcs, len, s, hull_sink(h_hull, cap, h), &hh,
                                            raw);
    if (proven) *proven = ok ? 1 : 0;
    if (ok) return;
    const uint64_t total = len[0] + len[1] + len[2] + len[3];
    ohx::PVec all(total);
    ohx::copy_d2h(ctx, all.data(), d_arcs, total * 16, s);
    const ohx::P2* arcs[4];
    uint64_t off = 0;
    for (int q = 0; q < 4; ++q) {
      arcs[q] = all.data() + off;
      off += len[q];
    }
    if (raw) {
      const ohx::PVec cyc = ohx::chain_arcs(arcs, len, {});
      ohx::copy_points(hull_sink(h_hull, cap, h)(cyc.size()), cyc.data(), cyc.size());
      return;
    }
    ohx::hull_from_sorted_arcs(arcs, len, {}, hull_sink(h_hull, cap, h));
  });
}

int ohx_chain(const double* h_xy, uint64_t n, double* h_out, uint64_t* m) {
  return guard([&] {
    const ohx::PVec c = ohx::chain_sorted(reinterpret_cast<const ohx::P2*>(h_xy), n);
    *m = c.size();
    ohx::copy_points(reinterpret_cast<ohx::P2*>(h_out), c.data(), c.size());
  });
}

int ohx_monotone_chain(const double* h_xy, uint64_t n, double* h_hull, uint64_t cap,
                       uint64_t* h) {
  return guard([&] {
    const octohull::HullPolygon hull = octohull::monotone_chain_hull(pts_of(h_xy, n));
    copy_hull(hull.vertices, h_hull, cap, h);
  });
}

int ohx_generate(int dist, uint64_t n, uint64_t seed, double distort_pct, double* h_xy,
                 int threads) {
  return guard([&] { ohx::generate_points(dist, n, seed, distort_pct, h_xy, threads); });
}

int ohx_generate_range(int dist, uint64_t n, uint64_t seed, double distort_pct, uint64_t lo,
                       uint64_t count, double* h_xy, int threads) {
  return guard([&] {
    ohx::generate_points_range(dist, n, seed, distort_pct, lo, count, h_xy, threads);
  });
}

int ohx_hull_from_queues(const double* h_xy, const uint64_t ext_axis[4],
                         const uint64_t* const q_idx[4], const uint64_t q_len[4],
                         double* h_hull, uint64_t cap, uint64_t* h) {
  return guard([&] {
    const auto* P = reinterpret_cast<const ohx::P2*>(h_xy);
    std::vector<ohx::P2> q[4];
    const ohx::P2* qp[4];
    for (int k = 0; k < 4; ++k) {
      q[k].resize(q_len[k]);
      for (uint64_t i = 0; i < q_len[k]; ++i) q[k][i] = P[q_idx[k][i]];
      qp[k] = q[k].data();
    }
    const ohx::P2 anchors[4] = {P[ext_axis[0]], P[ext_axis[1]], P[ext_axis[2]],
                                P[ext_axis[3]]};
    const ohx::PVec cyc = ohx::hull_from_queue_points(anchors, qp, q_len);
    *h = cyc.size();
    if (cyc.size() > cap) throw std::invalid_argument("hull output capacity too small");
    ohx::copy_points(reinterpret_cast<ohx::P2*>(h_hull), cyc.data(), cyc.size());
  });
}

int ohx_hull_from_queue_points(const double anchors_xy[8], const double* const q_xy[4],
                               const uint64_t q_len[4], double* h_hull, uint64_t cap,
                               uint64_t* h) {
  return guard([&] {
    const ohx::P2* qp[4];
    for (int k = 0; k < 4; ++k) qp[k] = reinterpret_cast<const ohx::P2*>(q_xy[k]);
    const auto* A = reinterpret_cast<const ohx::P2*>(anchors_xy);
    const ohx::PVec cyc = ohx::hull_from_queue_points(A, qp, q_len);
    *h = cyc.size();
    if (cyc.size() > cap) throw std::invalid_argument("hull output capacity too small");
    ohx::copy_points(reinterpret_cast<ohx::P2*>(h_hull), cyc.data(), cyc.size());
  });
}

}  // extern "C"
