// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference
// octohull library, compiled from /root/reference/proj/src by
// oracle/Makefile into oracle/_ref/libocto_ref.so.
//
// TEST INFRASTRUCTURE ONLY: used by tests/ (to pin oracle.c and generate
// golden fixtures) and by bench.py's reference arm / cpu_baseline leg.
// The reference is built with -Doctohull=octohull_ref so its C++ symbols
// can never interpose with the product library's octohull:: symbols.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <string>

#include "octohull/filter.hpp"
#include "octohull/hull.hpp"
#include "octohull/pointgen.hpp"

namespace R = octohull_ref;

namespace {
thread_local std::string g_err;

std::span<const R::Point2D> as_points(const double* xy, std::uint64_t n) {
  return {reinterpret_cast<const R::Point2D*>(xy), static_cast<std::size_t>(n)};
}

template <typename F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_generate(int dist, std::uint64_t n, std::uint64_t seed, double distort,
                 double* xy) {
  return guarded([&] {
    R::GenSpec spec;
    spec.dist = static_cast<R::Distribution>(dist);
    spec.n = n;
    spec.seed = seed;
    spec.distort_pct = distort;
    const R::PointSet pts = R::generate(spec);
    std::memcpy(xy, pts.data(), pts.size() * sizeof(R::Point2D));
    return 0;
  });
}

int ref_find_extremes(const double* xy, std::uint64_t n, std::uint64_t workers,
                      std::uint64_t chunk, std::uint64_t ext[8]) {
  return guarded([&] {
    R::ReduceEngine engine({chunk, workers});
    const R::ExtremeSet e = R::find_extremes(as_points(xy, n), engine);
    const std::uint64_t v[8] = {e.axis.east, e.axis.north, e.axis.west,
                                e.axis.south, e.corner.ne, e.corner.nw,
                                e.corner.sw, e.corner.se};
    std::memcpy(ext, v, sizeof(v));
    return 0;
  });
}

int ref_build_octagon(const double* xy, std::uint64_t n,
                      const std::uint64_t ext[8], double oct[16]) {
  return guarded([&] {
    R::ExtremeSet e;
    e.axis = {ext[0], ext[1], ext[2], ext[3]};
    e.corner = {ext[4], ext[5], ext[6], ext[7]};
    const R::Octagon o = R::build_octagon(as_points(xy, n), e);
    std::memcpy(oct, o.vertices.data(), o.vertices.size() * sizeof(R::Point2D));
    return static_cast<int>(o.vertices.size());
  });
}

int ref_find_queue(const double* p, const double* xy, std::uint64_t n,
                   const std::uint64_t ext[8]) {
  return guarded([&] {
    R::ExtremeSet e;
    e.axis = {ext[0], ext[1], ext[2], ext[3]};
    e.corner = {ext[4], ext[5], ext[6], ext[7]};
    return R::find_queue(R::Point2D{p[0], p[1]}, e, as_points(xy, n));
  });
}

int ref_classify(const double* xy, std::uint64_t n, std::uint64_t workers,
                 std::uint64_t chunk, std::uint8_t* labels) {
  return guarded([&] {
    R::ReduceEngine engine({chunk, workers});
    const auto pts = as_points(xy, n);
    const R::ExtremeSet e = R::find_extremes(pts, engine);
    const R::Octagon o = R::build_octagon(pts, e);
    const R::LabelArray l = R::classify_points(pts, o, e, engine);
    std::memcpy(labels, l.data(), l.size());
    return 0;
  });
}

// Full reference heaphull_run.  times = {filter_ms, hull_ms, total_ms}.
std::int64_t ref_heaphull_run(const double* xy, std::uint64_t n,
                              std::uint64_t workers, std::uint64_t chunk,
                              double* hull_xy, std::uint8_t* labels,
                              double* times) {
  std::int64_t h = -1;
  guarded([&] {
    R::ReduceEngine engine({chunk, workers});
    const R::HeaphullRun run = R::heaphull_run(as_points(xy, n), engine);
    std::memcpy(hull_xy, run.hull.vertices.data(),
                run.hull.vertices.size() * sizeof(R::Point2D));
    if (labels) std::memcpy(labels, run.labels.data(), run.labels.size());
    if (times) {
      times[0] = run.filter_ms;
      times[1] = run.hull_ms;
      times[2] = run.total_ms;
    }
    h = static_cast<std::int64_t>(run.hull.vertices.size());
    return 0;
  });
  return h;
}

std::int64_t ref_monotone_chain(const double* xy, std::uint64_t n,
                                double* hull_xy) {
  std::int64_t h = -1;
  guarded([&] {
    const R::HullPolygon hull = R::monotone_chain_hull(as_points(xy, n));
    std::memcpy(hull_xy, hull.vertices.data(),
                hull.vertices.size() * sizeof(R::Point2D));
    h = static_cast<std::int64_t>(hull.vertices.size());
    return 0;
  });
  return h;
}

// A persistent engine for timing loops (the reference arm of bench.py).
void* ref_engine_new(std::uint64_t workers, std::uint64_t chunk) {
  try {
    return new R::ReduceEngine({chunk, workers});
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_engine_free(void* eng) { delete static_cast<R::ReduceEngine*>(eng); }

std::int64_t ref_engine_heaphull(void* eng, const double* xy, std::uint64_t n,
                                 double* times) {
  std::int64_t h = -1;
  guarded([&] {
    const R::HeaphullRun run =
        R::heaphull_run(as_points(xy, n), *static_cast<R::ReduceEngine*>(eng));
    if (times) {
      times[0] = run.filter_ms;
      times[1] = run.hull_ms;
      times[2] = run.total_ms;
    }
    h = static_cast<std::int64_t>(run.hull.vertices.size());
    return 0;
  });
  return h;
}

}  // extern "C"
