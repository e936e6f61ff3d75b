// octohull_api.cpp -- the octohull C++ API (include/octohull/*.hpp) on top
// of the B200 layer.  Host-point entry points upload the points to the
// process-wide device context (ohx_ctx_default) and run the kernels there;
// the reference semantics each function keeps are cited inline
// (paths relative to /root/reference/proj).
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>

#include "internal.hpp"
#include "octohull/filter.hpp"
#include "octohull/geometry.hpp"
#include "octohull/hull.hpp"
#include "octohull/parallel.hpp"
#include "octohull/pointgen.hpp"
#include "pipeline.hpp"

namespace octohull {
namespace {

using Clock = std::chrono::steady_clock;

double ms(Clock::time_point a, Clock::time_point b) {
  return std::chrono::duration<double, std::milli>(b - a).count();
}

const double* raw(std::span<const Point2D> pts) {
  return reinterpret_cast<const double*>(pts.data());
}

// Exclusive use of the default device context for one API call; the
// caller's engine grants the call its host lanes (staging copies of
// pageable input and labels run on that many threads).
struct Device {
  ohx_ctx* c;
  std::unique_lock<std::mutex> lock;
  cudaStream_t s;
  explicit Device(std::size_t workers = 0)
      : c(ohx::default_ctx()), lock(ohx::ctx_mutex(c)), s(ohx::ctx_stream(c)) {
    ohx::ctx_bind(c);
    const int own = ohx::api_lanes_override();
    ohx::ctx_set_host_lanes(c, own >= 0 ? own : static_cast<int>(std::min<std::size_t>(workers, 1024)));
  }
  explicit Device(const ReduceEngine* e) : Device(e ? e->config().workers : 0) {}
  ~Device() { ohx::ctx_set_host_lanes(c, 0); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
};

ohx_extreme_set to_set(const ExtremeSet& e, std::span<const Point2D> pts) {
  ohx_extreme_set s{};
  const std::size_t idx[8] = {e.axis.east, e.axis.north, e.axis.west, e.axis.south,
                              e.corner.ne, e.corner.nw,  e.corner.sw, e.corner.se};
  for (int a = 0; a < 8; ++a) {
    if (idx[a] >= pts.size()) throw std::invalid_argument("extreme index out of range");
    s.ext[a] = idx[a];
    s.x[a] = pts[idx[a]].x;
    s.y[a] = pts[idx[a]].y;
  }
  return s;
}

ExtremeSet from_set(const ohx_extreme_set& s) {
  ExtremeSet e;
  e.axis = {s.ext[OHX_EAST], s.ext[OHX_NORTH], s.ext[OHX_WEST], s.ext[OHX_SOUTH]};
  e.corner = {s.ext[OHX_NE], s.ext[OHX_NW], s.ext[OHX_SW], s.ext[OHX_SE]};
  return e;
}

// Host hull on the device queues of the last filter (reference
// hull.cpp:164-183): survivor coordinates are gathered on the device in
// queue (= index) order and copied back, then chained on the host.
HullPolygon hull_from_device(Device& d, const ohx::FilterOut& f) {
  HullPolygon h;
  ohx::device_queues_hull(d.c, f, d.s, [&](std::size_t n) {
    h.vertices.resize(n);
    return reinterpret_cast<ohx::P2*>(h.vertices.data());
  });
  return h;
}

// ReduceConfig.workers mapped to devices (SURVEY §7 hard part 8): a call
// whose engine grants w > 1 workers shards its points over min(w, visible
// devices) GPUs through the NCCL layer (mg.cpp), a contiguous index range
// each; results are identical.  OHX_MG_VSHARDS=k (tests) routes every such
// call through that layer with k shards per device, also on one GPU.
struct MgPlan {
  int devices = 1, vshards = 1;
  bool use() const { return devices > 1 || vshards > 1; }
};
MgPlan mg_plan(std::size_t w) {
  static const int forced = [] {
    const char* v = std::getenv("OHX_MG_VSHARDS");
    return v ? std::max(0, std::atoi(v)) : 0;
  }();
  MgPlan p;
  int nd = 0;
  if (cudaGetDeviceCount(&nd) != cudaSuccess) {
    cudaGetLastError();
    nd = 0;
  }
  if (nd > 1 && w > 1) p.devices = static_cast<int>(std::min<std::size_t>(w, nd));
  if (forced >= 1) p.vshards = forced;
  return p;
}

}  // namespace

// ================================================================ geometry
PolygonLocation point_in_convex_polygon(const Point2D& p, std::span<const Point2D> poly) {
  // reference geometry.cpp:8-25
  if (poly.size() < 3)
    throw std::invalid_argument(
        "point_in_convex_polygon: polygon needs at least 3 vertices, got " +
        std::to_string(poly.size()));
  bool boundary = false;
  for (std::size_t i = 0; i < poly.size(); ++i) {
    const int o = orientation(poly[i], poly[i + 1 == poly.size() ? 0 : i + 1], p);
    if (o < 0) return PolygonLocation::Outside;
    boundary |= o == 0;
  }
  return boundary ? PolygonLocation::OnBoundary : PolygonLocation::StrictlyInside;
}

void require_finite(std::span<const Point2D> pts) {
  // reference geometry.cpp:27-34
  for (std::size_t j = 0; j < pts.size(); ++j)
    if (!std::isfinite(pts[j].x) || !std::isfinite(pts[j].y))
      throw std::invalid_argument("non-finite coordinate at point index " + std::to_string(j));
}

// ============================================================ ReduceEngine
ReduceEngine::ReduceEngine(ReduceConfig cfg) : cfg_(cfg) {
  // reference parallel.cpp:7-18
  if (cfg_.chunk_size < 1) throw std::invalid_argument("ReduceConfig.chunk_size must be >= 1");
  if (cfg_.workers < 1) throw std::invalid_argument("ReduceConfig.workers must be >= 1");
  for (std::size_t w = 1; w < cfg_.workers; ++w) pool_.emplace_back([this] { worker(); });
}

ReduceEngine::~ReduceEngine() {
  {
    std::lock_guard<std::mutex> g(mu_);
    quit_ = true;
  }
  wake_.notify_all();
  for (auto& t : pool_) t.join();
}

std::size_t ReduceEngine::argmin(std::span<const double> keys) {
  return argmin_by(keys.size(), [keys](std::size_t i) { return keys[i]; });
}

std::size_t ReduceEngine::argmax(std::span<const double> keys) {
  return argmax_by(keys.size(), [keys](std::size_t i) { return keys[i]; });
}

std::size_t ReduceEngine::lanes_for(std::size_t n) const {
  const std::size_t chunks = (n + cfg_.chunk_size - 1) / cfg_.chunk_size;
  return std::max<std::size_t>(1, std::min(cfg_.workers, chunks));
}

void ReduceEngine::for_each_lane(std::size_t n, const LaneFn& fn) {
  // contiguous chunk-aligned lane ranges; lane 0 on the caller
  const std::size_t lanes = lanes_for(n);
  const std::size_t chunks = (n + cfg_.chunk_size - 1) / cfg_.chunk_size;
  auto range = [&](std::size_t lane) {
    const std::size_t c0 = lane * chunks / lanes, c1 = (lane + 1) * chunks / lanes;
    fn(lane, c0 * cfg_.chunk_size, std::min(c1 * cfg_.chunk_size, n));
  };
  if (lanes == 1) {
    fn(0, 0, n);
    return;
  }
  const std::function<void(std::size_t)> task = range;
  {
    std::lock_guard<std::mutex> g(mu_);
    task_ = &task;
    task_lanes_ = lanes;
    next_ = 1;
  }
  wake_.notify_all();
  range(0);
  std::unique_lock<std::mutex> g(mu_);
  idle_.wait(g, [this] { return next_ >= task_lanes_ && busy_ == 0; });
  task_ = nullptr;
}

void ReduceEngine::worker() {
  std::unique_lock<std::mutex> g(mu_);
  for (;;) {
    wake_.wait(g, [this] { return quit_ || (task_ && next_ < task_lanes_); });
    if (quit_) return;
    const std::size_t lane = next_++;
    const auto* t = task_;
    ++busy_;
    g.unlock();
    (*t)(lane);
    g.lock();
    --busy_;
    if (next_ >= task_lanes_ && busy_ == 0) idle_.notify_all();
  }
}

// ================================================================ pointgen
std::string to_string(Distribution dist) {
  switch (dist) {
    case Distribution::Normal: return "normal";
    case Distribution::Square: return "square";
    case Distribution::Disk: return "disk";
    case Distribution::Circle: return "circle";
  }
  throw std::invalid_argument("unknown distribution value");
}

Distribution parse_distribution(const std::string& token) {
  if (token == "normal") return Distribution::Normal;
  if (token == "square") return Distribution::Square;
  if (token == "disk") return Distribution::Disk;
  if (token == "circle") return Distribution::Circle;
  throw std::invalid_argument("unknown distribution '" + token +
                              "' (expected normal|square|disk|circle)");
}

PointSet generate(const GenSpec& spec) {
  // reference pointgen.cpp:44-88, produced in parallel (pointgen.cpp here)
  if (spec.n < 1) throw std::invalid_argument("generate: n must be >= 1");
  PointSet pts(spec.n);
  ohx::generate_points(static_cast<int>(spec.dist), spec.n, spec.seed, spec.distort_pct,
                       reinterpret_cast<double*>(pts.data()), 0);
  return pts;
}

// ================================================================== filter
AxisExtremes find_axis_extremes(std::span<const Point2D> pts, ReduceEngine& engine) {
  // reference filter.cpp:8-23 -> K1
  if (pts.empty()) throw std::invalid_argument("find_axis_extremes: empty point set");
  Device d(&engine);
  const double* dx = ohx::stage_points(d.c, raw(pts), pts.size(), d.s);
  ohx_extremes_rec rec;
  ohx::extremes(d.c, dx, pts.size(), 0, &rec, d.s);
  return {rec.idx[OHX_EAST], rec.idx[OHX_NORTH], rec.idx[OHX_WEST], rec.idx[OHX_SOUTH]};
}

CornerExtremes find_corner_extremes(std::span<const Point2D> pts, const AxisExtremes& axis,
                                    ReduceEngine& engine) {
  // reference filter.cpp:25-45 -> K1b against the caller's axis extremes
  if (pts.empty()) throw std::invalid_argument("find_corner_extremes: empty point set");
  const double bbox[4] = {pts[axis.east].x, pts[axis.north].y, pts[axis.west].x,
                          pts[axis.south].y};
  Device d(&engine);
  const double* dx = ohx::stage_points(d.c, raw(pts), pts.size(), d.s);
  ohx_corner_rec rec;
  ohx::corners_exact(d.c, dx, pts.size(), 0, bbox, &rec, d.s);
  return {rec.idx[0], rec.idx[1], rec.idx[2], rec.idx[3]};
}

ExtremeSet find_extremes(std::span<const Point2D> pts, ReduceEngine& engine) {
  // reference filter.cpp:47-52 -> K1 + corner certificate (+ K1b)
  if (pts.empty()) throw std::invalid_argument("find_axis_extremes: empty point set");
  Device d(&engine);
  const double* dx = ohx::stage_points(d.c, raw(pts), pts.size(), d.s);
  ohx_extremes_rec rec;
  ohx::extremes(d.c, dx, pts.size(), 0, &rec, d.s);
  ohx_extreme_set set;
  if (ohx::resolve_extremes(rec, &set)) {
    const double bbox[4] = {rec.x[OHX_EAST], rec.y[OHX_NORTH], rec.x[OHX_WEST],
                            rec.y[OHX_SOUTH]};
    ohx_corner_rec cr;
    ohx::corners_exact(d.c, dx, pts.size(), 0, bbox, &cr, d.s);
    ohx::apply_corners(cr, &set);
  }
  return from_set(set);
}

Octagon build_octagon(std::span<const Point2D> pts, const ExtremeSet& ext) {
  // reference filter.cpp:54-86 (host; <= 8 points)
  double cand[16], oct[16];
  const auto c = ext.candidates();
  for (int k = 0; k < 8; ++k) {
    cand[2 * k] = pts[c[k]].x;
    cand[2 * k + 1] = pts[c[k]].y;
  }
  const int m = ohx::build_octagon(cand, oct);
  Octagon o;
  o.vertices.resize(m);
  std::memcpy(static_cast<void*>(o.vertices.data()), oct, sizeof(double) * 2 * m);
  return o;
}

int find_queue(const Point2D& p, const ExtremeSet& ext, std::span<const Point2D> pts) {
  // reference filter.cpp:88-102 (single point, host)
  const Point2D& e = pts[ext.axis.east];
  const Point2D& n = pts[ext.axis.north];
  const Point2D& w = pts[ext.axis.west];
  const Point2D& s = pts[ext.axis.south];
  if (orientation(e, n, p) < 0) return 1;
  if (orientation(n, w, p) < 0) return 2;
  if (orientation(w, s, p) < 0) return 3;
  if (orientation(s, e, p) < 0) return 4;
  return 1;
}

LabelArray classify_points(std::span<const Point2D> pts, const Octagon& oct,
                           const ExtremeSet& ext, ReduceEngine& engine) {
  // reference filter.cpp:104-131 -> K2 with the caller's octagon/extremes
  if (pts.empty()) return {};
  const ohx_extreme_set set = to_set(ext, pts);
  if (oct.vertices.size() > 8) {  // any vertex list is accepted (filter.cpp:118-128)
    Device d(&engine);
    const double* dx = ohx::stage_points(d.c, raw(pts), pts.size(), d.s);
    std::uint8_t* dl = ohx::stage_labels(d.c, pts.size());
    ohx::polygon_labels(d.c, dx, pts.size(), reinterpret_cast<const double*>(oct.vertices.data()),
                        static_cast<int>(oct.vertices.size()), set, dl, d.s);
    LabelArray labels(pts.size());
    ohx::fetch_labels(d.c, labels.data(), dl, pts.size(), d.s);
    ohx::check_cuda(cudaStreamSynchronize(d.s), "classify_points");
    return labels;
  }
  ohx_filter_plan plan;
  ohx::make_plan(set, reinterpret_cast<const double*>(oct.vertices.data()),
                 static_cast<int>(oct.vertices.size()), &plan);
  Device d(&engine);
  const double* dx = ohx::stage_points(d.c, raw(pts), pts.size(), d.s);
  std::uint8_t* dl = ohx::stage_labels(d.c, pts.size());
  std::uint64_t counts[4];
  ohx::filter(d.c, dx, pts.size(), 0, plan, dl, counts, d.s);
  LabelArray labels(pts.size());
  ohx::fetch_labels(d.c, labels.data(), dl, pts.size(), d.s);
  ohx::check_cuda(cudaStreamSynchronize(d.s), "classify_points");
  return labels;
}

// ==================================================================== hull
QuadQueues build_queues(const LabelArray& labels) {
  // reference hull.cpp:124-131 (host labels in, host queues out)
  QuadQueues q;
  for (std::size_t j = 0; j < labels.size(); ++j)
    if (labels[j] != 0) q.queue[labels[j] - 1].push_back(j);
  return q;
}

std::vector<Point2D> quadrant_hull(std::vector<Point2D> pts, int quadrant) {
  std::vector<ohx::P2> p(pts.size());
  std::memcpy(p.data(), pts.data(), pts.size() * sizeof(Point2D));
  const ohx::PVec c = ohx::quadrant_chain(std::move(p), quadrant);
  std::vector<Point2D> out(c.size());
  std::memcpy(static_cast<void*>(out.data()), c.data(), c.size() * sizeof(Point2D));
  return out;
}

HeaphullRun heaphull_run(std::span<const Point2D> pts, ReduceEngine& engine) {
  // reference hull.cpp:152-194: same stages and timer boundaries
  if (pts.empty()) throw std::invalid_argument("heaphull: empty point set");
  const auto t0 = Clock::now();
  if (const MgPlan mp = mg_plan(engine.config().workers); mp.use()) {
    HeaphullRun run;
    run.labels.resize(pts.size());
    ohx_mg_info info;
    ohx::mg_heaphull_host(ohx::mg_default(mp.devices), raw(pts), pts.size(), mp.vshards,
                          run.labels.data(), [&](std::size_t h) {
                            run.hull.vertices.resize(h);
                            return reinterpret_cast<ohx::P2*>(run.hull.vertices.data());
                          }, &info);
    run.total_ms = ms(t0, Clock::now());
    run.filter_ms = info.ms[0] + info.ms[1];
    run.hull_ms = std::max(0.0, run.total_ms - run.filter_ms);
    return run;
  }
  Device d(&engine);
  const double* dx = ohx::stage_points(d.c, raw(pts), pts.size(), d.s);
  std::uint8_t* dl = ohx::stage_labels(d.c, pts.size());
  const ohx::FilterOut f = ohx::device_filter(d.c, dx, pts.size(), dl, d.s);
  HeaphullRun run;
  run.labels.resize(pts.size());
  ohx::fetch_labels(d.c, run.labels.data(), dl, pts.size(), d.s);
  ohx::check_cuda(cudaStreamSynchronize(d.s), "heaphull_run");
  const auto t1 = Clock::now();
  run.hull = hull_from_device(d, f);
  const auto t2 = Clock::now();
  run.filter_ms = ms(t0, t1);
  run.hull_ms = ms(t1, t2);
  run.total_ms = ms(t0, t2);
  return run;
}

namespace {
// heaphull over `workers` host lanes / devices (labels not materialised)
HullPolygon heaphull_with(std::span<const Point2D> pts, std::size_t workers) {
  if (pts.empty()) throw std::invalid_argument("heaphull: empty point set");
  if (const MgPlan mp = mg_plan(workers); mp.use()) {
    HullPolygon hull;
    ohx::mg_heaphull_host(ohx::mg_default(mp.devices), raw(pts), pts.size(), mp.vshards, nullptr,
                          [&](std::size_t h) {
                            hull.vertices.resize(h);
                            return reinterpret_cast<ohx::P2*>(hull.vertices.data());
                          }, nullptr);
    return hull;
  }
  Device d(workers);
  const double* dx = ohx::stage_points(d.c, raw(pts), pts.size(), d.s);
  const ohx::FilterOut f = ohx::device_filter(d.c, dx, pts.size(), nullptr, d.s);
  return hull_from_device(d, f);
}
}  // namespace

HullPolygon heaphull(std::span<const Point2D> pts, ReduceEngine& engine) {
  // reference hull.cpp:196-198
  return heaphull_with(pts, engine.config().workers);
}

HullPolygon heaphull(std::span<const Point2D> pts, ReduceConfig cfg) {
  // reference hull.cpp:200-203; the config is validated as ReduceEngine
  // would (parallel.cpp:8-13), without starting its threads
  if (cfg.chunk_size < 1) throw std::invalid_argument("ReduceConfig.chunk_size must be >= 1");
  if (cfg.workers < 1) throw std::invalid_argument("ReduceConfig.workers must be >= 1");
  return heaphull_with(pts, cfg.workers);
}

HullPolygon monotone_chain_hull(std::span<const Point2D> pts) {
  // reference hull.cpp:205-232 (host; the independent check)
  if (pts.empty()) throw std::invalid_argument("monotone_chain_hull: empty point set");
  const ohx::PVec c =
      ohx::monotone_chain(reinterpret_cast<const ohx::P2*>(pts.data()), pts.size());
  HullPolygon h;
  h.vertices.resize(c.size());
  std::memcpy(static_cast<void*>(h.vertices.data()), c.data(), c.size() * sizeof(Point2D));
  return h;
}

double filter_rate(const LabelArray& labels) {
  // reference hull.cpp:234-241
  if (labels.empty()) throw std::invalid_argument("filter_rate: empty label array");
  const auto zeros = static_cast<double>(std::count(labels.begin(), labels.end(), Label{0}));
  return zeros / static_cast<double>(labels.size());
}

bool same_cycle(std::span<const Point2D> a, std::span<const Point2D> b) {
  // reference hull.cpp:243-255
  if (a.size() != b.size()) return false;
  if (a.empty()) return true;
  for (std::size_t s = 0; s < b.size(); ++s) {
    if (!(b[s] == a[0])) continue;
    std::size_t i = 1;
    while (i < a.size() && a[i] == b[(s + i) % b.size()]) ++i;
    if (i == a.size()) return true;
  }
  return false;
}

}  // namespace octohull
