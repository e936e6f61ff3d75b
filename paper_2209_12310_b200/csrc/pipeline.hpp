// pipeline.hpp -- internal orchestration shared by the pipeline-level C ABI
// (pipeline.cpp) and the C++ API (octohull_api.cpp).  Functions throw
// std::invalid_argument for contract violations and ohx::Error otherwise;
// callers hold ctx_mutex(ctx) and have bound the context's device.
#pragma once

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "internal.hpp"
#include "ohx.h"

namespace ohx {

struct FilterOut {
  ohx_extreme_set ext;  // resolved ExtremeSet (+ coordinates)
  double oct[16];       // octagon (build_octagon) ...
  int m;                // ... and its vertex count
  ohx_filter_plan plan;
  std::uint64_t counts[4];
  bool corner_pass;  // the certificate failed and K1b ran
  bool fused;        // single pass: K2 ran on the fused pass's candidates only
  std::uint64_t candidates;
  std::uint32_t fuse_state;  // ohx_run_info.fuse_state
  double sample_coverage;
};

// Host lanes of C++ API calls made on this thread (-1: the caller's
// ReduceEngine workers decide).  The C ABI's pipeline wrappers, which
// construct a one-worker engine only to call the C++ API, grant all cores.
int api_lanes_override();
struct ApiLanes {
  explicit ApiLanes(int lanes);
  ~ApiLanes();
  int saved;
};

ohx_ctx* create_ctx(int device);
void destroy_ctx(ohx_ctx* c);
void trim_ctx(ohx_ctx* c);
ohx_ctx* default_ctx(int device = -1);
cudaStream_t ctx_stream(ohx_ctx* c);
std::mutex& ctx_mutex(ohx_ctx* c);
void ctx_bind(ohx_ctx* c);
// host threads of the staging copies for the calls that follow (0: all)
void ctx_set_host_lanes(ohx_ctx* c, int lanes);

const double* stage_points(ohx_ctx* c, const double* h_xy, std::uint64_t n,
                           cudaStream_t s);
std::uint8_t* stage_labels(ohx_ctx* c, std::uint64_t n);
// a PTS2 file into the context's device point buffer (*n points)
const double* stage_pts2(ohx_ctx* c, const std::string& path, std::uint64_t* n, cudaStream_t s);
// labels back into a (possibly pageable) host buffer; synchronous
void fetch_labels(ohx_ctx* c, std::uint8_t* h_labels, const std::uint8_t* d_labels,
                  std::uint64_t n, cudaStream_t s);

void extremes(ohx_ctx* c, const double* d_xy, std::uint64_t n, std::uint64_t base,
              ohx_extremes_rec* out, cudaStream_t s);
void corners_exact(ohx_ctx* c, const double* d_xy, std::uint64_t n,
                   std::uint64_t base, const double bbox[4], ohx_corner_rec* out,
                   cudaStream_t s);
void combine_extremes(const ohx_extremes_rec* recs, int k, ohx_extremes_rec* out);
void combine_corners(const ohx_corner_rec* recs, int k, ohx_corner_rec* out);
std::uint32_t resolve_extremes(const ohx_extremes_rec& r, ohx_extreme_set* out);
void apply_corners(const ohx_corner_rec& c, ohx_extreme_set* ext);
int build_octagon(const double cand[16], double oct[16]);
// with_box = false leaves the certified interior box empty (K2 then tests
// every point exactly): the fused pass's K2 sees only points outside its
// provisional region, which the box would not hold -- ensure_box fills it
// in when the call falls back to a K2 over all points
void make_plan(const ohx_extreme_set& e, const double* oct, int m,
               ohx_filter_plan* p, bool with_box = true);
void ensure_box(ohx_filter_plan* p);
void filter(ohx_ctx* c, const double* d_xy, std::uint64_t n, std::uint64_t base,
            const ohx_filter_plan& plan, std::uint8_t* d_labels,
            std::uint64_t counts[4], cudaStream_t s);
// classify_points' labels against a caller's polygon of m > 8 vertices
void polygon_labels(ohx_ctx* c, const double* d_xy, std::uint64_t n, const double* poly, int m,
                    const ohx_extreme_set& ext, std::uint8_t* d_labels, cudaStream_t s);
void queue_fetch(ohx_ctx* c, int q, std::uint64_t* h_idx, double* h_xy,
                 std::uint64_t cap, cudaStream_t s);

// survivor coordinates of all four queues, packed [q1|q2|q3|q4], one launch
void queues_fetch_xy(ohx_ctx* c, double* h_xy, cudaStream_t s);

// hull stage on survivor coordinates packed on the device [q1|q2|q3|q4]
// (dev: sink hands out DEVICE memory -- the hull stays on the device)
std::size_t hull_from_packed(ohx_ctx* c, const double* d_packed, const std::uint64_t counts[4],
                             const P2 anchors[4], cudaStream_t s, const HullSink& sink,
                             bool dev = false);
// hull stage on survivor coordinates already in host memory, packed
// [q1|q2|q3|q4]: the host hull stage below device_sort_min() survivors,
// else one H2D through the context's gather buffer and hull_from_packed
std::size_t hull_from_host_packed(ohx_ctx* c, const P2* h_packed, const std::uint64_t counts[4],
                                  const P2 anchors[4], cudaStream_t s, const HullSink& sink);
// host hull stage on the queues of the last filter (survivors gathered and
// copied back in one launch)
PVec device_queues_hull(ohx_ctx* c, const FilterOut& f, cudaStream_t s);
// ... written to sink(h) instead (the caller's buffer); returns h
std::size_t device_queues_hull(ohx_ctx* c, const FilterOut& f, cudaStream_t s,
                               const HullSink& sink, bool dev = false);

// K1 -> certificate -> (K1b) -> octagon -> plan -> K2 on one device
FilterOut device_filter(ohx_ctx* c, const double* d_xy, std::uint64_t n,
                        std::uint8_t* d_labels, cudaStream_t s);

// ---- multi-GPU (mg.cpp)
// process-wide single-process communicator over devices 0..ndev-1
ohx_mg* mg_default(int ndev);
// host points over the handle's devices (vshards shards each), labels
// (nullable) for every point; the hull to sink
std::size_t mg_heaphull_host(ohx_mg* M, const double* h_xy, std::uint64_t n, int vshards,
                             std::uint8_t* h_labels, const HullSink& sink, ohx_mg_info* info);

}  // namespace ohx
