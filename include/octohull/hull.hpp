// octohull/hull.hpp -- B200 build of the octohull public API.
//
// Declaration-compatible with the reference header
// (/root/reference/proj/include/octohull/hull.hpp:15-73).  heaphull_run and
// heaphull filter on the GPU (kernels K1/K2, survivors compacted into the
// four queues on the device) and then run the host hull stage with the
// reference's semantics on the survivors only.
#pragma once

#include <array>
#include <span>
#include <vector>

#include "octohull/filter.hpp"
#include "octohull/geometry.hpp"
#include "octohull/parallel.hpp"

namespace octohull {

// Surviving indices per quadrant, ascending; q is 1-based.
struct QuadQueues {
  std::array<std::vector<std::size_t>, 4> queue;

  std::vector<std::size_t>& operator[](int q) { return queue[q - 1]; }
  const std::vector<std::size_t>& operator[](int q) const { return queue[q - 1]; }
};

// CCW cycle of strict hull vertices (1 or 2 for degenerate inputs).
struct HullPolygon {
  std::vector<Point2D> vertices;

  std::size_t h() const { return vertices.size(); }
};

QuadQueues build_queues(const LabelArray& labels);

std::vector<Point2D> quadrant_hull(std::vector<Point2D> pts, int quadrant);

struct HeaphullRun {
  HullPolygon hull;
  LabelArray labels;
  double filter_ms = 0.0;  // extremes + octagon + labels (device work included)
  double hull_ms = 0.0;    // queues + chains + assembly
  double total_ms = 0.0;
};

HeaphullRun heaphull_run(std::span<const Point2D> pts, ReduceEngine& engine);

HullPolygon heaphull(std::span<const Point2D> pts, ReduceEngine& engine);
HullPolygon heaphull(std::span<const Point2D> pts, ReduceConfig cfg = {});

HullPolygon monotone_chain_hull(std::span<const Point2D> pts);

double filter_rate(const LabelArray& labels);

bool same_cycle(std::span<const Point2D> a, std::span<const Point2D> b);

}  // namespace octohull
