// octohull/filter.hpp -- B200 build of the octohull public API.
//
// Declaration-compatible with the reference header
// (/root/reference/proj/include/octohull/filter.hpp:15-90).  The point
// passes run on an sm_100a GPU through the C ABI of include/ohx.h:
//   find_axis_extremes / find_extremes -> kernel K1 (one streaming pass,
//     corner extremes certified bit-exact, else kernel K1b),
//   find_corner_extremes               -> kernel K1b,
//   classify_points                    -> kernel K2 (labels materialised),
// build_octagon and the single-point find_queue stay on the host.  There is
// no CPU fallback: without a usable device these throw std::runtime_error.
#pragma once

#include <array>
#include <cstdint>
#include <span>
#include <vector>

#include "octohull/geometry.hpp"
#include "octohull/parallel.hpp"

namespace octohull {

// argmax x, argmax y, argmin x, argmin y (ties -> smaller index)
struct AxisExtremes {
  std::size_t east = 0;
  std::size_t north = 0;
  std::size_t west = 0;
  std::size_t south = 0;
};

// Manhattan-closest points to the bounding-box corners
struct CornerExtremes {
  std::size_t ne = 0;
  std::size_t nw = 0;
  std::size_t sw = 0;
  std::size_t se = 0;
};

struct ExtremeSet {
  AxisExtremes axis;
  CornerExtremes corner;

  // CCW candidate order starting at east
  std::array<std::size_t, 8> candidates() const {
    return {axis.east, corner.ne, axis.north, corner.nw,
            axis.west, corner.sw, axis.south, corner.se};
  }
};

// Strictly convex CCW filter polygon; < 3 vertices = degenerate input.
struct Octagon {
  std::vector<Point2D> vertices;

  bool degenerate() const { return vertices.size() < 3; }
};

// 0 = filtered out, 1..4 = quadrant queue
using Label = std::uint8_t;
using LabelArray = std::vector<Label>;

AxisExtremes find_axis_extremes(std::span<const Point2D> pts, ReduceEngine& engine);
CornerExtremes find_corner_extremes(std::span<const Point2D> pts,
                                    const AxisExtremes& axis, ReduceEngine& engine);
ExtremeSet find_extremes(std::span<const Point2D> pts, ReduceEngine& engine);
Octagon build_octagon(std::span<const Point2D> pts, const ExtremeSet& ext);
int find_queue(const Point2D& p, const ExtremeSet& ext, std::span<const Point2D> pts);
LabelArray classify_points(std::span<const Point2D> pts, const Octagon& oct,
                           const ExtremeSet& ext, ReduceEngine& engine);

}  // namespace octohull
