// octohull/pointgen.hpp -- B200 build of the octohull public API.
//
// Declaration-compatible with the reference header
// (/root/reference/proj/include/octohull/pointgen.hpp:10-70).  generate()
// here is multi-threaded yet produces the reference's exact byte stream.
#pragma once

#include <cstdint>
#include <string>

#include "octohull/geometry.hpp"

namespace octohull {

enum class Distribution { Normal, Square, Disk, Circle };

std::string to_string(Distribution dist);
Distribution parse_distribution(const std::string& token);

struct GenSpec {
  Distribution dist = Distribution::Normal;
  std::size_t n = 0;
  std::uint64_t seed = 0;
  double distort_pct = 0.0;  // circle only
};

// splitmix64 with the published constants; next_unit() = top 53 bits / 2^53.
class SplitMix64 {
 public:
  explicit SplitMix64(std::uint64_t seed) : s_(seed) {}

  std::uint64_t next() {
    s_ += 0x9E3779B97F4A7C15ULL;
    std::uint64_t z = s_;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }

  double next_unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }

 private:
  std::uint64_t s_;
};

// Seeded synthetic corpora (normal / square / disk / circle); same spec,
// same bytes as the reference.  Throws std::invalid_argument on bad specs.
PointSet generate(const GenSpec& spec);

}  // namespace octohull
