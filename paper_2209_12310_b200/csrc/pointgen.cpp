// pointgen.cpp -- multi-threaded generator, bit-identical to the reference's
// single-threaded generate() (reference pointgen.cpp:44-88).
//
// splitmix64 is counter-based: after k draws from seed s the state is
// s + k*0x9E3779B97F4A7C15 (mod 2^64), so draw k can be computed directly.
// square/disk/circle consume two draws per point and parallelise
// trivially.  normal uses Marsaglia's polar rejection (two draws per
// attempt): a counting pass finds how many attempts of each block of
// attempts are accepted, an exclusive scan gives every block its first
// output slot, and an emitting pass writes the accepted points.  The
// arithmetic (including glibc libm sqrt/log/cos/sin) is the reference's.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numbers>
#include <stdexcept>
#include <thread>
#include <vector>

#include "internal.hpp"

namespace ohx {
namespace {

constexpr std::uint64_t kGamma = 0x9E3779B97F4A7C15ULL;

inline std::uint64_t mix(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// value of the k-th draw (k >= 1) of a stream seeded with `seed`
inline double unit_at(std::uint64_t seed, std::uint64_t k) {
  return static_cast<double>(mix(seed + k * kGamma) >> 11) * 0x1.0p-53;
}

template <class F>
void parallel_for(std::uint64_t count, int threads, F&& body) {
  if (threads <= 1 || count < 2) {
    for (std::uint64_t b = 0; b < count; ++b) body(b);
    return;
  }
  std::vector<std::thread> pool;
  const int t = static_cast<int>(std::min<std::uint64_t>(threads, count));
  for (int w = 0; w < t; ++w)
    pool.emplace_back([&, w] {
      for (std::uint64_t b = w; b < count; b += t) body(b);
    });
  for (auto& th : pool) th.join();
}

constexpr std::uint64_t kAttemptBlock = 1u << 16;
constexpr std::uint64_t kPointBlock = 1u << 16;

// attempt a (0-based) of the normal generator, reference pointgen.cpp:30-40
inline bool normal_attempt(std::uint64_t seed, std::uint64_t a, double& x, double& y) {
  const double v1 = 2.0 * unit_at(seed, 2 * a + 1) - 1.0;
  const double v2 = 2.0 * unit_at(seed, 2 * a + 2) - 1.0;
  const double s = v1 * v1 + v2 * v2;
  if (s >= 1.0 || s == 0.0) return false;
  const double f = std::sqrt(-2.0 * std::log(s) / s);
  x = v1 * f;
  y = v2 * f;
  return true;
}

inline bool normal_accepts(std::uint64_t seed, std::uint64_t a) {
  const double v1 = 2.0 * unit_at(seed, 2 * a + 1) - 1.0;
  const double v2 = 2.0 * unit_at(seed, 2 * a + 2) - 1.0;
  const double s = v1 * v1 + v2 * v2;
  return !(s >= 1.0 || s == 0.0);
}

// outputs [lo, lo + cnt) of the normal stream: attempts are counted block
// by block until lo + cnt points are accepted; only the blocks whose
// outputs meet the range are emitted
void gen_normal(std::uint64_t lo, std::uint64_t cnt, std::uint64_t seed, double* xy,
                int threads) {
  const std::uint64_t end = lo + cnt;
  std::vector<std::uint64_t> accepted;  // per attempt block
  std::uint64_t have = 0;
  while (have < end) {
    // acceptance is pi/4; overshoot slightly, then extend if still short
    const std::uint64_t want = end - have;
    const std::uint64_t more =
        std::max<std::uint64_t>(1, (want * 1.28 + 4096) / kAttemptBlock + 1);
    const std::uint64_t first = accepted.size();
    accepted.resize(first + more);
    parallel_for(more, threads, [&](std::uint64_t b) {
      const std::uint64_t a0 = (first + b) * kAttemptBlock;
      std::uint64_t c = 0;
      for (std::uint64_t a = a0; a < a0 + kAttemptBlock; ++a) c += normal_accepts(seed, a);
      accepted[first + b] = c;
    });
    for (std::uint64_t b = first; b < accepted.size(); ++b) have += accepted[b];
  }
  std::vector<std::uint64_t> start(accepted.size());
  std::uint64_t run = 0;
  for (std::size_t b = 0; b < accepted.size(); ++b) {
    start[b] = run;
    run += accepted[b];
  }
  parallel_for(accepted.size(), threads, [&](std::uint64_t b) {
    std::uint64_t out = start[b];
    if (out >= end || out + accepted[b] <= lo) return;
    const std::uint64_t a0 = b * kAttemptBlock;
    for (std::uint64_t a = a0; a < a0 + kAttemptBlock && out < end; ++a) {
      double x, y;
      if (normal_attempt(seed, a, x, y)) {
        if (out >= lo) {
          xy[2 * (out - lo)] = x;
          xy[2 * (out - lo) + 1] = y;
        }
        ++out;
      }
    }
  });
}

}  // namespace

void generate_points(int dist, std::uint64_t n, std::uint64_t seed,
                     double distort_pct, double* xy, int threads) {
  generate_points_range(dist, n, seed, distort_pct, 0, n, xy, threads);
}

void generate_points_range(int dist, std::uint64_t n, std::uint64_t seed, double distort_pct,
                           std::uint64_t lo, std::uint64_t cnt, double* xy, int threads) {
  // validation and messages of reference pointgen.cpp:45-55
  if (n < 1) throw std::invalid_argument("generate: n must be >= 1");
  if (distort_pct < 0.0) throw std::invalid_argument("generate: distort_pct must be >= 0");
  if (dist != OHX_CIRCLE && distort_pct != 0.0)
    throw std::invalid_argument("generate: distortion applies to the circle distribution only");
  if (dist < OHX_NORMAL || dist > OHX_CIRCLE)
    throw std::invalid_argument("unknown distribution value");
  if (lo > n || cnt > n - lo) throw std::invalid_argument("generate: range outside [0, n)");
  if (cnt == 0) return;
  if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  if (lo + cnt < 4 * kPointBlock) threads = 1;

  if (dist == OHX_NORMAL) {
    gen_normal(lo, cnt, seed, xy, threads);
    return;
  }
  constexpr double two_pi = 2.0 * std::numbers::pi;
  const double scale = distort_pct / 100.0;
  const std::uint64_t blocks = (cnt + kPointBlock - 1) / kPointBlock;
  parallel_for(blocks, threads, [&](std::uint64_t b) {
    const std::uint64_t i1 = lo + std::min(cnt, (b + 1) * kPointBlock);
    for (std::uint64_t i = lo + b * kPointBlock; i < i1; ++i) {
      const double u1 = unit_at(seed, 2 * i + 1);
      const double u2 = unit_at(seed, 2 * i + 2);
      double x, y;
      if (dist == OHX_SQUARE) {
        x = u1;
        y = u2;
      } else if (dist == OHX_DISK) {
        const double r = std::sqrt(u1);
        const double th = two_pi * u2;
        x = r * std::cos(th);
        y = r * std::sin(th);
      } else {
        const double th = two_pi * u1;
        const double u = 2.0 * u2 - 1.0;
        const double r = 1.0 + u * scale;
        x = r * std::cos(th);
        y = r * std::sin(th);
      }
      xy[2 * (i - lo)] = x;
      xy[2 * (i - lo) + 1] = y;
    }
  });
}

}  // namespace ohx
