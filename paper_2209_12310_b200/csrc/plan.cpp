// plan.cpp -- the host geometry between the kernels: the corner
// certificate, extremes records (combine / resolve), build_octagon, the K2
// plan with its certified interior box, and the fused pass's provisional
// region (fit + exact certification).
//
// Host arithmetic that must match the reference (orientation, manhattan,
// edge constants) is plain binary64 in a TU built with -ffp-contract=off and
// no -march, like the reference objects.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <omp.h>
#include <unistd.h>

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

#include "host.hpp"
#include "internal.hpp"
#include "ohx.h"
#include "pipeline.hpp"

namespace ohx {

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
               ohx_filter_plan* p, bool with_box) {
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
  p->box[0] = 1.0;
  p->box[1] = 0.0;
  p->box[2] = 1.0;
  p->box[3] = 0.0;  // empty
  if (with_box) fit_box(oct, m, p->ea, p->ec, p->box);
}

void ensure_box(ohx_filter_plan* p) {
  if (p->box[0] <= p->box[1] || p->m < 3) return;  // has one (or no octagon to fit)
  double oct[16];
  for (int i = 0; i < p->m; ++i) {
    oct[2 * i] = p->ax[i];
    oct[2 * i + 1] = p->ay[i];
  }
  fit_box(oct, p->m, p->ea, p->ec, p->box);
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
// Part of the convex polygon `poly` on the left of a -> b (Sutherland-Hodgman
// step; heuristic geometry, the box is certified exactly after the pass).
void clip_left(const std::vector<P2>& poly, P2 a, P2 b, std::vector<P2>& out) {
  out.clear();
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
// a provisional region: at most 8 + 7 * 8 vertices (one octagon clipped by seven)
constexpr std::size_t kMaxRegion = 64;

struct REdge {
  double ax, ay, ex, ey;  // edge start, edge vector
};

bool region_inside(const double b[8], const REdge* R, std::size_t r) {
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
  for (int v = 0; v < m; ++v) {
    const P2 p = poly[v];
    for (std::size_t i = 0; i < r; ++i)
      if (R[i].ex * (p.y - R[i].ay) - R[i].ey * (p.x - R[i].ax) < 0) return false;
  }
  return true;
}

bool fit_region(const std::vector<P2>& R, const double lim[8], KFRegion* q) {
  if (R.size() < 3) return false;
  double cx = 0, cy = 0;
  for (const P2& p : R) {
    cx += p.x;
    cy += p.y;
  }
  cx /= double(R.size());
  cy /= double(R.size());
  const std::size_t nr = R.size();
  REdge E[kMaxRegion];
  if (nr > kMaxRegion) return false;
  for (std::size_t i = 0; i < nr; ++i) {
    const P2 a = R[i], c = R[i + 1 == nr ? 0 : i + 1];
    E[i] = {a.x, a.y, c.x - a.x, c.y - a.y};
  }
  auto inside = [&](const double* bb) { return region_inside(bb, E, nr); };
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
  if (!inside(b)) return false;
  // bisections to ~1e-3 of the span (Q is pulled 0.2 % inwards afterwards),
  // then one round of per-slot bisections: more rounds or steps add host
  // time on the pass's critical path but no measurable coverage
  for (int it = 0; it < 10; ++it) {
    const double mid = (lo + hi) / 2;
    at(mid, b);
    if (inside(b)) lo = mid;
    else hi = mid;
  }
  at(lo, b);
  for (int a = 0; a < 8; ++a) {
    double good = b[a], bad = h[a];
    for (int it = 0; it < 6; ++it) {
      double t[8];
      std::memcpy(t, b, sizeof(t));
      t[a] = (good + bad) / 2;
      if (inside(t)) good = t[a];
      else bad = t[a];
    }
    b[a] = good;
  }
  // pulled 0.2 % towards the centre (OHX_REGION_PULL overrides; tuning hook)
  static const double keep = [] {
    const char* e = std::getenv("OHX_REGION_PULL");
    const double p = e ? std::atof(e) : -1.0;
    return p >= 0.0 && p < 0.5 ? 1.0 - p : 0.998;
  }();
  double r[8];
  for (int a = 0; a < 8; ++a) {
    r[a] = c0[a] + keep * (b[a] - c0[a]);
    const double below = std::nextafter(lim[a], -INFINITY);
    if (r[a] > below) r[a] = below;
  }
  *q = KFRegion{-r[2], r[0], -r[3], r[1], -r[6], r[4], -r[5], r[7]};
  return q->x0 < q->x1 && q->y0 < q->y1 && q->t0 < q->t1 && q->d0 < q->d1;
}

}  // namespace ohx
