// hull.cpp -- the host hull stage that runs on the filter's survivors.
//
// The north star keeps this stage on the host with the reference's own
// semantics (reference hull.cpp:18-150, 205-232): per-quadrant sweep sort +
// strict-left-turn chain, then cycle clean-up (de-duplication, collinear
// collapse, strict_cycle peeling, rotation to the east-most vertex).
// Outputs are coordinate-identical to the reference for every input; the
// implementation differs where that cannot change the result: the four
// quadrant chains run concurrently and large sorts use the libstdc++
// parallel sort (equal points are indistinguishable, so any sort order of
// ties yields the same chain).
#include <parallel/algorithm>

#include <algorithm>
#include <cstdint>
#include <thread>
#include <vector>

#include "internal.hpp"

namespace ohx {

int orient(const P2& a, const P2& b, const P2& c) {
  // reference geometry.hpp:27-32
  const double det = (b.x - a.x) * (c.y - a.y) - (b.y - a.y) * (c.x - a.x);
  return det > 0.0 ? 1 : (det < 0.0 ? -1 : 0);
}

namespace {

bool same(const P2& a, const P2& b) { return a.x == b.x && a.y == b.y; }

// CCW sweep keys of the four quadrant arcs (reference hull.cpp:18-30)
struct SweepLess {
  int q;
  bool operator()(const P2& a, const P2& b) const {
    switch (q) {
      case 1: return a.x != b.x ? a.x > b.x : a.y < b.y;
      case 2: return a.y != b.y ? a.y > b.y : a.x > b.x;
      case 3: return a.x != b.x ? a.x < b.x : a.y > b.y;
      default: return a.y != b.y ? a.y < b.y : a.x < b.x;
    }
  }
};

bool lex(const P2& a, const P2& b) { return a.x != b.x ? a.x < b.x : a.y < b.y; }

template <class Cmp>
void big_sort(std::vector<P2>& v, Cmp cmp) {
  if (v.size() >= (1u << 17)) __gnu_parallel::sort(v.begin(), v.end(), cmp);
  else std::sort(v.begin(), v.end(), cmp);
}

// Peel every vertex that does not turn strictly left, re-examining the
// neighbours of each removal (LIFO worklist, reference hull.cpp:54-92; the
// visiting order is kept so degenerate cycles reduce identically).
std::vector<P2> peel(const std::vector<P2>& cyc) {
  const std::size_t m = cyc.size();
  std::vector<std::size_t> prv(m), nxt(m), stack;
  std::vector<unsigned char> alive(m, 1), pending(m, 1);
  stack.reserve(m);
  for (std::size_t i = 0; i < m; ++i) {
    prv[i] = (i + m - 1) % m;
    nxt[i] = (i + 1) % m;
    stack.push_back(i);
  }
  std::size_t live = m;
  while (!stack.empty() && live > 2) {
    const std::size_t i = stack.back();
    stack.pop_back();
    pending[i] = 0;
    if (!alive[i] || orient(cyc[prv[i]], cyc[i], cyc[nxt[i]]) > 0) continue;
    alive[i] = 0;
    --live;
    nxt[prv[i]] = nxt[i];
    prv[nxt[i]] = prv[i];
    for (std::size_t nb : {prv[i], nxt[i]})
      if (alive[nb] && !pending[nb]) {
        stack.push_back(nb);
        pending[nb] = 1;
      }
  }
  std::vector<P2> out;
  out.reserve(live);
  std::size_t s = 0;
  while (!alive[s]) ++s;
  std::size_t i = s;
  do {
    out.push_back(cyc[i]);
    i = nxt[i];
  } while (i != s);
  return out;
}

}  // namespace

std::vector<P2> quadrant_chain(std::vector<P2> pts, int quadrant) {
  // reference hull.cpp:133-150
  if (pts.empty()) return {};
  big_sort(pts, SweepLess{quadrant});
  std::vector<P2> chain;
  chain.reserve(std::min<std::size_t>(pts.size(), 1u << 20));
  for (const P2& p : pts) {
    while (chain.size() >= 2 && orient(chain[chain.size() - 2], chain.back(), p) <= 0)
      chain.pop_back();
    chain.push_back(p);
  }
  chain.pop_back();  // the sweep's last point is the next arc's entry
  return chain;
}

std::vector<P2> finalize_cycle(std::vector<P2> cycle) {
  // reference hull.cpp:94-120
  std::vector<P2> d;
  d.reserve(cycle.size());
  for (const P2& p : cycle)
    if (d.empty() || !same(d.back(), p)) d.push_back(p);
  while (d.size() > 1 && same(d.front(), d.back())) d.pop_back();
  if (d.size() > 2) {
    bool flat = true;
    for (std::size_t k = 2; k < d.size() && flat; ++k) flat = orient(d[0], d[1], d[k]) == 0;
    if (flat) {
      const auto mm = std::minmax_element(d.begin(), d.end(), lex);
      d = {*mm.first, *mm.second};
    } else {
      d = peel(d);
    }
  }
  if (d.size() >= 2) {
    // start at max x, ties to the smaller y (reference hull.cpp:35-49)
    std::size_t best = 0;
    for (std::size_t i = 1; i < d.size(); ++i) {
      const P2 &a = d[i], &b = d[best];
      if (a.x != b.x ? a.x > b.x : a.y < b.y) best = i;
    }
    std::rotate(d.begin(), d.begin() + static_cast<std::ptrdiff_t>(best), d.end());
  }
  return d;
}

std::vector<P2> hull_from_queue_points(const P2 anchors[4], const P2* const q_pts[4],
                                       const std::uint64_t q_len[4]) {
  // reference hull.cpp:164-183: arc q runs from anchor q-1 (entry) to
  // anchor q (exit) over the queue's members, in queue order
  std::vector<P2> chains[4];
  auto arc = [&](int q) {
    std::vector<P2> cand;
    cand.reserve(q_len[q] + 2);
    cand.push_back(anchors[q]);
    cand.insert(cand.end(), q_pts[q], q_pts[q] + q_len[q]);
    cand.push_back(anchors[(q + 1) % 4]);
    chains[q] = quadrant_chain(std::move(cand), q + 1);
  };
  const std::uint64_t total = q_len[0] + q_len[1] + q_len[2] + q_len[3];
  if (total >= (1u << 16)) {
    std::vector<std::thread> th;
    for (int q = 0; q < 4; ++q) th.emplace_back(arc, q);
    for (auto& t : th) t.join();
  } else {
    for (int q = 0; q < 4; ++q) arc(q);
  }
  std::vector<P2> cycle;
  for (int q = 0; q < 4; ++q) cycle.insert(cycle.end(), chains[q].begin(), chains[q].end());
  return finalize_cycle(std::move(cycle));
}

std::vector<P2> monotone_chain(const P2* pts, std::uint64_t n) {
  // reference hull.cpp:205-232
  std::vector<P2> s(pts, pts + n);
  big_sort(s, lex);
  s.erase(std::unique(s.begin(), s.end(), same), s.end());
  if (s.size() <= 2) return s;
  std::vector<P2> lo, hi;
  for (const P2& p : s) {
    while (lo.size() >= 2 && orient(lo[lo.size() - 2], lo.back(), p) <= 0) lo.pop_back();
    lo.push_back(p);
  }
  for (auto it = s.rbegin(); it != s.rend(); ++it) {
    while (hi.size() >= 2 && orient(hi[hi.size() - 2], hi.back(), *it) <= 0) hi.pop_back();
    hi.push_back(*it);
  }
  std::vector<P2> cyc(lo.begin(), lo.end() - 1);
  cyc.insert(cyc.end(), hi.begin(), hi.end() - 1);
  return cyc;
}

}  // namespace ohx
