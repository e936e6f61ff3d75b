/*
 * oracle.c -- plain-C restatement of the octohull heaphull filter path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Each function cites the
 * reference file:line (under /root/reference/proj) whose behaviour it
 * restates.  Compile with -O2 -ffp-contract=off.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define PX(xy, j) ((xy)[2 * (size_t)(j)])
#define PY(xy, j) ((xy)[2 * (size_t)(j) + 1])

/* ---------------------------------------------------------------- rng --
 * splitmix64, pointgen.hpp:42-48; unit draw pointgen.hpp:50-52 */
uint64_t orc_splitmix_next(uint64_t* state) {
  *state += 0x9E3779B97F4A7C15ULL;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

double orc_splitmix_unit(uint64_t* state) {
  return (double)(orc_splitmix_next(state) >> 11) * 0x1.0p-53;
}

/* pointgen.cpp:44-88 (Marsaglia polar at :30-40) */
int orc_generate(int dist, uint64_t n, uint64_t seed, double distort_pct,
                 double* xy) {
  if (n < 1 || distort_pct < 0.0) return -1;
  if (dist != ORC_CIRCLE && distort_pct != 0.0) return -1;
  const double two_pi = 2.0 * 3.141592653589793;
  uint64_t st = seed;
  for (uint64_t i = 0; i < n; ++i) {
    double x = 0.0, y = 0.0;
    if (dist == ORC_NORMAL) {
      for (;;) {
        const double v1 = 2.0 * orc_splitmix_unit(&st) - 1.0;
        const double v2 = 2.0 * orc_splitmix_unit(&st) - 1.0;
        const double s = v1 * v1 + v2 * v2;
        if (s >= 1.0 || s == 0.0) continue;
        const double f = sqrt(-2.0 * log(s) / s);
        x = v1 * f;
        y = v2 * f;
        break;
      }
    } else if (dist == ORC_SQUARE) {
      x = orc_splitmix_unit(&st);
      y = orc_splitmix_unit(&st);
    } else if (dist == ORC_DISK) {
      const double r = sqrt(orc_splitmix_unit(&st));
      const double th = two_pi * orc_splitmix_unit(&st);
      x = r * cos(th);
      y = r * sin(th);
    } else if (dist == ORC_CIRCLE) {
      const double th = two_pi * orc_splitmix_unit(&st);
      const double u = 2.0 * orc_splitmix_unit(&st) - 1.0;
      const double r = 1.0 + u * (distort_pct / 100.0);
      x = r * cos(th);
      y = r * sin(th);
    } else {
      return -1;
    }
    xy[2 * i] = x;
    xy[2 * i + 1] = y;
  }
  return 0;
}

/* ----------------------------------------------------------- geometry --
 * geometry.hpp:27-32 and :35-37 */
int orc_orientation(const double* a, const double* b, const double* c) {
  const double det = (b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0]);
  return det > 0.0 ? 1 : (det < 0.0 ? -1 : 0);
}

double orc_manhattan(const double* a, const double* b) {
  return fabs(a[0] - b[0]) + fabs(a[1] - b[1]);
}

/* ------------------------------------------------------------ extremes --
 * A sequential scan with a strict comparison is the reference's
 * chunk/lane-invariant arg reduction (parallel.hpp:34-43, :91-116;
 * tests/test_support.hpp:24-38): ties keep the smaller index. */
int orc_axis_extremes(const double* xy, uint64_t n, uint64_t axis[4]) {
  /* filter.cpp:8-23 */
  if (n == 0) return -1;
  uint64_t e = 0, no = 0, w = 0, s = 0;
  for (uint64_t j = 1; j < n; ++j) {
    if (PX(xy, j) > PX(xy, e)) e = j;
    if (PY(xy, j) > PY(xy, no)) no = j;
    if (PX(xy, j) < PX(xy, w)) w = j;
    if (PY(xy, j) < PY(xy, s)) s = j;
  }
  axis[0] = e; axis[1] = no; axis[2] = w; axis[3] = s;
  return 0;
}

int orc_corner_extremes(const double* xy, uint64_t n, const uint64_t axis[4],
                        uint64_t corner[4]) {
  /* filter.cpp:25-45: corners ne (xmax,ymax), nw (xmin,ymax),
   * sw (xmin,ymin), se (xmax,ymin); argmin of the Manhattan key */
  if (n == 0) return -1;
  const double xmax = PX(xy, axis[0]), ymax = PY(xy, axis[1]);
  const double xmin = PX(xy, axis[2]), ymin = PY(xy, axis[3]);
  const double c[4][2] = {{xmax, ymax}, {xmin, ymax}, {xmin, ymin}, {xmax, ymin}};
  for (int k = 0; k < 4; ++k) {
    uint64_t best = 0;
    double bkey = orc_manhattan(&xy[0], c[k]);
    for (uint64_t j = 1; j < n; ++j) {
      const double key = orc_manhattan(&xy[2 * j], c[k]);
      if (key < bkey) { bkey = key; best = j; }
    }
    corner[k] = best;
  }
  return 0;
}

int orc_find_extremes(const double* xy, uint64_t n, uint64_t ext[8]) {
  /* filter.cpp:47-52 */
  if (orc_axis_extremes(xy, n, ext) != 0) return -1;
  return orc_corner_extremes(xy, n, ext, ext + 4);
}

/* ------------------------------------------------------------ octagon --
 * filter.cpp:54-86.  Candidate order E, NE, N, NW, W, SW, S, SE
 * (filter.hpp:37-40). */
static int pt_eq(const double* a, const double* b) {
  return a[0] == b[0] && a[1] == b[1];
}

int orc_build_octagon(const double* xy, const uint64_t ext[8], double oct[16]) {
  const uint64_t order[8] = {ext[0], ext[4], ext[1], ext[5],
                             ext[2], ext[6], ext[3], ext[7]};
  double cyc[16];
  int m = 0;
  for (int k = 0; k < 8; ++k) {
    const double* p = &xy[2 * order[k]];
    if (m == 0 || !pt_eq(&cyc[2 * (m - 1)], p)) {
      cyc[2 * m] = p[0];
      cyc[2 * m + 1] = p[1];
      ++m;
    }
  }
  while (m > 1 && pt_eq(&cyc[0], &cyc[2 * (m - 1)])) --m;
  int removed = 1;
  while (removed && m > 2) {
    removed = 0;
    for (int i = 0; i < m; ++i) {
      const double* prev = &cyc[2 * ((i + m - 1) % m)];
      const double* next = &cyc[2 * ((i + 1) % m)];
      if (orc_orientation(prev, &cyc[2 * i], next) <= 0) {
        memmove(&cyc[2 * i], &cyc[2 * i + 2], sizeof(double) * 2 * (m - 1 - i));
        --m;
        removed = 1;
        break;
      }
    }
  }
  memcpy(oct, cyc, sizeof(double) * 2 * m);
  return m;
}

/* ------------------------------------------------------------ classify -- */
int orc_find_queue(const double* p, const double* xy, const uint64_t ext[8]) {
  /* filter.cpp:88-102 */
  const double* e = &xy[2 * ext[0]];
  const double* no = &xy[2 * ext[1]];
  const double* w = &xy[2 * ext[2]];
  const double* s = &xy[2 * ext[3]];
  if (orc_orientation(e, no, p) < 0) return 1;
  if (orc_orientation(no, w, p) < 0) return 2;
  if (orc_orientation(w, s, p) < 0) return 3;
  if (orc_orientation(s, e, p) < 0) return 4;
  return 1;
}

void orc_classify(const double* xy, uint64_t n, const double* oct, int oct_n,
                  const uint64_t ext[8], uint8_t* labels) {
  /* filter.cpp:104-131: kept overrides (E,1)(NE,1)(N,2)(NW,2)(W,3)(SW,3)
   * (S,4)(SE,4), first match wins; then the octagon test
   * (geometry.cpp:8-25: Outside iff some edge determinant < 0) */
  const uint64_t kidx[8] = {ext[0], ext[4], ext[1], ext[5],
                            ext[2], ext[6], ext[3], ext[7]};
  const uint8_t klab[8] = {1, 1, 2, 2, 3, 3, 4, 4};
  const int degenerate = oct_n < 3;
  for (uint64_t j = 0; j < n; ++j) {
    int lab = -1;
    for (int k = 0; k < 8 && lab < 0; ++k)
      if (kidx[k] == j) lab = klab[k];
    if (lab < 0) {
      const double* p = &xy[2 * j];
      int outside = degenerate;
      for (int i = 0; i < oct_n && !outside; ++i) {
        const double* a = &oct[2 * i];
        const double* b = &oct[2 * ((i + 1) % oct_n)];
        if (orc_orientation(a, b, p) < 0) outside = 1;
      }
      lab = outside ? orc_find_queue(p, xy, ext) : 0;
    }
    labels[j] = (uint8_t)lab;
  }
}

/* -------------------------------------------------------------- queues --
 * hull.cpp:124-131 */
void orc_queue_counts(const uint8_t* labels, uint64_t n, uint64_t counts[4]) {
  counts[0] = counts[1] = counts[2] = counts[3] = 0;
  for (uint64_t j = 0; j < n; ++j)
    if (labels[j]) ++counts[labels[j] - 1];
}

void orc_build_queues(const uint8_t* labels, uint64_t n, uint64_t* q1,
                      uint64_t* q2, uint64_t* q3, uint64_t* q4) {
  uint64_t* q[4] = {q1, q2, q3, q4};
  uint64_t c[4] = {0, 0, 0, 0};
  for (uint64_t j = 0; j < n; ++j) {
    const int l = labels[j];
    if (l) q[l - 1][c[l - 1]++] = j;
  }
}

/* --------------------------------------------------------------- hull --
 * quadrant sweep orders, hull.cpp:18-30 */
static int cmp_q1(const void* A, const void* B) {
  const double *a = A, *b = B;  /* x desc, then y asc */
  if (a[0] != b[0]) return a[0] > b[0] ? -1 : 1;
  return a[1] < b[1] ? -1 : (a[1] > b[1] ? 1 : 0);
}
static int cmp_q2(const void* A, const void* B) {
  const double *a = A, *b = B;  /* y desc, then x desc */
  if (a[1] != b[1]) return a[1] > b[1] ? -1 : 1;
  return a[0] > b[0] ? -1 : (a[0] < b[0] ? 1 : 0);
}
static int cmp_q3(const void* A, const void* B) {
  const double *a = A, *b = B;  /* x asc, then y desc */
  if (a[0] != b[0]) return a[0] < b[0] ? -1 : 1;
  return a[1] > b[1] ? -1 : (a[1] < b[1] ? 1 : 0);
}
static int cmp_q4(const void* A, const void* B) {
  const double *a = A, *b = B;  /* y asc, then x asc */
  if (a[1] != b[1]) return a[1] < b[1] ? -1 : 1;
  return a[0] < b[0] ? -1 : (a[0] > b[0] ? 1 : 0);
}
static int cmp_lex(const void* A, const void* B) {
  const double *a = A, *b = B;
  if (a[0] != b[0]) return a[0] < b[0] ? -1 : 1;
  return a[1] < b[1] ? -1 : (a[1] > b[1] ? 1 : 0);
}

uint64_t orc_quadrant_hull(double* pts, uint64_t m, int quadrant,
                           double* chain) {
  /* hull.cpp:133-150.  Equal points are indistinguishable, so an unstable
   * sort yields the same chain as std::sort. */
  if (m == 0) return 0;
  int (*cmp)(const void*, const void*) =
      quadrant == 1 ? cmp_q1 : quadrant == 2 ? cmp_q2 : quadrant == 3 ? cmp_q3 : cmp_q4;
  qsort(pts, m, 2 * sizeof(double), cmp);
  uint64_t c = 0;
  for (uint64_t i = 0; i < m; ++i) {
    const double* p = &pts[2 * i];
    while (c >= 2 && orc_orientation(&chain[2 * (c - 2)], &chain[2 * (c - 1)], p) <= 0) --c;
    chain[2 * c] = p[0];
    chain[2 * c + 1] = p[1];
    ++c;
  }
  return c - 1; /* the key-wise last point is the exit extreme */
}

/* strict_cycle, hull.cpp:53-91: LIFO worklist peeling of non-left turns;
 * the visiting order is replicated so degenerate inputs match. */
static uint64_t strict_cycle(double* cyc, uint64_t m) {
  uint64_t* prev = malloc(sizeof(uint64_t) * m);
  uint64_t* next = malloc(sizeof(uint64_t) * m);
  uint64_t* work = malloc(sizeof(uint64_t) * m);
  char* alive = malloc(m);
  char* queued = malloc(m);
  uint64_t top = 0, alive_n = m;
  for (uint64_t i = 0; i < m; ++i) {
    prev[i] = (i + m - 1) % m;
    next[i] = (i + 1) % m;
    work[top++] = i;
    alive[i] = 1;
    queued[i] = 1;
  }
  while (top > 0 && alive_n > 2) {
    const uint64_t i = work[--top];
    queued[i] = 0;
    if (!alive[i]) continue;
    if (orc_orientation(&cyc[2 * prev[i]], &cyc[2 * i], &cyc[2 * next[i]]) > 0) continue;
    alive[i] = 0;
    --alive_n;
    next[prev[i]] = next[i];
    prev[next[i]] = prev[i];
    const uint64_t nb[2] = {prev[i], next[i]};
    for (int k = 0; k < 2; ++k) {
      if (alive[nb[k]] && !queued[nb[k]]) {
        work[top++] = nb[k];
        queued[nb[k]] = 1;
      }
    }
  }
  double* out = malloc(sizeof(double) * 2 * alive_n);
  uint64_t start = 0, o = 0;
  while (!alive[start]) ++start;
  uint64_t i = start;
  do {
    out[2 * o] = cyc[2 * i];
    out[2 * o + 1] = cyc[2 * i + 1];
    ++o;
    i = next[i];
  } while (i != start);
  memcpy(cyc, out, sizeof(double) * 2 * o);
  free(out); free(prev); free(next); free(work); free(alive); free(queued);
  return o;
}

/* starts_before / rotate_to_start, hull.cpp:35-49 */
static void rotate_to_start(double* cyc, uint64_t m) {
  if (m < 2) return;
  uint64_t best = 0;
  for (uint64_t i = 1; i < m; ++i) {
    const double* a = &cyc[2 * i];
    const double* b = &cyc[2 * best];
    const int before = a[0] != b[0] ? a[0] > b[0] : a[1] < b[1];
    if (before) best = i;
  }
  if (best == 0) return;
  double* tmp = malloc(sizeof(double) * 2 * m);
  memcpy(tmp, &cyc[2 * best], sizeof(double) * 2 * (m - best));
  memcpy(&tmp[2 * (m - best)], cyc, sizeof(double) * 2 * best);
  memcpy(cyc, tmp, sizeof(double) * 2 * m);
  free(tmp);
}

/* finalize_cycle, hull.cpp:94-120; cyc is rewritten, returns h */
static uint64_t finalize_cycle(double* cyc, uint64_t m) {
  uint64_t d = 0;
  for (uint64_t i = 0; i < m; ++i) {
    if (d == 0 || !pt_eq(&cyc[2 * (d - 1)], &cyc[2 * i])) {
      cyc[2 * d] = cyc[2 * i];
      cyc[2 * d + 1] = cyc[2 * i + 1];
      ++d;
    }
  }
  while (d > 1 && pt_eq(&cyc[0], &cyc[2 * (d - 1)])) --d;
  if (d > 2) {
    int collinear = 1;
    for (uint64_t k = 2; k < d && collinear; ++k)
      collinear = orc_orientation(&cyc[0], &cyc[2], &cyc[2 * k]) == 0;
    if (collinear) {
      /* std::minmax_element: first smallest, last largest (lex order) */
      uint64_t lo = 0, hi = 0;
      for (uint64_t k = 1; k < d; ++k) {
        if (cmp_lex(&cyc[2 * k], &cyc[2 * lo]) < 0) lo = k;
        if (cmp_lex(&cyc[2 * k], &cyc[2 * hi]) >= 0) hi = k;
      }
      const double l0 = cyc[2 * lo], l1 = cyc[2 * lo + 1];
      const double h0 = cyc[2 * hi], h1 = cyc[2 * hi + 1];
      cyc[0] = l0; cyc[1] = l1; cyc[2] = h0; cyc[3] = h1;
      d = 2;
    } else {
      d = strict_cycle(cyc, d);
    }
  }
  rotate_to_start(cyc, d);
  return d;
}

int64_t orc_heaphull(const double* xy, uint64_t n, double* hull_xy,
                     uint8_t* labels_out) {
  /* hull.cpp:152-194 */
  if (n == 0) return -1;
  uint64_t ext[8];
  orc_find_extremes(xy, n, ext);
  double oct[16];
  const int m = orc_build_octagon(xy, ext, oct);
  uint8_t* labels = labels_out ? labels_out : malloc(n);
  orc_classify(xy, n, oct, m, ext, labels);

  uint64_t counts[4];
  orc_queue_counts(labels, n, counts);
  const uint64_t total = counts[0] + counts[1] + counts[2] + counts[3];
  double* cycle = malloc(sizeof(double) * 2 * (total + 8));
  uint64_t clen = 0;
  const double* anchor[4] = {&xy[2 * ext[0]], &xy[2 * ext[1]], &xy[2 * ext[2]],
                             &xy[2 * ext[3]]};
  for (int q = 1; q <= 4; ++q) {
    const uint64_t cm = counts[q - 1] + 2;
    double* cand = malloc(sizeof(double) * 2 * cm);
    double* chain = malloc(sizeof(double) * 2 * cm);
    uint64_t c = 0;
    cand[2 * c] = anchor[q - 1][0];
    cand[2 * c + 1] = anchor[q - 1][1];
    ++c;
    for (uint64_t j = 0; j < n; ++j) {
      if (labels[j] == q) {
        cand[2 * c] = PX(xy, j);
        cand[2 * c + 1] = PY(xy, j);
        ++c;
      }
    }
    cand[2 * c] = anchor[q % 4][0];
    cand[2 * c + 1] = anchor[q % 4][1];
    ++c;
    const uint64_t len = orc_quadrant_hull(cand, c, q, chain);
    memcpy(&cycle[2 * clen], chain, sizeof(double) * 2 * len);
    clen += len;
    free(cand);
    free(chain);
  }
  const uint64_t h = finalize_cycle(cycle, clen);
  memcpy(hull_xy, cycle, sizeof(double) * 2 * h);
  free(cycle);
  if (!labels_out) free(labels);
  return (int64_t)h;
}

int64_t orc_monotone_chain(const double* xy, uint64_t n, double* hull_xy) {
  /* hull.cpp:205-232 */
  if (n == 0) return -1;
  double* s = malloc(sizeof(double) * 2 * n);
  memcpy(s, xy, sizeof(double) * 2 * n);
  qsort(s, n, 2 * sizeof(double), cmp_lex);
  uint64_t u = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (u == 0 || !pt_eq(&s[2 * (u - 1)], &s[2 * i])) {
      s[2 * u] = s[2 * i];
      s[2 * u + 1] = s[2 * i + 1];
      ++u;
    }
  }
  if (u <= 2) {
    memcpy(hull_xy, s, sizeof(double) * 2 * u);
    free(s);
    return (int64_t)u;
  }
  double* lo = malloc(sizeof(double) * 2 * u);
  double* hi = malloc(sizeof(double) * 2 * u);
  uint64_t nl = 0, nh = 0;
  for (uint64_t i = 0; i < u; ++i) {
    const double* p = &s[2 * i];
    while (nl >= 2 && orc_orientation(&lo[2 * (nl - 2)], &lo[2 * (nl - 1)], p) <= 0) --nl;
    lo[2 * nl] = p[0]; lo[2 * nl + 1] = p[1]; ++nl;
  }
  for (uint64_t i = u; i-- > 0;) {
    const double* p = &s[2 * i];
    while (nh >= 2 && orc_orientation(&hi[2 * (nh - 2)], &hi[2 * (nh - 1)], p) <= 0) --nh;
    hi[2 * nh] = p[0]; hi[2 * nh + 1] = p[1]; ++nh;
  }
  uint64_t h = 0;
  memcpy(&hull_xy[0], lo, sizeof(double) * 2 * (nl - 1));
  h += nl - 1;
  memcpy(&hull_xy[2 * h], hi, sizeof(double) * 2 * (nh - 1));
  h += nh - 1;
  free(s); free(lo); free(hi);
  return (int64_t)h;
}

double orc_filter_rate(const uint8_t* labels, uint64_t n) {
  /* hull.cpp:234-241 */
  uint64_t zeros = 0;
  for (uint64_t j = 0; j < n; ++j) zeros += labels[j] == 0;
  return (double)zeros / (double)n;
}
