/*
 * oracle.h -- CPU restatement of the octohull heaphull filter path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * B200 path; it is imported by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py and nowhere else.  The product path never
 * links or calls it.
 *
 * Every function is a plain-C restatement of the reference algorithm at
 * the cited file:line of /root/reference/proj (octohull).  Points are AoS
 * interleaved doubles xy[2*j] = x_j, xy[2*j+1] = y_j (the reference's
 * Point2D layout, geometry.hpp:10-15).  Arithmetic is IEEE binary64 with
 * no FMA contraction (build with -ffp-contract=off), matching the
 * reference objects (0 vfmadd).
 *
 * Pinned against: the reference's own KATs (test_filter.cpp, test_hull.cpp,
 * test_pointgen.cpp), tests/data/bench_golden.json, and the reference
 * library itself compiled into oracle/_ref (see tests/test_oracle.py).
 */
#ifndef OHX_ORACLE_H
#define OHX_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_NORMAL = 0, ORC_SQUARE = 1, ORC_DISK = 2, ORC_CIRCLE = 3 };

/* pointgen.hpp:42-52 */
uint64_t orc_splitmix_next(uint64_t* state);
double orc_splitmix_unit(uint64_t* state);

/* pointgen.cpp:44-88; returns 0 or -1 on an invalid spec */
int orc_generate(int dist, uint64_t n, uint64_t seed, double distort_pct,
                 double* xy);

/* geometry.hpp:27-37 */
int orc_orientation(const double* a, const double* b, const double* c);
double orc_manhattan(const double* a, const double* b);

/* filter.cpp:8-23 -> axis[4] = {east, north, west, south}; -1 if n == 0 */
int orc_axis_extremes(const double* xy, uint64_t n, uint64_t axis[4]);

/* filter.cpp:25-45 -> corner[4] = {ne, nw, sw, se} */
int orc_corner_extremes(const double* xy, uint64_t n, const uint64_t axis[4],
                        uint64_t corner[4]);

/* filter.cpp:47-52 -> ext[8] = {east, north, west, south, ne, nw, sw, se} */
int orc_find_extremes(const double* xy, uint64_t n, uint64_t ext[8]);

/* filter.cpp:54-86; oct_xy receives <= 8 vertices, returns the count */
int orc_build_octagon(const double* xy, const uint64_t ext[8],
                      double oct_xy[16]);

/* filter.cpp:88-102 */
int orc_find_queue(const double* p, const double* xy, const uint64_t ext[8]);

/* filter.cpp:104-131 */
void orc_classify(const double* xy, uint64_t n, const double* oct_xy,
                  int oct_n, const uint64_t ext[8], uint8_t* labels);

/* hull.cpp:124-131: counts[4]; if queues != NULL, queues[q] (capacity
 * counts) receive the indices in input order */
void orc_queue_counts(const uint8_t* labels, uint64_t n, uint64_t counts[4]);
void orc_build_queues(const uint8_t* labels, uint64_t n, uint64_t* q1,
                      uint64_t* q2, uint64_t* q3, uint64_t* q4);

/* hull.cpp:133-150; pts (m points) is sorted in place, chain receives the
 * open chain, returns its length */
uint64_t orc_quadrant_hull(double* pts, uint64_t m, int quadrant,
                           double* chain);

/* hull.cpp:152-194 minus timing: full heaphull.  hull_xy needs room for n
 * points; labels may be NULL.  Returns h, or -1 on empty input. */
int64_t orc_heaphull(const double* xy, uint64_t n, double* hull_xy,
                     uint8_t* labels);

/* hull.cpp:205-232 */
int64_t orc_monotone_chain(const double* xy, uint64_t n, double* hull_xy);

/* hull.cpp:234-241 */
double orc_filter_rate(const uint8_t* labels, uint64_t n);

#ifdef __cplusplus
}
#endif

#endif
