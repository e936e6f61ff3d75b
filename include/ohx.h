/*
 * ohx.h -- C ABI of the B200 (sm_100a) heaphull filter layer.
 *
 * This is the drop-in boundary under the reference's public C++ API
 * (/root/reference/proj/include/octohull/{filter,hull}.hpp).  The
 * reference has no C ABI of its own -- its only FFI is the pybind11
 * module python/module.cpp -- so each entry point below names the
 * reference interface it replaces (file:line, paths relative to
 * /root/reference/proj).  INTEGRATION.md shows the bindings a
 * maintainer adds (ctypes stub, pybind11 module relink, C++ relink).
 *
 * Conventions
 *   - Every function returns OHX_OK (0) or a negative OHX_E* code and never
 *     throws or aborts across the ABI; ohx_last_error() returns a
 *     thread-local message for the last failure on the calling thread.
 *   - Points are the reference's AoS Point2D layout (geometry.hpp:10-15):
 *     interleaved IEEE binary64, xy[2j] = x_j, xy[2j+1] = y_j, 16-byte
 *     aligned.  Coordinates must be finite (the reference enforces this at
 *     ingestion, geometry.cpp:27-34); the filter does not re-check.
 *   - Indices are 64-bit global point indices.  Sharded callers pass
 *     `index_base` = first global index of the shard so that the
 *     smallest-index tie rule (parallel.hpp:34-43) holds across shards.
 *   - d_* pointers are device pointers (cudaMalloc / torch), h_* are host.
 *   - `stream` is a cudaStream_t passed as void*; NULL = the context's own
 *     stream.  Shard-level calls are synchronous w.r.t. their small host
 *     outputs (they end with a stream sync) unless stated otherwise.
 *   - There is no CPU fallback: without a usable sm_100 device every
 *     compute entry point fails with OHX_E_CUDA / OHX_E_NODEVICE.
 */
#ifndef OHX_H
#define OHX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OHX_ABI_VERSION 1

enum {
  OHX_OK = 0,
  OHX_E_INVALID = -1,  /* std::invalid_argument in the reference */
  OHX_E_CUDA = -2,     /* CUDA runtime error (std::runtime_error) */
  OHX_E_NODEVICE = -3, /* no sm_100 device visible */
  OHX_E_NOMEM = -4,    /* device or pinned allocation failed */
  OHX_E_INTERNAL = -5,
  OHX_E_IO = -6        /* file error (std::runtime_error in the reference's io) */
};

/* Distributions of pointgen.hpp:10 (generate, pointgen.cpp:44-88). */
enum { OHX_NORMAL = 0, OHX_SQUARE = 1, OHX_DISK = 2, OHX_CIRCLE = 3 };

/* Direction slots of an extremes record.  Slots 0..3 are the axis extremes
 * (AxisExtremes, filter.hpp:15-20), 4..7 the corner extremes
 * (CornerExtremes, filter.hpp:24-29). */
enum {
  OHX_EAST = 0, OHX_NORTH = 1, OHX_WEST = 2, OHX_SOUTH = 3,
  OHX_NE = 4, OHX_NW = 5, OHX_SW = 6, OHX_SE = 7
};

/* One shard's single-pass extremes (kernel K1).  Every slot is an argmax of
 * a maximised key with ties to the smaller global index:
 *   east x, north y, west -x, south -y,
 *   ne fl(x+y), nw fl(y-x), sw -fl(x+y), se fl(x-y).
 * second[k] is the second-largest diagonal key (as a multiset) of slot 4+k;
 * it feeds the corner certificate (see ohx_extremes_resolve).  x/y are the
 * coordinates of each slot's winner. */
typedef struct {
  double key[8];
  uint64_t idx[8];
  double second[4];
  double x[8];
  double y[8];
  uint64_t n; /* points covered by this record */
} ohx_extremes_rec;

/* Exact Manhattan corner argmins (kernel K1b), corners ne, nw, sw, se as in
 * find_corner_extremes (filter.cpp:25-45); key = the reference's
 * manhattan() value (geometry.hpp:35-37). */
typedef struct {
  double key[4];
  uint64_t idx[4];
  double x[4];
  double y[4];
  uint64_t n;
} ohx_corner_rec;

/* The resolved ExtremeSet (filter.hpp:33-41): ext[8] in slot order
 * {east, north, west, south, ne, nw, sw, se}, with coordinates. */
typedef struct {
  uint64_t ext[8];
  double x[8];
  double y[8];
} ohx_extreme_set;

/* Everything kernel K2 needs, built on the host from an Octagon and an
 * ExtremeSet (ohx_filter_plan_build).  Edge constants are the reference's
 * (b.x-a.x), (b.y-a.y) of orientation() (geometry.hpp:27-32). */
typedef struct {
  double ax[8], ay[8];   /* octagon edge origin a_i (padded: 0) */
  double ea[8], ec[8];   /* fl(b.x-a.x), fl(b.y-a.y) (padded: 0 => never < 0) */
  double qax[4], qay[4]; /* find_queue edges E->N, N->W, W->S, S->E */
  double qa[4], qc[4];
  double box[4];         /* certified interior box xlo,xhi,ylo,yhi (empty if xlo>xhi) */
  uint64_t kept[8];      /* kept indices in override order E,NE,N,NW,W,SW,S,SE */
  uint8_t kept_label[8]; /* 1,1,2,2,3,3,4,4 */
  int32_t m;             /* octagon vertices; < 3 = degenerate (filter nothing) */
  int32_t pad;
} ohx_filter_plan;

typedef struct ohx_ctx ohx_ctx;

/* ---- runtime ----------------------------------------------------------- */
int ohx_abi_version(void);
const char* ohx_last_error(void);
int ohx_device_count(int* n);
/* Per-device context: stream, workspaces (grow-only, reused across calls),
 * pinned staging.  One call at a time per context (ReduceEngine contract,
 * parallel.hpp:50-52); distinct contexts may run concurrently. */
int ohx_ctx_create(int device, ohx_ctx** out);
int ohx_ctx_destroy(ohx_ctx* ctx);
/* Releases the context's grow-only device / pinned workspaces and the
 * library's cache of large host blocks (the hull stage's); later calls
 * regrow what they need.  Drops a pending ohx_fused_extremes. */
int ohx_ctx_trim(ohx_ctx* ctx);
/* Process-wide lazily created context for `device` (used by the C++ API). */
int ohx_ctx_default(int device, ohx_ctx** out);
int ohx_ctx_device(const ohx_ctx* ctx);
/* Kernels launched by this context since creation (evidence counter). */
uint64_t ohx_ctx_launches(const ohx_ctx* ctx);
/* How the last pipeline-level call on this context ran. */
typedef struct {
  uint32_t fused;       /* 1: single pass (KF) + K2 on the candidates only */
  uint32_t corner_pass; /* 1: the corner certificate failed and K1b ran */
  uint64_t candidates;  /* points outside the provisional region (fused pass) */
  uint64_t counts[4];   /* queue lengths */
  uint32_t fuse_state;  /* 0 not tried (small n / disabled), 1 fused, 2 no
                           sample region, 3 sample coverage too low, 4 region
                           not certified in the true octagon, 5 too many
                           candidates */
  uint32_t hull_path;   /* hull stage: 0 host sort + chains (small survivor
                           sets), 1 device sort + device chains, 2 device
                           chains unproven -> host chains, 3 device sort +
                           host chains (OHX_DEVICE_CHAIN=0) */
  double sample_coverage; /* fraction of the sample inside the provisional region */
} ohx_run_info;
int ohx_ctx_last_run(const ohx_ctx* ctx, ohx_run_info* info);
/* Device duration (CUDA events on the launching stream) of the last launch
 * of each stage in this context: ms[0] K1 (or, fused, the KF filter pass),
 * ms[1] K1b, ms[2] K2, ms[3] the fused path's candidate stage (ordered
 * compaction + K1 over the candidates); -1 for a stage that did not run
 * (a pipeline call resets all four). */
int ohx_ctx_kernel_ms(ohx_ctx* ctx, double ms[4]);
/* Running sums of those stage times over the calls since the last reset
 * (each call's stages counted once, when they have completed; count[k] =
 * calls that ran stage k): a timing loop reads them once at its end
 * instead of querying events between calls.  reset != 0 zeroes them. */
int ohx_ctx_kernel_ms_sum(ohx_ctx* ctx, double sum[4], uint64_t count[4], int reset);

/* ---- kernel-level (one shard, device-resident points) ------------------ */

/* K1. Replaces the 8 reduction passes of find_axis_extremes
 * (filter.cpp:8-23) + find_corner_extremes (filter.cpp:25-45) by one
 * streaming pass.  n >= 1. */
int ohx_extremes(ohx_ctx* ctx, const double* d_xy, uint64_t n,
                 uint64_t index_base, ohx_extremes_rec* h_rec, void* stream);

/* Associative, commutative merge of shard records (ties -> smaller global
 * index); every rank computes the identical result.  Host only. */
int ohx_extremes_combine(const ohx_extremes_rec* recs, int k,
                         ohx_extremes_rec* out);

/* Axis extremes + certified corner extremes from a (global) record.
 * Corner slot k is certified when the reference's Manhattan argmin is
 * provably the diagonal winner (gap between best and second diagonal key
 * exceeds the binary64 rounding bound).  Uncertified slots are reported in
 * *uncertified_mask (bit k = corner 4+k) and must be resolved with
 * ohx_corners_exact.  Host only. */
int ohx_extremes_resolve(const ohx_extremes_rec* rec, ohx_extreme_set* out,
                         uint32_t* uncertified_mask);

/* Fused single pass over one shard (replaces K1 + the K2 read of every
 * point; SURVEY §8f "one read").  Samples the shard, fits a provisional
 * region Q, streams the points once (KF) keeping only those outside Q, and
 * runs K1 over those candidates.  *fused = 1: h_rec is the shard's extremes
 * record, exactly what ohx_extremes returns (global indices).  *fused = 0:
 * nothing usable (small shard, poor sample coverage, candidate overflow) --
 * call ohx_extremes.  The candidates stay in the context for
 * ohx_filter_fused. */
int ohx_fused_extremes(ohx_ctx* ctx, const double* d_xy, uint64_t n, uint64_t index_base,
                       ohx_extremes_rec* h_rec, int* fused, void* stream);
/* Second half of the fused pass, same points: classify with the global
 * ExtremeSet and plan (filter.cpp:104-131, hull.cpp:124-131).  K2 runs over
 * the candidates only when Q is certified inside the plan's octagon and
 * holds none of the kept points (*fused = 1), else over all n points
 * (*fused = 0).  Same outputs as ohx_filter (queues via ohx_queue_fetch;
 * labels of dropped points 0).  OHX_E_INVALID without a pending
 * ohx_fused_extremes over (d_xy, n, index_base) in this context. */
int ohx_filter_fused(ohx_ctx* ctx, const double* d_xy, uint64_t n, uint64_t index_base,
                     const ohx_extreme_set* ext, const ohx_filter_plan* plan, uint8_t* d_labels,
                     uint64_t h_counts[4], int* fused, void* stream);

/* K1b. Exact corner argmins against the bounding box
 * bbox = {x_max, y_max, x_min, y_min} (filter.cpp:28-43). */
int ohx_corners_exact(ohx_ctx* ctx, const double* d_xy, uint64_t n,
                      uint64_t index_base, const double bbox[4],
                      ohx_corner_rec* h_rec, void* stream);
int ohx_corners_combine(const ohx_corner_rec* recs, int k, ohx_corner_rec* out);

/* build_octagon (filter.cpp:54-86) on the 8 candidate coordinates in
 * candidate order E,NE,N,NW,W,SW,S,SE (filter.hpp:37-40).  Host only. */
int ohx_build_octagon(const double cand_xy[16], double oct_xy[16], int* m);

/* K2 plan from an octagon (m vertices, CCW) and the extreme set. Host only. */
int ohx_filter_plan_build(const ohx_extreme_set* ext, const double* oct_xy,
                          int m, ohx_filter_plan* plan);

/* K2. Replaces classify_points (filter.cpp:104-131) + build_queues
 * (hull.cpp:124-131): labels every point of the shard and compacts the
 * survivors, in index order, into four per-quadrant queues held in the
 * context.  d_labels (nullable) receives the n labels (LabelArray,
 * filter.hpp:53-54).  h_counts receives the four queue lengths. */
int ohx_filter(ohx_ctx* ctx, const double* d_xy, uint64_t n,
               uint64_t index_base, const ohx_filter_plan* plan,
               uint8_t* d_labels, uint64_t h_counts[4], void* stream);

/* Copy queue q (1..4) of the last ohx_filter to the host: global indices
 * (nullable) and survivor coordinates (nullable, gathered on the device). */
int ohx_queue_fetch(ohx_ctx* ctx, int q, uint64_t* h_idx, double* h_xy,
                    uint64_t cap, void* stream);
/* Device pointer + element width (4 or 8 bytes, shard-local indices) of
 * queue q of the last ohx_filter. */
int ohx_queue_device(ohx_ctx* ctx, int q, const void** d_idx,
                     int* idx_bytes, uint64_t* count);

/* Hull vertex indices (the north star's parity output; the reference itself
 * emits coordinates only, hull.cpp:196-203): for each of the h vertices of
 * a hull computed by the last pipeline / filter call on ctx (NULL: the
 * default context, i.e. after ohx_heaphull), the smallest input index with
 * equal coordinates (-0.0 == +0.0), in the hull's order.  OHX_E_INVALID if
 * a vertex is not among that call's survivors. */
int ohx_hull_indices(ohx_ctx* ctx, const double* h_hull, uint64_t h,
                     uint64_t* h_idx, void* stream);
/* Same over one shard's survivors (global indices: index_base of the
 * shard's filter call added); UINT64_MAX where the shard holds no point with
 * a vertex's coordinates, no error.  The job's answer is the minimum over
 * the shards (sharded.py: an all-reduce MIN). */
int ohx_hull_indices_partial(ohx_ctx* ctx, const double* h_hull, uint64_t h,
                             uint64_t* h_idx, void* stream);

/* ---- pipeline-level (host buffers; the reference's bound entry points) --- */

/* heaphull (hull.cpp:196-203; python/module.cpp:62-75): host points in,
 * CCW hull coordinates out (h_hull capacity `cap` points, *h = size).
 * timings (nullable) = {filter_ms, hull_ms, total_ms, h2d_ms}. */
int ohx_heaphull(const double* h_xy, uint64_t n, double* h_hull, uint64_t cap,
                 uint64_t* h, double* timings);
/* Same, points already on the device of `ctx`. */
int ohx_heaphull_device(ohx_ctx* ctx, const double* d_xy, uint64_t n,
                        double* h_hull, uint64_t cap, uint64_t* h,
                        double* timings);
/* The same with the hull left in DEVICE memory (d_hull, capacity cap
 * points, on ctx's device): for a consumer on the GPU, the hull stage skips
 * the PCIe copy of the hull (96.8M vertices = 1.55 GB for points on a
 * circle).  Small survivor sets still chain on the host; their hull is
 * copied up. */
int ohx_heaphull_device_out(ohx_ctx* ctx, const double* d_xy, uint64_t n, double* d_hull,
                            uint64_t cap, uint64_t* h, double* timings);
/* classify (python/module.cpp:91-108): find_extremes + build_octagon +
 * classify_points, labels to the host. */
int ohx_classify(const double* h_xy, uint64_t n, uint8_t* h_labels);
/* classify_points (filter.cpp:104-131) with the caller's polygon (m
 * vertices, any m -- build_octagon makes <= 8, callers may pass more) and
 * ExtremeSet ext[8] in slot order; labels to the host. */
int ohx_classify_points(const double* h_xy, uint64_t n, const double* poly_xy, uint64_t m,
                        const uint64_t ext[8], uint8_t* h_labels);
/* heaphull_run (hull.cpp:152-194): hull + labels + timings. */
int ohx_heaphull_run(const double* h_xy, uint64_t n, double* h_hull,
                     uint64_t cap, uint64_t* h, uint8_t* h_labels,
                     double* timings);
/* ---- point files (io.cpp:87-124, the binary PTS2 layout) -------------- */
/* Validated header -> point count (OHX_E_IO with the reference's message:
 * bad magic, count 0, size mismatch, cannot open). */
int ohx_pts2_count(const char* path, uint64_t* n);
/* The file's points straight into device memory d_xy (capacity cap
 * points): pread into pinned chunks overlapped with the H2D copies, then a
 * device scan rejects the first non-finite point ("non-finite coordinate in
 * point i at byte 12+16i", OHX_E_IO). */
int ohx_pts2_load_device(ohx_ctx* ctx, const char* path, double* d_xy, uint64_t cap,
                         uint64_t* n, void* stream);
/* read_points(path, Binary) + heaphull (tools/octohull_main.cpp) with the
 * file loaded straight into device memory; timings[3] = file -> device ms. */
int ohx_heaphull_pts2(const char* path, double* h_hull, uint64_t cap, uint64_t* h,
                      double* timings);

/* find_extremes (filter.cpp:47-52) from host points: ext[8] slot order. */
int ohx_find_extremes(const double* h_xy, uint64_t n, uint64_t ext[8]);

/* monotone_chain_hull (hull.cpp:205-232; python/module.cpp:77-89): the
 * independent full-set reference hull, host only. */
int ohx_monotone_chain(const double* h_xy, uint64_t n, double* h_hull,
                       uint64_t cap, uint64_t* h);

/* generate (pointgen.cpp:44-88), multi-threaded and bit-identical to the
 * reference's single-threaded stream; threads = 0 -> all cores. */
int ohx_generate(int dist, uint64_t n, uint64_t seed, double distort_pct,
                 double* h_xy, int threads);
/* Points [lo, lo + count) of the same n-point corpus: a shard's slice of
 * generate({dist, n, seed, distort}) without generating the rest (normal:
 * the rejection attempts before lo are counted, not emitted). */
int ohx_generate_range(int dist, uint64_t n, uint64_t seed, double distort_pct,
                       uint64_t lo, uint64_t count, double* h_xy, int threads);

/* The strict-left-turn chain of an arc already in sweep order (the loop of
 * quadrant_hull, hull.cpp:140-149, without its sort): h_out receives the
 * chain without the arc's last point (*m entries; capacity n).  Long arcs
 * run in parallel chunks with the reference loop's exact decisions. */
int ohx_chain(const double* h_xy, uint64_t n, double* h_out, uint64_t* m);

/* The hull stage on the four arcs [anchor q, queue q, anchor q+1] already
 * in their quadrant's sweep order (what the device sort hands the host:
 * hull.cpp:133-150 without the sort, then 94-120); h_hull capacity cap. */
int ohx_hull_from_sorted_arcs(const double* const arcs_xy[4], const uint64_t len[4],
                              double* h_hull, uint64_t cap, uint64_t* h);

/* The same hull stage with the arcs sorted in DEVICE memory (back to back,
 * len[q] points each): the chains are replayed on the device in chunks and
 * proven equal to the reference loop's (hullchain.cu); *proven = 0 when the
 * proof fails, and the host chains produce the hull instead.  Either way
 * the hull is the reference's.  flags & OHX_ARCS_RAW_CYCLE: write the
 * chained cycle itself (the four chains, each without its last point,
 * before finalize_cycle) -- a test hook for the chains alone. */
#define OHX_ARCS_RAW_CYCLE 1
int ohx_hull_from_sorted_arcs_device(ohx_ctx* ctx, const double* d_arcs, const uint64_t len[4],
                                     double* h_hull, uint64_t cap, uint64_t* h, int* proven,
                                     int flags, void* stream);

/* Host hull stage of heaphull_run (hull.cpp:164-183) on given queues:
 * pts = all points (host), queues as global indices. */
int ohx_hull_from_queues(const double* h_xy, const uint64_t ext_axis[4],
                         const uint64_t* const q_idx[4],
                         const uint64_t q_len[4], double* h_hull,
                         uint64_t cap, uint64_t* h);
/* Same, survivor coordinates given directly per queue (index order). */
int ohx_hull_from_queue_points(const double anchors_xy[8],
                               const double* const q_xy[4],
                               const uint64_t q_len[4], double* h_hull,
                               uint64_t cap, uint64_t* h);

/* ---- multi-GPU (the reference's ReduceConfig.workers,
 * parallel.hpp:18-21, mapped to devices) ---------------------------------
 * One NCCL rank per GPU.  The job's points are contiguous index-range
 * shards; each rank filters its own (fused pass or K1, then K2), the
 * 296-byte extremes records and the queue lengths are exchanged with
 * ncclAllGather (the same exact combine on every rank), and the survivors'
 * coordinates go to rank 0 only (one ncclSend/ncclRecv per queue and rank,
 * straight into place), which runs the hull stage.  Results equal the
 * single-device pipeline's bit for bit.  A rank may hold several virtual
 * shards (vshards): the same exchange with several shards per device.
 * NCCL is loaded at run time (libnccl.so.2); without it these calls fail
 * with OHX_E_NODEVICE.  A call that fails mid-exchange aborts the
 * communicator: destroy and recreate the handle. */
typedef struct ohx_mg ohx_mg;
typedef struct {
  uint64_t ext[8];       /* the job's ExtremeSet, slot order (global indices) */
  uint64_t counts[4];    /* the job's queue lengths */
  uint64_t n_total;      /* points in the job */
  uint32_t corner_pass;  /* the corner certificate failed: K1b ran on every shard */
  uint32_t fused_shards; /* shards whose K2 ran on their fused-pass candidates only */
  uint32_t shards;       /* shards in the job */
  uint32_t pad;
  double ms[4];          /* this rank's host wall time: extremes + exchange,
                            K2, survivor gather, hull stage (root) */
} ohx_mg_info;
/* ncclGetUniqueId, for the process of rank 0 to hand to the others. */
int ohx_mg_unique_id(uint8_t id[128]);
/* One process per GPU: this process is `rank` of `world`, on `device`
 * (ncclCommInitRank; collective over the world). */
int ohx_mg_init_rank(const uint8_t id[128], int world, int rank, int device, ohx_mg** out);
/* One process driving `ndev` GPUs, one thread per device in every call
 * (ncclCommInitAll); devices NULL = 0..ndev-1. */
int ohx_mg_init_all(int ndev, const int* devices, ohx_mg** out);
int ohx_mg_destroy(ohx_mg* mg);
int ohx_mg_world(const ohx_mg* mg, int* world, int* local_ranks);
int ohx_mg_nccl_version(int* version);
/* The context of shard `shard` of local rank `local_rank` (created if need
 * be; owned by the handle): its launch counter, stage times and last run
 * describe that shard's part of the last call. */
int ohx_mg_ctx(ohx_mg* mg, int local_rank, int shard, ohx_ctx** ctx);
/* Collective (ohx_mg_init_rank handles): this rank's device-resident shard
 * [index_base, index_base + n) of the job, split into vshards virtual
 * shards; every rank calls it with its own range, ranks in index order.
 * Rank 0 receives the hull (h_hull capacity cap, *h); elsewhere *h = 0.
 * h_labels (nullable): this shard's n labels. */
int ohx_mg_heaphull_shard(ohx_mg* mg, const double* d_xy, uint64_t n, uint64_t index_base,
                          int vshards, uint8_t* h_labels, double* h_hull, uint64_t cap,
                          uint64_t* h, ohx_mg_info* info);
/* Single process (ohx_mg_init_all): nshards device-resident shards, in
 * index order, nshards / ndev consecutive ones on each device. */
int ohx_mg_heaphull_device(ohx_mg* mg, int nshards, const double* const* d_xy, const uint64_t* n,
                           uint8_t* h_labels, double* h_hull, uint64_t cap, uint64_t* h,
                           ohx_mg_info* info);
/* Single process: host points split evenly over the devices (vshards
 * each), every device staging its own slice (heaphull / heaphull_run of
 * the C++ API with ReduceConfig.workers > 1 on a multi-GPU box). */
int ohx_mg_heaphull(ohx_mg* mg, const double* h_xy, uint64_t n, int vshards, uint8_t* h_labels,
                    double* h_hull, uint64_t cap, uint64_t* h, ohx_mg_info* info);

#ifdef __cplusplus
}
#endif

#endif /* OHX_H */
