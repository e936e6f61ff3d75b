// capi.cpp -- the C ABI of include/ohx.h: thin exception-safe wrappers
// over context.cpp / plan.cpp / device.cpp.
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

// =================================================================== C ABI
using namespace ohx;

extern "C" {

int ohx_abi_version(void) { return OHX_ABI_VERSION; }

const char* ohx_last_error(void) { return last_error(); }

int ohx_device_count(int* n) {
  return guard([&] {
    int k = 0;
    check_cuda(cudaGetDeviceCount(&k), "cudaGetDeviceCount");
    *n = k;
  });
}

int ohx_ctx_create(int device, ohx_ctx** out) {
  return guard([&] { *out = create_ctx(device); });
}

int ohx_ctx_destroy(ohx_ctx* ctx) {
  return guard([&] { destroy_ctx(ctx); });
}

int ohx_ctx_trim(ohx_ctx* ctx) {
  return guard([&] {
    std::lock_guard<std::mutex> g(ctx->mu);
    trim_ctx(ctx);
  });
}

int ohx_ctx_default(int device, ohx_ctx** out) {
  return guard([&] { *out = default_ctx(device); });
}

int ohx_ctx_device(const ohx_ctx* ctx) { return ctx ? ctx->device : -1; }

// both read state that pipeline calls write under the context's lock
uint64_t ohx_ctx_launches(const ohx_ctx* ctx) {
  if (!ctx) return 0;
  std::lock_guard<std::mutex> g(const_cast<ohx_ctx*>(ctx)->mu);
  return ctx->launches;
}

int ohx_ctx_last_run(const ohx_ctx* ctx, ohx_run_info* info) {
  return guard([&] {
    std::lock_guard<std::mutex> g(const_cast<ohx_ctx*>(ctx)->mu);
    *info = ctx->last_run;
  });
}

int ohx_ctx_kernel_ms(ohx_ctx* ctx, double ms[4]) {
  return guard([&] {
    std::lock_guard<std::mutex> g(ctx->mu);
    bind(ctx);
    for (int k = 0; k < 4; ++k) {
      ms[k] = -1.0;
      if (!ctx->timed[k]) continue;
      float v = 0.f;
      check_cuda(cudaEventSynchronize(ctx->ev[k][1]), "cudaEventSynchronize");
      check_cuda(cudaEventElapsedTime(&v, ctx->ev[k][0], ctx->ev[k][1]), "cudaEventElapsedTime");
      ms[k] = v;
    }
  });
}

int ohx_ctx_kernel_ms_sum(ohx_ctx* ctx, double sum[4], uint64_t count[4], int reset) {
  return guard([&] {
    std::lock_guard<std::mutex> g(ctx->mu);
    bind(ctx);
    fold_stage_times(ctx, true);
    for (int k = 0; k < 4; ++k) {
      sum[k] = ctx->ksum[k];
      count[k] = ctx->kcnt[k];
      if (reset) {
        ctx->ksum[k] = 0;
        ctx->kcnt[k] = 0;
      }
    }
  });
}

int ohx_extremes(ohx_ctx* ctx, const double* d_xy, uint64_t n, uint64_t index_base,
                 ohx_extremes_rec* h_rec, void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> g(ctx->mu);
    bind(ctx);
    extremes(ctx, d_xy, n, index_base, h_rec, pick(ctx, stream));
  });
}

int ohx_pts2_count(const char* path, uint64_t* n) {
  return guard([&] { *n = pts2_count(path); });
}

int ohx_pts2_load_device(ohx_ctx* ctx, const char* path, double* d_xy, uint64_t cap, uint64_t* n,
                         void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> g(ctx->mu);
    bind(ctx);
    *n = load_pts2_device(ctx, path, d_xy, cap, pick(ctx, stream));
  });
}

int ohx_fused_extremes(ohx_ctx* ctx, const double* d_xy, uint64_t n, uint64_t index_base,
                       ohx_extremes_rec* h_rec, int* fused, void* stream) {
  return guard([&] {
    if (n == 0) throw std::invalid_argument("find_extremes: empty point set");
    std::lock_guard<std::mutex> g(ctx->mu);
    bind(ctx);
    for (bool& t : ctx->timed) t = false;
    FilterOut f{};
    Trace tr;
    *fused = fused_begin(ctx, d_xy, n, index_base, f, h_rec, pick(ctx, stream), tr) ? 1 : 0;
    ctx->last_run = {};
    ctx->last_run.candidates = f.candidates;
    ctx->last_run.fuse_state = f.fuse_state;
    ctx->last_run.sample_coverage = f.sample_coverage;
  });
}

int ohx_filter_fused(ohx_ctx* ctx, const double* d_xy, uint64_t n, uint64_t index_base,
                     const ohx_extreme_set* ext, const ohx_filter_plan* plan, uint8_t* d_labels,
                     uint64_t h_counts[4], int* fused, void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> g(ctx->mu);
    bind(ctx);
    FilterOut f{};
    fused_finish(ctx, d_xy, n, index_base, *ext, *plan, d_labels, h_counts, f, pick(ctx, stream));
    *fused = f.fused ? 1 : 0;
    ctx->last_run.fused = f.fused;
    ctx->last_run.fuse_state = f.fuse_state;
    for (int q = 0; q < 4; ++q) ctx->last_run.counts[q] = h_counts[q];
  });
}

int ohx_extremes_combine(const ohx_extremes_rec* recs, int k, ohx_extremes_rec* out) {
  return guard([&] { combine_extremes(recs, k, out); });
}

int ohx_extremes_resolve(const ohx_extremes_rec* rec, ohx_extreme_set* out,
                         uint32_t* uncertified_mask) {
  return guard([&] {
    const std::uint32_t m = resolve_extremes(*rec, out);
    if (uncertified_mask) *uncertified_mask = m;
  });
}

int ohx_corners_exact(ohx_ctx* ctx, const double* d_xy, uint64_t n,
                      uint64_t index_base, const double bbox[4],
                      ohx_corner_rec* h_rec, void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> g(ctx->mu);
    bind(ctx);
    corners_exact(ctx, d_xy, n, index_base, bbox, h_rec, pick(ctx, stream));
  });
}

int ohx_corners_combine(const ohx_corner_rec* recs, int k, ohx_corner_rec* out) {
  return guard([&] { combine_corners(recs, k, out); });
}

int ohx_build_octagon(const double cand_xy[16], double oct_xy[16], int* m) {
  return guard([&] { *m = build_octagon(cand_xy, oct_xy); });
}

int ohx_filter_plan_build(const ohx_extreme_set* ext, const double* oct_xy, int m,
                          ohx_filter_plan* plan) {
  return guard([&] { make_plan(*ext, oct_xy, m, plan); });
}

int ohx_filter(ohx_ctx* ctx, const double* d_xy, uint64_t n, uint64_t index_base,
               const ohx_filter_plan* plan, uint8_t* d_labels, uint64_t h_counts[4],
               void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> g(ctx->mu);
    bind(ctx);
    filter(ctx, d_xy, n, index_base, *plan, d_labels, h_counts, pick(ctx, stream));
  });
}

int ohx_queue_fetch(ohx_ctx* ctx, int q, uint64_t* h_idx, double* h_xy, uint64_t cap,
                    void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> g(ctx->mu);
    bind(ctx);
    queue_fetch(ctx, q, h_idx, h_xy, cap, pick(ctx, stream));
  });
}

namespace {
void hull_indices_impl(ohx_ctx* ctx, const double* h_hull, uint64_t h, uint64_t* h_idx,
                       void* stream, bool partial) {
  {
    if (!ctx) ctx = default_ctx(-1);
    std::lock_guard<std::mutex> g(ctx->mu);
    bind(ctx);
    if (ctx->last_n == 0) throw std::invalid_argument("hull_indices: no filter result in this context");
    if (h == 0) return;
    if (h >= 0xffffffffull) throw std::invalid_argument("hull_indices: hull too large");
    cudaStream_t s = pick(ctx, stream);
    std::uint64_t nslots = 1;
    while (nslots < 2 * h) nslots <<= 1;
    // one stream-ordered scratch block: hull copy, result, table
    const std::uint64_t bytes = h * 16 + h * 8 + nslots * 4;
    void* scratch = nullptr;
    check_cuda(cudaMallocAsync(&scratch, bytes, s), "cudaMallocAsync(hull indices)");
    auto* d_hull = static_cast<double*>(scratch);
    auto* d_res = reinterpret_cast<unsigned long long*>(d_hull + 2 * h);
    auto* d_slots = reinterpret_cast<std::uint32_t*>(d_res + h);
    cudaError_t err = cudaMemcpyAsync(d_hull, h_hull, h * 16, cudaMemcpyHostToDevice, s);
    if (err == cudaSuccess) {
      launch_hull_indices(ctx->last_xy, ctx->d_queues, ctx->last_idx_bytes, ctx->last_cap,
                          ctx->last_counts, ctx->last_base, d_hull, h, d_slots, nslots, d_res, s);
      ctx->launches += 2;
      err = cudaMemcpyAsync(h_idx, d_res, h * 8, cudaMemcpyDeviceToHost, s);
    }
    cudaFreeAsync(scratch, s);
    check_cuda(err, "hull indices");
    check_cuda(cudaStreamSynchronize(s), "hull indices");
    for (std::uint64_t i = 0; i < h && !partial; ++i)
      if (h_idx[i] == ~0ull)
        throw std::invalid_argument("hull_indices: a vertex is not among the last call's survivors");
  }
}
}  // namespace

int ohx_hull_indices(ohx_ctx* ctx, const double* h_hull, uint64_t h, uint64_t* h_idx,
                     void* stream) {
  return guard([&] { hull_indices_impl(ctx, h_hull, h, h_idx, stream, false); });
}

int ohx_hull_indices_partial(ohx_ctx* ctx, const double* h_hull, uint64_t h, uint64_t* h_idx,
                             void* stream) {
  return guard([&] { hull_indices_impl(ctx, h_hull, h, h_idx, stream, true); });
}

int ohx_queue_device(ohx_ctx* ctx, int q, const void** d_idx, int* idx_bytes,
                     uint64_t* count) {
  return guard([&] {
    if (q < 1 || q > 4) throw std::invalid_argument("queue must be 1..4");
    *d_idx = static_cast<const char*>(ctx->d_queues) +
             std::uint64_t(q - 1) * ctx->last_cap * ctx->last_idx_bytes;
    *idx_bytes = ctx->last_idx_bytes;
    *count = ctx->last_counts[q - 1];
  });
}

}  // extern "C"
