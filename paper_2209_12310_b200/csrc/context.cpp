// context.cpp -- device contexts and their workspaces: grow-only device /
// pinned buffers, the pinned staging ring for pageable user buffers, the
// PTS2 loader straight to device memory, error plumbing.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <omp.h>
#include <unistd.h>
#include <emmintrin.h>

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

bool dev_grow(void** p, std::uint64_t* have, std::uint64_t need, const char* what) {
  if (*have >= need && *p) return false;
  if (*p) check_cuda(cudaFree(*p), "cudaFree");
  *p = nullptr;
  *have = 0;
  cudaError_t e = cudaMalloc(p, need);
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(OHX_E_NOMEM, std::string("cudaMalloc(") + what + ", " +
                                 std::to_string(need) + " bytes) failed: " +
                                 cudaGetErrorString(e));
  }
  *have = need;
  return true;
}

cudaStream_t pick(ohx_ctx* c, void* s) {
  return s ? static_cast<cudaStream_t>(s) : c->stream;
}

void bind(ohx_ctx* c) { check_cuda(cudaSetDevice(c->device), "cudaSetDevice"); }

void ensure_partials(ohx_ctx* c, int grid) {
  if (grid <= c->partial_cap) return;
  if (c->d_partials) check_cuda(cudaFree(c->d_partials), "cudaFree");
  c->d_partials = nullptr;
  check_cuda(cudaMalloc(&c->d_partials, sizeof(K1Partial) * grid), "cudaMalloc(partials)");
  c->partial_cap = grid;
}
namespace {
thread_local std::string g_last_error;
}  // namespace
void set_last_error(const char* msg) { g_last_error = msg; }
const char* last_error() { return g_last_error.c_str(); }

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    const int code = (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
                         ? OHX_E_NODEVICE
                         : (e == cudaErrorMemoryAllocation ? OHX_E_NOMEM : OHX_E_CUDA);
    throw Error(code, std::string(what) + ": " + cudaGetErrorString(e));
  }
}
// =================================================== internal pipeline API
cudaStream_t ctx_stream(ohx_ctx* c) { return c->stream; }
std::mutex& ctx_mutex(ohx_ctx* c) { return c->mu; }
void ctx_bind(ohx_ctx* c) { bind(c); }
void ctx_set_host_lanes(ohx_ctx* c, int lanes) { c->host_lanes = lanes; }

// ---- host <-> device copies of user buffers.  Page-locked memory is
// copied directly; pageable memory (std::vector, numpy: what the reference's
// API and bindings pass) would go through the driver's staging at ~11 GB/s,
// so it goes through the context's ring of pinned chunks instead: host
// threads copy chunk k into a pinned buffer while the copy engine moves
// chunk k-1 (PCIe-bound, ~55 GB/s).
constexpr std::uint64_t kStageChunk = 64ull << 20;  // bytes per pinned chunk
constexpr std::uint64_t kStageMin = 1ull << 20;     // smaller copies go direct

bool is_pinned(const void* h) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void ensure_stage(ohx_ctx* c) {
  if (c->h_stage[0]) return;
  for (int b = 0; b < ohx_ctx::kStageBufs; ++b) {
    check_cuda(cudaMallocHost(&c->h_stage[b], kStageChunk), "cudaMallocHost(staging)");
    check_cuda(cudaEventCreateWithFlags(&c->stage_ev[b], cudaEventDisableTiming),
               "cudaEventCreate(staging)");
  }
}

// Copy with non-temporal stores: the staged bytes are not read again by
// this core (a user buffer filled from the ring, or a ring chunk the copy
// engine reads next), so streaming stores skip the read-for-ownership of
// every destination line and leave the caches alone.
void stream_copy(char* dst, const char* src, std::uint64_t bytes) {
  const std::uint64_t head = std::min<std::uint64_t>(bytes, (64 - (reinterpret_cast<std::uintptr_t>(dst) & 63)) & 63);
  std::memcpy(dst, src, head);
  dst += head;
  src += head;
  bytes -= head;
  const std::uint64_t body = bytes & ~std::uint64_t(63);
  if (reinterpret_cast<std::uintptr_t>(src) & 15) {  // unaligned source
    for (std::uint64_t k = 0; k < body; k += 64)
      for (int u = 0; u < 4; ++u)
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + k + 16 * u),
                         _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + k + 16 * u)));
  } else {
    for (std::uint64_t k = 0; k < body; k += 64)
      for (int u = 0; u < 4; ++u)
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + k + 16 * u),
                         _mm_load_si128(reinterpret_cast<const __m128i*>(src + k + 16 * u)));
  }
  _mm_sfence();
  std::memcpy(dst + body, src + body, bytes - body);
}

void host_memcpy(void* dst, const void* src, std::uint64_t bytes, int lanes) {
  if (bytes < (8ull << 20) || lanes == 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
#pragma omp parallel num_threads(team(lanes > 0 ? lanes : omp_get_max_threads()))
  {
    const int t = omp_get_thread_num(), nt = omp_get_num_threads();
    const std::uint64_t b = bytes * t / nt, e = bytes * (t + 1) / nt;
    stream_copy(static_cast<char*>(dst) + b, static_cast<const char*>(src) + b, e - b);
  }
}

void copy_h2d(ohx_ctx* c, void* d, const void* h, std::uint64_t bytes, cudaStream_t s) {
  if (bytes < kStageMin || is_pinned(h)) {
    check_cuda(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s), "cudaMemcpyAsync(H2D)");
    return;
  }
  ensure_stage(c);
  const std::uint64_t chunks = (bytes + kStageChunk - 1) / kStageChunk;
  for (std::uint64_t k = 0; k < chunks; ++k) {
    const int b = static_cast<int>(k % ohx_ctx::kStageBufs);
    const std::uint64_t off = k * kStageChunk, len = std::min(kStageChunk, bytes - off);
    if (k >= ohx_ctx::kStageBufs)
      check_cuda(cudaEventSynchronize(c->stage_ev[b]), "cudaEventSynchronize(staging)");
    host_memcpy(c->h_stage[b], static_cast<const char*>(h) + off, len, c->host_lanes);
    check_cuda(cudaMemcpyAsync(static_cast<char*>(d) + off, c->h_stage[b], len,
                               cudaMemcpyHostToDevice, s), "cudaMemcpyAsync(H2D chunk)");
    check_cuda(cudaEventRecord(c->stage_ev[b], s), "cudaEventRecord(staging)");
  }
}

void copy_d2h(ohx_ctx* c, void* h, const void* d, std::uint64_t bytes, cudaStream_t s) {
  if (bytes < kStageMin || is_pinned(h)) {
    check_cuda(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync(D2H)");
    check_cuda(cudaStreamSynchronize(s), "D2H");
    return;
  }
  ensure_stage(c);
  const std::uint64_t chunks = (bytes + kStageChunk - 1) / kStageChunk;
  auto drain = [&](std::uint64_t k) {  // chunk k has been issued: copy it out
    const int b = static_cast<int>(k % ohx_ctx::kStageBufs);
    const std::uint64_t off = k * kStageChunk, len = std::min(kStageChunk, bytes - off);
    check_cuda(cudaEventSynchronize(c->stage_ev[b]), "cudaEventSynchronize(staging)");
    host_memcpy(static_cast<char*>(h) + off, c->h_stage[b], len, c->host_lanes);
  };
  for (std::uint64_t k = 0; k < chunks; ++k) {
    const int b = static_cast<int>(k % ohx_ctx::kStageBufs);
    if (k >= ohx_ctx::kStageBufs) drain(k - ohx_ctx::kStageBufs);
    const std::uint64_t off = k * kStageChunk, len = std::min(kStageChunk, bytes - off);
    check_cuda(cudaMemcpyAsync(c->h_stage[b], static_cast<const char*>(d) + off, len,
                               cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync(D2H chunk)");
    check_cuda(cudaEventRecord(c->stage_ev[b], s), "cudaEventRecord(staging)");
  }
  for (std::uint64_t k = chunks > ohx_ctx::kStageBufs ? chunks - ohx_ctx::kStageBufs : 0;
       k < chunks; ++k)
    drain(k);
}

// A PTS2 file straight into device memory: the payload
// streams through the pinned staging ring -- host threads pread chunk k
// while the copy engine moves chunk k-1 -- and a device scan finds the
// first non-finite point (reference io.cpp:87-124 semantics and messages).
std::uint64_t load_pts2_device(ohx_ctx* c, const std::string& path, double* d_xy,
                               std::uint64_t cap, cudaStream_t s) {
  const std::uint64_t n = pts2_count(path);
  if (n > cap) throw std::invalid_argument(path + ": " + std::to_string(n) +
                                           " points exceed the device buffer (" +
                                           std::to_string(cap) + ")");
  const int fd = ::open(path.c_str(), O_RDONLY);
  if (fd < 0) io_fail(path, "cannot open for reading");
  ensure_stage(c);
  const std::uint64_t bytes = 16 * n;
  const std::uint64_t chunks = (bytes + kStageChunk - 1) / kStageChunk;
  bool ok = true;
  for (std::uint64_t k = 0; k < chunks && ok; ++k) {
    const int b = static_cast<int>(k % ohx_ctx::kStageBufs);
    const std::uint64_t off = k * kStageChunk, len = std::min(kStageChunk, bytes - off);
    if (k >= ohx_ctx::kStageBufs)
      check_cuda(cudaEventSynchronize(c->stage_ev[b]), "cudaEventSynchronize(staging)");
    char* dst = static_cast<char*>(c->h_stage[b]);
#pragma omp parallel num_threads(team(len >= (16u << 20) ? 8 : 1)) reduction(&& : ok)
    {
      const int t = omp_get_thread_num(), nt = omp_get_num_threads();
      std::uint64_t p = len * t / nt, e = len * (t + 1) / nt;
      while (p < e && ok) {
        const ssize_t r = ::pread(fd, dst + p, static_cast<std::size_t>(e - p),
                                  static_cast<off_t>(12 + off + p));
        if (r <= 0) ok = false;
        else p += static_cast<std::uint64_t>(r);
      }
    }
    if (!ok) break;
    check_cuda(cudaMemcpyAsync(reinterpret_cast<char*>(d_xy) + off, dst, len,
                               cudaMemcpyHostToDevice, s), "cudaMemcpyAsync(PTS2 chunk)");
    check_cuda(cudaEventRecord(c->stage_ev[b], s), "cudaEventRecord(staging)");
  }
  ::close(fd);
  if (!ok) {
    check_cuda(cudaStreamSynchronize(s), "PTS2 load");
    io_fail(path, "read error");
  }
  launch_first_nonfinite(d_xy, n, c->d_cnt, s);
  ++c->launches;
  check_cuda(cudaMemcpyAsync(c->h_cnt, c->d_cnt, 8, cudaMemcpyDeviceToHost, s),
             "cudaMemcpyAsync(non-finite)");
  check_cuda(cudaStreamSynchronize(s), "PTS2 load");
  if (*c->h_cnt < n) io_fail(path, nonfinite_message(*c->h_cnt));
  return n;
}

const double* stage_pts2(ohx_ctx* c, const std::string& path, std::uint64_t* n, cudaStream_t s) {
  const std::uint64_t count = pts2_count(path);
  dev_grow(reinterpret_cast<void**>(&c->d_pts), &c->pts_bytes, count * 16, "points");
  *n = load_pts2_device(c, path, c->d_pts, count, s);
  return c->d_pts;
}

const double* stage_points(ohx_ctx* c, const double* h_xy, std::uint64_t n,
                           cudaStream_t s) {
  const std::uint64_t bytes = n * 16;
  dev_grow(reinterpret_cast<void**>(&c->d_pts), &c->pts_bytes, bytes, "points");
  copy_h2d(c, c->d_pts, h_xy, bytes, s);
  return c->d_pts;
}

void fetch_labels(ohx_ctx* c, std::uint8_t* h_labels, const std::uint8_t* d_labels,
                  std::uint64_t n, cudaStream_t s) {
  copy_d2h(c, h_labels, d_labels, n, s);
}

std::uint8_t* stage_labels(ohx_ctx* c, std::uint64_t n) {
  dev_grow(reinterpret_cast<void**>(&c->d_labels), &c->labels_bytes, n, "labels");
  return c->d_labels;
}
void host_grow(void** p, std::uint64_t* have, std::uint64_t need, const char* what) {
  if (*have >= need && *p) return;
  if (*p) check_cuda(cudaFreeHost(*p), "cudaFreeHost");
  *p = nullptr;
  *have = 0;
  check_cuda(cudaMallocHost(p, need), what);
  *have = need;
}
ohx_ctx* create_ctx(int device) {
  int ndev = 0;
  check_cuda(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (device < 0 || device >= ndev)
    throw Error(OHX_E_NODEVICE, "device " + std::to_string(device) + " not visible (" +
                                    std::to_string(ndev) + " devices)");
  cudaDeviceProp prop;
  check_cuda(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (prop.major != 10)
    throw Error(OHX_E_NODEVICE, std::string("device ") + prop.name +
                                    " is not sm_100 (this library is built for sm_100a only)");
  auto c = std::make_unique<ohx_ctx>();
  c->device = device;
  bind(c.get());
  check_cuda(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
  check_cuda(cudaMalloc(&c->d_ticket, 256), "cudaMalloc(ticket)");
  check_cuda(cudaMemset(c->d_ticket, 0, 256), "cudaMemset(ticket)");
  // the extremes record and the four counts side by side (one copy brings
  // both back after the fused pass's candidate stage)
  check_cuda(cudaMalloc(&c->d_rec, kRecBlock), "cudaMalloc(rec)");
  check_cuda(cudaMemset(c->d_rec, 0, kRecBlock), "cudaMemset(rec)");  // the gap is copied too
  check_cuda(cudaMalloc(&c->d_crec, sizeof(ohx_corner_rec)), "cudaMalloc(crec)");
  c->d_counts = rec_counts(c->d_rec);
  check_cuda(cudaMallocHost(&c->h_rec, kRecBlock), "cudaMallocHost");
  check_cuda(cudaMallocHost(&c->h_srec, 8 * sizeof(ohx_extremes_rec)), "cudaMallocHost");
  check_cuda(cudaMallocHost(&c->h_crec, sizeof(ohx_corner_rec)), "cudaMallocHost");
  c->h_counts = rec_counts(c->h_rec);
  check_cuda(cudaMalloc(&c->d_cnt, 64), "cudaMalloc(cnt)");
  check_cuda(cudaMallocHost(&c->h_cnt, 64), "cudaMallocHost");
  for (auto& pair : c->ev)
    for (auto& e : pair) check_cuda(cudaEventCreate(&e), "cudaEventCreate");
  return c.release();
}

void destroy_ctx(ohx_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (void* p : {static_cast<void*>(c->d_partials), static_cast<void*>(c->d_ticket),
                  static_cast<void*>(c->d_rec), static_cast<void*>(c->d_crec),
                  static_cast<void*>(c->d_status),
                  c->d_queues, static_cast<void*>(c->d_pts),
                  static_cast<void*>(c->d_labels), static_cast<void*>(c->d_gather),
                  static_cast<void*>(c->d_sample), c->d_cand, static_cast<void*>(c->d_cnt),
                  c->d_regions, static_cast<void*>(c->d_cpts), c->d_hsort, c->d_hchain, c->d_poly,
                  static_cast<void*>(c->d_cycfull),
                  c->d_k2op, static_cast<void*>(c->d_spec)})
    if (p) cudaFree(p);
  for (void* p : {static_cast<void*>(c->h_rec), static_cast<void*>(c->h_srec),
                  static_cast<void*>(c->h_crec),
                  static_cast<void*>(c->h_cnt), c->h_sorted, c->h_packed,
                  static_cast<void*>(c->h_spec)})
    if (p) cudaFreeHost(p);
  for (int b = 0; b < ohx_ctx::kStageBufs; ++b) {
    if (c->h_stage[b]) cudaFreeHost(c->h_stage[b]);
    if (c->stage_ev[b]) cudaEventDestroy(c->stage_ev[b]);
  }
  for (auto& e : c->arc_ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->pipe_ev)
    if (e) cudaEventDestroy(e);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  for (auto& pair : c->ev)
    for (auto& e : pair)
      if (e) cudaEventDestroy(e);
  cudaStreamDestroy(c->stream);
  delete c;
}

// Frees the context's grow-only workspaces (device, pinned) and the host
// block cache; the next call regrows what it needs.  Any pending fused pass
// or filter result of the context is dropped.
void trim_ctx(ohx_ctx* c) {
  bind(c);
  check_cuda(cudaStreamSynchronize(c->stream), "trim");
  auto dfree = [](auto*& p, std::uint64_t* bytes) {
    if (p) cudaFree(p);
    p = nullptr;
    if (bytes) *bytes = 0;
  };
  dfree(c->d_status, &c->status_bytes);
  dfree(c->d_queues, &c->queue_bytes);
  dfree(c->d_pts, &c->pts_bytes);
  dfree(c->d_labels, &c->labels_bytes);
  dfree(c->d_gather, &c->gather_bytes);
  dfree(c->d_k2op, &c->k2op_bytes);
  dfree(c->d_spec, &c->dspec_bytes);
  c->spec_zeroed = false;
  c->qxy_valid = false;
  dfree(c->d_sample, &c->sample_bytes);
  dfree(c->d_cand, &c->cand_bytes);
  dfree(c->d_regions, &c->regions_bytes);
  dfree(c->d_cpts, &c->cpts_bytes);
  dfree(c->d_hsort, &c->hsort_bytes);
  dfree(c->d_hchain, &c->hchain_bytes);
  dfree(c->d_poly, &c->poly_bytes);
  dfree(c->d_cycfull, &c->cycfull_bytes);
  if (c->h_sorted) cudaFreeHost(c->h_sorted);
  c->h_sorted = nullptr;
  c->h_sorted_bytes = 0;
  if (c->h_packed) cudaFreeHost(c->h_packed);
  c->h_packed = nullptr;
  c->h_packed_bytes = 0;
  for (int b = 0; b < ohx_ctx::kStageBufs; ++b) {
    if (c->h_stage[b]) cudaFreeHost(c->h_stage[b]);
    if (c->stage_ev[b]) cudaEventDestroy(c->stage_ev[b]);
    c->h_stage[b] = nullptr;
    c->stage_ev[b] = nullptr;
  }
  c->fz.active = false;
  c->last_n = 0;
  c->spec_n = ~0ull;
  big_cache_trim();
}

ohx_ctx* default_ctx(int device) {
  static std::mutex mu;
  static std::vector<ohx_ctx*> ctxs;  // intentionally leaked at exit
  std::lock_guard<std::mutex> g(mu);
  if (device < 0) {
    const char* env = std::getenv("OHX_DEVICE");
    device = env ? std::atoi(env) : 0;
  }
  if (static_cast<int>(ctxs.size()) <= device) ctxs.resize(device + 1, nullptr);
  if (!ctxs[device]) ctxs[device] = create_ctx(device);
  return ctxs[device];
}

}  // namespace ohx
