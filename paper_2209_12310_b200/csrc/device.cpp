// device.cpp -- the filter pipeline on one device: K1 / K1b / K2 launches
// and their host steps, the fused single pass (provisional region, KF,
// candidate extremes, certified K2 on the candidates), the queues and the
// hull stage's device sweep sort.
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

// stage k's events bracket a launch of this call
void mark_timed(ohx_ctx* c, int k) {
  c->timed[k] = true;
  c->folded[k] = false;
}
// add this call's completed stage times to the context's running sums
// (wait: block until the events complete, else leave unfinished ones)
void fold_stage_times(ohx_ctx* c, bool wait) {
  for (int k = 0; k < 4; ++k) {
    if (!c->timed[k] || c->folded[k]) continue;
    if (wait) check_cuda(cudaEventSynchronize(c->ev[k][1]), "cudaEventSynchronize");
    float v = 0.f;
    const cudaError_t e = cudaEventElapsedTime(&v, c->ev[k][0], c->ev[k][1]);
    if (e == cudaErrorNotReady) {  // (not waiting: left for a later fold)
      cudaGetLastError();
      continue;
    }
    check_cuda(e, "cudaEventElapsedTime");
    c->ksum[k] += v;
    ++c->kcnt[k];
    c->folded[k] = true;
  }
}

void extremes(ohx_ctx* c, const double* d_xy, std::uint64_t n, std::uint64_t base,
              ohx_extremes_rec* out, cudaStream_t s) {
  if (n == 0) throw std::invalid_argument("find_axis_extremes: empty point set");
  const int grid = k1_grid(c->device, n);
  ensure_partials(c, grid);
  check_cuda(cudaEventRecord(c->ev[0][0], s), "cudaEventRecord");
  launch_k1(d_xy, n, base, c->d_partials, grid, c->d_ticket, c->d_rec, s);
  check_cuda(cudaEventRecord(c->ev[0][1], s), "cudaEventRecord");
  mark_timed(c, 0);
  ++c->launches;
  check_cuda(cudaMemcpyAsync(c->h_rec, c->d_rec, sizeof(ohx_extremes_rec),
                             cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync(rec)");
  check_cuda(cudaStreamSynchronize(s), "k1_extremes");
  *out = *c->h_rec;
}

void corners_exact(ohx_ctx* c, const double* d_xy, std::uint64_t n,
                   std::uint64_t base, const double bbox[4], ohx_corner_rec* out,
                   cudaStream_t s) {
  if (n == 0) throw std::invalid_argument("find_corner_extremes: empty point set");
  const int grid = k1_grid(c->device, n);
  ensure_partials(c, grid);
  check_cuda(cudaEventRecord(c->ev[1][0], s), "cudaEventRecord");
  launch_k1b(d_xy, n, base, bbox, c->d_partials, grid, c->d_ticket, c->d_crec, s);
  check_cuda(cudaEventRecord(c->ev[1][1], s), "cudaEventRecord");
  mark_timed(c, 1);
  ++c->launches;
  check_cuda(cudaMemcpyAsync(c->h_crec, c->d_crec, sizeof(ohx_corner_rec),
                             cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync(crec)");
  check_cuda(cudaStreamSynchronize(s), "k1b_corners");
  *out = *c->h_crec;
}
KPlan make_kplan(const ohx_filter_plan& plan, std::uint64_t base, std::uint64_t n) {
  KPlan kp;
  std::memcpy(kp.ax, plan.ax, sizeof(kp.ax));
  std::memcpy(kp.ay, plan.ay, sizeof(kp.ay));
  std::memcpy(kp.ea, plan.ea, sizeof(kp.ea));
  std::memcpy(kp.ec, plan.ec, sizeof(kp.ec));
  std::memcpy(kp.qax, plan.qax, sizeof(kp.qax));
  std::memcpy(kp.qay, plan.qay, sizeof(kp.qay));
  std::memcpy(kp.qa, plan.qa, sizeof(kp.qa));
  std::memcpy(kp.qc, plan.qc, sizeof(kp.qc));
  std::memcpy(kp.box, plan.box, sizeof(kp.box));
  for (int k = 0; k < 8; ++k) {
    const std::uint64_t g = plan.kept[k];
    kp.kept[k] = (g >= base && g - base < n) ? g - base : ~0ull;
    kp.kept_label[k] = plan.kept_label[k];
  }
  kp.m = plan.m;
  return kp;
}

// OHX_K2_ONEPASS=0: K2 over a candidate list as k2_filter + k2_compact +
// the survivors' coordinate gather (A/B hook), default: one launch writing
// queues and coordinates
bool k2_one_pass_mode() {
  static const bool v = [] {
    const char* e = std::getenv("OHX_K2_ONEPASS");
    return !(e && std::string(e) == "0");
  }();
  return v;
}

// K2 over the n points of a shard, or (d_cand != null) over the n_cand
// candidates listed there (shard-local indices, same width as the queues).
void filter_core(ohx_ctx* c, const double* d_xy, std::uint64_t n, std::uint64_t base,
                 const ohx_filter_plan& plan, std::uint8_t* d_labels, std::uint64_t counts[4],
                 cudaStream_t s, const void* d_cand, std::uint64_t n_cand,
                 const double* d_cpts) {
  Trace tr;
  const KPlan kp = make_kplan(plan, base, n);
  const std::uint64_t items = d_cand ? n_cand : n;
  const int idx_bytes = n <= 0xffffffffull ? 4 : 8;
  c->spec_n = ~0ull;
  c->qxy_valid = false;
  if (items == 0) {  // no candidates at all
    for (int q = 0; q < 4; ++q) counts[q] = 0;
  } else {
    const std::uint64_t ntiles = (items + kK2Tile - 1) / kK2Tile;
    // candidate lists: one K2 launch that also writes the survivors'
    // coordinates; all points: k2_filter + k2_compact + a coordinate gather
    const bool one_pass = d_cand != nullptr && d_cpts != nullptr &&
                          ntiles <= kK2OnePassMaxTiles && k2_one_pass_mode();
    if (!one_pass)
      dev_grow(reinterpret_cast<void**>(&c->d_status), &c->status_bytes, k2_work_bytes(ntiles),
               "k2 work area");
    // queue capacity: 1/16 of the items (at least 1M); grown to the exact
    // counts and re-run on overflow (counts are exact even when stores are
    // dropped)
    std::uint64_t cap =
        std::min<std::uint64_t>(items, std::max<std::uint64_t>(1u << 20, items / 16));
    if (c->queue_bytes / (4ull * idx_bytes) > cap)
      cap = std::min<std::uint64_t>(items, c->queue_bytes / (4ull * idx_bytes));
    constexpr std::uint64_t kSpec = ohx_ctx::kSpecSurvivors;
    constexpr std::uint32_t kSpecQ = kSpec / 4;
    host_grow(reinterpret_cast<void**>(&c->h_spec), &c->spec_bytes,
              k2_one_pass_spec_bytes(kSpecQ), "cudaMallocHost(survivors)");
    if (one_pass) {
      // work words: zeroed once here, then left zeroed by the kernel;
      // the returned block: defined once (its copy reads unused slots)
      if (dev_grow(&c->d_k2op, &c->k2op_bytes, k2_one_pass_work_bytes(), "k2 one-pass work"))
        check_cuda(cudaMemsetAsync(c->d_k2op, 0, c->k2op_bytes, s), "cudaMemsetAsync(k2 work)");
      if (dev_grow(reinterpret_cast<void**>(&c->d_spec), &c->dspec_bytes,
                   k2_one_pass_spec_bytes(kSpecQ), "k2 survivor block"))
        check_cuda(cudaMemsetAsync(c->d_spec, 0, c->dspec_bytes, s), "cudaMemsetAsync(spec)");
    }
    for (int attempt = 0; attempt < 2; ++attempt) {
      dev_grow(&c->d_queues, &c->queue_bytes, 4ull * idx_bytes * cap, "queues");
      // the first survivors' coordinates ride along with the counts: a
      // small survivor set needs no second round trip (queues_fetch_xy)
      // one pass: the first spec_q of each quadrant + the counts in one
      // copy; else the first kSpec packed [q1|q2|q3|q4] by gather_xy4_dev
      const auto spec_q = static_cast<std::uint32_t>(std::min<std::uint64_t>(kSpecQ, cap));
      grow_gather(c, one_pass ? 4 * cap * 16 : kSpec * 16);
      if (!one_pass && !c->spec_zeroed) {  // the fixed-size copy below reads past the
        // survivors actually gathered: make those bytes defined (initcheck)
        check_cuda(cudaMemsetAsync(c->d_gather, 0, kSpec * 16, s), "cudaMemsetAsync(gather)");
        c->spec_zeroed = true;
      }
      tr.fine("  k2 prep");
      check_cuda(cudaEventRecord(c->ev[2][0], s), "cudaEventRecord");
      const K2OnePassBufs ob{c->d_k2op, c->d_gather, c->d_spec, spec_q};
      launch_k2(d_xy, items, kp, c->d_status, ntiles, c->d_queues, idx_bytes, cap, d_labels,
                c->d_counts, s, d_cand, d_cpts, one_pass ? &ob : nullptr);
      check_cuda(cudaEventRecord(c->ev[2][1], s), "cudaEventRecord");
      mark_timed(c, 2);
      const unsigned long long* hc = c->h_counts;
      if (one_pass) {
        ++c->launches;
        check_cuda(cudaMemcpyAsync(c->h_spec, c->d_spec, k2_one_pass_spec_bytes(spec_q),
                                   cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync(survivors)");
        hc = reinterpret_cast<const unsigned long long*>(c->h_spec + 8ull * spec_q);
      } else {  // k2_filter + k2_compact, then the survivors' coordinates
        c->launches += 3;
        launch_gather4_dev(d_xy, c->d_queues, idx_bytes, cap, c->d_counts, kSpec, c->d_gather, s);
        check_cuda(cudaMemcpyAsync(c->h_counts, c->d_counts, 4 * sizeof(unsigned long long),
                                   cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync(counts)");
        check_cuda(cudaMemcpyAsync(c->h_spec, c->d_gather, kSpec * 16, cudaMemcpyDeviceToHost, s),
                   "cudaMemcpyAsync(survivors)");
      }
      tr.fine("  k2 issued");
      check_cuda(cudaStreamSynchronize(s), "k2_filter");
      tr.fine("  k2 synced");
      std::uint64_t mx = 0, total = 0;
      for (int q = 0; q < 4; ++q) {
        counts[q] = hc[q];
        mx = std::max<std::uint64_t>(mx, counts[q]);
        total += counts[q];
      }
      if (mx <= cap) {
        if (!one_pass) {
          if (total <= kSpec) c->spec_n = total;
        } else if (mx <= spec_q) {  // every quadrant's survivors came back: pack them
          std::uint64_t off = 0;
          for (int q = 0; q < 4; ++q) {
            std::memmove(c->h_spec + 2 * off, c->h_spec + 2 * q * spec_q, counts[q] * 16);
            off += counts[q];
          }
          c->spec_n = total;
        }
        break;
      }
      if (attempt == 1) throw Error(OHX_E_INTERNAL, "k2_filter: queue overflow after regrow");
      cap = std::min<std::uint64_t>(items, mx + mx / 8 + 1024);
    }
    c->last_cap = cap;
    c->qxy_valid = one_pass;
  }
  fold_stage_times(c, false);  // every stage of this call has completed (K2 synced)
  c->last_xy = d_xy;
  c->last_n = n;
  c->last_base = base;
  c->last_idx_bytes = idx_bytes;
  for (int q = 0; q < 4; ++q) c->last_counts[q] = counts[q];
}


void filter(ohx_ctx* c, const double* d_xy, std::uint64_t n, std::uint64_t base,
            const ohx_filter_plan& plan, std::uint8_t* d_labels, std::uint64_t counts[4],
            cudaStream_t s) {
  if (n == 0) throw std::invalid_argument("classify_points: empty point set");
  filter_core(c, d_xy, n, base, plan, d_labels, counts, s, nullptr, 0, nullptr);
}
void polygon_labels(ohx_ctx* c, const double* d_xy, std::uint64_t n, const double* poly, int m,
                    const ohx_extreme_set& ext, std::uint8_t* d_labels, cudaStream_t s) {
  // kept overrides and find_queue edges from an ordinary plan; the
  // polygon's own edges (reference orientation constants) go separately
  ohx_filter_plan plan;
  make_plan(ext, nullptr, 0, &plan);
  const KPlan kp = make_kplan(plan, 0, n);
  std::vector<double> e(4 * static_cast<std::size_t>(m));
  for (int i = 0; i < m; ++i) {
    const int j = i + 1 == m ? 0 : i + 1;
    e[4 * i] = poly[2 * i];
    e[4 * i + 1] = poly[2 * i + 1];
    e[4 * i + 2] = poly[2 * j] - poly[2 * i];          // (b.x - a.x)
    e[4 * i + 3] = poly[2 * j + 1] - poly[2 * i + 1];  // (b.y - a.y)
  }
  dev_grow(&c->d_poly, &c->poly_bytes, e.size() * 8, "polygon edges");
  check_cuda(cudaMemcpyAsync(c->d_poly, e.data(), e.size() * 8, cudaMemcpyHostToDevice, s),
             "cudaMemcpyAsync(polygon)");
  launch_polygon_labels(d_xy, n, static_cast<const double*>(c->d_poly), m, kp, d_labels, s);
  ++c->launches;
  check_cuda(cudaStreamSynchronize(s), "k3_polygon_labels");  // e is freed on return
}

void queue_fetch(ohx_ctx* c, int q, std::uint64_t* h_idx, double* h_xy,
                 std::uint64_t cap, cudaStream_t s) {
  if (q < 1 || q > 4) throw std::invalid_argument("queue must be 1..4");
  if (c->last_n == 0) throw std::invalid_argument("no filter result in this context");
  const std::uint64_t cnt = c->last_counts[q - 1];
  if (cnt > cap) throw std::invalid_argument("queue larger than the output capacity");
  if (cnt == 0) return;
  const auto* qbase = static_cast<const char*>(c->d_queues) +
                      std::uint64_t(q - 1) * c->last_cap * c->last_idx_bytes;
  if (h_xy && c->qxy_valid) {  // the one-pass K2 wrote them already
    check_cuda(cudaMemcpyAsync(h_xy, c->d_gather + 2 * std::uint64_t(q - 1) * c->last_cap,
                               cnt * 16, cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync(queue xy)");
  } else if (h_xy) {
    grow_gather(c, cnt * 16);
    c->qxy_valid = false;
    launch_gather(c->last_xy, qbase, c->last_idx_bytes, cnt, c->d_gather, s);
    ++c->launches;
    check_cuda(cudaMemcpyAsync(h_xy, c->d_gather, cnt * 16, cudaMemcpyDeviceToHost, s),
               "cudaMemcpyAsync(queue xy)");
  }
  if (h_idx) {
    if (c->last_idx_bytes == 8) {
      check_cuda(cudaMemcpyAsync(h_idx, qbase, cnt * 8, cudaMemcpyDeviceToHost, s),
                 "cudaMemcpyAsync(queue idx)");
      check_cuda(cudaStreamSynchronize(s), "queue fetch");
    } else {
      std::vector<std::uint32_t> tmp(cnt);
      check_cuda(cudaMemcpyAsync(tmp.data(), qbase, cnt * 4, cudaMemcpyDeviceToHost, s),
                 "cudaMemcpyAsync(queue idx)");
      check_cuda(cudaStreamSynchronize(s), "queue fetch");
      for (std::uint64_t k = 0; k < cnt; ++k) h_idx[k] = c->last_base + tmp[k];
    }
    if (c->last_idx_bytes == 8 && c->last_base)
      for (std::uint64_t k = 0; k < cnt; ++k) h_idx[k] += c->last_base;
  }
  check_cuda(cudaStreamSynchronize(s), "queue fetch");
}

void queues_fetch_xy(ohx_ctx* c, double* h_xy, cudaStream_t s) {
  if (c->last_n == 0) throw std::invalid_argument("no filter result in this context");
  const std::uint64_t total =
      c->last_counts[0] + c->last_counts[1] + c->last_counts[2] + c->last_counts[3];
  if (total == 0) return;
  if (c->spec_n == total) {  // already fetched with the counts
    std::memcpy(h_xy, c->h_spec, total * 16);
    return;
  }
  if (c->qxy_valid) {  // the one-pass K2 wrote them per quadrant: plain copies
    std::uint64_t off = 0;
    for (int q = 0; q < 4; ++q) {
      if (c->last_counts[q])
        check_cuda(cudaMemcpyAsync(h_xy + 2 * off, c->d_gather + 2 * std::uint64_t(q) * c->last_cap,
                                   c->last_counts[q] * 16, cudaMemcpyDeviceToHost, s),
                   "cudaMemcpyAsync(queues xy)");
      off += c->last_counts[q];
    }
    check_cuda(cudaStreamSynchronize(s), "queues fetch");
    return;
  }
  grow_gather(c, total * 16);
  launch_gather4(c->last_xy, c->d_queues, c->last_idx_bytes, c->last_cap, c->last_counts,
                 c->d_gather, s, c->last_n);
  ++c->launches;
  check_cuda(cudaMemcpyAsync(h_xy, c->d_gather, total * 16, cudaMemcpyDeviceToHost, s),
             "cudaMemcpyAsync(queues xy)");
  check_cuda(cudaStreamSynchronize(s), "queues fetch");
}
// Survivor counts from which the hull stage's sweep sort runs on the device
// (OHX_DEVICE_SORT_MIN overrides; a test and tuning hook)
std::uint64_t device_sort_min() {
  static const std::uint64_t v = [] {
    const char* e = std::getenv("OHX_DEVICE_SORT_MIN");
    return e && *e ? static_cast<std::uint64_t>(std::atoll(e)) : std::uint64_t(1) << 17;
  }();
  return v;
}
// OHX_DEVICE_CHAIN=0: the hull stage's chains on the host even when the
// device chains could prove them (test and comparison hook)
bool device_chain_mode() {
  static const bool v = [] {
    const char* e = std::getenv("OHX_DEVICE_CHAIN");
    return !(e && std::string(e) == "0");
  }();
  return v;
}
// A host-computed hull into the sink (a device sink: one H2D copy).
std::size_t emit_host_hull(const PVec& cyc, const HullSink& sink, bool dev, cudaStream_t s) {
  P2* out = sink(cyc.size());
  if (!dev) {
    copy_points(out, cyc.data(), cyc.size());
  } else if (!cyc.empty()) {
    check_cuda(cudaMemcpyAsync(out, cyc.data(), cyc.size() * 16, cudaMemcpyHostToDevice, s),
               "cudaMemcpyAsync(hull H2D)");
    check_cuda(cudaStreamSynchronize(s), "hull H2D");
  }
  return cyc.size();
}
// bytes of device memory into the sink (host: the staging path; device: D2D)
void emit_device_bytes(ohx_ctx* c, P2* out, const double* d_src, std::uint64_t bytes, bool dev,
                       cudaStream_t s) {
  if (!bytes) return;
  if (!dev) {
    copy_d2h(c, out, d_src, bytes, s);
    return;
  }
  check_cuda(cudaMemcpyAsync(out, d_src, bytes, cudaMemcpyDeviceToDevice, s),
             "cudaMemcpyAsync(hull D2D)");
}

// The chains and the cycle scan on the device over arcs already sorted on
// the device (len[q] points each, back to back); the hull goes to sink.
// false: the chunked replay could not prove every chunk -- nothing was
// written, the host chains must run.
bool hull_device_chains(ohx_ctx* c, const double* d_sorted, const std::uint64_t len[4],
                        cudaStream_t s, const HullSink& sink, std::size_t* h, bool raw,
                        bool dev) {
  Trace tr;
  dev_grow(&c->d_hchain, &c->hchain_bytes, device_chain_work_bytes(len), "hull chain work");
  DeviceCycle dc;
  const bool ok = device_chains(d_sorted, len, c->d_hchain, s, &dc, dev ? c->dev_out : nullptr,
                                dev ? c->dev_out_cap : 0);
  c->launches += dc.launches;
  c->last_run.hull_path = ok ? 1 : 2;
  tr.mark(ok ? "dev chains" : "dev chains (unproven: host chains)");
  if (!ok) return false;
  const std::uint64_t m = dc.m;
  const bool direct = dev && dc.d_cycle == c->dev_out;  // the cycle is in the caller's buffer
  if (raw) {  // the chained cycle itself (test hook)
    P2* out = sink(m);
    if (!(direct && reinterpret_cast<double*>(out) == dc.d_cycle))
      emit_device_bytes(c, out, dc.d_cycle, m * 16, dev, s);
    if (dev) check_cuda(cudaStreamSynchronize(s), "hull D2D");
    *h = m;
    return true;
  }
  if (m > 2 && !dc.front_eq_back && !dc.dups && !dc.flat && dc.bad == 0) {
    // finalize_cycle keeps every vertex: the hull is the cycle rotated to
    // its start vertex, copied straight into the caller's buffer
    P2* out = sink(m);
    const std::uint64_t b = dc.best;
    const double* cyc = dc.d_cycle;
    if (direct && reinterpret_cast<double*>(out) == dc.d_cycle) {
      if (b == 0) {  // already the hull, in place
        tr.mark("hull in place (fast path)");
        *h = m;
        return true;
      }
      check_cuda(cudaMemcpyAsync(dc.d_scratch, dc.d_cycle, m * 16, cudaMemcpyDeviceToDevice, s),
                 "cudaMemcpyAsync(cycle)");
      cyc = dc.d_scratch;
    }
    emit_device_bytes(c, out, cyc + 2 * b, (m - b) * 16, dev, s);
    emit_device_bytes(c, out + (m - b), cyc, b * 16, dev, s);
    if (dev) check_cuda(cudaStreamSynchronize(s), "hull D2D");
    tr.mark(dev ? "hull D2D (fast path)" : "hull D2H (fast path)");
    *h = m;
    return true;
  }
  // the general clean-up on the host (duplicates, collinear, peel)
  PVec cyc(m);
  if (m) copy_d2h(c, cyc.data(), dc.d_cycle, m * 16, s);
  const PVec d = finalize_cycle(std::move(cyc));
  emit_host_hull(d, sink, dev, s);
  tr.mark("hull D2H + finalize");
  *h = d.size();
  return true;
}

// OHX_HULL_PIPE=0: the hull stage of a large survivor set never pipelined
// with its own transfer (A/B and test hook)
bool hull_pipe_mode() {
  static const bool v = [] {
    const char* e = std::getenv("OHX_HULL_PIPE");
    return !(e && std::string(e) == "0");
  }();
  return v;
}
// survivors from which pipelining pays (OHX_HULL_PIPE_MIN overrides; test hook)
std::uint64_t pipe_min() {
  static const std::uint64_t v = [] {
    const char* e = std::getenv("OHX_HULL_PIPE_MIN");
    return e && *e ? static_cast<std::uint64_t>(std::atoll(e)) : std::uint64_t(1) << 22;
  }();
  return v;
}

// The hull stage of a large survivor set whose hull goes to PINNED host
// memory, arc by arc: each arc is sorted and chained on the device and its
// chain copied to the host on a second stream while the next arc is
// sorted and chained -- the hull's own transfer (1.55 GB for the circle's
// 96.8M vertices, 28 ms over PCIe) then hides most of the device work.
// The statistics over the whole cycle decide at the end: the cycle is the
// hull as is (the usual case), a rotation of it, or the host clean-up runs
// from the copy already in the caller's buffer.  false: not taken (the
// caller runs the regular stage; nothing was returned).
bool hull_pipelined(ohx_ctx* c, const double* d_packed, const std::uint64_t counts[4],
                    const P2 anchors[4], cudaStream_t s, const HullSink& sink, std::size_t* h) {
  const std::uint64_t total = counts[0] + counts[1] + counts[2] + counts[3];
  if (total < pipe_min() || !hull_pipe_mode() || !device_chain_mode()) return false;
  const std::uint64_t arcs_n = total + 8;
  // a C-ABI call's page-locked output with room for every arc point
  if (c->host_out == nullptr || c->host_out_cap < arcs_n || !is_pinned(c->host_out)) return false;
  auto* out = reinterpret_cast<P2*>(c->host_out);
  Trace tr;
  dev_grow(&c->d_hsort, &c->hsort_bytes, sort_arcs_work_bytes(counts) + arcs_n * 16,
           "hull sort work");
  auto* d_sorted = reinterpret_cast<double*>(static_cast<unsigned char*>(c->d_hsort) +
                                             sort_arcs_work_bytes(counts));
  std::uint64_t len[4];
  for (int q = 0; q < 4; ++q) len[q] = counts[q] + 2;
  dev_grow(&c->d_hchain, &c->hchain_bytes, device_chain_work_bytes(len), "hull chain work");
  dev_grow(reinterpret_cast<void**>(&c->d_cycfull), &c->cycfull_bytes, arcs_n * 16, "hull cycle");
  if (!c->copy_stream)
    check_cuda(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking),
               "cudaStreamCreate(copy)");
  if (!c->pipe_ev[0])
    for (auto& e : c->pipe_ev)
      check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate(pipe)");
  std::uint64_t off = 0;
  for (int q = 0; q < 4; ++q) {
    sort_arcs(d_packed, counts, reinterpret_cast<const double*>(anchors), c->d_hsort, d_sorted, s,
              q);
    DeviceCycle dc;  // arc q's chain written straight after the arcs before it
    const bool ok = device_chains(d_sorted, len, c->d_hchain, s, &dc, c->d_cycfull + 2 * off,
                                  arcs_n - off, q);
    c->launches += 4 + dc.launches;
    if (!ok) {  // an arc the chunked chains cannot prove: the regular stage
      check_cuda(cudaStreamSynchronize(c->copy_stream), "hull copy");
      return false;
    }
    if (dc.m) {  // (a chain not written in place: copied there -- not expected)
      if (dc.d_cycle != c->d_cycfull + 2 * off)
        check_cuda(cudaMemcpyAsync(c->d_cycfull + 2 * off, dc.d_cycle, dc.m * 16,
                                   cudaMemcpyDeviceToDevice, s), "cudaMemcpyAsync(arc chain)");
      check_cuda(cudaEventRecord(c->pipe_ev[q], s), "cudaEventRecord(pipe)");
      check_cuda(cudaStreamWaitEvent(c->copy_stream, c->pipe_ev[q], 0), "cudaStreamWaitEvent");
      check_cuda(cudaMemcpyAsync(out + off, c->d_cycfull + 2 * off, dc.m * 16,
                                 cudaMemcpyDeviceToHost, c->copy_stream), "cudaMemcpyAsync(arc D2H)");
    }
    off += dc.m;
  }
  tr.mark("arcs sorted + chained");
  const std::uint64_t m = off;
  DeviceCycle st;
  device_cycle_stats(c->d_cycfull, m, len, c->d_hchain, s, &st);
  c->launches += st.launches;
  check_cuda(cudaStreamSynchronize(c->copy_stream), "hull copy");
  tr.mark("hull D2H (pipelined)");
  c->last_run.hull_path = 1;
  if (m > 2 && !st.front_eq_back && !st.dups && !st.flat && st.bad == 0) {
    const std::uint64_t b = st.best;
    if (b != 0) {  // the hull starts elsewhere in the cycle: rotated from the device copy
      copy_d2h(c, out, c->d_cycfull + 2 * b, (m - b) * 16, s);
      copy_d2h(c, out + (m - b), c->d_cycfull, b * 16, s);
    }
    sink(m);
    *h = m;
    return true;
  }
  // the general clean-up on the host, from the copy already there
  const PVec d = finalize_cycle(PVec(out, out + m));
  *h = emit_host_hull(d, sink, false, s);
  return true;
}

// The hull stage (reference hull.cpp:164-183) on survivors' coordinates
// already packed on the device as [q1|q2|q3|q4] in index order; the hull
// goes to sink.  Large sets: the arcs are built and sorted on the device
// and come back in sweep order, the chains and the clean-up run on the
// host; small sets: one D2H, then the host hull stage.
std::size_t hull_from_packed(ohx_ctx* c, const double* d_packed, const std::uint64_t counts[4],
                             const P2 anchors[4], cudaStream_t s, const HullSink& sink,
                             bool dev) {
  const std::uint64_t total = counts[0] + counts[1] + counts[2] + counts[3];
  if (total < device_sort_min()) {
    host_grow(&c->h_packed, &c->h_packed_bytes, std::max<std::uint64_t>(16, total * 16),
              "cudaMallocHost(survivors)");
    const auto* packed = static_cast<const P2*>(c->h_packed);
    if (total) {
      check_cuda(cudaMemcpyAsync(c->h_packed, d_packed, total * 16, cudaMemcpyDeviceToHost, s),
                 "cudaMemcpyAsync(survivors)");
      check_cuda(cudaStreamSynchronize(s), "survivors D2H");
    }
    const P2* qp[4];
    std::uint64_t off = 0;
    for (int k = 0; k < 4; ++k) {
      qp[k] = packed + off;
      off += counts[k];
    }
    return emit_host_hull(hull_from_queue_points(anchors, qp, counts), sink, dev, s);
  }
  if (!dev) {
    std::size_t h = 0;
    if (hull_pipelined(c, d_packed, counts, anchors, s, sink, &h)) return h;
  }
  const std::uint64_t arcs_n = total + 8;
  dev_grow(&c->d_hsort, &c->hsort_bytes, sort_arcs_work_bytes(counts) + arcs_n * 16,
           "hull sort work");
  auto* d_sorted = reinterpret_cast<double*>(static_cast<unsigned char*>(c->d_hsort) +
                                             sort_arcs_work_bytes(counts));
  c->last_run.hull_path = 3;
  Trace tr;
  sort_arcs(d_packed, counts, reinterpret_cast<const double*>(anchors), c->d_hsort, d_sorted, s);
  c->launches += 2 + 4 * 4;  // build/gather + four radix sorts
  if (tr.on) {
    check_cuda(cudaStreamSynchronize(s), "hull sort");
    tr.mark("hull dev sort");
  }
  std::uint64_t len[4];
  for (int q = 0; q < 4; ++q) len[q] = counts[q] + 2;
  if (device_chain_mode()) {
    std::size_t h = 0;
    if (hull_device_chains(c, d_sorted, len, s, sink, &h, false, dev)) return h;
  }
  host_grow(&c->h_sorted, &c->h_sorted_bytes, arcs_n * 16, "cudaMallocHost(sorted arcs)");
  // one copy per arc: arc q's chain starts as soon as its copy lands
  if (!c->arc_ev[0])
    for (auto& e : c->arc_ev)
      check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate(arc)");
  const P2* arcs[4];
  std::uint64_t off = 0;
  for (int q = 0; q < 4; ++q) {
    arcs[q] = static_cast<const P2*>(c->h_sorted) + off;
    len[q] = counts[q] + 2;
    check_cuda(cudaMemcpyAsync(static_cast<P2*>(c->h_sorted) + off,
                               reinterpret_cast<const P2*>(d_sorted) + off, len[q] * 16,
                               cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync(sorted arc)");
    check_cuda(cudaEventRecord(c->arc_ev[q], s), "cudaEventRecord(arc)");
    off += len[q];
  }
  std::atomic<int> failed{cudaSuccess};  // set by the arc threads (no throwing there)
  std::size_t h = 0;
  PVec host_out;  // a device sink: the host result, copied up once
  const HullSink host_sink = [&](std::size_t hh) {
    host_out.resize(hh);
    return host_out.data();
  };
  try {
    h = hull_from_sorted_arcs(
        arcs, len,
        [&](int q) {
          const cudaError_t e = cudaEventSynchronize(c->arc_ev[q]);
          if (e != cudaSuccess) failed = e;
          return e == cudaSuccess;
        },
        dev ? host_sink : sink);
  } catch (...) {  // a lost arc: report the CUDA error behind it
    check_cuda(static_cast<cudaError_t>(failed.load()), "cudaEventSynchronize(sorted arc)");
    throw;
  }
  if (dev) emit_host_hull(host_out, sink, true, s);
  tr.mark("hull D2H + host");
  return h;
}

std::size_t hull_from_host_packed(ohx_ctx* c, const P2* h_packed, const std::uint64_t counts[4],
                                  const P2 anchors[4], cudaStream_t s, const HullSink& sink) {
  const std::uint64_t total = counts[0] + counts[1] + counts[2] + counts[3];
  if (total >= device_sort_min()) {  // (the same stage as the device-resident survivors)
    grow_gather(c, total * 16);
    c->qxy_valid = false;
    check_cuda(cudaMemcpyAsync(c->d_gather, h_packed, total * 16, cudaMemcpyHostToDevice, s),
               "cudaMemcpyAsync(survivors H2D)");
    return hull_from_packed(c, c->d_gather, counts, anchors, s, sink);
  }
  const P2* qp[4];
  std::uint64_t off = 0;
  for (int k = 0; k < 4; ++k) {
    qp[k] = h_packed + off;
    off += counts[k];
  }
  return emit_host_hull(hull_from_queue_points(anchors, qp, counts), sink, false, s);
}

std::size_t device_queues_hull(ohx_ctx* c, const FilterOut& f, cudaStream_t s,
                               const HullSink& sink, bool dev) {
  // reference hull.cpp:164-183 on the device queues of the last filter
  const std::uint64_t total = f.counts[0] + f.counts[1] + f.counts[2] + f.counts[3];
  const P2 anchors[4] = {{f.ext.x[OHX_EAST], f.ext.y[OHX_EAST]},
                         {f.ext.x[OHX_NORTH], f.ext.y[OHX_NORTH]},
                         {f.ext.x[OHX_WEST], f.ext.y[OHX_WEST]},
                         {f.ext.x[OHX_SOUTH], f.ext.y[OHX_SOUTH]}};
  if (total >= device_sort_min()) {
    grow_gather(c, total * 16);
    c->qxy_valid = false;
    launch_gather4(c->last_xy, c->d_queues, c->last_idx_bytes, c->last_cap, c->last_counts,
                   c->d_gather, s, c->last_n);
    ++c->launches;
    return hull_from_packed(c, c->d_gather, f.counts, anchors, s, sink, dev);
  }
  // small sets: the survivors' coordinates (usually already fetched with
  // the K2 counts; else copied into a pinned buffer -- pageable copies
  // went through the driver's staging, ~0.1 ms for the square's 16K), then
  // the host hull stage reads them in place
  const P2* packed = reinterpret_cast<const P2*>(c->h_spec);
  if (c->spec_n != total) {
    host_grow(&c->h_packed, &c->h_packed_bytes, std::max<std::uint64_t>(16, total * 16),
              "cudaMallocHost(survivors)");
    queues_fetch_xy(c, static_cast<double*>(c->h_packed), s);
    packed = static_cast<const P2*>(c->h_packed);
  }
  const P2* qp[4];
  std::uint64_t off = 0;
  for (int k = 0; k < 4; ++k) {
    qp[k] = packed + off;
    off += f.counts[k];
  }
  return emit_host_hull(hull_from_queue_points(anchors, qp, f.counts), sink, dev, s);
}

PVec device_queues_hull(ohx_ctx* c, const FilterOut& f, cudaStream_t s) {
  PVec out;
  device_queues_hull(c, f, s, [&](std::size_t h) {
    out.resize(h);
    return out.data();
  });
  return out;
}
void finish_extremes(ohx_ctx* c, const double* d_xy, std::uint64_t n,
                     const ohx_extremes_rec& rec, FilterOut& f, cudaStream_t s,
                     bool with_box) {
  const std::uint32_t mask = resolve_extremes(rec, &f.ext);
  f.corner_pass = mask != 0;
  if (mask) {
    const double bbox[4] = {rec.x[OHX_EAST], rec.y[OHX_NORTH], rec.x[OHX_WEST],
                            rec.y[OHX_SOUTH]};
    ohx_corner_rec cr;
    corners_exact(c, d_xy, n, 0, bbox, &cr, s);
    apply_corners(cr, &f.ext);
  }
  const int slot[8] = {OHX_EAST, OHX_NE, OHX_NORTH, OHX_NW,
                       OHX_WEST, OHX_SW, OHX_SOUTH, OHX_SE};
  double cand[16];
  for (int k = 0; k < 8; ++k) {
    cand[2 * k] = f.ext.x[slot[k]];
    cand[2 * k + 1] = f.ext.y[slot[k]];
  }
  f.m = build_octagon(cand, f.oct);
  make_plan(f.ext, f.oct, f.m, &f.plan, with_box);
}

constexpr std::uint64_t kFuseMinPoints = 1ull << 23;  // below: both passes are cheap

// OHX_FUSE: unset/"auto" = fused pass when it pays, "0" = always two passes,
// "fallback" = run the fused pass but reject its region (exercises the
// verification-failure path), "force" = fuse whatever the sample coverage
// (exercises heavy candidate lists).  The last two are for tests.
int fuse_mode() {
  static const int mode = [] {
    const char* e = std::getenv("OHX_FUSE");
    if (!e || !*e || std::string(e) == "auto") return 1;
    if (std::string(e) == "0") return 0;
    if (std::string(e) == "fallback") return 2;
    if (std::string(e) == "force") return 3;
    return 1;
  }();
  return mode;
}
constexpr int kSampleLen = 8192;     // points per sample run
static_assert(kSampleLen % 2048 == 0, "k1_small reads sample runs 2048 points at a time");
constexpr int kCoverageRuns = 64;     // coverage counted on 64 evenly spaced runs
int coverage_step(int segs) {  // OHX_COVERAGE_STEP overrides (tuning hook)
  static const int v = [] {
    const char* e = std::getenv("OHX_COVERAGE_STEP");
    return e ? std::atoi(e) : 0;
  }();
  return v >= 1 ? v : std::max(1, segs / kCoverageRuns);
}
constexpr int kSampleMaxSegs = 512;  // runs (4M points, 64 MB) for n >= 2^26
// OHX_SAMPLE_SEGS overrides the cap (experiment switch)
int sample_max_segs() {
  static const int v = [] {
    const char* e = std::getenv("OHX_SAMPLE_SEGS");
    const int k = e ? std::atoi(e) : 0;
    return k >= 64 ? k : kSampleMaxSegs;
  }();
  return v;
}
// Four disjoint sub-samples (tools/sample_config_sweep.py, normal 1e9 over
// seeds: 8 x 128 runs -> 1.19M candidates, 2.570 ms; 4 x 128 -> 0.68M,
// 2.521 ms; 3 -> 0.61M, 2.510 ms; 2 sub-samples left a 30M-point region
// uncertified once -- fewer octagons to intersect, a larger but riskier Q).
constexpr int kMaxSubSamples = 8;
constexpr int kSubSamples = 4;
int sub_samples() {  // OHX_SUBSAMPLES overrides (1..8; tuning hook)
  static const int v = [] {
    const char* e = std::getenv("OHX_SUBSAMPLES");
    const int k = e ? std::atoi(e) : 0;
    return k >= 1 && k <= kMaxSubSamples ? k : kSubSamples;
  }();
  return v;
}
constexpr double kFuseMinCoverage = 0.8;
// The provisional region of the fused pass.  A sample of about n/16 points
// (up to 4M: runs of kSampleLen consecutive points at evenly spaced offsets,
// read in place) is split into kSubSamples disjoint sub-samples (run b goes
// to sub-sample b % kSubSamples, so each spans the whole index range); each
// one's eight extremes (one batched launch) give an octagon, and Q is fitted
// inside the INTERSECTION of those octagons.  The sub-sample octagons
// scatter the way the true octagon may sit relative to any one sample's, so
// a region inside all of them rarely leaves the true octagon (checked
// exactly after the pass; a miss costs the regular second pass).  Q's bounds
// are also kept strictly below the whole sample's extremes keys, which is
// what lets the fused pass skip the extremes test for points inside Q.
// Returns false when fusing does not pay (small input, no region, sample
// coverage below kFuseMinCoverage).
bool provisional_region(ohx_ctx* c, const double* d_xy, std::uint64_t n, KFRegion* q,
                        std::uint64_t* sampled, cudaStream_t s, FilterOut& f, Trace& tr) {
  if (n < kFuseMinPoints || fuse_mode() == 0) return false;
  f.fuse_state = 2;
  // about n/16 sampled points, 64..1024 runs, a multiple of the sub-samples
  const int subs = sub_samples();
  const int segs = static_cast<int>(std::clamp<std::uint64_t>(
                       n / (16ull * kSampleLen), 64, sample_max_segs())) / subs * subs;
  dev_grow(reinterpret_cast<void**>(&c->d_sample), &c->sample_bytes,
           kMaxSubSamples * sizeof(ohx_extremes_rec), "sample records");
  auto* d_recs = reinterpret_cast<ohx_extremes_rec*>(c->d_sample);
  ensure_partials(c, segs);
  launch_k1_sample(d_xy, n, segs, kSampleLen, subs, c->d_partials, c->d_ticket, d_recs, c->d_cnt, s);
  ++c->launches;
  tr.fine("  sample issued");
  static_assert(kMaxSubSamples <= 8, "h_srec holds 8 records");
  const ohx_extremes_rec* rs = c->h_srec;  // pinned: a direct DMA, no staging copy
  check_cuda(cudaMemcpyAsync(c->h_srec, d_recs, subs * sizeof(ohx_extremes_rec),
                             cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync(sample recs)");
  check_cuda(cudaStreamSynchronize(s), "sample extremes");
  tr.mark("sample k1");
  const int slot[8] = {OHX_EAST, OHX_NE, OHX_NORTH, OHX_NW,
                       OHX_WEST, OHX_SW, OHX_SOUTH, OHX_SE};
  std::vector<P2> region, clipped;
  region.reserve(64);
  clipped.reserve(64);
  for (int g = 0; g < subs; ++g) {
    ohx_extreme_set es;
    resolve_extremes(rs[g], &es);  // heuristic octagons: diagonal winners need no certificate
    double cand[16], oct[16];
    for (int k = 0; k < 8; ++k) {
      cand[2 * k] = es.x[slot[k]];
      cand[2 * k + 1] = es.y[slot[k]];
    }
    const int m = build_octagon(cand, oct);
    if (m < 3) return false;
    if (g == 0) {
      for (int i = 0; i < m; ++i) region.push_back({oct[2 * i], oct[2 * i + 1]});
      continue;
    }
    for (int i = 0; i < m && region.size() >= 3; ++i) {
      const int j = i + 1 == m ? 0 : i + 1;
      clip_left(region, {oct[2 * i], oct[2 * i + 1]}, {oct[2 * j], oct[2 * j + 1]}, clipped);
      region.swap(clipped);
    }
    if (region.size() < 3) return false;
  }
  // the whole sample's best (axis) / second (diagonal) keys
  ohx_extremes_rec all;
  combine_extremes(rs, subs, &all);
  double lim[8];
  for (int a = 0; a < 8; ++a) lim[a] = a < 4 ? all.key[a] : all.second[a - 4];
  if (!fit_region(region, lim, q)) return false;
  tr.mark("region fit");
  // the coverage count stays on the device: KF reads it and runs only when
  // enough of the sample falls inside Q (no host round trip here)
  const int step = coverage_step(segs);
  launch_count_in_region(d_xy, n, segs, kSampleLen, step, *q, c->d_cnt, s);
  ++c->launches;
  *sampled = std::uint64_t((segs + step - 1) / step) * kSampleLen;
  f.fuse_state = 3;
  return true;
}


FilterOut device_filter_impl(ohx_ctx* c, const double* d_xy, std::uint64_t n,
                             std::uint8_t* d_labels, cudaStream_t s);

FilterOut device_filter(ohx_ctx* c, const double* d_xy, std::uint64_t n,
                        std::uint8_t* d_labels, cudaStream_t s) {
  const FilterOut f = device_filter_impl(c, d_xy, n, d_labels, s);
  c->last_run.fused = f.fused;
  c->last_run.corner_pass = f.corner_pass;
  c->last_run.candidates = f.candidates;
  c->last_run.fuse_state = f.fuse_state;
  c->last_run.sample_coverage = f.sample_coverage;
  c->last_run.hull_path = 0;
  for (int q = 0; q < 4; ++q) c->last_run.counts[q] = f.counts[q];
  return f;
}


// Fused pass, first half, over the n points of one shard (global indices
// base + j): provisional region -> KF -> ordered candidate list -> K1 over
// the candidates.  Returns true with the shard's extremes record in *rec
// (what K1 over all points would have produced) when the fused pass ran;
// false (f.fuse_state says why) when the caller must run K1 instead.
bool fused_begin(ohx_ctx* c, const double* d_xy, std::uint64_t n, std::uint64_t base,
                 FilterOut& f, ohx_extremes_rec* rec, cudaStream_t s, Trace& tr) {
  c->fz.active = false;
  KFRegion q;
  std::uint64_t sampled = 0;
  tr.fine("  enter");
  if (!provisional_region(c, d_xy, n, &q, &sampled, s, f, tr)) return false;
  const int idx_bytes = n <= 0xffffffffull ? 4 : 8;
  const int grid = kf_grid(c->device);
  const std::uint64_t nw = std::uint64_t(grid) * kKFWarpsPerBlock;
  const std::uint64_t per = ((n + 255) / 256 + nw - 1) / nw * 256;  // points per warp
  // KF runs (device-side gate) when >= kFuseMinCoverage of the sample is in
  // Q; each warp region has room for 1.5x the miss rate that allows (+256).
  // A region that overflows sends the call down the two-pass path.
  const double min_cov = fuse_mode() == 3 ? 0.0 : kFuseMinCoverage;
  const auto gate_min = static_cast<std::uint64_t>(std::ceil(min_cov * double(sampled)));
  const std::uint64_t cap_w = std::min<std::uint64_t>(
      per, 256 + static_cast<std::uint64_t>(1.5 * (1.0 - min_cov) * double(per)));
  dev_grow(&c->d_regions, &c->regions_bytes, nw * cap_w * idx_bytes, "kf regions");
  dev_grow(reinterpret_cast<void**>(&c->d_status), &c->status_bytes, nw * 4 + 16, "kf counts");
  auto* d_wcounts = reinterpret_cast<std::uint32_t*>(c->d_status);
  check_cuda(cudaEventRecord(c->ev[0][0], s), "cudaEventRecord");
  launch_kf(d_xy, n, q, grid, c->d_regions, idx_bytes, cap_w, d_wcounts, c->d_cnt, gate_min, s);
  check_cuda(cudaEventRecord(c->ev[0][1], s), "cudaEventRecord");
  mark_timed(c, 0);
  ++c->launches;
  // candidate list + coordinates and K1 over them, sized on the device: the
  // list buffers hold cap_c candidates (more: regrown and redone below)
  check_cuda(cudaEventRecord(c->ev[3][0], s), "cudaEventRecord");
  std::uint64_t cap_c = std::max<std::uint64_t>(c->cpts_bytes / 16,
                                                std::max<std::uint64_t>(1u << 20, n / 32));
  auto candidates = [&](std::uint64_t cap) {
    dev_grow(&c->d_cand, &c->cand_bytes, cap * idx_bytes, "candidates");
    dev_grow(reinterpret_cast<void**>(&c->d_cpts), &c->cpts_bytes, cap * 16, "candidate points");
    launch_kf_gather(d_xy, c->d_regions, idx_bytes, cap_w, d_wcounts, nw, c->d_cnt, c->d_counts,
                     c->d_cand, c->d_cpts, cap, s);
    // grid sized for ~16 candidates per thread from the last call's count
    // (a hint only: the kernel covers the device-side count whatever the grid)
    const int k1g = k1_list_grid(c->cand_hint ? std::min<std::uint64_t>(cap, c->cand_hint) : cap);
    ensure_partials(c, k1g);
    launch_k1_list(c->d_cpts, cap, c->d_counts, c->d_cand, idx_bytes, base, c->d_partials, k1g,
                   c->d_ticket, c->d_rec, s);
    c->launches += 2;
    // the record and the counts after it: one copy
    check_cuda(cudaMemcpyAsync(c->h_rec, c->d_rec, kRecCountsOff + 4 * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync(rec + counts)");
    tr.fine("  cand issued");
    check_cuda(cudaStreamSynchronize(s), "kf + candidate extremes");
  };
  tr.fine("  kf issued");
  candidates(cap_c);
  tr.mark("kf+cand-k1");
  f.sample_coverage = double(c->h_counts[2]) / double(sampled);
  const std::uint64_t n_cand = c->h_counts[0];
  f.candidates = n_cand;
  if (c->h_counts[2] < gate_min) return false;  // KF did not run: low coverage
  if (n_cand == 0 || c->h_counts[1] != 0) {
    f.fuse_state = 5;  // a warp region overflowed: the two-pass path
    return false;
  }
  if (n_cand > cap_c) {  // more candidates than the list buffers held
    cap_c = n_cand;
    candidates(cap_c);
  }
  check_cuda(cudaEventRecord(c->ev[3][1], s), "cudaEventRecord");
  mark_timed(c, 3);
  *rec = *c->h_rec;
  rec->n = n;
  c->fz = {true, q, d_xy, n, base, n_cand};
  c->cand_hint = n_cand;
  return true;
}

// Fused pass, second half: with the (global) ExtremeSet and plan, the
// points KF dropped have the reference label 0 iff Q lies inside the
// octagon (exact error bounds) and holds none of the eight kept points;
// then K2 runs over the candidates only, otherwise over all n points.
void fused_finish(ohx_ctx* c, const double* d_xy, std::uint64_t n, std::uint64_t base,
                  const ohx_extreme_set& ext, const ohx_filter_plan& plan,
                  std::uint8_t* d_labels, std::uint64_t counts[4], FilterOut& f,
                  cudaStream_t s) {
  if (!c->fz.active || c->fz.d_xy != d_xy || c->fz.n != n || c->fz.base != base)
    throw std::invalid_argument("filter_fused: no fused pass over these points in this context");
  c->fz.active = false;
  const KFRegion& q = c->fz.q;
  bool ok = region_certified(plan, q) && fuse_mode() != 2;
  f.fuse_state = 4;
  for (int a = 0; a < 8 && ok; ++a) ok = !in_region_host(q, ext.x[a], ext.y[a]);
  if (!ok) {  // not certified: the regular K2 pass over all points
    ohx_filter_plan full = plan;
    ensure_box(&full);
    filter(c, d_xy, n, base, full, d_labels, counts, s);
    return;
  }
  f.fuse_state = 1;
  f.fused = true;
  Trace().fine("  certified");
  if (d_labels) check_cuda(cudaMemsetAsync(d_labels, 0, n, s), "cudaMemsetAsync(labels)");
  filter_core(c, d_xy, n, base, plan, d_labels, counts, s, c->d_cand, c->fz.n_cand, c->d_cpts);
}

// OHX_FUSED_BOX=1: fit the certified interior box in the fused path too
// (A/B hook: K2 there sees only candidates, outside the provisional region)
bool fused_box() {
  static const bool v = [] {
    const char* e = std::getenv("OHX_FUSED_BOX");
    return e && std::string(e) == "1";
  }();
  return v;
}

FilterOut device_filter_impl(ohx_ctx* c, const double* d_xy, std::uint64_t n,
                             std::uint8_t* d_labels, cudaStream_t s) {
  if (n == 0) throw std::invalid_argument("heaphull: empty point set");
  FilterOut f{};
  for (bool& t : c->timed) t = false;  // kernel_ms reports this pipeline's stages
  Trace tr;
  ohx_extremes_rec rec;
  if (fused_begin(c, d_xy, n, 0, f, &rec, s, tr)) {
    finish_extremes(c, d_xy, n, rec, f, s, fused_box());
    tr.mark("octagon+plan");
    fused_finish(c, d_xy, n, 0, f.ext, f.plan, d_labels, f.counts, f, s);
    tr.mark("k2");
    return f;
  }
  // ---- two passes: K1, then K2
  extremes(c, d_xy, n, 0, &rec, s);
  finish_extremes(c, d_xy, n, rec, f, s, true);
  filter(c, d_xy, n, 0, f.plan, d_labels, f.counts, s);
  return f;
}

}  // namespace ohx
