// mg.cpp -- the multi-GPU heaphull in the C host layer, over
// NCCL: one NCCL rank per GPU, either one process per GPU
// (ohx_mg_init_rank, the torchrun / MPI shape) or one process driving every
// GPU from its own thread (ohx_mg_init_all, ncclCommInitAll -- what the C++
// API uses when a ReduceEngine grants more than one worker on a multi-GPU
// box).
//
// The job's points are split into contiguous index ranges (shards); every
// index stays global, so the reference's smallest-index tie rule
// (parallel.hpp:34-43) holds across shards.  Per rank:
//   1. each of its shards: the fused pass (or K1) -> one extremes record
//   2. ncclAllGather of the rank records (296 B each); every rank runs the
//      same associative combine -> the identical global record
//   3. corner certificate; on failure K1b per shard + a second all-gather
//   4. build_octagon + plan on the host (identical on every rank)
//   5. K2 per shard (candidates only when the shard's fused region is
//      certified against the global octagon)
//   6. ncclAllGather of one fixed-size block per rank: its queue lengths
//      and, when they fit (up to kMgBlock, already on the host with the K2
//      counts), its survivors' coordinates [q1..q4]; if every rank's fit,
//      the root runs the host hull stage on them and the call ends here
//   7. else: the shard's survivors' coordinates packed on its device
//   8. survivors to the root only: each queue of each rank is one
//      ncclSend / ncclRecv straight into its place in the root's
//      [Q1|Q2|Q3|Q4] buffer (rank order = global index order, so the
//      concatenation equals build_queues, hull.cpp:124-131)
//   9. the root runs the hull stage on the device-resident survivors.
// A rank may hold several "virtual" shards (each with its own context):
// the same per-shard path as separate GPUs, which lets one device check the
// multi-shard exchange bit for bit.
//
// NCCL is loaded at run time (dlopen of libnccl.so.2, reusing the copy
// torch already loaded if any), so single-GPU use never depends on it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <functional>
#include <atomic>
#include <chrono>
#include <cstring>
#include <exception>
#include <future>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "host.hpp"
#include "internal.hpp"
#include "ohx.h"
#include "pipeline.hpp"

namespace ohx {
namespace {

// ---- NCCL, resolved at run time
struct Nccl {
  void* lib = nullptr;
  std::string why;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommInitAll) CommInitAll = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclCommAbort) CommAbort = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclBroadcast) Broadcast = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  decltype(&ncclGetVersion) GetVersion = nullptr;

  static const Nccl& get() {
    static const Nccl n = [] {
      Nccl r;
      r.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's copy, if loaded
      if (!r.lib) r.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
      if (!r.lib) r.lib = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
      if (!r.lib) {
        const char* e = dlerror();
        r.why = e ? e : "libnccl.so.2 not found";
        return r;
      }
      auto sym = [&](auto& fn, const char* name) {
        fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(r.lib, name));
        if (!fn && r.why.empty()) r.why = std::string("NCCL symbol missing: ") + name;
      };
      sym(r.GetUniqueId, "ncclGetUniqueId");
      sym(r.CommInitRank, "ncclCommInitRank");
      sym(r.CommInitAll, "ncclCommInitAll");
      sym(r.CommDestroy, "ncclCommDestroy");
      sym(r.CommAbort, "ncclCommAbort");
      sym(r.AllGather, "ncclAllGather");
      sym(r.AllReduce, "ncclAllReduce");
      sym(r.Broadcast, "ncclBroadcast");
      sym(r.Send, "ncclSend");
      sym(r.Recv, "ncclRecv");
      sym(r.GroupStart, "ncclGroupStart");
      sym(r.GroupEnd, "ncclGroupEnd");
      sym(r.GetErrorString, "ncclGetErrorString");
      sym(r.GetVersion, "ncclGetVersion");
      return r;
    }();
    if (!n.why.empty()) throw Error(OHX_E_NODEVICE, "NCCL unavailable: " + n.why);
    return n;
  }
};

// survivors per rank that travel inside the fixed-size exchange block
// (step 6): 16 KB per rank, the whole survivor set of a normal corpus
constexpr std::uint64_t kMgBlock = 1024;

void check_nccl(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  throw Error(OHX_E_CUDA, std::string(what) + ": " + Nccl::get().GetErrorString(r));
}

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t).count();
}

}  // namespace
}  // namespace ohx

// One NCCL rank held by this process: its communicator, its device, the
// contexts of its (virtual) shards and the exchange buffers.
struct ohx_mg_rank {
  int rank = 0;
  int device = 0;
  ncclComm_t comm = nullptr;
  std::vector<ohx_ctx*> shards;  // shard contexts, created on demand (owned)
  void* d_x = nullptr;           // records / counts exchange
  std::uint64_t x_bytes = 0;
  void* h_x = nullptr;           // pinned mirror of d_x
  std::uint64_t hx_bytes = 0;
  void* d_pack = nullptr;        // this rank's survivors, [q1|q2|q3|q4]
  std::uint64_t pack_bytes = 0;
  void* d_recv = nullptr;        // root: the job's survivors, [Q1|Q2|Q3|Q4]
  std::uint64_t recv_bytes = 0;
  void* h_blk = nullptr;         // pinned: this rank's block, then every rank's
  std::uint64_t hblk_bytes = 0;
  void* h_job = nullptr;         // pinned, root: small job survivors [Q1|Q2|Q3|Q4]
  std::uint64_t hjob_bytes = 0;
};

struct ohx_mg {
  std::mutex mu;
  int world = 1;
  bool single_process = false;
  bool broken = false;
  std::vector<ohx_mg_rank> ranks;  // the ranks this process drives
};

namespace ohx {
namespace {

struct ShardIn {
  const double* d_xy;
  std::uint64_t n, base;
  std::uint8_t* h_labels;  // nullable: this shard's labels (host)
  const double* h_xy;      // nullable: stage these host points first
};

struct RankOut {
  ohx_mg_info info{};
  std::size_t h = 0;
};

ohx_ctx* shard_ctx(ohx_mg_rank& R, std::size_t i) {
  while (R.shards.size() <= i) R.shards.push_back(create_ctx(R.device));
  return R.shards[i];
}

// all-gather of `bytes` per rank through the rank's exchange buffers
void allgather_host(const Nccl& N, ohx_mg_rank& R, int world, const void* mine, void* all,
                    std::uint64_t bytes, cudaStream_t s) {
  const std::uint64_t need = bytes * (world + 1);
  dev_grow(&R.d_x, &R.x_bytes, need, "mg exchange");
  host_grow(&R.h_x, &R.hx_bytes, need, "cudaMallocHost(mg exchange)");
  auto* hx = static_cast<unsigned char*>(R.h_x);
  auto* dx = static_cast<unsigned char*>(R.d_x);
  std::memcpy(hx, mine, bytes);
  check_cuda(cudaMemcpyAsync(dx, hx, bytes, cudaMemcpyHostToDevice, s), "cudaMemcpyAsync(mg)");
  check_nccl(N.AllGather(dx, dx + bytes, bytes, ncclUint8, R.comm, s), "ncclAllGather");
  check_cuda(cudaMemcpyAsync(hx + bytes, dx + bytes, bytes * world, cudaMemcpyDeviceToHost, s),
             "cudaMemcpyAsync(mg)");
  check_cuda(cudaStreamSynchronize(s), "mg all-gather");
  std::memcpy(all, hx + bytes, bytes * world);
}

// Steps 1-9 of the file comment for one rank over its shards.
RankOut run_rank(ohx_mg& M, ohx_mg_rank& R, const std::vector<ShardIn>& in, int root,
                 const HullSink& sink) {
  const Nccl& N = Nccl::get();
  check_cuda(cudaSetDevice(R.device), "cudaSetDevice");
  const int k = static_cast<int>(in.size());
  std::vector<ohx_ctx*> C(k);
  std::vector<std::unique_lock<std::mutex>> held;  // the pipeline calls' contract
  for (int i = 0; i < k; ++i) {
    C[i] = shard_ctx(R, i);
    held.emplace_back(ctx_mutex(C[i]));
  }
  cudaStream_t s = ctx_stream(C[0]);
  RankOut out;
  auto t0 = Clock::now();

  // 1. per-shard extremes (host points, when given, staged first)
  std::vector<const double*> d_xy(k);
  std::vector<FilterOut> F(k);
  std::vector<bool> fused(k, false);
  std::vector<ohx_extremes_rec> recs(k);
  for (int i = 0; i < k; ++i) {
    d_xy[i] = in[i].h_xy ? stage_points(C[i], in[i].h_xy, in[i].n, ctx_stream(C[i]))
                         : in[i].d_xy;
    for (bool& t : C[i]->timed) t = false;
    Trace tr;
    fused[i] = in[i].n > 0 &&
               fused_begin(C[i], d_xy[i], in[i].n, in[i].base, F[i], &recs[i], ctx_stream(C[i]), tr);
    if (!fused[i] && in[i].n > 0)
      extremes(C[i], d_xy[i], in[i].n, in[i].base, &recs[i], ctx_stream(C[i]));
  }
  // a rank with no points contributes the combine's identity (n = 0)
  ohx_extremes_rec local{};
  std::vector<ohx_extremes_rec> nonempty;
  for (int i = 0; i < k; ++i)
    if (in[i].n) nonempty.push_back(recs[i]);
  if (!nonempty.empty()) combine_extremes(nonempty.data(), static_cast<int>(nonempty.size()), &local);

  // 2. all-gather + the same combine everywhere
  std::vector<ohx_extremes_rec> all(M.world);
  allgather_host(N, R, M.world, &local, all.data(), sizeof(local), s);
  std::vector<ohx_extremes_rec> live;
  for (const auto& r : all)
    if (r.n) live.push_back(r);
  if (live.empty()) throw std::invalid_argument("heaphull: empty point set");
  ohx_extremes_rec g;
  combine_extremes(live.data(), static_cast<int>(live.size()), &g);

  // 3. corner certificate (+ exact corner pass on failure)
  ohx_extreme_set ext;
  const std::uint32_t mask = resolve_extremes(g, &ext);
  if (mask) {
    const double bbox[4] = {g.x[OHX_EAST], g.y[OHX_NORTH], g.x[OHX_WEST], g.y[OHX_SOUTH]};
    std::vector<ohx_corner_rec> crs;
    for (int i = 0; i < k; ++i) {
      if (!in[i].n) continue;
      ohx_corner_rec cr;
      corners_exact(C[i], d_xy[i], in[i].n, in[i].base, bbox, &cr, ctx_stream(C[i]));
      crs.push_back(cr);
    }
    ohx_corner_rec cl{};
    if (!crs.empty()) combine_corners(crs.data(), static_cast<int>(crs.size()), &cl);
    std::vector<ohx_corner_rec> call(M.world), clive;
    allgather_host(N, R, M.world, &cl, call.data(), sizeof(cl), s);
    for (const auto& c : call)
      if (c.n) clive.push_back(c);
    ohx_corner_rec cg;
    combine_corners(clive.data(), static_cast<int>(clive.size()), &cg);
    apply_corners(cg, &ext);
  }

  // 4. octagon + plan
  const int slot[8] = {OHX_EAST, OHX_NE, OHX_NORTH, OHX_NW, OHX_WEST, OHX_SW, OHX_SOUTH, OHX_SE};
  double cand[16], oct[16];
  for (int a = 0; a < 8; ++a) {
    cand[2 * a] = ext.x[slot[a]];
    cand[2 * a + 1] = ext.y[slot[a]];
  }
  const int m = build_octagon(cand, oct);
  ohx_filter_plan plan;
  bool all_fused = true;
  for (int i = 0; i < k; ++i) all_fused = all_fused && (fused[i] || in[i].n == 0);
  make_plan(ext, oct, m, &plan, !all_fused);  // fused shards' K2 needs no box
  out.info.ms[0] = ms_since(t0);
  t0 = Clock::now();

  // 5. K2 per shard
  std::vector<std::array<std::uint64_t, 4>> cnt(k);
  std::uint64_t mine[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // counts[4], fused, shards, points
  for (int i = 0; i < k; ++i) {
    cnt[i] = {0, 0, 0, 0};
    if (!in[i].n) continue;
    cudaStream_t si = ctx_stream(C[i]);
    std::uint8_t* dl = in[i].h_labels ? stage_labels(C[i], in[i].n) : nullptr;
    if (fused[i]) {
      fused_finish(C[i], d_xy[i], in[i].n, in[i].base, ext, plan, dl, cnt[i].data(), F[i], si);
    } else {
      ohx_filter_plan full = plan;
      ensure_box(&full);
      filter(C[i], d_xy[i], in[i].n, in[i].base, full, dl, cnt[i].data(), si);
    }
    if (dl) {
      fetch_labels(C[i], in[i].h_labels, dl, in[i].n, si);
      check_cuda(cudaStreamSynchronize(si), "mg labels");
    }
    ohx_run_info& lr = C[i]->last_run;  // what this shard's part of the call did
    lr.fused = F[i].fused;
    lr.corner_pass = mask != 0;
    lr.candidates = F[i].candidates;
    lr.fuse_state = F[i].fuse_state;
    lr.sample_coverage = F[i].sample_coverage;
    for (int q = 0; q < 4; ++q) lr.counts[q] = cnt[i][q];
    for (int q = 0; q < 4; ++q) mine[q] += cnt[i][q];
    mine[4] += F[i].fused ? 1 : 0;
    mine[5] += 1;
    mine[6] += in[i].n;
  }
  out.info.ms[1] = ms_since(t0);
  t0 = Clock::now();

  // 6. small survivor sets (the common case) travel in ONE fixed-size
  //    all-gather with the queue lengths: every shard's survivors came back
  //    to the host with its K2 counts (ctx->h_spec, packed [q1..q4]), so
  //    the rank's block is [counts, fused, shards, points, flag | up to
  //    kMgBlock survivors, q1..q4 with the shards in index order]; the root
  //    then runs the host hull on them -- no device pack, no second
  //    exchange, no send / recv, no survivor D2H.  Any rank over the block
  //    (or a shard whose survivors stayed on the device) sends every rank
  //    down steps 7-9 below with the lengths already known.
  const std::uint64_t my_total = mine[0] + mine[1] + mine[2] + mine[3];
  bool small = my_total <= kMgBlock;
  for (int i = 0; i < k && small; ++i) {
    const std::uint64_t t = cnt[i][0] + cnt[i][1] + cnt[i][2] + cnt[i][3];
    small = !in[i].n || t == 0 || C[i]->spec_n == t;
  }
  mine[7] = small ? 1 : 0;
  constexpr std::uint64_t kBlockBytes = 64 + kMgBlock * 16;
  host_grow(&R.h_blk, &R.hblk_bytes, kBlockBytes * (M.world + 1), "cudaMallocHost(mg block)");
  auto* blk = static_cast<unsigned char*>(R.h_blk);  // [mine | all ranks' blocks]
  std::memcpy(blk, mine, 64);
  if (small) {
    auto* dst = reinterpret_cast<P2*>(blk + 64);
    std::uint64_t off = 0;
    for (int q = 0; q < 4; ++q)
      for (int i = 0; i < k; ++i) {
        if (!cnt[i][q]) continue;
        std::uint64_t qo = 0;  // q's start in shard i's packed survivors
        for (int u = 0; u < q; ++u) qo += cnt[i][u];
        std::memcpy(dst + off, reinterpret_cast<const P2*>(C[i]->h_spec) + qo, cnt[i][q] * 16);
        off += cnt[i][q];
      }
  }
  allgather_host(N, R, M.world, blk, blk + kBlockBytes, kBlockBytes, s);
  std::vector<std::uint64_t> allc(8 * M.world);
  bool all_small = true;
  for (int r = 0; r < M.world; ++r) {
    std::memcpy(&allc[8 * r], blk + kBlockBytes * (r + 1), 64);
    all_small = all_small && allc[8 * r + 7] == 1;
  }
  std::uint64_t tq[4] = {0, 0, 0, 0};
  for (int r = 0; r < M.world; ++r) {
    for (int q = 0; q < 4; ++q) tq[q] += allc[8 * r + q];
    out.info.fused_shards += static_cast<std::uint32_t>(allc[8 * r + 4]);
    out.info.shards += static_cast<std::uint32_t>(allc[8 * r + 5]);
  }
  const std::uint64_t total = tq[0] + tq[1] + tq[2] + tq[3];
  const P2 anchors[4] = {{ext.x[OHX_EAST], ext.y[OHX_EAST]},
                         {ext.x[OHX_NORTH], ext.y[OHX_NORTH]},
                         {ext.x[OHX_WEST], ext.y[OHX_WEST]},
                         {ext.x[OHX_SOUTH], ext.y[OHX_SOUTH]}};
  if (all_small) {
    out.info.ms[2] = ms_since(t0);
    t0 = Clock::now();
    if (R.rank == root) {  // the job's [Q1|Q2|Q3|Q4]: queue q of rank 0, 1, ...
      host_grow(&R.h_job, &R.hjob_bytes, std::max<std::uint64_t>(16, total * 16),
                "cudaMallocHost(mg job survivors)");
      auto* job = static_cast<P2*>(R.h_job);
      std::uint64_t off = 0;
      for (int q = 0; q < 4; ++q)
        for (int r = 0; r < M.world; ++r) {
          const std::uint64_t c = allc[8 * r + q];
          if (!c) continue;
          std::uint64_t qo = 0;
          for (int u = 0; u < q; ++u) qo += allc[8 * r + u];
          std::memcpy(job + off, reinterpret_cast<const P2*>(blk + kBlockBytes * (r + 1) + 64) + qo,
                      c * 16);
          off += c;
        }
      out.h = hull_from_host_packed(C[0], job, tq, anchors, s, sink);
    }
  } else {
    // 7. this rank's survivors packed on its device [q1|q2|q3|q4]
    dev_grow(&R.d_pack, &R.pack_bytes, std::max<std::uint64_t>(16, my_total * 16),
             "mg survivors");
    auto* pack = static_cast<double*>(R.d_pack);
    {
      std::uint64_t off = 0;
      for (int q = 0; q < 4; ++q) {
        for (int i = 0; i < k; ++i) {
          const std::uint64_t c = cnt[i][q];
          if (!c) continue;
          const auto* qbase = static_cast<const char*>(C[i]->d_queues) +
                              std::uint64_t(q) * C[i]->last_cap * C[i]->last_idx_bytes;
          launch_gather(C[i]->last_xy, qbase, C[i]->last_idx_bytes, c, pack + 2 * off,
                        ctx_stream(C[i]));
          ++C[i]->launches;
          off += c;
        }
      }
      for (int i = 0; i < k; ++i)
        check_cuda(cudaStreamSynchronize(ctx_stream(C[i])), "mg survivor pack");
    }

    // 8. survivors to the root only, each queue slice straight into its place
    if (R.rank == root) {
      dev_grow(&R.d_recv, &R.recv_bytes, std::max<std::uint64_t>(16, total * 16),
               "mg job survivors");
    }
    auto* recv = static_cast<double*>(R.d_recv);
    check_nccl(N.GroupStart(), "ncclGroupStart");
    {
      std::uint64_t qoff = 0;  // start of Q_q in the job buffer
      std::uint64_t my_off = 0;  // start of q in this rank's pack
      for (int q = 0; q < 4; ++q) {
        std::uint64_t pos = qoff;
        for (int r = 0; r < M.world; ++r) {
          const std::uint64_t c = allc[8 * r + q];
          if (c) {
            if (R.rank == root && r == root) {
              check_cuda(cudaMemcpyAsync(recv + 2 * pos, pack + 2 * my_off, c * 16,
                                         cudaMemcpyDeviceToDevice, s), "cudaMemcpyAsync(mg own)");
            } else if (R.rank == root) {
              check_nccl(N.Recv(recv + 2 * pos, 2 * c, ncclFloat64, r, R.comm, s), "ncclRecv");
            } else if (r == R.rank) {
              check_nccl(N.Send(pack + 2 * my_off, 2 * c, ncclFloat64, root, R.comm, s),
                         "ncclSend");
            }
          }
          pos += c;
        }
        my_off += allc[8 * R.rank + q];
        qoff += tq[q];
      }
    }
    check_nccl(N.GroupEnd(), "ncclGroupEnd");
    check_cuda(cudaStreamSynchronize(s), "mg survivor gather");
    out.info.ms[2] = ms_since(t0);
    t0 = Clock::now();
    // 9. the hull stage on the root, on the device-resident survivors
    if (R.rank == root) out.h = hull_from_packed(C[0], recv, tq, anchors, s, sink);
  }
  for (int a = 0; a < 8; ++a) out.info.ext[a] = ext.ext[a];
  for (int q = 0; q < 4; ++q) out.info.counts[q] = tq[q];
  out.info.n_total = g.n;
  out.info.corner_pass = mask != 0;
  out.info.ms[3] = ms_since(t0);
  return out;
}

// Runs fn(rank index) for every local rank: the calling thread takes rank 0,
// one thread each for the others.  A failing rank aborts every local
// communicator so the others' collectives return instead of waiting for it;
// the handle is then unusable (recreate it).
void run_local(ohx_mg& M, const std::function<void(std::size_t)>& fn) {
  const std::size_t L = M.ranks.size();
  if (L == 1) {
    try {
      fn(0);
    } catch (...) {
      if (M.world > 1) {
        Nccl::get().CommAbort(M.ranks[0].comm);
        M.ranks[0].comm = nullptr;
        M.broken = true;
      }
      throw;
    }
    return;
  }
  std::vector<std::exception_ptr> err(L);
  std::atomic<bool> aborted{false};
  std::mutex abort_mu;
  auto body = [&](std::size_t r) {
    try {
      fn(r);
    } catch (...) {
      err[r] = std::current_exception();
      std::lock_guard<std::mutex> g(abort_mu);
      if (!aborted.exchange(true))
        for (auto& rk : M.ranks) Nccl::get().CommAbort(rk.comm);
    }
  };
  std::vector<std::thread> th;
  for (std::size_t r = 1; r < L; ++r) th.emplace_back(body, r);
  body(0);
  for (auto& t : th) t.join();
  if (aborted) {
    for (auto& rk : M.ranks) rk.comm = nullptr;
    M.broken = true;
  }
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

ohx_mg* new_mg() { return new ohx_mg(); }

void usable(ohx_mg* M) {
  if (!M) throw std::invalid_argument("mg: null handle");
  if (M->broken)
    throw Error(OHX_E_CUDA, "mg: a previous call failed and aborted the communicator; recreate it");
}

HullSink caller_sink(double* h_hull, std::uint64_t cap, std::uint64_t* h) {
  return [=](std::size_t hh) {
    *h = hh;
    if (hh > cap) throw std::invalid_argument("hull output capacity too small");
    return reinterpret_cast<P2*>(h_hull);
  };
}

}  // namespace

// The C++ API's multi-GPU route (octohull_api.cpp): a process-wide
// single-process communicator over the first `ndev` devices.
ohx_mg* mg_default(int ndev) {
  static std::mutex mu;
  static std::vector<ohx_mg*> cache(64, nullptr);  // intentionally leaked at exit
  std::lock_guard<std::mutex> g(mu);
  if (ndev < 1 || ndev >= static_cast<int>(cache.size()))
    throw std::invalid_argument("mg: bad device count");
  if (!cache[ndev] || cache[ndev]->broken) {
    // the reference API never mentions NCCL: a process-wide NCCL_DEBUG
    // (VERSION / WARN print a banner on stdout at the first init) must not
    // leak into the output of a program that only called heaphull --
    // e.g. the reference CLI's `verify`, whose first line must be "OK h=".
    // OHX_NCCL_DEBUG=1 keeps NCCL's own setting.
    static const bool quiet = [] {
      const char* k = std::getenv("OHX_NCCL_DEBUG");
      if (!(k && std::string(k) == "1")) unsetenv("NCCL_DEBUG");
      return true;
    }();
    (void)quiet;
    std::vector<int> devs(ndev);
    for (int d = 0; d < ndev; ++d) devs[d] = d;
    ohx_mg* m = nullptr;
    const int rc = ohx_mg_init_all(ndev, devs.data(), &m);
    if (rc != OHX_OK) throw Error(rc, last_error());
    cache[ndev] = m;
  }
  return cache[ndev];
}

// host points [0, n) split into contiguous shards over the handle's ranks
// (vshards per rank); labels (nullable) for every point
std::size_t mg_heaphull_host(ohx_mg* M, const double* h_xy, std::uint64_t n, int vshards,
                             std::uint8_t* h_labels, const HullSink& sink, ohx_mg_info* info) {
  usable(M);
  if (!M->single_process) throw std::invalid_argument("mg: host-point calls need ohx_mg_init_all");
  if (n == 0) throw std::invalid_argument("heaphull: empty point set");
  if (vshards < 1) throw std::invalid_argument("mg: vshards must be >= 1");
  const std::size_t L = M->ranks.size();
  const std::uint64_t S = L * vshards;
  std::vector<RankOut> outs(L);
  std::size_t h = 0;
  run_local(*M, [&](std::size_t r) {
    std::vector<ShardIn> in;
    for (int v = 0; v < vshards; ++v) {
      const std::uint64_t j = r * vshards + v;
      const std::uint64_t b0 = n * j / S, b1 = n * (j + 1) / S;
      in.push_back({nullptr, b1 - b0, b0, h_labels ? h_labels + b0 : nullptr, h_xy + 2 * b0});
    }
    outs[r] = run_rank(*M, M->ranks[r], in, 0, sink);
    if (r == 0) h = outs[r].h;
  });
  if (info) *info = outs[0].info;
  return h;
}

}  // namespace ohx

using ohx::check_cuda;
using ohx::guard;

extern "C" {

int ohx_mg_unique_id(uint8_t id[128]) {
  return guard([&] {
    ncclUniqueId u;
    ohx::check_nccl(ohx::Nccl::get().GetUniqueId(&u), "ncclGetUniqueId");
    static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id, &u, 128);
  });
}

int ohx_mg_init_rank(const uint8_t id[128], int world, int rank, int device, ohx_mg** out) {
  return guard([&] {
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("mg: bad rank/world");
    const auto& N = ohx::Nccl::get();
    std::unique_ptr<ohx_mg> M(ohx::new_mg());
    M->world = world;
    M->ranks.resize(1);
    auto& R = M->ranks[0];
    R.rank = rank;
    R.device = device;
    ohx::check_cuda(cudaSetDevice(device), "cudaSetDevice");
    ohx::shard_ctx(R, 0);  // validates the device (sm_100)
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    ohx::check_nccl(N.CommInitRank(&R.comm, world, u, rank), "ncclCommInitRank");
    *out = M.release();
  });
}

int ohx_mg_init_all(int ndev, const int* devices, ohx_mg** out) {
  return guard([&] {
    if (ndev < 1) throw std::invalid_argument("mg: ndev must be >= 1");
    const auto& N = ohx::Nccl::get();
    std::unique_ptr<ohx_mg> M(ohx::new_mg());
    M->world = ndev;
    M->single_process = true;
    M->ranks.resize(ndev);
    std::vector<ncclComm_t> comms(ndev);
    for (int r = 0; r < ndev; ++r) {
      M->ranks[r].rank = r;
      M->ranks[r].device = devices ? devices[r] : r;
      ohx::check_cuda(cudaSetDevice(M->ranks[r].device), "cudaSetDevice");
      ohx::shard_ctx(M->ranks[r], 0);
    }
    std::vector<int> devs(ndev);
    for (int r = 0; r < ndev; ++r) devs[r] = M->ranks[r].device;
    ohx::check_nccl(N.CommInitAll(comms.data(), ndev, devs.data()), "ncclCommInitAll");
    for (int r = 0; r < ndev; ++r) M->ranks[r].comm = comms[r];
    *out = M.release();
  });
}

int ohx_mg_destroy(ohx_mg* mg) {
  return guard([&] {
    if (!mg) return;
    {
      std::lock_guard<std::mutex> g(mg->mu);
      for (auto& R : mg->ranks) {
        cudaSetDevice(R.device);
        if (R.comm) ohx::Nccl::get().CommDestroy(R.comm);
        for (ohx_ctx* c : R.shards) ohx::destroy_ctx(c);
        for (void* p : {R.d_x, R.d_pack, R.d_recv})
          if (p) cudaFree(p);
        for (void* p : {R.h_x, R.h_blk, R.h_job})
          if (p) cudaFreeHost(p);
      }
    }
    delete mg;
  });
}

int ohx_mg_world(const ohx_mg* mg, int* world, int* local_ranks) {
  return guard([&] {
    if (!mg) throw std::invalid_argument("mg: null handle");
    if (world) *world = mg->world;
    if (local_ranks) *local_ranks = static_cast<int>(mg->ranks.size());
  });
}

int ohx_mg_ctx(ohx_mg* mg, int local_rank, int shard, ohx_ctx** ctx) {
  return guard([&] {
    if (!mg) throw std::invalid_argument("mg: null handle");
    std::lock_guard<std::mutex> g(mg->mu);
    if (local_rank < 0 || local_rank >= static_cast<int>(mg->ranks.size()) || shard < 0)
      throw std::invalid_argument("mg: no such rank");
    auto& R = mg->ranks[local_rank];
    check_cuda(cudaSetDevice(R.device), "cudaSetDevice");
    *ctx = ohx::shard_ctx(R, shard);
  });
}

int ohx_mg_nccl_version(int* version) {
  return guard([&] { ohx::check_nccl(ohx::Nccl::get().GetVersion(version), "ncclGetVersion"); });
}

int ohx_mg_heaphull_shard(ohx_mg* mg, const double* d_xy, uint64_t n, uint64_t index_base,
                          int vshards, uint8_t* h_labels, double* h_hull, uint64_t cap,
                          uint64_t* h, ohx_mg_info* info) {
  return guard([&] {
    ohx::usable(mg);
    std::lock_guard<std::mutex> g(mg->mu);
    if (mg->ranks.size() != 1)
      throw std::invalid_argument("mg: ohx_mg_heaphull_shard needs a one-rank handle (ohx_mg_init_rank)");
    if (vshards < 1) throw std::invalid_argument("mg: vshards must be >= 1");
    std::vector<ohx::ShardIn> in;
    for (int v = 0; v < vshards; ++v) {
      const std::uint64_t b0 = n * v / vshards, b1 = n * (v + 1) / vshards;
      in.push_back({d_xy + 2 * b0, b1 - b0, index_base + b0, h_labels ? h_labels + b0 : nullptr,
                    nullptr});
    }
    *h = 0;
    ohx::RankOut o;
    ohx::run_local(*mg, [&](std::size_t) {
      o = ohx::run_rank(*mg, mg->ranks[0], in, 0, ohx::caller_sink(h_hull, cap, h));
    });
    if (info) *info = o.info;
  });
}

int ohx_mg_heaphull_device(ohx_mg* mg, int nshards, const double* const* d_xy, const uint64_t* n,
                           uint8_t* h_labels, double* h_hull, uint64_t cap, uint64_t* h,
                           ohx_mg_info* info) {
  return guard([&] {
    ohx::usable(mg);
    std::lock_guard<std::mutex> g(mg->mu);
    if (!mg->single_process)
      throw std::invalid_argument("mg: ohx_mg_heaphull_device needs ohx_mg_init_all");
    const int L = static_cast<int>(mg->ranks.size());
    if (nshards < L || nshards % L != 0)
      throw std::invalid_argument("mg: nshards must be a positive multiple of the devices");
    const int k = nshards / L;
    std::vector<std::uint64_t> base(nshards + 1, 0);
    for (int j = 0; j < nshards; ++j) base[j + 1] = base[j] + n[j];
    if (base[nshards] == 0) throw std::invalid_argument("heaphull: empty point set");
    *h = 0;
    std::vector<ohx::RankOut> outs(L);
    ohx::run_local(*mg, [&](std::size_t r) {
      std::vector<ohx::ShardIn> in;
      for (int v = 0; v < k; ++v) {
        const int j = static_cast<int>(r) * k + v;
        in.push_back({d_xy[j], n[j], base[j], h_labels ? h_labels + base[j] : nullptr, nullptr});
      }
      outs[r] = ohx::run_rank(*mg, mg->ranks[r], in, 0, ohx::caller_sink(h_hull, cap, h));
    });
    if (info) *info = outs[0].info;
  });
}

int ohx_mg_heaphull(ohx_mg* mg, const double* h_xy, uint64_t n, int vshards, uint8_t* h_labels,
                    double* h_hull, uint64_t cap, uint64_t* h, ohx_mg_info* info) {
  return guard([&] {
    ohx::usable(mg);
    std::lock_guard<std::mutex> g(mg->mu);
    *h = 0;
    ohx::mg_heaphull_host(mg, h_xy, n, vshards, h_labels, ohx::caller_sink(h_hull, cap, h), info);
  });
}

}  // extern "C"
