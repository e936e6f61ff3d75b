#!/usr/bin/env python
"""Benchmark of the B200 heaphull filter (arXiv 2209.12310).

    python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference]
    (N > 1: launched by torch.distributed.run, one rank per GPU, NCCL)

Workload (the job's corpus is always ONE reference corpus,
generate({dist, points_total, seed}), so every number is checkable against
the reference on the same bytes):
  N = 1  BASELINE.json configs[2]: normal, 1e9 points, seed 7 (16 GB of AoS
         binary64 points, larger than the 126 MB L2: no flush needed).
  N > 1  BASELINE.json configs[4]: normal, 4e9 points in total, seed 7,
         strong scaling; rank r holds the contiguous slice
         [r*4e9/N, (r+1)*4e9/N) of that corpus, generated in place
         (ohx_generate_range).  --weak: 1e9 points per GPU instead.

A step is one full hull of the whole job's points:
  value  -- inputs resident in HBM: the fused single pass (sample ->
            provisional region -> KF filter pass -> K1 over the candidates)
            or, when it does not apply, K1; certificate -> (K1b) ->
            octagon -> K2 (candidates only when fused) -> survivors D2H ->
            host hull, Gpoints/s over all ranks,
  e2e    -- the same through the reference-facing API with host buffers:
            N = 1 the C ABI call ohx_heaphull (octohull::heaphull) on
            pinned host points, N > 1 each rank's pinned slice uploaded
            inside the step; e2e.roofline is the PCIe bound (the measured
            raw pinned H2D bandwidth of the same buffer).
Steps are timed with CUDA events after a barrier + synchronize on both
sides, max over ranks.  roofline: the dominant kernel's algorithmic bytes
per launch (16 B per point read; the fused KF pass also writes 4 B per
candidate index) over its CUDA-event duration on the launching stream,
against the measured HBM copy bandwidth in MEASURED_PEAKS.json.
cpu_baseline: the reference library itself (oracle/_ref, compiled from the
reference sources) timed on the host cores on the bench's own points (the
full per-GPU workload); the same leg checks the device results against it
(parity).  distributions: BASELINE configs[1] and configs[3] (square and
circle 1e8), timed device-resident and checked against the reference.

`--impl reference` times that reference CPU implementation on the same
metric and config (rank 0 only; the points come from the reference's own
generator, nothing of this repository's library is loaded), each step one
heaphull_run over the first --cpu-sample points of the job's corpus
(default: the whole corpus up to 1e9 points).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gpoints/s end-to-end hull and filter HBM GB/s vs peak at 1/2/4/8 B200"
UNIT = "Gpoints/s"
STRONG_TOTAL = 4_000_000_000  # BASELINE configs[4]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--dist", default="normal")
    ap.add_argument("--points", "--n", dest="n", type=float, default=1e9,
                    help="points per GPU at N = 1 (and with --weak)")
    ap.add_argument("--points-total", type=float, default=0,
                    help="points of the whole job at N > 1 (default 4e9: BASELINE configs[4])")
    ap.add_argument("--weak", action="store_true", help="N > 1: --points per GPU")
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--cpu-sample", type=float, default=0,
                    help="points of the CPU reference's sample (0: the corpus, up to 1e9)")
    ap.add_argument("--mg-vshards", type=int, default=1,
                    help="shards per rank through the native multi-GPU layer (N = 1: > 1 "
                         "routes the step through ohx_mg with that many shards on one GPU)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-dists", action="store_true",
                    help="skip the per-distribution lines (square / circle 1e8)")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the full-size parity checks against the reference library")
    return ap.parse_args()


def job(a, world: int) -> dict:
    """The job's corpus and how it is split over the ranks."""
    if world == 1:
        total, scaling = int(a.n), "weak"
    elif a.weak:
        total, scaling = world * int(a.n), "weak"
    else:
        total, scaling = int(a.points_total) or STRONG_TOTAL, "strong"
    return {"total": total, "scaling": scaling, "dist": a.dist, "seed": a.seed}


def shard_of(total: int, world: int, rank: int):
    """Rank r's contiguous slice [floor(r T / N), floor((r+1) T / N))."""
    b0 = total * rank // world
    return b0, total * (rank + 1) // world - b0


def config(a, world: int) -> dict:
    """The line's `config` -- identical for both arms."""
    j = job(a, world)
    per = j["total"] // world
    if world == 1 and j["dist"] == "normal" and j["total"] == 1_000_000_000 and j["seed"] == 7:
        name = "BASELINE configs[2]: normal-distribution 2D points N=1e9 on 1 B200"
    elif world > 1 and j["dist"] == "normal" and j["total"] == STRONG_TOTAL and j["seed"] == 7:
        name = f"BASELINE configs[4]: normal-distribution 4e9 points sharded across {world} B200"
    else:
        name = (f"{j['dist']}-distribution 2D points, {j['total']:.3g} in total on {world} B200"
                f" ({j['scaling']} scaling)")
    return {"workload": name, "dist": j["dist"], "seed": j["seed"], "points_total": j["total"],
            "points_per_gpu": per, "scaling": j["scaling"],
            "corpus": f"generate({{{j['dist']}, {j['total']}, {j['seed']}}}), rank r holds "
                      f"index range [r*T/N, (r+1)*T/N)",
            "parallelism": f"index-range shards x{world}",
            "l2": f"inputs {per * 16 / 1e9:.3g} GB/GPU vs 126 MB L2"
                  + (" (larger: no flush needed)" if per * 16 > 4 * 126e6
                     else " (L2-resident: not a roofline point)")}


# ---------------------------------------------------------------- clocks --
class ClockSampler:
    """SM clock + clock-event reasons sampled DURING the timed region.

    NVML is polled every 5 ms from a thread (the device-resident timed
    region of a 1e9-point run lasts only ~60 ms, too short for
    `nvidia-smi -lms 200`); `nvidia-smi` is the fallback."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40,
               "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4,
               "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period, self.rows = index, period_s, []
        self._stop = threading.Event()
        self.nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.nvml = (pynvml, h)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None
        self.t = threading.Thread(target=self._poll, daemon=True)
        self.t.start()
        return self

    def _poll(self):
        while not self._stop.is_set():
            try:
                if self.nvml:
                    pynvml, h = self.nvml
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append((sm, self.max_mhz, rs))
                else:
                    out = subprocess.run(
                        ["nvidia-smi", "-i", str(self.index),
                         "--query-gpu=clocks.sm,clocks.max.sm", "--format=csv,noheader,nounits"],
                        capture_output=True, text=True, timeout=5).stdout.split(",")
                    self.rows.append((float(out[0]), float(out[1]), 0))
            except Exception:
                pass
            self._stop.wait(self.period)

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [r[0] for r in self.rows]
        reasons = sorted({k for r in self.rows for k, bit in self.REASONS.items() if r[2] & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.rows[0][1],
                "reasons": reasons, "samples": len(self.rows),
                "source": "nvml" if self.nvml else "nvidia-smi"}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """dram bytes per point of K1/K2 from the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


# ------------------------------------------------------- CPU reference ----
def cpu_reference(pts, reps: int):
    """The reference heaphull_run (oracle/_ref) on all host cores over `pts`
    (the C restatement, single-threaded, where the reference was never
    built); -> {kind, cores, times}."""
    from oracle import Oracle, Reference

    cores = os.cpu_count() or 1
    if Reference.available():
        eng = Reference().engine(cores, 32)
        kind, run = "reference", eng.heaphull
    else:
        o = Oracle()
        kind, cores = "port", 1
        run = o.heaphull
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        run(pts)
        times.append(time.perf_counter() - t0)
    return {"kind": kind, "cores": cores, "times": times}


def reference_parity(ref, pts, ctx, hull_dev, ext_dev, counts=None) -> dict:
    """The device results of the last call on ctx (hull, extremes, queues)
    against the reference's own heaphull_run / find_extremes on the same
    points (outside every timed region; the reference is the checker).
    ctx None (a multi-shard call): the queue lengths `counts` are compared
    instead of the queues themselves."""
    import numpy as np

    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    ref_hull, ref_labels, _ = ref.heaphull_run(pts, cores, 32)
    ref_ext = ref.find_extremes(pts, cores, 32)
    ref_s = time.perf_counter() - t0
    queues_ok = True
    if ctx is not None:
        info = ctx.last_run()
        for q in range(4):
            want = np.flatnonzero(ref_labels == q + 1)
            got = ctx.queue(q + 1, info["counts"][q])[0]
            queues_ok &= bool(np.array_equal(got, want))
    else:
        queues_ok = [int((ref_labels == q + 1).sum()) for q in range(4)] == list(counts)
    out = {"checked_against": f"reference heaphull_run + find_extremes (oracle/_ref, {cores} "
                              f"workers) on the same {len(pts)} points",
           "hull_equal": bool(np.array_equal(hull_dev, ref_hull)),
           "extremes_equal": [int(v) for v in ext_dev] == [int(v) for v in ref_ext],
           "queues_equal": queues_ok,
           "survivors": int((ref_labels != 0).sum()), "h": int(len(ref_hull)),
           "reference_s": ref_s}
    del ref_labels
    return out


def run_reference_arm(a):
    """Rank 0 only: the reference's heaphull_run on the first `sample`
    points of the job's corpus, from the reference's own generator (the
    first k points of generate({dist, T, seed}) are generate({dist, k,
    seed})).  Nothing of this repository's library is loaded here."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from oracle import Oracle, Reference

    j = job(a, world)
    n = min(j["total"], int(a.cpu_sample) or 1_000_000_000)
    t0 = time.perf_counter()
    gen = Reference() if Reference.available() else Oracle()
    pts = gen.generate(j["dist"], n, j["seed"])
    gen_s = time.perf_counter() - t0
    r = cpu_reference(pts, a.warmup + a.steps)
    timed = r["times"][a.warmup:]
    ms = 1e3 * sum(timed) / len(timed)
    value = n / (ms * 1e-3) / 1e9
    sample = (f"{j['dist']} n={n} seed={j['seed']} ("
              + ("the whole corpus" if n == j["total"]
                 else f"the first {n} points of the {j['total']}-point corpus")
              + f"), full heaphull_run, ReduceEngine({{32, {r['cores']}}})")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": j["scaling"], "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic: the reference's own generator ({j['dist']}, seed {j['seed']})",
        "config": config(a, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "generate_s": gen_s,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- B200 arm --
def h2d_bandwidth(host, dev) -> float:
    """Raw pinned H2D GB/s of host -> dev (the e2e step's PCIe bound),
    best of 3 copies timed with CUDA events."""
    import torch

    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dev.copy_(host, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = max(best, host.numel() * host.element_size() / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return best


def distributions_leg(a, P, ctx, dev, start, stop, peak, check_parity):
    """BASELINE configs[1] (uniform square 1e8, pure streaming) and
    configs[3] (circumference 1e8, nothing filtered: compaction- and
    hull-bound), device-resident, 5 timed steps each, then checked against
    the reference's heaphull_run on the same points."""
    import numpy as np
    import torch

    out = []
    for dname, dn in (("square", 100_000_000), ("circle", 100_000_000)):
        hbuf = torch.empty((dn, 2), dtype=torch.float64, pin_memory=True)
        hp = hbuf.numpy()
        P.check(P.lib.ohx_generate(P.DISTS[dname], dn, a.seed, 0.0, hp.ctypes.data_as(P._dp), 0))
        dd = hbuf.to(dev)
        # the hull into one reused pinned host buffer (a 96.8M-vertex circle
        # hull is 1.55 GB: one direct DMA, no staging or first-touch faults)
        hout = torch.empty((dn + 8, 2), dtype=torch.float64, pin_memory=True)
        for _ in range(2):
            ctx.heaphull_device(dd, dn, out=hout)
        torch.cuda.synchronize()
        ctx.kernel_ms_sum(reset=True)
        start.record()
        for _ in range(5):
            hull, _ = ctx.heaphull_device(dd, dn, out=hout)
        stop.record()
        torch.cuda.synchronize()
        dms = start.elapsed_time(stop) / 5
        ksum = ctx.kernel_ms_sum()
        info = ctx.last_run()
        stream_ms = ksum["k1"][0] / max(1, ksum["k1"][1])
        k_bytes = 16 * dn + (4 * info["candidates"] if info["fused"] else 0)
        row = {"dist": dname, "points": dn, "seed": a.seed, "value": dn / (dms * 1e-3) / 1e9,
               "unit": UNIT, "ms_per_step": dms, "api": "ohx_heaphull_device (hull to a reused "
                                                        "pinned host buffer)",
               "fused": info["fused"],
               "survivors": sum(info["counts"]), "h": int(len(hull)),
               "streaming_kernel": "kf_filter" if info["fused"] else "k1_extremes",
               "streaming_ms": stream_ms,
               "streaming_gbs": k_bytes / (stream_ms * 1e-3) / 1e9,
               "streaming_frac": k_bytes / (stream_ms * 1e-3) / 1e9 / peak,
               "k2_ms": ksum["k2"][0] / max(1, ksum["k2"][1])}
        # the same pipeline with the hull left in device memory
        # (ohx_heaphull_device_out): no PCIe copy of a 96.8M-vertex hull
        dbuf = torch.empty((dn + 8, 2), dtype=torch.float64, device=dev)  # reused output
        dh, _ = ctx.heaphull_device(dd, dn, out=dbuf)
        torch.cuda.synchronize()
        start.record()
        for _ in range(5):
            dh, _ = ctx.heaphull_device(dd, dn, out=dbuf)
        stop.record()
        torch.cuda.synchronize()
        dms_dev = start.elapsed_time(stop) / 5
        row["hull_on_device"] = {"value": dn / (dms_dev * 1e-3) / 1e9, "unit": UNIT,
                                 "ms_per_step": dms_dev, "api": "ohx_heaphull_device_out",
                                 "hull_path": ctx.last_run()["hull_path"],
                                 "hull_equal": bool(np.array_equal(dh.cpu().numpy(), hull))}
        del dh, dbuf
        if check_parity:
            from oracle import Reference
            if Reference.available():
                rec = ctx.extremes(dd, dn)  # the library's find_extremes on the device points
                e, mask = P.resolve_extremes(rec)
                if mask:
                    e = P.apply_corners(e, ctx.corners_exact(dd, dn, (rec.x[0], rec.y[1],
                                                                      rec.x[2], rec.y[3])))
                hull, _ = ctx.heaphull_device(dd, dn)  # the queues of this very call are checked
                row["parity"] = reference_parity(Reference(), hp, ctx, hull, list(e.ext))
        out.append(row)
        del dd, hbuf, hp, hout
        torch.cuda.empty_cache()
    return out


class Runner:
    """One step of the job on this rank, in one of three shapes:
      single  -- N = 1: ctx.heaphull_device (the device pipeline)
      mg      -- the native multi-GPU layer (ohx_mg_*, NCCL): N > 1 over
                 NCCL, or N = 1 with --mg-vshards k (k shards on one GPU)
      sharded -- N > 1 with OHX_BENCH_BACKEND=gloo: sharded.py over gloo
                 (ranks sharing a GPU; a test mode of the multi-rank code)
    first() -> (hull, stats) with stats: counts (this rank), job_counts,
    uncertified, ext, fused; step() -> hull (rank 0) or None."""

    def __init__(self, mode, P, ctx, d, n, base, world, rank, local_dev, xdev, vshards):
        self.mode, self.P, self.d, self.n, self.base = mode, P, d, n, base
        self.world, self.rank, self.xdev, self.vshards = world, rank, xdev, vshards
        self.ctx = ctx
        if mode == "mg":
            import torch
            import torch.distributed as dist
            from paper_2209_12310_b200.mg import MultiGPU, unique_id
            uid = torch.zeros(128, dtype=torch.uint8, device=xdev)
            if rank == 0:
                uid.copy_(torch.frombuffer(bytearray(unique_id()), dtype=torch.uint8))
            if world > 1:
                dist.broadcast(uid, 0)
            self.mg = MultiGPU.init_rank(bytes(uid.cpu().numpy()), world, rank, local_dev)
            self.ctx = self.mg.shard_context(0, 0)  # stage times / launches of shard 0
            self.ctxs = [self.mg.shard_context(0, v) for v in range(vshards)]
        elif mode == "sharded":
            from paper_2209_12310_b200.sharded import CudaShard
            self.shard = CudaShard(ctx, d, n, base)

    def launches(self) -> int:
        cs = self.ctxs if self.mode == "mg" else [self.ctx]
        return sum(c.launches for c in cs)

    def step(self, d=None):
        d = self.d if d is None else d
        if self.mode == "single":
            return self.ctx.heaphull_device(d, self.n)[0]
        if self.mode == "mg":
            return self.mg.heaphull_shard(d, self.n, self.base, self.vshards)[0]
        from paper_2209_12310_b200.sharded import CudaShard, sharded_heaphull
        sh = self.shard if d is self.d else CudaShard(self.ctx, d, self.n, self.base)
        return sharded_heaphull(sh, device=self.xdev)

    def first(self):
        import numpy as np
        if self.mode == "mg":
            hull, info = self.mg.heaphull_shard(self.d, self.n, self.base, self.vshards)
            mine = [sum(c.last_run()["counts"][q] for c in self.ctxs) for q in range(4)]
            return hull, {"counts": mine, "job_counts": info["counts"],
                          "uncertified": int(info["corner_pass"]), "ext": info["ext"],
                          "fused": info["fused_shards"] == info["shards"], "mg": info}
        from paper_2209_12310_b200.sharded import sharded_heaphull
        stats = {}
        shard = self.shard if self.mode == "sharded" else \
            __import__("paper_2209_12310_b200.sharded", fromlist=["CudaShard"]).CudaShard(
                self.ctx, self.d, self.n, self.base)
        hull = sharded_heaphull(shard, device=self.xdev, stats=stats)
        stats["job_counts"] = None
        if self.mode == "sharded":  # the job's queue lengths: a sum over ranks
            import torch
            import torch.distributed as dist
            t = torch.tensor(stats["counts"], dtype=torch.int64, device=self.xdev)
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            stats["job_counts"] = [int(v) for v in t.tolist()]
        if self.mode == "single":
            assert np.array_equal(hull, self.step()), "pipeline disagreement"
            stats["job_counts"] = stats["counts"]
        return hull, stats


def run_b200_arm(a):
    import numpy as np  # noqa: F811
    import torch
    import torch.distributed as dist

    import paper_2209_12310_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.gpus != world:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    # OHX_BENCH_BACKEND=gloo: a test mode for the N > 1 code path on a box
    # with fewer GPUs than ranks (ranks share devices, exchanges go through
    # host memory); the measured configuration is always NCCL
    backend = os.environ.get("OHX_BENCH_BACKEND", "nccl")
    local_dev = local % max(1, torch.cuda.device_count()) if backend == "gloo" else local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    xdev = dev if backend == "nccl" else torch.device("cpu")  # collective buffers
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    mode = ("mg" if backend == "nccl" and (world > 1 or a.mg_vshards > 1)
            else "sharded" if world > 1 else "single")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=xdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v: int) -> int:
        if world == 1:
            return int(v)
        t = torch.tensor([int(v)], dtype=torch.int64, device=xdev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return int(t.item())

    j = job(a, world)
    total = j["total"]
    base, n = shard_of(total, world, rank)
    t0 = time.perf_counter()
    try:  # pinned: the e2e step's H2D runs at PCIe speed
        host = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
    except RuntimeError:  # e.g. 8 ranks x 16 GB beyond the host's pinnable memory
        host = torch.empty((n, 2), dtype=torch.float64)
    hp = host.numpy()
    P.generate_range(a.dist, total, base, n, a.seed, out=hp)
    d = host.to(dev)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    ctx0 = P.Context(local_dev)
    run = Runner(mode, P, ctx0, d, n, base, world, rank, local_dev, xdev, max(1, a.mg_vshards))
    ctx = run.ctx  # the (first) shard's context: stage times, last run

    def step_device():
        return run.step()

    # correctness gate on this very workload (single: the pipeline equals the
    # kernel-level path; K1/K2 are oracle-checked in tests) + the run's stats
    hull0, stats = run.first()
    survivors_job = (sum(stats["job_counts"]) if stats["job_counts"] is not None
                     else sum_over_ranks(sum(stats["counts"])))

    # ---------------- device-resident timed region
    for _ in range(a.warmup):
        step_device()
    launches0 = run.launches()
    # per-stage CUDA-event sums, read once after the loop; with several
    # (virtual) shards per rank their stages run one after another on this
    # GPU, so a step's stage time is the sum over the shards' contexts
    kctxs = run.ctxs if mode == "mg" else [ctx]
    for c in kctxs:
        c.kernel_ms_sum(reset=True)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_dev) as clocks:
        barrier()
        start.record()
        for _ in range(a.steps):
            step_device()
        stop.record()
        barrier()
    launches = run.launches() - launches0
    ksums = [c.kernel_ms_sum() for c in kctxs]
    ksum = {k: (sum(ks[k][0] for ks in ksums), ksums[0][k][1]) for k in ksums[0]}
    k1, k2, kc = ([ksum[k][0] / ksum[k][1]] if ksum[k][1] else [-1.0] for k in ("k1", "k2", "kc"))
    last = ctx.last_run()
    runs = [dict(last, fused=last["fused"] and ksum["kc"][1] == a.steps)]
    ms = max_over_ranks(start.elapsed_time(stop) / a.steps)
    value = total / (ms * 1e-3) / 1e9

    # ---------------- e2e through the host-buffer API
    e2e = None
    clocks_e2e_summary = None
    if not a.no_e2e:
        if mode == "single":
            s_local = sum(stats["counts"])
            out = np.empty((n + 8, 2), dtype=np.float64) if n < 10_000_000 else np.empty((s_local + 8 + 64, 2))
            h = P.C.c_uint64(0)

            def step_e2e():
                P.check(P.lib.ohx_heaphull(hp.ctypes.data_as(P._dp), n, out.ctypes.data_as(P._dp),
                                           len(out), P.C.byref(h), None))
            api = "ohx_heaphull (C ABI) on {} host points"
        else:
            d2 = torch.empty_like(d)

            def step_e2e():
                d2.copy_(host, non_blocking=True)
                torch.cuda.current_stream().synchronize()
                run.step(d2)
            api = ("ohx_mg_heaphull_shard (C ABI, NCCL) after each rank's H2D of its {} slice"
                   if mode == "mg" else "sharded_heaphull (gloo) after each rank's H2D of its {} slice")
        for _ in range(a.warmup):
            step_e2e()
        with ClockSampler(local_dev) as clocks_e2e:
            barrier()
            start.record()
            for _ in range(a.steps):
                step_e2e()
            stop.record()
            barrier()
        ms_e2e = max_over_ranks(start.elapsed_time(stop) / a.steps)
        # the bound of this step: the raw pinned H2D of the same buffer
        h2d = h2d_bandwidth(host, d if mode == "single" else d2) if host.is_pinned() else None
        h2d = max_over_ranks(h2d or 0.0) if world > 1 else h2d
        e2e_gbs = total * 16 / (ms_e2e * 1e-3) / 1e9
        if mode == "mg":
            # the layer's read-backs on every rank: the record all-gather
            # (296 B per rank) and the exchange block (16448 B per rank:
            # queue lengths + up to 1024 survivors); survivors over the
            # block go to the root's device and come back once
            per_rank = max_over_ranks(float(sum(stats["counts"])))
            d2h = world * world * (296 + 16448) + (0 if per_rank <= 1024 else survivors_job * 16)
        else:
            # survivors' coordinates (16 B each) + the small records
            d2h = survivors_job * 16 + world * 2 * 320
        e2e = {"value": total / (ms_e2e * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": ms_e2e,
               "h2d_bytes_per_step": total * 16,
               "d2h_bytes_per_step": d2h,
               "api": api.format("pinned" if host.is_pinned() else "pageable"),
               "roofline": {"bound": "pcie", "achieved": e2e_gbs, "unit": "GB/s",
                            "peak": h2d * world if (h2d and world > 1) else h2d,
                            "frac": e2e_gbs / (h2d * world) if h2d else None,
                            "peak_source": "raw pinned H2D of the same buffer, measured in this "
                                           "run (best of 3, CUDA events)"
                                           + (" x ranks (one PCIe link each)" if world > 1 else "")}}
        clocks_e2e_summary = clocks_e2e.summary()

    # ---------------- roofline of the dominant kernel
    # algorithmic bytes per launch: every point read once by the
    # streaming pass (16 B); fused, KF also writes its candidates' indices
    # (idx B each) and the candidate stage / K2 touch only the candidates
    peak, peak_src = measured_peak()
    s_local = sum(stats["counts"])
    idx_b = 4 if n < 2**32 else 8
    fused = bool(runs) and all(r["fused"] for r in runs)
    cand = runs[-1]["candidates"] if runs else 0
    k1_ms, k2_ms = statistics.mean(k1), statistics.mean(k2)
    if fused:
        kern = {
            "kf_filter": {"ms": k1_ms, "bytes": 16 * n + idx_b * cand,
                          "note": "fused pass: region test + candidate append"},
            "candidate_stage": {"ms": statistics.mean(kc),
                                "bytes": cand * (idx_b * 2 + 16 * 2 + 16),
                                "note": "ordered gather + K1 over the candidates (+ host sync)"},
            "k2_gather": {"ms": k2_ms, "bytes": cand * (idx_b + 16) + (idx_b + 16) * s_local,
                          "note": "K2 on the candidates only (one launch: survivors' indices "
                                  "and coordinates straight into the queues)"},
        }
    else:
        kern = {
            "k1_extremes": {"ms": k1_ms, "bytes": 16 * n},
            "k2_filter_compact": {"ms": k2_ms, "bytes": 16 * n + idx_b * s_local},
        }
    for v in kern.values():
        v["gbs"] = v["bytes"] / (v["ms"] * 1e-3) / 1e9
        v["frac"] = v["gbs"] / peak
    dom = max(kern, key=lambda k: kern[k]["ms"])
    traffic, traffic_src = None, None
    tr = ncu_traffic()
    if tr and dom in tr:
        traffic = tr[dom]["dram_bytes_per_point"] * n
        traffic_src = (f"not measured in this run: dram__bytes_read.sum + dram__bytes_write.sum "
                       f"per point from the committed ncu --set full capture "
                       f"({tr.get('source', 'profiles/ncu_traffic.json')}) x {n} points")
    roofline = {"bound": "hbm", "kernel": dom, "achieved": kern[dom]["gbs"], "peak": peak,
                "unit": "GB/s", "frac": kern[dom]["gbs"] / peak, "traffic": traffic,
                "traffic_source": traffic_src, "peak_source": peak_src,
                "algorithmic_bytes": kern[dom]["bytes"],
                "kernels": kern,
                "pipeline": "fused single pass (KF)" if fused else "two passes (K1, K2)",
                "candidates": cand}

    # ---------------- CPU baseline (rank 0, N = 1) + full-size parity check
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not a.no_cpu:
        ns = min(n, int(a.cpu_sample) or n)
        pts = hp[:ns]
        r = cpu_reference(pts, 2)
        t = statistics.mean(r["times"])
        cpu = {"value": ns / t / 1e9, "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
               "sample": f"{a.dist} n={ns} seed={a.seed}"
                         f"{' (the bench workload itself)' if ns == n else ' (the first points of the workload)'}"
                         f", reference heaphull_run x2 (ReduceEngine chunk 32, {r['cores']} workers), "
                         f"mean {t:.3f} s"}
        if not a.no_parity and r["kind"] == "reference" and ns == n:
            from oracle import Reference
            hull_dev = step_device()
            parity = reference_parity(Reference(), hp, ctx if mode == "single" else None,
                                      hull_dev, stats["ext"], stats["job_counts"])
    if world > 1 and not a.no_parity:
        # N > 1: the job's hull, extremes and queue lengths (one multi-GPU
        # step, collective) against the reference on the WHOLE corpus, which
        # rank 0 regenerates on its host cores (configs[4]: 4e9 points,
        # 64 GB, about a minute); the other ranks wait at the barrier
        hull_dev = step_device()
        if rank == 0:
            need = 16 * total * 2.2  # the points + the reference's labels and copies
            have = os.sysconf("SC_PHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
            from oracle import Reference
            if not Reference.available():
                parity = {"skipped": "reference library not built (oracle/_ref)"}
            elif need > have * 0.6:
                parity = {"skipped": f"host RAM {have / 2**30:.0f} GiB < the corpus + checker "
                                     f"({need / 2**30:.0f} GiB at 60 %)"}
            else:
                full = P.generate(a.dist, total, a.seed)
                parity = reference_parity(Reference(), full, None, hull_dev, stats["ext"],
                                          stats["job_counts"])
                parity["corpus"] = f"generate({{{a.dist}, {total}, {a.seed}}}) on rank 0"
                del full
        barrier()

    # ---------------- the other distributions (rank 0, N = 1)
    dists = None
    if rank == 0 and world == 1 and not a.no_dists:
        del d
        torch.cuda.empty_cache()
        dists = distributions_leg(a, P, ctx0, dev, start, stop, peak, not a.no_parity)

    if rank == 0:
        clk = clocks.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": j["scaling"], "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic: generate({a.dist}, {total}, seed {a.seed}) -- bit-identical to "
                    f"the reference generator, each rank generating its own slice",
            "config": config(a, world),
            "run": {"survivors": survivors_job, "survivors_rank0": stats["counts"],
                    "corner_certificate": "pass" if not stats["uncertified"]
                    else f"fallback mask {stats['uncertified']}", "fused": stats.get("fused"),
                    "path": {"single": "ohx_heaphull_device (one device pipeline)",
                             "mg": f"ohx_mg_heaphull_shard (NCCL, {world} rank(s), "
                                   f"{max(1, a.mg_vshards)} shard(s) per rank)",
                             "sharded": "sharded.py over gloo (test mode)"}[mode]},
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "parity": parity,
            "distributions": dists, "clocks": clk,
            "clocks_e2e": clocks_e2e_summary, "gpu_launches": launches,
            "setup_s": setup_s,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        run_reference_arm(a)
    else:
        run_b200_arm(a)


if __name__ == "__main__":
    main()
