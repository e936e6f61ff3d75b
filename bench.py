#!/usr/bin/env python
"""Benchmark of the B200 heaphull filter (arXiv 2209.12310).

    python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference]
    (N > 1: launched by torch.distributed.run, one rank per GPU, NCCL)

Workload: BASELINE.json configs[2] -- normal-distribution 2D points,
N = 1e9 per GPU (16 GB of AoS binary64 points, larger than the 126 MB L2,
so no flush is needed), seed 7 + rank.  Weak scaling: every rank owns a
1e9-point shard of the global index range; the shards are filtered
independently and only the ~300 B extremes records and the survivors
cross GPUs (sharded.py).

A step is one full hull of the whole job's points:
  value  -- inputs resident in HBM: the fused single pass (sample ->
            provisional region -> KF filter pass -> K1 over the candidates)
            or, when it does not apply, K1; certificate -> (K1b) ->
            octagon -> K2 (candidates only when fused) -> survivors D2H ->
            host hull, Gpoints/s over all ranks,
  e2e    -- the same through the reference-facing API with host buffers:
            N = 1 the C ABI call ohx_heaphull (octohull::heaphull) on
            pinned host points, N > 1 the sharded API with each rank's
            pinned shard uploaded inside the step.
Steps are timed with CUDA events after a barrier + synchronize on both
sides, max over ranks.  roofline: the dominant kernel's algorithmic bytes
per launch (16 B per point read; the fused KF pass also writes 4 B per
candidate index) over its CUDA-event duration on the launching stream,
against the measured HBM copy bandwidth in MEASURED_PEAKS.json.
cpu_baseline: the reference library itself (oracle/_ref, compiled from the reference sources) timed on
the host cores on the bench's own points (the full per-GPU workload).

`--impl reference` times that reference CPU implementation on the same
metric (rank 0 only), each step one heaphull_run over the full per-GPU
workload (--cpu-sample bounds it).
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
WORKLOAD = "normal-distribution 2D points, 1e9 per GPU (BASELINE configs[2]; C5 shape at N>1)"


def workload(dist: str, n: int) -> str:
    """The workload name: BASELINE configs[2] at its defaults, else what ran."""
    if dist == "normal" and n == 1_000_000_000:
        return WORKLOAD
    return f"{dist}-distribution 2D points, {n:.3g} per GPU (BASELINE configs[2] shape)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--dist", default="normal")
    ap.add_argument("--points", "--n", dest="n", type=float, default=1e9, help="points per GPU")
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--cpu-sample", type=float, default=0,
                    help="points of the CPU reference's sample (0: the full per-GPU workload)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-dists", action="store_true",
                    help="skip the per-distribution lines (square / circle 1e8)")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the full-size parity gate against the reference library")
    return ap.parse_args()


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
def cpu_reference(n_sample: int, reps: int, seed: int, dist: str, pts=None):
    """The reference heaphull_run (oracle/_ref) on all host cores, on `pts`
    (the bench's own points) or a generated sample of n_sample points."""
    import numpy as np

    import paper_2209_12310_b200 as P
    from oracle import Oracle, Reference

    if pts is None:
        pts = P.generate(dist, n_sample, seed)
    n_sample = len(pts)
    cores = os.cpu_count() or 1
    if Reference.available():
        eng = Reference().engine(cores, 32)
        kind = "reference"
        run = eng.heaphull
    else:  # the C restatement, single-threaded
        o = Oracle()
        kind, cores = "port", 1

        def run(a):
            t0 = time.perf_counter()
            h = o.heaphull(a)
            return len(h), {"total_ms": (time.perf_counter() - t0) * 1e3}
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        run(pts)
        times.append(time.perf_counter() - t0)
    del np
    return {"kind": kind, "cores": cores, "times": times, "n": n_sample}


def run_reference_arm(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = int(a.cpu_sample) or int(a.n)
    r = cpu_reference(n, a.warmup + a.steps, a.seed, a.dist)
    timed = r["times"][a.warmup:]
    ms = 1e3 * sum(timed) / len(timed)
    value = n / (ms * 1e-3) / 1e9
    sample = (f"{a.dist} n={n} seed={a.seed} ("
              + ("the full per-GPU workload" if n == int(a.n)
                 else f"bounded sample of the {workload(a.dist, int(a.n))} workload")
              + "), full heaphull_run")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator, seed 7)",
        "config": {"workload": workload(a.dist, int(a.n)), "dist": a.dist, "sample_points": n,
                   "parallelism": f"ReduceEngine({{32, {r['cores']}}}) host lanes"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- B200 arm --
def run_b200_arm(a):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2209_12310_b200 as P
    from paper_2209_12310_b200.sharded import CudaShard, sharded_heaphull

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

    n = int(a.n)
    base = rank * n
    t0 = time.perf_counter()
    try:  # pinned: the e2e step's H2D runs at PCIe speed
        host = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
    except RuntimeError:  # e.g. 8 ranks x 16 GB beyond the host's pinnable memory
        host = torch.empty((n, 2), dtype=torch.float64)
    hp = host.numpy()
    P.check(P.lib.ohx_generate(P.DISTS[a.dist], n, a.seed + rank, 0.0,
                               hp.ctypes.data_as(P._dp), 0))
    d = host.to(dev)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    ctx = P.Context(local_dev)
    shard = CudaShard(ctx, d, n, base)

    def step_device(stats=None):
        if world == 1:
            hull, _ = ctx.heaphull_device(d, n)
            return hull
        return sharded_heaphull(shard, device=xdev, stats=stats)

    # correctness gate on this very workload: the sharded / single pipeline
    # must equal the kernel-level path (and K1/K2 are oracle-checked in tests)
    stats = {}
    hull0 = sharded_heaphull(shard, device=xdev, stats=stats)
    if rank == 0 and world == 1:
        hull1 = step_device()
        assert np.array_equal(hull0, hull1), "pipeline disagreement"

    # ---------------- device-resident timed region
    for _ in range(a.warmup):
        step_device()
    launches0 = ctx.launches
    ctx.kernel_ms_sum(reset=True)  # per-stage CUDA-event sums, read once after the loop
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_dev) as clocks:
        barrier()
        start.record()
        for _ in range(a.steps):
            step_device()
        stop.record()
        barrier()
    launches = ctx.launches - launches0
    ksum = ctx.kernel_ms_sum()
    k1, k2, kc = ([ksum[k][0] / ksum[k][1]] if ksum[k][1] else [-1.0] for k in ("k1", "k2", "kc"))
    last = ctx.last_run()
    runs = [dict(last, fused=last["fused"] and ksum["kc"][1] == a.steps)]
    ms = max_over_ranks(start.elapsed_time(stop) / a.steps)
    value = world * n / (ms * 1e-3) / 1e9

    # ---------------- e2e through the host-buffer API
    e2e = None
    if not a.no_e2e:
        s_local = sum(stats["counts"])
        if world == 1:
            out = np.empty((n + 8, 2), dtype=np.float64) if n < 10_000_000 else np.empty((s_local + 8 + 64, 2))
            h = P.C.c_uint64(0)

            def step_e2e():
                P.check(P.lib.ohx_heaphull(hp.ctypes.data_as(P._dp), n, out.ctypes.data_as(P._dp),
                                           len(out), P.C.byref(h), None))
        else:
            d2 = torch.empty_like(d)

            def step_e2e():
                d2.copy_(host, non_blocking=True)
                torch.cuda.current_stream().synchronize()
                sharded_heaphull(CudaShard(ctx, d2, n, base), device=xdev)
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
        e2e = {"value": world * n / (ms_e2e * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": ms_e2e,
               "h2d_bytes_per_step": world * n * 16,
               "d2h_bytes_per_step": sum(stats["counts"]) * 16 * world + 2 * 320,
               "api": ("ohx_heaphull (C ABI) on {} host points" if world == 1
                       else "sharded_heaphull with per-rank {} shard H2D").format(
                           "pinned" if host.is_pinned() else "pageable")}
        clocks_e2e_summary = clocks_e2e.summary()
    else:
        clocks_e2e_summary = None

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
            "k2_gather": {"ms": k2_ms, "bytes": cand * (idx_b + 16) + idx_b * s_local,
                          "note": "K2 on the candidates only"},
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
    traffic = None
    tr = ncu_traffic()
    if tr and dom in tr:
        traffic = tr[dom]["dram_bytes_per_point"] * n
    roofline = {"bound": "hbm", "kernel": dom, "achieved": kern[dom]["gbs"], "peak": peak,
                "unit": "GB/s", "frac": kern[dom]["gbs"] / peak, "traffic": traffic,
                "peak_source": peak_src,
                "algorithmic_bytes": kern[dom]["bytes"],
                "kernels": kern,
                "pipeline": "fused single pass (KF)" if fused else "two passes (K1, K2)",
                "candidates": cand}

    # ---------------- CPU baseline (rank 0, N = 1) + full-size parity check
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not a.no_cpu:
        ns = int(a.cpu_sample)
        r = cpu_reference(ns, 2, a.seed, a.dist, pts=None if ns else hp)
        ns = r["n"]
        t = statistics.mean(r["times"])
        cpu = {"value": ns / t / 1e9, "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
               "sample": f"{a.dist} n={ns} seed={a.seed}"
                         f"{' (the bench workload itself)' if ns == n else ''}, reference "
                         f"heaphull_run x2 (ReduceEngine chunk 32, {r['cores']} workers), "
                         f"mean {t:.3f} s"}
        # the same leg checks the device results against the reference's
        # own heaphull_run / find_extremes on these very points (outside
        # every timed region; the reference is the checker here)
        if not a.no_parity and r["kind"] == "reference" and ns == n:
            from oracle import Reference
            if Reference.available():
                ref = Reference()
                cores = os.cpu_count() or 1
                t0 = time.perf_counter()
                ref_hull, ref_labels, _ = ref.heaphull_run(hp, cores, 32)
                ref_ext = ref.find_extremes(hp, cores, 32)
                ref_s = time.perf_counter() - t0
                hull_dev = step_device()
                info = ctx.last_run()
                queues_ok = True
                for q in range(4):
                    want = np.flatnonzero(ref_labels == q + 1)
                    got = ctx.queue(q + 1, info["counts"][q])[0]
                    queues_ok &= bool(np.array_equal(got, want))
                parity = {"checked_against": f"reference heaphull_run + find_extremes (oracle/_ref, "
                                             f"{cores} workers) on the same {n} points",
                          "hull_equal": bool(np.array_equal(hull_dev, ref_hull)),
                          "extremes_equal": stats["ext"] == [int(v) for v in ref_ext],
                          "queues_equal": queues_ok,
                          "survivors": int((ref_labels != 0).sum()), "h": int(len(ref_hull)),
                          "reference_s": ref_s}
                del ref_labels
            else:
                parity = {"checked_against": None, "why": "oracle/_ref not built"}

    # ---------------- the other distributions (rank 0, N = 1): BASELINE
    # configs[1] (uniform square 1e8, pure streaming) and configs[3]
    # (circumference 1e8, nothing filtered: compaction- and hull-bound),
    # device-resident, 5 timed steps each
    dists = None
    if rank == 0 and world == 1 and not a.no_dists:
        dists = []
        for dname, dn in (("square", 100_000_000), ("circle", 100_000_000)):
            hbuf = torch.empty((dn, 2), dtype=torch.float64, pin_memory=True)
            P.check(P.lib.ohx_generate(P.DISTS[dname], dn, a.seed, 0.0,
                                       hbuf.numpy().ctypes.data_as(P._dp), 0))
            dd = hbuf.to(dev)
            del hbuf
            for _ in range(2):
                ctx.heaphull_device(dd, dn)
            torch.cuda.synchronize()
            start.record()
            kms = []
            for _ in range(5):
                ctx.heaphull_device(dd, dn)
                kms.append(ctx.kernel_ms())
            stop.record()
            torch.cuda.synchronize()
            dms = start.elapsed_time(stop) / 5
            info = ctx.last_run()
            k_ms = statistics.mean(k["k1"] for k in kms)
            k_bytes = 16 * dn + (4 * info["candidates"] if info["fused"] else 0)
            dists.append({"dist": dname, "points": dn, "value": dn / (dms * 1e-3) / 1e9,
                          "unit": UNIT, "ms_per_step": dms, "fused": info["fused"],
                          "survivors": sum(info["counts"]),
                          "streaming_kernel": "kf_filter" if info["fused"] else "k1_extremes",
                          "streaming_gbs": k_bytes / (k_ms * 1e-3) / 1e9,
                          "streaming_frac": k_bytes / (k_ms * 1e-3) / 1e9 / peak})
            del dd
            torch.cuda.empty_cache()

    if rank == 0:
        clk = clocks.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic: reference generator ({a.dist}, seed {a.seed}+rank), bit-identical",
            "config": {"workload": workload(a.dist, n), "dist": a.dist, "points_per_gpu": n,
                       "points_total": world * n, "parallelism": f"index-range shards x{world}",
                       "l2": f"inputs {n * 16 / 1e9:.3g} GB/GPU vs 126 MB L2"
                             + (" (no flush needed)" if n * 16 > 4 * 126e6 else " (L2-resident: not a roofline point)"),
                       "survivors": stats["counts"], "corner_certificate": "pass" if not
                       stats["uncertified"] else f"fallback mask {stats['uncertified']}"},
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
