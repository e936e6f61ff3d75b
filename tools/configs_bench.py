"""Every BASELINE.json config through the device pipeline and the host API,
next to the reference CPU heaphull_run (oracle/_ref) on the same points.

  python tools/configs_bench.py [--reps 3] [--ref-max 1e8]

Per config: device-resident pipeline (ohx_heaphull_device: filter_ms up to
the queues, hull_ms = survivor D2H + host hull), the host-buffer API
(ohx_heaphull on pinned memory, H2D included), the run info (fused,
candidates, survivors, hull size) and the reference CPU time (all cores).
One JSON line per config."""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2209_12310_b200 as P  # noqa: E402
from oracle import Reference  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--ref-max", type=float, default=1e8)
ap.add_argument("--only", default="")
a = ap.parse_args()

CONFIGS = [("C1 normal 1e6", "normal", 1_000_000, 7, 0.0),
           ("C2 square 1e8", "square", 100_000_000, 7, 0.0),
           ("C3 normal 1e9", "normal", 1_000_000_000, 7, 0.0),
           ("C4 circle 1e8", "circle", 100_000_000, 7, 0.0),
           ("disk 1e8", "disk", 100_000_000, 7, 0.0),
           ("circle+2% 1e7", "circle", 10_000_000, 7, 2.0)]
ctx = P.Context(0)
ref = Reference() if Reference.available() else None
for name, dist, n, seed, distort in CONFIGS:
    if a.only and a.only not in name:
        continue
    host = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
    hp = host.numpy()
    P.check(P.lib.ohx_generate(P.DISTS[dist], n, seed, distort, hp.ctypes.data_as(P._dp), 0))
    d = host.cuda()
    dev_ms, filt_ms, hull_ms = [], [], []
    hull = None
    for r in range(a.reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hull, t = ctx.heaphull_device(d, n)
        t1 = time.perf_counter()
        if r:
            dev_ms.append((t1 - t0) * 1e3)
            filt_ms.append(t["filter_ms"])
            hull_ms.append(t["hull_ms"])
    info = ctx.last_run()
    del d
    torch.cuda.empty_cache()
    out = np.empty((len(hull) + 64, 2))
    h = P.C.c_uint64(0)
    api_ms = []
    for r in range(a.reps + 1):
        t0 = time.perf_counter()
        P.check(P.lib.ohx_heaphull(hp.ctypes.data_as(P._dp), n, out.ctypes.data_as(P._dp),
                                   len(out), P.C.byref(h), None))
        if r:
            api_ms.append((time.perf_counter() - t0) * 1e3)
    assert np.array_equal(out[: h.value], hull)
    line = {"config": name, "n": n, "fused": info["fused"], "fuse_state": info["fuse_state"],
            "candidates": info["candidates"], "survivors": sum(info["counts"]), "h": len(hull),
            "device_ms": statistics.median(dev_ms), "filter_ms": statistics.median(filt_ms),
            "hull_ms": statistics.median(hull_ms), "host_api_ms": statistics.median(api_ms),
            "device_gpts": n / statistics.median(dev_ms) / 1e6,
            "host_api_gpts": n / statistics.median(api_ms) / 1e6}
    if ref is not None and n <= a.ref_max:
        eng = ref.engine(os.cpu_count() or 1, 32)
        ts = []
        for r in range(2):
            t0 = time.perf_counter()
            eng.heaphull(hp)
            ts.append((time.perf_counter() - t0) * 1e3)
        line["ref_ms"] = min(ts)
        line["ref_cores"] = os.cpu_count()
        line["speedup_host_api_vs_ref"] = line["ref_ms"] / line["host_api_ms"]
        # parity on the same bytes: the reference's hull, labels and
        # extremes against the device pipeline's hull, queues and extremes
        ref_hull, ref_labels, _ = ref.heaphull_run(hp, os.cpu_count() or 1, 32)
        d = host.cuda()
        hull_dev, _ = ctx.heaphull_device(d, n)
        info = ctx.last_run()
        q_ok = all(np.array_equal(ctx.queue(q + 1, info["counts"][q])[0],
                                  np.flatnonzero(ref_labels == q + 1)) for q in range(4))
        line["parity"] = {"hull_equal": bool(np.array_equal(hull_dev, ref_hull)),
                          "queues_equal": bool(q_ok),
                          "extremes_equal": [int(v) for v in ref.find_extremes(hp, os.cpu_count() or 1)]
                          == [int(v) for v in P.find_extremes(hp)],
                          "h_ref": int(len(ref_hull))}
        del d, ref_labels
        torch.cuda.empty_cache()
    print(json.dumps(line), flush=True)
