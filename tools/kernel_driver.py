"""Minimal driver for ncu captures: K1 -> (K1b) -> K2 on device-resident
points, `--reps` times.  Usage (under gpurun):

  ncu --set full --clock-control none --import-source on \
      -k regex:"k1_extremes|k2_filter" -s 2 -c 2 -o gpurun_out/prof \
      python tools/kernel_driver.py --dist normal --n 1e8 --reps 2
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2209_12310_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dist", default="normal")
ap.add_argument("--n", type=float, default=1e8)
ap.add_argument("--seed", type=int, default=7)
ap.add_argument("--distort", type=float, default=0.0)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--pipeline", action="store_true",
                help="time the whole device pipeline (fused pass when it applies)")
a = ap.parse_args()
n = int(a.n)
pts = P.generate(a.dist, n, a.seed, a.distort)
d = torch.from_numpy(pts).cuda()
ctx = P.Context(0)
if a.pipeline:
    import time
    for _ in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hull, _ = ctx.heaphull_device(d, n)
        t1 = time.perf_counter()
        info = ctx.last_run()
        print(a.dist, n, "pipeline ms %.3f" % ((t1 - t0) * 1e3), "h", len(hull), "fused", info["fused"],
              info["fuse_state"], "cand", info["candidates"], "cov %.4f" % info["sample_coverage"],
              ctx.kernel_ms(), flush=True)
    sys.exit(0)
for _ in range(a.reps):
    rec = ctx.extremes(d, n)
    ext, mask = P.resolve_extremes(rec)
    if mask:
        ext = P.apply_corners(ext, ctx.corners_exact(d, n, (rec.x[0], rec.y[1], rec.x[2], rec.y[3])))
    plan = P.make_plan(ext, P.build_octagon_from_set(ext))
    counts = ctx.filter(d, n, plan)
    print(a.dist, n, "mask", mask, "counts", counts, ctx.kernel_ms(), flush=True)
