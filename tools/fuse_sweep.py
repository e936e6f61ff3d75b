"""Robustness sweep of the fused pass: how often the provisional region is
certified (fuse_state) across distributions, sizes and seeds, with the hull
checked against the oracle.  Usage (GPU): python tools/fuse_sweep.py"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2209_12310_b200 as P  # noqa: E402
from oracle import Oracle  # noqa: E402

o = Oracle()
ctx = P.Context(0)
stats = collections.Counter()
bad = 0
for dist, sizes, seeds in [("normal", [9_000_000, 30_000_000, 100_000_000], range(12)),
                           ("square", [9_000_000, 30_000_000], range(8)),
                           ("circle", [10_000_000], [0]), ("disk", [10_000_000], [0])]:
    for n in sizes:
        for seed in seeds:
            pts = P.generate(dist, n, seed)
            hull, _ = ctx.heaphull_device(torch.from_numpy(pts).cuda(), n)
            info = ctx.last_run()
            ok = np.array_equal(hull, o.heaphull(pts))
            bad += not ok
            stats[(dist, info["fuse_state"])] += 1
            print(dist, n, seed, info["fuse_state"], info["candidates"],
                  "%.5f" % info["sample_coverage"], "OK" if ok else "MISMATCH", flush=True)
print(dict(stats), "mismatches", bad)
