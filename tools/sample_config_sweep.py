"""Provisional-region sample configuration sweep (experiment tool): for the
current OHX_SUBSAMPLES / OHX_SAMPLE_SEGS settings, the fused pass's
candidate count, state and device time over sizes and seeds (no parity
check -- tools/fuse_sweep.py and tools/sweep_full.py do that).
Usage (GPU): OHX_SUBSAMPLES=4 python tools/sample_config_sweep.py"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2209_12310_b200 as P  # noqa: E402

ctx = P.Context(0)
tag = (f"subs={os.environ.get('OHX_SUBSAMPLES', 'default')} "
       f"segs={os.environ.get('OHX_SAMPLE_SEGS', 'default')} pull={os.environ.get('OHX_REGION_PULL', 'default')}")
for dist, n, seeds in [("normal", 30_000_000, range(6)), ("normal", 100_000_000, range(6)),
                       ("square", 100_000_000, range(3)), ("normal", 1_000_000_000, range(3))]:
    d = torch.empty((n, 2), dtype=torch.float64, device="cuda")
    cands, ms, states = [], [], set()
    for seed in seeds:
        d.copy_(torch.from_numpy(P.generate(dist, n, 100 + seed)))
        for r in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ctx.heaphull_device(d, n)
            t = (time.perf_counter() - t0) * 1e3
        info = ctx.last_run()
        cands.append(info["candidates"])
        ms.append(t)
        states.add(info["fuse_state"])
    print(f"{tag:22s} {dist} {n:>11d} cand mean {statistics.mean(cands):>10.0f} "
          f"max {max(cands):>9d} ms {statistics.mean(ms):7.3f} {sorted(states)}", flush=True)
    del d
    torch.cuda.empty_cache()
