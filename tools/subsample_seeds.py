"""Certification rate of the fused pass's provisional region over many
seeds (experiment tool): for each seed, the fused state, candidate count and
step time of ctx.heaphull_device on generate(dist, n, seed); run under
different OHX_SUBSAMPLES / OHX_SAMPLE_SEGS / OHX_REGION_PULL settings.
Usage (GPU): OHX_SUBSAMPLES=1 python tools/subsample_seeds.py normal 1e9 20"""
import collections
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2209_12310_b200 as P  # noqa: E402

dist, n, seeds = sys.argv[1], int(float(sys.argv[2])), int(sys.argv[3])
ctx = P.Context(0)
tag = (f"subs={os.environ.get('OHX_SUBSAMPLES', 'default')} "
       f"segs={os.environ.get('OHX_SAMPLE_SEGS', 'default')} "
       f"pull={os.environ.get('OHX_REGION_PULL', 'default')}")
d = torch.empty((n, 2), dtype=torch.float64, device="cuda")
host = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
states, cands, ms = collections.Counter(), [], []
for seed in range(seeds):
    P.check(P.lib.ohx_generate(P.DISTS[dist], n, 1000 + seed, 0.0,
                               host.numpy().ctypes.data_as(P._dp), 0))
    d.copy_(host)
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.heaphull_device(d, n)
        best = min(best, (time.perf_counter() - t0) * 1e3)
    info = ctx.last_run()
    states[info["fuse_state"]] += 1
    cands.append(info["candidates"])
    ms.append(best)
print(f"{tag} {dist} {n} seeds {seeds}: states {dict(states)} cand mean {statistics.mean(cands):.0f} "
      f"max {max(cands)} ms median {statistics.median(ms):.3f} max {max(ms):.3f}", flush=True)
