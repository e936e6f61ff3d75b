"""Full-size robustness + parity sweep (GPU box): BASELINE shapes over many
seeds, the device pipeline against the reference library (oracle/_ref, all
host cores): hull, extremes and the four queues; fused state recorded.
Usage: python tools/sweep_full.py [seeds] [dist:n,dist:n,...]
Every case also checks the hull written to a pinned host buffer (the
pipelined stage for large survivor sets) and left in device memory."""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2209_12310_b200 as P  # noqa: E402
from oracle import Reference  # noqa: E402

seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ref = Reference()
cores = os.cpu_count() or 1
ctx = P.Context(0)
stats = collections.Counter()
shapes = [("normal", 1_000_000_000), ("square", 100_000_000), ("normal", 100_000_000)]
if len(sys.argv) > 2:
    shapes = [(a.split(":")[0], int(float(a.split(":")[1]))) for a in sys.argv[2].split(",")]
for dist, n in shapes:
    host = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
    hp = host.numpy()
    d = torch.empty((n, 2), dtype=torch.float64, device="cuda")
    for seed in range(100, 100 + seeds):
        P.check(P.lib.ohx_generate(P.DISTS[dist], n, seed, 0.0, hp.ctypes.data_as(P._dp), 0))
        d.copy_(host)
        t0 = time.perf_counter()
        hull, _ = ctx.heaphull_device(d, n)
        dt = time.perf_counter() - t0
        info = ctx.last_run()
        qs = [ctx.queue(q + 1, info["counts"][q])[0] for q in range(4)]
        pin = torch.empty(((n if n < 2**28 else len(hull)) + 8, 2), dtype=torch.float64,
                          pin_memory=True)
        ph, _ = ctx.heaphull_device(d, n, out=pin)
        dbuf = torch.empty((n + 8, 2), dtype=torch.float64, device="cuda") if n < 2**28 else None
        dh = ctx.heaphull_device(d, n, out=dbuf)[0].cpu().numpy() if dbuf is not None else hull
        del dbuf
        rh, rl, _ = ref.heaphull_run(hp, cores, 32)
        ok = np.array_equal(hull, rh) and np.array_equal(ph, rh) and np.array_equal(dh, rh) and all(
            np.array_equal(qs[q], np.flatnonzero(rl == q + 1)) for q in range(4))
        stats[(dist, n, info["fuse_state"], ok)] += 1
        print(f"{dist} {n:>10} seed {seed} {info['fuse_state']:18s} cand {info['candidates']:8d} "
              f"cov {info['sample_coverage']:.4f} {dt * 1e3:7.2f} ms {'OK' if ok else 'MISMATCH'}",
              flush=True)
        del rl
    del d, host
    torch.cuda.empty_cache()
print(dict(stats))
