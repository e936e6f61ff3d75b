"""Per-call cost of the native multi-GPU layer on ONE GPU: a 1-rank NCCL
world with one shard (ohx_mg_heaphull_shard) against the single-context
call (Context.heaphull_device) on the same device-resident points -- the
layer's own overhead (record all-gather, survivor hand-off to the root,
the extra host round trips), which is what every rank pays per step at
N > 1.  Usage: python tools/mg_overhead.py [n ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2209_12310_b200 as P  # noqa: E402
from paper_2209_12310_b200.mg import MultiGPU, unique_id  # noqa: E402

sizes = [float(v) for v in sys.argv[1:]] or [1e9, 5e8]
ctx = P.Context(0)
mg = MultiGPU.init_rank(unique_id(), 1, 0, 0)
for nf in sizes:
    n = int(nf)
    d = torch.from_numpy(P.generate("normal", n, 7)).cuda()
    ref = None
    for name, fn in (("context", lambda: ctx.heaphull_device(d, n)[0]),
                     ("mg 1 rank", lambda: mg.heaphull_shard(d, n, 0)[0]),
                     ("context", lambda: ctx.heaphull_device(d, n)[0]),
                     ("mg 1 rank", lambda: mg.heaphull_shard(d, n, 0)[0])):
        for _ in range(3):
            h = fn()
        if ref is None:
            ref = h
        assert h.shape == ref.shape and (h == ref).all(), name
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        t0 = time.perf_counter()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        print(f"n={n:.0e} {name:10s} device {e0.elapsed_time(e1) / reps:.4f} ms/call  "
              f"wall {(t1 - t0) * 1e3 / reps:.4f} ms/call", flush=True)
    _, info = mg.heaphull_shard(d, n, 0)
    print("  mg info", info, flush=True)
    del d
    torch.cuda.empty_cache()
