"""Per-step cost of the sharded orchestration (sharded.py) against the
single-call device pipeline, world size 1, on one GPU."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2209_12310_b200 as P  # noqa: E402
from paper_2209_12310_b200.sharded import CudaShard, sharded_heaphull  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000_000
host = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
P.check(P.lib.ohx_generate(P.DISTS["normal"], n, 7, 0.0, host.numpy().ctypes.data_as(P._dp), 0))
d = host.cuda()
ctx = P.Context(0)
shard = CudaShard(ctx, d, n, 0)
for name, f in (("device", lambda: ctx.heaphull_device(d, n)),
                ("sharded", lambda: sharded_heaphull(shard, device=torch.device("cpu")))):
    for _ in range(3):
        f()
    ts = []
    for _ in range(10):
        torch.cuda.synchronize()
        t = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t) * 1e3)
    print(name, "median ms %.3f" % np.median(ts), flush=True)
