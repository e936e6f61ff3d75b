"""Does H2D from pinned memory go faster split over several streams / copy
engines?  16 GB pinned -> device as 1, 2, 4, 8 concurrent chunked copies
(experiment tool; GPU box only)."""
import os
import sys
import time

import torch

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000_000
host = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
host.fill_(1.0)
d = torch.empty((n, 2), dtype=torch.float64, device="cuda")
gb = n * 16 / 1e9
for k in (1, 2, 3, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    parts = [(i * n // k, (i + 1) * n // k) for i in range(k)]
    for chunk in (0, 64 << 20):  # whole parts, or 64 MB chunks round-robin
        def run():
            if chunk == 0:
                for s, (a, b) in zip(streams, parts):
                    with torch.cuda.stream(s):
                        d[a:b].copy_(host[a:b], non_blocking=True)
            else:
                per = chunk // 16
                j = 0
                for a in range(0, n, per):
                    b = min(n, a + per)
                    with torch.cuda.stream(streams[j % k]):
                        d[a:b].copy_(host[a:b], non_blocking=True)
                    j += 1
            torch.cuda.synchronize()
        run()
        best = 1e30
        for _ in range(3):
            t = time.perf_counter()
            run()
            best = min(best, time.perf_counter() - t)
        print(f"streams {k} chunk {chunk >> 20:3d} MB: {best * 1e3:7.1f} ms {gb / best:6.1f} GB/s",
              flush=True)
