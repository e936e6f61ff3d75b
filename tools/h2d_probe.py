"""Host-API transfer probe: raw H2D (pinned / pageable) against the C-ABI
pipeline on pinned and pageable host points.  GPU box only."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2209_12310_b200 as P  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000_000
pinned = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
hp = pinned.numpy()
P.check(P.lib.ohx_generate(P.DISTS["normal"], n, 7, 0.0, hp.ctypes.data_as(P._dp), 0))
pageable = np.empty_like(hp)
pageable[:] = hp
d = torch.empty((n, 2), dtype=torch.float64, device="cuda")


def timeit(f, reps=3):
    f()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        t = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best


gb = n * 16 / 1e9
t = timeit(lambda: d.copy_(pinned, non_blocking=True))
print(f"raw H2D pinned    {t * 1e3:8.1f} ms {gb / t:6.1f} GB/s", flush=True)
pg = torch.from_numpy(pageable)
t = timeit(lambda: d.copy_(pg))
print(f"raw H2D pageable  {t * 1e3:8.1f} ms {gb / t:6.1f} GB/s", flush=True)
del d
torch.cuda.empty_cache()
out = np.empty((4096, 2))
h = P.C.c_uint64(0)
for name, arr in (("pinned", hp), ("pageable", pageable)):
    t = timeit(lambda: P.check(P.lib.ohx_heaphull(arr.ctypes.data_as(P._dp), n,
                                                  out.ctypes.data_as(P._dp), len(out),
                                                  P.C.byref(h), None)))
    print(f"ohx_heaphull {name:9s} {t * 1e3:8.1f} ms {n / t / 1e9:6.2f} Gpts/s", flush=True)
