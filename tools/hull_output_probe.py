"""Hull-stage output cost on a hull-heavy input (experiment tool): the same
device-resident circle through ohx_heaphull_device into (a) a fresh numpy
buffer per call (the Python wrapper's behaviour), (b) one reused,
pre-faulted buffer, and (c) a device buffer (ohx_heaphull_device_out: the
hull stays on the GPU).  Run with OHX_TRACE=1 for the stage split."""
import argparse
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2209_12310_b200 as P  # noqa: E402
from paper_2209_12310_b200 import lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dist", default="circle")
ap.add_argument("--n", type=float, default=1e8)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
n = int(a.n)
pts = P.generate(a.dist, n, 7)
d = torch.from_numpy(pts).cuda()
ctx = P.Context(0)
dp = C.POINTER(C.c_double)
ptr = C.c_void_p(d.data_ptr())
reused = np.ones((n + 8, 2))
for mode in ("fresh", "reused") * a.reps:
    buf = np.empty((n + 8, 2)) if mode == "fresh" else reused
    h = C.c_uint64(0)
    t = np.zeros(4)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    P.check(lib.ohx_heaphull_device(ctx.h, ptr, n, buf.ctypes.data_as(dp), len(buf), C.byref(h),
                                    t.ctypes.data_as(dp)))
    print(f"{mode:7s} {a.dist} {n} h={h.value} wall {1e3 * (time.perf_counter() - t0):.1f} ms "
          f"filter {t[0]:.2f} hull {t[1]:.2f}", flush=True)
dbuf = torch.empty((n + 8, 2), dtype=torch.float64, device="cuda")
for _ in range(a.reps):
    h = C.c_uint64(0)
    t = np.zeros(4)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    P.check(lib.ohx_heaphull_device_out(ctx.h, ptr, n, C.c_void_p(dbuf.data_ptr()), n + 8,
                                        C.byref(h), t.ctypes.data_as(dp)))
    print(f"device  {a.dist} {n} h={h.value} wall {1e3 * (time.perf_counter() - t0):.1f} ms "
          f"filter {t[0]:.2f} hull {t[1]:.2f}", flush=True)
