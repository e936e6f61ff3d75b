"""Host gap between back-to-back ohx_heaphull_device calls (normal 1e9).

Per call: the device-timed step (CUDA events around K calls), the C-side
wall time of the call (timings[2]) and the Python wall time of the call; the
difference between the device step and the C-side time is the GPU-idle gap
between calls (return to Python, the bench loop, re-entry).
"""
import sys
import time

import numpy as np
import torch

import paper_2209_12310_b200 as P

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000_000
K = int(sys.argv[2]) if len(sys.argv) > 2 else 100
hp = torch.empty((n, 2), dtype=torch.float64).pin_memory()
P.generate_range("normal", n, 0, n, 7, out=hp.numpy())
d = hp.to("cuda:0")
ctx = P.Context(0)
for _ in range(5):
    ctx.heaphull_device(d, n)
torch.cuda.synchronize()
for rep in range(3):
    cms, pys = [], []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(K):
        t = time.perf_counter()
        _, tm = ctx.heaphull_device(d, n)
        pys.append((time.perf_counter() - t) * 1e3)
        cms.append(tm["total_ms"])
    e1.record()
    torch.cuda.synchronize()
    dev = e0.elapsed_time(e1) / K
    print(f"rep {rep}: device step {dev:.4f} ms  C call {np.mean(cms):.4f} ms  "
          f"python call {np.mean(pys):.4f} ms  gap {dev - np.mean(cms):.4f} ms  "
          f"python overhead {np.mean(pys) - np.mean(cms):.4f} ms", flush=True)

# bare ctypes round trip of a trivial entry point
t = time.perf_counter()
for _ in range(10000):
    ctx.launches
print(f"ctx.launches: {(time.perf_counter() - t) / 10000 * 1e6:.2f} us/call")
