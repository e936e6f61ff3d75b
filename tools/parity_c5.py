"""BASELINE configs[4] corpus (normal, 4e9 points, seed 7) on ONE B200
against the reference library on the host, same bytes:

  python tools/parity_c5.py [--n 4e9] [--seed 7] [--shards 1,2,4,8]

The corpus (64 GB) is generated in pinned host memory, copied to the
device, run through the device pipeline (64-bit indices), then the
reference's heaphull_run + find_extremes (oracle/_ref, all host cores)
run on the same host buffer: hull coordinates, extremes and all four
queues are compared.  --shards additionally runs the multi-GPU pipeline
(ohx_mg, NCCL 1-rank communicator) with k virtual shards on this device
and compares it with the single-shard result."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2209_12310_b200 as P  # noqa: E402
from oracle import Reference  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=float, default=4e9)
ap.add_argument("--seed", type=int, default=7)
ap.add_argument("--shards", default="")
a = ap.parse_args()
n = int(a.n)
cores = os.cpu_count() or 1
log = {"corpus": f"generate({{normal, {n}, {a.seed}}})", "cores": cores}
t0 = time.perf_counter()
host = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
hp = host.numpy()
P.generate_range("normal", n, 0, n, a.seed, out=hp)
log["generate_s"] = time.perf_counter() - t0
d = host.cuda()
ctx = P.Context(0)
t0 = time.perf_counter()
hull, tm = ctx.heaphull_device(d, n)
hull, tm = ctx.heaphull_device(d, n)
log["device_ms"] = (time.perf_counter() - t0) * 1e3 / 2
info = ctx.last_run()
log["run"] = info
queues = [ctx.queue(q + 1, info["counts"][q])[0] for q in range(4)]
rec = ctx.extremes(d, n)
ext, mask = P.resolve_extremes(rec)
if mask:
    ext = P.apply_corners(ext, ctx.corners_exact(d, n, (rec.x[0], rec.y[1], rec.x[2], rec.y[3])))
ext = [int(v) for v in ext.ext]
mg = {}
for k in [int(s) for s in a.shards.split(",") if s]:
    t0 = time.perf_counter()
    h2, st = P.mg_heaphull_device([d], n, shards=k)
    mg[k] = {"hull_equal": bool(np.array_equal(h2, hull)), "ms": (time.perf_counter() - t0) * 1e3,
             "counts": st["counts"], "ext_equal": st["ext"] == ext}
log["mg_virtual_shards"] = mg
del d
torch.cuda.empty_cache()
ref = Reference()
t0 = time.perf_counter()
ref_hull, ref_labels, rt = ref.heaphull_run(hp, cores, 32)
ref_ext = [int(v) for v in ref.find_extremes(hp, cores, 32)]
log["reference_s"] = time.perf_counter() - t0
log["reference_ms"] = rt
log["hull_equal"] = bool(np.array_equal(hull, ref_hull))
log["h"] = [int(len(hull)), int(len(ref_hull))]
log["extremes_equal"] = ext == ref_ext
log["extremes"] = ext
log["queues_equal"] = all(np.array_equal(queues[q], np.flatnonzero(ref_labels == q + 1))
                          for q in range(4))
log["survivors"] = int((ref_labels != 0).sum())
print(json.dumps(log), flush=True)
