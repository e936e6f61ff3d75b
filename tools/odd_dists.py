"""Fused-pass behaviour on unusual inputs (GPU box): heavy tails, clusters,
skew, thin rotated ellipses, a parabola; hull checked against the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2209_12310_b200 as P  # noqa: E402
from oracle import Oracle  # noqa: E402

o = Oracle()
ctx = P.Context(0)
rng = np.random.default_rng(3)
n = 20_000_000
cases = {
    "cauchy": lambda: rng.standard_cauchy((n, 2)),
    "two_clusters": lambda: rng.normal(0, 1, (n, 2)) + np.where(rng.random((n, 1)) < 0.5, [[-50, 0]], [[50, 20]]),
    "exponential": lambda: rng.exponential(1.0, (n, 2)),
    "thin_ellipse": lambda: (rng.normal(0, 1, (n, 2)) * [1000.0, 0.01]) @ np.array([[0.8, 0.6], [-0.6, 0.8]]),
    "parabola": lambda: (lambda t: np.stack([t, t * t], 1))(rng.uniform(-1, 1, n)),
    "lattice_normal": lambda: np.round(rng.normal(0, 30, (n, 2))),
    "tiny_spread": lambda: 1e300 + rng.normal(0, 1e284, (n, 2)),
}
for name, make in cases.items():
    pts = np.ascontiguousarray(make())
    hull, _ = ctx.heaphull_device(torch.from_numpy(pts).cuda(), n)
    info = ctx.last_run()
    ok = np.array_equal(hull, o.heaphull(pts))
    print(f"{name:15s} fused={info['fused']!s:5s} {info['fuse_state']:22s} cand={info['candidates']:9d} "
          f"cov={info['sample_coverage']:.4f} h={len(hull):6d} {'OK' if ok else 'MISMATCH'}", flush=True)
