"""Small runs of every kernel for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck):

  compute-sanitizer --tool memcheck python tools/sanitize_driver.py

two-pass K1 + K2 (+ labels) on normal 200k, K1b on a circle (the corner
certificate fails there), the fused pass (sample K1, count, KF, kf_gather,
candidate K1, K2 gather mode) on normal 9M, the device sweep sort + hull
indices on a 300k circle, the K2 look-back across many tile groups
(normal 3M two-pass with labels), the PTS2 loader's non-finite scan; the
hull into a device buffer (in place) and into pinned host memory (the
pipelined stage: OHX_HULL_PIPE_MIN lowered for the 300k circle).
Every result is checked against the oracle, so a sanitizer run is also a
parity run."""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OHX_DEVICE_SORT_MIN", "100000")
os.environ.setdefault("OHX_HULL_PIPE_MIN", "100000")  # the pipelined stage on the 300k circle
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2209_12310_b200 as P  # noqa: E402
from oracle import Oracle  # noqa: E402

o = Oracle()
ctx = P.Context(0)
cases = [("normal", 200_000, 7, 0.0), ("circle", 60_000, 3, 0.0), ("normal", 3_000_000, 5, 0.0),
         ("normal", 9_000_000, 7, 0.0), ("circle", 300_000, 2, 0.0)]
which = sys.argv[1:] or None
for k, (dist, n, seed, dd) in enumerate(cases):
    if which and str(k) not in which:
        continue
    pts = P.generate(dist, n, seed, dd)
    d = torch.from_numpy(pts).cuda()
    want_hull, want = o.heaphull(pts, with_labels=True)
    if n < 8_000_000:  # two-pass kernels with labels
        rec = ctx.extremes(d, n)
        ext, mask = P.resolve_extremes(rec)
        if mask:
            ext = P.apply_corners(ext, ctx.corners_exact(d, n, (rec.x[0], rec.y[1], rec.x[2],
                                                                rec.y[3])))
        octg = P.build_octagon_from_set(ext)
        labels = torch.empty(n, dtype=torch.uint8, device="cuda")
        counts = ctx.filter(d, n, P.make_plan(ext, octg), d_labels=labels)
        assert np.array_equal(labels.cpu().numpy(), want), (dist, n)
        print(f"case {k} {dist} {n}: two-pass labels ok, corner mask {mask}, counts {counts}",
              flush=True)
    hull, _ = ctx.heaphull_device(d, n)
    assert np.array_equal(hull, want_hull), (dist, n)
    info = ctx.last_run()
    idx = ctx.hull_indices(hull)
    assert (idx >= 0).all()
    dh, _ = ctx.heaphull_device(d, n, out="device")  # the hull left on the device
    assert np.array_equal(dh.cpu().numpy(), hull), (dist, n)
    pin = torch.empty((n + 8, 2), dtype=torch.float64, pin_memory=True)
    ph, _ = ctx.heaphull_device(d, n, out=pin)  # pinned host output (pipelined when large)
    assert np.array_equal(ph, hull), (dist, n)
    print(f"case {k} {dist} {n}: pipeline ok, fused {info['fused']}, hull path "
          f"{info['hull_path']}, h {len(hull)}", flush=True)
if not which or "pts2" in which:
    pts = P.generate("square", 100_000, 1)
    pts[77_777, 1] = np.inf
    with tempfile.TemporaryDirectory() as t:
        path = os.path.join(t, "p.pts2")
        P.write_pts2(pts, path)
        try:
            ctx.load_pts2(path)
            raise SystemExit("non-finite point not rejected")
        except P.OhxError as e:
            assert "77777" in str(e), e
    print("pts2 scan ok", flush=True)
torch.cuda.synchronize()
print("sanitize driver done", flush=True)
