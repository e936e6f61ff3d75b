"""Parity of the sm_100a path against the oracle and the reference's golden
fixtures, through the C ABI (ctypes).  Bit-exact everywhere: extreme
indices, labels, the four queues in order, hull coordinates."""

import os

import numpy as np
import pytest

import paper_2209_12310_b200 as P
from paper_2209_12310_b200 import _lib
from conftest import ROOT, sha

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    c = P.Context(0)
    yield c
    c.close()


def dev(pts):
    return torch.from_numpy(np.ascontiguousarray(pts)).cuda()


def ext_set(pts, ext):
    s = _lib.ExtremeSet()
    for k, j in enumerate(ext):
        s.ext[k], s.x[k], s.y[k] = int(j), pts[int(j), 0], pts[int(j), 1]
    return s


def run_kernels(ctx, pts, oracle, base=0):
    """K1 -> certificate -> K1b -> octagon -> K2 through the kernel-level ABI."""
    d = dev(pts)
    n = len(pts)
    rec = ctx.extremes(d, n, base)
    ext, mask = P.resolve_extremes(rec)
    if mask:
        bbox = (rec.x[0], rec.y[1], rec.x[2], rec.y[3])
        ext = P.apply_corners(ext, ctx.corners_exact(d, n, bbox, base))
    octg = P.build_octagon_from_set(ext)
    plan = P.make_plan(ext, octg)
    labels = torch.empty(n, dtype=torch.uint8, device="cuda")
    counts = ctx.filter(d, n, plan, base, d_labels=labels)
    queues = [ctx.queue(q + 1, counts[q])[0] for q in range(4)]
    return rec, ext, mask, octg, labels.cpu().numpy(), counts, queues


# ------------------------------------------------------------- golden ----
@pytest.mark.parametrize("k", range(23))
def test_api_matches_reference_golden(golden, k):
    c = golden["cases"][k]
    pts = P.generate(c["dist"], c["n"], c["seed"], c["distort"])
    assert sha(pts) == c["points_sha256"]
    assert [int(v) for v in P.find_extremes(pts)] == c["ext"]
    hull, labels, t = P.heaphull_run(pts)
    assert [int((labels == v).sum()) for v in range(5)] == c["label_hist"]
    assert sha(labels) == c["labels_sha256"]
    assert len(hull) == c["h"] and sha(hull) == c["hull_sha256"]
    if "hull" in c:
        assert hull.tolist() == c["hull"]
    assert np.array_equal(P.heaphull(pts), hull)
    assert np.array_equal(P.classify(pts), labels)
    assert P.filter_rate(labels) == c["filter_rate"]


@pytest.mark.parametrize("k", range(23))
def test_kernels_match_oracle(ctx, oracle, golden, k):
    c = golden["cases"][k]
    pts = P.generate(c["dist"], c["n"], c["seed"], c["distort"])
    rec, ext, mask, octg, labels, counts, queues = run_kernels(ctx, pts, oracle)
    # K1 axis slots and diagonal winners/seconds against a host scan
    x, y = pts[:, 0], pts[:, 1]
    keys = [x, y, -x, -y, x + y, y - x, -(x + y), x - y]
    for a, kk in enumerate(keys):
        j = int(np.flatnonzero(kk == kk.max())[0])
        assert rec.idx[a] == j and rec.x[a] == x[j] and rec.y[a] == y[j]
        if a >= 4:
            rest = np.delete(kk, j)
            assert rec.second[a - 4] == (rest.max() if rest.size else -np.inf)
    assert [int(v) for v in ext.ext] == c["ext"]
    assert octg.tolist() == c["octagon"]
    assert sha(labels) == c["labels_sha256"]
    assert counts == c["queue_len"]
    assert sha(np.concatenate(queues)) == c["queues_sha256"]
    assert np.array_equal(labels, oracle.classify(pts))


def test_degenerate_grids_match_reference(grid_trials):
    # test_hull.cpp:223-249, 5000 tiny integer grids: ties, duplicates, lines
    for t in grid_trials:
        a = np.array(t["pts"], dtype=float)
        assert [int(v) for v in P.find_extremes(a)] == t["ext"]
        hull, labels, _ = P.heaphull_run(a)
        assert labels.tolist() == t["labels"]
        assert hull.tolist() == t["hull"]


def test_exact_corner_kernel_matches_oracle(ctx, oracle):
    rng = np.random.default_rng(11)
    for n in (1, 5, 1000, 70001):
        pts = (rng.integers(-5, 6, size=(n, 2)) / 4.0).astype(float)
        axis = oracle.find_extremes(pts)[:4]
        bbox = (pts[axis[0], 0], pts[axis[1], 1], pts[axis[2], 0], pts[axis[3], 1])
        crec = ctx.corners_exact(dev(pts), n, bbox)
        assert [int(v) for v in crec.idx] == [int(v) for v in oracle.corner_extremes(pts, axis)]


# ---------------------------------------------------- shapes and tiles ----
@pytest.mark.parametrize("n", [1, 2, 3, 31, 32, 33, 255, 256, 2047, 2048, 2049,
                               4095, 4096, 4097, 3 * 2048 + 5, 65537, 300007])
def test_tile_boundaries_ragged_sizes(ctx, oracle, n):
    rng = np.random.default_rng(n)
    # coarse grid: heavy ties, duplicates, collinear runs, and plenty of survivors
    pts = (rng.integers(-40, 41, size=(n, 2)) / 8.0).astype(float)
    rec, ext, mask, octg, labels, counts, queues = run_kernels(ctx, pts, oracle)
    assert np.array_equal(ext.ext, oracle.find_extremes(pts))
    want = oracle.classify(pts)
    assert np.array_equal(labels, want)
    for q in range(4):
        assert np.array_equal(queues[q], np.flatnonzero(want == q + 1))
    hull = P.heaphull(pts)
    assert np.array_equal(hull, oracle.heaphull(pts))


def test_all_points_survive_circle(ctx, oracle):
    pts = P.generate("circle", 500000, 21)
    rec, ext, mask, octg, labels, counts, queues = run_kernels(ctx, pts, oracle)
    want = oracle.classify(pts)
    assert np.array_equal(labels, want)
    assert sum(counts) == int((want != 0).sum()) and sum(counts) > 0.99 * len(pts)
    assert np.array_equal(P.heaphull(pts), oracle.heaphull(pts))


def test_degenerate_octagon_filters_nothing(ctx, oracle):
    # collinear input: octagon has 2 vertices, every point goes to a queue
    n = 10000
    t = np.linspace(-1, 1, n)
    pts = np.stack([t, 0.5 * t], axis=1)
    rec, ext, mask, octg, labels, counts, queues = run_kernels(ctx, pts, oracle)
    assert len(octg) < 3
    assert np.array_equal(labels, oracle.classify(pts))
    assert (labels != 0).all()


@pytest.mark.parametrize("m", [3, 8, 9, 37, 1000])
def test_classify_points_any_polygon(oracle, m):
    # classify_points takes the caller's polygon (filter.cpp:104-131 accepts
    # any vertex list): regular m-gons inside a disk, ties on the boundary,
    # plus a reversed (clockwise) one; kept overrides from find_extremes
    pts = P.generate("disk", 300_001, 5)
    th = np.linspace(0, 2 * np.pi, m, endpoint=False)
    poly = np.stack([0.9 * np.cos(th), 0.9 * np.sin(th)], axis=1)
    pts[:m] = poly  # points exactly on the vertices
    ext = oracle.find_extremes(pts)
    for pg in (poly, poly[::-1].copy()):
        got = P.classify_points(pts, pg, ext)
        assert np.array_equal(got, oracle.classify(pts, ext, pg)), m


# ------------------------------------------------------------ sharding ----
@pytest.mark.parametrize("shards", [2, 3, 7])
def test_shard_records_combine_to_whole(ctx, oracle, shards):
    pts = P.generate("disk", 200001, 17)
    n = len(pts)
    bounds = np.linspace(0, n, shards + 1).astype(int)
    recs = [ctx.extremes(dev(pts[b0:b1]), b1 - b0, b0) for b0, b1 in zip(bounds[:-1], bounds[1:])]
    whole = ctx.extremes(dev(pts), n)
    g = P.combine_extremes(recs)
    assert list(g.idx) == list(whole.idx) and list(g.second) == list(whole.second)
    ext, mask = P.resolve_extremes(g)
    if mask:
        bbox = (g.x[0], g.y[1], g.x[2], g.y[3])
        crecs = [ctx.corners_exact(dev(pts[b0:b1]), b1 - b0, bbox, b0)
                 for b0, b1 in zip(bounds[:-1], bounds[1:])]
        ext = P.apply_corners(ext, P.combine_corners(crecs))
    assert np.array_equal(ext.ext, oracle.find_extremes(pts))
    plan = P.make_plan(ext, P.build_octagon_from_set(ext))
    want = oracle.classify(pts)
    for b0, b1 in zip(bounds[:-1], bounds[1:]):
        counts = ctx.filter(dev(pts[b0:b1]), b1 - b0, plan, b0)
        for q in range(4):
            got = ctx.queue(q + 1, counts[q])[0]
            assert np.array_equal(got, b0 + np.flatnonzero(want[b0:b1] == q + 1))


@pytest.mark.parametrize("dist,shards", [("normal", 3), ("square", 2)])
def test_fused_shards_match_whole(oracle, dist, shards):
    # the fused pass per shard (each with its own context, region and
    # candidates) combines to the reference result of the whole input: the
    # records equal K1's, the per-shard queues equal build_queues' slices
    pts = P.generate(dist, 30_000_000, 11)
    n = len(pts)
    bounds = np.linspace(0, n, shards + 1).astype(int)
    ctxs = [P.Context(0) for _ in range(shards)]
    devs = [dev(pts[b0:b1]) for b0, b1 in zip(bounds[:-1], bounds[1:])]
    recs = []
    for c, d, b0, b1 in zip(ctxs, devs, bounds[:-1], bounds[1:]):
        rec = c.fused_extremes(d, b1 - b0, b0)
        assert rec is not None, c.last_run()
        k1 = c.extremes(d, b1 - b0, b0)
        assert list(rec.idx) == list(k1.idx) and list(rec.second) == list(k1.second)
        assert list(rec.key) == list(k1.key)
        recs.append(rec)
    g = P.combine_extremes(recs)
    ext, mask = P.resolve_extremes(g)
    assert mask == 0
    want_ext = oracle.find_extremes(pts)
    assert np.array_equal(ext.ext, want_ext)
    octg = P.build_octagon_from_set(ext)
    plan = P.make_plan(ext, octg)
    want = oracle.classify(pts, want_ext, octg)
    for c, d, b0, b1 in zip(ctxs, devs, bounds[:-1], bounds[1:]):
        counts, fused = c.filter_fused(d, b1 - b0, ext, plan, b0)
        assert fused
        for q in range(4):
            got = c.queue(q + 1, counts[q])[0]
            assert np.array_equal(got, b0 + np.flatnonzero(want[b0:b1] == q + 1))
    with pytest.raises(ValueError):  # no pending fused pass any more
        ctxs[0].filter_fused(devs[0], bounds[1], ext, plan, 0)
    for c in ctxs:
        c.close()


# ---------------------------------------------------------- large sizes ----
def test_normal_1e8_matches_oracle(ctx, oracle):
    pts = P.generate("normal", 100_000_000, 7)
    d = dev(pts)
    rec = ctx.extremes(d, len(pts))
    ext, mask = P.resolve_extremes(rec)
    assert mask == 0  # certified on the normal corpus
    want_ext = oracle.find_extremes(pts)
    assert np.array_equal(ext.ext, want_ext)
    octg = P.build_octagon_from_set(ext)
    plan = P.make_plan(ext, octg)
    counts = ctx.filter(d, len(pts), plan)
    want = oracle.classify(pts, want_ext, octg)
    nz = np.flatnonzero(want)
    assert sum(counts) == len(nz)
    for q in range(4):
        got = ctx.queue(q + 1, counts[q])[0]
        assert np.array_equal(got, nz[want[nz] == q + 1])
    hull, _ = ctx.heaphull_device(d, len(pts))
    del d
    assert np.array_equal(hull, oracle.heaphull(pts))


def test_launch_counter_proves_native_path(ctx):
    before = ctx.launches
    pts = P.generate("square", 10000, 3)
    run_kernels(ctx, pts, None)
    assert ctx.launches >= before + 2


# ------------------------------------------------------- fused single pass ----
FUSED_CASES = [("normal", 10_000_000, 7, 0.0, True), ("normal", 12_000_000, 1, 0.0, True),
               ("normal", 20_000_000, 2, 0.0, True), ("normal", 30_000_000, 3, 0.0, True),
               ("square", 9_000_000, 3, 0.0, True), ("square", 20_000_000, 4, 0.0, True),
               ("disk", 9_000_000, 5, 0.0, False), ("circle", 9_000_000, 9, 1.0, False)]


@pytest.mark.parametrize("dist,n,seed,d,fused", FUSED_CASES)
def test_fused_pipeline_matches_oracle(ctx, oracle, dist, n, seed, d, fused):
    pts = P.generate(dist, n, seed, d)
    dpts = dev(pts)
    hull, _ = ctx.heaphull_device(dpts, n)
    info = ctx.last_run()
    assert info["fused"] == fused, info["fuse_state"]
    want_hull, want_labels = oracle.heaphull(pts, with_labels=True)
    assert np.array_equal(hull, want_hull)
    assert info["counts"] == [int((want_labels == q).sum()) for q in (1, 2, 3, 4)]
    # the queues themselves, in order
    for q in range(4):
        idx, _ = ctx.queue(q + 1, info["counts"][q])
        assert np.array_equal(idx, np.flatnonzero(want_labels == q + 1))
    if fused:
        assert 0 < info["candidates"] < n // 8


def test_fused_labels_through_the_host_api(oracle):
    pts = P.generate("normal", 9_000_000, 21)
    hull, labels, _ = P.heaphull_run(pts)
    want_hull, want_labels = oracle.heaphull(pts, with_labels=True)
    assert np.array_equal(labels, want_labels)
    assert np.array_equal(hull, want_hull)


def test_fused_verification_failure_falls_back(tmp_path):
    # OHX_FUSE=fallback rejects the provisional box after the fused pass:
    # the result must still be exact (the regular second pass runs)
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, paper_2209_12310_b200 as P\n"
        "from oracle import Oracle\n"
        "pts = P.generate('normal', 9_000_000, 5)\n"
        "ctx = P.Context(0)\n"
        "hull, _ = ctx.heaphull_device(torch.from_numpy(pts).cuda(), len(pts))\n"
        "info = ctx.last_run()\n"
        "assert not info['fused'], info\n"
        "assert np.array_equal(hull, Oracle().heaphull(pts))\n"
        "print('fallback ok')\n")
    env = dict(os.environ, OHX_FUSE="fallback", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       timeout=600)
    assert r.returncode == 0 and "fallback ok" in r.stdout, r.stderr[-3000:]


@pytest.mark.parametrize("fuse", ["auto", "0"])
def test_tma_streaming_variant_matches_oracle(fuse):
    # OHX_STREAM=tma selects the TMA bulk-copy (cp.async.bulk + mbarrier)
    # K1 instead of the register-staged default: same results, bit for bit
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, paper_2209_12310_b200 as P\n"
        "from oracle import Oracle\n"
        "o = Oracle()\n"
        "ctx = P.Context(0)\n"
        "for dist, n, seed, d in [('normal', 9_000_000, 5, 0.0), ('square', 8_500_003, 2, 0.0),\n"
        "                         ('circle', 1_000_003, 4, 1.0), ('normal', 777_777, 3, 0.0)]:\n"
        "    pts = P.generate(dist, n, seed, d)\n"
        "    hull, _ = ctx.heaphull_device(torch.from_numpy(pts).cuda(), n)\n"
        "    want_hull, want_labels = o.heaphull(pts, with_labels=True)\n"
        "    assert np.array_equal(hull, want_hull), dist\n"
        "    info = ctx.last_run()\n"
        "    assert info['counts'] == [int((want_labels == q).sum()) for q in (1, 2, 3, 4)]\n"
        "print('tma ok')\n")
    env = dict(os.environ, OHX_STREAM="tma", OHX_FUSE=fuse, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       timeout=600)
    assert r.returncode == 0 and "tma ok" in r.stdout, r.stderr[-3000:]


@pytest.mark.parametrize("one_pass", ["1", "0"])
def test_forced_fusion_heavy_candidates_match_oracle(one_pass):
    # OHX_FUSE=force fuses even when the provisional region covers the data
    # poorly (disk: ~25 % candidates, most warp tiles spill past their
    # 15-offset slot); the result must still be exact -- with K2 over the
    # candidates in one launch (up to 2048 tiles; a 20M-point disk's 5M
    # candidates take the two kernels) and as k2_filter + k2_compact
    # (OHX_K2_ONEPASS=0)
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, paper_2209_12310_b200 as P\n"
        "from oracle import Oracle\n"
        "o = Oracle()\n"
        "ctx = P.Context(0)\n"
        "cases = [('disk', 9_000_000, 5), ('square', 8_500_003, 2), ('normal', 8_388_700, 9)]\n"
        "if one_pass: cases.append(('disk', 20_000_000, 6))  # > 2048 candidate tiles: two kernels\n"
        "for dist, n, seed in cases:\n"
        "    pts = P.generate(dist, n, seed)\n"
        "    hull, _ = ctx.heaphull_device(torch.from_numpy(pts).cuda(), n)\n"
        "    info = ctx.last_run()\n"
        "    assert info['fused'], (dist, info)\n"
        "    want_hull, want_labels = o.heaphull(pts, with_labels=True)\n"
        "    assert np.array_equal(hull, want_hull), dist\n"
        "    assert info['counts'] == [int((want_labels == q).sum()) for q in (1, 2, 3, 4)]\n"
        "    for q in range(4):\n"
        "        idx, _ = ctx.queue(q + 1, info['counts'][q])\n"
        "        assert np.array_equal(idx, np.flatnonzero(want_labels == q + 1)), (dist, q)\n"
        "print('force ok')\n").replace("one_pass", repr(one_pass == "1"))
    env = dict(os.environ, OHX_FUSE="force", OHX_K2_ONEPASS=one_pass, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       timeout=600)
    assert r.returncode == 0 and "force ok" in r.stdout, r.stderr[-3000:]


def test_sorted_input_overflows_warp_regions_and_stays_exact(ctx, oracle):
    # points sorted by radius: the sample still covers the region well (the
    # fused pass runs), but every candidate sits in the last warps' ranges,
    # whose KF regions overflow -> the call takes the two-pass path
    pts = P.generate("normal", 9_000_000, 13)
    pts = np.ascontiguousarray(pts[np.argsort(np.hypot(pts[:, 0], pts[:, 1]), kind="stable")])
    n = len(pts)
    hull, _ = ctx.heaphull_device(dev(pts), n)
    info = ctx.last_run()
    assert not info["fused"] and info["fuse_state"] == "too-many-candidates", info
    want_hull, want_labels = oracle.heaphull(pts, with_labels=True)
    assert np.array_equal(hull, want_hull)
    assert info["counts"] == [int((want_labels == q).sum()) for q in (1, 2, 3, 4)]


def test_device_sweep_sort_forced_on_small_survivor_sets():
    # OHX_DEVICE_SORT_MIN=0 sends every survivor set -- empty queues, single
    # points, lattices full of duplicates and collinear runs -- through the
    # device sweep sort (default: 2^17 survivors and up); hulls must match
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, paper_2209_12310_b200 as P\n"
        "from oracle import Oracle\n"
        "o = Oracle()\n"
        "ctx = P.Context(0)\n"
        "cases = [P.generate('normal', 1_000_000, 7), P.generate('square', 70_001, 3),\n"
        "         P.generate('circle', 5_000, 2), P.generate('disk', 3, 1),\n"
        "         np.array([[0.0, 0.0], [1.0, 0.0], [2.0, 0.0]]),\n"
        "         np.array([[1.0, 1.0]] * 5), np.array([[0.0, -0.0], [-0.0, 0.0], [1.0, 1.0]])]\n"
        "g = np.stack(np.meshgrid(np.arange(-40, 41.0), np.arange(-40, 41.0)), -1).reshape(-1, 2)\n"
        "cases.append(np.ascontiguousarray(np.concatenate([g, g[::7]])))\n"
        "rng = np.random.default_rng(3)\n"
        "cases.append(np.ascontiguousarray(np.round(rng.normal(size=(20_000, 2)) * 3)))\n"
        "for pts in cases:\n"
        "    pts = np.ascontiguousarray(pts, dtype=np.float64)\n"
        "    hull, _ = ctx.heaphull_device(torch.from_numpy(pts).cuda(), len(pts))\n"
        "    assert np.array_equal(hull, o.heaphull(pts)), len(pts)\n"
        "    assert np.array_equal(P.heaphull(pts), hull)\n"
        "print('dsort ok')\n")
    env = dict(os.environ, OHX_DEVICE_SORT_MIN="0", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       timeout=600)
    assert r.returncode == 0 and "dsort ok" in r.stdout, r.stderr[-3000:]


@pytest.mark.parametrize("scale", [50.0, 3000.0, 1e6])
def test_device_sorted_hull_on_degenerate_survivors(oracle, scale):
    # survivor sets past the device sweep-sort threshold, full of duplicates,
    # collinear runs and -0.0 / +0.0 coordinates (np.round(-0.3) == -0.0)
    rng = np.random.default_rng(int(scale))
    t = rng.uniform(0, 2 * np.pi, 300_000)
    pts = np.ascontiguousarray(np.round(np.stack([np.cos(t), np.sin(t)], 1) * scale))
    assert np.signbit(pts).any() and (scale > 1e4 or (pts == 0).any())
    hull = P.heaphull(pts)
    assert np.array_equal(hull, oracle.heaphull(pts))



def test_u64_indices_on_a_tiled_4p5e9_point_input(ctx):
    # 4.5e9 points (72 GB of HBM) = the same 9e8-point block tiled 5 times:
    # every shard-local index needs 64 bits (K1/K2/KF/queues take their u64
    # paths).  Size-independent properties: the extremes are the block's
    # (first occurrence wins), the hull is the block's hull, and every queue
    # is the block's queue repeated with offsets t*B -- except that in the
    # later tiles the copies of the eight kept points are plain boundary
    # points of the octagon (reference label 0: only the kept INDICES carry
    # the override, filter.cpp:108-124).
    free, _ = torch.cuda.mem_get_info()
    B, T = 900_000_000, 5
    if free < (B * T * 16) * 1.25:
        pytest.skip(f"needs ~{B * T * 16 * 1.25 / 2**30:.0f} GiB of free device memory")
    n = B * T
    blk = P.generate("normal", B, 3)
    d = torch.empty((n, 2), dtype=torch.float64, device="cuda")
    d[:B].copy_(torch.from_numpy(blk))
    del blk
    for t in range(1, T):
        d[t * B:(t + 1) * B].copy_(d[:B])
    # the block alone (u32 paths)
    hull_b, _ = ctx.heaphull_device(d[:B], B)
    info_b = ctx.last_run()
    qb = [ctx.queue(q + 1, info_b["counts"][q])[0] for q in range(4)]
    rec_b = ctx.extremes(d[:B], B)
    ext_b, mask_b = P.resolve_extremes(rec_b)
    if mask_b:
        ext_b = P.apply_corners(ext_b, ctx.corners_exact(
            d[:B], B, (rec_b.x[0], rec_b.y[1], rec_b.x[2], rec_b.y[3])))
    kept = np.array(list(ext_b.ext), dtype=np.uint64)
    want = [np.concatenate([qb[q]] + [qb[q][~np.isin(qb[q], kept)] + np.uint64(t * B)
                                      for t in range(1, T)]) for q in range(4)]
    # fused pipeline over the tiled input
    hull, _ = ctx.heaphull_device(d, n)
    info = ctx.last_run()
    assert info["fused"], info
    assert np.array_equal(hull, hull_b)
    assert info["counts"] == [len(w) for w in want]
    for q in range(4):
        assert np.array_equal(ctx.queue(q + 1, info["counts"][q])[0], want[q]), q
    # two-pass kernels (K1, K2) over the tiled input
    rec = ctx.extremes(d, n)
    assert list(rec.idx) == list(rec_b.idx) and rec.n == n
    ext, mask = P.resolve_extremes(rec)
    if mask:
        ext = P.apply_corners(ext, ctx.corners_exact(d, n, (rec.x[0], rec.y[1], rec.x[2], rec.y[3])))
    assert list(ext.ext) == list(ext_b.ext)
    plan = P.make_plan(ext, P.build_octagon_from_set(ext))
    counts = ctx.filter(d, n, plan)
    assert counts == info["counts"]
    for q in range(4):
        assert np.array_equal(ctx.queue(q + 1, counts[q])[0], want[q]), q
    del d
    torch.cuda.empty_cache()


# ------------------------------------------------------------ PTS2 files
def test_pts2_straight_to_device(ctx, oracle, tmp_path):
    # file -> pinned chunks -> device, bit-exact; the first non-finite point
    # is reported with its index and byte offset (reference io.cpp:117-120)
    pts = P.generate("normal", 9_000_017, 19)  # > one 64 MB staging chunk
    f = tmp_path / "p.bin"
    P.write_pts2(pts, f)
    n, d = ctx.load_pts2(f)
    assert n == len(pts)
    assert np.array_equal(d.cpu().numpy(), pts)
    hull = P.heaphull_file(f)
    assert np.array_equal(hull, oracle.heaphull(pts))
    for bad in (8_999_999, 4_194_305, 0):
        q = pts.copy()
        q[bad, bad % 2] = np.inf if bad else np.nan
        q[bad + 7, 0] = np.nan  # a later one must not be the one reported
        P.write_pts2(q, f)
        with pytest.raises(P.OhxError, match=f"point {bad} at byte {12 + 16 * bad}"):
            ctx.load_pts2(f)


@pytest.mark.parametrize("shape", ["same", "line", "two", "grid"])
def test_degenerate_large_inputs(ctx, oracle, shape):
    # large inputs (past the fused-pass threshold) whose octagon degenerates
    # or whose extremes tie massively: every pipeline stage must agree with
    # the oracle (fused or not)
    n = 9_000_000
    rng = np.random.default_rng(7)
    if shape == "same":
        pts = np.full((n, 2), 1.5)
    elif shape == "line":
        t = rng.uniform(-1, 1, n)
        pts = np.stack([t, 3 * t + 0.25], 1)
    elif shape == "two":
        pts = np.where(rng.random((n, 1)) < 0.5, [[0.0, 0.0]], [[1.0, -2.0]])
    else:
        pts = rng.integers(-40, 41, size=(n, 2)).astype(float)
    pts = np.ascontiguousarray(pts)
    hull, _ = ctx.heaphull_device(dev(pts), n)
    want_hull, want_labels = oracle.heaphull(pts, with_labels=True)
    assert np.array_equal(hull, want_hull), shape
    info = ctx.last_run()
    assert info["counts"] == [int((want_labels == q).sum()) for q in (1, 2, 3, 4)], (shape, info)


def test_trim_releases_and_regrows(oracle):
    c = P.Context(0)
    pts = P.generate("circle", 2_000_000, 5, 1.0)
    d = dev(pts)
    h1, _ = c.heaphull_device(d, len(pts))
    c.trim()
    h2, _ = c.heaphull_device(d, len(pts))
    assert np.array_equal(h1, h2) and np.array_equal(h1, oracle.heaphull(pts))
    c.close()


@pytest.mark.parametrize("scale,offset", [(1e300, 0.0), (1e-300, 0.0), (1e-310, 0.0),
                                          (1.0, 1e15), (3e-9, -7.0)])
@pytest.mark.parametrize("n", [1_000_003, 9_000_000])
def test_extreme_magnitudes_match_oracle(ctx, oracle, scale, offset, n):
    # x + y overflowing to +-inf (1e300), subnormal coordinates (1e-300,
    # 1e-310), and points whose spread is a few ulps of their offset (ties
    # galore): the fused pass's region, its certification and the two-pass
    # path must still give the reference's results bit for bit
    pts = np.ascontiguousarray(P.generate("normal", n, 11) * scale + offset)
    assert np.isfinite(pts).all()
    hull, _ = ctx.heaphull_device(dev(pts), n)
    info = ctx.last_run()
    want_hull, want_labels = oracle.heaphull(pts, with_labels=True)
    assert np.array_equal(hull, want_hull), info
    assert info["counts"] == [int((want_labels == q).sum()) for q in (1, 2, 3, 4)], info
    for q in range(4):
        idx, _ = ctx.queue(q + 1, info["counts"][q])
        assert np.array_equal(idx, np.flatnonzero(want_labels == q + 1)), q


def _min_index_of(pts, hull):
    """For each hull vertex, the smallest index j with pts[j] == vertex."""
    z = pts + 0.0  # -0.0 -> +0.0: the reference compares with ==
    order = np.lexsort((np.arange(len(z)), z[:, 1], z[:, 0]))
    zs = z[order]
    first = np.ones(len(zs), dtype=bool)
    first[1:] = (zs[1:] != zs[:-1]).any(axis=1)
    keys = {(a, b): int(j) for (a, b), j in zip(map(tuple, zs[first]), order[first])}
    return np.array([keys[(a + 0.0, b + 0.0)] for a, b in hull], dtype=np.int64)


@pytest.mark.parametrize("case", ["normal_1e6", "normal_9e6", "lattice_dups", "circle",
                                  "signed_zeros", "collinear"])
def test_hull_vertex_indices(ctx, oracle, case):
    # the north star's parity output "hull vertex indices": the smallest
    # input index with each vertex's coordinates, in the hull's order
    rng = np.random.default_rng(3)
    if case == "normal_1e6":
        pts = P.generate("normal", 1_000_000, 7)
    elif case == "normal_9e6":
        pts = P.generate("normal", 9_000_000, 7)
    elif case == "lattice_dups":  # every vertex repeated, later copies first in the array
        g = rng.integers(-30, 31, size=(2_000_000, 2)).astype(float)
        pts = np.concatenate([g[::-1], g])
    elif case == "circle":
        pts = P.generate("circle", 300_000, 5)
    elif case == "signed_zeros":
        g = rng.integers(-2, 3, size=(200_000, 2)).astype(float)
        g[rng.random(len(g)) < 0.5] *= -1.0  # -0.0 copies of the zero coordinates
        pts = g
    else:
        t = rng.integers(0, 1000, 100_000).astype(float)
        pts = np.stack([t, 2 * t], 1)
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    hull, _ = ctx.heaphull_device(dev(pts), len(pts))
    assert np.array_equal(hull, oracle.heaphull(pts))
    idx = ctx.hull_indices(hull)
    assert np.array_equal(idx, _min_index_of(pts, hull)), case
    assert np.array_equal(pts[idx] + 0.0, hull + 0.0)
    # the host API and the default context
    assert np.array_equal(P.heaphull(pts), hull)
    assert np.array_equal(P.hull_indices(hull), idx)


def test_stage_time_sums_count_each_call_once(ctx):
    # ohx_ctx_kernel_ms_sum: per-stage CUDA-event sums over the calls since
    # the reset, each call's stages counted once (the bench reads them once
    # after its timed loop instead of querying events between steps)
    pts = P.generate("normal", 9_000_000, 7)
    d = dev(pts)
    ctx.heaphull_device(d, len(pts))
    ctx.kernel_ms_sum(reset=True)
    for _ in range(3):
        ctx.heaphull_device(d, len(pts))
    s = ctx.kernel_ms_sum()
    assert ctx.last_run()["fused"]
    assert s["k1"][1] == 3 and s["kc"][1] == 3 and s["k2"][1] == 3 and s["k1b"][1] == 0, s
    assert all(s[k][0] > 0 for k in ("k1", "kc", "k2")), s
    assert ctx.kernel_ms_sum() == s  # reading does not count again
    assert ctx.kernel_ms_sum(reset=True) == s and ctx.kernel_ms_sum()["k1"] == (0.0, 0)
