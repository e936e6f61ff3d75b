"""The hull stage's chains on the device (csrc/hullchain.cu): chunked local
runs, the replay-until-coincidence proof per chunk, the cycle scan and the
rotated copy.  Every result is compared with the host chains (themselves
pinned to the reference loop in test_host.py) and the oracle; the device
path must either prove a chunk decomposition or hand over to the host --
never return a different chain."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2209_12310_b200 as P
from conftest import ROOT

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    c = P.Context(0)
    yield c
    c.close()


def seq_chain(a):
    """The reference loop (hull.cpp:140-149) in Python doubles, last point dropped."""
    st = []
    for x, y in a.tolist():
        while len(st) >= 2:
            (ax, ay), (bx, by) = st[-2], st[-1]
            if (bx - ax) * (y - ay) - (by - ay) * (x - ax) > 0.0:
                break
            st.pop()
        st.append((x, y))
    return np.array(st[:-1], dtype=np.float64).reshape(-1, 2)


def host_cycle(arcs):
    dp = P._dp
    import ctypes as C
    out = []
    for a in arcs:
        a = np.ascontiguousarray(a, dtype=np.float64)
        o = np.empty_like(a)
        m = C.c_uint64()
        P.check(P.lib.ohx_chain(a.ctypes.data_as(dp), len(a), o.ctypes.data_as(dp), C.byref(m)))
        out.append(o[: m.value])
    return np.concatenate(out)


def host_hull(arcs):
    import ctypes as C
    dp = P._dp
    arcs = [np.ascontiguousarray(a, dtype=np.float64) for a in arcs]
    ptrs = (dp * 4)(*[a.ctypes.data_as(dp) for a in arcs])
    lens = (C.c_uint64 * 4)(*[len(a) for a in arcs])
    out = np.empty((sum(len(a) for a in arcs) + 8, 2))
    h = C.c_uint64()
    P.check(P.lib.ohx_hull_from_sorted_arcs(ptrs, lens, out.ctypes.data_as(dp), len(out),
                                            C.byref(h)))
    return out[: h.value]


def device_run(ctx, arcs, raw):
    allp = np.ascontiguousarray(np.concatenate(arcs), dtype=np.float64)
    d = torch.from_numpy(allp).cuda()
    return ctx.hull_from_sorted_arcs_device(d, [len(a) for a in arcs], raw_cycle=raw)


def arc_sequences(n=20000, seed=11):
    rng = np.random.default_rng(seed)
    seqs = {}
    # quadrant 1's sweep runs east -> north: x descending, CCW (a convex arc
    # turns left at every point); reversed, every point pops its predecessor
    t = np.sort(rng.uniform(0, np.pi / 2, n))
    seqs["convex"] = np.stack([np.cos(t), np.sin(t)], 1)
    seqs["reflex"] = seqs["convex"][::-1].copy()
    seqs["noisy_convex"] = np.stack([np.cos(t), np.sin(t)], 1) * (1 + rng.normal(0, 1e-3, (n, 1)))
    x = np.sort(rng.uniform(0, 1, n))[::-1]
    seqs["cloud"] = np.stack([x, rng.uniform(0, 1, n)], 1)
    z = np.arange(float(n))
    seqs["zigzag"] = np.stack([-z, (z % 2) * 3.0 + z * 1e-3], 1)
    seqs["blocks"] = np.stack([-z, np.where(z % 1000 < 500, 0.0, 1e6 - z)], 1)
    g = rng.integers(0, 30, size=(n, 2)).astype(float)
    seqs["grid"] = g[np.lexsort((g[:, 1], -g[:, 0]))]
    seqs["collinear"] = np.stack([-z, 2 * z], 1)
    w = np.cumsum(rng.normal(0, 1, (n, 2)), 0)
    seqs["walk"] = w[np.argsort(-w[:, 0], kind="stable")]
    # a long convex run, then a point that pops deep into earlier chunks
    tt = np.linspace(0.0, np.pi / 2, n)
    deep = np.stack([np.cos(tt), np.sin(tt)], 1)
    deep[n // 2] = (deep[n // 2, 0], 50.0)
    seqs["deep_pop"] = deep
    # rounding-level non-convexity everywhere (the circle's regime)
    tc = np.sort(rng.uniform(0, np.pi / 2, n))
    seqs["fp_circle"] = np.stack([np.cos(tc), np.sin(tc)], 1)
    return seqs


@pytest.mark.parametrize("name", list(arc_sequences(2000).keys()))
def test_device_chains_equal_the_reference_loop(ctx, name):
    a = arc_sequences()[name]
    small = [a[:2].copy(), a[:3].copy(), np.array([[0.0, 0.0], [1.0, 1.0]])]
    arcs = [a] + small
    cyc, proven = device_run(ctx, arcs, raw=True)
    want = np.concatenate([seq_chain(x) for x in arcs])
    assert np.array_equal(cyc, want), (name, proven)
    assert np.array_equal(host_cycle(arcs), want)
    if name in ("convex", "fp_circle"):
        assert proven, name  # these decompose: the device path must carry them


def fuzz_arc(rng, kind, n):
    """One sweep-ordered arc of quadrant 1 (x descending), of a given texture."""
    if kind == "noisy_circle":  # rounding-level to visible noise
        t = np.sort(rng.uniform(0, np.pi / 2, n))
        r = 1 + rng.normal(0, 10.0 ** rng.uniform(-16, -6), (n, 1))
        a = np.stack([np.cos(t), np.sin(t)], 1) * r
    elif kind == "grid":  # duplicates, collinear runs
        a = rng.integers(0, int(rng.integers(3, 60)), size=(n, 2)).astype(float)
    elif kind == "walk":
        a = np.cumsum(rng.normal(0, 1, (n, 2)), 0)
    elif kind == "crescent":  # a disk's survivor arc: thin band, many pops
        t = rng.uniform(0, np.pi / 2, n)
        r = 1 - rng.uniform(0, 0.02, (n, 1)) ** 2
        a = np.stack([np.cos(t), np.sin(t)], 1) * r
    else:  # "mixed": convex runs broken by outliers
        t = np.sort(rng.uniform(0, np.pi / 2, n))
        a = np.stack([np.cos(t), np.sin(t)], 1)
        k = rng.integers(0, n, size=max(1, n // 500))
        a[k] *= rng.uniform(0.5, 1.5, (len(k), 1))
    a = a[np.lexsort((a[:, 1], -a[:, 0]))]  # the sweep order (hull.cpp:18-22)
    return np.ascontiguousarray(a)


@pytest.mark.parametrize("seed", range(12))
def test_device_chains_fuzz(ctx, seed):
    # whatever the texture, the device path either proves its chunks and
    # returns the reference loop's chains, or hands over to the host chains
    rng = np.random.default_rng(1000 + seed)
    kinds = ["noisy_circle", "grid", "walk", "crescent", "mixed"]
    arcs = [fuzz_arc(rng, kinds[(seed + q) % len(kinds)], int(rng.integers(2, 9000)))
            for q in range(4)]
    cyc, proven = device_run(ctx, arcs, raw=True)
    assert np.array_equal(cyc, np.concatenate([seq_chain(x) for x in arcs])), proven
    hull, _ = device_run(ctx, arcs, raw=False)
    assert np.array_equal(hull, host_hull(arcs))


@pytest.mark.parametrize("n", [2, 3, 1023, 1024, 2047, 2048, 2049, 5000, 70001])
def test_device_chains_chunk_boundaries(ctx, n):
    rng = np.random.default_rng(n)
    t = np.sort(rng.uniform(0, np.pi / 2, n))
    arcs = []
    for q in range(4):
        r = 1.0 + rng.normal(0, 1e-12, (n, 1))
        arcs.append(np.stack([np.cos(t), np.sin(t)], 1) * r)
    cyc, proven = device_run(ctx, arcs, raw=True)
    want = np.concatenate([seq_chain(x) for x in arcs])
    assert np.array_equal(cyc, want)
    assert proven
    hull, _ = device_run(ctx, arcs, raw=False)
    assert np.array_equal(hull, host_hull(arcs))


def quadrant_arcs(oracle, pts):
    ext = oracle.find_extremes(pts)
    lab = oracle.classify(pts)
    anchors = pts[ext[:4].astype(np.int64)]
    arcs = []
    for q in range(4):
        arc = np.concatenate([anchors[q:q + 1], pts[lab == q + 1],
                              anchors[(q + 1) % 4:(q + 1) % 4 + 1]])
        x, y = arc[:, 0], arc[:, 1]
        keys = {0: (y, -x), 1: (-x, -y), 2: (-y, x), 3: (x, y)}[q]
        arcs.append(np.ascontiguousarray(arc[np.lexsort(keys)]))
    return arcs


@pytest.mark.parametrize("dist,n,seed,d", [("circle", 400_000, 3, 0.0), ("circle", 300_000, 4, 1.0),
                                           ("disk", 400_000, 5, 0.0), ("normal", 200_000, 6, 0.0)])
def test_device_hull_from_sorted_arcs_matches_oracle(ctx, oracle, dist, n, seed, d):
    pts = oracle.generate(dist, n, seed, d)
    arcs = quadrant_arcs(oracle, pts)
    hull, proven = device_run(ctx, arcs, raw=False)
    assert np.array_equal(hull, oracle.heaphull(pts)), (dist, proven)
    if dist == "circle" and d == 0.0:
        assert proven


def test_device_hull_general_cleanup(ctx, oracle):
    # duplicates / ties / a start vertex that is not the east anchor: the
    # device cycle goes through the host's general clean-up
    rng = np.random.default_rng(9)
    t = rng.uniform(0, 2 * np.pi, 120_000)
    cases = [np.round(np.stack([np.cos(t), np.sin(t)], 1) * 3000.0)]
    dd = oracle.generate("circle", 60_000, 8, 0.0) * 900.0
    dd[0], dd[5] = (1e3, 1.0), (1e3, -1.0)
    cases.append(dd)
    for pts in cases:
        pts = np.ascontiguousarray(pts)
        hull, _ = device_run(ctx, quadrant_arcs(oracle, pts), raw=False)
        assert np.array_equal(hull, oracle.heaphull(pts))


PIPE_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, ROOT_DIR); sys.path.insert(0, ROOT_DIR + "/tests")
import paper_2209_12310_b200 as P
from oracle import Oracle
o = Oracle(); ctx = P.Context(0)
for dist, n, seed, d, want_path in [("circle", 1_000_000, 3, 0.0, "device-chains"),
                                    ("circle", 1_000_000, 5, 2.0, None),
                                    ("disk", 2_000_000, 7, 0.0, None),
                                    ("normal", 300_000, 2, 0.0, "host")]:
    pts = P.generate(dist, n, seed, d)
    dx = torch.from_numpy(pts).cuda()
    hull, _ = ctx.heaphull_device(dx, n)
    info = ctx.last_run()
    assert np.array_equal(hull, o.heaphull(pts)), (dist, n, info)
    dh, _ = ctx.heaphull_device(dx, n, out="device")  # the hull left on the device
    assert dh.is_cuda and np.array_equal(dh.cpu().numpy(), hull), (dist, n)
    assert want_path is None or info["hull_path"] == want_path, info
    print(dist, n, info["hull_path"], len(hull))
print("pipeline ok")
"""


def test_pipeline_device_chains_match_oracle():
    env = dict(os.environ, OHX_DEVICE_SORT_MIN="100000")
    code = PIPE_SCRIPT.replace("ROOT_DIR", repr(ROOT))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       timeout=900)
    assert r.returncode == 0 and "pipeline ok" in r.stdout, r.stdout + r.stderr[-3000:]


def test_pipeline_device_chains_64bit_sort_tier():
    # OHX_HULL_SORT=u64 skips the sweep sort's 32-bit linear-key tier: the
    # 64-bit primary-key tier (and its 128-bit fallback) against the oracle
    env = dict(os.environ, OHX_DEVICE_SORT_MIN="100000", OHX_HULL_SORT="u64")
    code = PIPE_SCRIPT.replace("ROOT_DIR", repr(ROOT))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       timeout=900)
    assert r.returncode == 0 and "pipeline ok" in r.stdout, r.stdout + r.stderr[-3000:]


ROTATED_SCRIPT = r"""
import sys
sys.path.insert(0, ROOT_DIR)
import numpy as np, torch, paper_2209_12310_b200 as P
from oracle import Oracle
o = Oracle()
ctx = P.Context(0)
pts = P.generate("circle", 1_200_000, 8)
e = int(np.argmax(pts[:, 0]))
# a second point at the largest x, below the east extreme and with a larger
# index: it joins the S -> E arc and is the hull's first vertex (max x, then
# min y), so the chained cycle must be rotated
extra = np.array([[pts[e, 0], pts[e, 1] - 1e-7]])
pts = np.ascontiguousarray(np.concatenate([pts, extra]))
n = len(pts)
dx = torch.from_numpy(pts).cuda()
want = o.heaphull(pts)
assert want[0, 0] == pts[e, 0] and want[0, 1] == extra[0, 1], want[:2]
hull, _ = ctx.heaphull_device(dx, n)
assert np.array_equal(hull, want)
buf = torch.empty((n + 8, 2), dtype=torch.float64, device="cuda")
dh, _ = ctx.heaphull_device(dx, n, out=buf)  # the cycle written into buf, then rotated
info = ctx.last_run()
assert info["hull_path"] == "device-chains", info
assert np.array_equal(dh.cpu().numpy(), want)
print("rotated ok")
"""


def test_device_hull_rotated_into_caller_buffer():
    # the device hull stage writes its cycle straight into the caller's
    # device buffer; when the hull's first vertex is not the cycle's first
    # point the cycle is copied aside and rotated back into it
    env = dict(os.environ, OHX_DEVICE_SORT_MIN="100000")
    code = ROTATED_SCRIPT.replace("ROOT_DIR", repr(ROOT))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       timeout=600)
    assert r.returncode == 0 and "rotated ok" in r.stdout, r.stdout + r.stderr[-3000:]


PIPE_OUT_SCRIPT = r"""
import sys
sys.path.insert(0, ROOT_DIR)
import numpy as np, torch, paper_2209_12310_b200 as P
from oracle import Oracle
o = Oracle()
ctx = P.Context(0)
cases = []
pts = P.generate("circle", 5_000_000, 9)
cases.append(("circle", pts, "device-chains"))
e = int(np.argmax(pts[:, 0]))
extra = np.array([[pts[e, 0], pts[e, 1] - 1e-7]])  # the hull starts mid-cycle: a rotation
cases.append(("circle, rotated", np.ascontiguousarray(np.concatenate([pts, extra])), "device-chains"))
cases.append(("disk", P.generate("disk", 40_000_000, 3), None))  # chains unproven: regular stage
for name, pts, want_path in cases:
    n = len(pts)
    dx = torch.from_numpy(pts).cuda()
    out = torch.empty((n + 8, 2), dtype=torch.float64, pin_memory=True)
    hull, _ = ctx.heaphull_device(dx, n, out=out)
    info = ctx.last_run()
    want = o.heaphull(pts)
    assert np.array_equal(hull, want), (name, info)
    assert want_path is None or info["hull_path"] == want_path, (name, info)
    print(name, n, info["hull_path"], len(hull))
print("pipe ok")
"""


@pytest.mark.parametrize("pipe", ["1", "0"])
def test_pipelined_hull_stage_to_pinned_host_memory(pipe):
    # a large survivor set with the hull going to pinned host memory: arcs
    # sorted and chained one at a time, each arc's chain copied to the host
    # behind the next arc's work (OHX_HULL_PIPE=0: the regular stage)
    env = dict(os.environ, OHX_HULL_PIPE=pipe)
    code = PIPE_OUT_SCRIPT.replace("ROOT_DIR", repr(ROOT))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       timeout=900)
    assert r.returncode == 0 and "pipe ok" in r.stdout, r.stdout + r.stderr[-3000:]


PIPE_DEGEN_SCRIPT = r"""
import sys
sys.path.insert(0, ROOT_DIR)
import numpy as np, torch, paper_2209_12310_b200 as P
from oracle import Oracle
o = Oracle()
ctx = P.Context(0)
rng = np.random.default_rng(5)
for scale in (1000.0, 3e4, 1e7):
    t = rng.uniform(0, 2 * np.pi, 1_300_000)
    pts = np.ascontiguousarray(np.round(np.stack([np.cos(t), np.sin(t)], 1) * scale))
    n = len(pts)
    out = torch.empty((n + 8, 2), dtype=torch.float64, pin_memory=True)
    hull, _ = ctx.heaphull_device(torch.from_numpy(pts).cuda(), n, out=out)
    assert np.array_equal(hull, o.heaphull(pts)), (scale, ctx.last_run())
    print(scale, ctx.last_run()["hull_path"], len(hull))
print("degenerate pipe ok")
"""


def test_pipelined_hull_stage_on_degenerate_survivors():
    # duplicates, collinear runs and -0.0 through the pipelined stage (its
    # threshold lowered): the cycle statistics send these to the host
    # clean-up, from the copy already in the caller's buffer
    env = dict(os.environ, OHX_DEVICE_SORT_MIN="100000", OHX_HULL_PIPE_MIN="100000")
    code = PIPE_DEGEN_SCRIPT.replace("ROOT_DIR", repr(ROOT))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       timeout=900)
    assert r.returncode == 0 and "degenerate pipe ok" in r.stdout, r.stdout + r.stderr[-3000:]
