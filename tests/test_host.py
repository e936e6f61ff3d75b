"""CPU-side tests of the product library (no GPU needed): the C ABI loads and
exports everything include/ohx.h declares, the host stages between and after
the kernels (generator, extremes combine + corner certificate, build_octagon,
the K2 plan and its certified box, the host hull) match the oracle, and the
device entry points fail loudly when there is no GPU."""

import os
import re

import numpy as np
import pytest

import paper_2209_12310_b200 as P
from paper_2209_12310_b200 import _lib
from conftest import ROOT, sha
from emulate import emulate_corners, emulate_k1


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ohx.h")).read()
    return sorted(set(re.findall(r"\b(ohx_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (ohx_\w+)", out))
    declared = declared_symbols()
    assert len(declared) >= 25
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    # and the ctypes stub binds every one of them
    bound = {name for name, _, _ in _lib.PROTOTYPES}
    assert set(declared) <= bound
    assert P.lib.ohx_abi_version() == 1


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


@pytest.mark.parametrize("dist,n,seed,d", [
    ("normal", 1, 0, 0.0), ("normal", 300001, 9, 0.0), ("square", 262145, 4, 0.0),
    ("disk", 300000, 5, 0.0), ("circle", 300000, 6, 3.5), ("circle", 70000, 6, 0.0)])
def test_generator_bit_exact(oracle, dist, n, seed, d):
    a = P.generate(dist, n, seed, d)
    assert np.array_equal(a, oracle.generate(dist, n, seed, d))
    assert np.array_equal(a, P.generate(dist, n, seed, d, threads=3))


@pytest.mark.parametrize("dist,d", [("normal", 0.0), ("square", 0.0), ("disk", 0.0),
                                    ("circle", 2.0)])
def test_generator_range_is_a_slice_of_the_corpus(oracle, dist, d):
    # a shard's slice (bench.py at N > 1: rank r generates only its range
    # of generate({dist, n_total, seed}))
    n = 1_000_003
    whole = oracle.generate(dist, n, 11, d)
    for lo, cnt in [(0, 1), (0, n), (1, 262144), (333_333, 333_334), (n - 5, 5), (n, 0)]:
        got = P.generate_range(dist, n, lo, cnt, 11, d, threads=4)
        assert np.array_equal(got, whole[lo: lo + cnt]), (lo, cnt)
    with pytest.raises(ValueError):
        P.generate_range(dist, n, n - 1, 2, 11, d)


def test_generator_errors():
    with pytest.raises(ValueError):
        P.generate("triangle", 10)
    with pytest.raises(ValueError):
        P.generate("normal", 10, distort=2.0)
    with pytest.raises(ValueError):
        P.generate("circle", 10, distort=-1.0)
    with pytest.raises(ValueError):
        P.generate("normal", 0)


def test_monotone_chain_matches_oracle(oracle, golden):
    for c in golden["cases"][:12]:
        pts = oracle.generate(c["dist"], c["n"], c["seed"], c["distort"])
        assert np.array_equal(P.monotone_chain(pts), oracle.monotone_chain(pts))


# ---------------------------------------------------------------- host hull
def hull_via_library(oracle, pts):
    """Oracle labels -> queues -> the product's host hull stage."""
    ext = oracle.find_extremes(pts)
    lab = oracle.classify(pts)
    anchors = pts[ext[:4].astype(np.int64)]
    queues = [pts[np.flatnonzero(lab == q)] for q in (1, 2, 3, 4)]
    return P.hull_from_queue_points(anchors, queues)


def test_host_hull_matches_oracle_on_golden(oracle, golden):
    for c in golden["cases"]:
        pts = oracle.generate(c["dist"], c["n"], c["seed"], c["distort"])
        hull = hull_via_library(oracle, pts)
        assert len(hull) == c["h"] and sha(hull) == c["hull_sha256"], c


def test_host_hull_matches_oracle_on_degenerate_grids(oracle, grid_trials):
    for t in grid_trials:
        a = np.array(t["pts"], dtype=float)
        assert hull_via_library(oracle, a).tolist() == t["hull"]


def test_host_hull_large_degenerate_sets(oracle):
    # sizes past the parallel thresholds of the host hull stage (compaction,
    # collinearity reduction, the scan-skipping peel) on inputs full of
    # duplicates, collinear runs and non-strict seams
    rng = np.random.default_rng(5)
    cases = []
    for g in (3, 7, 40, 1000):
        cases.append(rng.integers(0, g, size=(150_000, 2)).astype(float))
    t = rng.uniform(0, 2 * np.pi, 200_000)
    for scale in (50.0, 3000.0):  # circle points snapped to a grid: collinear chords
        cases.append(np.round(np.stack([np.cos(t), np.sin(t)], 1) * scale))
    line = np.stack([np.arange(100_000.0), 2 * np.arange(100_000.0)], 1)
    cases.append(np.concatenate([line, line[::-1]]))  # fully collinear
    # mid-sized arcs (the radix sweep sort): duplicates and +/-0.0 ties
    for g in (5, 60):
        cases.append(rng.integers(-g, g + 1, size=(20_000, 2)).astype(float) * 0.5)
    t2 = rng.uniform(0, 2 * np.pi, 30_000)
    cases.append(np.round(np.stack([np.cos(t2), np.sin(t2)], 1) * 400.0))
    # coordinates that differ only below the radix passes' top 33 key bits
    # (the comparator orders those runs)
    cases.append(1.0 + rng.integers(0, 3000, size=(20_000, 2)) * 2.0 ** -40)
    cases.append(-1.0 - rng.uniform(0, 2.0 ** -25, size=(20_000, 2)))
    for a in cases:
        a = np.ascontiguousarray(a)
        assert np.array_equal(hull_via_library(oracle, a), oracle.heaphull(a))


# ------------------------------------------------- extremes combine + cert
def resolve_like_pipeline(pts, shards):
    """Shard -> K1 records -> combine -> certificate -> (exact corners)."""
    bounds = np.linspace(0, len(pts), shards + 1).astype(int)
    recs = [emulate_k1(pts[b0:b1], b0) for b0, b1 in zip(bounds[:-1], bounds[1:]) if b1 > b0]
    g = P.combine_extremes(recs)
    ext, mask = P.resolve_extremes(g)
    if mask:
        bbox = (g.x[0], g.y[1], g.x[2], g.y[3])
        crecs = [emulate_corners(pts[b0:b1], bbox, b0)
                 for b0, b1 in zip(bounds[:-1], bounds[1:]) if b1 > b0]
        ext = P.apply_corners(ext, P.combine_corners(crecs))
    return [int(v) for v in ext.ext], mask


@pytest.mark.parametrize("shards", [1, 2, 3, 8])
def test_certificate_and_combine_match_reference_extremes(oracle, golden, shards):
    for c in golden["cases"]:
        if c["n"] > 300000:
            continue
        pts = oracle.generate(c["dist"], c["n"], c["seed"], c["distort"])
        got, _ = resolve_like_pipeline(pts, shards)
        assert got == c["ext"], c


def test_certificate_on_degenerate_grids(grid_trials):
    uncertified = 0
    for t in grid_trials[:2000]:
        a = np.array(t["pts"], dtype=float)
        got, mask = resolve_like_pipeline(a, 1 + len(a) % 3)
        uncertified += mask != 0
        assert got == t["ext"]
    assert uncertified > 0  # ties on grids must exercise the exact fallback


def test_certificate_never_certifies_a_wrong_corner(oracle):
    # adversarial near-ties: points on a line x + y = const, perturbed by ulps
    rng = np.random.default_rng(1)
    for trial in range(200):
        n = 50
        base = rng.uniform(-1e3, 1e3)
        x = rng.uniform(-1, 1, n) * 10.0 ** rng.integers(-3, 4)
        y = base - x
        y = y + rng.integers(-3, 4, n) * np.spacing(np.abs(y) + 1e-300)
        pts = np.stack([x, y], axis=1)
        ext, mask = resolve_like_pipeline(pts, 1)
        assert ext == [int(v) for v in oracle.find_extremes(pts)]


# ----------------------------------------------------- octagon and K2 plan
def test_build_octagon_matches_oracle(oracle, golden, grid_trials):
    for c in golden["cases"]:
        pts = oracle.generate(c["dist"], c["n"], c["seed"], c["distort"])
        rec = emulate_k1(pts)
        ext, _ = P.resolve_extremes(rec)
        for k in range(8):  # use the reference's extremes
            j = c["ext"][k]
            ext.ext[k], ext.x[k], ext.y[k] = j, pts[j, 0], pts[j, 1]
        assert P.build_octagon_from_set(ext).tolist() == c["octagon"]
    for t in grid_trials[:500]:
        a = np.array(t["pts"], dtype=float)
        ext = _lib.ExtremeSet()
        for k, j in enumerate(t["ext"]):
            ext.ext[k], ext.x[k], ext.y[k] = j, a[j, 0], a[j, 1]
        e = np.array(t["ext"], dtype=np.uint64)
        assert np.array_equal(P.build_octagon_from_set(ext), oracle.build_octagon(a, e))


def orientation(a, b, c):
    det = (b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0])
    return int(det > 0) - int(det < 0)


def test_certified_box_is_strictly_inside(oracle):
    rng = np.random.default_rng(3)
    for dist, n, seed, d in [("normal", 100000, 7, 0.0), ("square", 100000, 7, 0.0),
                             ("disk", 100000, 7, 0.0), ("circle", 20000, 7, 5.0)]:
        pts = oracle.generate(dist, n, seed, d)
        e = oracle.find_extremes(pts)
        octg = oracle.build_octagon(pts, e)
        ext = _lib.ExtremeSet()
        for k, j in enumerate(e):
            ext.ext[k], ext.x[k], ext.y[k] = int(j), pts[j, 0], pts[j, 1]
        plan = P.make_plan(ext, octg)
        x0, x1, y0, y1 = plan.box
        assert x0 < x1 and y0 < y1, dist
        # corners, edges of the box and random interior points: every
        # reference orientation strictly positive
        xs = np.concatenate([[x0, x1], rng.uniform(x0, x1, 300)])
        ys = np.concatenate([[y0, y1], rng.uniform(y0, y1, 300)])
        m = len(octg)
        for px in xs[:40]:
            for py in ys[:40]:
                for i in range(m):
                    assert orientation(octg[i], octg[(i + 1) % m], (px, py)) == 1
        # plan edge constants are the reference's (b - a) differences
        for i in range(m):
            b = octg[(i + 1) % m]
            assert plan.ea[i] == b[0] - octg[i][0] and plan.ec[i] == b[1] - octg[i][1]
        # coverage: the box must catch most interior points of these corpora
        inside = ((pts[:, 0] >= x0) & (pts[:, 0] <= x1) & (pts[:, 1] >= y0) & (pts[:, 1] <= y1))
        floor = {"normal": 0.99, "square": 0.9, "disk": 0.6}.get(dist, 0.0)
        assert inside.mean() > floor, (dist, inside.mean())


def test_device_entry_points_fail_loudly_without_gpu():
    if P.device_count() if _has_driver() else 0:
        pytest.skip("a GPU is visible")
    pts = P.generate("normal", 100, 1)
    with pytest.raises(RuntimeError):
        P.heaphull(pts)
    with pytest.raises(RuntimeError):
        P.classify(pts)
    with pytest.raises(RuntimeError):
        P.Context(0)


def _has_driver():
    try:
        P.device_count()
        return True
    except RuntimeError:
        return False


def test_bad_input_raises_value_error():
    # tests/python/test_smoke.py:54-60
    with pytest.raises(ValueError):
        P.heaphull(np.zeros((3, 3)))
    with pytest.raises(ValueError):
        P.heaphull(np.array([[0.0, np.nan]]))
    with pytest.raises(ValueError):
        P.heaphull(np.zeros((0, 2)))
    with pytest.raises(ValueError):
        P.classify(np.zeros((4, 2)), threads=0)


# ------------------------------------------------------------ PTS2 files
def test_pts2_header_validation(tmp_path, oracle):
    import ctypes as C
    pts = oracle.generate("disk", 1000, 3)
    f = tmp_path / "p.bin"
    P.write_pts2(pts, f)
    assert f.stat().st_size == 12 + 16 * 1000
    n = C.c_uint64(0)
    P.check(P.lib.ohx_pts2_count(os.fsencode(f), C.byref(n)))
    assert n.value == 1000
    cases = {b"XXXX" + (3).to_bytes(8, "little"): "magic",
             b"PTS2" + (0).to_bytes(8, "little"): "empty",
             b"PTS2" + (2).to_bytes(8, "little") + b"\0" * 27: "size mismatch",
             b"PTS2": "truncated header"}
    for raw, what in cases.items():
        f.write_bytes(raw)
        assert P.lib.ohx_pts2_count(os.fsencode(f), C.byref(n)) == _lib.OHX_E_IO
        assert what in P.lib.ohx_last_error().decode()
    assert P.lib.ohx_pts2_count(os.fsencode(tmp_path / "nope.bin"), C.byref(n)) == _lib.OHX_E_IO
    assert "nope.bin" in P.lib.ohx_last_error().decode()


@pytest.mark.parametrize("chunks", ["2", "7", "64"])
def test_parallel_chain_matches_the_sequential_loop(chunks):
    # the host hull tests again with every arc of >= 64 points chained in
    # parallel chunks (OHX_CHAIN_PAR_MIN / OHX_CHAIN_CHUNKS test hooks):
    # golden corpora, the reference's degenerate grids, large degenerate sets
    import subprocess
    import sys
    env = dict(os.environ, OHX_CHAIN_PAR_MIN="64", OHX_CHAIN_CHUNKS=chunks)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_host.py"), "-k",
                        "host_hull and not parallel_chain"],
                       capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


CHAIN_SCRIPT = r"""
import sys, numpy as np, ctypes as C
sys.path.insert(0, ROOT_DIR)
import paper_2209_12310_b200 as P
dp = C.POINTER(C.c_double)

def seq_chain(a):  # the reference loop (hull.cpp:140-149), Python doubles
    st = []
    for x, y in a.tolist():
        while len(st) >= 2:
            (ax, ay), (bx, by) = st[-2], st[-1]
            if (bx - ax) * (y - ay) - (by - ay) * (x - ax) > 0.0:
                break
            st.pop()
        st.append((x, y))
    return np.array(st[:-1], dtype=np.float64).reshape(-1, 2)

def lib_chain(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    out = np.empty_like(a); m = C.c_uint64()
    P.check(P.lib.ohx_chain(a.ctypes.data_as(dp), len(a), out.ctypes.data_as(dp), C.byref(m)))
    return out[: m.value]

rng = np.random.default_rng(11)
seqs = []
t = np.sort(rng.uniform(0, np.pi / 2, 20000))[::-1]          # convex arc (nearly no pops)
seqs.append(np.stack([np.cos(t), np.sin(t)], 1))
seqs.append(np.stack([np.cos(t), np.sin(t)], 1) * (1 + rng.normal(0, 1e-3, (20000, 1))))
x = np.sort(rng.uniform(0, 1, 20000))[::-1]                   # random cloud, many pops
seqs.append(np.stack([x, rng.uniform(0, 1, 20000)], 1))
z = np.arange(20000.0)                                        # zigzag: pops across chunks
seqs.append(np.stack([-z, (z % 2) * 3.0 + z * 1e-3], 1))
seqs.append(np.stack([-z, np.where(z % 1000 < 500, 0.0, 1e6 - z)], 1))
g = rng.integers(0, 30, size=(20000, 2)).astype(float)        # grid: duplicates, collinear
seqs.append(g[np.lexsort((g[:, 1], -g[:, 0]))])
line = np.stack([-z, 2 * z], 1)                               # collinear
seqs.append(line)
w = np.cumsum(rng.normal(0, 1, (20000, 2)), 0)               # random walk
seqs.append(w[np.argsort(-w[:, 0], kind="stable")])
bad = 0
for a in seqs:
    a = np.ascontiguousarray(a)
    if not np.array_equal(lib_chain(a), seq_chain(a)):
        bad += 1
print("chains ok" if bad == 0 else f"{bad} mismatches")
"""


@pytest.mark.parametrize("chunks", ["2", "5", "16", "300"])
def test_parallel_chain_equals_the_reference_loop_directly(chunks):
    import subprocess
    import sys
    env = dict(os.environ, OHX_CHAIN_PAR_MIN="64", OHX_CHAIN_CHUNKS=chunks)
    code = CHAIN_SCRIPT.replace("ROOT_DIR", repr(ROOT))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       timeout=900)
    assert r.returncode == 0 and "chains ok" in r.stdout, r.stdout + r.stderr[-3000:]


SORTED_ARCS_SCRIPT = r"""
import sys, numpy as np, ctypes as C
sys.path.insert(0, ROOT_DIR)
sys.path.insert(0, ROOT_DIR + "/tests")
import paper_2209_12310_b200 as P
from oracle import Oracle
dp = C.POINTER(C.c_double)
o = Oracle()

def sweep_sorted(a, q):  # the reference comparator's order (hull.cpp:18-30)
    x, y = a[:, 0], a[:, 1]
    keys = {1: (y, -x), 2: (-x, -y), 3: (-y, x), 4: (x, y)}[q]
    return np.ascontiguousarray(a[np.lexsort(keys)])

def lib_hull(pts, cap=None, rc_want=0):
    ext = o.find_extremes(pts)
    lab = o.classify(pts)
    anchors = pts[ext[:4].astype(np.int64)]
    arcs = []
    for q in range(4):
        arc = np.concatenate([anchors[q:q + 1], pts[lab == q + 1], anchors[(q + 1) % 4:(q + 1) % 4 + 1]])
        arcs.append(sweep_sorted(arc, q + 1))
    ptrs = (dp * 4)(*[a.ctypes.data_as(dp) for a in arcs])
    lens = (C.c_uint64 * 4)(*[len(a) for a in arcs])
    out = np.empty((sum(len(a) for a in arcs) + 8, 2)); h = C.c_uint64()
    rc = P.lib.ohx_hull_from_sorted_arcs(ptrs, lens, out.ctypes.data_as(dp),
                                         len(out) if cap is None else cap, C.byref(h))
    if rc_want:
        assert rc == rc_want, rc
        return h.value
    P.check(rc)
    return out[: h.value]

rng = np.random.default_rng(9)
cases = [o.generate("circle", 200_000, 3, 0.0), o.generate("circle", 150_000, 4, 1.0),
         o.generate("disk", 200_000, 5, 0.0), o.generate("normal", 100_000, 6, 0.0)]
t = rng.uniform(0, 2 * np.pi, 120_000)
cases.append(np.round(np.stack([np.cos(t), np.sin(t)], 1) * 300.0))      # duplicates, ties
cases.append(rng.integers(-9, 10, size=(50_000, 2)).astype(float))       # degenerate grid
d = o.generate("disk", 50_000, 8, 0.0) * 900.0   # two east-most points: the start vertex is
d[0], d[5] = (1e3, 1.0), (1e3, -1.0)              # not the east anchor (smallest index)
cases.append(d)
bad = sum(not np.array_equal(lib_hull(np.ascontiguousarray(a)), o.heaphull(np.ascontiguousarray(a)))
          for a in cases)
# the output buffer sized to the hull exactly (smaller than the chained
# cycle when the clean-up drops vertices), and one vertex short
for a in cases:
    a = np.ascontiguousarray(a)
    want = o.heaphull(a)
    bad += not np.array_equal(lib_hull(a, cap=len(want)), want)
    bad += lib_hull(a, cap=len(want) - 1, rc_want=P.OHX_E_INVALID) != len(want)
print("arcs ok" if bad == 0 else f"{bad} mismatches")
"""


@pytest.mark.parametrize("par_min,chunks", [("1000000000", "16"), ("64", "3"), ("64", "16")])
def test_hull_from_sorted_arcs_matches_oracle(par_min, chunks):
    # the device-sort path's host half (chains, piece-cycle clean-up and the
    # single rotated copy) on arcs sorted here, sequential and chunked chains
    import subprocess
    import sys
    env = dict(os.environ, OHX_CHAIN_PAR_MIN=par_min, OHX_CHAIN_CHUNKS=chunks)
    code = SORTED_ARCS_SCRIPT.replace("ROOT_DIR", repr(ROOT))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       timeout=900)
    assert r.returncode == 0 and "arcs ok" in r.stdout, r.stdout + r.stderr[-3000:]


def test_host_hull_workers_survive_fork(oracle):
    # the arc workers and the OpenMP pool are process-local: a forked child
    # runs single-threaded (no hang waiting for threads it does not have),
    # with the same results
    import subprocess
    import sys
    code = (
        "import os, sys, numpy as np\n"
        f"sys.path.insert(0, {ROOT!r}); sys.path.insert(0, {ROOT!r} + '/tests')\n"
        "import paper_2209_12310_b200 as P\n"
        "from oracle import Oracle\n"
        "o = Oracle()\n"
        "pts = o.generate('disk', 400_000, 5, 0.0)\n"
        "ext = o.find_extremes(pts); lab = o.classify(pts)\n"
        "anchors = pts[ext[:4].astype(np.int64)]\n"
        "queues = [pts[np.flatnonzero(lab == q)] for q in (1, 2, 3, 4)]\n"
        "assert sum(len(q) for q in queues) >= 4096\n"
        "want = P.hull_from_queue_points(anchors, queues)\n"
        "t = np.random.default_rng(1).uniform(0, 2 * np.pi, 600_000)\n"
        "circ = np.ascontiguousarray(np.stack([np.cos(t), np.sin(t)], 1))\n"
        "mc = P.monotone_chain(circ)  # parallel sort + OpenMP clean-up in the parent\n"
        "pid = os.fork()\n"
        "if pid == 0:\n"
        "    got = P.hull_from_queue_points(anchors, queues)\n"
        "    ok = np.array_equal(got, want) and np.array_equal(P.monotone_chain(circ), mc)\n"
        "    os._exit(0 if ok else 3)\n"
        "_, st = os.waitpid(pid, 0)\n"
        "assert os.WEXITSTATUS(st) == 0, st\n"
        "assert np.array_equal(P.hull_from_queue_points(anchors, queues), want)\n"
        "print('fork ok')\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "fork ok" in r.stdout, r.stdout + r.stderr[-3000:]
