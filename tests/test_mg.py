"""The native multi-GPU layer (csrc/mg.cpp, ohx_mg_* over NCCL) on one
B200: a one-rank NCCL communicator with several virtual shards per device
runs the same per-shard pipeline, record all-gathers and survivor
gathers as separate GPUs would.  Every result must equal the single-device
pipeline and the oracle bit for bit."""

import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2209_12310_b200 as P
from conftest import ROOT
from paper_2209_12310_b200 import mg

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def handle():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    h = mg.MultiGPU.init_all([0])
    yield h
    h.close()


@pytest.mark.parametrize("dist,n,seed,d", [
    ("normal", 20_000_000, 7, 0.0),   # fused pass on every shard
    ("square", 12_000_000, 3, 0.0),
    ("circle", 1_000_000, 5, 0.0),    # all survive, the corner certificate fails
    ("disk", 3_000_000, 2, 0.0),
    ("circle", 400_000, 9, 2.0)])
@pytest.mark.parametrize("shards", [1, 2, 3, 7])
def test_virtual_shards_match_single_device(handle, oracle, dist, n, seed, d, shards):
    pts = P.generate(dist, n, seed, d)
    dd = torch.from_numpy(pts).cuda()
    ctx = P.Context(0)
    want, _ = ctx.heaphull_device(dd, n)
    hull, info = handle.heaphull_device(
        [(dd.data_ptr() + 16 * (n * j // shards), n * (j + 1) // shards - n * j // shards)
         for j in range(shards)])
    assert np.array_equal(hull, want)
    assert info["shards"] == shards and info["n_total"] == n
    assert info["ext"] == [int(v) for v in P.find_extremes(pts)]
    assert info["counts"] == ctx.last_run()["counts"]
    if n <= 3_000_000:
        assert np.array_equal(hull, oracle.heaphull(pts))


def test_ties_across_shard_seams(handle, oracle):
    # duplicates of every extreme in every shard: ties must go to the
    # smallest global index across shards
    rng = np.random.default_rng(3)
    base = (rng.integers(-6, 7, size=(5000, 2)) / 3.0).astype(float)
    pts = np.concatenate([base] * 6)
    dd = torch.from_numpy(pts).cuda()
    n = len(pts)
    for shards in (2, 5, 6):
        hull, info = handle.heaphull_device(
            [(dd.data_ptr() + 16 * (n * j // shards), n * (j + 1) // shards - n * j // shards)
             for j in range(shards)])
        assert np.array_equal(hull, oracle.heaphull(pts))
        assert info["ext"] == [int(v) for v in oracle.find_extremes(pts)]


def test_host_points_with_labels(handle, oracle):
    pts = P.generate("disk", 2_000_001, 11)
    hull, info, labels = handle.heaphull(pts, vshards=3, labels=True)
    want_hull, want = oracle.heaphull(pts, with_labels=True)
    assert np.array_equal(hull, want_hull)
    assert np.array_equal(labels, want)
    assert info["counts"] == [int((want == q).sum()) for q in (1, 2, 3, 4)]


def test_one_rank_communicator_shard_call():
    # the one-process-per-GPU entry (ohx_mg_init_rank) as a world of 1
    # 4 shards of 10M points: each above the fused pass's 2^23-point floor
    pts = P.generate("normal", 40_000_000, 9)
    dd = torch.from_numpy(pts).cuda()
    h = mg.MultiGPU.init_rank(mg.unique_id(), 1, 0, 0)
    try:
        assert h.world == 1 and h.local_ranks == 1
        for vs in (1, 4):
            hull, info = h.heaphull_shard(dd, len(pts), 0, vshards=vs)
            assert np.array_equal(hull, P.heaphull(pts))
            assert info["fused_shards"] == vs
        # per-shard contexts: counters and run info of the last call
        c = h.shard_context(0, 3)
        assert c.launches > 0 and c.last_run()["fused"]
    finally:
        h.close()


def test_empty_and_bad_calls(handle):
    dd = torch.zeros((4, 2), dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        handle.heaphull_device([(dd.data_ptr(), 0)])
    with pytest.raises(ValueError):
        handle.heaphull(np.zeros((0, 2)))


@pytest.mark.parametrize("suite", ["hull", "filter", "bench"])
def test_reference_suites_through_the_mg_layer(suite):
    # the reference's own suites with every heaphull / heaphull_run routed
    # through the NCCL layer (OHX_MG_VSHARDS=3: three shards on this GPU)
    path = os.path.join(ROOT, "oracle", "_ref", "reftests", f"test_{suite}")
    if not os.path.exists(path):
        pytest.skip("reference suites not built")
    r = subprocess.run([path], capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, OHX_MG_VSHARDS="3"))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_bench_through_the_mg_layer():
    # bench.py's N > 1 step shape (native NCCL layer) at N = 1 with 2 shards
    import json
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--points", "2e7",
                        "--steps", "3", "--warmup", "3", "--mg-vshards", "2", "--no-cpu",
                        "--no-dists"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["run"]["path"].startswith("ohx_mg_heaphull_shard")
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
