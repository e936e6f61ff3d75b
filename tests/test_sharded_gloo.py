"""The multi-GPU orchestration (paper_2209_12310_b200/sharded.py) on CPU:
world_size 2 (and 3) over gloo, every rank owning a contiguous index range,
the per-shard kernels emulated with reference semantics (tests/emulate.py).
The sharded result must equal the single-process oracle bit for bit."""

import os
import socket
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))

CORPORA = [("normal", 20000, 7, 0.0), ("circle", 3000, 12, 2.0), ("square", 5001, 3, 0.0),
           ("disk", 4000, 55, 0.0)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, HERE)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from emulate import EmulatedShard
    from oracle import Oracle
    from paper_2209_12310_b200.sharded import shard_range, sharded_heaphull

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = Oracle()
        out = []
        cases = CORPORA + [("grid", 0, 0, 0.0)]
        for dist_name, n, seed, d in cases:
            if dist_name == "grid":  # ties and duplicates across the shard seam
                rng = np.random.default_rng(1)
                pts = (rng.integers(-3, 4, size=(61, 2)) / 2.0).astype(float)
            else:
                pts = o.generate(dist_name, n, seed, d)
            b0, cnt = shard_range(len(pts), world, rank)
            stats = {}
            hull = sharded_heaphull(EmulatedShard(o, pts, b0, cnt), device="cpu", stats=stats)
            if rank == 0:
                want, labels = o.heaphull(pts, with_labels=True)
                out.append((dist_name, hull.tolist() == want.tolist(),
                            stats["ext"] == [int(v) for v in o.find_extremes(pts)],
                            stats["n_total"] == len(pts)))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_pipeline_matches_oracle(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for name, hull_ok, ext_ok, n_ok in res:
        assert hull_ok and ext_ok and n_ok, name


def _gpu_worker(rank, world, port, q):
    sys.path.insert(0, os.path.dirname(HERE))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import paper_2209_12310_b200 as P
    from oracle import Oracle
    from paper_2209_12310_b200.sharded import (CudaShard, shard_range, sharded_heaphull,
                                               sharded_hull_indices)

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = Oracle()
        ctx = P.Context(0)
        out = []
        for dist_name, n, seed in [("normal", 24_000_000, 5), ("square", 20_000_000, 8),
                                   ("disk", 3_000_000, 2)]:
            pts = P.generate(dist_name, n, seed)
            b0, cnt = shard_range(n, world, rank)
            d = torch.from_numpy(pts[b0:b0 + cnt]).cuda()
            stats = {}
            shard = CudaShard(ctx, d, cnt, b0)
            hull = sharded_heaphull(shard, device="cpu", stats=stats)
            idx = sharded_hull_indices(shard, hull, device="cpu")
            if rank == 0:
                want = o.heaphull(pts)
                ok = hull.tolist() == want.tolist()
                # vertex indices: the smallest global index with the vertex's
                # coordinates (brute force over the whole input)
                for v, j in zip(hull, idx):
                    ok = ok and int(j) == int(np.flatnonzero((pts[:, 0] == v[0]) &
                                                             (pts[:, 1] == v[1]))[0])
                out.append((dist_name, ok, stats["fused"]))
        if rank == 0:
            q.put(out)
        ctx.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_cuda_shards_over_gloo_on_one_gpu():
    # the real per-shard backend (CudaShard: fused pass on each shard's own
    # sample, filter_fused against the global plan) in 2 processes sharing
    # cuda:0, exchanging records and survivors over gloo
    import torch
    if not torch.cuda.is_available():
        pytest.fail("needs a CUDA device")
    import torch.multiprocessing as mp
    mctx = mp.get_context("spawn")
    q = mctx.Queue()
    port = _free_port()
    procs = [mctx.Process(target=_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for name, hull_ok, fused in res:
        assert hull_ok, name
    assert [fused for _, _, fused in res] == [True, True, False]


@pytest.mark.gpu
def test_bench_multi_rank_path_on_one_gpu(tmp_path):
    # bench.py's N > 1 code path (barriers, max over ranks, sharded fused
    # pipeline, e2e with per-rank H2D) as 2 torchrun ranks sharing cuda:0;
    # OHX_BENCH_BACKEND=gloo only swaps the collective backend
    import json
    import subprocess
    root = os.path.dirname(HERE)
    env = dict(os.environ, OHX_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(root, "bench.py"), "--gpus", "2", "--points-total", "2.4e7", "--steps", "3",
           "--warmup", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["config"]["points_total"] == 24_000_000
    assert line["scaling"] == "strong" and line["config"]["points_per_gpu"] == 12_000_000
    assert line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
    par = line["parity"]  # the 2-rank job against the reference on the whole corpus
    assert par["hull_equal"] and par["extremes_equal"] and par["queues_equal"], par
