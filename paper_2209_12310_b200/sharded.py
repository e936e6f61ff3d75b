"""Multi-GPU heaphull over index-range shards.

One process per GPU (torch.distributed; NCCL on GPUs, gloo in the CPU
tests).  Rank r owns the contiguous global index range
[base_r, base_r + n_r); indices stay global, so the smallest-index tie rule
of the reference (parallel.hpp:34-43) holds across shards.

  1. K1 on every shard                       -> one ~300 B extremes record
     (or the fused pass: KF streams the shard once against a provisional
     region fitted on the shard's own sample and K1 runs on the points
     outside it -- the same record from one read)
  2. all_gather of the records + the same associative combine on every rank
     (NCCL has no arg-min over (f64, u64) pairs; the combine is exact and
     order-independent, so every rank derives the identical ExtremeSet)
  3. corner certificate; only if it fails: K1b per shard + all_gather
  4. build_octagon + K2 plan (host, identical on every rank)
  5. K2 on every shard -> four index-ordered queues per shard (fused: on the
     shard's candidates only, once its region is certified inside the
     global octagon)
  6. survivor coordinates sent to the root only, in rank order (= global
     index order, so the concatenation equals build_queues of the whole)
  7. the root runs the host hull stage (reference semantics) on them.

The only exchanges are those small collectives and the survivors' trip to
the root: the data path itself is never communicated.  This is the
torch.distributed rendering of the protocol (gloo in the CPU tests, ranks
sharing one GPU); the production multi-GPU path is the native NCCL layer
behind the C ABI (csrc/mg.cpp, ohx_mg_*), which runs the same steps with
the survivors moving device to device.  The per-shard compute sits behind a tiny interface
(`extremes`, `corners_exact`, `filter`, `queue_xy`) implemented here by
`CudaShard` over the C ABI; the CPU tests plug in an emulated shard to
exercise the orchestration with world_size 2 over gloo.
"""

from __future__ import annotations

import numpy as np

from . import (CornerRec, ExtremesRec, apply_corners, build_octagon_from_set,
               combine_corners, combine_extremes, hull_from_queue_points, make_plan,
               resolve_extremes)


class CudaShard:
    """A shard of device-resident points on one GPU (the product backend)."""

    def __init__(self, ctx, d_xy, n: int, base: int):
        self.ctx, self.d_xy, self.n, self.base = ctx, d_xy, int(n), int(base)
        self.counts = None

    def extremes(self) -> ExtremesRec:
        return self.ctx.extremes(self.d_xy, self.n, self.base)

    def fused_extremes(self):
        return self.ctx.fused_extremes(self.d_xy, self.n, self.base)

    def filter_fused(self, ext, plan):
        self.counts, _ = self.ctx.filter_fused(self.d_xy, self.n, ext, plan, self.base)
        return self.counts

    def corners_exact(self, bbox) -> CornerRec:
        return self.ctx.corners_exact(self.d_xy, self.n, bbox, self.base)

    def filter(self, plan):
        self.counts = self.ctx.filter(self.d_xy, self.n, plan, self.base)
        return self.counts

    def hull_indices(self, hull) -> np.ndarray:
        """This shard's part of the hull vertex indices (-1: none here)."""
        return self.ctx.hull_indices(hull, partial=True)

    def queue_xy(self, q: int, count: int) -> np.ndarray:
        if count == 0:
            return np.zeros((0, 2), dtype=np.float64)
        return self.ctx.queue(q, count, with_idx=False, with_xy=True)[1]


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def _allgather_structs(obj, cls, device):
    """all_gather of a ctypes struct as raw bytes -> list of structs."""
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return [obj]
    import torch
    raw = torch.frombuffer(bytearray(bytes(obj)), dtype=torch.uint8).to(device)
    out = [torch.empty_like(raw) for _ in range(dist.get_world_size())]
    dist.all_gather(out, raw)
    return [cls.from_buffer_copy(t.cpu().numpy().tobytes()) for t in out]


def _gather_queues(queues, device, root):
    """Survivor coordinates of the 4 queues from every rank to `root` only
    (exact-size point-to-point sends after an all-gather of the 4 queue
    lengths), concatenated per quadrant in rank order.  Returns the 4
    arrays on `root`, None elsewhere."""
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return queues
    import torch
    world, rank = dist.get_world_size(), dist.get_rank()
    counts = torch.tensor([len(q) for q in queues], dtype=torch.int64, device=device)
    all_counts = [torch.empty_like(counts) for _ in range(world)]
    dist.all_gather(all_counts, counts)
    all_counts = [c.cpu().numpy() for c in all_counts]
    if rank != root:
        mine = np.concatenate(queues) if sum(len(q) for q in queues) else np.zeros((0, 2))
        if len(mine):
            dist.send(torch.from_numpy(np.ascontiguousarray(mine)).to(device), dst=root)
        return None
    per_rank = []
    for r in range(world):
        k = int(all_counts[r].sum())
        if r == root:
            per_rank.append(np.concatenate(queues) if k else np.zeros((0, 2)))
        elif k:
            buf = torch.empty((k, 2), dtype=torch.float64, device=device)
            dist.recv(buf, src=r)
            per_rank.append(buf.cpu().numpy())
        else:
            per_rank.append(np.zeros((0, 2)))
    out = []
    for q in range(4):
        parts = []
        for r in range(world):
            off = int(all_counts[r][:q].sum())
            parts.append(per_rank[r][off: off + int(all_counts[r][q])])
        out.append(np.concatenate(parts))
    return out


def sharded_heaphull(shard, device=None, root: int = 0, stats: dict | None = None):
    """Run the sharded pipeline; returns the hull (h, 2) on `root`, None
    elsewhere.  `stats` (optional) receives counts / certificate info."""
    dist = _dist()
    rank = dist.get_rank() if dist else 0
    # one read per shard when the fused pass applies (its record equals K1's)
    rec = shard.fused_extremes() if hasattr(shard, "fused_extremes") else None
    fused = rec is not None
    if not fused:
        rec = shard.extremes()
    g = combine_extremes(_allgather_structs(rec, ExtremesRec, device))
    ext, mask = resolve_extremes(g)
    if mask:
        bbox = (g.x[0], g.y[1], g.x[2], g.y[3])
        crec = shard.corners_exact(bbox)
        ext = apply_corners(ext, combine_corners(_allgather_structs(crec, CornerRec, device)))
    octagon = build_octagon_from_set(ext)
    plan = make_plan(ext, octagon)
    counts = shard.filter_fused(ext, plan) if fused else shard.filter(plan)
    queues = [shard.queue_xy(q + 1, counts[q]) for q in range(4)]
    if stats is not None:
        stats.update(counts=list(counts), uncertified=mask, fused=fused,
                     ext=[int(v) for v in ext.ext],
                     octagon=octagon.tolist(), n_total=int(g.n))
    gathered = _gather_queues(queues, device, root)
    if rank != root:
        return None
    anchors = [(ext.x[s], ext.y[s]) for s in range(4)]
    return hull_from_queue_points(anchors, gathered)


def sharded_hull_indices(shard, hull, device=None, root: int = 0):
    """Hull vertex indices of the last sharded_heaphull (the hull given on
    `root`): the smallest global input index with each vertex's
    coordinates -- every shard maps the vertices over its own survivors,
    then a MIN all-reduce.  Returns the (h,) int64 array on `root`."""
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        idx = shard.hull_indices(hull)
        if (idx < 0).any():
            raise ValueError("hull_indices: a vertex is not among the survivors")
        return idx
    import torch
    rank = dist.get_rank()
    h = torch.tensor([len(hull) if rank == root else 0], dtype=torch.int64, device=device)
    dist.broadcast(h, root)
    hv = torch.zeros((int(h.item()), 2), dtype=torch.float64, device=device)
    if rank == root:
        hv.copy_(torch.from_numpy(np.ascontiguousarray(hull, dtype=np.float64)))
    dist.broadcast(hv, root)
    part = shard.hull_indices(hv.cpu().numpy())
    big = np.iinfo(np.int64).max
    t = torch.from_numpy(np.where(part < 0, big, part)).to(device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    if rank != root:
        return None
    idx = t.cpu().numpy()
    if (idx == big).any():
        raise ValueError("hull_indices: a vertex is not among the survivors")
    return idx


def shard_range(n_total: int, world: int, rank: int):
    """Contiguous index range of `rank`: [floor(r n / G), floor((r+1) n / G))."""
    b0 = (n_total * rank) // world
    b1 = (n_total * (rank + 1)) // world
    return b0, b1 - b0


__all__ = ["CudaShard", "sharded_heaphull", "sharded_hull_indices", "shard_range"]
