"""Test-side emulation of one shard's kernel outputs with reference
semantics (numpy + the oracle).  Used to exercise the host orchestration
(combine, certificate, octagon, plan, gather, host hull) without a GPU."""

import numpy as np

from paper_2209_12310_b200 import _lib


def emulate_k1(pts, base=0):
    """One shard's K1 record: argmax of the 8 maximised keys (smallest index
    on ties) plus the second-largest diagonal key."""
    x, y = pts[:, 0], pts[:, 1]
    t = x + y
    d = x - y
    keys = [x, y, -x, -y, t, -d, -t, d]
    rec = _lib.ExtremesRec()
    for a, k in enumerate(keys):
        j = int(np.flatnonzero(k == k.max())[0])
        rec.key[a] = k[j]
        rec.idx[a] = base + j
        rec.x[a] = x[j]
        rec.y[a] = y[j]
        if a >= 4:
            rest = np.delete(k, j)
            rec.second[a - 4] = rest.max() if rest.size else -np.inf
    rec.n = len(pts)
    return rec


def emulate_corners(pts, bbox, base=0):
    xmax, ymax, xmin, ymin = bbox
    rec = _lib.CornerRec()
    for a, (cx, cy) in enumerate([(xmax, ymax), (xmin, ymax), (xmin, ymin), (xmax, ymin)]):
        m = np.abs(pts[:, 0] - cx) + np.abs(pts[:, 1] - cy)
        j = int(np.flatnonzero(m == m.min())[0])
        rec.key[a], rec.idx[a], rec.x[a], rec.y[a] = m[j], base + j, pts[j, 0], pts[j, 1]
    rec.n = len(pts)
    return rec


class EmulatedShard:
    """The `sharded.py` shard interface over host arrays.  `filter` labels
    the shard with the oracle using the plan's octagon and kept indices."""

    def __init__(self, oracle, all_pts, base, n):
        self.o, self.all, self.base, self.n = oracle, all_pts, base, n
        self.pts = all_pts[base: base + n]
        self.labels = None

    def extremes(self):
        return emulate_k1(self.pts, self.base)

    def corners_exact(self, bbox):
        return emulate_corners(self.pts, bbox, self.base)

    def filter(self, plan):
        ext = np.array([plan.kept[k] for k in (0, 2, 4, 6, 1, 3, 5, 7)], dtype=np.uint64)
        m = plan.m
        octagon = np.array([[plan.ax[i], plan.ay[i]] for i in range(m)]) if m >= 3 else \
            np.zeros((0, 2))
        if m < 3:  # degenerate: pass the (<3) vertices the oracle expects
            octagon = np.zeros((max(m, 0), 2))
        full = self.o.classify(self.all, ext, octagon)
        self.labels = full[self.base: self.base + self.n]
        return [int((self.labels == q).sum()) for q in (1, 2, 3, 4)]

    def queue_xy(self, q, count):
        return self.pts[self.labels == q]
