"""B200-native heaphull filter (arXiv 2209.12310) -- Python front-end.

Drop-in for the reference Python package ``octohull``
(/root/reference/proj/python/octohull/__init__.py and python/module.cpp):
the same functions with the same arguments, return types and errors --
``generate``, ``heaphull``, ``monotone_chain``, ``classify``,
``filter_rate`` -- backed by the C ABI of ``include/ohx.h`` whose filter
runs as sm_100a kernels.  ``threads``/``chunk`` are accepted for
compatibility (the reference's CPU lane geometry); results never depend
on them, as in the reference.

``Context`` exposes the kernel-level entry points for device-resident
points (torch CUDA tensors or raw device pointers), which is what the
benchmarks and the multi-GPU sharded path (``sharded.py``) use.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from ._lib import (DISTS, OHX_E_INVALID, SLOTS, CornerRec, ExtremeSet, ExtremesRec, FilterPlan,
                   OhxError, RunInfo, check, lib)

__all__ = ["classify", "classify_points", "filter_rate", "generate", "generate_range", "heaphull", "heaphull_file", "hull_indices", "write_pts2",
           "monotone_chain",
           "heaphull_run", "find_extremes", "Context", "OhxError", "device_count"]

_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)
_u8p = C.POINTER(C.c_uint8)


def _points(points) -> np.ndarray:
    """python/module.cpp:18-28: (n, 2) C-contiguous float64, finite."""
    a = np.ascontiguousarray(points, dtype=np.float64)
    if a.ndim != 2 or a.shape[1] != 2:
        raise ValueError("expected an array of shape (n, 2)")
    if a.size:
        bad = ~np.isfinite(a).all(axis=1)
        if bad.any():
            raise ValueError(f"non-finite coordinate at point index {int(np.argmax(bad))}")
    return a


def _check_cfg(threads: int, chunk: int) -> None:
    # ReduceConfig validation, reference parallel.cpp:8-13
    if chunk < 1:
        raise ValueError("ReduceConfig.chunk_size must be >= 1")
    if threads < 1:
        raise ValueError("ReduceConfig.workers must be >= 1")


def generate(dist: str, n: int, seed: int = 0, distort: float = 0.0, threads: int = 0) -> np.ndarray:
    """Seeded synthetic points: normal | square | disk | circle (bit-identical
    to the reference generator; multi-threaded)."""
    if dist not in DISTS:
        raise ValueError(f"unknown distribution '{dist}' (expected normal|square|disk|circle)")
    out = np.empty((max(int(n), 0), 2), dtype=np.float64)
    check(lib.ohx_generate(DISTS[dist], int(n), int(seed), float(distort),
                           out.ctypes.data_as(_dp), int(threads)))
    return out


def generate_range(dist: str, n: int, lo: int, count: int, seed: int = 0, distort: float = 0.0,
                   threads: int = 0, out=None) -> np.ndarray:
    """Points [lo, lo + count) of generate(dist, n, seed, distort) -- a
    shard's slice of the corpus, without generating the rest.  `out`
    (optional) is a C-contiguous (count, 2) float64 buffer to fill."""
    if dist not in DISTS:
        raise ValueError(f"unknown distribution '{dist}' (expected normal|square|disk|circle)")
    if out is None:
        out = np.empty((max(int(count), 0), 2), dtype=np.float64)
    if out.shape != (int(count), 2) or out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError("out must be a C-contiguous (count, 2) float64 array")
    check(lib.ohx_generate_range(DISTS[dist], int(n), int(seed), float(distort), int(lo),
                                 int(count), out.ctypes.data_as(_dp), int(threads)))
    return out


def heaphull(points, threads: int = 1, chunk: int = 32) -> np.ndarray:
    """Octagon-filtered convex hull; returns the CCW vertex cycle (h, 2)."""
    _check_cfg(threads, chunk)
    a = _points(points)
    hull = np.empty((len(a) + 8, 2), dtype=np.float64)
    h = C.c_uint64(0)
    check(lib.ohx_heaphull(a.ctypes.data_as(_dp), len(a), hull.ctypes.data_as(_dp),
                           len(hull), C.byref(h), None))
    # small hulls are copied out of the (virtual, n-sized) buffer
    return hull[: h.value].copy() if h.value < (1 << 20) else hull[: h.value]


def hull_indices(hull) -> np.ndarray:
    """Vertex indices of the hull the last heaphull call returned (default
    context): for each vertex, the smallest input index with those
    coordinates, in the hull's order."""
    hv = np.ascontiguousarray(hull, dtype=np.float64).reshape(-1, 2)
    idx = np.empty(len(hv), dtype=np.uint64)
    check(lib.ohx_hull_indices(None, hv.ctypes.data_as(_dp), len(hv), idx.ctypes.data_as(_u64p),
                               None))
    return idx.astype(np.int64)


def heaphull_run(points):
    """heaphull_run (hull.cpp:152-194): (hull, labels, timings dict)."""
    a = _points(points)
    hull = np.empty((len(a) + 8, 2), dtype=np.float64)
    labels = np.empty(len(a), dtype=np.uint8)
    t = np.zeros(4, dtype=np.float64)
    h = C.c_uint64(0)
    check(lib.ohx_heaphull_run(a.ctypes.data_as(_dp), len(a), hull.ctypes.data_as(_dp),
                               len(hull), C.byref(h), labels.ctypes.data_as(_u8p),
                               t.ctypes.data_as(_dp)))
    return hull[: h.value].copy(), labels, dict(filter_ms=t[0], hull_ms=t[1], total_ms=t[2])


def heaphull_file(path) -> np.ndarray:
    """heaphull of a PTS2 point file (reference io.cpp binary layout), the
    file streamed straight into device memory."""
    n = C.c_uint64(0)
    check(lib.ohx_pts2_count(os.fsencode(path), C.byref(n)))
    hull = np.empty((n.value + 8, 2), dtype=np.float64)
    h = C.c_uint64(0)
    check(lib.ohx_heaphull_pts2(os.fsencode(path), hull.ctypes.data_as(_dp), len(hull),
                                C.byref(h), None))
    return hull[: h.value].copy() if h.value < (1 << 20) else hull[: h.value]


def write_pts2(points, path) -> None:
    """Write a PTS2 file (magic, u64 LE count, LE (x, y) doubles); like the
    reference's write_points it does not validate the values."""
    a = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
    with open(path, "wb") as f:
        f.write(b"PTS2" + len(a).to_bytes(8, "little"))
        f.write(a.astype("<f8", copy=False).tobytes())


def monotone_chain(points) -> np.ndarray:
    """Full-set reference hull (Andrew's monotone chain), host only."""
    a = _points(points)
    hull = np.empty((len(a) + 2, 2), dtype=np.float64)
    h = C.c_uint64(0)
    check(lib.ohx_monotone_chain(a.ctypes.data_as(_dp), len(a), hull.ctypes.data_as(_dp),
                                 len(hull), C.byref(h)))
    return hull[: h.value].copy()


def classify(points, threads: int = 1, chunk: int = 32) -> np.ndarray:
    """Filter labels per point: 0 = discarded, 1..4 = quadrant queue."""
    _check_cfg(threads, chunk)
    a = _points(points)
    labels = np.empty(len(a), dtype=np.uint8)
    if len(a) == 0:
        raise ValueError("find_axis_extremes: empty point set")
    check(lib.ohx_classify(a.ctypes.data_as(_dp), len(a), labels.ctypes.data_as(_u8p)))
    return labels


def classify_points(points, polygon, ext) -> np.ndarray:
    """classify_points with a given polygon (any vertex count) and
    ExtremeSet (8 indices {east, north, west, south, ne, nw, sw, se})."""
    a = _points(points)
    poly = np.ascontiguousarray(polygon, dtype=np.float64).reshape(-1, 2)
    e = np.ascontiguousarray(ext, dtype=np.uint64)
    if e.shape != (8,):
        raise ValueError("ext must hold 8 indices")
    labels = np.empty(len(a), dtype=np.uint8)
    check(lib.ohx_classify_points(a.ctypes.data_as(_dp), len(a), poly.ctypes.data_as(_dp),
                                  len(poly), e.ctypes.data_as(_u64p),
                                  labels.ctypes.data_as(_u8p)))
    return labels


def find_extremes(points) -> np.ndarray:
    """ExtremeSet as 8 indices {east, north, west, south, ne, nw, sw, se}."""
    a = _points(points)
    ext = np.zeros(8, dtype=np.uint64)
    check(lib.ohx_find_extremes(a.ctypes.data_as(_dp), len(a), ext.ctypes.data_as(_u64p)))
    return ext


def filter_rate(labels) -> float:
    """Fraction of points discarded by the filter (label == 0)."""
    labels = np.asarray(labels)
    if labels.size == 0:
        raise ValueError("empty label array")
    return float((labels == 0).mean())


def device_count() -> int:
    n = C.c_int(0)
    check(lib.ohx_device_count(C.byref(n)))
    return n.value


def _ptr(x) -> int:
    """Device address of a torch tensor (or an int pointer)."""
    if isinstance(x, int):
        return x
    return int(x.data_ptr())


def _stream(s):
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return int(s.cuda_stream)  # torch.cuda.Stream


def rec_to_dict(rec: ExtremesRec) -> dict:
    return {
        "idx": [int(v) for v in rec.idx], "key": list(rec.key), "x": list(rec.x),
        "y": list(rec.y), "second": list(rec.second), "n": int(rec.n),
    }


class Context:
    """A device context (stream + grow-only workspaces) of the C ABI."""

    def __init__(self, device: int = 0, default: bool = False):
        h = C.c_void_p()
        check((lib.ohx_ctx_default if default else lib.ohx_ctx_create)(device, C.byref(h)))
        self.h = h
        self.device = device
        self._owned = not default
        self._hbuf = None  # heaphull_device's host output scratch (small hulls are copied out)

    def trim(self):
        """Release this context's grow-only workspaces (and the host block
        cache); later calls regrow them."""
        check(lib.ohx_ctx_trim(self.h))
        self._hbuf = None

    def close(self):
        if self._owned and self.h:
            lib.ohx_ctx_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(lib.ohx_ctx_launches(self.h))

    def kernel_ms(self) -> dict:
        """CUDA-event durations (ms) of the last launch of each stage: K1 (or
        the fused KF filter pass), K1b, K2, and the fused candidate stage."""
        out = (C.c_double * 4)()
        check(lib.ohx_ctx_kernel_ms(self.h, out))
        return {"k1": out[0], "k1b": out[1], "k2": out[2], "kc": out[3]}

    def kernel_ms_sum(self, reset: bool = False) -> dict:
        """Running sums of the stage durations over the calls since the last
        reset: {stage: (total_ms, calls)} (read once after a timing loop)."""
        tot = (C.c_double * 4)()
        cnt = (C.c_uint64 * 4)()
        check(lib.ohx_ctx_kernel_ms_sum(self.h, tot, cnt, 1 if reset else 0))
        return {k: (tot[i], int(cnt[i])) for i, k in enumerate(("k1", "k1b", "k2", "kc"))}

    def last_run(self) -> dict:
        """How the last pipeline call on this context ran (fused single pass
        or two passes, corner fallback, candidates, queue lengths)."""
        r = RunInfo()
        check(lib.ohx_ctx_last_run(self.h, C.byref(r)))
        return {"fused": bool(r.fused), "corner_pass": bool(r.corner_pass),
                "candidates": int(r.candidates), "counts": [int(v) for v in r.counts],
                "fuse_state": ("off", "fused", "no-sample-region", "low-sample-coverage",
                               "region-not-certified", "too-many-candidates")[r.fuse_state],
                "sample_coverage": float(r.sample_coverage),
                "hull_path": ("host", "device-chains", "device-chains-unproven",
                              "device-sort-host-chains")[r.hull_path]}

    # ---- kernel level --------------------------------------------------
    def extremes(self, d_xy, n: int, index_base: int = 0, stream=None) -> ExtremesRec:
        rec = ExtremesRec()
        check(lib.ohx_extremes(self.h, _ptr(d_xy), n, index_base, C.byref(rec), _stream(stream)))
        return rec

    def fused_extremes(self, d_xy, n: int, index_base: int = 0, stream=None):
        """Fused single pass over a shard: the extremes record from one read
        (KF + K1 over the candidates), or None when the pass did not apply
        (then use `extremes`).  Pair with `filter_fused`."""
        rec = ExtremesRec()
        fused = C.c_int(0)
        check(lib.ohx_fused_extremes(self.h, _ptr(d_xy), n, index_base, C.byref(rec),
                                     C.byref(fused), _stream(stream)))
        return rec if fused.value else None

    def filter_fused(self, d_xy, n: int, ext: ExtremeSet, plan: FilterPlan, index_base: int = 0,
                     d_labels=None, stream=None):
        """Second half of the fused pass -> (queue counts, K2 ran on the
        candidates only)."""
        counts = (C.c_uint64 * 4)()
        fused = C.c_int(0)
        check(lib.ohx_filter_fused(self.h, _ptr(d_xy), n, index_base, C.byref(ext), C.byref(plan),
                                   None if d_labels is None else _ptr(d_labels), counts,
                                   C.byref(fused), _stream(stream)))
        return [int(c) for c in counts], bool(fused.value)

    def corners_exact(self, d_xy, n: int, bbox, index_base: int = 0, stream=None) -> CornerRec:
        b = (C.c_double * 4)(*bbox)
        rec = CornerRec()
        check(lib.ohx_corners_exact(self.h, _ptr(d_xy), n, index_base, b, C.byref(rec),
                                    _stream(stream)))
        return rec

    def filter(self, d_xy, n: int, plan: FilterPlan, index_base: int = 0, d_labels=None,
               stream=None) -> list:
        counts = (C.c_uint64 * 4)()
        check(lib.ohx_filter(self.h, _ptr(d_xy), n, index_base, C.byref(plan),
                             None if d_labels is None else _ptr(d_labels), counts,
                             _stream(stream)))
        return [int(c) for c in counts]

    def queue(self, q: int, count: int, with_idx: bool = True, with_xy: bool = False,
              stream=None):
        idx = np.empty(count, dtype=np.uint64) if with_idx else None
        xy = np.empty((count, 2), dtype=np.float64) if with_xy else None
        check(lib.ohx_queue_fetch(self.h, q, None if idx is None else idx.ctypes.data_as(_u64p),
                                  None if xy is None else xy.ctypes.data_as(_dp), count,
                                  _stream(stream)))
        return idx, xy

    def hull_indices(self, hull, partial: bool = False, stream=None) -> np.ndarray:
        """Vertex indices of a hull from this context's last pipeline call:
        the smallest input index with each vertex's coordinates.  partial:
        over this shard's survivors only, -1 where it has none."""
        hv = np.ascontiguousarray(hull, dtype=np.float64).reshape(-1, 2)
        idx = np.empty(len(hv), dtype=np.uint64)
        fn = lib.ohx_hull_indices_partial if partial else lib.ohx_hull_indices
        check(fn(self.h, hv.ctypes.data_as(_dp), len(hv), idx.ctypes.data_as(_u64p),
                 _stream(stream)))
        return idx.astype(np.int64)  # UINT64_MAX -> -1

    def load_pts2(self, path, d_xy=None, stream=None):
        """A PTS2 file into device memory -> (n, tensor or the given buffer)."""
        n = C.c_uint64(0)
        check(lib.ohx_pts2_count(os.fsencode(path), C.byref(n)))
        if d_xy is None:
            import torch
            d_xy = torch.empty((n.value, 2), dtype=torch.float64, device=f"cuda:{self.device}")
        cap = d_xy.numel() // 2
        check(lib.ohx_pts2_load_device(self.h, os.fsencode(path), _ptr(d_xy), cap, C.byref(n),
                                       _stream(stream)))
        return n.value, d_xy

    def hull_from_sorted_arcs_device(self, d_arcs, lens, raw_cycle=False, stream=None):
        """The hull stage on four arcs already in sweep order in device memory
        (back to back, lens[q] points each) -> (hull, proven): proven is
        False when the device chains could not prove a chunk and the host
        chains ran instead (the hull is the reference's either way).
        raw_cycle: the chained cycle before finalize_cycle (a test hook)."""
        ln = (C.c_uint64 * 4)(*[int(v) for v in lens])
        cap = sum(int(v) for v in lens) + 8
        hull = np.empty((cap, 2), dtype=np.float64)
        h = C.c_uint64(0)
        proven = C.c_int(0)
        check(lib.ohx_hull_from_sorted_arcs_device(self.h, _ptr(d_arcs), ln, hull.ctypes.data_as(_dp),
                                                   cap, C.byref(h), C.byref(proven),
                                                   1 if raw_cycle else 0, _stream(stream)))
        return hull[: h.value].copy(), bool(proven.value)

    def heaphull_device(self, d_xy, n: int, out="host"):
        """Full pipeline on device-resident points -> (hull, timings).
        out="device": the hull stays in device memory (a torch tensor on this
        context's device) -- ohx_heaphull_device_out; out=<(cap, 2) float64
        CUDA tensor>: written there (a reused buffer), a view returned;
        out=<(cap, 2) float64 C-contiguous host array or CPU tensor>: the
        hull copied there (a reused -- e.g. pinned -- host buffer: pinned
        memory takes one direct DMA), a view returned."""
        if isinstance(out, np.ndarray) or (not isinstance(out, str) and not out.is_cuda):
            host = out if isinstance(out, np.ndarray) else out.numpy()
            if host.dtype != np.float64 or not host.flags.c_contiguous or host.size % 2:
                raise ValueError("out: a C-contiguous float64 (cap, 2) host buffer")
            h = C.c_uint64(0)
            t = (C.c_double * 4)()
            check(lib.ohx_heaphull_device(self.h, _ptr(d_xy), n, host.ctypes.data_as(_dp),
                                          host.size // 2, C.byref(h), t))
            return host.reshape(-1, 2)[: h.value], dict(filter_ms=t[0], hull_ms=t[1],
                                                       total_ms=t[2])
        if not isinstance(out, str):  # a caller's device buffer
            cap = out.numel() // 2
            h = C.c_uint64(0)
            t = (C.c_double * 4)()
            check(lib.ohx_heaphull_device_out(self.h, _ptr(d_xy), n, _ptr(out), cap, C.byref(h),
                                              t))
            return out.view(-1, 2)[: h.value], dict(filter_ms=t[0], hull_ms=t[1], total_ms=t[2])
        if out == "device":
            import torch
            cap = n + 8 if n <= (1 << 26) else 1 << 24
            while True:
                hull = torch.empty((cap, 2), dtype=torch.float64, device=f"cuda:{self.device}")
                h = C.c_uint64(0)
                t = (C.c_double * 4)()
                rc = lib.ohx_heaphull_device_out(self.h, _ptr(d_xy), n, _ptr(hull), cap,
                                                 C.byref(h), t)
                if rc == OHX_E_INVALID and h.value > cap:
                    cap = h.value
                    continue
                check(rc)
                return hull[: h.value], dict(filter_ms=t[0], hull_ms=t[1], total_ms=t[2])
        if out != "host":
            raise ValueError("out must be 'host' or 'device'")
        # the output buffer is virtual until written: full size up to 2^28
        # points, else start at 2^24 and grow if the hull outgrows it.  It is
        # kept for the next call while hulls come back as copies (< 2^20
        # vertices); a larger hull is returned in it (the buffer goes with it)
        cap = n + 8 if n <= (1 << 28) else 1 << 24
        while True:
            # the scratch is kept with its ctypes pointer (numpy's .ctypes
            # costs microseconds per call on a 2.5 ms step)
            hb = self._hbuf
            if hb is not None and len(hb[0]) >= cap:
                hull, hptr = hb
            else:
                hull = np.empty((cap, 2), dtype=np.float64)
                hptr = hull.ctypes.data_as(_dp)
            self._hbuf = None
            h = C.c_uint64(0)
            t = (C.c_double * 4)()
            rc = lib.ohx_heaphull_device(self.h, _ptr(d_xy), n, hptr, len(hull), C.byref(h), t)
            if rc == OHX_E_INVALID and h.value > len(hull):  # the hull outgrew the buffer
                cap = h.value
                continue
            check(rc)
            if h.value < (1 << 20):
                self._hbuf = (hull, hptr)
                out = hull[: h.value].copy()
            else:
                out = hull[: h.value]
            return out, dict(filter_ms=t[0], hull_ms=t[1], total_ms=t[2])


# ---- host-only helpers of the C ABI (pure functions, no device) ---------
def combine_extremes(recs) -> ExtremesRec:
    arr = (ExtremesRec * len(recs))(*recs)
    out = ExtremesRec()
    check(lib.ohx_extremes_combine(arr, len(recs), C.byref(out)))
    return out


def combine_corners(recs) -> CornerRec:
    arr = (CornerRec * len(recs))(*recs)
    out = CornerRec()
    check(lib.ohx_corners_combine(arr, len(recs), C.byref(out)))
    return out


def resolve_extremes(rec: ExtremesRec):
    """-> (ExtremeSet, uncertified corner mask)."""
    out = ExtremeSet()
    mask = C.c_uint32(0)
    check(lib.ohx_extremes_resolve(C.byref(rec), C.byref(out), C.byref(mask)))
    return out, int(mask.value)


def apply_corners(ext: ExtremeSet, crec: CornerRec) -> ExtremeSet:
    for k in range(4):
        ext.ext[4 + k] = crec.idx[k]
        ext.x[4 + k] = crec.x[k]
        ext.y[4 + k] = crec.y[k]
    return ext


CANDIDATE_SLOTS = (0, 4, 1, 5, 2, 6, 3, 7)  # E, NE, N, NW, W, SW, S, SE


def build_octagon_from_set(ext: ExtremeSet) -> np.ndarray:
    cand = np.array([[ext.x[s], ext.y[s]] for s in CANDIDATE_SLOTS], dtype=np.float64)
    out = np.zeros((8, 2), dtype=np.float64)
    m = C.c_int(0)
    check(lib.ohx_build_octagon(cand.ctypes.data_as(_dp), out.ctypes.data_as(_dp), C.byref(m)))
    return out[: m.value].copy()


def make_plan(ext: ExtremeSet, octagon) -> FilterPlan:
    o = np.ascontiguousarray(octagon, dtype=np.float64).reshape(-1, 2)
    plan = FilterPlan()
    check(lib.ohx_filter_plan_build(C.byref(ext), o.ctypes.data_as(_dp), len(o), C.byref(plan)))
    return plan


def hull_from_queue_points(anchors, queues) -> np.ndarray:
    """Host hull stage on per-quadrant survivor coordinates (index order)."""
    a = np.ascontiguousarray(anchors, dtype=np.float64).reshape(4, 2)
    qs = [np.ascontiguousarray(q, dtype=np.float64).reshape(-1, 2) for q in queues]
    ptrs = (_dp * 4)(*[q.ctypes.data_as(_dp) for q in qs])
    lens = (C.c_uint64 * 4)(*[len(q) for q in qs])
    total = sum(len(q) for q in qs) + 8
    out = np.empty((total, 2), dtype=np.float64)
    h = C.c_uint64(0)
    check(lib.ohx_hull_from_queue_points(a.ctypes.data_as(_dp), ptrs, lens,
                                         out.ctypes.data_as(_dp), total, C.byref(h)))
    return out[: h.value].copy()


from .mg import MultiGPU, mg_heaphull_device  # noqa: E402  (multi-GPU, NCCL)
