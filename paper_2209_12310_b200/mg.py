"""Multi-GPU heaphull over NCCL (ctypes front-end of the ohx_mg_* C ABI,
csrc/mg.cpp).

Two shapes, both one NCCL rank per GPU:

* one process per GPU (torchrun): rank 0 calls ``unique_id()``, hands the
  bytes to the other ranks (e.g. a torch.distributed broadcast), every
  rank calls ``MultiGPU.init_rank(uid, world, rank, device)`` and then
  ``heaphull_shard(d_xy, n, base)`` with its own contiguous index range;
* one process driving several GPUs: ``MultiGPU.init_all(devices)`` and
  ``heaphull(points)`` (host points split over the devices) or
  ``heaphull_device(shards)``.

``vshards`` splits every rank's range into that many shards with their own
contexts -- the multi-GPU exchange exercised on one device.  The hull comes
back on rank 0 (``None`` elsewhere) with an info dict (job extremes, queue
lengths, fused shards, per-phase host times).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import MgInfo, check, lib

_dp = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)
_u64p = C.POINTER(C.c_uint64)


def unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(lib.ohx_mg_unique_id(buf))
    return bytes(buf)


def nccl_version() -> int:
    v = C.c_int(0)
    check(lib.ohx_mg_nccl_version(C.byref(v)))
    return v.value


def _info(i: MgInfo) -> dict:
    return {"ext": [int(v) for v in i.ext], "counts": [int(v) for v in i.counts],
            "n_total": int(i.n_total), "corner_pass": bool(i.corner_pass),
            "fused_shards": int(i.fused_shards), "shards": int(i.shards),
            "ms": {"extremes_exchange": i.ms[0], "filter": i.ms[1], "gather": i.ms[2],
                   "hull": i.ms[3]}}


def _ptr(x) -> int:
    return x if isinstance(x, int) else int(x.data_ptr())


class MultiGPU:
    def __init__(self, handle):
        self.h = handle
        w, lr = C.c_int(0), C.c_int(0)
        check(lib.ohx_mg_world(self.h, C.byref(w), C.byref(lr)))
        self.world, self.local_ranks = w.value, lr.value

    @classmethod
    def init_rank(cls, uid: bytes, world: int, rank: int, device: int) -> "MultiGPU":
        h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        check(lib.ohx_mg_init_rank(buf, world, rank, device, C.byref(h)))
        return cls(h)

    @classmethod
    def init_all(cls, devices) -> "MultiGPU":
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        check(lib.ohx_mg_init_all(len(devices), devs, C.byref(h)))
        return cls(h)

    def shard_context(self, local_rank: int = 0, shard: int = 0):
        """The (borrowed) Context of one shard of this handle: launches,
        kernel_ms_sum and last_run of that shard's part of the last call."""
        from . import Context
        h = C.c_void_p()
        check(lib.ohx_mg_ctx(self.h, local_rank, shard, C.byref(h)))
        c = Context.__new__(Context)
        c.h, c.device, c._owned = h, None, False
        return c

    def close(self):
        if self.h:
            lib.ohx_mg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _call(self, fn, cap):
        """fn(hull buffer, cap, &h) -> (hull, h); regrows when the hull outgrew cap.
        The output buffer (and its ctypes pointer) is kept for the next call
        while hulls come back as copies (< 2^20 vertices), as Context does:
        a fresh 256 MB buffer per call costs an mmap / munmap pair."""
        while True:
            hb = getattr(self, "_hbuf", None)
            if hb is not None and len(hb[0]) >= cap:
                hull, hptr = hb
            else:
                hull = np.empty((max(cap, 1), 2), dtype=np.float64)
                hptr = hull.ctypes.data_as(_dp)
            self._hbuf = None
            h = C.c_uint64(0)
            info = MgInfo()
            rc = fn(hptr, len(hull), C.byref(h), C.byref(info))
            if rc == -1 and h.value > len(hull):
                cap = h.value
                continue
            check(rc)
            if h.value < (1 << 20):
                self._hbuf = (hull, hptr)
                return hull[: h.value].copy(), info
            return hull[: h.value], info

    def heaphull_shard(self, d_xy, n: int, base: int, vshards: int = 1, labels=None,
                       cap: int | None = None):
        """Collective: this rank's device-resident range [base, base + n).
        -> (hull on rank 0 else None, info)."""
        lab = None if labels is None else labels.ctypes.data_as(_u8p)
        hull, info = self._call(
            lambda hp, c, h, i: lib.ohx_mg_heaphull_shard(self.h, _ptr(d_xy), n, base, vshards,
                                                          lab, hp, c, h, i),
            cap if cap is not None else min(n + 8, 1 << 24))
        return (hull if len(hull) else None), _info(info)

    def heaphull_device(self, shards, labels=None, cap: int | None = None):
        """shards: [(device tensor or pointer, n), ...] in index order, an
        equal number per device.  -> (hull, info)."""
        k = len(shards)
        ptrs = (C.c_void_p * k)(*[_ptr(d) for d, _ in shards])
        ns = (C.c_uint64 * k)(*[int(n) for _, n in shards])
        total = sum(int(n) for _, n in shards)
        lab = None if labels is None else labels.ctypes.data_as(_u8p)
        hull, info = self._call(
            lambda hp, c, h, i: lib.ohx_mg_heaphull_device(self.h, k, ptrs, ns, lab, hp, c, h, i),
            cap if cap is not None else min(total + 8, 1 << 24))
        return hull, _info(info)

    def heaphull(self, points, vshards: int = 1, labels: bool = False):
        """Host points over the handle's devices -> (hull, info[, labels])."""
        a = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
        lab = np.empty(len(a), dtype=np.uint8) if labels else None
        hull, info = self._call(
            lambda hp, c, h, i: lib.ohx_mg_heaphull(
                self.h, a.ctypes.data_as(_dp), len(a), vshards,
                None if lab is None else lab.ctypes.data_as(_u8p), hp, c, h, i),
            min(len(a) + 8, 1 << 24))
        return (hull, _info(info), lab) if labels else (hull, _info(info))


_single = {}


def mg_heaphull_device(tensors, n: int, shards: int = 1, devices=(0,)):
    """The multi-GPU pipeline over ONE device-resident array split into
    `shards` contiguous shards (per device: shards / len(devices)),
    through a cached single-process handle.  -> (hull, info)."""
    key = tuple(devices)
    if key not in _single:
        _single[key] = MultiGPU.init_all(list(devices))
    mg = _single[key]
    d = tensors[0]
    base = _ptr(d)
    parts = []
    for j in range(shards):
        b0, b1 = n * j // shards, n * (j + 1) // shards
        parts.append((base + 16 * b0, b1 - b0))
    return mg.heaphull_device(parts)


__all__ = ["MultiGPU", "unique_id", "nccl_version", "mg_heaphull_device"]
