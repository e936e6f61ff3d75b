"""ctypes front-end for the parity checkers (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg -- which also checks the device results against the
reference on the same points, outside every timed region -- and its
``--impl reference`` arm) may import this package.  The product path
(``paper_2209_12310_b200``) never does.

Two checkers live here:

* ``Oracle`` -- ``liboracle.so``, the plain-C restatement in ``oracle.c``
  of the reference filter path (each function cites the reference
  file:line it follows).
* ``Reference`` -- ``_ref/libocto_ref.so``, the unmodified reference
  library compiled from ``/root/reference/proj/src`` by ``Makefile``.
  Present in the build container and shipped to the GPU box as a built
  artefact; ``available()`` is False where it was never built.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libocto_ref.so")

DISTS = {"normal": 0, "square": 1, "disk": 2, "circle": 3}

_u64p = C.POINTER(C.c_uint64)
_dp = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)


def build(quiet: bool = True) -> None:
    """Compile liboracle.so (and _ref/ when /root/reference is present)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _pts(xy) -> np.ndarray:
    a = np.ascontiguousarray(xy, dtype=np.float64)
    if a.ndim != 2 or (a.size and a.shape[1] != 2):
        raise ValueError("expected an array of shape (n, 2)")
    return a


def _dptr(a):
    return a.ctypes.data_as(_dp)


class Oracle:
    """The C restatement (oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.orc_splitmix_next.restype = C.c_uint64
        L.orc_splitmix_next.argtypes = [_u64p]
        L.orc_splitmix_unit.restype = C.c_double
        L.orc_splitmix_unit.argtypes = [_u64p]
        L.orc_generate.restype = C.c_int
        L.orc_generate.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_double, _dp]
        L.orc_find_extremes.restype = C.c_int
        L.orc_find_extremes.argtypes = [_dp, C.c_uint64, _u64p]
        L.orc_axis_extremes.restype = C.c_int
        L.orc_axis_extremes.argtypes = [_dp, C.c_uint64, _u64p]
        L.orc_corner_extremes.restype = C.c_int
        L.orc_corner_extremes.argtypes = [_dp, C.c_uint64, _u64p, _u64p]
        L.orc_build_octagon.restype = C.c_int
        L.orc_build_octagon.argtypes = [_dp, _u64p, _dp]
        L.orc_find_queue.restype = C.c_int
        L.orc_find_queue.argtypes = [_dp, _dp, _u64p]
        L.orc_classify.restype = None
        L.orc_classify.argtypes = [_dp, C.c_uint64, _dp, C.c_int, _u64p, _u8p]
        L.orc_heaphull.restype = C.c_int64
        L.orc_heaphull.argtypes = [_dp, C.c_uint64, _dp, _u8p]
        L.orc_monotone_chain.restype = C.c_int64
        L.orc_monotone_chain.argtypes = [_dp, C.c_uint64, _dp]
        L.orc_filter_rate.restype = C.c_double
        L.orc_filter_rate.argtypes = [_u8p, C.c_uint64]

    # -- generator (pointgen.cpp:44-88)
    def generate(self, dist: str, n: int, seed: int = 0, distort: float = 0.0) -> np.ndarray:
        if dist not in DISTS:
            raise ValueError(f"unknown distribution '{dist}'")
        out = np.empty((n, 2), dtype=np.float64)
        if self.lib.orc_generate(DISTS[dist], n, seed, float(distort), _dptr(out)) != 0:
            raise ValueError("invalid generator spec")
        return out

    def splitmix(self, seed: int, k: int):
        st = C.c_uint64(seed)
        return [self.lib.orc_splitmix_next(C.byref(st)) for _ in range(k)]

    # -- filter stage (filter.cpp)
    def find_extremes(self, xy) -> np.ndarray:
        a = _pts(xy)
        ext = np.zeros(8, dtype=np.uint64)
        if self.lib.orc_find_extremes(_dptr(a), len(a), ext.ctypes.data_as(_u64p)) != 0:
            raise ValueError("empty point set")
        return ext

    def corner_extremes(self, xy, axis) -> np.ndarray:
        a = _pts(xy)
        ax = np.ascontiguousarray(axis, dtype=np.uint64)
        out = np.zeros(4, dtype=np.uint64)
        self.lib.orc_corner_extremes(_dptr(a), len(a), ax.ctypes.data_as(_u64p),
                                     out.ctypes.data_as(_u64p))
        return out

    def build_octagon(self, xy, ext) -> np.ndarray:
        a = _pts(xy)
        e = np.ascontiguousarray(ext, dtype=np.uint64)
        oct_ = np.zeros((8, 2), dtype=np.float64)
        m = self.lib.orc_build_octagon(_dptr(a), e.ctypes.data_as(_u64p), _dptr(oct_))
        return oct_[:m].copy()

    def find_queue(self, p, xy, ext) -> int:
        a = _pts(xy)
        pp = np.ascontiguousarray(p, dtype=np.float64)
        e = np.ascontiguousarray(ext, dtype=np.uint64)
        return self.lib.orc_find_queue(_dptr(pp), _dptr(a), e.ctypes.data_as(_u64p))

    def classify(self, xy, ext=None, octagon=None) -> np.ndarray:
        a = _pts(xy)
        e = self.find_extremes(a) if ext is None else np.ascontiguousarray(ext, dtype=np.uint64)
        o = self.build_octagon(a, e) if octagon is None else np.ascontiguousarray(octagon)
        labels = np.zeros(len(a), dtype=np.uint8)
        self.lib.orc_classify(_dptr(a), len(a), _dptr(o), len(o),
                              e.ctypes.data_as(_u64p), labels.ctypes.data_as(_u8p))
        return labels

    @staticmethod
    def build_queues(labels):
        """hull.cpp:124-131 -- the four index queues in input order."""
        lab = np.asarray(labels)
        return [np.flatnonzero(lab == q).astype(np.uint64) for q in (1, 2, 3, 4)]

    # -- hull (hull.cpp)
    def heaphull(self, xy, with_labels: bool = False):
        a = _pts(xy)
        if len(a) == 0:
            raise ValueError("heaphull: empty point set")
        hull = np.zeros((len(a) + 8, 2), dtype=np.float64)
        labels = np.zeros(len(a), dtype=np.uint8)
        h = self.lib.orc_heaphull(_dptr(a), len(a), _dptr(hull), labels.ctypes.data_as(_u8p))
        hull = hull[:h].copy()
        return (hull, labels) if with_labels else hull

    def monotone_chain(self, xy) -> np.ndarray:
        a = _pts(xy)
        if len(a) == 0:
            raise ValueError("monotone_chain_hull: empty point set")
        hull = np.zeros((len(a) + 2, 2), dtype=np.float64)
        h = self.lib.orc_monotone_chain(_dptr(a), len(a), _dptr(hull))
        return hull[:h].copy()


class Reference:
    """The unmodified reference library (oracle/_ref/libocto_ref.so)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self, path: str = REF_SO):
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_generate.restype = C.c_int
        L.ref_generate.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_double, _dp]
        L.ref_find_extremes.restype = C.c_int
        L.ref_find_extremes.argtypes = [_dp, C.c_uint64, C.c_uint64, C.c_uint64, _u64p]
        L.ref_build_octagon.restype = C.c_int
        L.ref_build_octagon.argtypes = [_dp, C.c_uint64, _u64p, _dp]
        L.ref_find_queue.restype = C.c_int
        L.ref_find_queue.argtypes = [_dp, _dp, C.c_uint64, _u64p]
        L.ref_classify.restype = C.c_int
        L.ref_classify.argtypes = [_dp, C.c_uint64, C.c_uint64, C.c_uint64, _u8p]
        L.ref_heaphull_run.restype = C.c_int64
        L.ref_heaphull_run.argtypes = [_dp, C.c_uint64, C.c_uint64, C.c_uint64, _dp, _u8p, _dp]
        L.ref_monotone_chain.restype = C.c_int64
        L.ref_monotone_chain.argtypes = [_dp, C.c_uint64, _dp]
        L.ref_engine_new.restype = C.c_void_p
        L.ref_engine_new.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_engine_free.restype = None
        L.ref_engine_free.argtypes = [C.c_void_p]
        L.ref_engine_heaphull.restype = C.c_int64
        L.ref_engine_heaphull.argtypes = [C.c_void_p, _dp, C.c_uint64, _dp]

    def _err(self):
        return ValueError(self.lib.ref_last_error().decode())

    def generate(self, dist: str, n: int, seed: int = 0, distort: float = 0.0) -> np.ndarray:
        out = np.empty((n, 2), dtype=np.float64)
        if self.lib.ref_generate(DISTS[dist], n, seed, float(distort), _dptr(out)) != 0:
            raise self._err()
        return out

    def find_extremes(self, xy, workers: int = 1, chunk: int = 32) -> np.ndarray:
        a = _pts(xy)
        ext = np.zeros(8, dtype=np.uint64)
        if self.lib.ref_find_extremes(_dptr(a), len(a), workers, chunk,
                                      ext.ctypes.data_as(_u64p)) != 0:
            raise self._err()
        return ext

    def build_octagon(self, xy, ext) -> np.ndarray:
        a = _pts(xy)
        e = np.ascontiguousarray(ext, dtype=np.uint64)
        oct_ = np.zeros((8, 2), dtype=np.float64)
        m = self.lib.ref_build_octagon(_dptr(a), len(a), e.ctypes.data_as(_u64p), _dptr(oct_))
        return oct_[:m].copy()

    def find_queue(self, p, xy, ext) -> int:
        a = _pts(xy)
        pp = np.ascontiguousarray(p, dtype=np.float64)
        e = np.ascontiguousarray(ext, dtype=np.uint64)
        return self.lib.ref_find_queue(_dptr(pp), _dptr(a), len(a), e.ctypes.data_as(_u64p))

    def classify(self, xy, workers: int = 1, chunk: int = 32) -> np.ndarray:
        a = _pts(xy)
        labels = np.zeros(len(a), dtype=np.uint8)
        if self.lib.ref_classify(_dptr(a), len(a), workers, chunk,
                                 labels.ctypes.data_as(_u8p)) != 0:
            raise self._err()
        return labels

    def heaphull_run(self, xy, workers: int = 1, chunk: int = 32):
        """-> (hull (h,2), labels (n,), {filter_ms, hull_ms, total_ms})"""
        a = _pts(xy)
        hull = np.zeros((len(a) + 8, 2), dtype=np.float64)
        labels = np.zeros(len(a), dtype=np.uint8)
        t = np.zeros(3, dtype=np.float64)
        h = self.lib.ref_heaphull_run(_dptr(a), len(a), workers, chunk, _dptr(hull),
                                      labels.ctypes.data_as(_u8p), _dptr(t))
        if h < 0:
            raise self._err()
        return hull[:h].copy(), labels, dict(filter_ms=t[0], hull_ms=t[1], total_ms=t[2])

    def monotone_chain(self, xy) -> np.ndarray:
        a = _pts(xy)
        hull = np.zeros((len(a) + 2, 2), dtype=np.float64)
        h = self.lib.ref_monotone_chain(_dptr(a), len(a), _dptr(hull))
        if h < 0:
            raise self._err()
        return hull[:h].copy()

    def engine(self, workers: int, chunk: int = 32):
        return _RefEngine(self, workers, chunk)


class _RefEngine:
    """A persistent reference ReduceEngine (for timing loops)."""

    def __init__(self, ref: Reference, workers: int, chunk: int):
        self.ref = ref
        self.h = ref.lib.ref_engine_new(workers, chunk)
        self.workers = workers

    def heaphull(self, xy):
        t = np.zeros(3, dtype=np.float64)
        h = self.ref.lib.ref_engine_heaphull(self.h, _dptr(xy), len(xy), _dptr(t))
        if h < 0:
            raise self.ref._err()
        return h, dict(filter_ms=t[0], hull_ms=t[1], total_ms=t[2])

    def close(self):
        if self.h:
            self.ref.lib.ref_engine_free(self.h)
            self.h = None

    def __del__(self):
        self.close()
