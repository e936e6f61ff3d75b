"""ctypes binding of the C ABI (include/ohx.h) -- the same stub a maintainer
adds on the reference side.

Loading fails loudly: if ``lib/libocto_b200.so`` is missing the import
raises instead of falling back to anything.
"""

from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "lib", "libocto_b200.so")

OHX_OK = 0
OHX_E_INVALID = -1
OHX_E_CUDA = -2
OHX_E_NODEVICE = -3
OHX_E_NOMEM = -4
OHX_E_INTERNAL = -5
OHX_E_IO = -6

DISTS = {"normal": 0, "square": 1, "disk": 2, "circle": 3}
SLOTS = ("east", "north", "west", "south", "ne", "nw", "sw", "se")

_u64 = C.c_uint64
_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)
_u8p = C.POINTER(C.c_uint8)
_vp = C.c_void_p


class ExtremesRec(C.Structure):
    _fields_ = [("key", C.c_double * 8), ("idx", _u64 * 8), ("second", C.c_double * 4),
                ("x", C.c_double * 8), ("y", C.c_double * 8), ("n", _u64)]


class CornerRec(C.Structure):
    _fields_ = [("key", C.c_double * 4), ("idx", _u64 * 4), ("x", C.c_double * 4),
                ("y", C.c_double * 4), ("n", _u64)]


class ExtremeSet(C.Structure):
    _fields_ = [("ext", _u64 * 8), ("x", C.c_double * 8), ("y", C.c_double * 8)]


class RunInfo(C.Structure):
    _fields_ = [("fused", C.c_uint32), ("corner_pass", C.c_uint32), ("candidates", _u64),
                ("counts", _u64 * 4), ("fuse_state", C.c_uint32), ("hull_path", C.c_uint32),
                ("sample_coverage", C.c_double)]


class FilterPlan(C.Structure):
    _fields_ = [("ax", C.c_double * 8), ("ay", C.c_double * 8),
                ("ea", C.c_double * 8), ("ec", C.c_double * 8),
                ("qax", C.c_double * 4), ("qay", C.c_double * 4),
                ("qa", C.c_double * 4), ("qc", C.c_double * 4),
                ("box", C.c_double * 4), ("kept", _u64 * 8),
                ("kept_label", C.c_uint8 * 8), ("m", C.c_int32), ("pad", C.c_int32)]


class MgInfo(C.Structure):
    _fields_ = [("ext", _u64 * 8), ("counts", _u64 * 4), ("n_total", _u64),
                ("corner_pass", C.c_uint32), ("fused_shards", C.c_uint32),
                ("shards", C.c_uint32), ("pad", C.c_uint32), ("ms", C.c_double * 4)]


# (name, restype, argtypes) of every entry point declared in include/ohx.h
PROTOTYPES = [
    ("ohx_abi_version", C.c_int, []),
    ("ohx_last_error", C.c_char_p, []),
    ("ohx_device_count", C.c_int, [C.POINTER(C.c_int)]),
    ("ohx_ctx_create", C.c_int, [C.c_int, C.POINTER(_vp)]),
    ("ohx_ctx_destroy", C.c_int, [_vp]),
    ("ohx_ctx_trim", C.c_int, [_vp]),
    ("ohx_ctx_default", C.c_int, [C.c_int, C.POINTER(_vp)]),
    ("ohx_ctx_device", C.c_int, [_vp]),
    ("ohx_ctx_launches", _u64, [_vp]),
    ("ohx_ctx_kernel_ms", C.c_int, [_vp, _dp]),
    ("ohx_ctx_kernel_ms_sum", C.c_int, [_vp, _dp, _u64p, C.c_int]),
    ("ohx_ctx_last_run", C.c_int, [_vp, C.POINTER(RunInfo)]),
    ("ohx_extremes", C.c_int, [_vp, _vp, _u64, _u64, C.POINTER(ExtremesRec), _vp]),
    ("ohx_fused_extremes", C.c_int, [_vp, _vp, _u64, _u64, C.POINTER(ExtremesRec),
                                     C.POINTER(C.c_int), _vp]),
    ("ohx_filter_fused", C.c_int, [_vp, _vp, _u64, _u64, C.POINTER(ExtremeSet),
                                   C.POINTER(FilterPlan), _vp, _u64p, C.POINTER(C.c_int), _vp]),
    ("ohx_extremes_combine", C.c_int, [C.POINTER(ExtremesRec), C.c_int, C.POINTER(ExtremesRec)]),
    ("ohx_extremes_resolve", C.c_int, [C.POINTER(ExtremesRec), C.POINTER(ExtremeSet),
                                       C.POINTER(C.c_uint32)]),
    ("ohx_corners_exact", C.c_int, [_vp, _vp, _u64, _u64, _dp, C.POINTER(CornerRec), _vp]),
    ("ohx_corners_combine", C.c_int, [C.POINTER(CornerRec), C.c_int, C.POINTER(CornerRec)]),
    ("ohx_build_octagon", C.c_int, [_dp, _dp, C.POINTER(C.c_int)]),
    ("ohx_filter_plan_build", C.c_int, [C.POINTER(ExtremeSet), _dp, C.c_int,
                                        C.POINTER(FilterPlan)]),
    ("ohx_filter", C.c_int, [_vp, _vp, _u64, _u64, C.POINTER(FilterPlan), _vp, _u64p, _vp]),
    ("ohx_queue_fetch", C.c_int, [_vp, C.c_int, _u64p, _dp, _u64, _vp]),
    ("ohx_queue_device", C.c_int, [_vp, C.c_int, C.POINTER(_vp), C.POINTER(C.c_int),
                                   C.POINTER(_u64)]),
    ("ohx_heaphull", C.c_int, [_dp, _u64, _dp, _u64, _u64p, _dp]),
    ("ohx_heaphull_device", C.c_int, [_vp, _vp, _u64, _dp, _u64, _u64p, _dp]),
    ("ohx_heaphull_device_out", C.c_int, [_vp, _vp, _u64, _vp, _u64, _u64p, _dp]),
    ("ohx_hull_indices", C.c_int, [_vp, _dp, _u64, _u64p, _vp]),
    ("ohx_hull_indices_partial", C.c_int, [_vp, _dp, _u64, _u64p, _vp]),
    ("ohx_classify", C.c_int, [_dp, _u64, _u8p]),
    ("ohx_classify_points", C.c_int, [_dp, _u64, _dp, _u64, _u64p, _u8p]),
    ("ohx_heaphull_run", C.c_int, [_dp, _u64, _dp, _u64, _u64p, _u8p, _dp]),
    ("ohx_pts2_count", C.c_int, [C.c_char_p, _u64p]),
    ("ohx_pts2_load_device", C.c_int, [_vp, C.c_char_p, _vp, _u64, _u64p, _vp]),
    ("ohx_heaphull_pts2", C.c_int, [C.c_char_p, _dp, _u64, _u64p, _dp]),
    ("ohx_find_extremes", C.c_int, [_dp, _u64, _u64p]),
    ("ohx_monotone_chain", C.c_int, [_dp, _u64, _dp, _u64, _u64p]),
    ("ohx_chain", C.c_int, [_dp, _u64, _dp, _u64p]),
    ("ohx_hull_from_sorted_arcs", C.c_int, [C.POINTER(_dp), _u64p, _dp, _u64, _u64p]),
    ("ohx_hull_from_sorted_arcs_device", C.c_int, [_vp, _vp, _u64p, _dp, _u64, _u64p,
                                                   C.POINTER(C.c_int), C.c_int, _vp]),
    ("ohx_generate", C.c_int, [C.c_int, _u64, _u64, C.c_double, _dp, C.c_int]),
    ("ohx_generate_range", C.c_int, [C.c_int, _u64, _u64, C.c_double, _u64, _u64, _dp, C.c_int]),
    ("ohx_hull_from_queues", C.c_int, [_dp, _u64p, C.POINTER(_u64p), _u64p, _dp, _u64, _u64p]),
    ("ohx_hull_from_queue_points", C.c_int, [_dp, C.POINTER(_dp), _u64p, _dp, _u64, _u64p]),
    ("ohx_mg_unique_id", C.c_int, [C.POINTER(C.c_uint8)]),
    ("ohx_mg_init_rank", C.c_int, [C.POINTER(C.c_uint8), C.c_int, C.c_int, C.c_int,
                                   C.POINTER(_vp)]),
    ("ohx_mg_init_all", C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(_vp)]),
    ("ohx_mg_destroy", C.c_int, [_vp]),
    ("ohx_mg_world", C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("ohx_mg_nccl_version", C.c_int, [C.POINTER(C.c_int)]),
    ("ohx_mg_ctx", C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(_vp)]),
    ("ohx_mg_heaphull_shard", C.c_int, [_vp, _vp, _u64, _u64, C.c_int, _u8p, _dp, _u64, _u64p,
                                        C.POINTER(MgInfo)]),
    ("ohx_mg_heaphull_device", C.c_int, [_vp, C.c_int, C.POINTER(_vp), _u64p, _u8p, _dp, _u64,
                                         _u64p, C.POINTER(MgInfo)]),
    ("ohx_mg_heaphull", C.c_int, [_vp, _dp, _u64, C.c_int, _u8p, _dp, _u64, _u64p,
                                  C.POINTER(MgInfo)]),
]


class OhxError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python paper_2209_12310_b200/build.py` "
            "(there is no CPU fallback for the filter)")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in PROTOTYPES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(code: int) -> None:
    """Raise for a non-zero status: ValueError for the reference's
    std::invalid_argument (as pybind11 maps it), RuntimeError otherwise."""
    if code == OHX_OK:
        return
    msg = lib.ohx_last_error().decode()
    if code == OHX_E_INVALID:
        raise ValueError(msg)
    raise OhxError(code, msg)
