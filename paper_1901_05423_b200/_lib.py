"""ctypes declarations of librtf.so (include/rtf.h).  Loading fails loudly when
the library is missing: there is no fallback implementation."""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "librtf.so")

RTF_OK, RTF_EINVAL, RTF_EALLZERO, RTF_ETOOLARGE, RTF_ENOSPACE, RTF_ECUDA, RTF_EDATA = range(7)
RTF_DATA_NAN, RTF_DATA_INF, RTF_DATA_NEG, RTF_DATA_ALLZERO = 1, 2, 4, 8
RTF_BUILD_DEFAULT, RTF_BUILD_SMALL_TILES = 0, 1


class rtf_header(ctypes.Structure):
    _fields_ = [("total", ctypes.c_uint64), ("recip", ctypes.c_uint64),
                ("n_pos", ctypes.c_uint32), ("exponent", ctypes.c_int32),
                ("scale_bits", ctypes.c_int32), ("status", ctypes.c_uint32),
                ("norm_shift", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


class rtf_forest(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint32), ("m", ctypes.c_uint32), ("rows", ctypes.c_uint32),
                ("flags", ctypes.c_uint32), ("nodes", ctypes.c_void_p),
                ("table", ctypes.c_void_p), ("header", ctypes.c_void_p)]


class rtf_forest2d(ctypes.Structure):
    _fields_ = [("W", ctypes.c_uint32), ("H", ctypes.c_uint32), ("mx", ctypes.c_uint32),
                ("my", ctypes.c_uint32), ("rows", rtf_forest), ("marginal", rtf_forest),
                ("rows_jmap", ctypes.c_void_p), ("marg_jmap", ctypes.c_void_p),
                ("weights", ctypes.c_void_p), ("rows_dense", ctypes.c_void_p)]


class rtf_shard_view(ctypes.Structure):
    _fields_ = [("spine", ctypes.c_void_p), ("scale", ctypes.c_void_p), ("total", ctypes.c_void_p),
                ("nt_local", ctypes.c_uint32), ("spine_row_bytes", ctypes.c_uint32),
                ("nt_cap", ctypes.c_uint32), ("reserved", ctypes.c_uint32),
                ("jbound", ctypes.c_void_p)]


# name -> (restype, argtypes)
_P, _U32, _U64, _I32, _SZ = (ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int,
                             ctypes.c_size_t)
_F = ctypes.POINTER(rtf_forest)
_H = ctypes.POINTER(rtf_header)
PROTOTYPES = {
    "rtf_forest_bytes": (_SZ, [_U32, _U32, _U32]),
    "rtf_workspace_bytes": (_SZ, [_U32, _U32, _U32]),
    "rtf_workspace_init": (_I32, [_P, _SZ, _U32, _U32, _U32, _P]),
    "rtf_build": (_I32, [_P, _U32, _U32, _U32, _P, _SZ, _P, _SZ, _P, _F]),
    "rtf_build_rows": (_I32, [_P, _U32, _U32, _U32, _P, _SZ, _P, _F]),
    "rtf_forest_view": (_I32, [_P, _SZ, _U32, _U32, _U32, _F]),
    "rtf_forest_status": (_I32, [_F, _P, _H]),
    "rtf_sample": (_I32, [_F, _P, _U64, _P, _P]),
    "rtf_sample_f32": (_I32, [_F, _P, _U64, _P, _P]),
    "rtf_sample_loads": (_I32, [_F, _P, _U64, _P, _P, _P]),
    "rtf_quad_bytes": (_SZ, [_U32]),
    "rtf_build_quad": (_I32, [_F, _P, _SZ, _P]),
    "rtf_sample_quad": (_I32, [_F, _P, _P, _U64, _P, _P]),
    "rtf_sample_rows": (_I32, [_F, _P, _P, _U64, _P, _P]),
    "rtf_build_cdf": (_I32, [_P, _U32, _P, _P, _P, _SZ, _P]),
    "rtf_sample_bsearch": (_I32, [_P, _U32, _P, _P, _U64, _P, _P]),
    "rtf_sample_alias": (_I32, [_P, _U32, _P, _U64, _P, _P]),
    "rtf_sample_alias_2d": (_I32, [_P, _U32, _P, _U32, _U32, _U32, _P, _P, _U64, _P, _P]),
    "rtf_fallback_bytes": (_SZ, [_U32]),
    "rtf_build_fallback": (_I32, [_F, _P, _SZ, _P]),
    "rtf_eytzinger_slots": (_U64, [_U32]),
    "rtf_build_eytzinger": (_I32, [_P, _U32, _P, _P]),
    "rtf_sample_eytzinger": (_I32, [_P, _U32, _P, _P, _U64, _P, _P]),
    "rtf_forest2d_bytes": (_SZ, [_U32, _U32, _U32, _U32]),
    "rtf_build_2d": (_I32, [_P, _U32, _U32, _U32, _U32, _P, _SZ, _P,
                            ctypes.POINTER(rtf_forest2d)]),
    "rtf_forest2d_status": (_I32, [ctypes.POINTER(rtf_forest2d), _P]),
    "rtf_sample_2d": (_I32, [ctypes.POINTER(rtf_forest2d), _P, _P, _U64, _P, _P, _P]),
    "rtf_build_cutpoint": (_I32, [_P, _U32, _U32, _P, _P]),
    "rtf_sample_cutpoint": (_I32, [_P, _U32, _P, _P, _U32, _I32, _P, _U64, _P, _P]),
    "rtf_build_host": (_I32, [_P, _U32, _U32, _U32, _P, _P, _SZ, _P, _SZ, _P, _F, _H]),
    "rtf_sample_host": (_I32, [_F, _P, _U64, _P, _P, _P, _U64, _P]),
    "rtf_philox_u32": (_I32, [_U64, _U64, _U64, _P, _P]),
    "rtf_shard_workspace_bytes": (_SZ, [_U32, _U32, _U32]),
    "rtf_shard_workspace_init": (_I32, [_P, _SZ, _U32, _U32, _U32, _P]),
    "rtf_shard_get_view": (_I32, [_P, _SZ, _U32, _U32, _U32, ctypes.POINTER(rtf_shard_view)]),
    "rtf_shard_scale": (_I32, [_P, _U32, _U32, _U32, _P, _SZ, _P]),
    "rtf_shard_totals": (_I32, [_P, _U32, _U32, _U32, _U32, _P, _SZ, _P]),
    "rtf_shard_build": (_I32, [_P, _U32, _U32, _U32, _U32, _U32, _U32, _P, _P, _SZ, _P, _SZ, _P,
                               _F]),
    "rtf_shard_finish": (_I32, [_U32, _U32, _U32, _P, _U32, _P, _SZ, _P, _SZ, _P, _F]),
    "rtf_shard_finish_range": (_I32, [_U32, _U32, _U32, _P, _U32, _U32, _U32, _P, _SZ, _P, _SZ,
                                      _P, _F]),
    "rtf_shard_build_peers": (_I32, [_P, _U32, _U32, _U32, _U32, _U32, _U32, _P, _P, _U32, _P,
                                     _SZ, _P, _SZ, _P, _F]),
    "rtf_shard_count_cells": (_I32, [_P, _SZ, _U32, _U32, _U32, _U32, _P, _U32, _P, _P]),
    "rtf_shard_set_peers": (_I32, [_P, _SZ, _U32, _U32, _U32, _P, _U32, _SZ, _P]),
    "rtf_shard_finish_own": (_I32, [_U32, _U32, _U32, _P, _U32, _U32, _P, _SZ, _P, _SZ, _P, _F]),
    "rtf_launch_count": (_U64, []),
    "rtf_status_string": (ctypes.c_char_p, [_I32]),
    "rtf_version": (ctypes.c_char_p, []),
}

_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run `python __graft_entry__.py` "
                              "(build()) -- there is no fallback implementation")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class RtfError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        name = load().rtf_status_string(status).decode()
        super().__init__(f"{what}: {name}" if what else name)
        self.status = status


def check(status: int, what: str = "") -> None:
    if status != RTF_OK:
        raise RtfError(status, what)
