"""Host-side comparison baselines reported by bench.py (not the product path,
not the oracle): cpu_bsearch.c, an OpenMP binary search over the full CDF."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cpu_bsearch.c")
_LIB = os.path.join(_HERE, "libcpu_bsearch.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-march=native", "-fopenmp", "-shared", "-fPIC",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        lib.cpu_bsearch.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p,
                                    ctypes.c_uint64, ctypes.c_void_p]
        lib.cpu_bsearch.restype = None
        lib.cpu_bsearch_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def threads() -> int:
    return int(_load().cpu_bsearch_threads())


def bsearch(cdf: np.ndarray, xi: np.ndarray) -> np.ndarray:
    cdf = np.ascontiguousarray(cdf, dtype=np.uint64)
    xi = np.ascontiguousarray(xi, dtype=np.uint32)
    out = np.empty(xi.size, np.int32)
    _load().cpu_bsearch(cdf.ctypes.data, cdf.size, xi.ctypes.data, xi.size, out.ctypes.data)
    return out
