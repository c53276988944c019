"""Host-side comparison baselines reported by bench.py (not the product path,
not the oracle): cpu_bsearch.c, an OpenMP binary search over the full CDF;
alias.c, the alias table (Vose) the GPU alias sampler reads."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = [os.path.join(_HERE, "cpu_bsearch.c"), os.path.join(_HERE, "alias.c")]
_LIB = os.path.join(_HERE, "libcpu_bsearch.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or any(os.path.getmtime(_LIB) < os.path.getmtime(f)
                                                for f in _SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-march=native", "-fopenmp", "-shared", "-fPIC",
                               "-o", tmp, *_SRC])
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
        lib.alias_build.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p,
                                    ctypes.c_void_p]
        lib.alias_build.restype = ctypes.c_int
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


def alias_table(cdf: np.ndarray):
    """Alias table over the 32-bit xi grid from the full fixed-point CDF
    (alias.c): (prob u32[2^k], alias i32[2^k], k)."""
    cdf = np.ascontiguousarray(cdf, dtype=np.uint64)
    k = 1
    while (1 << k) < cdf.size:
        k += 1
    prob = np.empty(1 << k, np.uint32)
    alias = np.empty(1 << k, np.int32)
    got = _load().alias_build(cdf.ctypes.data, cdf.size, prob.ctypes.data, alias.ctypes.data)
    if got != k:
        raise MemoryError("alias_build")
    return prob, alias, k


def alias_sample(prob: np.ndarray, alias: np.ndarray, k: int, xi: np.ndarray) -> np.ndarray:
    """The alias table's answer for each xi (numpy, the definition)."""
    x = np.asarray(xi, dtype=np.uint64)
    b = (x >> np.uint64(32 - k)).astype(np.int64)
    o = x & np.uint64((1 << (32 - k)) - 1)
    return np.where(o < prob[b].astype(np.uint64), b, alias[b]).astype(np.int32)
