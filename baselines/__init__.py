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
        lib.alias_build_counts.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_int,
                                           ctypes.c_void_p, ctypes.c_void_p]
        lib.alias_build_counts.restype = ctypes.c_int
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


def alias_from_counts(counts: np.ndarray):
    """Alias table realising per-item xi counts (summing to 2^32): (prob, alias, k)."""
    c = np.ascontiguousarray(counts, dtype=np.uint64)
    k = 1
    while (1 << k) < c.size:
        k += 1
    prob = np.empty(1 << k, np.uint32)
    alias = np.empty(1 << k, np.int32)
    if _load().alias_build_counts(c.ctypes.data, c.size, k, prob.ctypes.data, alias.ctypes.data):
        raise MemoryError("alias_build_counts")
    return prob, alias, k


def counts_from_cdf(K: np.ndarray) -> np.ndarray:
    """Exact xi counts the inverse mapping gives each item of a full fixed-point
    CDF K[0..n) (K_n = 2^63): c_i = ceil(K_{i+1}/2^31) - ceil(K_i/2^31)."""
    kc = (np.asarray(K, np.uint64) + np.uint64((1 << 31) - 1)) >> np.uint64(31)
    return np.diff(np.append(kc, np.uint64(1 << 32)).astype(np.int64)).astype(np.uint64)


def alias_2d(K_marg: np.ndarray, K_rows):
    """Tables of the 2-D alias baseline: the marginal over the rows' fixed-point
    CDF K_marg and one table per row (K_rows[y], or None for a zero-weight row,
    which the marginal never selects: uniform filler).  Returns ((prob, alias,
    ky), (prob[H, 2^kx], alias[H, 2^kx], kx))."""
    marg = alias_from_counts(counts_from_cdf(K_marg))
    W = max(len(K) for K in K_rows if K is not None)
    kx = 1
    while (1 << kx) < W:
        kx += 1
    H = len(K_rows)
    prob = np.empty((H, 1 << kx), np.uint32)
    alias = np.empty((H, 1 << kx), np.int32)
    for y, K in enumerate(K_rows):
        if K is None:
            prob[y], alias[y] = np.uint32(1 << (32 - kx)), np.arange(1 << kx, dtype=np.int32)
            continue
        c = counts_from_cdf(K)
        c = np.concatenate([c, np.zeros((1 << kx) - c.size, np.uint64)])
        prob[y], alias[y], _ = alias_from_counts(c)
    return marg, (prob, alias, kx)
