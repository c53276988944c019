"""CPU oracle for the radix-tree-forest sampler (arXiv 1901.05423).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product package ``paper_1901_05423_b200`` never imports it and
shares no code with it (the oracle is plain serial C in ``rtf_oracle.c``, built
with gcc; this module is argument marshalling only).

Every function follows the paper step by step; see the header of
``rtf_oracle.c`` for the step list (O1..O12) with PAPER.md line citations, and
DESIGN.md section 3 for the readings (R1..R17) and the pin of each function.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rtf_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, EINVAL, EALLZERO, ETOOLARGE = 0, 1, 2, 3
ONE = 1 << 63  # fixed-point 1.0 (reading R4)


def build_oracle(force: bool = False) -> str:
    """Compile rtf_oracle.c with gcc (plain C, -O2, single thread)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-shared",
                               "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build_oracle())
        P = ctypes.c_void_p
        u32, u64, i32 = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32
        lib.orc_quantize.argtypes = [P, u32, P, P, P]
        lib.orc_cdf_all.argtypes = [P, u32, P, P]
        lib.orc_build.argtypes = [P, u32, u32, P, P, P, P, P, P, P, P, P]
        lib.orc_sample.argtypes = [P, P, P, P, u32, P, u64, P, P]
        lib.orc_sample.restype = None
        lib.orc_sample_bsearch.argtypes = [P, u32, P, u64, P]
        lib.orc_sample_bsearch.restype = None
        lib.orc_build_rows.argtypes = [P, u32, u32, u32, P, P, P, P, P, P, P, P, P, P]
        for f in (lib.orc_quantize, lib.orc_cdf_all, lib.orc_build, lib.orc_build_rows):
            f.restype = i32
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


class OracleError(ValueError):
    def __init__(self, status: int):
        super().__init__({EINVAL: "EINVAL", EALLZERO: "EALLZERO",
                          ETOOLARGE: "ETOOLARGE"}.get(status, str(status)))
        self.status = status


def _f32(p) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(p, dtype=np.float32))


def quantize(p):
    """O1-O3: returns (w uint64[n], E, B)."""
    p = _f32(p)
    w = np.zeros(max(p.size, 1), dtype=np.uint64)
    E, B = ctypes.c_int(0), ctypes.c_int(0)
    st = _load().orc_quantize(_ptr(p), p.size, _ptr(w), ctypes.byref(E), ctypes.byref(B))
    if st:
        raise OracleError(st)
    return w[: p.size], E.value, B.value


def cdf_all(p):
    """Fixed-point CDF over all n entries (zeros included): (K uint64[n], T)."""
    p = _f32(p)
    K = np.zeros(max(p.size, 1), dtype=np.uint64)
    T = ctypes.c_uint64(0)
    st = _load().orc_cdf_all(_ptr(p), p.size, _ptr(K), ctypes.byref(T))
    if st:
        raise OracleError(st)
    return K[: p.size], T.value


@dataclass
class Forest:
    """Oracle forest.  Arrays are indexed by the compacted leaf / node index j."""
    n: int
    m: int
    n_pos: int
    T: int
    key: np.ndarray      # uint64[n_pos]
    orig: np.ndarray     # int32[n_pos]
    cell: np.ndarray     # uint32[n_pos]
    lam: np.ndarray      # uint8[n_pos]   split levels (64 = boundary)
    child0: np.ndarray   # int32[n_pos]
    child1: np.ndarray   # int32[n_pos]
    table: np.ndarray    # int32[m]

    def records(self) -> np.ndarray:
        """The 16-byte node records {u64 key; i32 child0; i32 child1} as a
        structured array (the layout of Sec.3.2 P:1082-1083 interleaving)."""
        r = np.zeros(self.n_pos, dtype=[("key", "<u8"), ("c0", "<i4"), ("c1", "<i4")])
        r["key"], r["c0"], r["c1"] = self.key, self.child0, self.child1
        return r

    def sample(self, xi, with_loads: bool = False):
        xi = np.ascontiguousarray(np.asarray(xi, dtype=np.uint32))
        out = np.empty(xi.size, dtype=np.int32)
        loads = np.empty(xi.size, dtype=np.uint32) if with_loads else None
        _load().orc_sample(_ptr(self.key), _ptr(self.child0), _ptr(self.child1),
                           _ptr(self.table), self.m, _ptr(xi), xi.size, _ptr(out),
                           _ptr(loads) if with_loads else None)
        return (out, loads) if with_loads else out

    def table2(self) -> np.ndarray:
        """O13: the guide table with the paper's "exactly two intervals" flag
        (Sec.3.2: "further information could also be stored in the
        reference, such as a flag that there are exactly two intervals that
        overlap the cell.  Then, only one comparison must be performed and
        there is no need to explicitly store a node"; reading R18).  Entry
        (key32, ref), from the O10 table, written out cell by cell:
          * empty cell (table = ~i):              (0, ~i)
          * a cell holding exactly one leaf a, overlapped by intervals a-1 and a,
            with orig(a) = orig(a-1) + 1 (no zero weight between them):
            (ceil(key_a / 2^31), ~orig(a)) -- xi < key32 means interval a-1,
            whose reference ~orig(a-1) is ~orig(a) + 1;
            if ceil(key_a / 2^31) = 2^32 no xi of the cell reaches a: (0, ~orig(a-1));
            if a = 0 (key 0) every xi of the cell is in a: (0, ~orig(0))
          * any other non-empty cell: (0, anchor a) -- the node of O10.
        Sampling: ref >= 0 -> Alg. 2 from node ref; ref < 0 -> the leaf
        ~(xi < key32 ? ref + 1 : ref)."""
        return table2_of(self.table, self.key, self.orig, self.cell, self.m)

    def table3(self) -> np.ndarray:
        """O16: the guide table with three-interval cells packed (R20); the
        table the build produces."""
        return table3_of(self.table2(), self.key, self.orig, self.cell, self.m)

    def sample_table3(self, xi) -> np.ndarray:
        """Alg. 2 through the O16 table: plain Python loop."""
        t3 = self.table3()
        rec = self.records()
        shift = 32 - (self.m.bit_length() - 1)
        out = np.empty(len(xi), dtype=np.int32)
        for k, x in enumerate(np.asarray(xi, dtype=np.uint64).tolist()):
            g = (x * self.m) >> 32
            key32, ref = int(t3[g]["key32"]), int(t3[g]["ref"])
            if ref >= 0 and key32:  # three intervals: ref = orig(a-1)
                xi0 = g << shift
                out[k] = ref + (x >= xi0 + (key32 & 0xFFFF)) + (x >= xi0 + (key32 >> 16))
                continue
            if ref < 0:
                out[k] = ~(ref + 1 if x < key32 else ref)
                continue
            j = ref
            while j >= 0:
                j = int(rec[j]["c0"]) if (x << 31) < int(rec[j]["key"]) else int(rec[j]["c1"])
            out[k] = ~j
        return out

    def cell_depths(self) -> tuple[np.ndarray, np.ndarray]:
        """O17 helper: per cell g, (D_g, k_g).  k_g = leaves whose cell is g;
        D_g = the most node records Alg. 2 (through the O10 table)
        visits for any 32-bit xi of cell g: 1 for the anchor's left child
        (interval a-1), else the visits to the leaf j that xi_j =
        ceil(key_j / 2^31) reaches, over the leaves j reachable by a 32-bit xi
        (ceil(key_j / 2^31) < ceil(key_{j+1} / 2^31), key_{n'} = 2^63), each
        counted in the cell of xi_j (every xi mapping to leaf j follows the
        same path, and xi_j is the first of them).  D_g = 0 for cells without
        an anchor."""
        kc = np.array([-(-int(k) >> 31) for k in self.key] + [1 << 32], dtype=np.uint64)
        reach = np.flatnonzero(kc[:-1] < kc[1:])
        xs = kc[reach].astype(np.uint32)
        _, loads = self.sample(xs, with_loads=True)
        cells = ((xs.astype(np.uint64) * np.uint64(self.m)) >> np.uint64(32)).astype(np.int64)
        D = np.zeros(self.m, dtype=np.int64)
        np.maximum.at(D, cells, loads.astype(np.int64) - 1)
        D[self.table >= 0] = np.maximum(D[self.table >= 0], 1)
        k = np.bincount(self.cell.astype(np.int64), minlength=self.m)
        return D, k

    def table4(self) -> np.ndarray:
        """O17: the O16 table with degenerate cells marked for bisection (R21)."""
        D, k = self.cell_depths()
        return table4_of(self.table3(), D, k)

    def sample_table4(self, xi, with_loads: bool = False):
        """Alg. 2 through the O17 table: a marked cell is searched by bisection
        of the index interval [a-1, a+k) of the intervals overlapping it (Sec.6
        P:1545-1548: "the implicit balanced tree is traversed by consecutive
        bisection of the index interval"); every other cell as sample_table3.
        with_loads: also the node records read after the table (bisection:
        one per probe)."""
        t4 = self.table4()
        rec = self.records()
        shift = 32 - (self.m.bit_length() - 1)
        out = np.empty(len(xi), dtype=np.int32)
        visits = np.zeros(len(xi), dtype=np.int32)
        for q, x in enumerate(np.asarray(xi, dtype=np.uint64).tolist()):
            g = (x * self.m) >> 32
            key32, ref = int(t4[g]["key32"]), int(t4[g]["ref"])
            if ref >= 0 and key32 >> 30 == 3:  # bisection over the intervals a-1 .. a+k-1
                a, kk = ref, key32 & 0x3FFFFFFF
                lo, hi = a - 1, a + kk  # key_lo <= x 2^31 < key_hi
                while hi - lo > 1:
                    mid = (lo + hi) // 2
                    visits[q] += 1
                    if int(self.key[mid]) <= (x << 31):
                        lo = mid
                    else:
                        hi = mid
                out[q] = int(self.orig[lo])
                continue
            if ref >= 0 and key32:  # three intervals (O16)
                xi0 = g << shift
                out[q] = ref + (x >= xi0 + (key32 & 0xFFFF)) + (x >= xi0 + (key32 >> 16))
                continue
            if ref < 0:
                out[q] = ~(ref + 1 if x < key32 else ref)
                continue
            j = ref
            while j >= 0:
                visits[q] += 1
                j = int(rec[j]["c0"]) if (x << 31) < int(rec[j]["key"]) else int(rec[j]["c1"])
            out[q] = ~j
        return (out, visits) if with_loads else out

    def sample_table2(self, xi) -> np.ndarray:
        """Alg. 2 through the O13 table: plain Python loop."""
        t2 = self.table2()
        rec = self.records()
        out = np.empty(len(xi), dtype=np.int32)
        for k, x in enumerate(np.asarray(xi, dtype=np.uint64).tolist()):
            key32, ref = int(t2[(x * self.m) >> 32]["key32"]), int(t2[(x * self.m) >> 32]["ref"])
            if ref < 0:
                out[k] = ~(ref + 1 if x < key32 else ref)
                continue
            j = ref
            while j >= 0:
                j = int(rec[j]["c0"]) if (x << 31) < int(rec[j]["key"]) else int(rec[j]["c1"])
            out[k] = ~j
        return out


PACK_MIN_M = 1 << 17  # O16 packs cells of m >= 2^17 power-of-two tables (R20)


def table3_of(t2, key, orig, cell, m) -> np.ndarray:
    """O16 (reading R20): the O13 table with every cell that holds exactly two
    leaves a, a+1 -- overlapped by the three intervals a-1, a, a+1 --
    stored in the 8-byte entry itself, carrying the paper's idea that
    "further information could also be stored in the reference" so that
    "there is no need to explicitly store a node" (Sec.3.2) one
    step further than the two-interval flag.  Only for a power-of-two m >=
    2^17 (a cell is then at most 2^15 xi values wide, xi0 = g 2^32 / m its
    first xi), when a >= 1 and orig(a+1) = orig(a-1) + 2 (no zero weight
    between the three intervals):
        key32 = s1 | s2 << 16,  s = ceil(key / 2^31) - xi0 for key_a, key_{a+1}
        ref   = orig(a-1)  (>= 0, as an anchor's; key32 != 0 tells them apart:
                            s2 >= 1 because key_{a+1} > xi0 2^31)
    Sampling: ref + [xi >= xi0 + s1] + [xi >= xi0 + s2] (xi 2^31 < key <=>
    xi < ceil(key / 2^31), so the comparisons are Alg. 2's).  Every other
    cell and any other m: the O13 entry."""
    out = np.array(t2, dtype=TABLE2_DTYPE, copy=True)
    if m < PACK_MIN_M or (m & (m - 1)):
        return out
    shift = 32 - (m.bit_length() - 1)  # xi0 = g << shift
    leaves_per_cell = np.bincount(cell.astype(np.int64), minlength=m)
    for g in np.flatnonzero((out["ref"] >= 0) & (leaves_per_cell == 2)).tolist():
        a = int(out["ref"][g])  # the anchor: the cell's first leaf
        if a == 0 or int(orig[a + 1]) != int(orig[a - 1]) + 2:
            continue
        xi0 = g << shift
        s1 = -(-int(key[a]) >> 31) - xi0
        s2 = -(-int(key[a + 1]) >> 31) - xi0
        out[g] = (s1 | (s2 << 16), int(orig[a - 1]))
    return out


FALLBACK_SLACK = 4  # O17 (reading R21): the depth allowed above binary search


def bisect_visits(k: int) -> int:
    """Node records a bisection of the k + 1 intervals overlapping a cell with
    k leaves reads at most: ceil(log2(k + 1))."""
    return (k).bit_length() if k > 0 else 0  # ceil(log2(k + 1)) for k >= 0


def table4_of(t3, D, k) -> np.ndarray:
    """O17 (reading R21): the fallback of Sec.3 P:983-984 ("for degenerate
    hierarchical structures the worst case may increase ... a fallback method
    constructs such a structure upon detection to guarantee logarithmic
    complexity"), with the balanced tree of Sec.6 P:1545-1548 that "does not
    need to be built" (bisection of the index interval) and the criterion of
    Sec.4 P:1516-1518 (an explicit tree only pays "if the maximum depth does
    not exceed the number of comparisons required for binary search").  A cell
    whose O16 entry is an anchor (key32 = 0, ref = a >= 0) and that holds k_g <
    2^30 leaves is marked when its radix depth D_g exceeds the bisection's
    ceil(log2(k_g + 1)) node reads by more than FALLBACK_SLACK:
        key32 = 3 << 30 | k_g,  ref = a
    (an O16 packed entry never has both top bits set: s2 <= 2^15, and s2 =
    2^15 leaves s1 < 2^15 in the low bits).  Every other entry: the O16 entry."""
    out = np.array(t3, dtype=TABLE2_DTYPE, copy=True)
    for g in np.flatnonzero((out["ref"] >= 0) & (out["key32"] == 0)).tolist():
        kk = int(k[g])
        if kk < (1 << 30) and int(D[g]) > bisect_visits(kk) + FALLBACK_SLACK:
            out[g] = ((3 << 30) | kk, int(out["ref"][g]))
    return out


def is_bisect(t4) -> np.ndarray:
    """O17 marks: ref >= 0 and both top bits of key32 set."""
    return (t4["ref"] >= 0) & ((t4["key32"] >> 30) == 3)


def table2_of(table, key, orig, cell, m) -> np.ndarray:
    """O13 for one distribution's O10 table, keys, original indices and cells
    (see Forest.table2)."""
    out = np.zeros(m, dtype=TABLE2_DTYPE)
    out["ref"] = table
    leaves_per_cell = np.bincount(cell.astype(np.int64), minlength=m)
    one = np.flatnonzero((table >= 0) & (leaves_per_cell == 1))  # two intervals
    a = table[one].astype(np.int64)
    kc = [-(-int(k) >> 31) for k in key[a]]  # ceil(key_a / 2^31), exact ints
    for g, ai, c in zip(one.tolist(), a.tolist(), kc):
        if c == 0:                  # a = 0: the cell lies inside interval a
            out[g] = (0, ~int(orig[ai]))
        elif c == 1 << 32:          # no xi of the cell reaches interval a
            out[g] = (0, ~int(orig[ai - 1]))
        elif int(orig[ai]) == int(orig[ai - 1]) + 1:
            out[g] = (c, ~int(orig[ai]))
    return out


TABLE2_DTYPE = np.dtype([("key32", "<u4"), ("ref", "<i4")])


def build(p, m: int) -> Forest:
    """O1-O11 for one distribution."""
    p = _f32(p)
    n = p.size
    nn = max(n, 1)
    key = np.zeros(nn, np.uint64)
    orig = np.zeros(nn, np.int32)
    cell = np.zeros(nn, np.uint32)
    lam = np.zeros(nn, np.uint8)
    c0 = np.zeros(nn, np.int32)
    c1 = np.zeros(nn, np.int32)
    table = np.zeros(max(m, 1), np.int32)
    T = ctypes.c_uint64(0)
    npos = ctypes.c_uint32(0)
    st = _load().orc_build(_ptr(p), n, m, _ptr(key), _ptr(orig), _ptr(cell), _ptr(lam),
                           _ptr(c0), _ptr(c1), _ptr(table), ctypes.byref(T), ctypes.byref(npos))
    if st:
        raise OracleError(st)
    k = npos.value
    return Forest(n, m, k, T.value, key[:k], orig[:k], cell[:k], lam[:k], c0[:k], c1[:k],
                  table[:m])


def sample_bsearch(K: np.ndarray, xi) -> np.ndarray:
    """Binary search on the full fixed-point CDF (Sec.2.2): independent of the forest."""
    K = np.ascontiguousarray(K, dtype=np.uint64)
    xi = np.ascontiguousarray(np.asarray(xi, dtype=np.uint32))
    out = np.empty(xi.size, dtype=np.int32)
    _load().orc_sample_bsearch(_ptr(K), K.size, _ptr(xi), xi.size, _ptr(out))
    return out


def build_rows(p, rows: int, n_row: int, m_row: int):
    """Batched independent rows (Sec.5).  Returns dict of arrays laid
    out row-major with per-row stride n_row (nodes) / m_row (table), plus the
    per-row T, n_pos and status."""
    p = _f32(p).reshape(-1)
    assert p.size == rows * n_row
    N = rows * n_row
    out = dict(key=np.zeros(N, np.uint64), orig=np.zeros(N, np.int32),
               cell=np.zeros(N, np.uint32), lam=np.zeros(N, np.uint8),
               child0=np.zeros(N, np.int32), child1=np.zeros(N, np.int32),
               table=np.zeros(rows * m_row, np.int32), T=np.zeros(rows, np.uint64),
               n_pos=np.zeros(rows, np.uint32), status=np.zeros(rows, np.int32))
    _load().orc_build_rows(_ptr(p), rows, n_row, m_row, *(_ptr(out[k]) for k in (
        "key", "orig", "cell", "lam", "child0", "child1", "table", "T", "n_pos", "status")))
    return out


# ---------------------------------------------------------------- 2-D (Sec.6)

def _f32_floor_log2(x: np.float32) -> int:
    """floor(log2 x) of a positive finite float32, from its bits (O2)."""
    b = int(np.float32(x).view(np.uint32))
    e = (b >> 23) & 0xFF
    if e:
        return e - 127
    return (b & 0x7FFFFF).bit_length() - 1 - 149


def marginal_weights(p2d) -> np.ndarray:
    """O14: the row weights of a 2-D distribution (Sec.6: "first
    calculating the cumulative distribution function of the image rows").  Row
    y's quantised mass is T_y 2^(E_y - B_y) (O2-O5 applied to the row alone,
    reading R15); with K = max over non-empty rows of E_y - B_y the weight is
    q_y = float32(float64(T_y) * 2^(E_y - B_y - K)) (two round-to-nearest steps,
    reading R19); an all-zero row gets 0."""
    p2d = np.ascontiguousarray(np.asarray(p2d, dtype=np.float32))
    H, W = p2d.shape
    B = 62 - max(0, (W - 1).bit_length())
    T, k = [], []
    for y in range(H):
        row = p2d[y]
        if not np.any(row > 0):
            T.append(0)
            k.append(None)
            continue
        f = build(row, 1)
        T.append(int(f.T))
        k.append(_f32_floor_log2(row.max()) - B)
    K = max(v for v in k if v is not None)
    q = np.zeros(H, np.float32)
    for y in range(H):
        if T[y]:
            q[y] = np.float32(math.ldexp(float(T[y]), k[y] - K))
    return q


def _f32_rz(d):
    """float64 -> float32 rounded toward zero (element-wise)."""
    d = np.asarray(d, np.float64)
    f = d.astype(np.float32)
    over = np.abs(f.astype(np.float64)) > np.abs(d)
    f[over] = np.nextafter(f[over], np.float32(0))
    return f


@dataclass
class Forest2D:
    """O14-O15: marginal forest over the row weights + one conditional forest
    per row (Sec.6)."""
    W: int
    H: int
    marginal: Forest
    rows: list  # Forest per row (None for an all-zero row)

    @staticmethod
    def _positions(f: Forest, idx: np.ndarray, xi: np.ndarray) -> np.ndarray:
        """Relative position of each xi inside interval idx of forest f (the
        sub-pixel rescale of P:1526-1528): float64(xi 2^31 - key_j) /
        float64(key_{j+1} - key_j), each integer rounded to nearest once
        (numpy's uint64 -> float64 conversion rounds to nearest, as
        Python's float(int) does); j is the leaf of original index idx."""
        j_of = np.full(f.n, -1, np.int64)
        j_of[f.orig] = np.arange(f.n_pos)
        j = j_of[np.asarray(idx, np.int64)]
        keys = np.append(f.key.astype(np.uint64), np.uint64(ONE))  # key_{n'} = "1"
        lo, hi = keys[j], keys[j + 1]
        num = (np.asarray(xi, np.uint64) << np.uint64(31)) - lo
        return num.astype(np.float64) / (hi - lo).astype(np.float64)

    def sample(self, xi1, xi2):
        """O15: y = marginal^-1(xi1); x = row_y^-1(xi2); the continuous position
        ((x + v) / W, (y + u) / H) in float64, rounded toward zero to float32
        (so it stays below 1, reading R19), u and v the relative
        positions inside the chosen intervals.  Returns (pixel = y W + x,
        pos float32[N, 2] as (x, y)).  The samples of one row go through that
        row's forest together."""
        xi1 = np.asarray(xi1, dtype=np.uint32)
        xi2 = np.asarray(xi2, dtype=np.uint32)
        ys = self.marginal.sample(xi1).astype(np.int64)
        xs = np.empty(xi1.size, np.int64)
        v = np.empty(xi1.size, np.float64)
        order = np.argsort(ys, kind="stable")
        ys_sorted = ys[order]
        bounds = np.flatnonzero(np.diff(ys_sorted)) + 1
        for sel in np.split(order, bounds):
            if sel.size == 0:
                continue
            fr = self.rows[int(ys[sel[0]])]
            xs[sel] = fr.sample(xi2[sel])
            v[sel] = self._positions(fr, xs[sel], xi2[sel])
        u = self._positions(self.marginal, ys, xi1)
        pix = (ys * self.W + xs).astype(np.int32)
        pos = np.empty((xi1.size, 2), np.float32)
        pos[:, 0] = _f32_rz((xs.astype(np.float64) + v) / float(self.W))
        pos[:, 1] = _f32_rz((ys.astype(np.float64) + u) / float(self.H))
        return pix, pos


def build_2d(p2d, m_x: int, m_y: int) -> Forest2D:
    p2d = np.ascontiguousarray(np.asarray(p2d, dtype=np.float32))
    H, W = p2d.shape
    q = marginal_weights(p2d)
    rows = [build(p2d[y], m_x) if np.any(p2d[y] > 0) else None for y in range(H)]
    return Forest2D(W, H, build(q, m_y), rows)
