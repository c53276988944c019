"""paper_1901_05423_b200 -- radix-tree-forest sampling (Binder & Keller,
arXiv 1901.05423) on NVIDIA B200.

A thin binding over librtf.so (C ABI, include/rtf.h).  This module only
marshals arguments: device memory and streams come from PyTorch, every step of
the build and of sampling runs in the library's sm_100a kernels.  If the
library is missing, importing the ops raises -- there is no CPU fallback.

    import torch, paper_1901_05423_b200 as rtf
    f = rtf.build(p_cuda_float32, m)            # guide table + radix forest
    idx = rtf.sample(f, xi_cuda_uint32)         # Alg. 2, original indices
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import (RTF_BUILD_DEFAULT, RTF_BUILD_SMALL_TILES, RTF_DATA_ALLZERO,  # noqa: F401
                   RTF_DATA_INF, RTF_DATA_NAN, RTF_DATA_NEG, RtfError, check, rtf_forest,
                   rtf_forest2d, rtf_header)

__all__ = ["Forest", "RowsForest", "Forest2D", "build", "build_rows", "build_2d", "sample", "sample_rows",
           "build_cdf", "sample_bsearch", "philox", "build_host", "sample_host",
           "launch_count", "RtfError", "lib"]

NODE_DTYPE = np.dtype([("key", "<u8"), ("c0", "<i4"), ("c1", "<i4")])
CELL_DTYPE = np.dtype([("key32", "<u4"), ("ref", "<i4")])  # rtf_ref


def lib():
    return _lib.load()


def _stream(stream=None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def _u32_view(t: torch.Tensor) -> torch.Tensor:
    if t.dtype not in (torch.int32, torch.uint32):
        raise TypeError(f"expected a 32-bit integer tensor of fixed-point xi/2^32, got {t.dtype}")
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("xi must be a contiguous CUDA tensor")
    return t


def _bytes_tensor(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


@dataclass
class _Buffers:
    forest: torch.Tensor
    ws: torch.Tensor | None


class Forest:
    """A guide table + radix forest over n weights with m cells, in device memory
    owned by this object (forest buffer + build workspace)."""

    def __init__(self, n: int, m: int, flags: int = RTF_BUILD_DEFAULT, device="cuda"):
        L = lib()
        self.n, self.m, self.flags = int(n), int(m), int(flags)
        self.device = torch.device(device)
        fb = L.rtf_forest_bytes(self.n, self.m, 1)
        wb = L.rtf_workspace_bytes(self.n, self.m, self.flags)
        self._buf = _Buffers(_bytes_tensor(fb, self.device), _bytes_tensor(wb, self.device))
        self.view = rtf_forest()
        check(L.rtf_forest_view(_ptr(self._buf.forest), fb, self.n, self.m, 1,
                                ctypes.byref(self.view)), "rtf_forest_view")
        check(L.rtf_workspace_init(_ptr(self._buf.ws), wb, self.n, self.m, self.flags,
                                   _stream()), "rtf_workspace_init")

    @classmethod
    def from_buffer(cls, n: int, m: int, forest_buf: torch.Tensor) -> "Forest":
        """A read-only view (sampling, inspection) of a forest buffer built
        elsewhere, e.g. by the sharded build (paper_1901_05423_b200.sharded)."""
        f = cls.__new__(cls)
        f.n, f.m, f.flags, f.device = int(n), int(m), 0, forest_buf.device
        f._buf = _Buffers(forest_buf, None)
        f.view = rtf_forest()
        check(lib().rtf_forest_view(_ptr(forest_buf), forest_buf.numel(), f.n, f.m, 1,
                                    ctypes.byref(f.view)), "rtf_forest_view")
        return f

    # ---------------------------------------------------------------- build
    def build(self, p: torch.Tensor, stream=None) -> "Forest":
        if p.dtype != torch.float32 or not p.is_cuda or not p.is_contiguous():
            raise TypeError("p must be a contiguous float32 CUDA tensor")
        if p.numel() != self.n:
            raise ValueError(f"p has {p.numel()} entries, forest was sized for {self.n}")
        self._p = p  # keep alive while kernels run
        self._rec4_valid = False  # the 4-ary records describe the previous forest
        self._marked = False      # a rebuild writes an unmarked table
        check(lib().rtf_build(_ptr(p), self.n, self.m, self.flags, _ptr(self._buf.forest),
                              self._buf.forest.numel(), _ptr(self._buf.ws),
                              self._buf.ws.numel(), _stream(stream), ctypes.byref(self.view)),
              "rtf_build")
        return self

    # ---------------------------------------------------------------- sampling
    def sample(self, xi: torch.Tensor, out: torch.Tensor | None = None, stream=None):
        """xi: int32/uint32 fixed point xi/2^32, or float32 in [0, 1)."""
        if xi.dtype == torch.float32:
            if not xi.is_cuda or not xi.is_contiguous():
                raise ValueError("xi must be a contiguous CUDA tensor")
            if out is None:
                out = torch.empty(xi.numel(), dtype=torch.int32, device=xi.device)
            check(lib().rtf_sample_f32(ctypes.byref(self.view), _ptr(xi), xi.numel(), _ptr(out),
                                       _stream(stream)), "rtf_sample_f32")
            return out
        xi = _u32_view(xi)
        if out is None:
            out = torch.empty(xi.numel(), dtype=torch.int32, device=xi.device)
        check(lib().rtf_sample(ctypes.byref(self.view), _ptr(xi), xi.numel(), _ptr(out),
                               _stream(stream)), "rtf_sample")
        return out

    # ------------------------------------------- 4-ary collapsed records
    def build_quad(self, stream=None) -> "Forest":
        """32-B records deciding two levels per load (rtf_build_quad); call after build()."""
        L = lib()
        nb = L.rtf_quad_bytes(self.n)
        if getattr(self, "_rec4", None) is None or self._rec4.numel() < nb:
            self._rec4 = _bytes_tensor(nb, self._buf.forest.device)
        check(L.rtf_build_quad(ctypes.byref(self.view), _ptr(self._rec4), self._rec4.numel(),
                               _stream(stream)), "rtf_build_quad")
        self._rec4_valid = True
        return self

    def sample_quad(self, xi: torch.Tensor, out: torch.Tensor | None = None, stream=None):
        """rtf_sample's indices through the quad records (build_quad() first)."""
        if getattr(self, "_rec4", None) is None or not getattr(self, "_rec4_valid", False):
            raise RuntimeError("sample_quad needs build_quad() after the latest build()")
        if getattr(self, "_marked", False):
            raise RuntimeError("sample_quad does not read tables marked by build_fallback()")
        xi = _u32_view(xi)
        if out is None:
            out = torch.empty(xi.numel(), dtype=torch.int32, device=xi.device)
        check(lib().rtf_sample_quad(ctypes.byref(self.view), _ptr(self._rec4), _ptr(xi),
                                    xi.numel(), _ptr(out), _stream(stream)), "rtf_sample_quad")
        return out

    # ------------------------------------------- degenerate-cell fallback (R21)
    def build_fallback(self, stream=None) -> "Forest":
        """Mark the cells whose radix trees are deeper than bisection + 4 reads
        (rtf_build_fallback); rtf_sample then bisects them.  Call after build()."""
        L = lib()
        nb = L.rtf_fallback_bytes(self.m)
        if getattr(self, "_fb_ws", None) is None or self._fb_ws.numel() < nb:
            self._fb_ws = _bytes_tensor(nb, self._buf.forest.device)
        check(L.rtf_build_fallback(ctypes.byref(self.view), _ptr(self._fb_ws), self._fb_ws.numel(),
                                   _stream(stream)), "rtf_build_fallback")
        self._marked = True
        return self

    def cell_depths(self):
        """After build_fallback(): per cell the radix depth (node reads of the
        deepest xi, anchor cells; else 0) and the cell's last leaf, as int64 numpy."""
        if getattr(self, "_fb_ws", None) is None:
            raise RuntimeError("cell_depths needs build_fallback()")
        torch.cuda.synchronize(self._buf.forest.device)
        w = self._fb_ws[: 8 * self.m].view(torch.int32).cpu().numpy().astype(np.int64)
        return w[: self.m], w[self.m: 2 * self.m]

    def sample_loads(self, xi: torch.Tensor, stream=None, plain: bool = False):
        """Per-sample memory loads of Alg. 2 (1 table cell + nodes visited);
        with plain=True also the count without the two-interval flag."""
        xi = _u32_view(xi)
        out = torch.empty(xi.numel(), dtype=torch.int32, device=xi.device)
        op = torch.empty_like(out) if plain else None
        check(lib().rtf_sample_loads(ctypes.byref(self.view), _ptr(xi), xi.numel(), _ptr(out),
                                     _ptr(op) if plain else None, _stream(stream)),
              "rtf_sample_loads")
        return (out, op) if plain else out

    # ---------------------------------------------------------------- inspection
    def header(self, stream=None) -> rtf_header:
        h = rtf_header()
        self.last_status = lib().rtf_forest_status(ctypes.byref(self.view), _stream(stream),
                                                   ctypes.byref(h))
        return h

    def status(self, stream=None) -> int:
        self.header(stream)
        return self.last_status

    def n_pos(self) -> int:
        return int(self.header().n_pos)

    def _section(self, ptr, nbytes) -> torch.Tensor:
        base = self._buf.forest.data_ptr()
        off = ptr - base
        return self._buf.forest[off: off + nbytes]

    def nodes_numpy(self) -> np.ndarray:
        k = self.n_pos()
        raw = self._section(self.view.nodes, 16 * k).cpu().numpy()
        return raw.view(NODE_DTYPE)

    def table_numpy(self) -> np.ndarray:
        """The guide table as (key32, ref) cells (rtf_ref)."""
        return self._section(self.view.table, 8 * self.m).cpu().numpy().view(CELL_DTYPE)


class RowsForest:
    """`rows` independent forests of n_row entries / m_row cells (config 5)."""

    def __init__(self, rows: int, n_row: int, m_row: int, device="cuda"):
        L = lib()
        self.rows, self.n, self.m = int(rows), int(n_row), int(m_row)
        fb = L.rtf_forest_bytes(self.n, self.m, self.rows)
        self._forest = _bytes_tensor(fb, torch.device(device))
        self.view = rtf_forest()
        check(L.rtf_forest_view(_ptr(self._forest), fb, self.n, self.m, self.rows,
                                ctypes.byref(self.view)), "rtf_forest_view")

    def build(self, p: torch.Tensor, stream=None) -> "RowsForest":
        if p.dtype != torch.float32 or not p.is_cuda or not p.is_contiguous():
            raise TypeError("p must be a contiguous float32 CUDA tensor")
        if p.numel() != self.rows * self.n:
            raise ValueError("p must hold rows * n_row weights")
        self._p = p
        check(lib().rtf_build_rows(_ptr(p), self.rows, self.n, self.m, _ptr(self._forest),
                                   self._forest.numel(), _stream(stream),
                                   ctypes.byref(self.view)), "rtf_build_rows")
        return self

    def sample(self, row: torch.Tensor, xi: torch.Tensor, out=None, stream=None):
        xi = _u32_view(xi)
        row = _u32_view(row)
        if out is None:
            out = torch.empty(xi.numel(), dtype=torch.int32, device=xi.device)
        check(lib().rtf_sample_rows(ctypes.byref(self.view), _ptr(row), _ptr(xi), xi.numel(),
                                    _ptr(out), _stream(stream)), "rtf_sample_rows")
        return out

    def headers(self, stream=None) -> np.ndarray:
        arr = (rtf_header * self.rows)()
        self.last_status = lib().rtf_forest_status(ctypes.byref(self.view), _stream(stream),
                                                   ctypes.cast(arr, ctypes.POINTER(rtf_header)))
        return np.ctypeslib.as_array(arr)

    def _section(self, ptr, nbytes):
        off = ptr - self._forest.data_ptr()
        return self._forest[off: off + nbytes]

    def nodes_numpy(self) -> np.ndarray:
        return self._section(self.view.nodes, 16 * self.rows * self.n).cpu().numpy().view(NODE_DTYPE)

    def table_numpy(self) -> np.ndarray:
        return self._section(self.view.table, 8 * self.rows * self.m).cpu().numpy().view(CELL_DTYPE)


class Forest2D:
    """A 2-D distribution (Sec.6): marginal forest over the rows + one forest per
    row (rtf_build_2d / rtf_sample_2d)."""

    def __init__(self, W: int, H: int, mx: int, my: int, device="cuda"):
        L = lib()
        self.W, self.H, self.mx, self.my = int(W), int(H), int(mx), int(my)
        self._buf = _bytes_tensor(L.rtf_forest2d_bytes(self.W, self.H, self.mx, self.my),
                                  torch.device(device))
        self.view = rtf_forest2d()

    def build(self, p: torch.Tensor, stream=None) -> "Forest2D":
        if p.dtype != torch.float32 or not p.is_cuda or not p.is_contiguous():
            raise TypeError("p must be a contiguous float32 CUDA tensor")
        if p.numel() != self.W * self.H:
            raise ValueError("p must hold H x W weights")
        self._p = p
        check(lib().rtf_build_2d(_ptr(p), self.W, self.H, self.mx, self.my, _ptr(self._buf),
                                 self._buf.numel(), _stream(stream), ctypes.byref(self.view)),
              "rtf_build_2d")
        return self

    def status(self, stream=None) -> int:
        return lib().rtf_forest2d_status(ctypes.byref(self.view), _stream(stream))

    def sample(self, xi1: torch.Tensor, xi2: torch.Tensor, pixel=None, pos=None,
               with_pos: bool = True, stream=None):
        """Returns pixel (int32, y W + x) and, with_pos, pos (float32 [N, 2], (x, y) in [0,1))."""
        xi1, xi2 = _u32_view(xi1), _u32_view(xi2)
        if xi1.numel() != xi2.numel():
            raise ValueError("xi1 and xi2 must have the same length")
        n = xi1.numel()
        if pixel is None:
            pixel = torch.empty(n, dtype=torch.int32, device=xi1.device)
        if with_pos and pos is None:
            pos = torch.empty((n, 2), dtype=torch.float32, device=xi1.device)
        check(lib().rtf_sample_2d(ctypes.byref(self.view), _ptr(xi1), _ptr(xi2), n, _ptr(pixel),
                                  _ptr(pos) if with_pos else None, _stream(stream)),
              "rtf_sample_2d")
        return (pixel, pos) if with_pos else pixel

    def weights(self) -> np.ndarray:
        off = self.view.weights - self._buf.data_ptr()
        return self._buf[off: off + 4 * self.H].cpu().numpy().view(np.float32)

    def dense_rows(self) -> np.ndarray:
        """bool[H]: row y has no zero weight (rows_dense bit y)."""
        off = self.view.rows_dense - self._buf.data_ptr()
        words = self._buf[off: off + 4 * ((self.H + 31) // 32)].cpu().numpy().view(np.uint32)
        return ((words[np.arange(self.H) // 32] >> (np.arange(self.H) % 32)) & 1).astype(bool)


def build_2d(p: torch.Tensor, mx: int, my: int, stream=None) -> Forest2D:
    H, W = p.shape
    return Forest2D(W, H, mx, my, device=p.device).build(p.contiguous().view(-1), stream)


# -------------------------------------------------------------------- functional API

def build(p: torch.Tensor, m: int, flags: int = RTF_BUILD_DEFAULT, stream=None) -> Forest:
    return Forest(p.numel(), m, flags, device=p.device).build(p, stream)


def sample(forest: Forest, xi: torch.Tensor, out=None, stream=None) -> torch.Tensor:
    return forest.sample(xi, out, stream)


def build_rows(p: torch.Tensor, m_row: int, stream=None) -> RowsForest:
    rows, n_row = p.shape
    return RowsForest(rows, n_row, m_row, device=p.device).build(p.contiguous().view(-1), stream)


def sample_rows(forest: RowsForest, row, xi, out=None, stream=None):
    return forest.sample(row, xi, out, stream)


class Cdf:
    """The full fixed-point CDF (zeros included) for the binary-search baseline."""

    def __init__(self, n: int, device="cuda"):
        self.n = int(n)
        self.cdf = torch.empty(self.n, dtype=torch.int64, device=device)
        self.header = torch.zeros(48, dtype=torch.uint8, device=device)
        wb = lib().rtf_workspace_bytes(self.n, 1, 0)
        self.ws = _bytes_tensor(wb, torch.device(device))
        check(lib().rtf_workspace_init(_ptr(self.ws), self.ws.numel(), self.n, 1, 0, _stream()),
              "rtf_workspace_init")

    def build(self, p: torch.Tensor, stream=None) -> "Cdf":
        self._p = p
        check(lib().rtf_build_cdf(_ptr(p), self.n, _ptr(self.cdf), _ptr(self.header),
                                  _ptr(self.ws), self.ws.numel(), _stream(stream)),
              "rtf_build_cdf")
        return self

    def sample(self, xi: torch.Tensor, out=None, stream=None) -> torch.Tensor:
        xi = _u32_view(xi)
        if out is None:
            out = torch.empty(xi.numel(), dtype=torch.int32, device=xi.device)
        check(lib().rtf_sample_bsearch(_ptr(self.cdf), self.n, _ptr(self.header), _ptr(xi),
                                       xi.numel(), _ptr(out), _stream(stream)),
              "rtf_sample_bsearch")
        return out


    def eytzinger(self, stream=None) -> "Eytzinger":
        """The same CDF as a breadth-first search tree (the Eytzinger baseline)."""
        return Eytzinger(self, stream)

    def cutpoint(self, m: int, stream=None) -> "Cutpoint":
        """The cutpoint table (m cells) over this CDF, for the cutpoint baselines."""
        return Cutpoint(self, m, stream)


class Eytzinger:
    """Binary search over a Cdf in breadth-first (Eytzinger) order, top levels
    in shared memory: the competent GPU binary-search baseline."""

    def __init__(self, cdf: Cdf, stream=None):
        self.cdf = cdf
        slots = int(lib().rtf_eytzinger_slots(cdf.n))
        self.eyt = torch.empty(slots, dtype=torch.int64, device=cdf.cdf.device)
        check(lib().rtf_build_eytzinger(_ptr(cdf.cdf), cdf.n, _ptr(self.eyt), _stream(stream)),
              "rtf_build_eytzinger")

    def sample(self, xi: torch.Tensor, out=None, stream=None) -> torch.Tensor:
        xi = _u32_view(xi)
        if out is None:
            out = torch.empty(xi.numel(), dtype=torch.int32, device=xi.device)
        check(lib().rtf_sample_eytzinger(_ptr(self.eyt), self.cdf.n, _ptr(self.cdf.header),
                                         _ptr(xi), xi.numel(), _ptr(out), _stream(stream)),
              "rtf_sample_eytzinger")
        return out


class Alias:
    """The alias-method baseline (rtf_sample_alias) over a host-built table
    {prob, alias} of 2^k buckets (baselines.alias_table): argument marshalling."""

    def __init__(self, prob: np.ndarray, alias: np.ndarray, k: int, device="cuda"):
        tab = np.empty((prob.size, 2), np.uint32)
        tab[:, 0], tab[:, 1] = prob, alias.view(np.uint32)
        self.k = int(k)
        self.table = torch.from_numpy(tab.view(np.int32)).to(device)

    def sample(self, xi: torch.Tensor, out=None, stream=None) -> torch.Tensor:
        xi = _u32_view(xi)
        if out is None:
            out = torch.empty(xi.numel(), dtype=torch.int32, device=xi.device)
        check(lib().rtf_sample_alias(_ptr(self.table), self.k, _ptr(xi), xi.numel(), _ptr(out),
                                     _stream(stream)), "rtf_sample_alias")
        return out


class Alias2D:
    """The 2-D alias baseline (rtf_sample_alias_2d) over host-built tables
    (baselines.alias_2d): marginal {prob, alias} of 2^ky buckets, H row
    tables of 2^kx buckets each.  Argument marshalling."""

    def __init__(self, marg, rows, W: int, H: int, device="cuda"):
        (mp, ma, ky), (rp, ra, kx) = marg, rows
        def pack(prob, alias):
            t = np.empty(prob.shape + (2,), np.uint32)
            t[..., 0], t[..., 1] = prob, alias.view(np.uint32)
            return torch.from_numpy(t.view(np.int32)).to(device)
        self.W, self.H, self.ky, self.kx = int(W), int(H), int(ky), int(kx)
        self.marg, self.rows = pack(mp, ma), pack(rp, ra)

    def sample(self, xi1: torch.Tensor, xi2: torch.Tensor, pixel=None, stream=None):
        xi1, xi2 = _u32_view(xi1), _u32_view(xi2)
        if xi1.numel() != xi2.numel():
            raise ValueError("xi1 and xi2 must have the same length")
        if pixel is None:
            pixel = torch.empty(xi1.numel(), dtype=torch.int32, device=xi1.device)
        check(lib().rtf_sample_alias_2d(_ptr(self.marg), self.ky, _ptr(self.rows), self.kx,
                                        self.W, self.H, _ptr(xi1), _ptr(xi2), xi1.numel(),
                                        _ptr(pixel), _stream(stream)), "rtf_sample_alias_2d")
        return pixel


class Cutpoint:
    """Classic cutpoint guide table over a Cdf (baselines of Sec.2.3 / Table 1)."""

    def __init__(self, cdf: Cdf, m: int, stream=None):
        self.cdf, self.m = cdf, int(m)
        self.cut = torch.empty(self.m + 1, dtype=torch.int32, device=cdf.cdf.device)
        check(lib().rtf_build_cutpoint(_ptr(cdf.cdf), cdf.n, self.m, _ptr(self.cut),
                                       _stream(stream)), "rtf_build_cutpoint")

    def sample(self, xi: torch.Tensor, out=None, binary: bool = True, stream=None):
        xi = _u32_view(xi)
        if out is None:
            out = torch.empty(xi.numel(), dtype=torch.int32, device=xi.device)
        check(lib().rtf_sample_cutpoint(_ptr(self.cdf.cdf), self.cdf.n, _ptr(self.cdf.header),
                                        _ptr(self.cut), self.m, int(binary), _ptr(xi),
                                        xi.numel(), _ptr(out), _stream(stream)),
              "rtf_sample_cutpoint")
        return out


def build_cdf(p: torch.Tensor, stream=None) -> Cdf:
    return Cdf(p.numel(), p.device).build(p, stream)


def sample_bsearch(cdf: Cdf, xi: torch.Tensor, out=None, stream=None) -> torch.Tensor:
    return cdf.sample(xi, out, stream)


def philox(count: int, seed: int = 0x5EED, start: int = 0, out=None, device="cuda",
           stream=None) -> torch.Tensor:
    if out is None:
        out = torch.empty(int(count), dtype=torch.int32, device=device)
    check(lib().rtf_philox_u32(seed, start, int(count), _ptr(out), _stream(stream)),
          "rtf_philox_u32")
    return out


def build_host(forest: Forest, p_host: torch.Tensor, p_dev: torch.Tensor, stream=None) -> int:
    """End-to-end build from a (pinned) host float32 tensor; synchronous."""
    h = rtf_header()
    st = lib().rtf_build_host(ctypes.c_void_p(p_host.data_ptr()), forest.n, forest.m,
                              forest.flags, _ptr(p_dev), _ptr(forest._buf.forest),
                              forest._buf.forest.numel(), _ptr(forest._buf.ws),
                              forest._buf.ws.numel(), _stream(stream),
                              ctypes.byref(forest.view), ctypes.byref(h))
    if st not in (_lib.RTF_OK, _lib.RTF_EALLZERO, _lib.RTF_EDATA):
        check(st, "rtf_build_host")
    return st


def sample_host(forest: Forest, xi_host: torch.Tensor, out_host: torch.Tensor,
                xi_dev: torch.Tensor, out_dev: torch.Tensor, stream=None) -> None:
    """End-to-end sampling host -> host through pipelined staging buffers
    (xi_dev / out_dev hold 2 chunks each); synchronous."""
    chunk = xi_dev.numel() // 2
    check(lib().rtf_sample_host(ctypes.byref(forest.view), ctypes.c_void_p(xi_host.data_ptr()),
                                xi_host.numel(), ctypes.c_void_p(out_host.data_ptr()),
                                _ptr(xi_dev), _ptr(out_dev), chunk, _stream(stream)),
          "rtf_sample_host")


def launch_count() -> int:
    return int(lib().rtf_launch_count())
