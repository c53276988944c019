"""Sharded build across GPUs (config 4): cross-GPU scan of per-shard totals plus
a per-shard build, then replication so every GPU can sample the whole forest.

Only orchestration lives here: every step of the method runs in librtf's
kernels (rtf_shard_* in include/rtf.h); this module moves bytes between shards
with collectives.  Two communicators implement the same four collectives:

  DistComm   one shard per process, torch.distributed (NCCL over NVLink on a
             B200 box; gloo in CPU tests of the orchestration)
  LocalComm  several shards in one process on one GPU (virtual shards), used
             by the single-GPU parity tests

Protocol (include/rtf.h, "sharded build"): scale -> MAX-reduce -> totals ->
gather (the cross-GPU scan) -> per-shard build -> replicate records (broadcast
from the owner), table (MAX-reduce), tile spine rows (gather) -> finish (the
cross-tile links) on every shard.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import check, rtf_forest, rtf_shard_view


def shard_range(n: int, world: int, rank: int, align: int = 4096):
    """Contiguous shard [base, base + n_local) of rank; shard sizes are a
    multiple of `align` entries (tile boundaries, 16-B aligned) except the last."""
    per = -(-n // world)
    per = -(-per // align) * align
    base = min(n, rank * per)
    return base, max(0, min(per, n - base))


# --------------------------------------------------------------------- collectives

class LocalComm:
    """Virtual shards in one process: each collective takes the list of the
    shards' tensors."""

    def allreduce_max(self, ts):
        mx = ts[0].clone()
        for t in ts[1:]:
            torch.maximum(mx, t, out=mx)
        for t in ts:
            t.copy_(mx)

    def allgather(self, ts):
        cat = torch.cat([t.reshape(-1) for t in ts])
        return [cat for _ in ts]

    def broadcast(self, ts, src):
        for i, t in enumerate(ts):
            if i != src:
                t.copy_(ts[src])


class DistComm:
    """One shard per process (torch.distributed); lists hold the local tensor."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def allreduce_max(self, ts):
        self.dist.all_reduce(ts[0], op=self.dist.ReduceOp.MAX, group=self.group)

    def allgather(self, ts):
        t = ts[0].reshape(-1).contiguous()
        world = self.dist.get_world_size(self.group)
        if t.is_cuda:  # NCCL: one fused all-gather
            out = torch.empty(world * t.numel(), dtype=t.dtype, device=t.device)
            self.dist.all_gather_into_tensor(out, t, group=self.group)
            return [out]
        parts = [torch.empty_like(t) for _ in range(world)]  # gloo
        self.dist.all_gather(parts, t, group=self.group)
        return [torch.cat(parts)]

    def broadcast(self, ts, src):
        self.dist.broadcast(ts[0], src=src, group=self.group)


# --------------------------------------------------------------------- shard state

def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


@dataclass
class Shard:
    rank: int
    count: int
    n_global: int
    m: int
    base: int
    n_local: int
    p: torch.Tensor                      # this shard's weights (device, float32)
    forest: torch.Tensor = field(init=False)
    ws: torch.Tensor = field(init=False)
    view: rtf_shard_view = field(init=False)
    fview: rtf_forest = field(init=False)

    def __post_init__(self):
        L = _lib.load()
        dev = self.p.device
        fb = L.rtf_forest_bytes(self.n_global, self.m, 1)
        wb = L.rtf_shard_workspace_bytes(self.n_local, self.n_global, self.m)
        self.forest = torch.empty(fb, dtype=torch.uint8, device=dev)
        self.ws = torch.empty(wb, dtype=torch.uint8, device=dev)
        self.view = rtf_shard_view()
        self.fview = rtf_forest()
        args = (self.n_local, self.n_global, self.m)
        check(L.rtf_shard_workspace_init(_ptr(self.ws), wb, *args, _stream()), "shard ws init")
        check(L.rtf_shard_get_view(_ptr(self.ws), wb, *args, ctypes.byref(self.view)), "view")
        check(L.rtf_forest_view(_ptr(self.forest), fb, self.n_global, self.m, 1,
                                ctypes.byref(self.fview)), "forest view")

    # device tensors aliasing the workspace / forest (for the collectives)
    def _ws_slice(self, ptr, nbytes):
        off = ptr - self.ws.data_ptr()
        return self.ws[off: off + nbytes]

    def _forest_slice(self, ptr, nbytes):
        off = ptr - self.forest.data_ptr()
        return self.forest[off: off + nbytes]

    def scale_words(self):
        return self._ws_slice(self.view.scale, 16).view(torch.int32)

    def total_bytes(self):
        return self._ws_slice(self.view.total, 16)

    def node_bytes(self, j0, cnt):
        return self._forest_slice(self.fview.nodes + 16 * j0, 16 * cnt)

    def table_words(self):
        # 8-B cells {u32 key32, i32 ref} as little-endian int64: ref is the high
        # half, so a MAX-reduction keeps the owner's cell over {0, INT32_MIN}
        return self._forest_slice(self.fview.table, 8 * self.m).view(torch.int64)

    def spine_bytes(self):
        return self._ws_slice(self.view.spine, self.view.spine_row_bytes * self.view.nt_local)


def _padded(t: torch.Tensor, nbytes: int, fill: int) -> torch.Tensor:
    out = torch.full((nbytes,), fill, dtype=torch.uint8, device=t.device)
    out[: t.numel()] = t
    return out


def build_sharded(shards: list[Shard], comm) -> None:
    """Run the sharded build for the local shards (all of them for LocalComm,
    the process's own for DistComm).  On return every shard's forest buffer
    holds the full forest."""
    L = _lib.load()
    st = _stream()
    sh0 = shards[0]
    args = lambda s: (s.n_local, s.n_global, s.m)  # noqa: E731
    # 1. per-shard scale, MAX across shards
    for s in shards:
        check(L.rtf_shard_scale(_ptr(s.p), *args(s), _ptr(s.ws), s.ws.numel(), st), "shard scale")
    comm.allreduce_max([s.scale_words() for s in shards])
    # 2. per-shard totals; gather = the cross-GPU scan input
    for s in shards:
        check(L.rtf_shard_totals(_ptr(s.p), *args(s), s.base, _ptr(s.ws), s.ws.numel(), st),
              "shard totals")
    totals = comm.allgather([s.total_bytes() for s in shards])
    # 3. per-shard build with the global prefix
    for s, tot in zip(shards, totals):
        check(L.rtf_shard_build(_ptr(s.p), *args(s), s.base, s.rank, s.count, _ptr(tot),
                                _ptr(s.forest), s.forest.numel(), _ptr(s.ws), s.ws.numel(), st,
                                ctypes.byref(s.fview)), "shard build")
    # 4. replication: owner ranges from the gathered totals (16 B per shard)
    tot = totals[0].cpu().numpy().view(np.dtype([("W", "<u8"), ("cnt", "<u4"), ("last", "<i4")]))
    starts = np.concatenate([[0], np.cumsum(tot["cnt"].astype(np.int64))])
    for r in range(sh0.count):
        j0, cnt = int(starts[r]), int(tot["cnt"][r])
        if cnt:
            comm.broadcast([s.node_bytes(j0, cnt) for s in shards], src=r)
    comm.allreduce_max([s.table_words() for s in shards])
    nt_max = max(s.view.nt_local for s in shards)
    if hasattr(comm, "dist"):  # shards of other processes may have more tiles
        t = torch.tensor([nt_max], dtype=torch.int64, device=sh0.p.device)
        comm.allreduce_max([t])
        nt_max = int(t.item())
    row = sh0.view.spine_row_bytes
    spine_all = comm.allgather([_padded(s.spine_bytes(), row * nt_max, 0) for s in shards])
    # 5. cross-tile links over all shards' spine rows, on every shard
    for s, sa in zip(shards, spine_all):
        check(L.rtf_shard_finish(*args(s), _ptr(sa), s.count * nt_max, _ptr(s.forest),
                                 s.forest.numel(), _ptr(s.ws), s.ws.numel(), st,
                                 ctypes.byref(s.fview)), "shard finish")


def make_shards_local(p_local: torch.Tensor, n: int, m: int, rank: int, count: int,
                      base: int) -> list[Shard]:
    """The one shard this process holds (multi-GPU: one shard per rank)."""
    return [Shard(rank, count, n, m, base, p_local.numel(), p_local)]


def make_shards(p: torch.Tensor, m: int, count: int, ranks=None) -> list[Shard]:
    """Shards of a (device) weight vector; `ranks` selects which to create
    locally (default: all, for virtual shards)."""
    n = p.numel()
    out = []
    for r in (range(count) if ranks is None else ranks):
        base, nl = shard_range(n, count, r)
        if nl == 0:
            raise ValueError("more shards than 4096-entry blocks")
        out.append(Shard(r, count, n, m, base, nl, p[base: base + nl]))
    return out
