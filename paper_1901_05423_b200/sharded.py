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

    def allreduce_sum(self, ts):
        tot = ts[0].clone()
        for t in ts[1:]:
            tot += t
        for t in ts:
            t.copy_(tot)

    def alltoallv(self, sends, recvs):
        """sends[q][r]: shard q's piece for shard r; recvs[r][q]: where shard r
        receives shard q's piece (None on the diagonal: already in place)."""
        for r in range(len(sends)):
            for q in range(len(sends)):
                if q != r and sends[q][r] is not None and sends[q][r].numel():
                    recvs[r][q].copy_(sends[q][r])

    def reduce_scatter_max(self, full, lo, hi):
        """full[r]: shard r's whole array; on return full[r][lo[r]:hi[r]] holds
        the element-wise maximum over all shards of that slice."""
        for r in range(len(full)):
            mx = full[0][lo[r]: hi[r]].clone()
            for t in full[1:]:
                torch.maximum(mx, t[lo[r]: hi[r]], out=mx)
            full[r][lo[r]: hi[r]].copy_(mx)


def _local_peers(shards):
    return [s.forest.data_ptr() for s in shards]


class DistComm:
    """One shard per process (torch.distributed); lists hold the local tensor.

    NCCL (one process per GPU): device tensors go straight into the
    collectives, and the fused build's peer pointers come from CUDA symmetric
    memory (NVLink).  gloo (CPU tests, or several processes sharing one GPU in
    the single-GPU multi-process tests): device tensors are staged through host
    memory, and peer pointers are CUDA IPC mappings of the other processes'
    forest buffers (valid when the processes share the device)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.host = dist.get_backend(group) == "gloo"
        self._ipc_keep = []  # opened IPC storages stay mapped while the comm lives

    def _run(self, t, fn):
        """fn(tensor) on t, or on a host copy of it (gloo), written back."""
        if self.host and t.is_cuda:
            h = t.cpu()
            fn(h)
            t.copy_(h)
        else:
            fn(t)

    def allreduce_max(self, ts):
        self._run(ts[0], lambda t: self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX,
                                                        group=self.group))

    def allgather(self, ts):
        t = ts[0].reshape(-1).contiguous()
        world = self.dist.get_world_size(self.group)
        if t.is_cuda and not self.host:  # NCCL: one fused all-gather
            out = torch.empty(world * t.numel(), dtype=t.dtype, device=t.device)
            self.dist.all_gather_into_tensor(out, t, group=self.group)
            return [out]
        src = t.cpu() if t.is_cuda else t
        parts = [torch.empty_like(src) for _ in range(world)]  # gloo
        self.dist.all_gather(parts, src, group=self.group)
        return [torch.cat(parts).to(t.device)]

    def broadcast(self, ts, src):
        self._run(ts[0], lambda t: self.dist.broadcast(t, src=src, group=self.group))

    def allreduce_sum(self, ts):
        self._run(ts[0], lambda t: self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM,
                                                        group=self.group))

    # fused ranged sharding: forest buffers in CUDA symmetric memory, so every
    # rank's kernels can store into every peer's buffer over NVLink
    def alloc(self, nbytes, device):
        if self.host:
            return torch.empty(nbytes, dtype=torch.uint8, device=device)
        import torch.distributed._symmetric_memory as symm_mem
        return symm_mem.empty(nbytes, dtype=torch.uint8, device=device)

    def peer_ptrs(self, buf):
        if self.host:  # processes sharing one device: CUDA IPC handles
            st = buf.untyped_storage()
            handle = st._share_cuda_()
            off = buf.data_ptr() - st.data_ptr()
            world = self.dist.get_world_size(self.group)
            allh = [None] * world
            self.dist.all_gather_object(allh, (handle, off), group=self.group)
            me = self.dist.get_rank(self.group)
            ptrs = []
            for r, (h, o) in enumerate(allh):
                if r == me:
                    ptrs.append(buf.data_ptr())
                    continue
                peer = torch.UntypedStorage._new_shared_cuda(*h)
                self._ipc_keep.append(peer)
                ptrs.append(peer.data_ptr() + o)
            return ptrs
        import torch.distributed._symmetric_memory as symm_mem
        group = self.group if self.group is not None else self.dist.group.WORLD
        hdl = symm_mem.rendezvous(buf, group)
        return [int(x) for x in hdl.buffer_ptrs]

    def alltoallv(self, sends, recvs):
        """Grouped point-to-point transfers of the local pieces (sends[0][r] to
        rank r, recvs[0][q] from rank q) straight between their final places
        (gloo: through host copies)."""
        me = self.dist.get_rank(self.group)
        if self.host:
            hs = [None if t is None else t.cpu() for t in sends[0]]
            hr = [None if t is None else torch.empty(t.shape, dtype=t.dtype) for t in recvs[0]]
            ops = []
            for r, t in enumerate(hs):
                if r != me and t is not None and t.numel():
                    ops.append(self.dist.P2POp(self.dist.isend, t, r, group=self.group))
            for q, t in enumerate(hr):
                if q != me and t is not None and t.numel():
                    ops.append(self.dist.P2POp(self.dist.irecv, t, q, group=self.group))
            if ops:
                for w in self.dist.batch_isend_irecv(ops):
                    w.wait()
            for q, t in enumerate(hr):
                if q != me and t is not None and t.numel():
                    recvs[0][q].copy_(t)
            return
        ops = []
        for r, t in enumerate(sends[0]):
            if r != me and t is not None and t.numel():
                ops.append(self.dist.P2POp(self.dist.isend, t, r, group=self.group))
        for q, t in enumerate(recvs[0]):
            if q != me and t is not None and t.numel():
                ops.append(self.dist.P2POp(self.dist.irecv, t, q, group=self.group))
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()

    def reduce_scatter_max(self, full, lo, hi):
        me = self.dist.get_rank(self.group)
        t = full[0]
        equal = len(set(int(h) - int(l) for l, h in zip(lo, hi))) == 1 and int(lo[0]) == 0
        if self.host:  # gloo (no reduce-scatter): the all-reduce covers the slice
            self.allreduce_max([t])
            return
        if t.is_cuda and equal and int(hi[-1]) == t.numel():  # NCCL: one reduce-scatter
            out = torch.empty(int(hi[me]) - int(lo[me]), dtype=t.dtype, device=t.device)
            self.dist.reduce_scatter_tensor(out, t, op=self.dist.ReduceOp.MAX, group=self.group)
            t[int(lo[me]): int(hi[me])].copy_(out)
        else:  # gloo (no reduce-scatter): the all-reduce covers the slice
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)


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

    alloc: object = None                 # forest allocator (symmetric memory when fused)

    def __post_init__(self):
        L = _lib.load()
        dev = self.p.device
        fb = L.rtf_forest_bytes(self.n_global, self.m, 1)
        wb = L.rtf_shard_workspace_bytes(self.n_local, self.n_global, self.m)
        self.forest = (self.alloc(fb, dev) if self.alloc is not None
                       else torch.empty(fb, dtype=torch.uint8, device=dev))
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

    def node_words(self, j0, cnt):
        """Records [j0, j0 + cnt) as int64 pairs (2 words per 16-B record)."""
        return self._forest_slice(self.fview.nodes + 16 * j0, 16 * cnt).view(torch.int64)

    def spine_bytes(self):
        return self._ws_slice(self.view.spine, self.view.spine_row_bytes * self.view.nt_local)


def _padded(t: torch.Tensor, nbytes: int, fill: int) -> torch.Tensor:
    out = torch.full((nbytes,), fill, dtype=torch.uint8, device=t.device)
    out[: t.numel()] = t
    return out


def build_sharded(shards: list[Shard], comm, ranged: bool = False, fused: bool = False) -> None:
    """Run the sharded build for the local shards (all of them for LocalComm,
    the process's own for DistComm).  On return every shard's forest buffer
    holds the full forest -- or, with ranged=True, shard r holds the cells
    [g_r, g_{r+1}) = [r m / N, (r + 1) m / N) (node slots [J_r, J_{r+1}),
    stored in s.cells / s.slots), the xi range it samples.  fused=True (ranged
    only): the per-shard build stores records and table cells straight into
    their owners' buffers (rtf_shard_build_peers: peer memory), so no
    all-to-all and no reduce-scatter remain -- only the gather of the spine
    rows and a MAX-reduce of N + 1 boundary words."""
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
    if fused and sh0.count > 1:
        _build_fused(shards, comm, totals, st)
        return
    # 3. per-shard build with the global prefix
    for s, tot in zip(shards, totals):
        check(L.rtf_shard_build(_ptr(s.p), *args(s), s.base, s.rank, s.count, _ptr(tot),
                                _ptr(s.forest), s.forest.numel(), _ptr(s.ws), s.ws.numel(), st,
                                ctypes.byref(s.fview)), "shard build")
    # 4. replication: owner ranges from the gathered totals (16 B per shard)
    tot = totals[0].cpu().numpy().view(np.dtype([("W", "<u8"), ("cnt", "<u4"), ("last", "<i4")]))
    starts = np.concatenate([[0], np.cumsum(tot["cnt"].astype(np.int64))])
    if ranged and sh0.count > 1:
        _redistribute_and_finish(shards, comm, starts, tot["cnt"].astype(np.int64), st)
        return
    if ranged:  # one shard: its cell range is everything
        shards[0].cells, shards[0].slots = (0, sh0.m), (0, int(starts[-1]))
    for r in range(sh0.count):
        j0, cnt = int(starts[r]), int(tot["cnt"][r])
        if cnt:
            comm.broadcast([s.node_bytes(j0, cnt) for s in shards], src=r)
    comm.allreduce_max([s.table_words() for s in shards])
    nt_max = _nt_max(shards, comm)
    row = sh0.view.spine_row_bytes
    spine_all = comm.allgather([_padded(s.spine_bytes(), row * nt_max, 0) for s in shards])
    # 5. cross-tile links over all shards' spine rows, on every shard
    for s, sa in zip(shards, spine_all):
        check(L.rtf_shard_finish(*args(s), _ptr(sa), s.count * nt_max, _ptr(s.forest),
                                 s.forest.numel(), _ptr(s.ws), s.ws.numel(), st,
                                 ctypes.byref(s.fview)), "shard finish")


def make_shards_local(p_local: torch.Tensor, n: int, m: int, rank: int, count: int,
                      base: int, alloc=None) -> list[Shard]:
    """The one shard this process holds (multi-GPU: one shard per rank);
    alloc=DistComm().alloc puts its forest in symmetric memory (fused mode)."""
    return [Shard(rank, count, n, m, base, p_local.numel(), p_local, alloc)]


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


def _redistribute_and_finish(shards, comm, starts, counts, st) -> None:
    """Ranged sharding (include/rtf.h): records to the rank of their cells (an
    all-to-all of contiguous slices), the table reduce-scattered by cell slice,
    the spine rows gathered, then the cross-tile links of the own slots."""
    L = _lib.load()
    sh0 = shards[0]
    N, m, dev = sh0.count, sh0.m, sh0.p.device
    g = np.array([k * m // N for k in range(N + 1)], np.int64)
    bounds = torch.from_numpy(g.astype(np.uint32).view(np.int32)).to(dev)
    # J_k: global index of the first leaf with cell >= g_k (sum of the shards' counts)
    cts = []
    for s in shards:
        c = torch.empty(N + 1, dtype=torch.int32, device=dev)
        check(L.rtf_shard_count_cells(_ptr(s.forest), s.forest.numel(), s.n_global, m,
                                      int(starts[s.rank]), int(counts[s.rank]), _ptr(bounds),
                                      N + 1, _ptr(c), _stream()), "count cells")
        cts.append(c.to(torch.int64))
    comm.allreduce_sum(cts)
    J = cts[0].cpu().numpy().astype(np.int64)
    own = [(int(starts[q]), int(starts[q] + counts[q])) for q in range(N)]
    need = [(int(J[r]), int(J[r + 1])) for r in range(N)]

    def piece(s, a, b):  # records [max(a0, b0), min(a1, b1)) of shard s's buffer
        lo, hi = max(a[0], b[0]), min(a[1], b[1])
        return s.node_words(lo, hi - lo) if hi > lo else None

    # a record stays at its global slot: the piece a rank already holds (its
    # own cells among its own entries) does not move
    sends = [[piece(s, own[s.rank], need[r]) for r in range(N)] for s in shards]
    recvs = [[piece(s, own[q], need[s.rank]) for q in range(N)] for s in shards]
    comm.alltoallv(sends, recvs)
    # table: each rank's cell slice, MAX over the shards' partial tables
    comm.reduce_scatter_max([s.table_words() for s in shards], g[:-1], g[1:])
    nt_max = _nt_max(shards, comm)
    row = sh0.view.spine_row_bytes
    spine_all = comm.allgather([_padded(s.spine_bytes(), row * nt_max, 0) for s in shards])
    args = lambda s: (s.n_local, s.n_global, s.m)  # noqa: E731
    for s, sa in zip(shards, spine_all):
        lo, hi = need[s.rank]
        check(L.rtf_shard_finish_range(*args(s), _ptr(sa), s.count * nt_max, lo, hi,
                                       _ptr(s.forest), s.forest.numel(), _ptr(s.ws),
                                       s.ws.numel(), st, ctypes.byref(s.fview)),
              "shard finish (ranged)")
        s.cells = (int(g[s.rank]), int(g[s.rank + 1]))
        s.slots = (lo, hi)


def ranged_xi(xi: torch.Tensor, rank: int, count: int, m: int) -> torch.Tensor:
    """Map u32 xi (as int32) into rank's xi range [g_r 2^32 / m, g_{r+1} 2^32 / m)
    for a power-of-two count: xi' = g_r 2^32 / m + (xi >> log2 count) -- a
    stratified split of the unit interval (input generation, not the method)."""
    if count & (count - 1):
        raise ValueError("ranged sampling needs a power-of-two shard count")
    if m % count:
        # the strata [g_r 2^32 / m, g_{r+1} 2^32 / m) are 2^32 / count wide only
        # when count divides m; otherwise xi would land in another rank's cells
        raise ValueError("ranged sampling needs m divisible by the shard count")
    lo = (rank * m // count) * (1 << 32) // m
    v = (xi.to(torch.int64) & 0xFFFFFFFF) >> (count.bit_length() - 1)
    return ((v + lo) & 0xFFFFFFFF).to(torch.int32)


def _nt_max(shards, comm) -> int:
    """The most tile rows any shard has (the spine gather pads to it); fixed by
    the shard sizes, so computed once and cached on the shards."""
    sh0 = shards[0]
    if getattr(sh0, "_nt_max", None) is None:
        nt_max = max(s.view.nt_local for s in shards)
        if hasattr(comm, "dist"):  # shards of other processes may have more tiles
            t = torch.tensor([nt_max], dtype=torch.int64, device=sh0.p.device)
            comm.allreduce_max([t])
            nt_max = int(t.item())
        for s in shards:
            s._nt_max = nt_max
    return sh0._nt_max


def _build_fused(shards, comm, totals, st) -> None:
    """Fused ranged build: step 3 writes each record / table cell into the
    buffer of the rank owning its cell; then the boundaries J and the spine
    rows are exchanged and each rank finishes its own cells.  The peer
    pointers are uploaded once (rtf_shard_set_peers) and J stays on the device
    (rtf_shard_finish_own), so repeated builds enqueue work without any host
    round trip (s.slots is read back lazily, after the build)."""
    L = _lib.load()
    sh0 = shards[0]
    N, m = sh0.count, sh0.m
    if m % N:
        raise ValueError("fused ranged sharding needs m divisible by the shard count")
    args = lambda s: (s.n_local, s.n_global, s.m)  # noqa: E731
    for s, tot in zip(shards, totals):
        if not getattr(s, "_peers_set", False):
            peers = _local_peers(shards) if isinstance(comm, LocalComm) else comm.peer_ptrs(s.forest)
            arr = (ctypes.c_void_p * N)(*peers)
            check(L.rtf_shard_set_peers(_ptr(s.ws), s.ws.numel(), *args(s), arr, N,
                                        s.forest.numel(), st), "shard peers")
            s._peers_set = True
        check(L.rtf_shard_build_peers(_ptr(s.p), *args(s), s.base, s.rank, s.count, _ptr(tot),
                                      None, N, _ptr(s.forest), s.forest.numel(), _ptr(s.ws),
                                      s.ws.numel(), st, ctypes.byref(s.fview)),
              "shard build (fused)")
    jb = [s._ws_slice(s.view.jbound, 4 * (N + 1)).view(torch.int32) for s in shards]
    comm.allreduce_max(jb)
    nt_max = _nt_max(shards, comm)
    row = sh0.view.spine_row_bytes
    spine_all = comm.allgather([s.spine_bytes() if s.view.nt_local == nt_max
                                else _padded(s.spine_bytes(), row * nt_max, 0) for s in shards])
    for s, sa in zip(shards, spine_all):
        check(L.rtf_shard_finish_own(*args(s), _ptr(sa), s.count * nt_max, s.rank,
                                     _ptr(s.forest), s.forest.numel(), _ptr(s.ws),
                                     s.ws.numel(), st, ctypes.byref(s.fview)),
              "shard finish (fused)")
        s.cells = (s.rank * m // N, (s.rank + 1) * m // N)
        s._jb = jb[shards.index(s)]
        s.slots = None  # [J_r, J_{r+1}) read back on demand: slots_of(s)


def slots_of(s) -> tuple[int, int]:
    """The node slots [J_r, J_{r+1}) a ranged shard holds (a host read of the
    device boundaries after a fused build)."""
    if s.slots is None:
        J = s._jb.cpu().numpy().astype(np.int64)
        s.slots = (int(J[s.rank]), int(J[s.rank + 1]))
    return s.slots
