"""Multi-process (world_size 2, gloo, CPU) checks of the N>1 host paths:

* DistComm (one shard per process, torch.distributed) implements exactly the
  collectives LocalComm (virtual shards, used by the single-GPU parity tests)
  implements, on the tensor shapes and dtypes the sharded build exchanges;
* shard ranges tile [0, n) and are 4096-entry aligned;
* bench.py's max-over-ranks timing reduction.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1901_05423_b200.sharded import DistComm, LocalComm, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs(rank):
    g = torch.Generator().manual_seed(100 + rank)
    return {
        "scale": torch.randint(0, 2**31 - 1, (4,), generator=g, dtype=torch.int32),
        "total": torch.randint(0, 255, (16,), generator=g, dtype=torch.uint8),
        "table": torch.randint(-2**63, 2**63 - 1, (1000,), generator=g, dtype=torch.int64),
        "pend": torch.randint(0, 255, (64,), generator=g, dtype=torch.uint8),
        "records": torch.randint(0, 255, (16 * 37,), generator=g, dtype=torch.uint8),
        "nt": torch.tensor([3 + rank], dtype=torch.int64),
        "counts": torch.randint(0, 1000, (3,), generator=g, dtype=torch.int64),
        "table2": torch.randint(-2**63, 2**63 - 1, (10,), generator=g, dtype=torch.int64),
        # ranged sharding: shard q owns records [OWN[q]), rank r needs [NEED[r])
        "own": torch.randint(-2**62, 2**62, (2 * (OWN[rank][1] - OWN[rank][0]),),
                             generator=g, dtype=torch.int64),
    }


OWN = [(0, 7), (7, 12)]    # record ranges built by shards 0, 1
NEED = [(0, 4), (4, 12)]   # record ranges of the cell slices of ranks 0, 1
SLICE_LO, SLICE_HI = [0, 5], [5, 10]


def _pieces(glob, me):
    """Views of a rank's record buffer (global slots): what it sends to r, where
    it receives from q (the same global slots on both sides)."""
    def view(a, b):
        lo, hi = max(a[0], b[0]), min(a[1], b[1])
        return glob[2 * lo: 2 * hi] if hi > lo else None
    return ([view(OWN[me], NEED[r]) for r in range(2)], [view(OWN[q], NEED[me]) for q in range(2)])


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = DistComm()
        x = _inputs(rank)
        comm.allreduce_max([x["scale"]])
        comm.allreduce_max([x["table"]])
        comm.allreduce_max([x["nt"]])
        tot = comm.allgather([x["total"]])[0]
        pend = comm.allgather([x["pend"]])[0]
        comm.broadcast([x["records"]], src=1)
        comm.allreduce_sum([x["counts"]])
        comm.reduce_scatter_max([x["table2"]], SLICE_LO, SLICE_HI)
        glob = torch.zeros(2 * 12, dtype=torch.int64)  # this rank's record buffer
        glob[2 * OWN[rank][0]: 2 * OWN[rank][1]] = x["own"]
        sends, recvs = _pieces(glob, rank)
        comm.alltoallv([sends], [recvs])
        x["mine"] = glob[2 * NEED[rank][0]: 2 * NEED[rank][1]].clone()
        x["table2"] = x["table2"][SLICE_LO[rank]:SLICE_HI[rank]]
        # bench.py: max over ranks of the device times
        t = torch.tensor([1.5 + rank, 7.0 - rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        # plain lists: tensors through a Queue die with the sending process
        q.put((rank, {k: v.tolist() for k, v in x.items()}, tot.tolist(), pend.tolist(),
               t.tolist()))
    finally:
        dist.destroy_process_group()


def test_distcomm_matches_localcomm():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(world):
        r, x, tot, pend, t = q.get(timeout=120)
        res[r] = (x, tot, pend, t)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # the same collectives in one process (virtual shards)
    local = [_inputs(r) for r in range(world)]
    lc = LocalComm()
    for k in ("scale", "table", "nt"):
        lc.allreduce_max([d[k] for d in local])
    tot = lc.allgather([d["total"] for d in local])
    pend = lc.allgather([d["pend"] for d in local])
    lc.broadcast([d["records"] for d in local], src=1)
    lc.allreduce_sum([d["counts"] for d in local])
    lc.reduce_scatter_max([d["table2"] for d in local], SLICE_LO, SLICE_HI)
    globs = [torch.zeros(2 * 12, dtype=torch.int64) for _ in range(world)]
    for r in range(world):
        globs[r][2 * OWN[r][0]: 2 * OWN[r][1]] = local[r]["own"]
    pieces = [_pieces(globs[r], r) for r in range(world)]
    lc.alltoallv([p[0] for p in pieces], [p[1] for p in pieces])
    # the records' move: global record j lands at its place on the rank needing it
    truth = torch.cat([d["own"] for d in local])
    for r in range(world):
        mine = globs[r][2 * NEED[r][0]: 2 * NEED[r][1]]
        assert torch.equal(mine, truth[2 * NEED[r][0]: 2 * NEED[r][1]])
        local[r]["mine"] = mine.clone()
        local[r]["table2"] = local[r]["table2"][SLICE_LO[r]:SLICE_HI[r]]
    for r in range(world):
        x, dtot, dpend, t = res[r]
        for k in ("scale", "table", "nt", "records", "counts", "table2", "mine"):
            assert x[k] == local[r][k].tolist(), k
        assert dtot == tot[r].tolist() and dpend == pend[r].tolist()
        assert t == [2.5, 7.0]


@pytest.mark.parametrize("n,world", [(1 << 20, 8), (100003, 3), (4096, 1), (5000, 2)])
def test_shard_ranges(n, world):
    ranges = [shard_range(n, world, r) for r in range(world)]
    pos = 0
    for base, nl in ranges:
        assert base == pos or nl == 0
        assert base % 4096 == 0
        pos = base + nl
    assert pos == n
