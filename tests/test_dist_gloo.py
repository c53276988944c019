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
    }


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
    for r in range(world):
        x, dtot, dpend, t = res[r]
        for k in ("scale", "table", "nt", "records"):
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
