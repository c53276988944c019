"""The sharded build (config 4) across PROCESSES through
DistComm with the real kernels: two ranks on cuda:0 over gloo (collectives
staged through host memory, the fused build's peer stores into the other
process's forest buffer through a CUDA IPC mapping).  Every rank's cell slice
(records, table cells) and its samples are compared byte for byte with the
single-GPU build and with the oracle; the replicated protocol's full forest
too.  (A one-GPU lease cannot run NCCL with two ranks; the NVLink path is the
same code with symmetric memory and NCCL collectives.)"""
import os
import socket
import tempfile

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, outdir, mode, workload):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    import oracle
    import paper_1901_05423_b200 as rtf
    from paper_1901_05423_b200 import sharded
    from workloads import philox_xi, power_law, spikes

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        n = 1 << 18
        p = power_law(n, "A") if workload == "powerlaw" else spikes(n)
        m = 1 << 16
        comm = sharded.DistComm()
        base, nl = sharded.shard_range(n, world, rank)
        pd = torch.from_numpy(p).cuda()
        shards = sharded.make_shards_local(pd[base: base + nl].clone(), n, m, rank, world, base,
                                           alloc=comm.alloc if mode == "fused" else None)
        for _ in range(2):  # the second build reuses the uploaded peer pointers
            sharded.build_sharded(shards, comm, ranged=mode != "replicated",
                                  fused=mode == "fused")
        torch.cuda.synchronize()
        dist.barrier()
        s = shards[0]
        single = rtf.build(pd, m)
        ref = oracle.build(p, m)
        nodes, table = single.nodes_numpy(), single.table_numpy()
        f = rtf.Forest.from_buffer(n, m, s.forest)
        allrec = f._section(f.view.nodes, 16 * ref.n_pos).cpu().numpy().view(rtf.NODE_DTYPE)
        if mode == "replicated":
            assert allrec.tobytes() == nodes.tobytes(), f"rank {rank}: replicated records"
            assert f.table_numpy().tobytes() == table.tobytes(), f"rank {rank}: replicated table"
            assert np.array_equal(allrec["key"], ref.key)
            xi = philox_xi(1 << 16, seed=rank + 3)
            got = f.sample(torch.from_numpy(xi.view(np.int32)).cuda()).cpu().numpy()
            assert np.array_equal(got, ref.sample(xi)), f"rank {rank}: samples"
            covered = ref.n_pos if rank == 0 else 0
        else:
            (j0, j1), (g0, g1) = sharded.slots_of(s), s.cells
            assert allrec[j0:j1].tobytes() == nodes[j0:j1].tobytes(), f"rank {rank}: records"
            assert f.table_numpy()[g0:g1].tobytes() == table[g0:g1].tobytes(), f"rank {rank}: table"
            assert np.array_equal(allrec["key"][j0:j1], ref.key[j0:j1])
            xi = philox_xi(1 << 16, seed=rank + 3)
            xr = sharded.ranged_xi(torch.from_numpy(xi.view(np.int32)), rank, world, m)
            got = f.sample(xr.cuda()).cpu().numpy()
            assert np.array_equal(got, ref.sample(xr.numpy().view(np.uint32))), \
                f"rank {rank}: samples"
            covered = j1 - j0
        with open(os.path.join(outdir, f"r{rank}"), "w") as fh:
            fh.write(f"{covered} {ref.n_pos}")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["fused", "ranged", "replicated"])
@pytest.mark.parametrize("workload", ["powerlaw", "spikes"])
def test_sharded_build_two_processes(mode, workload):
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import torch.multiprocessing as mp
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, mode, workload), nprocs=world, join=True)
        got = [open(os.path.join(d, f"r{r}")).read().split() for r in range(world)]
    covered = sum(int(c) for c, _ in got)
    assert covered == int(got[0][1]), "the ranks' slots cover every node exactly once"
