"""Sharded build (config 4) on one GPU with virtual shards: the shards run the
per-shard kernels on their own buffers and exchange through LocalComm (the
same collectives NCCL performs across GPUs).  Every shard must end with the
forest the single-GPU build (and the oracle) produces, byte for byte."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from workloads import philox_xi, power_law, random_small, spikes  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rtf():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1901_05423_b200 as rtf
    rtf.lib()
    return rtf


def _check(rtf, p, m, count):
    from paper_1901_05423_b200 import sharded
    pd = torch.from_numpy(p).cuda()
    shards = sharded.make_shards(pd, m, count)
    sharded.build_sharded(shards, sharded.LocalComm())
    ref = oracle.build(p, m)
    single = rtf.build(pd, m)
    want_nodes = single.nodes_numpy().tobytes()
    want_table = single.table_numpy().tobytes()
    assert np.array_equal(single.nodes_numpy()["c1"], ref.child1)
    assert want_table == ref.table3().tobytes()
    for s in shards:
        f = rtf.Forest.from_buffer(s.n_global, m, s.forest)
        assert f.status() == 0
        assert f.n_pos() == ref.n_pos
        assert f.nodes_numpy().tobytes() == want_nodes, f"shard {s.rank} records"
        assert f.table_numpy().tobytes() == want_table, f"shard {s.rank} table"
        xi = philox_xi(1 << 16, seed=s.rank)
        got = f.sample(torch.from_numpy(xi.view(np.int32)).cuda()).cpu().numpy()
        assert np.array_equal(got, ref.sample(xi))


@pytest.mark.parametrize("count", [1, 2, 3, 4])
def test_sharded_power_law(rtf, count):
    # the giant cell of p_i ~ i^20 spans every shard: many cross-shard merges
    _check(rtf, power_law(1 << 18, "A"), 1 << 16, count)


@pytest.mark.parametrize("count", [2, 5])
def test_sharded_spikes_and_random(rtf, count):
    _check(rtf, spikes(3 << 16), 1 << 15, count)
    rng = np.random.default_rng(count)
    _check(rtf, random_small(rng, 100003, zero_frac=0.3, dyn=12.0), 77777, count)


def test_sharded_config4_shape(rtf):
    """Config 4's distribution (4 spikes, uniform background) at 2^22 over 8 shards."""
    _check(rtf, spikes(1 << 22), 1 << 20, 8)


def test_config4_full_size_sampled(rtf):
    """Config 4 at its full size (n = 2^28 spikes, m = 2^22, the bench's shape):
    the single-GPU build and the sharded protocol over 4 virtual shards give
    byte-identical forests, and 2^20 Philox samples match the oracle's binary
    search over the oracle's full fixed-point CDF (O1-O6 + the P:61-63
    definition, computed independently of any forest) one by one."""
    from paper_1901_05423_b200 import sharded
    n, m = 1 << 28, 1 << 22
    p = spikes(n)
    K, _ = oracle.cdf_all(p)
    xi = philox_xi(1 << 20, seed=0x5EED)
    want = oracle.sample_bsearch(K, xi)
    del K
    pd = torch.from_numpy(p).cuda()
    xd = torch.from_numpy(xi.view(np.int32)).cuda()
    single = rtf.build(pd, m)
    assert single.status() == 0
    assert np.array_equal(single.sample(xd).cpu().numpy(), want)
    nodes = single.nodes_numpy()
    table = single.table_numpy()
    del single
    torch.cuda.empty_cache()
    shards = sharded.make_shards(pd, m, 4)
    sharded.build_sharded(shards, sharded.LocalComm())
    for s in shards[:2]:  # every shard holds the same forest; compare two
        f = rtf.Forest.from_buffer(s.n_global, m, s.forest)
        assert f.nodes_numpy().tobytes() == nodes.tobytes(), f"shard {s.rank} records"
        assert f.table_numpy().tobytes() == table.tobytes(), f"shard {s.rank} table"
        assert np.array_equal(f.sample(xd).cpu().numpy(), want)


def _check_ranged(rtf, p, m, count, fused=False):
    from paper_1901_05423_b200 import sharded
    pd = torch.from_numpy(p).cuda()
    single = rtf.build(pd, m)
    nodes, table = single.nodes_numpy(), single.table_numpy()
    ref = oracle.build(p, m)
    shards = sharded.make_shards(pd, m, count)
    sharded.build_sharded(shards, sharded.LocalComm(), ranged=True, fused=fused)
    covered = 0
    for s in shards:
        f = rtf.Forest.from_buffer(s.n_global, m, s.forest)
        (j0, j1), (g0, g1) = sharded.slots_of(s), s.cells
        covered += j1 - j0
        allrec = f._section(f.view.nodes, 16 * ref.n_pos).cpu().numpy().view(rtf.NODE_DTYPE)
        assert allrec[j0:j1].tobytes() == nodes[j0:j1].tobytes(), f"shard {s.rank} records"
        assert f.table_numpy()[g0:g1].tobytes() == table[g0:g1].tobytes(), f"shard {s.rank} table"
        xi = philox_xi(1 << 15, seed=s.rank + 7)
        xr = sharded.ranged_xi(torch.from_numpy(xi.view(np.int32)), s.rank, count, m)
        cells = (xr.numpy().view(np.uint32).astype(np.uint64) * m) >> 32
        assert np.all((cells >= g0) & (cells < g1))
        got = f.sample(xr.cuda()).cpu().numpy()
        assert np.array_equal(got, ref.sample(xr.numpy().view(np.uint32))), f"shard {s.rank} samples"
    assert covered == ref.n_pos


@pytest.mark.parametrize("count", [1, 2, 4, 8])
def test_sharded_ranged_power_law(rtf, count):
    # cell 0 of p_i ~ i^20 holds half the leaves: shard 0's cell range owns
    # records built by most other shards
    _check_ranged(rtf, power_law(1 << 18, "A"), 1 << 16, count)


@pytest.mark.parametrize("count", [2, 4])
def test_sharded_ranged_spikes_random(rtf, count):
    _check_ranged(rtf, spikes(3 << 16), 1 << 15, count)
    rng = np.random.default_rng(10 + count)
    _check_ranged(rtf, random_small(rng, 100003, zero_frac=0.3, dyn=12.0), 1 << 16, count)


@pytest.mark.parametrize("count", [2, 4, 8])
def test_sharded_fused_peer_stores(rtf, count):
    """Fused ranged build: records and table cells stored straight into the
    owner's buffer by the build kernel (peer pointers = the virtual shards'
    buffers); byte-equal cell slices, exact samples."""
    _check_ranged(rtf, power_law(1 << 18, "A"), 1 << 16, count, fused=True)
    _check_ranged(rtf, spikes(3 << 16), 1 << 15, count, fused=True)
    rng = np.random.default_rng(20 + count)
    _check_ranged(rtf, random_small(rng, 4096 * 3 * count - 100, zero_frac=0.3, dyn=12.0),
                  1 << 16, count, fused=True)


def test_config4_full_size_records_vs_oracle(rtf):
    """Config 4 at its full size (n = 2^28 spikes, m = 2^22): EVERY node record
    (key and both children) and EVERY guide-table cell of the single-GPU build
    equal the oracle's (O1-O13, about 8 GB of host arrays); then the fused
    ranged build over 4 virtual shards (the N > 1 default: peer stores into the
    owner's buffer) gives byte-equal cell slices, and 2^20 samples of each
    shard's xi stratum equal the single forest's."""
    from paper_1901_05423_b200 import sharded
    n, m = 1 << 28, 1 << 22
    p = spikes(n)
    pd = torch.from_numpy(p).cuda()
    single = rtf.build(pd, m)
    assert single.status() == 0
    nodes = single.nodes_numpy()
    table = single.table_numpy()
    del single
    torch.cuda.empty_cache()
    ref = oracle.build(p, m)
    assert nodes.size == ref.n_pos
    assert np.array_equal(nodes["key"], ref.key), "keys"
    assert np.array_equal(nodes["c0"], ref.child0), "left children"
    assert np.array_equal(nodes["c1"], ref.child1), "right children"
    assert table.tobytes() == ref.table3().tobytes(), "guide table"
    del ref
    shards = sharded.make_shards(pd, m, 4)
    sharded.build_sharded(shards, sharded.LocalComm(), ranged=True, fused=True)
    covered = 0
    for s in shards:
        f = rtf.Forest.from_buffer(s.n_global, m, s.forest)
        (j0, j1), (g0, g1) = sharded.slots_of(s), s.cells
        covered += j1 - j0
        recs = f._section(f.view.nodes + 16 * j0, 16 * (j1 - j0)).cpu().numpy()
        assert recs.tobytes() == nodes[j0:j1].tobytes(), f"shard {s.rank} records"
        assert f.table_numpy()[g0:g1].tobytes() == table[g0:g1].tobytes(), f"shard {s.rank} table"
        xi = philox_xi(1 << 20, seed=40 + s.rank)
        xr = sharded.ranged_xi(torch.from_numpy(xi.view(np.int32)), s.rank, 4, m).cuda()
        got = f.sample(xr).cpu().numpy()
        # the definition on the verified keys: the last key <= xi 2^31;
        # no zero weights here (n' = n), so leaf index = original index
        want = np.searchsorted(nodes["key"], xr.cpu().numpy().view(np.uint32).astype(np.uint64)
                               << np.uint64(31), side="right") - 1
        assert np.all((want >= j0) & (want < j1)), f"shard {s.rank}: xi outside its stratum"
        assert np.array_equal(got, want.astype(np.int32)), f"shard {s.rank} samples"
    assert covered == nodes.size == n


@pytest.mark.parametrize("count", [2, 3, 8])
def test_sharded_packed_cells(rtf, count):
    """Packed three-interval cells (R20, m = 2^17 and 2^18 power-of-two
    tables with m near n) across shard boundaries, in the replicated, ranged
    and fused builds: every shard's table equals the single build's (and the
    oracle's O16 table), including cells whose two leaves sit on two shards."""
    rng = np.random.default_rng(60 + count)
    p = random_small(rng, 4096 * 40 * count + 77, zero_frac=0.05, dyn=3.0)
    _check(rtf, p, 1 << 17, count)
    if (1 << 17) % count == 0:  # ranged shards own m / count cells each
        _check_ranged(rtf, p, 1 << 17, count)
    if (1 << 18) % count == 0:
        _check_ranged(rtf, random_small(rng, 4096 * 70 * count, zero_frac=0.0, dyn=2.0),
                      1 << 18, count, fused=True)
