"""4-ary collapsed records (rtf_build_quad / rtf_sample_quad): the
indices equal rtf_sample's and the oracle's on the same forests and xi, and a
32-B record holds its node's and its children's decisions."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from workloads import (FIG6_WEIGHTS, env_map, philox_xi, power_law, random_small,  # noqa: E402
                       spikes)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rtf():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1901_05423_b200 as rtf
    rtf.lib()
    return rtf


def dev_f32(p):
    return torch.from_numpy(np.ascontiguousarray(p, dtype=np.float32)).cuda()


def dev_u32(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint32).view(np.int32)).cuda()


def boundary_xi(ref, rng, k):
    """xi at, just below and just above interval boundaries (ceil(key / 2^31))."""
    key = ref.key.astype(np.uint64)
    c = (key >> np.uint64(31)) + ((key & np.uint64(0x7FFFFFFF)) != 0)
    pick = c[rng.integers(0, c.size, k)]
    xs = np.concatenate([pick, pick - 1, pick + 1, [0, 2**32 - 1]])
    return np.clip(xs, 0, 2**32 - 1).astype(np.uint32)


def check(rtf, p, m, xi):
    ref = oracle.build(p, m)
    f = rtf.build(dev_f32(p), m).build_quad()
    got = f.sample_quad(dev_u32(xi)).cpu().numpy()
    want = f.sample(dev_u32(xi)).cpu().numpy()
    assert np.array_equal(got, want)
    assert np.array_equal(got, ref.sample(xi))
    return f, ref


def test_quad_records_fig6(rtf):
    p = np.array(FIG6_WEIGHTS, np.float32)
    f, ref = check(rtf, p, 12, np.arange(0, 2**32, 2**20, dtype=np.uint64).astype(np.uint32))
    rec = f._rec4[: 32 * ref.n_pos].cpu().numpy().view(np.uint32).reshape(-1, 8)
    for j in range(ref.n_pos):
        k = ref.key.astype(np.uint64)
        ceil = lambda v: int((int(v) + (1 << 31) - 1) >> 31)
        assert rec[j, 0] == ceil(k[j]) & 0xFFFFFFFF
        for i, c in enumerate((ref.child0[j], ref.child1[j])):
            g = rec[j, 4 + 2 * i: 6 + 2 * i].view(np.int32)
            if c >= 0:
                assert rec[j, 1 + i] == ceil(k[c]) & 0xFFFFFFFF
                assert g[0] == ref.child0[c] and g[1] == ref.child1[c]
            else:
                assert g[0] == c and g[1] == c


def test_quad_random_small(rtf):
    rng = np.random.default_rng(31)
    for t in range(60):
        n = int(rng.choice([1, 2, 3, 17, 100, 4096, 4097, 9000]))
        m = int(rng.integers(1, 2 * n + 3))
        p = random_small(rng, n, zero_frac=0.3)
        ref = oracle.build(p, m)
        check(rtf, p, m, np.concatenate([philox_xi(4093, seed=t), boundary_xi(ref, rng, 200)]))


def test_quad_power_law_spikes_envmap(rtf):
    rng = np.random.default_rng(5)
    for p, m in ((power_law(1 << 20, "A"), 1 << 18), (spikes(1 << 22), 1 << 20),
                 (env_map(), 2048 * 1024)):
        ref = oracle.build(p, m)
        check(rtf, p, m, np.concatenate([philox_xi(1 << 20, seed=9), boundary_xi(ref, rng, 4096)]))


def test_quad_poisoned_and_deep(rtf):
    p = np.array([1.0, np.nan, 2.0], np.float32)
    f = rtf.build(dev_f32(p), 4).build_quad()
    assert np.all(f.sample_quad(dev_u32(philox_xi(64, seed=1))).cpu().numpy() == 2**31 - 1)
    g = np.exp2(-np.arange(120, dtype=np.float64)).astype(np.float32)  # a deep chain
    check(rtf, g, 2, np.concatenate([philox_xi(4096, seed=2), boundary_xi(oracle.build(g, 2),
                                                                           np.random.default_rng(0), 256)]))


def test_quad_records_invalidated_by_rebuild(rtf):
    """After build(p1); build_quad(); build(p2) the 4-ary records describe p1:
    sample_quad must refuse until build_quad() runs again, then match p2."""
    p1 = power_law(1 << 14, "A")
    p2 = env_map(128, 128, seed=4)
    m = 1 << 12
    f = rtf.Forest(p1.size, m).build(dev_f32(p1)).build_quad()
    xi = dev_u32(philox_xi(1 << 14, seed=3))
    f.build(dev_f32(p2))
    with pytest.raises(RuntimeError):
        f.sample_quad(xi)
    f.build_quad()
    assert torch.equal(f.sample_quad(xi), f.sample(xi))
    ref = oracle.build(p2, m)
    assert np.array_equal(f.sample(xi).cpu().numpy(), ref.sample(xi.cpu().numpy().view(np.uint32)))
