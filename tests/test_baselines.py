"""The comparison baselines bench.py reports give the inverse-CDF answers of
the oracle: the OpenMP binary search (CPU) here, the GPU cutpoint baselines in
the -m gpu part."""
import numpy as np
import pytest

import baselines
import oracle
from workloads import philox_xi, power_law, random_small


def test_cpu_bsearch_matches_oracle():
    rng = np.random.default_rng(31)
    for n in (1, 2, 17, 5000, 70001):
        p = random_small(rng, n, zero_frac=0.3, dyn=8.0)
        K, _ = oracle.cdf_all(p)
        xi = philox_xi(50000, seed=n)
        assert np.array_equal(baselines.bsearch(K, xi), oracle.build(p, 64).sample(xi))


@pytest.mark.gpu
def test_gpu_cutpoint_baselines_match_oracle():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1901_05423_b200 as rtf
    rng = np.random.default_rng(32)
    cases = [(random_small(rng, n, zero_frac=z, dyn=8.0), m)
             for n, m, z in ((1, 1, 0.0), (17, 5, 0.3), (4097, 4096, 0.5), (70001, 333, 0.2))]
    cases.append((power_law(1 << 18, "A"), 1 << 16))
    for p, m in cases:
        ref = oracle.build(p, m)
        cdf = rtf.build_cdf(torch.from_numpy(p).cuda())
        cut = cdf.cutpoint(m)
        xi = np.concatenate([philox_xi(1 << 16, seed=m),
                             ((np.arange(m, dtype=np.uint64) << 32) // m).astype(np.uint32)])
        xd = torch.from_numpy(xi.view(np.int32)).cuda()
        want = ref.sample(xi)
        for binary in (True, False):
            got = cut.sample(xd, binary=binary).cpu().numpy()
            assert np.array_equal(got, want), (p.size, m, binary)


@pytest.mark.gpu
def test_gpu_eytzinger_baseline_matches_oracle():
    """The Eytzinger-layout binary search returns the oracle's inverse CDF:
    trees of height 0 (n = 1) to 20, shallower and deeper than the 13
    shared-memory levels, ragged sample counts (scalar tail), zero weights."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1901_05423_b200 as rtf
    rng = np.random.default_rng(33)
    cases = [random_small(rng, n, zero_frac=z, dyn=8.0)
             for n, z in ((1, 0.0), (2, 0.0), (3, 0.3), (4096, 0.5), (8193, 0.2), (70001, 0.3))]
    cases.append(power_law(1 << 20, "A"))
    for p in cases:
        ref = oracle.build(p, 64)
        cdf = rtf.build_cdf(torch.from_numpy(p).cuda())
        ey = cdf.eytzinger()
        K, _ = oracle.cdf_all(p)
        edges = np.clip(np.concatenate([K[:64] >> 31, (K[:64] >> 31) + 1, (K[-64:] >> 31) - 1,
                                        K[-64:] >> 31]), 0, 2**32 - 1).astype(np.uint32)
        xi = np.concatenate([philox_xi((1 << 16) + 3, seed=p.size), edges,
                             np.array([0, 2**32 - 1], np.uint32)])
        want = ref.sample(xi)
        for xs, w in ((xi, want), (xi[1:], want[1:])):  # aligned, then misaligned (scalar path)
            got = ey.sample(torch.from_numpy(xs.view(np.int32)).cuda()).cpu().numpy()
            assert np.array_equal(got, w), p.size


def _alias_counts(prob, alias, k):
    """xi count per item that the table realises (bucket b keeps prob[b] of its
    2^(32-k) values for item b and gives the rest to alias[b])."""
    s = 1 << (32 - k)
    cnt = np.zeros(prob.size, np.int64)
    np.add.at(cnt, np.arange(prob.size), prob.astype(np.int64))
    np.add.at(cnt, alias.astype(np.int64), s - prob.astype(np.int64))
    return cnt


def test_alias_table_realises_the_inverse_cdf_counts():
    """The alias table (baselines/alias.c, the comparison system of Sec.2.6
    P:203-239) gives every item exactly the number of 32-bit xi the inverse
    mapping gives it (ceil(K_{i+1}/2^31) - ceil(K_i/2^31), from the oracle's
    CDF); padding buckets own nothing; brute force over all xi of a few
    buckets agrees with the counts."""
    rng = np.random.default_rng(71)
    for n in (1, 2, 3, 17, 1000, 4097, 70000):
        p = random_small(rng, n, zero_frac=0.3, dyn=10.0)
        K, _ = oracle.cdf_all(p)
        prob, alias, k = baselines.alias_table(K)
        kc = np.array([-(-int(x) >> 31) for x in K] + [1 << 32], dtype=np.int64)
        cnt = _alias_counts(prob, alias, k)
        assert np.array_equal(cnt[:n], np.diff(kc)), n
        assert int(cnt[n:].sum()) == 0
    # every xi of 8 buckets, item by item
    p = random_small(rng, 300, zero_frac=0.2, dyn=6.0)
    K, _ = oracle.cdf_all(p)
    prob, alias, k = baselines.alias_table(K)
    for b in (0, 1, 7, 100, 255, 299, 300, 511):
        xs = np.arange(b << (32 - k), (b + 1) << (32 - k), dtype=np.uint64).astype(np.uint32)
        got = baselines.alias_sample(prob, alias, k, xs)
        want = np.where(np.arange(xs.size) < prob[b], b, alias[b])
        assert np.array_equal(got, want), b


@pytest.mark.gpu
def test_gpu_alias_sampler_matches_table():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1901_05423_b200 as rtf
    rng = np.random.default_rng(72)
    for n in (2, 1000, 70001, 1 << 20):
        p = random_small(rng, n, zero_frac=0.3, dyn=10.0)
        K, _ = oracle.cdf_all(p)
        prob, alias, k = baselines.alias_table(K)
        a = rtf.Alias(prob, alias, k)
        xi = np.concatenate([philox_xi((1 << 18) + 3, seed=n), np.array([0, 2**32 - 1], np.uint32)])
        for xs in (xi, xi[1:]):  # vector and scalar paths
            got = a.sample(torch.from_numpy(xs.view(np.int32)).cuda()).cpu().numpy()
            assert np.array_equal(got, baselines.alias_sample(prob, alias, k, xs)), n


def _alias_2d_case(rng, W=37, H=11):
    p2d = np.stack([random_small(rng, W, zero_frac=0.3, dyn=8.0) for _ in range(H)])
    p2d[3] = 0.0  # a zero row: the marginal never selects it
    q = oracle.marginal_weights(p2d)
    K_marg, _ = oracle.cdf_all(q)
    K_rows = [oracle.cdf_all(p2d[y])[0] if np.any(p2d[y] > 0) else None for y in range(H)]
    return p2d, K_marg, K_rows


def test_alias_2d_tables_realise_the_inverse_counts():
    """The 2-D alias baseline's tables (baselines.alias_2d): the marginal table
    gives row y exactly the xi1 count the marginal inverse mapping gives it, and
    row y's table gives column x exactly the xi2 count of row y's inverse
    mapping (both from the oracle's fixed-point CDFs, P:61-63 and Sec.6
    P:1523-1529); padding buckets own nothing."""
    rng = np.random.default_rng(73)
    p2d, K_marg, K_rows = _alias_2d_case(rng)
    H, W = p2d.shape
    (mp, ma, ky), (rp, ra, kx) = baselines.alias_2d(K_marg, K_rows)
    want_m = np.diff(np.array([-(-int(x) >> 31) for x in K_marg] + [1 << 32], dtype=np.int64))
    cm = _alias_counts(mp, ma, ky)
    assert np.array_equal(cm[:H], want_m) and cm[3] == 0 and int(cm[H:].sum()) == 0
    for y in range(H):
        if K_rows[y] is None:
            continue
        want = np.diff(np.array([-(-int(x) >> 31) for x in K_rows[y]] + [1 << 32], dtype=np.int64))
        c = _alias_counts(rp[y], ra[y], kx)
        assert np.array_equal(c[:W], want), y
        assert int(c[W:].sum()) == 0


@pytest.mark.gpu
def test_gpu_alias_2d_sampler_matches_tables():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1901_05423_b200 as rtf
    rng = np.random.default_rng(74)
    p2d, K_marg, K_rows = _alias_2d_case(rng, W=300, H=70)
    H, W = p2d.shape
    marg, rows = baselines.alias_2d(K_marg, K_rows)
    a = rtf.Alias2D(marg, rows, W, H)
    x1 = np.concatenate([philox_xi(1 << 18, seed=1), np.array([0, 2**32 - 1], np.uint32)])
    x2 = np.concatenate([philox_xi(1 << 18, seed=2), np.array([2**32 - 1, 0], np.uint32)])
    got = a.sample(torch.from_numpy(x1.view(np.int32)).cuda(),
                   torch.from_numpy(x2.view(np.int32)).cuda()).cpu().numpy()
    y = baselines.alias_sample(*marg, x1)
    (rp, ra, kx) = rows
    b = (x2 >> np.uint32(32 - kx)).astype(np.int64)
    frac = x2.astype(np.int64) & ((1 << (32 - kx)) - 1)
    x = np.where(frac < rp[y, b], b, ra[y, b])
    assert np.array_equal(got, (y * W + x).astype(np.int32))
    assert not np.any(y == 3)
