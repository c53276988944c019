"""GPU parity of the degenerate-cell fallback (reading R21, oracle O17;
Sec.3, Sec.4, Sec.6): the marked table
equals the oracle's O17 table, sampled indices stay the inverse CDF's, and a
marked cell is answered in at most ceil(log2(k + 1)) node reads."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from workloads import philox_xi, power_law, random_small  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rtf():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1901_05423_b200 as rtf
    rtf.lib()
    return rtf


def dev_u32(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint32).view(np.int32)).cuda()


def geometric_mix(rng, n_parts):
    parts = []
    for _ in range(n_parts):
        if rng.random() < 0.6:
            L = int(rng.integers(8, 60))
            parts.append(np.exp2(-np.arange(L, dtype=np.float64) * rng.uniform(0.7, 1.5))
                         * rng.uniform(1e-6, 1.0))
        else:
            parts.append(random_small(rng, int(rng.integers(1, 3000)), zero_frac=0.2, dyn=8.0))
    return np.concatenate(parts).astype(np.float32)


def check(rtf, p, m, rng, nx=1 << 16):
    ref = oracle.build(p, m)
    f = rtf.build(torch.from_numpy(p).cuda(), m).build_fallback()
    want = ref.table4()
    got = f.table_numpy()
    bad = np.flatnonzero((got["ref"] != want["ref"]) | (got["key32"] != want["key32"]))
    assert bad.size == 0, f"{bad.size} table cells differ, first at {bad[:5]}"
    marked = np.flatnonzero(oracle.is_bisect(want))
    # xi: every leaf boundary +-1, random, and a dense sweep of the marked cells
    ks = ref.key.astype(np.uint64)
    b = ((ks + np.uint64((1 << 31) - 1)) >> np.uint64(31)).astype(np.int64)
    xs = [b - 1, b, b + 1, rng.integers(0, 2**32, nx)]
    for g in marked[:64].tolist():
        lo, hi = -(-(g << 32) // m), -(-((g + 1) << 32) // m)
        xs.append(np.linspace(lo, hi - 1, 512).astype(np.int64))
    xs = np.concatenate(xs)
    xs = xs[(xs >= 0) & (xs < 2**32)].astype(np.uint32)
    out = f.sample(dev_u32(xs)).cpu().numpy()
    assert np.array_equal(out, ref.sample(xs)), "sampled indices"
    loads = f.sample_loads(dev_u32(xs)).cpu().numpy()
    cells = ((xs.astype(np.uint64) * np.uint64(m)) >> np.uint64(32)).astype(np.int64)
    for g in marked.tolist():
        sel = cells == g
        if np.any(sel):
            k = int(want["key32"][g]) & 0x3FFFFFFF
            assert int(loads[sel].max()) <= 1 + oracle.bisect_visits(k), g
    return marked.size


def test_fallback_random(rtf):
    rng = np.random.default_rng(51)
    marked = 0
    for t in range(16):
        p = geometric_mix(rng, int(rng.integers(1, 5)))
        if not np.any(p > 0):
            continue
        m = int(rng.choice([1, 3, 64, 1000, 1 << 17]))
        marked += check(rtf, p, m, rng)
    assert marked > 5


def test_fallback_power_law_full(rtf):
    """Config 3's distribution (family A, n = 2^24, m = 2^22): cell 0 holds
    about half of the leaves in a radix tree deeper than bisection + 4."""
    rng = np.random.default_rng(52)
    p = power_law(1 << 24, "A")
    assert check(rtf, p, 1 << 22, rng, nx=1 << 18) >= 1


def test_fallback_idempotent_and_rebuild(rtf):
    rng = np.random.default_rng(53)
    p = geometric_mix(rng, 3)
    f = rtf.build(torch.from_numpy(p).cuda(), 7)
    plain = f.table_numpy().tobytes()
    f.build_fallback()
    once = f.table_numpy().tobytes()
    f.build_fallback()
    assert f.table_numpy().tobytes() == once
    f.build(torch.from_numpy(p).cuda())
    assert f.table_numpy().tobytes() == plain
