"""GPU parity of the 2-D sampler (Sec.6; oracle O14/O15, reading R19):
row weights, pixels and sub-pixel positions bit-exact against the oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from workloads import env_map, philox_xi, random_small  # noqa: E402

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


def check(rtf, p, mx, my, xi1, xi2, sample_all=True):
    H, W = p.shape
    f = rtf.build_2d(torch.from_numpy(np.ascontiguousarray(p)).cuda(), mx, my)
    assert f.status() == 0
    q = oracle.marginal_weights(p)
    assert f.weights().tobytes() == q.tobytes(), "row weights"
    assert np.array_equal(f.dense_rows(), np.all(p > 0, axis=1)), "dense-row bits"
    pix, pos = f.sample(dev_u32(xi1), dev_u32(xi2))
    pix, pos = pix.cpu().numpy(), pos.cpu().numpy()
    ref = oracle.build_2d(p, mx, my)
    sel = np.arange(xi1.size) if sample_all else np.linspace(0, xi1.size - 1, 4096).astype(np.int64)
    rp, rpos = ref.sample(xi1[sel], xi2[sel])
    assert np.array_equal(pix[sel], rp), "pixels"
    assert pos[sel].tobytes() == rpos.tobytes(), "sub-pixel positions"
    # every sample: inside its pixel, never a zero-weight pixel
    y, x = pix // W, pix % W
    assert np.all(p.reshape(-1)[pix] > 0)
    assert np.all((pos[:, 0] >= x / W - 2.0**-23) & (pos[:, 0] < (x + 1) / W))
    assert np.all((pos[:, 1] >= y / H - 2.0**-23) & (pos[:, 1] < (y + 1) / H))


def test_2d_random_small(rtf):
    rng = np.random.default_rng(11)
    for t in range(30):
        H, W = int(rng.integers(1, 40)), int(rng.integers(1, 70))
        # zero-free rows (identity index maps) mixed with rows holding zeros
        p = np.stack([random_small(rng, W, zero_frac=0.3 if (t + y) % 2 else 0.0)
                      for y in range(H)])
        if t % 3 == 0:
            p[int(rng.integers(H))] = 0.0
            if not np.any(p > 0):
                p[0, 0] = 1.0
        n = 2000
        xi1 = np.concatenate([philox_xi(n, seed=t), [0, 2**32 - 1]]).astype(np.uint32)
        xi2 = np.concatenate([philox_xi(n, seed=100 + t), [2**32 - 1, 0]]).astype(np.uint32)
        check(rtf, p, int(rng.integers(1, 2 * W + 3)), int(rng.integers(1, 2 * H + 3)), xi1, xi2)


def test_2d_constant_image_identity(rtf):
    H, W = 512, 1024
    p = np.full((H, W), 2.5, np.float32)
    xi1, xi2 = philox_xi(1 << 16, seed=1), philox_xi(1 << 16, seed=2)
    f = rtf.build_2d(torch.from_numpy(p).cuda(), W, H)
    pix, pos = f.sample(dev_u32(xi1), dev_u32(xi2))
    a, b = xi1.astype(np.uint64), xi2.astype(np.uint64)
    assert np.array_equal(pix.cpu().numpy(), ((a * H >> 32) * W + (b * W >> 32)).astype(np.int32))
    # (xi2, xi1) / 2^32 truncated to float32: exact here
    want = np.stack([b, a], axis=1)
    drop = np.maximum(0, np.floor(np.log2(np.maximum(want, 1))).astype(np.int64) + 1 - 24)
    want = ((want >> drop.astype(np.uint64)) << drop.astype(np.uint64)).astype(np.float64) / 2**32
    assert np.array_equal(pos.cpu().numpy(), want.astype(np.float32))


def test_2d_envmap_full(rtf):
    """The C2 environment map (2048 x 1024) as a 2-D distribution: weights
    bit-exact, all 2^20 samples (pixels and positions) against the oracle."""
    p = env_map().reshape(1024, 2048)
    xi1, xi2 = philox_xi(1 << 20, seed=21), philox_xi(1 << 20, seed=22)
    check(rtf, p, 2048, 1024, xi1, xi2)


def test_2d_data_errors(rtf):
    p = np.ones((8, 16), np.float32)
    p[3, 5] = np.nan
    f = rtf.build_2d(torch.from_numpy(p).cuda(), 16, 8)
    assert f.status() == rtf._lib.RTF_EDATA
    pix = f.sample(dev_u32(philox_xi(100, seed=3)), dev_u32(philox_xi(100, seed=4)), with_pos=False)
    assert np.all(pix.cpu().numpy() == np.iinfo(np.int32).max)
    f = rtf.build_2d(torch.zeros((8, 16), dtype=torch.float32).cuda(), 16, 8)
    assert f.status() == rtf._lib.RTF_EALLZERO


def test_2d_quadratic_error_qmc_vs_mc(rtf):
    """The paper's convergence measure: e = sum_i (p_i - c_i/n)^2.
    Pseudo-random pairs give E[e] = sum p_i (1 - p_i) / n; the Hammersley set
    through the monotone inverse mapping keeps its stratification and lands
    well below that (tools/convergence.py, profiles/r01_convergence.jsonl)."""
    W, H, k = 2048, 1024, 20
    n = 1 << k
    img = env_map(W, H)
    dev = torch.device("cuda", 0)
    p = torch.from_numpy(img.astype(np.float64) / img.astype(np.float64).sum()).to(dev)
    f = rtf.build_2d(torch.from_numpy(img).reshape(H, W).to(dev), W, H)
    idx = np.arange(n, dtype=np.uint64)
    rev = np.zeros(n, dtype=np.uint64)
    for b in range(32):
        rev |= ((idx >> np.uint64(b)) & np.uint64(1)) << np.uint64(31 - b)
    qmc = (dev_u32((idx << np.uint64(32 - k)).astype(np.uint32)), dev_u32(rev.astype(np.uint32)))
    mc = (dev_u32(philox_xi(n, seed=5)), dev_u32(philox_xi(n, seed=6)))

    def err(x1, x2):
        pix = f.sample(x1, x2, with_pos=False)
        c = torch.bincount(pix.to(torch.int64), minlength=W * H).to(torch.float64)
        return float(((p - c / n) ** 2).sum())

    expected = float((p * (1 - p)).sum()) / n
    e_mc, e_qmc = err(*mc), err(*qmc)
    assert 0.8 * expected < e_mc < 1.2 * expected
    assert e_qmc < e_mc / 3


def test_2d_beyond_row_kernel(rtf):
    """Maps beyond the row kernel's 4096 entries / cells (Sec.6
    sets no size limit): rows of 8192 pixels (the 8192 x 4096 lat-long map,
    rows built by the cooperative kernel), more than 4096 rows (a cooperative
    marginal), and more than 4096 cells per row, with zeros and an all-zero
    row; weights, pixels and positions bit-exact vs oracle O14/O15."""
    rng = np.random.default_rng(12)
    cases = [(env_map(8192, 4096, seed=4).reshape(4096, 8192), 8192, 4096, 1 << 18)]
    p = np.stack([random_small(rng, 700, zero_frac=0.2 * (y % 3 == 0)) for y in range(5000)])
    p[17] = 0.0
    cases.append((p, 700, 6000, 1 << 16))
    p = np.stack([random_small(rng, 3000, zero_frac=0.5 * (y % 2)) for y in range(40)])
    cases.append((p, 5000, 40, 1 << 16))
    for k, (p, mx, my, ns) in enumerate(cases):
        xi1 = np.concatenate([philox_xi(ns, seed=30 + k), [0, 2**32 - 1]]).astype(np.uint32)
        xi2 = np.concatenate([philox_xi(ns, seed=40 + k), [2**32 - 1, 0]]).astype(np.uint32)
        check(rtf, p.astype(np.float32), mx, my, xi1, xi2)
