"""A small run of every kernel family for compute-sanitizer (tests/test_gpu_sanitize.py):
the cooperative build in both tile configurations (4096- and 256-entry
tiles, power-of-two and general m, zeros, one-leaf cells), the small-build
row kernel, the batched rows, sampling, the 4-ary collapse and its sampler,
the 2-D build and sampler.  Exits 0 when every result equals the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1901_05423_b200 as rtf  # noqa: E402
from workloads import env_map, philox_xi, power_law, random_small  # noqa: E402


def dev(a, dt=np.float32):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).cuda()


def main():
    rng = np.random.default_rng(5)
    xi = philox_xi(1 << 14, seed=9)
    xi_d = dev(xi.view(np.int32), np.int32)
    cases = [(power_law(20000, "A"), 1 << 12), (random_small(rng, 9000, 0.3), 2000),
             (env_map(96, 64, seed=2), 96 * 64)]
    for p, m in cases:
        ref = oracle.build(p, m)
        for flags in (rtf.RTF_BUILD_DEFAULT, rtf.RTF_BUILD_SMALL_TILES):
            f = rtf.build(dev(p), m, flags)
            assert np.array_equal(f.nodes_numpy()["key"], ref.key)
            got = f.sample(xi_d).cpu().numpy()
            assert np.array_equal(got, ref.sample(xi)), "samples"
        f.build_quad()
        assert torch.equal(f.sample_quad(xi_d), f.sample(xi_d))
    small = rtf.build(dev(power_law(3000, "A")), 1024)  # n, m <= 4096: the row kernel
    assert small.status() == 0
    rows = np.abs(rng.standard_normal((64, 1024))).astype(np.float32)
    rf = rtf.build_rows(dev(rows), 256)
    torch.cuda.synchronize()
    img = env_map(128, 64, seed=3)
    f2 = rtf.build_2d(dev(img.reshape(64, 128)), 128, 64)
    pix = torch.empty(1 << 12, dtype=torch.int32, device="cuda")
    pos = torch.empty((1 << 12, 2), dtype=torch.float32, device="cuda")
    f2.sample(xi_d[: 1 << 12], xi_d[1 << 12: 2 << 12], pix, pos)
    torch.cuda.synchronize()
    del rf
    # round 2: packed three-interval cells (m = 2^17) in both tile configurations,
    # the degenerate-cell fallback and its bisecting sampler
    pk = random_small(rng, 150000, zero_frac=0.05, dyn=3.0)
    refp = oracle.build(pk, 1 << 17)
    for flags in (rtf.RTF_BUILD_DEFAULT, rtf.RTF_BUILD_SMALL_TILES):
        fp = rtf.build(dev(pk), 1 << 17, flags)
        assert np.array_equal(fp.table_numpy().view(np.uint64), refp.table3().view(np.uint64))
        assert np.array_equal(fp.sample(xi_d).cpu().numpy(), refp.sample(xi)), "packed samples"
    chain = np.concatenate([np.exp2(-np.arange(40, dtype=np.float64)), np.ones(5000)])
    chain = chain.astype(np.float32)
    refc = oracle.build(chain, 3)
    fc = rtf.build(dev(chain), 3).build_fallback()
    assert np.array_equal(fc.table_numpy().view(np.uint64), refc.table4().view(np.uint64))
    assert np.array_equal(fc.sample(xi_d).cpu().numpy(), refc.sample(xi)), "fallback samples"
    fc.sample_loads(xi_d)
    # baselines: Eytzinger and alias
    import baselines
    q = power_law(20000, "A")
    cdf = rtf.build_cdf(dev(q))
    assert np.array_equal(cdf.eytzinger().sample(xi_d).cpu().numpy(), oracle.build(q, 64).sample(xi))
    K, _ = oracle.cdf_all(q)
    prob, alias, ak = baselines.alias_table(K)
    got = rtf.Alias(prob, alias, ak).sample(xi_d).cpu().numpy()
    assert np.array_equal(got, baselines.alias_sample(prob, alias, ak, xi)), "alias"
    # 2-D rows wider than the row kernel (cooperative per-row builds + index maps)
    wide = np.stack([random_small(rng, 4200, zero_frac=0.2 * (y % 2)) for y in range(3)])
    f2w = rtf.build_2d(dev(wide), 5000, 3)
    pw = torch.empty(1 << 12, dtype=torch.int32, device="cuda")
    qw = torch.empty((1 << 12, 2), dtype=torch.float32, device="cuda")
    f2w.sample(xi_d[: 1 << 12], xi_d[1 << 12: 2 << 12], pw, qw)
    rp, _ = oracle.build_2d(wide, 5000, 3).sample(xi[: 1 << 12], xi[1 << 12: 2 << 12])
    assert np.array_equal(pw.cpu().numpy(), rp), "2-D wide rows"
    torch.cuda.synchronize()
    print("sanitize target ok")


if __name__ == "__main__":
    main()
