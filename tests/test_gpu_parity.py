"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element
by element on the same seeded inputs.  Everything here is integer / index work,
so the bar is bit-exact."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from workloads import (FIG6_WEIGHTS, SPEC_WEIGHTS, TEASER_WEIGHTS, env_map,  # noqa: E402
                       hammersley_xi, philox_xi, power_law, random_small, rows_lognormal,
                       sine64, sobol0_xi, spikes, stratified_xi)

pytestmark = pytest.mark.gpu

DEV = "cuda"


@pytest.fixture(scope="module")
def rtf():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1901_05423_b200 as rtf
    rtf.lib()
    return rtf


def dev_f32(p):
    return torch.from_numpy(np.ascontiguousarray(p, dtype=np.float32)).to(DEV)


def dev_u32(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint32).view(np.int32)).to(DEV)


def assert_forest_equal(f, ref, what=""):
    assert f.status() == 0, what
    h = f.header()
    assert h.n_pos == ref.n_pos and h.total == ref.T, what
    nodes = f.nodes_numpy()
    assert np.array_equal(nodes["key"], ref.key), f"{what}: keys"
    bad = np.flatnonzero((nodes["c0"] != ref.child0) | (nodes["c1"] != ref.child1))
    assert bad.size == 0, f"{what}: {bad.size} node records differ, first at {bad[:5]}"
    tab = f.table_numpy()
    want = ref.table3()  # the table the build produces (O16: packed two-leaf cells)
    badt = np.flatnonzero((tab["ref"] != want["ref"]) | (tab["key32"] != want["key32"]))
    assert badt.size == 0, f"{what}: {badt.size} table cells differ, first at {badt[:5]}"


def boundary_xi(ref, rng, extra=4096):
    ks = ref.key.astype(np.uint64)
    b = ((ks + np.uint64((1 << 31) - 1)) >> np.uint64(31)).astype(np.int64)  # ceil(k / 2^31)
    xs = np.concatenate([b - 1, b, b + 1, rng.integers(0, 2**32, extra),
                         (np.arange(ref.m, dtype=np.int64) << 32) // ref.m, [0, 2**32 - 1]])
    xs = xs[(xs >= 0) & (xs < 2**32)]
    return xs.astype(np.uint32)


def check_sampling(f, ref, xi):
    got = f.sample(dev_u32(xi)).cpu().numpy()
    want = ref.sample(xi)
    bad = np.flatnonzero(got != want)
    assert bad.size == 0, f"{bad.size} samples differ; first xi={xi[bad[:3]]} got={got[bad[:3]]} want={want[bad[:3]]}"


# ---------------------------------------------------------------- paper examples

@pytest.mark.parametrize("flags", [0, 1])
def test_paper_examples(rtf, flags):
    rng = np.random.default_rng(0)
    for w, m in ((FIG6_WEIGHTS, 12), (SPEC_WEIGHTS, 4), (TEASER_WEIGHTS, 8), (sine64(), 64)):
        p = np.asarray(w, np.float32)
        f = rtf.build(dev_f32(p), m, flags)
        ref = oracle.build(p, m)
        assert_forest_equal(f, ref, f"m={m}")
        check_sampling(f, ref, boundary_xi(ref, rng))
    # teaser: the 1024-point Hammersley set (config 1) splits exactly 16 w
    f = rtf.build(dev_f32(TEASER_WEIGHTS), 8, flags)
    x, _ = hammersley_xi(1024)
    got = f.sample(dev_u32(x)).cpu().numpy()
    assert np.bincount(got, minlength=16).tolist() == [16 * v for v in TEASER_WEIGHTS]


# ---------------------------------------------------------------- random / edge cases

@pytest.mark.parametrize("flags", [0, 1])
def test_random_small(rtf, flags):
    rng = np.random.default_rng(1 + flags)
    for t in range(120):
        n = int(rng.choice([1, 2, 3, 5, 17, 127, 128, 129, 1000, 4095, 4096, 4097, 9000, 20000]))
        m = int(max(1, rng.choice([1, n // 7, n // 2, n, 2 * n + 3, 5])))
        p = random_small(rng, n, zero_frac=float(rng.choice([0, 0.2, 0.9])),
                         dyn=float(rng.choice([0.3, 4, 16, 40])))
        ref = oracle.build(p, m)
        f = rtf.build(dev_f32(p), m, flags)
        assert_forest_equal(f, ref, f"case {t} n={n} m={m}")
        check_sampling(f, ref, boundary_xi(ref, rng, 512))


@pytest.mark.parametrize("flags", [0, 1])
def test_packed_two_leaf_cells(rtf, flags):
    """Power-of-two tables with m >= 2^17 hold the packed three-interval cells
    of reading R20 (oracle O16): many two-leaf cells (m near n), zero weights
    between them (no packing then), cells across tile boundaries (small tiles
    put most of them there), the packing threshold m = 2^17 and below it."""
    rng = np.random.default_rng(11 + flags)
    for t, (n, m, z) in enumerate(((70000, 1 << 17, 0.0), (70000, 1 << 16, 0.0),
                                   (150000, 1 << 17, 0.3), (200000, 1 << 18, 0.05),
                                   (300000, 1 << 17, 0.0), (1 << 20, 1 << 19, 0.1))):
        p = random_small(rng, n, zero_frac=z, dyn=float(rng.choice([0.5, 4])))
        ref = oracle.build(p, m)
        f = rtf.build(dev_f32(p), m, flags)
        assert_forest_equal(f, ref, f"case {t} n={n} m={m}")
        t3 = ref.table3()
        packed = int(np.count_nonzero((t3["ref"] >= 0) & (t3["key32"] != 0)))
        assert (packed > 0) == (m >= 1 << 17), (t, packed)
        check_sampling(f, ref, boundary_xi(ref, rng, 4096))


def test_edge_cases(rtf):
    rng = np.random.default_rng(3)
    cases = []
    cases.append((np.array([3.0], np.float32), 1))                     # n = 1
    cases.append((np.array([0, 0, 5, 0, 0], np.float32), 3))           # single positive
    z = np.zeros(20000, np.float32); z[[0, 19999]] = 1; cases.append((z, 64))   # sparse ends
    z = np.zeros(20000, np.float32); z[9000:9010] = 2; cases.append((z, 7))     # zero tiles
    cases.append((np.full(10000, 1e-45, np.float32), 100))             # all subnormal
    g = np.exp2(-np.arange(200, dtype=np.float64)).astype(np.float32)  # geometric: deep chain
    cases.append((g, 4))
    cases.append((np.ones(70000, np.float32), 1))                      # m = 1: one radix tree
    cases.append((random_small(rng, 5000), 40000))                     # m >> n
    # one ragged tile in the cooperative kernel (n <= 4096 with m <= 4096 goes
    # to the row kernel instead)
    cases.append((random_small(rng, 3000), 5000))
    cases.append((random_small(rng, 100), 8192))
    big = np.ones(6000, np.float32); big[::3] = 3e38; cases.append((big, 999))  # huge values
    for k, (p, m) in enumerate(cases):
        ref = oracle.build(p, m)
        f = rtf.build(dev_f32(p), m)
        assert_forest_equal(f, ref, f"edge {k}")
        check_sampling(f, ref, boundary_xi(ref, rng, 256))


def test_data_errors_poison(rtf):
    xi = dev_u32(np.arange(0, 2**32, 2**24, dtype=np.uint64).astype(np.uint32))
    for bad, code in (([1.0, float("nan")], rtf._lib.RTF_EDATA),
                      ([1.0, -2.0], rtf._lib.RTF_EDATA),
                      ([float("inf"), 1.0], rtf._lib.RTF_EDATA),
                      ([0.0, 0.0, -0.0], rtf._lib.RTF_EALLZERO)):
        p = np.zeros(5000, np.float32)
        p[:len(bad)] = bad
        f = rtf.build(dev_f32(p), 16)
        assert f.status() == code
        out = f.sample(xi).cpu().numpy()
        assert np.all(out == np.iinfo(np.int32).max)
        # a later valid build on the same buffers recovers
        good = random_small(np.random.default_rng(0), 5000)
        f.build(dev_f32(good))
        assert_forest_equal(f, oracle.build(good, 16), "recovery")


def test_argument_errors(rtf):
    import ctypes
    L = rtf.lib()
    view = rtf.rtf_forest()
    assert L.rtf_build(None, 10, 4, 0, None, 0, None, 0, None, ctypes.byref(view)) == rtf._lib.RTF_EINVAL
    f = rtf.Forest(100, 10)
    p = dev_f32(np.ones(100))
    assert L.rtf_build(ctypes.c_void_p(p.data_ptr()), 100, 0, 0, ctypes.c_void_p(f._buf.forest.data_ptr()),
                       f._buf.forest.numel(), ctypes.c_void_p(f._buf.ws.data_ptr()), f._buf.ws.numel(),
                       None, ctypes.byref(view)) == rtf._lib.RTF_EINVAL
    assert L.rtf_build(ctypes.c_void_p(p.data_ptr()), 100, 10, 0, ctypes.c_void_p(f._buf.forest.data_ptr()),
                       16, ctypes.c_void_p(f._buf.ws.data_ptr()), f._buf.ws.numel(),
                       None, ctypes.byref(view)) == rtf._lib.RTF_ENOSPACE


# ---------------------------------------------------------------- schedule independence

def test_repeat_builds_byte_identical(rtf):
    p = power_law(1 << 20, "A")
    m = 1 << 18
    ref = oracle.build(p, m)
    for flags in (0, 1):
        f = rtf.Forest(p.size, m, flags)
        pd = dev_f32(p)
        first = None
        for rep in range(20 if flags == 0 else 5):
            f.build(pd)
            nodes = f.nodes_numpy().tobytes() + f.table_numpy().tobytes()
            if first is None:
                first = nodes
                assert_forest_equal(f, ref, f"flags={flags}")
            assert nodes == first, f"rep {rep} differs"


def test_small_builds_same_bytes_from_both_kernels(rtf):
    """n, m <= 4096 goes to the row kernel (one CTA); RTF_BUILD_SMALL_TILES keeps
    the cooperative kernel.  Records [0, n'), table and header agree byte for byte."""
    rng = np.random.default_rng(21)
    for n, m in ((1, 1), (7, 3), (100, 4096), (1000, 17), (4096, 4096), (4096, 1)):
        p = random_small(rng, n, zero_frac=0.2)
        a, b = rtf.build(dev_f32(p), m, 0), rtf.build(dev_f32(p), m, 1)
        ha, hb = a.header(), b.header()
        assert bytes(ha) == bytes(hb), (n, m)
        k = ha.n_pos
        assert a.nodes_numpy()[:k].tobytes() == b.nodes_numpy()[:k].tobytes(), (n, m)
        assert a.table_numpy().tobytes() == b.table_numpy().tobytes(), (n, m)


# ---------------------------------------------------------------- workloads at scale

@pytest.mark.parametrize("fam", ["A", "B", "C", "D"])
def test_power_law_families_2_20(rtf, fam):
    p = power_law(1 << 20, fam)
    m = 1 << 18
    ref = oracle.build(p, m)
    f = rtf.build(dev_f32(p), m)
    assert_forest_equal(f, ref, fam)
    rng = np.random.default_rng(5)
    check_sampling(f, ref, np.concatenate([philox_xi(1 << 20, seed=11), boundary_xi(ref, rng, 0)[:1 << 20]]))


def test_config2_envmap_full(rtf):
    """Config 2 at full size: 2048x1024 env map, m = n, 2^26 Sobol samples."""
    p = env_map()
    m = p.size
    ref = oracle.build(p, m)
    f = rtf.build(dev_f32(p), m)
    assert_forest_equal(f, ref, "envmap")
    xi = sobol0_xi(1 << 26)
    got = f.sample(dev_u32(xi)).cpu().numpy()
    assert np.array_equal(got, ref.sample(xi))


def test_config3_full_size(rtf):
    """Config 3 at full size (n = 2^24, m = 2^22) in the bench's launch
    configuration: every node record and table cell vs the oracle; 2^22 of the
    bench's Philox samples vs the oracle one by one; all 2^30 bench samples vs
    the binary-search baseline (an independent search over the CDF, itself
    checked against the oracle's CDF)."""
    p = power_law(1 << 24, "A")
    m = 1 << 22
    ref = oracle.build(p, m)
    pd = dev_f32(p)
    f = rtf.build(pd, m)
    assert_forest_equal(f, ref, "C3")
    xi_d = rtf.philox(1 << 30, seed=0x5EED)
    head = xi_d[: 1 << 22].cpu().numpy().view(np.uint32)
    assert np.array_equal(head, philox_xi(1 << 22, seed=0x5EED))
    got = f.sample(xi_d)
    assert np.array_equal(got[: 1 << 22].cpu().numpy(), ref.sample(head))
    cdf = rtf.build_cdf(pd)
    K, T = oracle.cdf_all(p)
    assert np.array_equal(cdf.cdf.cpu().numpy().view(np.uint64), K)
    bs = cdf.sample(xi_d)
    assert torch.equal(bs, got)


def test_config5_rows_full(rtf):
    """Config 5: 65536 independent rows of 1024 entries (m_row = 1024)."""
    rows, n_row, m_row = 65536, 1024, 1024
    p = rows_lognormal(rows, n_row)
    ref = oracle.build_rows(p, rows, n_row, m_row)
    f = rtf.build_rows(dev_f32(p), m_row)
    hd = f.headers()
    assert f.last_status == 0
    assert np.array_equal(hd["n_pos"], ref["n_pos"]) and np.array_equal(hd["total"], ref["T"])
    nodes = f.nodes_numpy()
    valid = (np.arange(n_row)[None, :] < ref["n_pos"][:, None]).reshape(-1)
    assert np.array_equal(nodes["key"][valid], ref["key"][valid])
    assert np.array_equal(nodes["c0"][valid], ref["child0"][valid])
    assert np.array_equal(nodes["c1"][valid], ref["child1"][valid])
    assert_cells_equal(f.table_numpy(), rows_table2(ref, rows, n_row, m_row), "rows")
    # sampling (row, xi) pairs against per-row oracle forests
    rng = np.random.default_rng(2)
    r = rng.integers(0, rows, 1 << 16).astype(np.uint32)
    xi = philox_xi(1 << 16, seed=3)
    got = f.sample(dev_u32(r), dev_u32(xi)).cpu().numpy()
    for k in np.unique(r)[:300]:
        sel = r == k
        fr = oracle.build(p[k], m_row)
        assert np.array_equal(got[sel], fr.sample(xi[sel]))


def rows_table2(ref, rows, n_row, m_row, ok=None):
    """O13 per row from the oracle's batched build (each row independent, R15)."""
    out = np.zeros(rows * m_row, dtype=[("key32", "<u4"), ("ref", "<i4")])
    for r in range(rows):
        if ok is None or ok[r]:
            k = int(ref["n_pos"][r])
            sl = slice(r * n_row, r * n_row + k)
            out[r * m_row:(r + 1) * m_row] = oracle.table2_of(
                ref["table"][r * m_row:(r + 1) * m_row], ref["key"][sl], ref["orig"][sl],
                ref["cell"][sl], m_row)
    return out


def assert_cells_equal(got, want, what=""):
    bad = np.flatnonzero((got["ref"] != want["ref"]) | (got["key32"] != want["key32"]))
    assert bad.size == 0, f"{what}: {bad.size} table cells differ, first at {bad[:5]}"


def test_rows_random_shapes(rtf):
    rng = np.random.default_rng(9)
    # every kernel configuration: 64x4 (<= 256), 256x4 (<= 1024), 256x8 (<= 2048), 512x8
    for n_row, m_row in ((1, 1), (3, 7), (64, 16), (255, 256), (256, 257), (1000, 333),
                         (1024, 1024), (1025, 64), (1500, 700), (2048, 2048), (1024, 4096),
                         (4096, 4096), (2500, 100)):
        rows = 37
        p = np.stack([random_small(rng, n_row, zero_frac=0.3) for _ in range(rows)])
        p[5] = 0.0          # an all-zero row
        ref = oracle.build_rows(p, rows, n_row, m_row)
        f = rtf.build_rows(dev_f32(p), m_row)
        hd = f.headers()
        assert hd["status"][5] == rtf.RTF_DATA_ALLZERO and f.last_status == rtf._lib.RTF_EALLZERO
        ok = ref["status"] == 0
        assert np.array_equal(hd["n_pos"][ok], ref["n_pos"][ok])
        nodes = f.nodes_numpy()
        valid = ((np.arange(n_row)[None, :] < ref["n_pos"][:, None]) & ok[:, None]).reshape(-1)
        assert np.array_equal(nodes["key"][valid], ref["key"][valid])
        assert np.array_equal(nodes["c0"][valid], ref["child0"][valid])
        assert np.array_equal(nodes["c1"][valid], ref["child1"][valid])
        tab = f.table_numpy().reshape(rows, m_row)
        want = rows_table2(ref, rows, n_row, m_row, ok).reshape(rows, m_row)
        assert_cells_equal(tab[ok].reshape(-1), want[ok].reshape(-1), f"rows {n_row}x{m_row}")
        r = np.repeat(np.arange(rows, dtype=np.uint32), 64)
        xi = philox_xi(r.size, seed=n_row)
        got = f.sample(dev_u32(r), dev_u32(xi)).cpu().numpy()
        assert np.all(got[r == 5] == np.iinfo(np.int32).max)


def test_spikes_2_22(rtf):
    p = spikes(1 << 22)
    m = 1 << 20
    ref = oracle.build(p, m)
    f = rtf.build(dev_f32(p), m)
    assert_forest_equal(f, ref, "spikes")
    check_sampling(f, ref, philox_xi(1 << 20, seed=4))


# ---------------------------------------------------------------- host entry points, generator

def test_philox_generator(rtf):
    for start, count in ((0, 1000), (3, 17), (1 << 33, 4099)):
        got = rtf.philox(count, seed=99, start=start).cpu().numpy().view(np.uint32)
        assert np.array_equal(got, philox_xi(count, seed=99, start=start))


def test_host_entry_points(rtf):
    p = env_map(512, 256, seed=5)
    m = p.size // 3
    ref = oracle.build(p, m)
    f = rtf.Forest(p.size, m)
    p_host = torch.from_numpy(p).pin_memory()
    p_dev = torch.empty(p.size, dtype=torch.float32, device=DEV)
    assert rtf.build_host(f, p_host, p_dev) == 0
    assert_forest_equal(f, ref, "host build")
    xi = philox_xi(1_000_003, seed=5)
    xi_host = torch.from_numpy(xi.view(np.int32)).pin_memory()
    out_host = torch.empty(xi.size, dtype=torch.int32).pin_memory()
    chunk = 1 << 17
    xi_dev = torch.empty(2 * chunk, dtype=torch.int32, device=DEV)
    out_dev = torch.empty(2 * chunk, dtype=torch.int32, device=DEV)
    rtf.sample_host(f, xi_host, out_host, xi_dev, out_dev)
    assert np.array_equal(out_host.numpy(), ref.sample(xi))


def test_host_build_chunked_scale(rtf):
    """rtf_build_host copies p in chunks and runs phase A per chunk while the
    rest lands: the largest weight in the last chunk, a smaller maximum after
    a larger one (the scale word is cleared per call), a ragged n, a NaN in
    the last chunk and an all-zero input."""
    cases = [(power_law((1 << 20) + 3, "A"), 1 << 18),  # max at the very end, ragged n
             (power_law(300001, "D"), 70001),             # max at the start
             (env_map(1024, 512, seed=8) * np.float32(1e-3), 1 << 17)]
    for p, m in cases:
        ref = oracle.build(p, m)
        f = rtf.Forest(p.size, m)
        p_host = torch.from_numpy(np.ascontiguousarray(p, np.float32)).pin_memory()
        p_dev = torch.empty(p.size, dtype=torch.float32, device=DEV)
        big = torch.full_like(p_host, 1e30).pin_memory()
        assert rtf.build_host(f, big, p_dev) == 0          # a larger maximum first
        assert rtf.build_host(f, p_host, p_dev) == 0
        assert_forest_equal(f, ref, "chunked host build")
        assert f.header().exponent == ref_exponent(p)
        bad = p_host.clone().pin_memory()
        bad[-1] = float("nan")
        st = rtf.build_host(f, bad, p_dev)
        assert st == rtf._lib.RTF_EDATA and (f.header().status & rtf.RTF_DATA_NAN)
        zero = torch.zeros_like(p_host).pin_memory()
        assert rtf.build_host(f, zero, p_dev) == rtf._lib.RTF_EALLZERO
        assert rtf.build_host(f, p_host, p_dev) == 0       # recovers
        assert_forest_equal(f, ref, "chunked host build after poisoned inputs")
    # the 256-entry-tile configuration through the chunked path, and a small
    # build (the row kernel: one copy, no chunks)
    for p, m, flags in ((power_law(70001, "B"), 9001, rtf.RTF_BUILD_SMALL_TILES),
                        (power_law(3001, "A"), 1000, rtf.RTF_BUILD_DEFAULT)):
        ref = oracle.build(p, m)
        f = rtf.Forest(p.size, m, flags)
        p_host = torch.from_numpy(np.ascontiguousarray(p, np.float32)).pin_memory()
        p_dev = torch.empty(p.size, dtype=torch.float32, device=DEV)
        assert rtf.build_host(f, p_host, p_dev) == 0
        assert_forest_equal(f, ref, f"host build flags={flags} n={p.size}")


def ref_exponent(p):
    return int(np.floor(np.log2(np.float64(np.max(p)))))


def test_stratified_histogram_closed_form_gpu(rtf):
    p = env_map(1024, 512, seed=2)
    f = rtf.build(dev_f32(p), 4096)
    ref = oracle.build(p, 4096)
    N = 1 << 24
    got = f.sample(dev_u32(stratified_xi(N)))
    c = torch.bincount(got.long(), minlength=p.size).cpu().numpy()
    ks = [int(k) for k in ref.key] + [1 << 63]
    exp = np.zeros(p.size, np.int64)
    for j in range(ref.n_pos):
        exp[ref.orig[j]] = -(-N * ks[j + 1] >> 63) - -(-N * ks[j] >> 63)
    assert np.array_equal(c, exp)


def test_corrupted_forest_terminates(rtf):
    """Fault injection (SPEC S:274-275 idea): a child pointer rewritten into a
    cycle must not hang Alg. 2; affected samples report INT32_MIN."""
    p = np.ones(1000, np.float32)
    f = rtf.build(dev_f32(p), 1)  # one radix tree: every sample descends ~10 levels
    ref = oracle.build(p, 1)
    root = int(ref.child1[0])
    assert root >= 0
    off = f.view.nodes - f._buf.forest.data_ptr()
    rec = f._buf.forest[off: off + 16 * f.n].view(torch.int32).view(-1, 4)
    rec[root, 2] = root  # child0 of the root points back to itself
    rec[root, 3] = root
    xi = dev_u32(np.arange(0, 2**32, 2**22, dtype=np.uint64).astype(np.uint32))
    out = f.sample(xi).cpu().numpy()
    assert np.all(out == np.iinfo(np.int32).min)


def test_float_xi_entry(rtf):
    """rtf_sample_f32: float xi in [0, 1) is mapped to floor(xi 2^32) exactly
    (reading R11), then sampled as usual; out-of-range values saturate."""
    rng = np.random.default_rng(17)
    p = random_small(rng, 30000, zero_frac=0.2)
    f = rtf.build(dev_f32(p), 4096)
    ref = oracle.build(p, 4096)
    xf = np.concatenate([rng.random(1 << 16).astype(np.float32),
                         np.array([0.0, 0.5, np.nextafter(np.float32(1), np.float32(0)), 1.0, 7.5,
                                   -0.25], np.float32)])
    want_u = np.clip(np.floor(xf.astype(np.float64) * 2.0 ** 32), 0, 2**32 - 1).astype(np.uint32)
    got = f.sample(torch.from_numpy(xf).cuda()).cpu().numpy()
    assert np.array_equal(got, ref.sample(want_u))


def test_concurrent_sampling_two_streams(rtf):
    """rtf.h: sampling is read-only on the forest, so calls on two streams may
    overlap; both give the oracle's indices."""
    p = power_law(1 << 20, "B")
    ref = oracle.build(p, 1 << 18)
    f = rtf.build(dev_f32(p), 1 << 18)
    torch.cuda.synchronize()
    xa, xb = philox_xi(1 << 22, seed=31), philox_xi(1 << 22, seed=32)
    da, db = dev_u32(xa), dev_u32(xb)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    oa = torch.empty_like(da)
    ob = torch.empty_like(db)
    for _ in range(3):
        with torch.cuda.stream(s1):
            f.sample(da, oa, stream=s1)
        with torch.cuda.stream(s2):
            f.sample(db, ob, stream=s2)
    torch.cuda.synchronize()
    assert np.array_equal(oa.cpu().numpy(), ref.sample(xa))
    assert np.array_equal(ob.cpu().numpy(), ref.sample(xb))


def test_rebuild_with_new_data(rtf):
    """One Forest object rebuilt with different distributions of its size:
    every build equals the oracle's (no state leaks between builds)."""
    rng = np.random.default_rng(41)
    n, m = 50000, 12345
    f = rtf.Forest(n, m)
    for t in range(6):
        p = random_small(rng, n, zero_frac=float(rng.choice([0, 0.5, 0.95])),
                         dyn=float(rng.choice([1, 10, 30])))
        f.build(dev_f32(p))
        assert_forest_equal(f, oracle.build(p, m), f"rebuild {t}")


def test_maximum_size(rtf):
    """n = 2^31 - 1, the largest n the leaf references allow (reading R3): the
    build completes, n' and T match the oracle's exact CDF (O1-O6), and 2^20
    samples equal the oracle's binary search over that CDF one by one."""
    n, m = (1 << 31) - 1, 1 << 24
    i = np.arange(n, dtype=np.int64)
    p = ((i % 1000) + 1).astype(np.float32)  # a sawtooth: no zeros, n' = n
    p[::7919] = 0.0                          # some zeros to compact
    del i
    K, T = oracle.cdf_all(p)
    xi = philox_xi(1 << 20, seed=77)
    want = oracle.sample_bsearch(K, xi)
    del K
    pd = torch.from_numpy(p).cuda()
    n_pos = int(np.count_nonzero(p))
    del p
    f = rtf.build(pd, m)
    h = f.header()
    assert f.last_status == 0
    assert h.n_pos == n_pos and h.total == T
    got = f.sample(dev_u32(xi)).cpu().numpy()
    assert np.array_equal(got, want)
    del f, pd
    torch.cuda.empty_cache()


def test_host_sampling_ragged_chunk_stays_in_staging(rtf):
    """rtf_sample_host with a chunk that is not a multiple of 4: the staging
    buffers hold exactly 2 * chunk entries (rtf.h) and nothing past them is
    written; indices still equal the oracle's."""
    p = env_map(256, 128, seed=11)
    m = p.size // 2
    ref = oracle.build(p, m)
    f = rtf.Forest(p.size, m).build(dev_f32(p))
    xi = philox_xi(100_003, seed=12)
    xi_host = torch.from_numpy(xi.view(np.int32)).pin_memory()
    out_host = torch.empty(xi.size, dtype=torch.int32).pin_memory()
    chunk = 1001
    guard = 64
    xi_big = torch.full((2 * chunk + guard,), 0x55AA55AA, dtype=torch.int32, device=DEV)
    out_big = torch.full((2 * chunk + guard,), 0x55AA55AA, dtype=torch.int32, device=DEV)
    rtf.sample_host(f, xi_host, out_host, xi_big[: 2 * chunk], out_big[: 2 * chunk])
    assert np.array_equal(out_host.numpy(), ref.sample(xi))
    assert bool((xi_big[2 * chunk:] == 0x55AA55AA).all()), "xi staging overrun"
    assert bool((out_big[2 * chunk:] == 0x55AA55AA).all()), "out staging overrun"
