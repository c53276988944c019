"""Pins of the CPU oracle against what the paper and the mathematics fix
(never against the oracle itself).  CPU only.

Pins used (DESIGN.md section 3 lists which pin covers which oracle step):
  * Fig. 6 worked example: cells, per-cell offsets, every TikZ
    edge, node enumeration, guide table            -> tests/golden/fig6.txt
  * Fig. 9 monotone histograms -> tests/golden/fig9_monotone.txt
  * xi = 0.5 lands in interval 3 (Fig. 2-5 captions P:107-109, P:123-125,
    P:164-166) on SPEC.md's (1,1,2,4) example
  * the paper's own Alg. 1, run bottom-up under random
    schedules (tests/alg1_sim.py), must give the oracle's topology
  * m = 1 gives a single radix tree (Alg. 1 caption P:1118-1119)
  * closed forms: floor properties of quantisation / fixed point, dyadic cases
  * brute force: the inverse-CDF definition P:61-63 evaluated in exact
    rational arithmetic on tiny inputs, for every boundary and a dense grid
  * stratified-set histogram closed form, chi-square, monotonicity
"""
from fractions import Fraction
import math
import random

import numpy as np
import pytest

import oracle
from workloads import (FIG6_WEIGHTS, SPEC_WEIGHTS, TEASER_WEIGHTS, hammersley_xi,
                       philox4x32_10, philox_xi, random_small, sine64, stratified_xi)
from tests.alg1_sim import alg1_forest

ONE = 1 << 63
F32 = np.float32


def xi_of(x: float) -> int:
    return int(x * 2**32)


# ---------------------------------------------------------------- Fig. 6

def test_fig6_cells_offsets_table(fig6):
    f = oracle.build(np.array(fig6["weights"], F32), fig6["m"])
    assert f.n_pos == 12
    assert f.cell.tolist() == fig6["cells"]
    # p1..p12 markers: number of leaves in cells < g+1
    offs = [int(np.sum(f.cell < g + 1)) for g in range(fig6["m"])]
    assert offs == fig6["offsets"]
    assert f.table.tolist() == fig6["table"]


def test_fig6_nodes_and_tikz_edges(fig6):
    f = oracle.build(np.array(fig6["weights"], F32), fig6["m"])
    for j, (c0, c1) in fig6["nodes"].items():
        assert (int(f.child0[j]), int(f.child1[j])) == (c0, c1), j
    # every TikZ edge is a parent-child relation of the oracle forest
    rel = set()
    for j in range(f.n_pos):
        for c in (int(f.child0[j]), int(f.child1[j])):
            rel.add((str(j), f"l{~c}" if c < 0 else str(c)))
    for e in fig6["edges"]:
        assert e in rel, e
    # and no drawn node has a child the figure lacks, except the anchors' left
    # children which the caption says are set manually
    anchors = {0, 4, 6, 7, 9, 10, 11}
    drawn = set(fig6["edges"])
    for (p, c) in rel:
        if (p, c) not in drawn:
            j = int(p)
            assert j in anchors and c == f"l{max(j - 1, 0)}", (p, c)


def test_fig6_keys_closed_form(fig6):
    # integer weights summing to 113: W = (0,5,6,9,11,17,23,30,36,64,66,80), key = floor(W 2^63/113)
    f = oracle.build(np.array(fig6["weights"], F32), fig6["m"])
    W = np.concatenate([[0], np.cumsum(fig6["weights"])[:-1]])
    assert [int(k) for k in f.key] == [(int(w) << 63) // 113 for w in W]


def test_fig6_alg1_every_schedule(fig6):
    f = oracle.build(np.array(fig6["weights"], F32), fig6["m"])
    keys = [int(k) for k in f.key]
    for seed in range(200):
        child, exch, other = alg1_forest(keys, fig6["m"], random.Random(seed))
        for j in range(12):
            got = tuple(~c[1] if c[0] == "leaf" else c[1] for c in child[j])
            assert got == fig6["nodes"][j]
        # paper-literal Alg.1 also exchanges at the C = 7 roots: 2(n'-C) + C = 17
        assert exch == 17


# ---------------------------------------------------------------- worked lookups

def test_spec_example_xi_half_is_interval_3():
    f = oracle.build(np.array(SPEC_WEIGHTS, F32), 4)
    assert [int(k) for k in f.key] == [0, 1 << 60, 1 << 61, 1 << 62]  # C = (0,.125,.25,.5)
    assert f.table.tolist() == [0, 2, 3, ~3]
    assert list(zip(f.child0.tolist(), f.child1.tolist())) == [(~0, 1), (~0, ~1), (~1, ~2), (~2, ~3)]
    out, loads = f.sample(np.array([xi_of(.8), xi_of(.3), xi_of(.15), xi_of(.5)], np.uint32), True)
    assert out.tolist() == [3, 2, 1, 3]
    assert loads.tolist() == [1, 2, 3, 2]


def test_teaser_config1():
    w = np.array(TEASER_WEIGHTS, F32)
    f = oracle.build(w, 8)
    assert f.cell.tolist() == [0, 0, 0, 2, 5, 5, 5, 5, 5, 6, 6, 6, 6, 6, 7, 7]
    assert f.table.tolist() == [0, ~2, 3, ~3, ~3, 4, 9, 14]
    x, _ = hammersley_xi(1024)
    out, loads = f.sample(x, True)
    # sum w = 64 is a power of two, so the 1024 stratified points split exactly 16 w
    assert np.bincount(out, minlength=16).tolist() == [16 * int(v) for v in TEASER_WEIGHTS]
    o, l = f.sample(np.array([1 << 31], np.uint32), True)
    assert o[0] == 3 and l[0] == 1  # xi = 0.5 -> interval 3 with a single table lookup


# ---------------------------------------------------------------- Fig. 9

@pytest.mark.parametrize("N", [512, 2048])
def test_fig9_monotone_histogram(fig9, N):
    f = oracle.build(sine64(), 64)
    c = np.bincount(f.sample(stratified_xi(N)), minlength=64)
    paper = np.array([round(fig9[N][i] * N) for i in range(64)])
    assert c.sum() == N == paper.sum()
    # The real CDF has exact ties with the stratified set: sum_{i<32} p_i = 31/64
    # and sum_{i<33} p_i = 33/64 (the cosine sum over a half period telescopes).
    # Those two points x = 31/64, 33/64 sit exactly on a boundary, where rounding
    # decides: the paper's float32 CDF put them in bins 31 and 33, the 63-bit
    # fixed point (reading R7) puts both in bin 32.  Every other point agrees.
    assert not np.array_equal(c, paper)
    ties = np.array([31 * N // 64, 33 * N // 64], np.uint32) * np.uint32(2**32 // N)
    assert f.sample(ties).tolist() == [32, 32]
    moved = paper.copy()
    moved[31] -= 1
    moved[33] -= 1
    moved[32] += 2
    assert c.tolist() == moved.tolist()


# ---------------------------------------------------------------- quantisation (O2, O3)

def test_quantize_dyadic_closed_form():
    # p = (1, 2, 3, 0.5): max 3 -> E = 1; n = 4 -> B = 62 - 2 = 60; w = p 2^59
    w, E, B = oracle.quantize([1, 2, 3, 0.5])
    assert (E, B) == (1, 60)
    assert [int(x) for x in w] == [1 << 59, 1 << 60, 3 << 59, 1 << 58]
    # n = 1 -> B = 62; single weight 0.75 -> E = -1 -> w = 0.75 2^63
    w, E, B = oracle.quantize([0.75])
    assert (E, B) == (-1, 62) and int(w[0]) == 3 << 61


def test_quantize_tiny_and_subnormal():
    tiny = np.float32(1e-45)  # smallest subnormal, 2^-149
    w, E, B = oracle.quantize(np.array([1.0, tiny, 0.0], F32))
    assert (E, B) == (0, 60)
    assert [int(x) for x in w] == [1 << 60, 1, 0]  # positive underflow clamps to 1 (R7)
    w, E, B = oracle.quantize(np.array([tiny, tiny * 2], F32))  # all subnormal
    assert (E, B) == (-148, 61)
    assert [int(x) for x in w] == [1 << 60, 1 << 61]


def test_quantize_floor_property_random():
    rng = np.random.default_rng(3)
    for _ in range(50):
        n = int(rng.integers(1, 300))
        p = random_small(rng, n, dyn=20.0)
        w, E, B = oracle.quantize(p)
        pmax = Fraction(float(p.max()))
        assert 2**E <= pmax < 2**(E + 1)
        assert B == 62 - math.ceil(math.log2(n)) if n > 1 else B == 62
        s = Fraction(2) ** (B - E)
        for pi, wi in zip(p.tolist(), w.tolist()):
            if pi == 0:
                assert wi == 0
            else:
                exact = Fraction(pi) * s
                assert wi == max(1, math.floor(exact))
        assert int(sum(int(x) for x in w)) < ONE  # T < 2^63


def test_errors():
    for bad in ([1.0, float("nan")], [1.0, -1.0], [float("inf"), 1.0], []):
        with pytest.raises(oracle.OracleError) as e:
            oracle.build(np.array(bad, F32), 4)
        assert e.value.status == oracle.EINVAL
    with pytest.raises(oracle.OracleError) as e:
        oracle.build(np.zeros(5, F32), 4)
    assert e.value.status == oracle.EALLZERO
    with pytest.raises(oracle.OracleError):
        oracle.build(np.ones(3, F32), 0)
    f = oracle.build(np.array([-0.0, 2.0], F32), 2)  # -0.0 is a zero weight
    assert f.n_pos == 1 and f.orig.tolist() == [1]


# ---------------------------------------------------------------- fixed point (O4-O8)

def _invariants(f: oracle.Forest, p: np.ndarray):
    w, _, _ = oracle.quantize(p)
    pos = np.flatnonzero(w > 0)
    assert f.orig.tolist() == pos.tolist()          # O4 compaction keeps order
    W = 0
    T = int(sum(int(x) for x in w))
    assert f.T == T
    for j, i in enumerate(pos.tolist()):
        k = int(f.key[j])
        assert k * T <= (W << 63) < (k + 1) * T      # key = floor(W 2^63 / T)
        assert int(f.cell[j]) == (k * f.m) >> 63    # cell = floor(key m / 2^63)
        W += int(w[i])
    assert int(f.key[0]) == 0 and np.all(np.diff(f.key.astype(object)) > 0)
    # lambda: 64 exactly at cell boundaries / end, else msb of the XOR
    for j in range(f.n_pos):
        if j + 1 == f.n_pos or f.cell[j] != f.cell[j + 1]:
            assert f.lam[j] == 64
        else:
            assert f.lam[j] == (int(f.key[j]) ^ int(f.key[j + 1])).bit_length() - 1


def _tree_invariants(f: oracle.Forest):
    """Structural facts of a radix forest (Sec.3.1-3.2): in-order leaves of each
    cell tree are its leaves in order; split levels strictly decrease root->leaf
    (so depth <= 64); every node slot written exactly once; k-1 internal nodes
    plus one anchor per cell with k leaves."""
    npos = f.n_pos
    seen_slots = np.zeros(npos, int)
    cells = {}
    for j in range(npos):
        cells.setdefault(int(f.cell[j]), []).append(j)

    def inorder(ref, lvl_above, out, depth):
        assert depth <= 64
        if ref < 0:
            out.append(~ref)
            return
        seen_slots[ref] += 1
        lam = int(f.lam[ref - 1])  # node ref splits between ref-1 and ref
        assert lam < lvl_above
        inorder(int(f.child0[ref]), lam, out, depth + 1)
        inorder(int(f.child1[ref]), lam, out, depth + 1)

    for g, leaves in cells.items():
        a = leaves[0]
        assert int(f.table[g]) == a
        seen_slots[a] += 1
        assert int(f.child0[a]) == ~int(f.orig[max(a - 1, 0)])
        got = []
        inorder(int(f.child1[a]), 65, got, 0)
        assert [int(f.orig[j]) for j in leaves] == got
    assert np.all(seen_slots == 1)
    for g in range(f.m):  # empty cells: the interval overlapping the cell
        if g not in cells:
            last = max(j for j in range(npos) if f.cell[j] < g)
            assert int(f.table[g]) == ~int(f.orig[last])


def test_invariants_random():
    rng = np.random.default_rng(11)
    for t in range(300):
        n = int(rng.integers(1, 80))
        m = int(rng.integers(1, 2 * n + 3))
        p = random_small(rng, n, zero_frac=0.25, dyn=float(rng.choice([0.5, 4, 12])))
        f = oracle.build(p, m)
        _invariants(f, p)
        _tree_invariants(f)


def test_alg1_random_cases_random_schedules():
    """Alg. 1 as printed (bottom-up, atomic exchange, random interleavings)
    gives exactly the oracle's per-cell top-down radix trees."""
    rng = np.random.default_rng(5)
    for t in range(300):
        n = int(rng.integers(1, 60))
        m = int(rng.integers(1, 2 * n + 3))
        f = oracle.build(random_small(rng, n, zero_frac=0.2, dyn=6.0), m)
        keys = [int(k) for k in f.key]
        child, exch, other = alg1_forest(keys, m, random.Random(t))
        C = len(set(f.cell.tolist()))
        assert exch == 2 * (f.n_pos - C) + C
        for j in range(f.n_pos):
            got = tuple(~int(f.orig[c[1]]) if c[0] == "leaf" else c[1] for c in child[j])
            assert got == (int(f.child0[j]), int(f.child1[j])), (t, j)


def test_m1_is_single_radix_tree():
    """Alg. 1 caption: omitting the coloured lines builds one
    radix tree; with m = 1 the forest is that tree."""
    rng = np.random.default_rng(9)
    for t in range(100):
        n = int(rng.integers(1, 70))
        f = oracle.build(random_small(rng, n), 1)
        keys = [int(k) for k in f.key]
        child, _, _ = alg1_forest(keys, 1, random.Random(t), forest=False)
        assert set(f.cell.tolist()) == {0}
        for j in range(f.n_pos):
            c1 = child[j][1]
            got = ~int(f.orig[c1[1]]) if c1[0] == "leaf" else c1[1]
            assert got == int(f.child1[j])
            if j > 0:
                c0 = child[j][0]
                assert (~int(f.orig[c0[1]]) if c0[0] == "leaf" else c0[1]) == int(f.child0[j])


# ---------------------------------------------------------------- sampling (O12)

def _definition_index(w, xi: int) -> int:
    """P^-1(x) = i <=> P_{i-1} <= x < P_i with P_i = floor(W_i 2^63/T)/2^63
    and x = xi/2^32, evaluated in exact integer arithmetic by a linear scan over
    ALL entries (zeros included): the last i with floor(W_i 2^63 / T) <= xi 2^31."""
    T = int(sum(int(v) for v in w))
    best, W = None, 0
    for i, wi in enumerate(int(v) for v in w):
        if wi > 0 and (W << 63) // T <= (xi << 31):
            best = i
        W += wi
    return best


def test_brute_force_inverse_cdf():
    rng = np.random.default_rng(21)
    for t in range(150):
        n = int(rng.integers(1, 40))
        m = int(rng.integers(1, 3 * n + 2))
        p = random_small(rng, n, zero_frac=0.3, dyn=float(rng.choice([1, 6, 16])))
        f = oracle.build(p, m)
        w, _, _ = oracle.quantize(p)
        # every boundary, its neighbours, cell boundaries and random points
        xs = set(rng.integers(0, 2**32, 200).tolist()) | {0, 2**32 - 1}
        for k in f.key.tolist():
            b = -(-int(k) >> 31)  # ceil(k / 2^31)
            xs |= {b - 1, b, b + 1}
        xs |= {(g << 32) // m for g in range(m)}
        xs = np.array(sorted(x for x in xs if 0 <= x < 2**32), np.uint32)
        got = f.sample(xs)
        for x, g in zip(xs.tolist(), got.tolist()):
            assert g == _definition_index(w, x), (t, x)
        assert np.all(np.diff(got) >= 0)           # monotone mapping (Sec.1)
        assert np.all(p[got] > 0)                  # zero weights never returned


def test_table2_fig6_hand_derived(fig6):
    """O13 on Fig. 6: cells 2, 6, 7, 8 hold exactly one leaf (6, 9, 10, 11; the
    figure's cell lines) and are overlapped by exactly two intervals
    (P:1335-1338): key32 = ceil(key_a / 2^31) with key_a = floor(W_a 2^63 / 113),
    ref = ~a (no zero weights: orig = index).  Cells 0, 1, 3 keep their anchor,
    the empty cells their leaf (the figure's table)."""
    f = oracle.build(np.array(fig6["weights"], F32), fig6["m"])
    W = np.concatenate([[0], np.cumsum(fig6["weights"])[:-1]]).tolist()
    per_cell = np.bincount(fig6["cells"], minlength=fig6["m"])
    want = []
    for g, t in enumerate(fig6["table"]):
        if t >= 0 and per_cell[g] == 1:
            key = (int(W[t]) << 63) // 113
            want.append((-(-key >> 31), ~t))
        else:
            want.append((0, t))
    assert sorted(g for g in range(12) if per_cell[g] == 1) == [2, 6, 7, 8]
    got = [(int(e["key32"]), int(e["ref"])) for e in f.table2()]
    assert got == want


def test_table2_special_cases():
    # a = 0 alone in cell 0: the whole cell is interval 0 -> (0, ~0)
    f = oracle.build(np.array([1.0, 1.0], F32), 2)
    assert [(int(e["key32"]), int(e["ref"])) for e in f.table2()] == [(0, ~0), (1 << 31, ~1)]
    # ceil(key_a / 2^31) = 2^32: no xi of cell 1 reaches interval 1 -> (0, ~0)
    f = oracle.build(np.array([1.0, 1e-30], F32), 2)
    assert int(f.key[1]) > (1 << 63) - (1 << 31)
    assert [(int(e["key32"]), int(e["ref"])) for e in f.table2()][1] == (0, ~0)
    assert f.sample(np.array([2**32 - 1], np.uint32)).tolist() == [0]
    # a zero weight between the two intervals: no flag, the anchor stays
    f = oracle.build(np.array([1.0, 0.0, 1.0], F32), 2)
    assert [(int(e["key32"]), int(e["ref"])) for e in f.table2()][1] == (0, 1)


def test_table2_descent_brute_force():
    """Alg. 2 through the O13 table reaches the inverse-CDF definition
    (exact integers) on every boundary, cell edge and random xi."""
    rng = np.random.default_rng(23)
    for t in range(80):
        n = int(rng.integers(1, 40))
        m = int(rng.integers(1, 3 * n + 2))
        p = random_small(rng, n, zero_frac=float(rng.choice([0.0, 0.3])), dyn=float(rng.choice([1, 6, 16])))
        f = oracle.build(p, m)
        w, _, _ = oracle.quantize(p)
        xs = set(rng.integers(0, 2**32, 64).tolist()) | {0, 2**32 - 1}
        for k in f.key.tolist():
            b = -(-int(k) >> 31)
            xs |= {b - 1, b, b + 1}
        xs |= {(g << 32) // m for g in range(m)} | {((g << 32) // m) - 1 for g in range(1, m)}
        xs = np.array(sorted(x for x in xs if 0 <= x < 2**32), np.uint32)
        got = f.sample_table2(xs)
        for x, g in zip(xs.tolist(), got.tolist()):
            assert g == _definition_index(w, x), (t, x)


def test_stratified_histogram_closed_form():
    """For a full stratified set of N = 2^k points, interval j receives
    ceil(N key_{j+1}/2^63) - ceil(N key_j/2^63) points (key_{n'} = 2^63)."""
    rng = np.random.default_rng(4)
    for t in range(40):
        n = int(rng.integers(1, 300))
        f = oracle.build(random_small(rng, n, dyn=5.0), int(rng.integers(1, 2 * n + 1)))
        N = 1 << int(rng.integers(4, 14))
        c = np.bincount(f.sample(stratified_xi(N)), minlength=n)
        ks = [int(k) for k in f.key] + [ONE]
        for j in range(f.n_pos):
            exp = -(-N * ks[j + 1] >> 63) - -(-N * ks[j] >> 63)
            assert c[int(f.orig[j])] == exp


def test_chi_square_philox():
    from scipy.stats import chisquare
    for fam_seed in range(3):
        rng = np.random.default_rng(100 + fam_seed)
        p = np.exp(2.0 * rng.standard_normal(64)).astype(F32)
        f = oracle.build(p, 32)
        w, _, _ = oracle.quantize(p)
        N = 1 << 18
        c = np.bincount(f.sample(philox_xi(N, seed=1234 + fam_seed)), minlength=64)
        expected = N * w.astype(np.float64) / float(sum(int(x) for x in w))
        assert chisquare(c, expected).pvalue > 1e-3


def test_bsearch_baseline_agrees_with_definition():
    rng = np.random.default_rng(8)
    for t in range(50):
        n = int(rng.integers(1, 50))
        p = random_small(rng, n, zero_frac=0.3)
        K, T = oracle.cdf_all(p)
        w, _, _ = oracle.quantize(p)
        xs = rng.integers(0, 2**32, 300, dtype=np.uint64).astype(np.uint32)
        got = oracle.sample_bsearch(K, xs)
        assert [_definition_index(w, int(x)) for x in xs] == got.tolist()


def test_rows_equal_independent_builds():
    rng = np.random.default_rng(12)
    rows, n_row, m_row = 7, 33, 17
    p = np.stack([random_small(rng, n_row) for _ in range(rows)])
    out = oracle.build_rows(p, rows, n_row, m_row)
    for r in range(rows):
        f = oracle.build(p[r], m_row)
        k = f.n_pos
        assert out["n_pos"][r] == k and out["T"][r] == f.T
        s = slice(r * n_row, r * n_row + k)
        assert np.array_equal(out["key"][s], f.key)
        assert np.array_equal(out["child0"][s], f.child0)
        assert np.array_equal(out["child1"][s], f.child1)
        assert np.array_equal(out["table"][r * m_row:(r + 1) * m_row], f.table)


# ---------------------------------------------------------------- input generator

def test_philox_known_answers():
    """Random123 known-answer vectors for philox4x32-10."""
    ctr = np.array([[0, 0, 0, 0], [0xFFFFFFFF] * 4,
                    [0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344]], np.uint32)
    keys = [0, 0xFFFFFFFFFFFFFFFF, 0x299F31D0A4093822]
    want = [[0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8],
            [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD],
            [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]]
    for c, k, wv in zip(ctr, keys, want):
        assert philox4x32_10(c[None, :], k)[0].tolist() == wv


def test_table3_hand_derived():
    """O16 (R20) on w = (2^20, 1, 2^20 - 1), m = 2^17: E = 20, B = 60, so the
    quantised weights are (2^60, 2^40, 2^60 - 2^40), T = 2^61 and the keys
    W 2^63 / T = 4 W are (0, 2^62, 2^62 + 2^42) -- cells key >> 46 = (0,
    65536, 65536).  Cell 65536 holds exactly the two leaves 1, 2: its first xi
    is 65536 2^15 = 2^31, ceil(key_1 / 2^31) = 2^31 (s1 = 0: interval 0 ends
    at the cell edge) and ceil(key_2 / 2^31) = 2^31 + 2^11 (s2 = 2048 = w_1 /
    T 2^32); entry (2048 << 16, orig(0) = 0).  Every other cell keeps O13."""
    p = np.array([2.0**20, 1.0, 2.0**20 - 1.0], F32)
    m = 1 << 17
    f = oracle.build(p, m)
    assert f.key.tolist() == [0, 1 << 62, (1 << 62) + (1 << 42)]
    t2, t3 = f.table2(), f.table3()
    diff = np.flatnonzero(t2.view(np.uint64) != t3.view(np.uint64)).tolist()
    assert diff == [65536]
    assert (int(t3[65536]["key32"]), int(t3[65536]["ref"])) == (2048 << 16, 0)
    xs = np.array([2**31 - 1, 2**31, 2**31 + 2047, 2**31 + 2048, 2**31 + 2**15 - 1], np.uint32)
    assert f.sample_table3(xs).tolist() == [0, 1, 1, 2, 2]
    w, _, _ = oracle.quantize(p)
    assert [_definition_index(w, int(x)) for x in xs] == [0, 1, 1, 2, 2]


def test_table3_not_packed():
    """No packing below m = 2^17 or for a non-power-of-two m (O16 = O13), for
    a = 0, or with a zero weight among the three intervals."""
    p = np.array([2.0**20, 1.0, 2.0**20 - 1.0], F32)
    for m in (1 << 16, (1 << 17) + 1):
        f = oracle.build(p, m)
        assert f.table3().tobytes() == f.table2().tobytes()
    f = oracle.build(np.array([1.0, 1.0, 2.0**30], F32), 1 << 17)  # leaves 0, 1 share cell 0
    assert f.table3().tobytes() == f.table2().tobytes()
    f = oracle.build(np.array([2.0**20, 0.0, 1.0, 2.0**20 - 1.0], F32), 1 << 17)
    assert f.table3().tobytes() == f.table2().tobytes()


def test_table3_descent_brute_force():
    """Alg. 2 through the O16 table equals the inverse-CDF definition (P:61-63,
    oracle.sample_bsearch over the exact fixed-point CDF) and the tree descent
    on every packed cell's boundaries +-1, its edges and random xi in it."""
    rng = np.random.default_rng(31)
    npack = 0
    for t, m in enumerate([1 << 17, 1 << 17, 1 << 18]):
        n = int(m * rng.uniform(0.7, 1.6))
        p = random_small(rng, n, zero_frac=float(rng.choice([0.0, 0.1])), dyn=float(rng.choice([2, 8])))
        f = oracle.build(p, m)
        t3 = f.table3()
        packed = np.flatnonzero((t3["ref"] >= 0) & (t3["key32"] != 0))
        npack += packed.size
        shift = 32 - (m.bit_length() - 1)
        xs = set()
        for g in packed[:: max(1, packed.size // 400)].tolist():
            x0, k = g << shift, int(t3[g]["key32"])
            for s in (k & 0xFFFF, k >> 16):
                xs |= {x0 + s - 1, x0 + s, x0 + s + 1}
            xs |= {x0, x0 + (1 << shift) - 1, x0 + int(rng.integers(1 << shift))}
        xs = np.array(sorted(x for x in xs if 0 <= x < 2**32), np.uint32)
        K, _ = oracle.cdf_all(p)
        want = oracle.sample_bsearch(K, xs)
        assert np.array_equal(f.sample_table3(xs), want), t
        assert np.array_equal(f.sample(xs), want), t
    assert npack > 1000  # the inputs do exercise the packed cells


# ---------------------------------------------------------------- O17 (reading R21): fallback

def test_table4_geometric_chain_hand_derived():
    """O17 on p_i = 2^-i (i < 20), m = 1: every split level is below the one
    before it (the keys halve their distance to the top), so Alg. 1 builds a
    chain -- the deepest leaf 19 sits under 19 internal nodes, 20 visits with
    the anchor -- while bisection of the 21 intervals needs ceil(log2 21) = 5:
    20 > 5 + 4, so the cell is marked (3 << 30 | 20, anchor 0), every xi is
    answered in at most 5 reads, and the answers are the definition's."""
    L = 20
    p = np.exp2(-np.arange(L, dtype=np.float64)).astype(F32)
    f = oracle.build(p, 1)
    assert np.all(np.diff(f.lam[:-1].astype(np.int64)) < 0)  # a strictly falling chain
    D, k = f.cell_depths()
    assert (int(D[0]), int(k[0])) == (L, L)
    assert oracle.bisect_visits(L) == 5
    t4 = f.table4()
    assert (int(t4[0]["key32"]), int(t4[0]["ref"])) == ((3 << 30) | L, 0)
    w, _, _ = oracle.quantize(p)
    xs = {0, 2**32 - 1}
    for key in f.key.tolist():
        b = -(-int(key) >> 31)
        xs |= {b - 1, b, b + 1}
    xs = np.array(sorted(x for x in xs if 0 <= x < 2**32), np.uint32)
    got, visits = f.sample_table4(xs, with_loads=True)
    assert [int(g) for g in got] == [_definition_index(w, int(x)) for x in xs]
    assert int(visits.max()) <= 5


def test_table4_balanced_not_marked():
    """Equal weights (n = 1024, m = 1): keys j 2^53, a perfect radix tree of
    10 internal levels -- 11 visits with the anchor, exactly the bisection's
    ceil(log2 1025) = 11 -- so nothing is marked (O17 = O16)."""
    f = oracle.build(np.ones(1024, F32), 1)
    D, k = f.cell_depths()
    assert (int(D[0]), int(k[0])) == (11, 1024)
    assert oracle.bisect_visits(1024) == 11
    assert f.table4().tobytes() == f.table3().tobytes()


def test_cell_depths_brute_force():
    """D_g from the reachable leaves equals the most visits over EVERY 32-bit
    xi of the cell (m = 2^20: cells of 4096 xi, enumerated)."""
    rng = np.random.default_rng(41)
    m = 1 << 20
    p = np.concatenate([np.exp2(-np.arange(30, dtype=np.float64)) * 1e-3,
                        random_small(rng, 3000, zero_frac=0.2, dyn=30.0)]).astype(F32)
    f = oracle.build(p, m)
    D, _ = f.cell_depths()
    cells = np.unique(f.cell)[:40].tolist() + np.flatnonzero(D == D.max())[:3].tolist()
    for g in cells:
        xs = np.arange(g << 12, (g + 1) << 12, dtype=np.uint64).astype(np.uint32)
        _, loads = f.sample(xs, with_loads=True)
        assert int(loads.max()) - 1 == int(D[g]), g


def test_table4_descent_brute_force():
    """Alg. 2 through the O17 table equals the inverse-CDF definition on
    distributions with degenerate cells (geometric runs) and ordinary ones;
    a marked cell never reads more than ceil(log2(k + 1)) records."""
    rng = np.random.default_rng(43)
    marked = 0
    for t in range(24):
        parts = []
        for _ in range(int(rng.integers(1, 4))):
            if rng.random() < 0.6:
                L = int(rng.integers(8, 40))
                parts.append(np.exp2(-np.arange(L, dtype=np.float64) * rng.uniform(0.7, 1.5))
                             * rng.uniform(1e-6, 1.0))
            else:
                parts.append(random_small(rng, int(rng.integers(1, 60)), zero_frac=0.2, dyn=8.0))
        p = np.concatenate(parts).astype(F32)
        if not np.any(p > 0):
            continue
        m = int(rng.choice([1, 2, 3, 7, 64]))
        f = oracle.build(p, m)
        w, _, _ = oracle.quantize(p)
        t4 = f.table4()
        mk = np.flatnonzero(oracle.is_bisect(t4))
        marked += mk.size
        xs = set(rng.integers(0, 2**32, 64).tolist()) | {0, 2**32 - 1}
        for key in f.key.tolist():
            b = -(-int(key) >> 31)
            xs |= {b - 1, b, b + 1}
        xs = np.array(sorted(x for x in xs if 0 <= x < 2**32), np.uint32)
        got, visits = f.sample_table4(xs, with_loads=True)
        for x, g in zip(xs.tolist(), got.tolist()):
            assert g == _definition_index(w, x), (t, x)
        cells = (xs.astype(np.uint64) * np.uint64(m)) >> np.uint64(32)
        for g in mk.tolist():
            sel = cells == g
            if np.any(sel):
                assert int(visits[sel].max()) <= oracle.bisect_visits(int(t4[g]["key32"]) & 0x3FFFFFFF)
    assert marked > 5


def test_table4_marks_never_collide_with_packed():
    """An O16 packed entry can carry bit 31 but never both top bits: p = (2^46,
    2^46 - 2^30, 2^30, 2^63 - 2^47) gives E = 62, B = 60, w = p / 4, T = 2^61
    and keys 4 W = (0, 2^46, 2^47 - 2^30, 2^47); with m = 2^17 (cells key >>
    46) cell 1 holds leaves 1, 2 and starts at xi0 = 2^15: s1 = 2^15 - xi0 =
    0, s2 = ceil(2^16 - 1/2) - xi0 = 2^15 -- entry (2^31, orig(0) = 0).  O17's
    marks are 3 << 30 | k, so this entry is no mark, and through the O17 table
    cell 1 still answers as O16 and the definition do."""
    p = np.array([2.0**46, 2.0**46 - 2.0**30, 2.0**30, 2.0**63 - 2.0**47], F32)
    f = oracle.build(p, 1 << 17)
    assert f.key.tolist() == [0, 1 << 46, (1 << 47) - (1 << 30), 1 << 47]
    t3, t4 = f.table3(), f.table4()
    assert (int(t3[1]["key32"]), int(t3[1]["ref"])) == (1 << 31, 0)
    assert not np.any(oracle.is_bisect(t4))
    xs = np.array([1 << 15, (1 << 16) - 2, (1 << 16) - 1], np.uint32)
    w, _, _ = oracle.quantize(p)
    want = [_definition_index(w, int(x)) for x in xs]
    assert want == [1, 1, 1]
    assert f.sample_table3(xs).tolist() == want
    assert f.sample_table4(xs).tolist() == want
