"""Pins of the 2-D oracle (O14 marginal weights, O15 component-wise sampling with
the sub-pixel rescale; Sec.6, readings R15/R19).  CPU only."""
from fractions import Fraction

import numpy as np

import oracle
from workloads import random_small


def _rz_u32_over_2_32(x: int) -> np.float32:
    """float32(x / 2^32) rounded toward zero, by truncating x to its top 24
    significant bits (then the quotient is exact in float32)."""
    if x == 0:
        return np.float32(0.0)
    drop = max(0, x.bit_length() - 24)
    return np.float32((x >> drop << drop) / 2.0 ** 32)


def _definition_index(w, xi: int) -> int:
    T = int(sum(int(v) for v in w))
    best, W = None, 0
    for i, wi in enumerate(int(v) for v in w):
        if wi > 0 and (W << 63) // T <= (xi << 31):
            best = i
        W += wi
    return best


def test_2d_constant_image_is_the_identity():
    """A constant W x H image (powers of two) maps (xi1, xi2) to the pixel
    (floor(xi1 H / 2^32), floor(xi2 W / 2^32)) and the position (xi2, xi1) / 2^32
    exactly: every key is a multiple of 2^63 / H or 2^63 / W."""
    rng = np.random.default_rng(5)
    for H, W in ((1, 1), (4, 8), (16, 2)):
        f = oracle.build_2d(np.full((H, W), 0.37, np.float32), W, H)
        xs1 = np.concatenate([[0, 2**32 - 1, 2**31], rng.integers(0, 2**32, 40)]).astype(np.uint32)
        xs2 = np.concatenate([[2**32 - 1, 0, 2**30], rng.integers(0, 2**32, 40)]).astype(np.uint32)
        pix, pos = f.sample(xs1, xs2)
        for k in range(xs1.size):
            a, b = int(xs1[k]), int(xs2[k])
            assert pix[k] == (a * H >> 32) * W + (b * W >> 32)
            assert pos[k, 0] == _rz_u32_over_2_32(b) and pos[k, 1] == _rz_u32_over_2_32(a)


def test_2d_marginal_weights_are_row_sums():
    """Small integer images: every quantisation step is exact, so the row
    weights are the row sums up to one common power of two."""
    rng = np.random.default_rng(6)
    for _ in range(20):
        H, W = int(rng.integers(1, 7)), int(rng.integers(1, 9))
        p = rng.integers(0, 9, (H, W)).astype(np.float32)
        p[rng.integers(H), rng.integers(W)] = 5.0
        q = oracle.marginal_weights(p)
        S = p.sum(axis=1).astype(np.int64)
        top = int(np.argmax(S))
        for y in range(H):
            assert Fraction(float(q[y])) / Fraction(float(q[top])) == Fraction(int(S[y]), int(S[top]))


def test_2d_brute_force_components():
    """Tiny random images with zeros: y is the inverse CDF of the quantised
    row weights, x the inverse CDF of row y's quantised weights; the
    position lies in pixel (x, y) and is monotone in xi1 along a column."""
    rng = np.random.default_rng(7)
    for t in range(40):
        H, W = int(rng.integers(1, 6)), int(rng.integers(1, 9))
        p = np.stack([random_small(rng, W, zero_frac=0.3) for _ in range(H)])
        if t % 5 == 0:
            p[int(rng.integers(H))] = 0.0  # an all-zero row is never chosen
            if not np.any(p > 0):
                p[0, 0] = 1.0
        f = oracle.build_2d(p, int(rng.integers(1, 2 * W + 2)), int(rng.integers(1, 2 * H + 2)))
        wq, _, _ = oracle.quantize(oracle.marginal_weights(p))
        xs1 = np.sort(rng.integers(0, 2**32, 30)).astype(np.uint32)
        xs2 = np.full(30, int(rng.integers(0, 2**32)), np.uint32)
        pix, pos = f.sample(xs1, xs2)
        for k in range(30):
            y, x = divmod(int(pix[k]), W)
            assert y == _definition_index(wq, int(xs1[k]))
            wr, _, _ = oracle.quantize(p[y])
            assert x == _definition_index(wr, int(xs2[k]))
            assert x / W - 2.0 ** -23 <= pos[k, 0] < (x + 1) / W
            assert y / H - 2.0 ** -23 <= pos[k, 1] < (y + 1) / H
        assert np.all(np.diff(pos[:, 1]) >= 0)
