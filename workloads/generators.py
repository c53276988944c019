"""Input generators (see package docstring).  DESIGN.md section 4 states each
recipe; the paper passage each workload imitates is cited per function."""
from __future__ import annotations

import numpy as np

__all__ = [
    "FIG6_WEIGHTS", "SPEC_WEIGHTS", "TEASER_WEIGHTS", "sine64", "env_map", "power_law",
    "spikes", "rows_lognormal", "random_small", "stratified_xi", "sobol0_xi",
    "radical_inverse2", "hammersley_xi", "philox4x32_10", "philox_xi", "WORKLOADS",
]

# Fig. 6: weights recovered from the bar coordinates x 113
# (P:1247-1258); they match the generator at P:1126 (first 7 <= ceil(0.12*64)).
FIG6_WEIGHTS = (5, 1, 3, 2, 6, 6, 7, 6, 28, 2, 14, 33)
# SPEC.md's worked example: C = (0, .125, .25, .5, 1).
SPEC_WEIGHTS = (1, 1, 2, 4)
# Config 1 (teaser, Fig. 1): the paper does not give its distribution;
# this n=16 one (sum 64) is invented.
TEASER_WEIGHTS = (2, 4, 10, 24, 3, 1, 1, 2, 1, 1, 1, 2, 3, 1, 4, 4)


def sine64() -> np.ndarray:
    """Fig. 9's 1-D target density: p_i = (1 - cos(2 pi i / 64)) / 64,
    i = 0..63 (p_0 = 0).  Computed in float64, rounded to float32."""
    i = np.arange(64, dtype=np.float64)
    return ((1.0 - np.cos(2.0 * np.pi * i / 64.0)) / 64.0).astype(np.float32)


def env_map(width: int = 2048, height: int = 1024, seed: int = 1) -> np.ndarray:
    """Synthetic lat-long HDR environment-map luminance (config 2; the paper's
    env-map use case P:1562-1567, Fig. 5, whose image is proprietary).
    Sky 1 + 2 cos(theta) for theta < pi/2; ground 0.2 exp(N(0,1)) with 5 % exact
    zeros; a sun 5e4 exp(-d^2 / (2 * 0.01^2)) at (theta, phi) = (0.6, 2.0); all
    times sin(theta) (solid-angle weight).  Row-major, n = width * height."""
    rng = np.random.default_rng(seed)
    theta = (np.arange(height, dtype=np.float64) + 0.5) / height * np.pi
    phi = (np.arange(width, dtype=np.float64) + 0.5) / width * 2.0 * np.pi
    th, ph = np.meshgrid(theta, phi, indexing="ij")
    sky = 1.0 + 2.0 * np.cos(th)
    ground = 0.2 * np.exp(rng.standard_normal(th.shape))
    ground[rng.random(th.shape) < 0.05] = 0.0
    lum = np.where(th < np.pi / 2, sky, ground)
    # great-circle distance to the sun
    ts, ps = 0.6, 2.0
    cosd = np.sin(th) * np.sin(ts) * np.cos(ph - ps) + np.cos(th) * np.cos(ts)
    d = np.arccos(np.clip(cosd, -1.0, 1.0))
    lum = lum + 5e4 * np.exp(-d * d / (2 * 0.01 ** 2))
    return (lum * np.sin(th)).astype(np.float32).reshape(-1)


def power_law(n: int, family: str = "A") -> np.ndarray:
    """Config 3 / Table 1 families, normalised in
    float64 then rounded to float32 (tiny entries underflow to 0, as the paper's
    own families do in float32):
      A: ((i+1)/n)^20          (p_i ~ i^20)
      B: (i mod 32 + 1)^25
      C: (i mod 64 + 1)^35
      D: 2^(-64 i / n)          (exponentially skewed)
    """
    i = np.arange(n, dtype=np.float64)
    if family == "A":
        x = np.exp(20.0 * np.log((i + 1.0) / n))
    elif family == "B":
        x = np.exp(25.0 * np.log(i % 32 + 1.0) - 25.0 * np.log(32.0))
    elif family == "C":
        x = np.exp(35.0 * np.log(i % 64 + 1.0) - 35.0 * np.log(64.0))
    elif family == "D":
        x = np.exp2(-64.0 * i / n)
    else:
        raise ValueError(family)
    return (x / x.sum()).astype(np.float32)


def spikes(n: int, n_spikes: int = 4, spike_mass: float = 0.24) -> np.ndarray:
    """Config 4 / Table 1 "4 spikes" (masses unstated in the paper):
    spikes at (2k+1) n / (2 n_spikes) with mass 0.24 each, uniform background
    carrying the remaining 0.04."""
    bg = (1.0 - n_spikes * spike_mass) / (n - n_spikes)
    p = np.full(n, bg, dtype=np.float64)
    for k in range(n_spikes):
        p[(2 * k + 1) * n // (2 * n_spikes)] = spike_mass
    return p.astype(np.float32)


def rows_lognormal(rows: int, n_row: int, seed: int = 7) -> np.ndarray:
    """Config 5 (batched rebuilds, Sec.5): p = exp(3 N(0,1)) per
    entry; every 16th row is a "4 spikes" row.  Shape (rows, n_row)."""
    rng = np.random.default_rng(seed)
    p = np.exp(3.0 * rng.standard_normal((rows, n_row)))
    if n_row >= 8:
        sp = spikes(n_row).astype(np.float64)
        p[::16] = sp
    return p.astype(np.float32)


def random_small(rng: np.random.Generator, n: int, zero_frac: float = 0.2,
                 dyn: float = 8.0) -> np.ndarray:
    """Random small test vectors with a high dynamic range and exact zeros."""
    # clip keeps every value finite and representable in float32 (tiny ones subnormal)
    p = np.exp(np.clip(dyn * rng.standard_normal(n), -100.0, 80.0))
    p[rng.random(n) < zero_frac] = 0.0
    if not np.any(p > 0):
        p[rng.integers(n)] = 1.0
    return p.astype(np.float32)


# ---------------- xi sequences (u32 fixed point xi / 2^32) ----------------

def stratified_xi(N: int) -> np.ndarray:
    """xi_k = k / N (Fig. 9's monotone experiment), N a power of two <= 2^32."""
    assert N & (N - 1) == 0
    return (np.arange(N, dtype=np.uint64) * (np.uint64(1 << 32) // np.uint64(N))).astype(np.uint32)


def _bitreverse32(k: np.ndarray) -> np.ndarray:
    x = k.astype(np.uint32)
    x = ((x >> 1) & 0x55555555) | ((x & 0x55555555) << 1)
    x = ((x >> 2) & 0x33333333) | ((x & 0x33333333) << 2)
    x = ((x >> 4) & 0x0F0F0F0F) | ((x & 0x0F0F0F0F) << 4)
    x = ((x >> 8) & 0x00FF00FF) | ((x & 0x00FF00FF) << 8)
    x = (x >> 16) | (x << 16)
    return x.astype(np.uint32)


def sobol0_xi(N: int, start: int = 0) -> np.ndarray:
    """Sobol' dimension 0 = van der Corput base 2 = bit-reversed index."""
    return _bitreverse32(np.arange(start, start + N, dtype=np.uint64))


def radical_inverse2(k: np.ndarray) -> np.ndarray:
    return _bitreverse32(k)


def hammersley_xi(N: int):
    """2-D Hammersley set (Fig. 1): (k/N, radical_inverse_2(k))."""
    return stratified_xi(N), radical_inverse2(np.arange(N, dtype=np.uint64))


_M0, _M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_W0, _W1 = 0x9E3779B9, 0xBB67AE85
_MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(counters: np.ndarray, key: int) -> np.ndarray:
    """Philox4x32-10 (Salmon et al. 2011, Random123): counters uint32[B,4],
    key = 64-bit -> uint32[B,4].  Counter-based, so the CUDA input generator
    (rtf_philox_u32) implements the identical function independently."""
    c = [counters[:, i].astype(np.uint64) for i in range(4)]
    k0, k1 = key & 0xFFFFFFFF, (key >> 32) & 0xFFFFFFFF
    for r in range(10):
        if r:
            k0, k1 = (k0 + _W0) & 0xFFFFFFFF, (k1 + _W1) & 0xFFFFFFFF
        p0 = _M0 * c[0]
        p1 = _M1 * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK
        c = [hi1 ^ c[1] ^ np.uint64(k0), lo1, hi0 ^ c[3] ^ np.uint64(k1), lo0]
    return np.stack([x.astype(np.uint32) for x in c], axis=1)


def philox_xi(N: int, seed: int = 0x5EED, start: int = 0) -> np.ndarray:
    """xi_k for k in [start, start+N): block b = k // 4 uses counter
    (b mod 2^32, b >> 32, 0, 0) and key = seed; xi_k is word k mod 4."""
    b0, b1 = start // 4, (start + N + 3) // 4
    b = np.arange(b0, b1, dtype=np.uint64)
    ctr = np.zeros((b.size, 4), dtype=np.uint32)
    ctr[:, 0] = (b & _MASK).astype(np.uint32)
    ctr[:, 1] = (b >> np.uint64(32)).astype(np.uint32)
    out = philox4x32_10(ctr, seed).reshape(-1)
    off = start - 4 * b0
    return np.ascontiguousarray(out[off: off + N])


# Named workloads (BASELINE.json configs).
WORKLOADS = {
    "c1_teaser": dict(n=16, m=8, samples=1024),
    "c2_envmap": dict(n=2048 * 1024, m=2048 * 1024, samples=1 << 26),
    "c3_powerlaw": dict(n=1 << 24, m=1 << 22, samples=1 << 30),
    "c4_spikes": dict(n=1 << 28, m=1 << 26, samples=1 << 32),
    "c5_rows": dict(rows=65536, n_row=1024, m_row=1024),
}
