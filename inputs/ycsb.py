"""YCSB input generators (seeded, synthetic).  See inputs/__init__.py for the contract.

Shapes follow PAPER.md:457-458 (YCSB, 2^20*10 rows, 16 single-tuple accesses per
transaction) and BASELINE.json configs[0..1].  Row payload: 16 x u64 = 128 B
(SURVEY.md §8(c) reading Z11: word j of row k starts as mix64(seed ^ (16k+j)) for
j < 15, word 15 is a write counter starting at 0).
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def mix64(z):
    """splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + _G
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def ycsb_rows(seed: int, n_rows: int, first: int = 0) -> np.ndarray:
    """Rows [first, first+n_rows) of the YCSB table S0 as an (n, 16) uint64 array."""
    k = np.arange(first, first + n_rows, dtype=np.uint64)[:, None]
    j = np.arange(16, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        x = np.uint64(seed & MASK64) ^ (k * np.uint64(16) + j)
    rows = mix64(x)
    rows[:, 15] = 0
    return np.ascontiguousarray(rows)


def ycsb_row(seed: int, k: int) -> np.ndarray:
    return ycsb_rows(seed, 1, k)[0]


def zipf_thresholds(n: int, theta: float) -> np.ndarray:
    """u64 thresholds T[r-1] = floor(2^64 * P(rank <= r)) for P(rank=r) ∝ r^-theta.

    A sampler draws a uniform u64 ``u`` and returns rank = min(#{j: T[j] <= u}, n-1) + 1.
    The last threshold (and any that round to 1.0) is 2^64-1.
    """
    if n < 1:
        raise ValueError("n must be >= 1")
    w = np.arange(1, n + 1, dtype=np.float64) ** (-float(theta))
    c = np.cumsum(w)
    cdf = c / c[-1]
    t = np.floor(cdf * 2.0 ** 64)
    out = np.empty(n, dtype=np.uint64)
    full = t >= 2.0 ** 64
    out[~full] = t[~full].astype(np.uint64)
    out[full] = np.uint64(MASK64)
    out[-1] = np.uint64(MASK64)
    return out


def harmonic(n: int, theta: float) -> float:
    """Generalised harmonic number H(n, theta) via the Hurwitz zeta closed form
    (independent of the cumulative sum used by zipf_thresholds)."""
    import mpmath
    if theta == 0:
        return float(n)
    if abs(theta - 1.0) < 1e-12:
        return float(mpmath.digamma(n + 1) + mpmath.euler)
    # H(n,θ) = ζ(θ, 1) - ζ(θ, n+1) (Hurwitz zeta, analytic continuation for θ != 1).
    return float(mpmath.zeta(theta, 1) - mpmath.zeta(theta, n + 1))


def scramble_mult(n: int) -> int:
    """Fixed odd multiplier coprime with n: key = ((rank-1) * A) mod n is a bijection
    on [0, n) (reading Z13: hot ranks land on distant rows)."""
    from math import gcd
    a = 0x9E3779B1
    while gcd(a, n) != 1:
        a += 2
    return a % n if n > 1 else 0


def random_batch(seed: int, n_txn: int, k: int, n_rows: int, w: float,
                 hot: int | None = None):
    """A small arbitrary batch for brute-force tests: distinct sorted keys per
    transaction, Bernoulli(w) writes, field in [0,15).  ``hot`` restricts keys to
    [0, hot) to force conflicts.  Returns (keys u32[n_txn*k], ops u8[n_txn*k]) where
    op bit7 = write and bits 0..3 = field."""
    rng = np.random.default_rng(seed)
    span = n_rows if hot is None else min(hot, n_rows)
    if span < k:
        raise ValueError("need at least k distinct rows")
    keys = np.empty((n_txn, k), dtype=np.uint32)
    for t in range(n_txn):
        keys[t] = np.sort(rng.choice(span, size=k, replace=False))
    wr = rng.random((n_txn, k)) < w
    field = rng.integers(0, 15, size=(n_txn, k))
    ops = (field | (wr.astype(np.int64) << 7)).astype(np.uint8)
    return keys.reshape(-1), ops.reshape(-1)
