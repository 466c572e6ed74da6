"""Synthetic inputs with the reference's own generator, vectorised.

SplitMix64 (proj/include/lseforge/rng.hpp:13-60) draws in make_instance's
order (proj/tests/support.hpp:27-37): ref-E [n x d] = U(-half, half) first,
then ref-C [d x v], then targets = bounded(v) — so the bench times exactly
the instance the reference library would build from the same seed
(SURVEY.md 8(d)).  The k-th draw of SplitMix64(seed) is mix(seed + k * golden),
so every block of draws is one numpy expression; bounded() rejections are
resolved by keeping the accepted candidates of the stream in order.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def mix(z: np.ndarray) -> np.ndarray:
    """SplitMix64::mix (rng.hpp:52-56), elementwise on uint64."""
    z = (z ^ (z >> np.uint64(30))) * M1
    z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def draws(seed: int, first: int, count: int) -> np.ndarray:
    """next() outputs first+1 .. first+count of SplitMix64(seed) (uint64)."""
    with np.errstate(over="ignore"):
        k = np.arange(first + 1, first + count + 1, dtype=np.uint64)
        return mix(np.uint64(seed) + k * GOLDEN)


def derived_seed(seed: int, index: int) -> int:
    """SplitMix64(seed).derived(index).seed() (rng.hpp:46-48)."""
    with np.errstate(over="ignore"):
        return int(mix(np.uint64(seed) + GOLDEN * np.uint64(index + 1)))


def symmetric_uniform(seed: int, first: int, count: int, half_width: float = 1.0,
                      chunk: int = 1 << 23) -> np.ndarray:
    """float((2 * uniform() - 1) * half_width) for `count` draws (support.hpp:22-24)."""
    out = np.empty(count, np.float32)
    for a in range(0, count, chunk):
        b = min(count, a + chunk)
        u = (draws(seed, first + a, b - a) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        out[a:b] = ((2.0 * u - 1.0) * half_width).astype(np.float32)
    return out


def bounded(seed: int, first: int, n: int, bound: int):
    """n successive bounded(bound) results from draw `first` on (rng.hpp:23-38);
    returns (values int64, draws consumed)."""
    mask = bound - 1
    for s in (1, 2, 4, 8, 16, 32):
        mask |= mask >> s
    out = np.empty(0, np.int64)
    pos = first
    while out.size < n:
        want = max(1024, 2 * (n - out.size) * (mask + 1) // bound + 64)
        cand = draws(seed, pos, want) & np.uint64(mask)
        ok = np.nonzero(cand < np.uint64(bound))[0]
        take = ok[: n - out.size]
        out = np.concatenate([out, cand[take].astype(np.int64)])
        pos += int(take[-1]) + 1 if out.size == n and take.size else want
    return out, pos - first


def make_instance(seed: int, n: int, d: int, v: int, half_width: float = 1.0):
    """(ref-E [n x d] float32, ref-C [d x v] float32, targets [n] int64)."""
    E = symmetric_uniform(seed, 0, n * d, half_width).reshape(n, d)
    Cm = symmetric_uniform(seed, n * d, d * v, half_width).reshape(d, v)
    t, _ = bounded(seed, n * d + d * v, n, v)
    return E, Cm, t
