"""Test helpers: the reference's seeded instance generators (tests/support/synthetic.hpp)
restated over the same SplitMix64 stream, so the cases are the reference's own."""
from __future__ import annotations

import numpy as np

from paper_2307_04904_b200.generators import SplitMix64


class ScalarRng:
    """Scalar view of SplitMix64 (rng.hpp:10-29) for small generators."""

    def __init__(self, seed: int):
        self.r = SplitMix64(seed)

    def next_below(self, n: int) -> int:
        return int(self.r.next_below(n, 1)[0])

    def next_double(self) -> float:
        return float(self.r.next_double(1)[0])


def random_int_series(rng: ScalarRng, max_length: int, low: int, high: int) -> np.ndarray:
    """synthetic.hpp:22-29."""
    length = 1 + rng.next_below(max_length)
    span = high - low + 1
    return np.array([float(low + rng.next_below(span)) for _ in range(length)])


def random_walk_series(rng: ScalarRng, length: int, start: float = 0.0) -> np.ndarray:
    """synthetic.hpp:32-41."""
    out = np.empty(length)
    level = start
    for t in range(length):
        level += rng.next_double() * 2.0 - 1.0
        out[t] = level
    return out


def blob_series(rng: ScalarRng, length: int, level: float, jitter: float) -> np.ndarray:
    """synthetic.hpp:44-49."""
    return np.array([level + (rng.next_double() * 2.0 - 1.0) * jitter for _ in range(length)])


def random_condensed(rng: ScalarRng, p: int, low: float = 0.1, high: float = 10.0) -> np.ndarray:
    """synthetic.hpp:52-57 (random_distance_matrix)."""
    return np.array([low + rng.next_double() * (high - low) for _ in range(p * (p - 1) // 2)])


def pack(rows):
    lens = np.array([len(r) for r in rows], dtype=np.int64)
    offsets = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(lens, out=offsets[1:])
    samples = np.concatenate([np.asarray(r, dtype=np.float64) for r in rows]) if rows else \
        np.zeros(0)
    return np.ascontiguousarray(samples), offsets


def bits(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def assert_bitwise(a, b, what=""):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    bad = np.nonzero(bits(a) != bits(b))[0]
    assert bad.size == 0, f"{what}: {bad.size} mismatches, first at {bad[:5]}: {a[bad[:5]]} vs {b[bad[:5]]}"
