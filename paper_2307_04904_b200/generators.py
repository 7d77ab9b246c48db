"""Seeded synthetic series generators for the five BASELINE.json configurations.

The paper measures on the UCR archive, which is not available here;
these seeded generators stand in for it with the shapes, lengths and value
distributions BASELINE.json names. Both the CUDA path and the
CPU reference consume the *same* arrays, so any platform difference in numpy's
transcendental functions cannot break parity.

RNG: the reference's SplitMix64 (rng.hpp:10-33) with seed ``2307049040 + c``.
SplitMix64's k-th output depends only on ``seed + k * golden``, so it vectorises
exactly in numpy. Gaussians: Box-Muller, ``sqrt(-2 ln(1-u1)) * cos(2 pi u2)``, one
draw per two consecutive uniforms. z-normalisation follows runner.hpp:82-95
(sequential sums, population std, constant series -> zeros).

Draw order per config (documented so it can be reproduced elsewhere):
  c1  per class (4): 3 x (f=1+9u, phi=2*pi*u); per series: shift U{-50..50};
      then all noise N(0, 0.1^2), series-major.
  c2  all N(0,1) steps, series-major; walk = running sum from 0.
  c3  per class (24): knot positions (two distinct U{1..44}, sorted), then 4 knot
      values N(0,1); per series: shift U{-3..3}; then all noise N(0, 0.2^2).
  c4  as c2 with L=2844.
  c5  per series: length U{50..1500}; per class (10): 3 x (f, phi); then noise
      N(0, 0.15^2) series-major over the ragged lengths.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

MASK64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
BASE_SEED = 2307049040


class SplitMix64:
    """rng.hpp:10-33, vectorised: output k is mix(seed + k*golden)."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next_u64(self, count: int) -> np.ndarray:
        k = np.arange(1, count + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            z = np.uint64(self.state) + k * np.uint64(_GOLDEN)
            z = (z ^ (z >> np.uint64(30))) * _M1
            z = (z ^ (z >> np.uint64(27))) * _M2
            z = z ^ (z >> np.uint64(31))
        self.state = (self.state + count * _GOLDEN) & MASK64
        return z

    def next_double(self, count: int) -> np.ndarray:
        """rng.hpp:22: (next() >> 11) * 2^-53."""
        return (self.next_u64(count) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)

    def next_below(self, n: int, count: int) -> np.ndarray:
        """rng.hpp:26-29: high 64 bits of next() * n (n < 2^32 here)."""
        assert 0 < n < (1 << 32)
        u = self.next_u64(count)
        nn = np.uint64(n)
        with np.errstate(over="ignore"):
            lo = (u & np.uint64(0xFFFFFFFF)) * nn
            hi = (u >> np.uint64(32)) * nn
            res = (hi + (lo >> np.uint64(32))) >> np.uint64(32)
        return res.astype(np.int64)

    def gaussian(self, count: int) -> np.ndarray:
        u = self.next_double(2 * count).reshape(count, 2)
        return np.sqrt(-2.0 * np.log1p(-u[:, 0])) * np.cos(2.0 * np.pi * u[:, 1])


def z_normalize_rows(values: np.ndarray) -> np.ndarray:
    """runner.hpp:82-95 applied to each row of an equal-length (N, L) block."""
    n = float(values.shape[1])
    mean = np.cumsum(values, axis=1)[:, -1] / n
    dev = values - mean[:, None]
    var = np.cumsum(dev * dev, axis=1)[:, -1]
    std = np.sqrt(var / n)
    out = np.zeros_like(values)
    ok = std > 0.0
    out[ok] = (values[ok] - mean[ok, None]) / std[ok, None]
    return out


def z_normalize_one(v: np.ndarray) -> np.ndarray:
    return z_normalize_rows(v[None, :])[0]


@dataclass
class Dataset:
    """A packed CSR dataset: series i is samples[offsets[i]:offsets[i+1]]."""

    samples: np.ndarray
    offsets: np.ndarray
    name: str = ""
    half_width: int = -1  # < 0: WarpWindow::unlimited()
    auto_widen: bool = False
    k: int = 0
    restarts: int = 10
    meta: dict = field(default_factory=dict)

    @property
    def p(self) -> int:
        return int(self.offsets.shape[0] - 1)

    @property
    def lengths(self) -> np.ndarray:
        return np.diff(self.offsets)

    def series(self, i: int) -> np.ndarray:
        return self.samples[self.offsets[i]:self.offsets[i + 1]]

    def subset(self, q: int) -> "Dataset":
        """First q series (used for bounded CPU samples)."""
        q = min(q, self.p)
        return Dataset(self.samples[: self.offsets[q]].copy(), self.offsets[: q + 1].copy(),
                       f"{self.name}[:{q}]", self.half_width, self.auto_widen, self.k,
                       self.restarts, dict(self.meta))


def from_rows(rows, name="", **kw) -> Dataset:
    lens = np.array([len(r) for r in rows], dtype=np.int64)
    offsets = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(lens, out=offsets[1:])
    samples = np.concatenate([np.asarray(r, dtype=np.float64) for r in rows]) if rows else \
        np.zeros(0, dtype=np.float64)
    return Dataset(samples, offsets, name, **kw)


def _from_block(block: np.ndarray, name: str, **kw) -> Dataset:
    n, L = block.shape
    offsets = np.arange(n + 1, dtype=np.int64) * L
    return Dataset(np.ascontiguousarray(block.reshape(-1)), offsets, name, **kw)


def _sinusoid_protos(rng: SplitMix64, classes: int):
    u = rng.next_double(classes * 6).reshape(classes, 3, 2)
    f = 1.0 + 9.0 * u[:, :, 0]
    phi = 2.0 * np.pi * u[:, :, 1]
    return f, phi


def config1(n: int = 100, length: int = 500) -> Dataset:
    rng = SplitMix64(BASE_SEED + 1)
    f, phi = _sinusoid_protos(rng, 4)
    t = np.arange(length, dtype=np.float64)
    protos = np.zeros((4, length))
    for c in range(4):
        for q in range(3):
            protos[c] += np.sin(2.0 * np.pi * f[c, q] * t / length + phi[c, q])
    shift = rng.next_below(101, n) - 50
    noise = rng.gaussian(n * length).reshape(n, length) * 0.1
    block = np.empty((n, length))
    for i in range(n):
        block[i] = np.roll(protos[i % 4], int(shift[i])) + noise[i]
    return _from_block(z_normalize_rows(block), "c1", half_width=-1, k=4, restarts=10)


def _random_walks(seed: int, n: int, length: int) -> np.ndarray:
    rng = SplitMix64(seed)
    steps = rng.gaussian(n * length).reshape(n, length)
    return z_normalize_rows(np.cumsum(steps, axis=1))


def config2(n: int = 1000, length: int = 1000, half_width: int = 100) -> Dataset:
    return _from_block(_random_walks(BASE_SEED + 2, n, length), "c2", half_width=half_width,
                       k=8, restarts=5)


def config3(n: int = 24000, length: int = 46) -> Dataset:
    rng = SplitMix64(BASE_SEED + 3)
    classes = 24
    t = np.arange(length, dtype=np.float64)
    protos = np.zeros((classes, length))
    for c in range(classes):
        a = int(rng.next_below(length - 2, 1)[0]) + 1
        b = a
        while b == a:
            b = int(rng.next_below(length - 2, 1)[0]) + 1
        knots_t = np.array([0, min(a, b), max(a, b), length - 1], dtype=np.float64)
        knots_v = rng.gaussian(4)
        protos[c] = np.interp(t, knots_t, knots_v)
    shift = rng.next_below(7, n) - 3
    noise = rng.gaussian(n * length).reshape(n, length) * 0.2
    idx = np.arange(length)
    block = np.empty((n, length))
    for i in range(n):
        src = np.clip(idx - int(shift[i]), 0, length - 1)
        block[i] = protos[i % classes][src] + noise[i]
    return _from_block(z_normalize_rows(block), "c3", half_width=-1, k=24, restarts=10)


def config4(n: int = 1000, length: int = 2844) -> Dataset:
    return _from_block(_random_walks(BASE_SEED + 4, n, length), "c4", half_width=-1)


def config5(n: int = 5000, lo: int = 50, hi: int = 1500, half_width: int = 100) -> Dataset:
    rng = SplitMix64(BASE_SEED + 5)
    lengths = rng.next_below(hi - lo + 1, n) + lo
    f, phi = _sinusoid_protos(rng, 10)
    noise = rng.gaussian(int(lengths.sum())) * 0.15
    rows = []
    pos = 0
    for i in range(n):
        L = int(lengths[i])
        u = np.arange(L, dtype=np.float64) / L
        c = i % 10
        v = np.zeros(L)
        for q in range(3):
            v += np.sin(2.0 * np.pi * f[c, q] * u + phi[c, q])
        v += noise[pos:pos + L]
        pos += L
        rows.append(z_normalize_one(v))
    return from_rows(rows, "c5", half_width=half_width, auto_widen=True, k=10, restarts=10)


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


def make_config(c: int, **kw) -> Dataset:
    return CONFIGS[c](**kw)


def pair_cells(n: np.ndarray, m: np.ndarray, hw) -> np.ndarray:
    """In-band cell count per pair, vectorised.

    hw may be an array (per-pair effective half-width) or scalar; < 0 = unlimited.
    cells = sum_{i=1..N} max(0, min(M, i+hw) - max(1, i-hw) + 1) with N >= M.
    """
    n = np.asarray(n, dtype=np.int64)
    m = np.asarray(m, dtype=np.int64)
    N = np.maximum(n, m)
    M = np.minimum(n, m)
    hw = np.broadcast_to(np.asarray(hw, dtype=np.int64), N.shape)
    full = hw < 0
    h = np.where(full, N, hw)
    # cells = N*M - (left triangle: cells with j < i - h) - (right: j > i + h)
    # left: rows i > h+1, count min(M, i-h-1); right: rows i < M-h, count M-(i+h)
    def tri_left(N, M, h):
        # sum_{i=h+2..N} min(M, i-h-1) = sum_{t=1..N-h-1} min(M, t)
        T = np.maximum(N - h - 1, 0)
        a = np.minimum(T, M)
        return a * (a + 1) // 2 + np.maximum(T - M, 0) * M

    def tri_right(N, M, h):
        # sum_{i=1..M-h-1} (M - h - i) = S(S+1)/2, S = M-h-1 (i <= N automatically since M <= N)
        S = np.maximum(M - h - 1, 0)
        return S * (S + 1) // 2

    cells = N * M - tri_left(N, M, h) - tri_right(N, M, h)
    return np.where(full, N * M, cells)


def effective_half_width(n: np.ndarray, m: np.ndarray, half_width: int, auto_widen: bool):
    """pairwise.hpp:29-33 pair_window, vectorised; < 0 = unlimited."""
    n = np.asarray(n, dtype=np.int64)
    m = np.asarray(m, dtype=np.int64)
    if half_width < 0:
        return np.full(np.broadcast(n, m).shape, -1, dtype=np.int64)
    gap = np.abs(n - m)
    if auto_widen:
        return np.where(gap > half_width, gap, half_width)
    return np.full(gap.shape, half_width, dtype=np.int64)


def total_cells(ds: Dataset, slot_begin: int = 0, slot_end: int | None = None) -> int:
    """Total in-band cells over the condensed pairs of a dataset (the GCUPS numerator)."""
    p = ds.p
    lens = ds.lengths
    total = 0
    if slot_end is None:
        slot_end = p * (p - 1) // 2
    if slot_begin == 0 and slot_end == p * (p - 1) // 2 and np.all(lens == lens[0]) and p > 1:
        hw = effective_half_width(lens[:1], lens[:1], ds.half_width, ds.auto_widen)
        return int(pair_cells(lens[:1], lens[:1], hw)[0]) * (p * (p - 1) // 2)
    for i in range(p - 1):
        row0 = i * p - i * (i + 1) // 2
        lo = max(slot_begin - row0, 0)
        hi = min(slot_end - row0, p - 1 - i)
        if hi <= lo:
            continue
        js = np.arange(i + 1 + lo, i + 1 + hi)
        hw = effective_half_width(lens[i], lens[js], ds.half_width, ds.auto_widen)
        total += int(pair_cells(np.full(js.shape, lens[i]), lens[js], hw).sum())
    return total
