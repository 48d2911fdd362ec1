"""Seeded synthetic point sets for the benchmark configurations C1-C5.

`generate_blobs` is the d-dimensional generalisation of the reference's
`generate_blobs` (pkg/src/densescan/core.py:181-222): the same rng call
sequence, lattice placement (pitch max(10*spread, 1), coordinate 0
fastest), remainder split and noise box, so at d=3 it returns the same
bits as the reference (pinned by tests/golden, see make_golden.py).

`generate_chain` is the C5 "skewed density" set defined in SURVEY.md §8(d):
a 1.6M-point serpentine chain, eight dense blobs and uniform noise.

`CONFIGS` names the five BASELINE.json configurations.
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass

import numpy as np

from .core import InvalidParams, PointSet


def _lattice_cells(k: int, d: int) -> np.ndarray:
    side = math.ceil(k ** (1.0 / d))
    # coordinate 0 varies fastest, as in the reference's (i, j, l) comprehension
    cells = itertools.islice(itertools.product(range(side), repeat=d), k)
    return np.array([c[::-1] for c in cells], dtype=np.float64).reshape(k, d)


def generate_blobs(n: int, k: int, spread: float, noise_fraction: float,
                   seed: int, d: int = 3) -> PointSet:
    """k Gaussian blobs on a lattice plus uniform noise, in d dimensions."""
    if not (isinstance(n, (int, np.integer)) and n >= 1):
        raise InvalidParams("n", f"point count must be >= 1, got {n!r}")
    if not (isinstance(k, (int, np.integer)) and 1 <= k <= n):
        raise InvalidParams("k", f"cluster count must satisfy 1 <= k <= n, got {k!r}")
    if not (isinstance(spread, (int, float)) and math.isfinite(spread) and spread >= 0):
        raise InvalidParams("spread", f"spread must be a finite real >= 0, got {spread!r}")
    if not (isinstance(noise_fraction, (int, float)) and 0.0 <= noise_fraction <= 1.0):
        raise InvalidParams("noise_fraction",
                            f"noise fraction must lie in [0, 1], got {noise_fraction!r}")
    if not (isinstance(d, (int, np.integer)) and d >= 1):
        raise InvalidParams("d", f"dimension must be >= 1, got {d!r}")

    rng = np.random.default_rng(seed)
    pitch = max(10.0 * float(spread), 1.0)
    centers = _lattice_cells(int(k), int(d)) * pitch

    n_noise = min(int(round(noise_fraction * n)), n - k)
    n_blob = n - n_noise
    per_blob = np.full(k, n_blob // k, dtype=np.int64)
    per_blob[: n_blob % k] += 1

    parts = [c + rng.normal(0.0, float(spread), size=(int(m), d))
             for c, m in zip(centers, per_blob)]
    if n_noise:
        lo = centers.min(axis=0) - pitch / 2.0
        hi = centers.max(axis=0) + pitch / 2.0
        parts.append(rng.uniform(lo, hi, size=(n_noise, d)))
    return PointSet(np.concatenate(parts, axis=0))


def generate_chain(n_chain: int = 1_600_000, n_blob_each: int = 47_500, n_blobs: int = 8,
                   n_noise: int = 20_000, seed: int = 5) -> PointSet:
    """C5: serpentine chain + dense blobs + noise.

    The chain has 40 horizontal runs of length 100 at y = 1.5*r, alternating
    direction, joined by vertical segments of length 1.5 (total arc length
    4058.5). Draw order: arc positions, perpendicular jitter N(0, 0.05),
    blobs N((6.25 + 12.5 i, 70), 0.3^2 I), noise x ~ U(-5, 105) then
    y ~ U(-5, 75).
    """
    rng = np.random.default_rng(seed)
    run, gap, runs = 100.0, 1.5, 40
    period = run + gap
    s = rng.uniform(0.0, runs * run + (runs - 1) * gap, size=n_chain)
    jitter = rng.normal(0.0, 0.05, size=n_chain)
    r = np.minimum(np.floor(s / period), runs - 1)
    u = s - r * period
    horizontal = u < run
    forward = (r % 2) == 0
    x = np.where(horizontal, np.where(forward, u, run - u), np.where(forward, run, 0.0))
    y = np.where(horizontal, gap * r, gap * r + (u - run))
    x = np.where(horizontal, x, x + jitter)
    y = np.where(horizontal, y + jitter, y)
    parts = [np.stack([x, y], axis=1)]
    for i in range(n_blobs):
        parts.append(np.array([6.25 + 12.5 * i, 70.0])
                     + rng.normal(0.0, 0.3, size=(n_blob_each, 2)))
    nx = rng.uniform(-5.0, 105.0, size=n_noise)
    ny = rng.uniform(-5.0, 75.0, size=n_noise)
    parts.append(np.stack([nx, ny], axis=1))
    return PointSet(np.concatenate(parts, axis=0))


@dataclass(frozen=True)
class BenchConfig:
    name: str
    n: int
    d: int
    eps: float
    min_pts: int
    description: str

    def points(self) -> PointSet:
        return _BUILDERS[self.name]()


_BUILDERS = {
    "C1": lambda: generate_blobs(10_000, 4, 0.5, 0.0, 1, 2),
    "C2": lambda: generate_blobs(200_000, 16, 1.0, 0.10, 2, 2),
    "C3": lambda: generate_blobs(1_000_000, 16, 1.0, 0.0, 3, 2),
    "C4": lambda: generate_blobs(500_000, 8, 0.5, 0.0, 4, 16),
    "C5": lambda: generate_chain(),
}

CONFIGS = {
    "C1": BenchConfig("C1", 10_000, 2, 0.3, 4,
                      "2-D Gaussian blobs N=10k, eps=0.3, MinPts=4"),
    "C2": BenchConfig("C2", 200_000, 2, 0.3, 8,
                      "2-D blobs + 10% uniform noise N=200k, eps=0.3, MinPts=8"),
    "C3": BenchConfig("C3", 1_000_000, 2, 0.3, 8,
                      "2-D blobs N=1M, eps=0.3, MinPts=8 (row-block sharded)"),
    "C4": BenchConfig("C4", 500_000, 16, 1.6, 8,
                      "16-D blobs N=500k, eps=1.6, MinPts=8"),
    "C5": BenchConfig("C5", 2_000_000, 2, 0.3, 8,
                      "skewed density N=2M: serpentine chain + dense blobs + noise"),
}
