"""Shared test configuration.

Markers: `gpu` (needs a B200 and the built library; run with -m gpu),
`slow` (full-size property checks). The CPU suite (-m "not gpu") covers the
oracle against the reference's golden vectors, the host-side API, the C-ABI
exports and the multi-process exchange logic.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device and the sm_100a library")
    config.addinivalue_line("markers", "slow: full-size property checks")


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


def load_golden(name: str):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated")
    return np.load(path, allow_pickle=False)


def golden_cases(npz):
    """(name, points, eps, eps_sq, min_pts) for fixtures with stored points."""
    for name in npz["names"]:
        name = str(name)
        eps, eps_sq, min_pts = npz[f"{name}/params"]
        yield name, npz[f"{name}/points"], float(eps), float(eps_sq), int(min_pts)


def random_specs(npz):
    from paper_1506_02226_b200.datasets import generate_blobs
    for t, spec in enumerate(npz["specs"]):
        n, k, spread, noise, seed, d, scale, offset, eps, min_pts = spec
        coords = generate_blobs(int(n), int(k), float(spread), float(noise), int(seed),
                                int(d)).coords_aos * scale + offset
        yield f"r{t:03d}", coords, float(eps), float(eps) * float(eps), int(min_pts)


def pad3(coords):
    coords = np.asarray(coords, dtype=np.float64)
    if coords.shape[1] == 3:
        return coords
    out = np.zeros((coords.shape[0], 3))
    out[:, : coords.shape[1]] = coords
    return out
