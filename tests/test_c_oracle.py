"""The C oracle (large-N checker) agrees with the numpy oracle and the reference."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_cases, load_golden, random_specs
from oracle import c_oracle
from oracle import densescan_oracle as oracle
from paper_1506_02226_b200.datasets import generate_blobs


def test_kat_and_lattices_match_reference():
    for fixture in ("kat.npz", "lattice.npz"):
        g = load_golden(fixture)
        for name, pts, _, eps_sq, min_pts in golden_cases(g):
            for fname, f in (("alg", 1), ("dir", 0)):
                labels, counts = c_oracle.dbscan(pts, eps_sq, min_pts, f, nthreads=2)
                assert np.array_equal(counts, g[f"{name}/{fname}/counts"]), (name, fname)
                assert np.array_equal(labels, g[f"{name}/{fname}/labels"]), (name, fname)


def test_random_unfiltered_match_reference():
    g = load_golden("random.npz")
    for name, pts, _, eps_sq, min_pts in random_specs(g):
        for fname, f in (("alg", 1), ("dir", 0)):
            labels, counts = c_oracle.dbscan(pts, eps_sq, min_pts, f, nthreads=3)
            assert np.array_equal(counts, g[f"{name}/{fname}/counts"]), (name, fname)
            assert np.array_equal(labels, g[f"{name}/{fname}/labels"]), (name, fname)


@pytest.mark.parametrize("d", [1, 5, 16])
def test_matches_numpy_oracle_any_dimension(rng, d):
    for _ in range(3):
        n = int(rng.integers(2, 1500))
        pts = generate_blobs(n, 3, 0.4, 0.2, int(rng.integers(2**31)), d).coords_aos * 3.0 + 20
        eps_sq = float(rng.uniform(0.5, 2.0)) ** 2 * d / 2
        mp = int(rng.integers(1, 9))
        for f in (0, 1):
            want, wc = oracle.dbscan(pts, eps_sq, mp, f)
            got, gc = c_oracle.dbscan(pts, eps_sq, mp, f, nthreads=4)
            assert np.array_equal(gc, wc) and np.array_equal(got, want)


def test_thread_count_independence(rng):
    pts = generate_blobs(3000, 4, 0.3, 0.2, 9, 2).coords_aos
    base = c_oracle.dbscan(pts, 0.01, 5, 1, nthreads=1)
    for t in (2, 3, 7):
        other = c_oracle.dbscan(pts, 0.01, 5, 1, nthreads=t)
        assert np.array_equal(base[0], other[0]) and np.array_equal(base[1], other[1])


@pytest.mark.slow
def test_c1_and_c2_full_against_reference():
    g1 = load_golden("c1.npz")
    pts = generate_blobs(10_000, 4, 0.5, 0.0, 1, 2).coords_aos
    for fname, f in (("alg", 1), ("dir", 0)):
        labels, counts = c_oracle.dbscan(pts, 0.3 * 0.3, 4, f)
        assert np.array_equal(labels, g1[f"{fname}/labels"])
        assert np.array_equal(counts, g1[f"{fname}/counts"])
    g2 = load_golden("c2.npz")
    pts = generate_blobs(200_000, 16, 1.0, 0.10, 2, 2).coords_aos
    labels, counts = c_oracle.dbscan(pts, 0.3 * 0.3, 8, 1)
    assert np.array_equal(labels, g2["labels"]) and np.array_equal(counts, g2["counts"])
