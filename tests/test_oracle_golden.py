"""Pin the CPU oracle against outputs of the reference itself (tests/golden).

The fixtures were produced by tests/golden/make_golden.py running the
reference package (fused_build / fused_build_algebraic + merge_iterative).
Here the oracle must reproduce them bit-for-bit; the GPU is then checked
against both (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import golden_cases, load_golden, pad3, random_specs
from oracle import densescan_oracle as oracle

FORMULAS = {"alg": oracle.ALGEBRAIC, "dir": oracle.DIRECT}


def sha(bits):
    return hashlib.sha256(np.ascontiguousarray(bits).tobytes()).hexdigest()


def check_case(g, name, pts, eps_sq, min_pts):
    for fname, f in FORMULAS.items():
        bits, counts = oracle.neighborhood(pts, eps_sq, f)
        assert sha(bits) == str(g[f"{name}/{fname}/bits_sha"]), (name, fname)
        if f"{name}/{fname}/bits" in g:
            assert np.array_equal(bits, g[f"{name}/{fname}/bits"])
        assert np.array_equal(counts, g[f"{name}/{fname}/counts"]), (name, fname)
        labels, _ = oracle.dbscan(pts, eps_sq, min_pts, f)
        assert np.array_equal(labels, g[f"{name}/{fname}/labels"]), (name, fname)
        assert np.array_equal(oracle.merge_labels(bits, counts, min_pts), labels)


def test_known_answer_cases():
    g = load_golden("kat.npz")
    names = []
    for name, pts, _, eps_sq, min_pts in golden_cases(g):
        check_case(g, name, pts, eps_sq, min_pts)
        names.append(name)
    # spot-check the hand-derived answers of the reference test-suite
    assert list(g["collinear/alg/labels"]) == [0, 0, 0]
    assert list(g["two_groups/alg/labels"]) == [0, 0, 1, 1]
    assert list(g["single/alg/labels"]) == [0]
    bt = g["border_tie/alg/labels"]
    assert bt[8] == bt[0] != bt[4]
    assert "lattice_ties" in names


def test_lattice_ties_and_far_offsets():
    g = load_golden("lattice.npz")
    for name, pts, _, eps_sq, min_pts in golden_cases(g):
        check_case(g, name, pts, eps_sq, min_pts)


def test_random_unfiltered():
    g = load_golden("random.npz")
    for name, pts, _, eps_sq, min_pts in random_specs(g):
        check_case(g, name, pts, eps_sq, min_pts)


def test_c1_native_2d_equals_reference_padded():
    from paper_1506_02226_b200.datasets import generate_blobs
    g = load_golden("c1.npz")
    pts = generate_blobs(10_000, 4, 0.5, 0.0, 1, 2).coords_aos
    for fname, f in FORMULAS.items():
        for coords in (pts, pad3(pts)):
            bits, counts = oracle.neighborhood(coords, 0.3 * 0.3, f)
            assert sha(bits) == str(g[f"{fname}/bits_sha"])
            assert np.array_equal(counts, g[f"{fname}/counts"])
        labels, _ = oracle.dbscan(pts, 0.3 * 0.3, 4, f)
        assert np.array_equal(labels, g[f"{fname}/labels"])
    lab = g["alg/labels"]
    assert len(set(lab.tolist()) - {-1}) == 4 and int((lab == -1).sum()) == 27


@pytest.mark.slow
def test_blob23040_counts():
    from paper_1506_02226_b200.datasets import generate_blobs
    g = load_golden("blob23040.npz")
    pts = generate_blobs(23040, 3, 0.03, 0.02, 1).coords_aos
    for fname, f in FORMULAS.items():
        labels, counts = oracle.dbscan(pts, 0.1 * 0.1, 8, f)
        assert np.array_equal(counts, g[f"{fname}/counts"])
        assert np.array_equal(labels, g[f"{fname}/labels"])


def test_formulas_really_differ_somewhere():
    """The far-offset lattice is a case where ALGEBRAIC != DIRECT: the fixtures
    exercise the rounding difference rather than two copies of one answer."""
    g = load_golden("lattice.npz")
    diffs = sum(not np.array_equal(g[f"{n}/alg/counts"], g[f"{n}/dir/counts"])
                for n in (str(x) for x in g["names"]))
    assert diffs >= 1


def test_reference_flow_port_matches_reference():
    """The threaded CPU baseline (bench.py cpu_baseline / --impl reference) computes the
    reference's labels and counts: C1 both formulas, the 48 random unfiltered sets."""
    from paper_1506_02226_b200.datasets import CONFIGS
    g = load_golden("c1.npz")
    pts = CONFIGS["C1"].points()
    for name, f in (("alg", 1), ("dir", 0)):
        labels, counts, _, _ = oracle.dbscan_reference_flow(pts.coords_aos, 0.3 * 0.3, 4, f,
                                                            threads=3)
        assert np.array_equal(labels, g[f"{name}/labels"])
        assert np.array_equal(counts, g[f"{name}/counts"])
    r = load_golden("random.npz")
    for name, coords, eps, eps_sq, min_pts in random_specs(r):
        labels, counts, _, _ = oracle.dbscan_reference_flow(coords, eps_sq, min_pts, 1, threads=2)
        assert np.array_equal(labels, r[f"{name}/alg/labels"]), name
