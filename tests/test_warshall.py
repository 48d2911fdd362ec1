"""Warshall backend (reference merge.py:169-238).

CPU: the oracle restatement against fixtures made by executing the reference
(tests/golden/make_golden_warshall.py). GPU: build_core_adjacency,
warshall_closure and merge_warshall through the C ABI against the same
fixtures, bit for bit, plus larger random relations against the oracle.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden


@pytest.fixture(scope="module")
def fx():
    return load_golden("warshall.npz")


def test_oracle_matches_reference_adjacency(fx):
    from oracle import densescan_oracle as oracle
    for name in fx["adj_names"]:
        name = str(name)
        ci, adj = oracle.core_adjacency(fx[f"adj/{name}/bits"], fx[f"adj/{name}/valid"])
        assert np.array_equal(ci, fx[f"adj/{name}/core_indices"]), name
        assert np.array_equal(adj, fx[f"adj/{name}/adj"]), name
        closed = oracle.warshall_closure_bits(adj, ci.size)
        assert np.array_equal(closed, fx[f"adj/{name}/closed"]), name


def test_oracle_matches_reference_closure(fx):
    from oracle import densescan_oracle as oracle
    for name in fx["cl_names"]:
        name = str(name)
        a = fx[f"cl/{name}/in"]
        assert np.array_equal(oracle.warshall_closure_bits(a, a.shape[0]), fx[f"cl/{name}/out"]), name


@pytest.fixture(scope="module")
def ds():
    import paper_1506_02226_b200 as pkg
    from paper_1506_02226_b200 import _native
    _native.load_library()
    return pkg


@pytest.mark.gpu
def test_gpu_core_adjacency_and_closure(ds, fx):
    for name in fx["adj_names"]:
        name = str(name)
        bits = fx[f"adj/{name}/bits"]
        valid = fx[f"adj/{name}/valid"].astype(bool)
        n = valid.size
        nbr = ds.NeighborhoodMatrix(n=n, bits=bits, neighbor_count=np.zeros(n, np.int64))
        vv = ds.ValidVector(valid=valid, min_pts=1)
        adj = ds.build_core_adjacency(nbr, vv)
        assert adj.m == int(valid.sum())
        assert np.array_equal(adj.core_indices, fx[f"adj/{name}/core_indices"]), name
        assert np.array_equal(adj.bits, fx[f"adj/{name}/adj"]), name
        before = adj.bits.copy()
        closed = ds.warshall_closure(adj)
        assert np.array_equal(adj.bits, before)  # input not mutated
        assert np.array_equal(closed.bits, fx[f"adj/{name}/closed"]), name
        assert np.array_equal(ds.merge_warshall(nbr, vv).labels, fx[f"adj/{name}/labels"]), name


@pytest.mark.gpu
def test_gpu_closure_reference_cases(ds, fx):
    for name in fx["cl_names"]:
        name = str(name)
        a = fx[f"cl/{name}/in"]
        m = a.shape[0]
        adj = ds.CoreAdjacency(m=m, core_indices=np.arange(m, dtype=np.int64), bits=a)
        assert np.array_equal(ds.warshall_closure(adj).bits, fx[f"cl/{name}/out"]), name


@pytest.mark.gpu
def test_gpu_closure_random_directed_vs_oracle(ds, rng):
    from oracle import densescan_oracle as oracle
    for m in (31, 32, 33, 95, 257, 700):
        for p in (0.002, 0.01, 0.05):
            rel = rng.random((m, m)) < p
            bits = np.packbits(rel, axis=-1)
            adj = ds.CoreAdjacency(m=m, core_indices=np.arange(m, dtype=np.int64), bits=bits)
            got = ds.warshall_closure(adj).bits
            assert np.array_equal(got, oracle.warshall_closure_bits(bits, m)), (m, p)


@pytest.mark.gpu
def test_gpu_merge_warshall_takes_valid_as_given(ds, fx):
    bits = fx["mw/bits"]
    valid = fx["mw/valid"].astype(bool)
    n = valid.size
    nbr = ds.NeighborhoodMatrix(n=n, bits=bits, neighbor_count=np.zeros(n, np.int64))
    labels = ds.merge_warshall(nbr, ds.ValidVector(valid=valid, min_pts=5)).labels
    assert np.array_equal(labels, fx["mw/labels"])


@pytest.mark.gpu
def test_gpu_core_adjacency_at_c1(ds):
    """build_core_adjacency + merge_warshall on C1 (10k points) against the oracle."""
    from oracle import densescan_oracle as oracle
    cfg = ds.CONFIGS["C1"]
    pts = cfg.points()
    params = ds.validate_params(cfg.eps, cfg.min_pts)
    nbr, valid = ds.fused_build_algebraic(pts, params, ds.KernelVariant(ds.VariantId.FUSED_ALGEBRAIC))
    adj = ds.build_core_adjacency(nbr, valid)
    ci, want = oracle.core_adjacency(nbr.bits, valid.valid)
    assert np.array_equal(adj.core_indices, ci) and np.array_equal(adj.bits, want)
    lab = ds.merge_warshall(nbr, valid).labels
    assert np.array_equal(lab, ds.merge_iterative(nbr, valid).labels)
