"""Materialising ladder: dist_baseline / dist_soa / dist_tiled,
build_clusters_from_dist and run_variant's BASELINE/SOA/TILED/TILED_UNROLLED rungs.

Golden vectors: tests/golden/dist.npz, made by executing the reference
(tests/golden/make_golden_dist.py). Bar: bit-exact float32 matrices (compared as
uint32 bit patterns), identical reference-layout bits, int64 counts and labels.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden

CASES = ["kat345", "lattice", "blobs257", "uniform101"]
LADDER = ["BASELINE", "SOA", "TILED", "TILED_UNROLLED"]


def _case(g, key):
    eps, eps_sq, min_pts = g[f"{key}/params"]
    return g[f"{key}/points"], float(eps), float(eps_sq), int(min_pts)


# ---- CPU: the oracle restatement is pinned to the reference's matrices ----
@pytest.mark.parametrize("key", CASES)
def test_oracle_direct_matrix_matches_reference(key):
    from oracle import densescan_oracle as oracle
    g = load_golden("dist.npz")
    pts, _, eps_sq, _ = _case(g, key)
    p32 = oracle.narrow(pts)
    d2 = oracle.block_d2_direct(p32, p32)
    assert d2.dtype == np.float32
    assert np.array_equal(d2.view(np.uint32), g[f"{key}/dist"].view(np.uint32))
    bits, counts = oracle.neighborhood(pts, eps_sq, oracle.DIRECT)
    assert np.array_equal(bits, g[f"{key}/bits"])
    assert np.array_equal(counts, g[f"{key}/counts"])


def test_dist_tiled_rejects_other_variants():
    import paper_1506_02226_b200 as ds
    pts = ds.PointSet(np.zeros((4, 3)))
    with pytest.raises(ValueError):
        ds.dist_tiled(pts, ds.KernelVariant(ds.VariantId.FUSED))


def test_ladder_capacity_guard():
    import paper_1506_02226_b200 as ds
    pts = ds.PointSet(np.zeros((100, 3)))
    with pytest.raises(ds.CapacityExceeded) as e:
        ds.dist_baseline(pts, mem_cap=4 * 100 * 100 - 1)
    assert e.value.required_bytes == 40000


# ---- GPU ----
@pytest.fixture(scope="module")
def ds():
    import paper_1506_02226_b200 as pkg
    from paper_1506_02226_b200 import _native
    _native.load_library()
    return pkg


@pytest.mark.gpu
@pytest.mark.parametrize("key", CASES)
def test_dist_matrix_bit_exact(ds, key):
    g = load_golden("dist.npz")
    pts, _, _, _ = _case(g, key)
    p = ds.PointSet(pts)
    want = g[f"{key}/dist"].view(np.uint32)
    for got in (ds.dist_baseline(p), ds.dist_soa(p),
                ds.dist_tiled(p, ds.KernelVariant(ds.VariantId.TILED, tile_size=64)),
                ds.dist_tiled(p, ds.KernelVariant(ds.VariantId.TILED_UNROLLED, tile_size=48,
                                                  unroll_width=5))):
        assert got.n == p.n and got.values.dtype == np.float32
        assert np.array_equal(got.values.view(np.uint32), want)


@pytest.mark.gpu
@pytest.mark.parametrize("key", CASES)
def test_build_clusters_from_dist(ds, key):
    g = load_golden("dist.npz")
    _, eps, eps_sq, min_pts = _case(g, key)
    dist = ds.DistSqMatrix(n=g[f"{key}/dist"].shape[0], values=g[f"{key}/dist"])
    params = ds.validate_params(eps, min_pts)
    assert params.eps_sq == eps_sq
    nbr, valid = ds.build_clusters_from_dist(dist, params)
    assert np.array_equal(nbr.bits, g[f"{key}/bits"])
    assert np.array_equal(nbr.neighbor_count, g[f"{key}/counts"])
    assert np.array_equal(valid.valid, g[f"{key}/counts"] >= min_pts)
    labels = ds.merge_iterative(nbr, valid).labels
    assert np.array_equal(labels, g[f"{key}/labels"])


@pytest.mark.gpu
@pytest.mark.parametrize("rung", LADDER)
def test_run_variant_materialising_rungs(ds, rung):
    g = load_golden("dist.npz")
    for key in CASES:
        pts, eps, _, min_pts = _case(g, key)
        v = ds.KernelVariant(getattr(ds.VariantId, rung))
        nbr, valid, dist_ms, cluster_ms, fused_ms = ds.run_variant(
            ds.PointSet(pts), ds.validate_params(eps, min_pts), v)
        assert fused_ms is None and dist_ms >= 0 and cluster_ms >= 0
        assert np.array_equal(nbr.bits, g[f"{key}/bits"])
        assert np.array_equal(nbr.neighbor_count, g[f"{key}/counts"])


@pytest.mark.gpu
@pytest.mark.parametrize("n,d", [(1, 3), (7, 2), (1000, 3), (3001, 5), (513, 16), (129, 24), (300, 40)])
def test_dist_matrix_vs_oracle_random(ds, n, d, rng):
    from oracle import densescan_oracle as oracle
    pts = rng.normal(0, 3, (n, d)) + rng.uniform(-50, 50, d)
    p32 = oracle.narrow(pts)
    want = oracle.block_d2_direct(p32, p32)
    got = ds.dist_baseline(ds.PointSet(pts)).values
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    eps = max(float(np.sqrt(np.median(want))), 1e-3)
    params = ds.validate_params(eps, 3)
    nbr, _ = ds.build_clusters_from_dist(ds.DistSqMatrix(n=n, values=got), params)
    bits, counts = oracle.neighborhood(pts, params.eps_sq, oracle.DIRECT)
    assert np.array_equal(nbr.bits, bits) and np.array_equal(nbr.neighbor_count, counts)
    # the materialising build agrees with the fused direct-formula kernel
    fb, _ = ds.fused_build(ds.PointSet(pts), params, ds.KernelVariant(ds.VariantId.FUSED))
    assert np.array_equal(fb.bits, bits)
