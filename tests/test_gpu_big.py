"""GPU parity at the full BASELINE sizes C3 (1M, 2-D), C4 (500k, 16-D) and C5
(2M: a 13.5k-hop chain + dense blobs, the union-find stress case), against
committed fixtures made by the pinned C oracle (tests/golden/make_golden_big.py;
the reference itself cannot run these sizes). Both the default
schedule (spatial order + culling) and the paper's dense all-pairs schedule are
compared, so a union-find bug shared by both schedules fails here.

Also the capacity path: a call that overflows its unit list or word buffer is
re-run with larger buffers until nothing overflows (never returned as OK with
dropped adjacency), checked with a forced tiny initial capacity, and a fresh
context needs at most two stage 1+2 launches at C3.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

MEM_CAP = 96 * 1024**3


@pytest.fixture(scope="module")
def ds():
    import paper_1506_02226_b200 as pkg
    from paper_1506_02226_b200 import _native
    _native.load_library()
    return pkg


def counts_sha(counts):
    return hashlib.sha256(np.ascontiguousarray(counts, dtype=np.int64).tobytes()).hexdigest()


def check_against_fixture(ds, name, prune, order):
    fx = load_golden(f"{name.lower()}.npz")
    cfg = ds.CONFIGS[name]
    pts = cfg.points()
    assert pts.n == int(fx["n"]) and pts.d == int(fx["d"])
    params = ds.validate_params(cfg.eps, cfg.min_pts)
    ctx = ds._native.context()
    prev = ctx.schedule()
    ctx.configure(prune, order)
    try:
        labels, counts, t = ctx.run_dbscan(pts.coords_aos, params.eps_sq, cfg.min_pts, 1,
                                           MEM_CAP, want_counts=True)
    finally:
        ctx.configure(*prev)
    want = fx["labels"].astype(np.int64)
    bad = np.nonzero(labels != want)[0]
    assert bad.size == 0, (f"{name}: {bad.size} labels differ, first at {bad[:5]} "
                           f"(got {labels[bad[:5]]}, want {want[bad[:5]]})")
    sample = counts[::97]
    assert np.array_equal(sample, fx["counts_sample"].astype(np.int64)), name
    assert counts_sha(counts) == str(fx["counts_sha"]), name
    assert t.core_count == int(fx["cores"])
    assert t.cluster_count == int(fx["clusters"])
    return t


@pytest.mark.parametrize("name", ["C5", "C3", "C4"])
def test_full_size_default_schedule(ds, name):
    check_against_fixture(ds, name, True, True)


@pytest.mark.parametrize("name", ["C5", "C3"])
def test_full_size_dense_schedule(ds, name):
    check_against_fixture(ds, name, False, False)


def test_c5_public_api(ds):
    """run_dbscan(default_config()) exactly as a reference user calls it."""
    fx = load_golden("c5.npz")
    cfg = ds.CONFIGS["C5"]
    pts = cfg.points()
    conf = ds.default_config()
    conf.mem_cap = MEM_CAP
    labeling, timings = ds.run_dbscan(pts, ds.validate_params(cfg.eps, cfg.min_pts), conf)
    assert np.array_equal(labeling.labels, fx["labels"].astype(np.int64))
    assert timings.fused_ms > 0 and timings.merge_ms > 0


def test_fresh_context_c3_at_most_two_launches(ds):
    fx = load_golden("c3.npz")
    cfg = ds.CONFIGS["C3"]
    pts = cfg.points()
    params = ds.validate_params(cfg.eps, cfg.min_pts)
    ctx = ds._native.Context(0)
    try:
        labels, _, t = ctx.run_dbscan(pts.coords_aos, params.eps_sq, cfg.min_pts, 1, MEM_CAP)
        assert t.tile_launches <= 2, t.tile_launches
        assert np.array_equal(labels, fx["labels"].astype(np.int64))
    finally:
        ctx.close()


@pytest.mark.parametrize("cull", [True, False])
def test_forced_tiny_capacity_regrows_to_exact_labels(ds, cull):
    """Start from 1 unit / 1 word and grow at most x2 per re-run: the call walks
    through many overflowing launches and must still return the oracle's labels."""
    from oracle import c_oracle
    pts = ds.generate_blobs(30_000, 6, 0.4, 0.05, 11, 2)
    params = ds.validate_params(0.3, 8)
    want, wc = c_oracle.dbscan(pts.coords_aos, params.eps_sq, 8, 1)
    ctx = ds._native.Context(0)
    try:
        ctx.configure(cull, cull)
        ctx.set_test_capacity(1)
        labels, counts, t = ctx.run_dbscan(pts.coords_aos, params.eps_sq, 8, 1, 0,
                                           want_counts=True)
        assert t.tile_launches >= 5, t.tile_launches
        assert np.array_equal(labels, want) and np.array_equal(counts, wc)
        # stage-level entry point and shard stage walk the same loop
        ctx.set_test_capacity(1)
        bits, counts2, _, t2 = ctx.fused_build(pts.coords_aos, params.eps_sq, 8, 1, 0,
                                               want_bits=False)
        assert t2.tile_launches >= 5 and np.array_equal(counts2, wc)
        ctx.set_test_capacity(0)
        labels3, _, t3 = ctx.run_dbscan(pts.coords_aos, params.eps_sq, 8, 1, 0)
        assert np.array_equal(labels3, want) and t3.tile_launches == 1
    finally:
        ctx.close()


def test_capacity_cap_still_raises(ds):
    """Growing stops at the memory cap with CapacityExceeded (never a partial result)."""
    pts = ds.generate_blobs(30_000, 1, 0.05, 0.0, 2, 2)
    params = ds.validate_params(0.5, 4)
    ctx = ds._native.Context(0)
    try:
        ctx.set_test_capacity(1)
        with pytest.raises(ds.CapacityExceeded):
            ctx.run_dbscan(pts.coords_aos, params.eps_sq, 4, 1, 12_000_000)
    finally:
        ctx.close()


@pytest.mark.parametrize("name,pairs,tiles", [("C2", 152_918_016, 3823)])
def test_spatial_sort_is_the_stable_key_order(ds, name, pairs, tiles):
    """The hand-written LSD radix sort (ds_sort.cu) must give the stable (key, index)
    order — the one round 1's library sort produced: the work counters of the culled
    schedule depend on the exact permutation, so they must equal the pinned numbers, on
    two independent contexts and on repeated calls. (Kept tile pairs: round 1's 3823.
    Pairs: round 1's 211,812,352 before the row-pair culling of the unit list, 152,918,016
    with it.)"""
    cfg = ds.CONFIGS[name]
    pts = cfg.points()
    params = ds.validate_params(cfg.eps, cfg.min_pts)
    seen = set()
    for _ in range(2):
        ctx = ds._native.Context(0)
        try:
            ctx.set_stable_order(True)  # the radix sort (C2 would take the counting sort)
            for _ in range(2):
                _, _, t = ctx.run_dbscan(pts.coords_aos, params.eps_sq, cfg.min_pts, 1, MEM_CAP)
                seen.add((t.pairs_evaluated, t.tiles_total))
        finally:
            ctx.close()
    assert seen == {(pairs, tiles)}


def test_counting_sort_order_gives_identical_results(ds):
    """C2 takes the counting-sort spatial order by default (arbitrary order inside a grid
    cell) and the stable radix sort with DS_OPT_STABLE_ORDER: labels and counts are
    identical (the reference's), only the schedule may differ."""
    cfg = ds.CONFIGS["C2"]
    pts = cfg.points()
    params = ds.validate_params(cfg.eps, cfg.min_pts)
    out = {}
    for stable in (False, True):
        ctx = ds._native.Context(0)
        try:
            ctx.set_stable_order(stable)
            for _ in range(3):  # eager, recorded, replayed
                labels, counts, t = ctx.run_dbscan(pts.coords_aos, params.eps_sq, cfg.min_pts, 1,
                                                   MEM_CAP, want_counts=True)
                out.setdefault(stable, []).append((labels.copy(), counts.copy()))
        finally:
            ctx.close()
    ref_labels, ref_counts = out[True][0]
    for stable in (False, True):
        for labels, counts in out[stable]:
            assert np.array_equal(labels, ref_labels)
            assert np.array_equal(counts, ref_counts)
