"""GPU parity: the sm_100a path against the reference's golden outputs and the oracle.

Bar: bit-exact. Neighbourhood bits, int64 counts and canonical
labels must be identical to what the reference package computes with the same
formula (FUSED_ALGEBRAIC -> algebraic, FUSED -> direct), including exact ties,
large offsets where the two formulas disagree, ragged tile edges and
unfiltered eps.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import golden_cases, load_golden, pad3, random_specs

pytestmark = pytest.mark.gpu

FORMULAS = {"alg": 1, "dir": 0}


@pytest.fixture(scope="module")
def ds():
    import paper_1506_02226_b200 as pkg
    from paper_1506_02226_b200 import _native
    _native.load_library()
    return pkg


@pytest.fixture(scope="module")
def oracle():
    from oracle import densescan_oracle
    return densescan_oracle


def variant(ds, fname):
    vid = ds.VariantId.FUSED_ALGEBRAIC if fname == "alg" else ds.VariantId.FUSED
    return ds.KernelVariant(vid)


def gpu_stage12(ds, coords, eps, eps_sq, min_pts, fname, want_bits=True):
    ctx = ds._native.context()
    bits, counts, valid, _ = ctx.fused_build(coords, eps_sq, min_pts, FORMULAS[fname], 0,
                                             want_bits=want_bits)
    return bits, counts, valid


def gpu_labels(ds, coords, eps, eps_sq, min_pts, fname):
    params = ds.DbscanParams(eps=eps, eps_sq=eps_sq, min_pts=min_pts)
    cfg = ds.PipelineConfig(variant=variant(ds, fname))
    labeling, _ = ds.run_dbscan(ds.PointSet(coords), params, cfg)
    return labeling.labels


def sha(bits):
    return hashlib.sha256(np.ascontiguousarray(bits).tobytes()).hexdigest()


# ---- reference golden vectors ------------------------------------------------------
def test_kat_cases(ds):
    g = load_golden("kat.npz")
    for name, pts, eps, eps_sq, min_pts in golden_cases(g):
        for fname in FORMULAS:
            bits, counts, valid = gpu_stage12(ds, pts, eps, eps_sq, min_pts, fname)
            assert sha(bits) == str(g[f"{name}/{fname}/bits_sha"]), (name, fname)
            assert np.array_equal(counts, g[f"{name}/{fname}/counts"]), (name, fname)
            labels = gpu_labels(ds, pts, eps, eps_sq, min_pts, fname)
            assert np.array_equal(labels, g[f"{name}/{fname}/labels"]), (name, fname)


@pytest.mark.parametrize("native_2d", [True, False])
def test_c1_full(ds, native_2d):
    g = load_golden("c1.npz")
    pts = ds.generate_blobs(10_000, 4, 0.5, 0.0, 1, 2).coords_aos
    if not native_2d:
        pts = pad3(pts)
    for fname in FORMULAS:
        bits, counts, _ = gpu_stage12(ds, pts, 0.3, 0.3 * 0.3, 4, fname)
        assert np.array_equal(bits[:64], g[f"{fname}/bits_rows0_64"])
        assert sha(bits) == str(g[f"{fname}/bits_sha"])
        assert np.array_equal(counts, g[f"{fname}/counts"])
        labels = gpu_labels(ds, pts, 0.3, 0.3 * 0.3, 4, fname)
        assert np.array_equal(labels, g[f"{fname}/labels"])


@pytest.mark.parametrize("fixture", ["lattice.npz", "random.npz"])
def test_boundary_dense_and_random(ds, fixture):
    g = load_golden(fixture)
    cases = golden_cases(g) if fixture == "lattice.npz" else random_specs(g)
    seen = 0
    for name, pts, eps, eps_sq, min_pts in cases:
        for fname in FORMULAS:
            bits, counts, _ = gpu_stage12(ds, pts, eps, eps_sq, min_pts, fname)
            assert sha(bits) == str(g[f"{name}/{fname}/bits_sha"]), (fixture, name, fname)
            assert np.array_equal(counts, g[f"{name}/{fname}/counts"]), (name, fname)
            labels = gpu_labels(ds, pts, eps, eps_sq, min_pts, fname)
            assert np.array_equal(labels, g[f"{name}/{fname}/labels"]), (name, fname)
        seen += 1
    assert seen > 0


def test_blob23040(ds):
    g = load_golden("blob23040.npz")
    pts = ds.generate_blobs(23040, 3, 0.03, 0.02, 1).coords_aos
    for fname in FORMULAS:
        _, counts, _ = gpu_stage12(ds, pts, 0.1, 0.01, 8, fname, want_bits=False)
        assert np.array_equal(counts, g[f"{fname}/counts"])
        labels = gpu_labels(ds, pts, 0.1, 0.1 * 0.1, 8, fname)
        assert np.array_equal(labels, g[f"{fname}/labels"])


def test_c2_full_reference_labels(ds):
    g = load_golden("c2.npz")
    cfg = ds.CONFIGS["C2"]
    pts = cfg.points()
    params = ds.validate_params(cfg.eps, cfg.min_pts)
    labeling, _ = ds.run_dbscan(pts, params, ds.default_config())
    assert np.array_equal(labeling.labels, g["labels"])
    _, counts, _ = gpu_stage12(ds, pts.coords_aos, cfg.eps, params.eps_sq, cfg.min_pts, "alg",
                               want_bits=False)
    assert np.array_equal(counts, g["counts"])


# ---- oracle comparisons beyond the reference's reach ---------------------------------
@pytest.mark.parametrize("d", [1, 2, 3, 5, 8, 13, 16, 17, 33])
@pytest.mark.parametrize("fname", ["alg", "dir"])
def test_oracle_any_dimension(ds, oracle, rng, d, fname):
    for n in (1, 2, 31, 511, 512, 513, 1500):
        k = int(rng.integers(1, min(4, n) + 1))
        pts = ds.generate_blobs(n, k, 0.3, 0.2, int(rng.integers(2**31)), d).coords_aos
        pts = pts * rng.choice([1.0, 7.0]) + rng.choice([0.0, 50.0])
        eps = float(rng.uniform(0.2, 1.2)) * np.sqrt(d / 2.0)
        eps_sq = eps * eps
        min_pts = int(rng.integers(1, 10))
        bits, counts, _ = gpu_stage12(ds, pts, eps, eps_sq, min_pts, fname)
        obits, ocounts = oracle.neighborhood(pts, eps_sq, FORMULAS[fname])
        assert np.array_equal(bits, obits), (d, n, fname)
        assert np.array_equal(counts, ocounts), (d, n, fname)
        labels = gpu_labels(ds, pts, eps, eps_sq, min_pts, fname)
        want, _ = oracle.dbscan(pts, eps_sq, min_pts, FORMULAS[fname])
        assert np.array_equal(labels, want), (d, n, fname)


@pytest.mark.parametrize("d", [5, 8, 16, 24])
@pytest.mark.parametrize("fname", ["alg", "dir"])
def test_exact_products_signed_zeros_and_subnormals(ds, oracle, rng, d, fname):
    """d >= 5 forms every product as FFMA2(a, b, -0): signed zeros,
    float32 subnormals and products that underflow must give the FMUL bits exactly."""
    n = 700
    vals = np.array([0.0, -0.0, 1e-39, -1e-39, 3e-42, 1e-20, -1e-20, 1e-19, 0.5, -0.25],
                    dtype=np.float64)
    pts = rng.choice(vals, size=(n, d))
    pts[: n // 2] += rng.normal(0.0, 1e-19, size=(n // 2, d))  # tiny spread: squares underflow
    for eps in (1e-19, 3e-19, 0.3):
        eps_sq = eps * eps
        bits, counts, _ = gpu_stage12(ds, pts, eps, eps_sq, 2, fname)
        obits, ocounts = oracle.neighborhood(pts, eps_sq, FORMULAS[fname])
        assert np.array_equal(bits, obits), (d, eps, fname)
        assert np.array_equal(counts, ocounts), (d, eps, fname)
        labels = gpu_labels(ds, pts, eps, eps_sq, 2, fname)
        want, _ = oracle.dbscan(pts, eps_sq, 2, FORMULAS[fname])
        assert np.array_equal(labels, want), (d, eps, fname)


def test_padding_is_bit_neutral(ds):
    pts = ds.generate_blobs(3000, 5, 0.4, 0.1, 11, 2).coords_aos
    for fname in FORMULAS:
        a = gpu_labels(ds, pts, 0.25, 0.0625, 5, fname)
        b = gpu_labels(ds, pad3(pts), 0.25, 0.0625, 5, fname)
        assert np.array_equal(a, b)


def test_overflow_range_uses_exact_compare(ds, oracle, rng):
    # squares overflow float32: the NaN/inf semantics must follow numpy's
    pts = rng.normal(size=(700, 2)) * 1e19
    pts[:5] = rng.normal(size=(5, 2))
    for fname in FORMULAS:
        eps_sq = 1e38
        bits, counts, _ = gpu_stage12(ds, pts, 1e19, eps_sq, 2, fname)
        obits, ocounts = oracle.neighborhood(pts, eps_sq, FORMULAS[fname])
        assert np.array_equal(bits, obits)
        assert np.array_equal(counts, ocounts)


def test_merge_from_reference_bits(ds, oracle, rng):
    g = load_golden("kat.npz")
    for name, pts, eps, eps_sq, min_pts in golden_cases(g):
        key = f"{name}/alg/bits"
        if key not in g:
            continue
        bits = g[key]
        counts = g[f"{name}/alg/counts"].astype(np.int64)
        nbr = ds.NeighborhoodMatrix(n=counts.size, bits=bits, neighbor_count=counts)
        valid = ds.ValidVector(valid=counts >= min_pts, min_pts=min_pts)
        assert np.array_equal(ds.merge_iterative(nbr, valid).labels, g[f"{name}/alg/labels"])
        assert np.array_equal(ds.merge_warshall(nbr, valid).labels, g[f"{name}/alg/labels"])
    pts = ds.generate_blobs(2000, 3, 0.1, 0.2, 3, 2)
    params = ds.validate_params(0.05, 4)
    nbr, valid = ds.fused_build_algebraic(pts, params,
                                          ds.KernelVariant(ds.VariantId.FUSED_ALGEBRAIC))
    want, _ = oracle.dbscan(pts.coords_aos, params.eps_sq, 4, 1)
    assert np.array_equal(ds.merge_iterative(nbr, valid).labels, want)
    valid.valid[0] = not valid.valid[0]
    with pytest.raises(ds.InconsistentInput):
        ds.merge_iterative(nbr, valid)


def test_determinism_and_permutation(ds, oracle, rng):
    pts = ds.generate_blobs(20_000, 9, 0.5, 0.1, 5, 2)
    params = ds.validate_params(0.12, 6)
    first, _ = ds.run_dbscan(pts, params, ds.default_config())
    for _ in range(3):
        again, _ = ds.run_dbscan(pts, params, ds.default_config())
        assert np.array_equal(first.labels, again.labels)
    # permuting the input permutes the core partition; border ties follow the new
    # index order (lowest in-range core), so compare those against the oracle
    perm = rng.permutation(pts.n)
    coords = pts.coords_aos[perm]
    permuted, _ = ds.run_dbscan(ds.PointSet(coords), params, ds.default_config())
    want, counts = oracle.dbscan(coords, params.eps_sq, 6, 1)
    assert np.array_equal(permuted.labels, want)
    core = counts >= 6
    a = ds.canonicalize(ds.Labeling(np.where(core, first.labels[perm], -1))).labels
    b = ds.canonicalize(ds.Labeling(np.where(core, permuted.labels, -1))).labels
    assert np.array_equal(a, b)


def test_capacity_regrow_and_error(ds):
    # a dense blob emits many words: a small cap must raise, a generous one regrows
    pts = ds.generate_blobs(6000, 1, 0.05, 0.0, 1, 2)
    params = ds.validate_params(0.5, 4)
    with pytest.raises(ds.CapacityExceeded) as exc:
        ds.run_dbscan(pts, params, ds.PipelineConfig(
            variant=ds.KernelVariant(ds.VariantId.FUSED_ALGEBRAIC), mem_cap=2_000_000))
    assert exc.value.cap_bytes == 2_000_000 and exc.value.required_bytes > 2_000_000
    labeling, t = ds.run_dbscan(pts, params, ds.default_config())
    assert labeling.cluster_count() == 1 and t.words_emitted > 0


@pytest.mark.parametrize("cull", [True, False])
@pytest.mark.parametrize("shards", [2, 3, 5])
def test_shard_stages_fold_to_reference_labels(ds, shards, cull):
    """The real device shard stages, run as `shards` virtual ranks on one GPU
    (one context each); the exchanges are done with torch ops exactly as the
    NCCL collectives would (sum, gather, min)."""
    import torch
    from paper_1506_02226_b200 import _native, distributed as D

    g = load_golden("c1.npz")
    pts = ds.generate_blobs(10_000, 4, 0.5, 0.0, 1, 2).coords_aos
    coords = torch.from_numpy(pts.copy()).cuda()
    n, d = pts.shape
    total = D.tile_items(n)
    ctxs = [_native.Context(0) for _ in range(shards)]
    counts = []
    for r, ctx in enumerate(ctxs):
        ctx.set_tile_cull(cull)  # every rank builds the same (ordered) item list
        c = torch.empty(n, dtype=torch.int32, device="cuda")
        ctx.shard_stage12(coords.data_ptr(), n, d, 0.09, 1, r, shards, 0, c.data_ptr())
        counts.append(c)
    total_counts = torch.stack(counts).sum(0).to(torch.int32)
    assert np.array_equal(total_counts.cpu().numpy(), g["alg/counts"])
    parents, bmins = [], []
    for ctx in ctxs:
        p = torch.empty(n, dtype=torch.int32, device="cuda")
        b = torch.empty(n, dtype=torch.int32, device="cuda")
        ctx.shard_stage3_local(total_counts.data_ptr(), n, 4, p.data_ptr(), b.data_ptr())
        parents.append(p)
        bmins.append(b)
    par = torch.stack(parents).contiguous()
    bmin = torch.stack(bmins).min(0).values.to(torch.int32).contiguous()
    labels = torch.empty(n, dtype=torch.int64, device="cuda")
    ctxs[0].shard_stage3_merge(total_counts.data_ptr(), n, 4, par.data_ptr(), shards,
                               bmin.data_ptr(), labels.data_ptr())
    assert np.array_equal(labels.cpu().numpy(), g["alg/labels"])
    for ctx in ctxs:
        ctx.close()


def _labels_counts(ds, coords, eps_sq, min_pts, formula, prune, order=True):
    ctx = ds._native.context()
    ctx.configure(prune, order)
    try:
        labels, counts, t = ctx.run_dbscan(coords, eps_sq, min_pts, formula, 0, want_counts=True)
    finally:
        ctx.configure(True, True)
    return labels, counts, t


def test_tile_culling_is_exact(ds, oracle, rng):
    """Culled and dense schedules give identical counts and labels, including
    tile pairs right at the eps boundary and far-from-origin data where the
    algebraic rounding error exceeds eps^2."""
    cases = []
    # blobs exactly eps apart across tile boundaries (direct: exact lattice arithmetic)
    a = np.stack(np.meshgrid(np.arange(23.0), np.arange(23.0)), -1).reshape(-1, 2)[:512]
    cases.append((np.concatenate([a, a + [30.0, 0.0], a + [52.0, 0.0]]), 64.0, 3))
    # same far from the origin, in the algebraic cancellation regime
    cases.append((np.concatenate([a, a + [22.5, 0.0]]) * 0.02 + 1000.0, 0.0004, 3))
    cases.append((rng.normal(size=(3000, 2)) * 0.05 + [[700.0, -300.0]], 0.0009, 4))
    # blob-ordered data where most tile pairs are culled
    cases.append((ds.generate_blobs(12_000, 9, 0.3, 0.05, 3, 2).coords_aos, 0.01, 5))
    cases.append((ds.generate_blobs(6_000, 5, 0.2, 0.0, 8, 16).coords_aos * 3.0, 0.5, 5))
    for coords, eps_sq, mp in cases:
        for f in (0, 1):
            lc, cc, tc = _labels_counts(ds, coords, eps_sq, mp, f, True)
            ld, cd, td = _labels_counts(ds, coords, eps_sq, mp, f, False, False)
            assert np.array_equal(cc, cd) and np.array_equal(lc, ld)
            want, wc = oracle.dbscan(coords, eps_sq, mp, f)
            assert np.array_equal(cc, wc) and np.array_equal(lc, want)
            assert tc.pairs_evaluated <= td.pairs_evaluated


def test_culling_skips_work_on_c2(ds):
    cfg = ds.CONFIGS["C2"]
    pts = cfg.points()
    params = ds.validate_params(cfg.eps, cfg.min_pts)
    _, t_cull = ds.run_dbscan(pts, params, ds.default_config())
    dense_cfg = ds.default_config()
    dense_cfg.prune = False
    lab_dense, t_dense = ds.run_dbscan(pts, params, dense_cfg)
    assert np.array_equal(lab_dense.labels, load_golden("c2.npz")["labels"])
    assert t_cull.pairs_evaluated < 0.5 * t_dense.pairs_evaluated


@pytest.mark.parametrize("prune,order", [(True, True), (True, False), (False, True),
                                         (False, False)])
def test_schedules_shuffled_input(ds, oracle, rng, prune, order):
    """Random input order (worst case for tiles) and border points shared by
    several clusters: the lowest-ORIGINAL-index core rule must survive the
    spatial permutation."""
    base = ds.generate_blobs(4000, 6, 0.25, 0.15, 17, 2).coords_aos
    coords = base[rng.permutation(base.shape[0])]
    # bridges of sparse points between blobs create multi-cluster border points
    bridge = np.stack([np.linspace(0, 5.0, 60), np.zeros(60)], 1)
    coords = np.concatenate([coords, bridge])[rng.permutation(coords.shape[0] + 60)]
    for f in (0, 1):
        labels, counts, _ = _labels_counts(ds, coords, 0.03, 6, f, prune, order)
        want, wc = oracle.dbscan(coords, 0.03, 6, f)
        assert np.array_equal(counts, wc) and np.array_equal(labels, want)
        nbr, valid = ds.fused_build_algebraic(ds.PointSet(coords), ds.validate_params(
            np.sqrt(0.03), 6), ds.KernelVariant(ds.VariantId.FUSED_ALGEBRAIC))
        obits, _ = oracle.neighborhood(coords, np.sqrt(0.03) ** 2, 1)
        assert np.array_equal(nbr.bits, obits)


def test_full_size_configs_schedule_invariance(ds):
    """C3 (1M) and C5 (2M, chain + dense blobs): the default schedule (spatial
    order + culling + sub-tile skipping) equals the paper's dense schedule, and
    repeated runs are identical. (Oracle parity at C3/C4 full size is recorded in
    DESIGN.md §5 from tools/run_configs.py: the C oracle needs minutes.)"""
    for name in ("C3", "C5"):
        cfg = ds.CONFIGS[name]
        pts = cfg.points()
        params = ds.validate_params(cfg.eps, cfg.min_pts)
        fast = ds.default_config()
        fast.mem_cap = 64 * 1024**3
        a, ta = ds.run_dbscan(pts, params, fast)
        b, _ = ds.run_dbscan(pts, params, fast)
        assert np.array_equal(a.labels, b.labels)
        dense = ds.default_config()
        dense.mem_cap = 64 * 1024**3
        dense.prune = False
        dense.spatial_order = False
        c, tc = ds.run_dbscan(pts, params, dense)
        assert np.array_equal(a.labels, c.labels), name
        assert ta.pairs_evaluated < 0.05 * tc.pairs_evaluated


def test_c4_shape_against_oracle(ds):
    """16-D blobs (C4's generator at 60k points): parity with the C oracle."""
    from oracle import c_oracle
    pts = ds.generate_blobs(60_000, 8, 0.5, 0.0, 4, 16)
    params = ds.validate_params(1.6, 8)
    labeling, _ = ds.run_dbscan(pts, params, ds.default_config())
    want, wc = c_oracle.dbscan(pts.coords_aos, params.eps_sq, 8, 1)
    assert np.array_equal(labeling.labels, want)
    ctx = ds._native.context()
    _, counts, _ = ctx.run_dbscan(pts.coords_aos, params.eps_sq, 8, 1, 0, want_counts=True)
    assert np.array_equal(counts, wc)


def test_graph_replay_with_new_data(ds, oracle):
    """Call 1 runs eagerly, call 2 records the CUDA graph, later calls replay it:
    replays on different data of the same shape must still be exact, and a
    word-buffer overflow on a denser input must fall back and stay exact."""
    ctx = ds._native.context()
    params = ds.validate_params(0.2, 5)
    sets = [ds.generate_blobs(6000, 5, 0.3, 0.1, s, 2).coords_aos for s in (1, 1, 2, 3)]
    sets.append(ds.generate_blobs(6000, 1, 0.05, 0.0, 4, 2).coords_aos)  # far denser
    for coords in sets + sets[:2]:
        labels, counts, t = ctx.run_dbscan(coords, params.eps_sq, 5, 1, 0, want_counts=True)
        want, wc = oracle.dbscan(coords, params.eps_sq, 5, 1)
        assert np.array_equal(counts, wc) and np.array_equal(labels, want)
    ctx.set_cuda_graph(False)
    labels, _, _ = ctx.run_dbscan(sets[2], params.eps_sq, 5, 1, 0)
    ctx.set_cuda_graph(True)
    assert np.array_equal(labels, oracle.dbscan(sets[2], params.eps_sq, 5, 1)[0])


def test_public_api_graph_replay_repoints_host_buffers(ds, oracle):
    """run_dbscan through the public API: page-locked PointSet coordinates and label
    buffers, so from the second call on the label copy is a recorded graph node that
    is re-pointed at every call's fresh buffer; alternate data sets of one shape."""
    params = ds.validate_params(0.2, 5)
    sets = [ds.generate_blobs(7000, 4, 0.3, 0.1, s, 2) for s in (11, 12, 13)]
    conf = ds.default_config()
    for rnd in range(3):
        for pts in sets:
            labeling, _ = ds.run_dbscan(pts, params, conf)
            want, _ = oracle.dbscan(pts.coords_aos, params.eps_sq, 5, 1)
            assert np.array_equal(labeling.labels, want), rnd


def _degenerate_cases(rng):
    """(name, coords, eps, min_pts): inputs that stress the spatial order, the
    culling bounds and the merge rather than the formula."""
    line = np.zeros((3000, 3))
    line[:, 0] = np.arange(3000) * 0.5  # spacing == eps: every neighbour an exact tie
    far = rng.normal(0, 1e-3, (6000, 3)) + np.array([1.5e4, -2.5e4, 7e3])
    far[::7] += rng.normal(0, 0.05, (len(far[::7]), 3))
    same = np.full((5000, 3), 3.25)
    same_out = same.copy()
    same_out[:4] = [[1e3, 0, 0], [-1e3, 5, 5], [0, 2e3, 0], [3.25, 3.25, 3.26]]
    grid = np.array([[x, y, 0.0] for x in range(80) for y in range(80)], dtype=float) * 0.1
    return [
        ("identical", same, 1e-3, 10),
        ("identical_outliers", same_out, 0.02, 10),
        ("line_ties", line, 0.5, 3),
        ("far_offset", far, 4e-3, 5),  # |x| ~ 2.5e4: the algebraic form cancels badly
        ("grid_ties", grid, 0.1, 5),
        ("all_noise", rng.uniform(0, 1, (4000, 3)), 0.05, 10_000),
        ("one_cluster", rng.uniform(0, 1, (4000, 3)), 10.0, 2),
    ]


def test_degenerate_inputs_against_oracle(ds, rng):
    """Identical points (zero-span bounding box, one Morton cell), exact ties on a line
    and a grid, a tiny cluster far from the origin, MinPts above n and eps above the
    diameter: labels and counts equal the C oracle's for both formulas, with the
    default (sorted, culled) and the dense schedule."""
    from oracle import c_oracle
    ctx = ds._native.context()
    for name, coords, eps, min_pts in _degenerate_cases(rng):
        params = ds.validate_params(eps, min_pts)
        for fname, formula in FORMULAS.items():
            want, wc = c_oracle.dbscan(coords, params.eps_sq, min_pts, formula)
            for prune in (True, False):
                ctx.configure(prune, prune)
                try:
                    labels, counts, _ = ctx.run_dbscan(coords, params.eps_sq, min_pts, formula,
                                                       0, want_counts=True)
                finally:
                    ctx.configure(True, True)
                assert np.array_equal(counts, wc), (name, fname, prune)
                assert np.array_equal(labels, want), (name, fname, prune)


def test_stage_timings_stamps_and_events(ds):
    """Stage times come from the kernels' %globaltimer stamps by default and from CUDA
    events with DS_OPT_EVENT_TIMING; both are positive, nested (tile <= stage 1+2) and
    leave the labels unchanged."""
    pts = ds.generate_blobs(30_000, 6, 0.4, 0.1, 9, 2)
    params = ds.validate_params(0.1, 5)
    ctx = ds._native.context()
    out = {}
    for ev in (False, True):
        ctx.set_event_timing(ev)
        try:
            for _ in range(3):  # eager, recorded, replayed
                labels, _, t = ctx.run_dbscan(pts.coords_aos, params.eps_sq, 5, 1, 0)
                assert 0 < t.tile_ms <= t.fused_ms and t.merge_ms > 0
                assert t.d2h_ms > 0 if ev else t.d2h_ms == 0  # copies timed with events only
                assert t.fused_ms + t.merge_ms < t.total_ms
        finally:
            ctx.set_event_timing(False)
        out[ev] = labels.copy()
    assert np.array_equal(out[False], out[True])
