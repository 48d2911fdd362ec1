"""Host-side API of the drop-in (no GPU needed): the reference's validation,
error types, containers and helpers behave as in pkg/src/densescan."""

from __future__ import annotations

import math

import numpy as np
import pytest

import paper_1506_02226_b200 as ds
from paper_1506_02226_b200 import datasets


class TestParams:
    def test_squares_eps(self):
        p = ds.validate_params(1.5, 4)
        assert (p.eps, p.eps_sq, p.min_pts) == (1.5, 2.25, 4)

    @pytest.mark.parametrize("eps", [0.0, -1.0, math.inf, math.nan, "1", None, False,
                                     np.float32(0.3), np.int64(1)])
    def test_rejects_bad_eps(self, eps):
        with pytest.raises(ds.InvalidParams) as exc:
            ds.validate_params(eps, 4)
        assert exc.value.field == "eps"

    @pytest.mark.parametrize("min_pts", [0, -3, 2.5, "4", False, np.float64(4.0)])
    def test_rejects_bad_min_pts(self, min_pts):
        with pytest.raises(ds.InvalidParams) as exc:
            ds.validate_params(1.0, min_pts)
        assert exc.value.field == "min_pts"

    def test_matches_reference_outcomes(self):
        """Every (type, value) case of tests/golden/params.json (made by running the
        reference's validate_params / PipelineConfig, core.py:86-93, pipeline.py:39-41):
        same accepted values, same rejected field."""
        import json
        import os
        import sys
        sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
        from make_golden_params import make
        with open(os.path.join(os.path.dirname(__file__), "golden", "params.json")) as fh:
            rows = json.load(fh)
        assert len(rows) >= 40

        def run(fn):
            try:
                return {"ok": fn()}
            except Exception as e:  # noqa: BLE001
                return {"error": type(e).__name__, "field": getattr(e, "field", None)}

        for row in rows:
            x = make(row["kind"], row["value"])
            got_eps = run(lambda: list(map(float, ds.validate_params(x, 4).__dict__.values())))
            got_pts = run(lambda: list(map(float, ds.validate_params(1.0, x).__dict__.values())))
            got_thr = run(lambda: int(ds.PipelineConfig(
                variant=ds.KernelVariant(ds.VariantId.FUSED), threads=x).threads))
            assert got_eps == row["eps"], (row["kind"], row["value"])
            assert got_pts == row["min_pts"], (row["kind"], row["value"])
            assert got_thr == row["threads"], (row["kind"], row["value"])

    def test_bool_and_float64_accepted_like_reference(self):
        assert ds.validate_params(True, 4).eps == 1.0
        assert ds.validate_params(1.0, True).min_pts == 1
        assert ds.validate_params(np.float64(0.3), np.int64(8)).min_pts == 8

    def test_threshold_is_float32_of_float64_square(self):
        # core.py:93 + kernels.py:355: eps^2 in float64, then narrowed
        p = ds.validate_params(0.1, 3)
        assert p.eps_sq_f32 == np.float32(0.1 * 0.1)
        assert p.eps_sq_f32 != np.float32(0.1) * np.float32(0.1)


class TestPointSet:
    def test_any_dimension_and_mirror(self, rng):
        for d in (1, 2, 3, 16):
            c = rng.normal(size=(7, d))
            p = ds.PointSet(c)
            assert (p.n, p.d) == (7, d)
            assert np.array_equal(p.coords_aos, p.coords_soa.T)

    def test_frozen(self, rng):
        p = ds.PointSet(rng.normal(size=(4, 3)))
        with pytest.raises(ValueError):
            p.coords_aos[0, 0] = 1.0

    @pytest.mark.parametrize("bad", [np.zeros((0, 3)), np.zeros(3), np.zeros((2, 65)),
                                     np.array([[0.0, np.nan]]), np.array([[np.inf, 0.0]])])
    def test_rejects(self, bad):
        with pytest.raises(ValueError):
            ds.PointSet(bad)


class TestVariants:
    def test_defaults_and_validation(self):
        v = ds.KernelVariant(ds.VariantId.TILED)
        assert (v.tile_size, v.unroll_width) == (256, 32)
        with pytest.raises(ds.InvalidParams):
            ds.KernelVariant(ds.VariantId.TILED, tile_size=8, unroll_width=16)
        with pytest.raises(ds.InvalidParams):
            ds.KernelVariant(ds.VariantId.TILED, tile_size=8, unroll_width=0)

    def test_formula_mapping(self):
        # FUSED_ALGEBRAIC -> algebraic; every other rung computes the direct values
        assert ds.KernelVariant(ds.VariantId.FUSED_ALGEBRAIC).formula == 1
        for vid in ds.VariantId:
            if vid is not ds.VariantId.FUSED_ALGEBRAIC:
                assert ds.KernelVariant(vid).formula == 0

    def test_dispatch_guards(self, rng):
        pts = ds.PointSet(rng.normal(size=(4, 3)))
        params = ds.validate_params(1.0, 2)
        with pytest.raises(ValueError):
            ds.fused_build(pts, params, ds.KernelVariant(ds.VariantId.TILED))
        with pytest.raises(ValueError):
            ds.fused_build_algebraic(pts, params, ds.KernelVariant(ds.VariantId.FUSED))

    def test_flop_counts(self):
        assert ds.flop_count(ds.FlopFormula.DIRECT) == 8
        assert ds.flop_count(ds.FlopFormula.ALGEBRAIC_INNER) == 6


class TestCapacity:
    def test_resolve_mem_cap(self, monkeypatch):
        monkeypatch.delenv(ds.MEM_CAP_ENV_VAR, raising=False)
        assert ds.resolve_mem_cap() == ds.DEFAULT_MEM_CAP == 4 * 1024**3
        monkeypatch.setenv(ds.MEM_CAP_ENV_VAR, "12345")
        assert ds.resolve_mem_cap() == 12345
        assert ds.resolve_mem_cap(7) == 7

    def test_fused_build_guard_before_device(self, rng):
        # the exported matrix needs n * ceil(n/8) bytes (kernels.py:318); the guard
        # fires on the host before any device call, with the reference's numbers
        pts = ds.PointSet(rng.normal(size=(1000, 3)))
        with pytest.raises(ds.CapacityExceeded) as exc:
            ds.fused_build(pts, ds.validate_params(0.5, 3), ds.KernelVariant(ds.VariantId.FUSED),
                           mem_cap=100_000)
        assert exc.value.required_bytes == 125_000 and exc.value.cap_bytes == 100_000

    def test_materialising_rungs_guard(self, rng):
        pts = ds.PointSet(rng.normal(size=(1000, 3)))
        cfg = ds.PipelineConfig(variant=ds.KernelVariant(ds.VariantId.SOA), mem_cap=1_000_000)
        with pytest.raises(ds.CapacityExceeded) as exc:
            ds.run_dbscan(pts, ds.validate_params(0.5, 3), cfg)
        assert exc.value.required_bytes == 4_000_000


class TestPipelineTypes:
    def test_default_config(self):
        c = ds.default_config()
        assert c.variant.id is ds.VariantId.FUSED_ALGEBRAIC
        assert c.merge_backend is ds.MergeBackend.ITERATIVE
        assert c.threads >= 1

    def test_threads_validation(self):
        with pytest.raises(ValueError):
            ds.PipelineConfig(variant=ds.KernelVariant(ds.VariantId.FUSED), threads=0)

    def test_labelings(self):
        L = ds.Labeling
        assert ds.labelings_equivalent(L(np.array([0, 0, 1])), L(np.array([5, 5, 2])))
        assert not ds.labelings_equivalent(L(np.array([0, 0, 1])), L(np.array([0, 1, 1])))
        assert not ds.labelings_equivalent(L(np.array([-1, 0])), L(np.array([0, -1])))
        with pytest.raises(ds.LengthMismatch):
            ds.labelings_equivalent(L(np.array([0])), L(np.array([0, 1])))
        assert ds.first_difference(L(np.array([0, 0, 1, -1])), L(np.array([7, 7, 7, -1]))) == 2

    def test_canonicalize(self):
        c = ds.canonicalize
        assert list(c(ds.Labeling(np.array([7, 7, 3, -1]))).labels) == [0, 0, 1, -1]
        assert list(c(ds.Labeling(np.array([-1, -1]))).labels) == [-1, -1]
        assert list(c(ds.Labeling(np.array([2, 1, 2]))).labels) == [0, 1, 0]
        x = ds.Labeling(np.array([4, -1, 9, 4, 2, 9]))
        assert np.array_equal(c(c(x)).labels, c(x).labels)

    def test_timings_kernel_ms(self):
        t = ds.StageTimings(dist_ms=1.0, cluster_ms=2.0)
        assert t.kernel_ms() == 3.0
        assert ds.StageTimings(fused_ms=4.0).kernel_ms() == 4.0


class TestIO:
    def test_round_trip(self, tmp_path, rng):
        pts = ds.PointSet(rng.normal(size=(20, 2)) * 1e3)
        path = tmp_path / "p.txt"
        ds.write_points(pts, path)
        back = ds.load_points(path)
        assert np.array_equal(back.coords_aos, pts.coords_aos)

    def test_parse_errors(self, tmp_path):
        f = tmp_path / "bad.txt"
        f.write_text("0 0 0\n1 2\n")
        with pytest.raises(ds.ParseError) as exc:
            ds.load_points(f)
        assert exc.value.line_no == 2
        f.write_text("# only a comment\n")
        with pytest.raises(ds.EmptyDataset):
            ds.load_points(f)

    def test_labels_file(self, tmp_path):
        path = tmp_path / "l.txt"
        ds.write_labels(ds.Labeling(np.array([0, 0, -1])), path)
        assert path.read_text() == "0\n0\n-1\n"


class TestDatasets:
    def test_deterministic(self):
        a = ds.generate_blobs(500, 3, 0.1, 0.1, 7, 2).coords_aos
        b = ds.generate_blobs(500, 3, 0.1, 0.1, 7, 2).coords_aos
        assert np.array_equal(a, b)

    def test_configs(self):
        assert set(ds.CONFIGS) == {"C1", "C2", "C3", "C4", "C5"}
        c1 = ds.CONFIGS["C1"].points()
        assert (c1.n, c1.d) == (10_000, 2)
        assert ds.CONFIGS["C4"].d == 16

    def test_chain_generator_shape(self):
        p = datasets.generate_chain(n_chain=2000, n_blob_each=100, n_blobs=2, n_noise=50, seed=1)
        assert p.n == 2250 and p.d == 2
        assert p.coords_aos[:, 0].min() > -6 and p.coords_aos[:, 0].max() < 106
