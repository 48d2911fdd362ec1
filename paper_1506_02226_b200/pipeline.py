"""End-to-end clustering: the drop-in for `densescan.pipeline`.

`run_dbscan(points, params, config)` keeps the reference signature and
return value (pkg/src/densescan/pipeline.py:70-92): a canonical Labeling
and a StageTimings. Underneath, one C-ABI call (`ds_run_dbscan`) copies the
float64 points to the device, runs the three stages as sm_100a kernels and
copies the int64 labels back. There is no CPU path.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _native
from .core import DensescanError, DbscanParams, Labeling, PointSet, canonicalize
from .kernels import KernelVariant, VariantId, ensure_capacity, resolve_mem_cap


class LengthMismatch(DensescanError):
    """Two labelings of different lengths cannot be compared (pipeline.py:21-22)."""


class MergeBackend(Enum):
    ITERATIVE = "iterative"
    WARSHALL = "warshall"


@dataclass
class PipelineConfig:
    """Kernel rung, merge backend, workers and memory cap (pipeline.py:30-41).

    `threads` is validated as in the reference but the device ignores it.
    `device` picks the CUDA ordinal (None: $DENSESCAN_DEVICE or 0).
    `devices` (a sequence of ordinals, optional) shards one call over several
    devices inside this process — the stage-1 tile pairs are dealt to the shards,
    counts / border minima / union-find forests are exchanged device to device
    (distributed.run_dbscan_multi) — the device analogue of the reference's
    worker threads (`threads`, _parallel.py:24-39). Labels do not depend on it.
    `prune` skips tile pairs whose bounding boxes prove every pair out of range
    (with a float32 error margin) and `spatial_order` visits the points in
    Morton order so tiles are compact; results are bit-identical either way,
    and prune=False, spatial_order=False is the paper's dense all-pairs schedule.
    """

    variant: KernelVariant
    merge_backend: MergeBackend = MergeBackend.ITERATIVE
    threads: int = 1
    mem_cap: int | None = None
    device: int | None = None
    devices: tuple | list | None = None
    prune: bool = True
    spatial_order: bool = True

    def __post_init__(self):
        # the reference's predicate exactly (pipeline.py:39-41): bool is an int
        if not (isinstance(self.threads, (int, np.integer)) and self.threads >= 1):
            raise ValueError(f"threads must be an integer >= 1, got {self.threads!r}")


def default_config() -> PipelineConfig:
    """FUSED_ALGEBRAIC + ITERATIVE + all host workers (pipeline.py:44-49)."""
    return PipelineConfig(variant=KernelVariant(VariantId.FUSED_ALGEBRAIC),
                          merge_backend=MergeBackend.ITERATIVE,
                          threads=os.cpu_count() or 1)


@dataclass
class StageTimings:
    """Per-stage times in ms (pipeline.py:52-67) plus device counters.

    dist/cluster are None for the fused rungs, fused_ms None otherwise; stage
    times are device times of the device work (%globaltimer stamps at kernel
    boundaries), total_ms the wall time of the whole call (host<->device copies
    included). h2d_ms is timed with CUDA events while the pipeline runs; d2h_ms
    only with event timing (DS_OPT_EVENT_TIMING), 0.0 otherwise.
    """

    dist_ms: float | None = None
    cluster_ms: float | None = None
    fused_ms: float | None = None
    merge_ms: float | None = None
    total_ms: float = 0.0
    tile_ms: float | None = None
    h2d_ms: float | None = None
    d2h_ms: float | None = None
    pairs_evaluated: int = 0
    tiles_total: int = 0
    tiles_nonempty: int = 0
    words_emitted: int = 0
    core_count: int = 0
    cluster_count: int = 0

    def kernel_ms(self) -> float:
        """Time spent producing the neighbourhood relation (stages 1+2)."""
        if self.fused_ms is not None:
            return self.fused_ms
        return (self.dist_ms or 0.0) + (self.cluster_ms or 0.0)


def _timings(t: "_native.Timings", variant: KernelVariant, total_ms: float) -> StageTimings:
    st = StageTimings(merge_ms=t.merge_ms, total_ms=total_ms, tile_ms=t.tile_ms,
                      h2d_ms=t.h2d_ms, d2h_ms=t.d2h_ms, pairs_evaluated=t.pairs_evaluated,
                      tiles_total=t.tiles_total, tiles_nonempty=t.tiles_nonempty,
                      words_emitted=t.words_emitted, core_count=t.core_count,
                      cluster_count=t.cluster_count)
    if variant.materializes_distance():
        st.dist_ms = t.tile_ms
        st.cluster_ms = max(t.fused_ms - t.tile_ms, 0.0)
    else:
        st.fused_ms = t.fused_ms
    return st


def run_dbscan(points: PointSet, params: DbscanParams, config: PipelineConfig):
    """Cluster `points`; returns (canonical Labeling, StageTimings).

    Raises CapacityExceeded when the device workspace would exceed the memory
    cap (config.mem_cap, else $DENSESCAN_MEM_CAP, else 4 GiB) and DeviceError
    on CUDA failures. The input PointSet is never mutated.
    """
    t0 = time.perf_counter()
    variant = config.variant
    mem_cap = resolve_mem_cap(config.mem_cap)
    if variant.materializes_distance():
        # the reference allocates the 4 n^2 float32 matrix for these rungs (kernels.py:156)
        ensure_capacity(4 * points.n * points.n, mem_cap)
    if config.devices is not None and len(config.devices) > 1:
        from .distributed import run_dbscan_multi
        labels, tm = run_dbscan_multi(points, params, config.devices, variant.formula, mem_cap,
                                      config.prune, config.spatial_order)
        st = StageTimings(fused_ms=tm.stage12_ms + tm.exchange1_ms,
                          merge_ms=tm.stage3_local_ms + tm.exchange2_ms + tm.stage3_merge_ms,
                          total_ms=(time.perf_counter() - t0) * 1e3, tile_ms=tm.tile_ms,
                          pairs_evaluated=tm.pairs_evaluated)
        return Labeling(labels), st
    ctx = _native.context(config.device if config.devices is None or not config.devices
                          else config.devices[0])
    ctx.configure(config.prune, config.spatial_order)
    _native.pin_frozen(points.coords_aos, points)
    labels, _, t = ctx.run_dbscan(points.coords_aos, params.eps_sq, params.min_pts,
                                  variant.formula, mem_cap)
    total = (time.perf_counter() - t0) * 1e3
    return Labeling(labels), _timings(t, variant, total)


def labelings_equivalent(a: Labeling, b: Labeling) -> bool:
    """Identical after canonicalization (pipeline.py:95-103)."""
    if a.n != b.n:
        raise LengthMismatch(f"labelings have lengths {a.n} and {b.n}")
    return bool(np.array_equal(canonicalize(a).labels, canonicalize(b).labels))


def first_difference(a: Labeling, b: Labeling) -> int | None:
    """Index of the first disagreement between canonical forms (pipeline.py:106-113)."""
    if a.n != b.n:
        raise LengthMismatch(f"labelings have lengths {a.n} and {b.n}")
    diff = np.nonzero(canonicalize(a).labels != canonicalize(b).labels)[0]
    return int(diff[0]) if diff.size else None
