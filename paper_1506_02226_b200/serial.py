"""The reference's float64 semantic oracle `serial_dbscan` (pkg/src/densescan/oracle.py:
29-111), run on the device (csrc/ds_serial.cu through ds_serial_dbscan).

The reference uses it as the CLI's `--variant serial` and as the `bench` equivalence
gate (cli.py:94-122, 152-234). Same contract: float64 direct-formula squared
distances, `<= eps_sq` in float64, counts incl. self, BFS components over core-core
pairs (= union-find components of the symmetric relation), borders to their
lowest-indexed in-range core, canonical labels; OracleTrace carries per-stage times
(device CUDA-event times here) and the core count.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _native
from .core import DbscanParams, Labeling, PointSet


@dataclass
class OracleTrace:
    """Per-stage times (ms) and the number of core points found (oracle.py:29-36)."""

    dist_sq_ms: float
    cluster_build_ms: float
    merge_ms: float
    core_count: int


def serial_dbscan(points: PointSet, params: DbscanParams, device=None):
    """float64 reference clustering on the GPU; returns (Labeling, OracleTrace)."""
    ctx = _native.context(device)
    labels, _, t = ctx.serial_dbscan(points.coords_aos, params.eps_sq, params.min_pts)
    return Labeling(labels), OracleTrace(dist_sq_ms=t.tile_ms, cluster_build_ms=t.fused_ms,
                                         merge_ms=t.merge_ms, core_count=int(t.core_count))
