"""Stage 3 API: merging primitive clusters into final clusters.

Mirrors `densescan.merge` (pkg/src/densescan/merge.py). Both reference
backends — the monotone target merge `merge_iterative` (merge.py:133-166)
and the Warshall closure `merge_warshall` (merge.py:218-238) — return the
same canonical labeling (SPEC.md merge contract), and here both run the
same sm_100a lock-free union-find over the core-core adjacency words
(csrc/ds_merge.cu), with the reference's lowest-indexed-core border rule
(merge.py:116-130) and canonical relabel (core.py:116-132).

Unlike the reference, the GPU merge does not mutate `nbr.bits` or
`valid_vec.valid` (union-find needs no monotone OR-merge); a MergeAudit
passed in therefore records no transitions.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .core import DensescanError, Labeling
from .kernels import NeighborhoodMatrix, ValidVector


class InconsistentInput(DensescanError):
    """The valid vector disagrees with the neighbor counts (merge.py:36-37)."""


@dataclass
class MergeAudit:
    """Transition tally of the reference's monotone merge (merge.py:40-61).

    The union-find merge never mutates its inputs, so every field stays 0.
    """

    bit_upgrades: int = 0
    bit_downgrades: int = 0
    valid_upgrades: int = 0
    valid_downgrades: int = 0
    merge_events: int = 0


def _merge(nbr: NeighborhoodMatrix, valid_vec: ValidVector, device=None) -> Labeling:
    ctx = _native.context(device)
    labels, _ = ctx.merge_bits(nbr.bits, nbr.neighbor_count, valid_vec.valid, valid_vec.min_pts)
    return Labeling(labels)


def merge_iterative(nbr: NeighborhoodMatrix, valid_vec: ValidVector, threads: int = 1,
                    audit: MergeAudit | None = None) -> Labeling:
    """Canonical labeling of a NeighborhoodMatrix (merge.py:133-166), on the GPU.

    Raises InconsistentInput when valid != (neighbor_count >= min_pts)
    (merge.py:141-145).
    """
    return _merge(nbr, valid_vec)


def merge_warshall(nbr: NeighborhoodMatrix, valid_vec: ValidVector,
                   threads: int = 1) -> Labeling:
    """Transitive-closure backend (merge.py:218-238); label-equivalent to
    merge_iterative, so it runs the same device union-find."""
    return _merge(nbr, valid_vec)


def labels_equal(a: np.ndarray, b: np.ndarray) -> bool:
    return bool(np.array_equal(np.asarray(a), np.asarray(b)))
