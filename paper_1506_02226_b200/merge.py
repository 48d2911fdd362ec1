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
    (merge.py:141-145). `audit` is accepted for signature compatibility and left
    at zero: the union-find merge performs none of the monotone bit/valid
    transitions the reference's MergeAudit tallies (merge.py:40-61), and it does
    not mutate `nbr.bits` or `valid_vec.valid`.
    """
    return _merge(nbr, valid_vec)


@dataclass
class CoreAdjacency:
    """Core-to-core in-range relation, packbits rows (m x ceil(m/8)), with the map
    from core rank back to point index (merge.py:169-176)."""

    m: int
    core_indices: np.ndarray
    bits: np.ndarray


def build_core_adjacency(nbr: NeighborhoodMatrix, valid_vec: ValidVector,
                         device=None) -> CoreAdjacency:
    """The neighbourhood matrix restricted to core rows and columns (merge.py:179-188),
    gathered on the GPU (csrc/ds_closure.cu core_gather_kernel)."""
    ctx = _native.context(device)
    core_indices, adj, _ = ctx.core_adjacency(nbr.bits, valid_vec.valid)
    return CoreAdjacency(m=int(core_indices.size), core_indices=core_indices, bits=adj)


def warshall_closure(adj: CoreAdjacency, threads: int = 1, device=None) -> CoreAdjacency:
    """Transitive closure of the core relation (merge.py:191-215), on the GPU.

    The blocked Warshall recurrence (32 pivots per phase, csrc/ds_closure.cu)
    yields the same closure as the reference's pivot loop for any input relation;
    the input is not mutated. `threads` is accepted for signature compatibility.
    """
    ctx = _native.context(device)
    closed, _ = ctx.warshall_closure(adj.bits, adj.m)
    return CoreAdjacency(m=adj.m, core_indices=adj.core_indices.copy(), bits=closed)


def merge_warshall(nbr: NeighborhoodMatrix, valid_vec: ValidVector,
                   threads: int = 1) -> Labeling:
    """Transitive-closure backend (merge.py:218-238), label-equivalent to
    merge_iterative (SPEC merge contract).

    Like the reference it takes the core set from `valid_vec.valid` as given
    and never raises InconsistentInput. Its clusters are the connected components
    of the core relation, so it runs the device union-find over (bits AND core x
    core) instead of the O(m^3) closure (identical labels for the symmetric
    relation stage 1+2 produces; warshall_closure is available on its own).
    """
    ctx = _native.context()
    labels, _ = ctx.merge_bits_core(nbr.bits, np.asarray(valid_vec.valid, dtype=bool))
    return Labeling(labels)


def labels_equal(a: np.ndarray, b: np.ndarray) -> bool:
    return bool(np.array_equal(np.asarray(a), np.asarray(b)))
