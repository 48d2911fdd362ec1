"""Stage 1+2 API: kernel variants, the capacity guard, and the fused builds.

Mirrors the reference module `densescan.kernels` (pkg/src/densescan/
kernels.py): the same VariantId ladder, KernelVariant validation, result
containers and CapacityExceeded error. The computation runs in sm_100a
kernels; the variant selects the formula and whether the distance matrix is
materialised:

  FUSED_ALGEBRAIC                 -> eps-tile kernel (csrc/ds_tile.cu), algebraic
                                     T + P - (X*x + Y*y + ...)  (default)
  FUSED                           -> eps-tile kernel, direct ((dx^2 + dy^2) + ...)
  BASELINE, SOA, TILED,           -> the n x n float32 direct-formula matrix in HBM
  TILED_UNROLLED                     (csrc/ds_dist.cu), thresholded into bits; the
                                     four rungs compute exactly these values
                                     (kernels.py:21-25), so do dist_baseline /
                                     dist_soa / dist_tiled

`tile_size` / `unroll_width` are validated exactly as in the reference but,
as there, never change a result (the device tiling is fixed at 512).
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _native
from .core import DbscanParams, DensescanError, InvalidParams, PointSet

DEFAULT_MEM_CAP = 4 * 1024**3
MEM_CAP_ENV_VAR = "DENSESCAN_MEM_CAP"

# absolute eps^2 band (unit-scale data) inside which the algebraic rewrite may
# classify pairs differently from the direct formula (kernels.py:46-48)
ALGEBRAIC_MARGIN = 1e-2


class CapacityExceeded(DensescanError):
    """An allocation would exceed the configured memory cap (kernels.py:55-63)."""

    def __init__(self, required_bytes: int, cap_bytes: int):
        super().__init__(
            f"requires {required_bytes} bytes but the memory cap is {cap_bytes} bytes"
            f" (override with {MEM_CAP_ENV_VAR} or mem_cap=)")
        self.required_bytes = required_bytes
        self.cap_bytes = cap_bytes


def resolve_mem_cap(mem_cap=None) -> int:
    """Explicit argument, else the environment variable, else 4 GiB (kernels.py:66-73)."""
    if mem_cap is not None:
        return int(mem_cap)
    env = os.environ.get(MEM_CAP_ENV_VAR)
    if env is not None:
        return int(env)
    return DEFAULT_MEM_CAP


def ensure_capacity(required_bytes: int, mem_cap) -> None:
    cap = resolve_mem_cap(mem_cap)
    if required_bytes > cap:
        raise CapacityExceeded(required_bytes, cap)


class VariantId(Enum):
    BASELINE = "baseline"
    SOA = "soa"
    TILED = "tiled"
    TILED_UNROLLED = "tiled-unrolled"
    FUSED = "fused"
    FUSED_ALGEBRAIC = "fused-algebraic"


@dataclass(frozen=True)
class KernelVariant:
    """A rung of the kernel ladder plus its blocking parameters (kernels.py:91-109)."""

    id: VariantId
    tile_size: int = 256
    unroll_width: int = 32

    def __post_init__(self):
        if not (isinstance(self.unroll_width, (int, np.integer)) and self.unroll_width >= 1):
            raise InvalidParams("unroll_width",
                                f"must be an integer >= 1, got {self.unroll_width!r}")
        if not (isinstance(self.tile_size, (int, np.integer))
                and self.tile_size >= self.unroll_width):
            raise InvalidParams("tile_size",
                                f"must be an integer >= unroll_width, got {self.tile_size!r}")

    def materializes_distance(self) -> bool:
        return self.id in (VariantId.BASELINE, VariantId.SOA,
                           VariantId.TILED, VariantId.TILED_UNROLLED)

    @property
    def formula(self) -> int:
        """The pair formula this rung evaluates on the device."""
        return (_native.FORMULA_ALGEBRAIC if self.id is VariantId.FUSED_ALGEBRAIC
                else _native.FORMULA_DIRECT)


@dataclass
class DistSqMatrix:
    """Dense float32 matrix of pairwise squared Euclidean distances (kernels.py:113-118)."""

    n: int
    values: np.ndarray


@dataclass
class NeighborhoodMatrix:
    """Bit-packed boolean matrix, reference layout (kernels.py:120-137).

    bits: uint8 [n, ceil(n/8)], numpy packbits MSB-first rows;
    neighbor_count: int64 popcount per row (includes the point itself).
    """

    n: int
    bits: np.ndarray
    neighbor_count: np.ndarray

    def row(self, i: int) -> np.ndarray:
        return np.unpackbits(self.bits[i], count=self.n).view(bool)

    def to_bool(self) -> np.ndarray:
        return np.unpackbits(self.bits, axis=-1, count=self.n).view(bool)


@dataclass
class ValidVector:
    """valid[i] iff neighbor_count[i] >= min_pts (kernels.py:140-145)."""

    valid: np.ndarray
    min_pts: int


def row_bytes(n: int) -> int:
    return (n + 7) // 8


def _fused(points: PointSet, params: DbscanParams, formula: int, mem_cap, device=None):
    n = points.n
    # the exported matrix is n x ceil(n/8) host bytes, guarded like kernels.py:318
    ensure_capacity(n * row_bytes(n), mem_cap)
    ctx = _native.context(device)
    # the stage-level entry points always run the default (culled, spatially ordered)
    # schedule; the caller's options on this thread's shared context are restored
    previous = ctx.schedule()
    ctx.configure(True, True)
    try:
        bits, counts, valid, t = ctx.fused_build(points.coords_aos, params.eps_sq,
                                                 params.min_pts, formula, 0)
    finally:
        ctx.configure(*previous)
    return (NeighborhoodMatrix(n=n, bits=bits, neighbor_count=counts),
            ValidVector(valid=valid, min_pts=params.min_pts), t)


def fused_build(points: PointSet, params: DbscanParams, variant: KernelVariant,
                threads: int = 1, mem_cap=None):
    """Stage 1+2 with the direct formula (kernels.py:420-428), on the GPU.

    `threads` is accepted for signature compatibility; results never depend on it.
    """
    if variant.id is not VariantId.FUSED:
        raise ValueError(f"fused_build cannot run variant {variant.id.value}")
    nbr, valid, _ = _fused(points, params, _native.FORMULA_DIRECT, mem_cap)
    return nbr, valid


def fused_build_algebraic(points: PointSet, params: DbscanParams, variant: KernelVariant,
                          threads: int = 1, mem_cap=None):
    """Stage 1+2 with the hoisted algebraic rewrite (kernels.py:431-442), on the GPU."""
    if variant.id is not VariantId.FUSED_ALGEBRAIC:
        raise ValueError(f"fused_build_algebraic cannot run variant {variant.id.value}")
    nbr, valid, _ = _fused(points, params, _native.FORMULA_ALGEBRAIC, mem_cap)
    return nbr, valid


# ---- materialising ladder (kernels.py:153-308) -------------------------------------
# All four rungs compute the same direct-formula values (kernels.py:21-25): on the
# device they are one HBM-write-bound kernel (csrc/ds_dist.cu); the rungs differ
# only in the reference's CPU memory access pattern, which has no device analogue.

def _dist(points: PointSet, mem_cap, device=None) -> DistSqMatrix:
    n = points.n
    ensure_capacity(4 * n * n, mem_cap)  # kernels.py:156 / 262
    ctx = _native.context(device)
    values, _ = ctx.dist_matrix(points.coords_aos, 0)
    return DistSqMatrix(n=n, values=values)


def dist_baseline(points: PointSet, threads: int = 1, mem_cap=None) -> DistSqMatrix:
    """Ladder rung 0 (kernels.py:177-180): the direct-formula matrix, on the GPU."""
    return _dist(points, mem_cap)


def dist_soa(points: PointSet, threads: int = 1, mem_cap=None) -> DistSqMatrix:
    """Ladder rung 1 (kernels.py:183-185): identical values to dist_baseline."""
    return _dist(points, mem_cap)


def dist_tiled(points: PointSet, variant: KernelVariant, threads: int = 1,
               mem_cap=None) -> DistSqMatrix:
    """Ladder rungs 2-3 (kernels.py:251-281): identical values to dist_baseline."""
    if variant.id not in (VariantId.TILED, VariantId.TILED_UNROLLED):
        raise ValueError(f"dist_tiled cannot run variant {variant.id.value}")
    return _dist(points, mem_cap)


def build_clusters_from_dist(dist: DistSqMatrix, params: DbscanParams,
                             threads: int = 1, mem_cap=None):
    """Stage 2 from a materialised matrix (kernels.py:284-308), on the GPU:
    bit (i, j) iff values[i, j] <= float32(eps_sq); (NeighborhoodMatrix, ValidVector)."""
    n = dist.n
    ensure_capacity(n * row_bytes(n), mem_cap)  # kernels.py:293
    ctx = _native.context()
    bits, counts, valid, _ = ctx.dist_threshold(dist.values, params.eps_sq, params.min_pts, 0)
    return (NeighborhoodMatrix(n=n, bits=bits, neighbor_count=counts),
            ValidVector(valid=valid, min_pts=params.min_pts))


def run_variant(points: PointSet, params: DbscanParams, variant: KernelVariant,
                threads: int = 1, mem_cap=None):
    """One ladder rung to (NeighborhoodMatrix, ValidVector) plus stage times
    (kernels.py:445-470): (nbr, valid, dist_ms, cluster_ms, fused_ms).

    Device times from CUDA events. The materialising rungs build the float32
    matrix in HBM (ds_dist_build: dist_ms = distance kernel, cluster_ms =
    threshold kernel) and never copy it to the host; the fused rungs run the
    eps-tile kernel (fused_ms = stage 1+2).
    """
    if variant.materializes_distance():
        n = points.n
        ensure_capacity(4 * n * n, mem_cap)  # kernels.py:156 / 262
        ensure_capacity(n * row_bytes(n), mem_cap)  # kernels.py:293
        ctx = _native.context()
        bits, counts, valid, t = ctx.dist_build(points.coords_aos, params.eps_sq,
                                                params.min_pts, 0)
        return (NeighborhoodMatrix(n=n, bits=bits, neighbor_count=counts),
                ValidVector(valid=valid, min_pts=params.min_pts), t.tile_ms, t.merge_ms, None)
    nbr, valid, t = _fused(points, params, variant.formula, mem_cap)
    return nbr, valid, None, None, t.fused_ms


class FlopFormula(Enum):
    DIRECT = "direct"
    ALGEBRAIC_INNER = "algebraic-inner"


def flop_count(formula: FlopFormula, pair=((1.0, 2.0, 3.0), (4.0, 6.0, 3.0))) -> int:
    """Paper §V-B operation counts per 3-D inner-loop evaluation (kernels.py:512-544):
    DIRECT 8 (3 sub, 3 mul, 2 add), ALGEBRAIC_INNER 6 (T+P hoisted).

    Counted by evaluating the formula with an op-counting scalar.
    """
    ops = [0]

    class _C:
        __slots__ = ("v",)

        def __init__(self, v):
            self.v = v

        def _op(self, other, f):
            ops[0] += 1
            return _C(f(self.v, other.v))

        def __add__(self, o):
            return self._op(o, lambda a, b: a + b)

        def __sub__(self, o):
            return self._op(o, lambda a, b: a - b)

        def __mul__(self, o):
            return self._op(o, lambda a, b: a * b)

    t, p = pair
    if formula is FlopFormula.DIRECT:
        d = [_C(a) - _C(b) for a, b in zip(t, p)]
        total = d[0] * d[0] + d[1] * d[1]
        total = total + d[2] * d[2]
    elif formula is FlopFormula.ALGEBRAIC_INNER:
        base = _C(sum(v * v for v in t) + sum(v * v for v in p))
        x2 = [_C(2.0 * v) for v in t]
        cross = x2[0] * _C(p[0]) + x2[1] * _C(p[1])
        cross = cross + x2[2] * _C(p[2])
        total = base - cross
    else:
        raise ValueError(f"unknown flop formula {formula!r}")
    assert total.v >= 0.0
    return ops[0]
