"""Multi-GPU DBSCAN: row-block sharding of the eps-tile work across ranks.

The reference parallelises stage 1 by handing disjoint row ranges to worker
threads (pkg/src/densescan/_parallel.py:24-39, kernels.py:322-335) and
merges serially. Here one process drives one GPU (torch.distributed over
NCCL for the exchanges):

  * every rank holds all n points (float64, <= 32 MB at every config);
  * the upper-triangle tile pairs (items, TILE = 512 points per side,
    numbered row-major by ds_tile_items) — after bounding-box culling, the
    list of tile pairs that can hold an in-range pair, built identically on
    every rank (deterministic sort and scan) — are dealt to the ranks
    cyclically (kept pair q goes to rank q mod world, which spreads dense and
    sparse regions evenly); with culling off, the work units of the dense
    triangle are split into contiguous equal ranges (shard_range);
  * stage 1+2 on the rank's items gives partial neighbour counts and the
    rank's adjacency words (ds_shard_stage12);
  * exchange 1: all_reduce(SUM) of the int32 counts -> identical core flags;
  * stage 3 on the rank's words gives a union-find forest and border minima
    (ds_shard_stage3_local);
  * exchange 2: all_gather of the int32 forests, all_reduce(MIN) of the
    border minima;
  * every rank folds the forests and emits the same canonical labels
    (ds_shard_stage3_merge).

Labels are identical for any rank count (the forest union and the border
minimum do not depend on how pairs were split), which tests/test_distributed.py
checks with world sizes 1-3 on the gloo backend with a CPU stand-in for the
device stages, and tests/test_gpu_parity.py with the real stages.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from . import _native
from .core import Labeling, PointSet, DbscanParams
from .kernels import resolve_mem_cap

TILE = 512
NONE = 0x7FFFFFFF


def n_tiles(n: int) -> int:
    return (n + TILE - 1) // TILE


def tile_items(n: int) -> int:
    t = n_tiles(n)
    return t * (t + 1) // 2


def item_to_tiles(q: int, t: int) -> tuple[int, int]:
    """Item q -> tile pair (a, b), a <= b, row-major over the upper triangle
    (the device's decode_item in csrc/ds_tile.cu)."""
    def off(a):
        return a * t - a * (a - 1) // 2
    tt = 2.0 * t + 1.0
    a = int(math.floor((tt - math.sqrt(tt * tt - 8.0 * q)) * 0.5))
    a = max(0, min(a, t - 1))
    while a + 1 <= t - 1 and off(a + 1) <= q:
        a += 1
    while a > 0 and off(a) > q:
        a -= 1
    return a, a + (q - off(a))


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, near-equal item range of one rank (like split_ranges, _parallel.py:16-21)."""
    return total * rank // world, total * (rank + 1) // world


class NativeShardBackend:
    """The device stages through the C ABI, on torch CUDA tensors."""

    def __init__(self, device: int):
        import torch
        self.torch = torch
        self.device = torch.device("cuda", device)
        self.ctx = _native.context(device)

    def stream(self) -> int:
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def to_device(self, coords: np.ndarray):
        return self.torch.from_numpy(np.ascontiguousarray(coords, dtype=np.float64).copy()).to(
            self.device)

    def stage12(self, coords, eps_sq, formula, rank, world, mem_cap):
        n, d = coords.shape
        counts = self.torch.empty(n, dtype=self.torch.int32, device=self.device)
        t = self.ctx.shard_stage12(coords.data_ptr(), n, d, eps_sq, formula, rank, world,
                                   mem_cap, counts.data_ptr(), self.stream())
        return counts, t

    def stage3_local(self, counts, min_pts):
        n = counts.shape[0]
        parent = self.torch.empty(n, dtype=self.torch.int32, device=self.device)
        bmin = self.torch.empty(n, dtype=self.torch.int32, device=self.device)
        self.ctx.shard_stage3_local(counts.data_ptr(), n, min_pts, parent.data_ptr(),
                                    bmin.data_ptr(), self.stream())
        return parent, bmin

    def stage3_merge(self, counts, min_pts, parents, bmin):
        n = counts.shape[0]
        labels = self.torch.empty(n, dtype=self.torch.int64, device=self.device)
        self.ctx.shard_stage3_merge(counts.data_ptr(), n, min_pts, parents.data_ptr(),
                                    parents.shape[0], bmin.data_ptr(), labels.data_ptr(),
                                    self.stream())
        return labels


@dataclass
class ShardTimings:
    stage12_ms: float = 0.0
    exchange1_ms: float = 0.0
    stage3_local_ms: float = 0.0
    exchange2_ms: float = 0.0
    stage3_merge_ms: float = 0.0
    total_ms: float = 0.0
    items: tuple = (0, 0)
    tile_ms: float = 0.0
    pairs_evaluated: int = 0


def run_dbscan_sharded(points, params: DbscanParams, formula: int = _native.FORMULA_ALGEBRAIC,
                       mem_cap=None, group=None, backend=None, coords=None):
    """Cluster `points` across the ranks of `group`; every rank returns the same
    canonical Labeling (and its own ShardTimings).

    `coords` may be a device-resident (n, d) float64 tensor (the benchmark's
    HBM-resident input); otherwise the PointSet is copied to the device.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if backend is None:
        backend = NativeShardBackend(torch.cuda.current_device())
    sync = torch.cuda.synchronize if torch.cuda.is_available() else (lambda: None)
    tm = ShardTimings()
    t0 = time.perf_counter()
    if coords is None:
        coords = backend.to_device(points.coords_aos if isinstance(points, PointSet) else points)
    n = coords.shape[0]
    tm.items = shard_range(tile_items(n), world, rank)  # dense share (culled: same fraction)
    cap = resolve_mem_cap(mem_cap)

    t = time.perf_counter()
    counts, st = backend.stage12(coords, params.eps_sq, formula, rank, world, cap)
    tm.tile_ms = getattr(st, "tile_ms", 0.0)
    tm.pairs_evaluated = getattr(st, "pairs_evaluated", 0)
    sync()
    tm.stage12_ms = (time.perf_counter() - t) * 1e3

    t = time.perf_counter()
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    sync()
    tm.exchange1_ms = (time.perf_counter() - t) * 1e3

    t = time.perf_counter()
    parent, bmin = backend.stage3_local(counts, params.min_pts)
    sync()
    tm.stage3_local_ms = (time.perf_counter() - t) * 1e3

    t = time.perf_counter()
    gathered = [torch.empty_like(parent) for _ in range(world)]
    dist.all_gather(gathered, parent, group=group)
    parents = torch.stack(gathered)
    dist.all_reduce(bmin, op=dist.ReduceOp.MIN, group=group)
    sync()
    tm.exchange2_ms = (time.perf_counter() - t) * 1e3

    t = time.perf_counter()
    labels = backend.stage3_merge(counts, params.min_pts, parents, bmin)
    sync()
    tm.stage3_merge_ms = (time.perf_counter() - t) * 1e3
    tm.total_ms = (time.perf_counter() - t0) * 1e3
    return Labeling(labels.cpu().numpy()), tm
