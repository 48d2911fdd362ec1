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
  * exchange 2: all_reduce(MIN) of the border minima, and a pairwise fold of
    the int32 forests by recursive doubling (fold_rounds: in round s rank r
    swaps forests with rank r XOR 2^s and folds the partner's into its own,
    ds_shard_fold), so after log2(world) rounds every rank holds the forest of
    all edges with O(n log world) work and traffic per rank (world sizes that
    are not powers of two fold their extra ranks in first and copy the result
    back last);
  * every rank turns the folded forest and the minima into the same canonical
    labels (ds_shard_stage3_merge), which stay on the device.

The same stages also run inside one process over several devices
(run_dbscan_multi, selected by PipelineConfig.devices): one context and host
thread per shard, the exchanges as device-to-device copies over NVLink. It is
the drop-in for the reference's fork-join over worker threads
(_parallel.py:24-39): one call, shards fanned out and joined internally.

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


def fold_rounds(world: int) -> list[list[tuple[str, int, int]]]:
    """Schedule of the pairwise forest exchange for `world` ranks.

    Each round is a list of steps ("fold", src, dst): dst folds src's forest into
    its own; ("swap", a, b): a and b exchange forests and both fold; ("copy", src,
    dst): dst replaces its forest by src's. With P the largest power of two <=
    world: ranks >= P fold into rank - P first, then log2(P) rounds of swaps
    between r and r XOR 2^s, then ranks >= P receive the result. Every rank ends
    with the union of all forests.
    """
    if world < 1:
        raise ValueError("world must be >= 1")
    p = 1
    while p * 2 <= world:
        p *= 2
    rounds = []
    extra = [("fold", r, r - p) for r in range(p, world)]
    if extra:
        rounds.append(extra)
    s = 1
    while s < p:
        rounds.append([("swap", r, r ^ s) for r in range(p) if r < (r ^ s)])
        s *= 2
    back = [("copy", r - p, r) for r in range(p, world)]
    if back:
        rounds.append(back)
    return rounds


def _fold_distributed(backend, parent, group):
    """Run this rank's part of fold_rounds over torch.distributed point-to-point."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    peer_rank = (lambda r: dist.get_global_rank(group, r)) if group is not None else (lambda r: r)
    # NCCL moves device tensors directly; gloo has no device point-to-point, so its
    # messages are staged through host memory (CPU tests, several ranks on one GPU)
    staged = parent.is_cuda and dist.get_backend(group) != "nccl"
    buf = torch.empty_like(parent)
    for rnd in fold_rounds(world):
        for kind, a, b in rnd:
            if rank not in (a, b):
                continue
            other = b if rank == a else a
            ops = []
            sends = kind == "swap" or (rank == a)
            recvs = kind == "swap" or (rank == b)
            out_t = parent.cpu() if staged else parent
            in_t = torch.empty_like(out_t) if staged else buf
            if sends:
                ops.append(dist.P2POp(dist.isend, out_t, peer_rank(other), group))
            if recvs:
                ops.append(dist.P2POp(dist.irecv, in_t, peer_rank(other), group))
            for req in dist.batch_isend_irecv(ops):
                req.wait()
            if recvs:
                if staged:
                    buf.copy_(in_t)
                if kind == "copy":
                    parent.copy_(buf)
                else:
                    backend.fold(parent, buf)
    return parent


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

    def fold(self, parent, other):
        """parent <- union of the forests parent and other (flattened), in place."""
        self.ctx.shard_fold(parent.data_ptr(), other.data_ptr(), parent.shape[0], self.stream())

    def stage3_merge(self, counts, min_pts, parents, bmin):
        n = counts.shape[0]
        if parents.dim() == 1:
            parents = parents.unsqueeze(0)
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
                       mem_cap=None, group=None, backend=None, coords=None,
                       return_device: bool = False):
    """Cluster `points` across the ranks of `group`; every rank returns the same
    canonical Labeling (and its own ShardTimings).

    `coords` may be a device-resident (n, d) float64 tensor (the benchmark's
    HBM-resident input); otherwise the PointSet is copied to the device. With
    return_device the labels stay a device int64 tensor (no host copy).
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
    dist.all_reduce(bmin, op=dist.ReduceOp.MIN, group=group)
    parent = _fold_distributed(backend, parent, group)
    sync()
    tm.exchange2_ms = (time.perf_counter() - t) * 1e3

    t = time.perf_counter()
    labels = backend.stage3_merge(counts, params.min_pts, parent, bmin)
    sync()
    tm.stage3_merge_ms = (time.perf_counter() - t) * 1e3
    tm.total_ms = (time.perf_counter() - t0) * 1e3
    if return_device:
        return labels, tm
    return Labeling(labels.cpu().numpy()), tm


# ---- one process, several devices (PipelineConfig.devices) -------------------------

class _MultiShards:
    """One native context per shard (shards may share a device: virtual shards)."""

    _cache: dict = {}

    @classmethod
    def get(cls, devices: tuple):
        import threading
        key = (threading.get_ident(), devices)
        shards = cls._cache.get(key)
        if shards is None:
            shards = cls._cache[key] = [_native.Context(dev) for dev in devices]
        return shards


def run_dbscan_multi(points: PointSet, params: DbscanParams, devices,
                     formula: int = _native.FORMULA_ALGEBRAIC, mem_cap=None,
                     prune: bool = True, spatial_order: bool = True):
    """run_dbscan over len(devices) shards inside this process: the drop-in for the
    reference's fork-join over worker threads (_parallel.py:24-39). One host thread
    per shard drives its device through the shard ABI; counts are summed, border
    minima min-reduced and forests folded pairwise (fold_rounds) by device-to-device
    copies; the first device computes the labels. Returns (labels int64 numpy,
    ShardTimings of the call)."""
    import torch
    from concurrent.futures import ThreadPoolExecutor

    devices = tuple(int(d) for d in devices)
    world = len(devices)
    ctxs = _MultiShards.get(devices)
    for c in ctxs:
        c.configure(prune, spatial_order)
    cap = resolve_mem_cap(mem_cap)
    tm = ShardTimings()
    t0 = time.perf_counter()
    host = np.ascontiguousarray(points.coords_aos, dtype=np.float64)
    n, d = host.shape
    dev = [torch.device("cuda", x) for x in devices]
    src = torch.from_numpy(host)
    if torch.cuda.is_available():
        _native.pin_frozen(points.coords_aos, points)
    coords = [src.to(dv, non_blocking=False) for dv in dev]
    counts = [torch.empty(n, dtype=torch.int32, device=dv) for dv in dev]

    def on(k, fn):
        with torch.cuda.device(dev[k]):
            return fn()

    with ThreadPoolExecutor(max_workers=world) as pool:
        t = time.perf_counter()
        sts = list(pool.map(lambda k: on(k, lambda: ctxs[k].shard_stage12(
            coords[k].data_ptr(), n, d, params.eps_sq, formula, k, world, cap,
            counts[k].data_ptr(), 0)), range(world)))
        tm.stage12_ms = (time.perf_counter() - t) * 1e3
        tm.tile_ms = max(s.tile_ms for s in sts)
        tm.pairs_evaluated = sum(s.pairs_evaluated for s in sts)

        t = time.perf_counter()
        total = counts[0].clone()
        for k in range(1, world):
            total += counts[k].to(dev[0])
        counts = [total] + [total.to(dv) for dv in dev[1:]]
        torch.cuda.synchronize(dev[0])
        tm.exchange1_ms = (time.perf_counter() - t) * 1e3

        t = time.perf_counter()
        parent = [torch.empty(n, dtype=torch.int32, device=dv) for dv in dev]
        bmin = [torch.empty(n, dtype=torch.int32, device=dv) for dv in dev]
        list(pool.map(lambda k: on(k, lambda: ctxs[k].shard_stage3_local(
            counts[k].data_ptr(), n, params.min_pts, parent[k].data_ptr(), bmin[k].data_ptr(),
            0)), range(world)))
        tm.stage3_local_ms = (time.perf_counter() - t) * 1e3

        t = time.perf_counter()
        bm = bmin[0].clone()
        for k in range(1, world):
            bm = torch.minimum(bm, bmin[k].to(dev[0]))
        for rnd in fold_rounds(world):
            def step(st):
                kind, a, b = st
                if kind == "swap":
                    pa, pb = parent[b].to(dev[a]), parent[a].to(dev[b])
                    on(a, lambda: ctxs[a].shard_fold(parent[a].data_ptr(), pa.data_ptr(), n, 0))
                    on(b, lambda: ctxs[b].shard_fold(parent[b].data_ptr(), pb.data_ptr(), n, 0))
                elif kind == "fold":
                    pa = parent[a].to(dev[b])
                    on(b, lambda: ctxs[b].shard_fold(parent[b].data_ptr(), pa.data_ptr(), n, 0))
                else:
                    parent[b].copy_(parent[a].to(dev[b]))
            list(pool.map(step, rnd))
        torch.cuda.synchronize(dev[0])
        tm.exchange2_ms = (time.perf_counter() - t) * 1e3

    t = time.perf_counter()
    labels = torch.empty(n, dtype=torch.int64, device=dev[0])
    on(0, lambda: ctxs[0].shard_stage3_merge(counts[0].data_ptr(), n, params.min_pts,
                                             parent[0].data_ptr(), 1, bm.data_ptr(),
                                             labels.data_ptr(), 0))
    out = labels.cpu().numpy()
    tm.stage3_merge_ms = (time.perf_counter() - t) * 1e3
    tm.total_ms = (time.perf_counter() - t0) * 1e3
    return out, tm
