"""Multi-process sharding logic on CPU (gloo, world sizes 1-3).

The exchange steps of distributed.run_dbscan_sharded run for real (gloo
collectives on CPU tensors). The three device stages are replaced by a numpy
stand-in that evaluates exactly the rank's tile-pair items with the oracle's
pair arithmetic, so the test checks: the item partition covers every tile
pair once, partial counts sum correctly, per-shard forests + border minima
fold into the reference labels, and labels do not depend on the rank count.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import densescan_oracle as oracle
from paper_1506_02226_b200 import distributed as D
from paper_1506_02226_b200.datasets import generate_blobs


class CpuShardBackend:
    """numpy stand-in for the three device stages (same contract as NativeShardBackend)."""

    def __init__(self, formula):
        self.formula = formula
        self.blocks = []

    def to_device(self, coords):
        return torch.from_numpy(np.ascontiguousarray(coords, dtype=np.float64))

    def stage12(self, coords, eps_sq, formula, rank, world, mem_cap):
        c = coords.numpy()
        n = c.shape[0]
        lo, hi = D.shard_range(D.tile_items(n), world, rank)
        p32 = oracle.narrow(c)
        norms = oracle.sq_norms(p32)
        thr = oracle.thr32(eps_sq)
        t = D.n_tiles(n)
        counts = np.zeros(n, dtype=np.int64)
        self.blocks = []
        for q in range(lo, hi):
            a, b = D.item_to_tiles(q, t)
            r0, r1 = a * D.TILE, min((a + 1) * D.TILE, n)
            c0, c1 = b * D.TILE, min((b + 1) * D.TILE, n)
            hit = oracle.in_range_block(p32, norms, r0, r1, thr, formula, c0, c1)
            counts[r0:r1] += hit.sum(axis=1)
            if a != b:
                counts[c0:c1] += hit.sum(axis=0)
            self.blocks.append((r0, c0, hit))
        self.n = n
        return torch.from_numpy(counts.astype(np.int32)), None

    def stage3_local(self, counts, min_pts):
        n = self.n
        core = counts.numpy() >= min_pts
        parent = np.arange(n, dtype=np.int64)

        def find(x):
            while parent[x] != x:
                parent[x] = parent[parent[x]]
                x = parent[x]
            return x

        bmin = np.full(n, D.NONE, dtype=np.int64)
        for r0, c0, hit in self.blocks:
            ii, jj = np.nonzero(hit)
            ii, jj = ii + r0, jj + c0
            for i, j in zip(ii.tolist(), jj.tolist()):
                if core[i] and core[j]:
                    ri, rj = find(i), find(j)
                    if ri != rj:
                        parent[max(ri, rj)] = min(ri, rj)
                elif core[i]:
                    bmin[j] = min(bmin[j], i)
                elif core[j]:
                    bmin[i] = min(bmin[i], j)
        return torch.from_numpy(parent.astype(np.int32)), torch.from_numpy(bmin.astype(np.int32))

    def fold(self, parent, other):
        """numpy stand-in of ds_shard_fold: union of two forests, flattened, in place."""
        par = parent.numpy().astype(np.int64)
        oth = other.numpy()

        def find(x):
            while par[x] != x:
                par[x] = par[par[x]]
                x = par[x]
            return x

        for i in np.nonzero(oth != np.arange(oth.size))[0].tolist():
            ri, rj = find(i), find(int(oth[i]))
            if ri != rj:
                par[max(ri, rj)] = min(ri, rj)
        parent.copy_(torch.from_numpy(np.array([find(i) for i in range(par.size)],
                                               dtype=np.int32)))

    def stage3_merge(self, counts, min_pts, parents, bmin):
        n = self.n
        core = counts.numpy() >= min_pts
        par = parents.numpy()
        if par.ndim == 1:
            par = par[None, :]
        src = np.concatenate([np.arange(n)[core & (p != np.arange(n))] for p in par])
        dst = np.concatenate([p[core & (p != np.arange(n))] for p in par])
        border = bmin.numpy().astype(np.int64)
        border[border == D.NONE] = -1
        border[core] = -1
        labels = oracle.labels_from_core_graph(n, core, src.astype(np.int64), dst.astype(np.int64),
                                               border)
        return torch.from_numpy(labels)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, coords, eps, min_pts, formula, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1506_02226_b200.core import validate_params
        params = validate_params(eps, min_pts)
        labeling, tm = D.run_dbscan_sharded(coords, params, formula=formula,
                                            backend=CpuShardBackend(formula))
        out[rank] = (labeling.labels.copy(), tm.items)
    finally:
        dist.destroy_process_group()


def run_world(world, coords, eps, min_pts, formula):
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, port, coords, eps, min_pts, formula, out), nprocs=world,
             join=True)
    return dict(out)


def test_item_decode_matches_enumeration():
    for t in (1, 2, 3, 7, 40):
        seen = [(a, b) for a in range(t) for b in range(a, t)]
        assert [D.item_to_tiles(q, t) for q in range(len(seen))] == seen
        assert D.tile_items(t * D.TILE) == len(seen)


def test_shard_ranges_partition_items():
    for total in (1, 6, 7, 76636):
        for world in (1, 2, 3, 8):
            ranges = [D.shard_range(total, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == total
            assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in ranges]
            assert max(sizes) - min(sizes) <= 1


def test_fold_rounds_reach_every_forest():
    """Simulate the schedule: each rank starts with its own set; after the rounds
    every rank must hold the union of all sets, for any world size."""
    for world in range(1, 13):
        held = [{r} for r in range(world)]
        for rnd in D.fold_rounds(world):
            new = [set(h) for h in held]
            for kind, a, b in rnd:
                if kind == "swap":
                    new[a] |= held[b]
                    new[b] |= held[a]
                elif kind == "fold":
                    new[b] |= held[a]
                else:
                    new[b] = set(held[a])
            held = new
        assert all(h == set(range(world)) for h in held), world
        # each rank takes part in at most one step per round (no conflicting writes)
        for rnd in D.fold_rounds(world):
            ranks = [r for _, a, b in rnd for r in (a, b)]
            assert len(ranks) == len(set(ranks))
        rounds = len(D.fold_rounds(world))
        p = 1 << (world.bit_length() - 1)
        assert rounds == (p.bit_length() - 1) + (2 if world > p else 0)


@pytest.mark.parametrize("formula", [1, 0])
def test_sharded_labels_equal_reference_any_world(formula):
    coords = generate_blobs(1300, 4, 0.15, 0.2, 21, 2).coords_aos
    eps, min_pts = 0.08, 5
    want, _ = oracle.dbscan(coords, eps * eps, min_pts, formula)
    for world in (1, 2, 3, 4, 5):
        out = run_world(world, coords, eps, min_pts, formula)
        items = sorted(v[1] for v in out.values())
        assert items[0][0] == 0 and items[-1][1] == D.tile_items(1300)
        for rank, (labels, _) in out.items():
            assert np.array_equal(labels, want), (world, rank)
