"""Several shards inside one process (PipelineConfig.devices -> run_dbscan_multi).

This run has one GPU, so the shards are *virtual*: devices=[0, 0, 0] gives three
contexts on device 0, each evaluating its dealt share of the tile pairs, with
the real exchange code (count sum, border minimum, pairwise forest fold by
fold_rounds, device-to-device copies). Labels must equal the reference's for
every shard count, culled and dense.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ds():
    import paper_1506_02226_b200 as pkg
    from paper_1506_02226_b200 import _native
    _native.load_library()
    return pkg


@pytest.mark.parametrize("shards", [2, 3, 4, 5, 8])
def test_virtual_shards_c2_reference_labels(ds, shards):
    g = load_golden("c2.npz")
    cfg = ds.CONFIGS["C2"]
    conf = ds.default_config()
    conf.devices = [0] * shards
    labeling, t = ds.run_dbscan(cfg.points(), ds.validate_params(cfg.eps, cfg.min_pts), conf)
    assert np.array_equal(labeling.labels, g["labels"])
    assert t.pairs_evaluated > 0 and t.merge_ms > 0


@pytest.mark.parametrize("prune", [True, False])
def test_virtual_shards_c1_both_schedules(ds, prune):
    g = load_golden("c1.npz")
    cfg = ds.CONFIGS["C1"]
    conf = ds.default_config()
    conf.devices = (0, 0, 0)
    conf.prune = prune
    conf.spatial_order = prune
    labeling, _ = ds.run_dbscan(cfg.points(), ds.validate_params(cfg.eps, cfg.min_pts), conf)
    assert np.array_equal(labeling.labels, g["alg/labels"])


def test_virtual_shards_c5_chain(ds):
    """The 2M-point chain (13.5k eps-hops through every shard's tile pairs)."""
    g = load_golden("c5.npz")
    cfg = ds.CONFIGS["C5"]
    conf = ds.default_config()
    conf.devices = [0] * 4
    conf.mem_cap = 96 * 1024**3
    labeling, _ = ds.run_dbscan(cfg.points(), ds.validate_params(cfg.eps, cfg.min_pts), conf)
    assert np.array_equal(labeling.labels, g["labels"].astype(np.int64))


def test_shard_fold_unions_forests(ds, rng):
    """ds_shard_fold on random forests: the result's components are the union's."""
    import torch
    from oracle import densescan_oracle as oracle
    n = 5000
    ctx = ds._native.context(0)
    for _ in range(5):
        forests, edges = [], []
        for _ in range(2):
            src = rng.integers(0, n, 800)
            dst = rng.integers(0, n, 800)
            roots = oracle.components(n, src, dst)
            forests.append(torch.from_numpy(roots.astype(np.int32)).cuda())
            edges.append((src, dst))
        ctx.shard_fold(forests[0].data_ptr(), forests[1].data_ptr(), n)
        got = forests[0].cpu().numpy()
        src = np.concatenate([e[0] for e in edges])
        dst = np.concatenate([e[1] for e in edges])
        want = oracle.components(n, src, dst)
        assert np.array_equal(got, want)


def _two_rank_worker(rank, world, port, out_dir):
    import os
    import torch
    import torch.distributed as dist
    import paper_1506_02226_b200 as ds
    from paper_1506_02226_b200.distributed import NativeShardBackend, run_dbscan_sharded
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = ds.CONFIGS["C2"]
        labels, tm = run_dbscan_sharded(cfg.points(), ds.validate_params(cfg.eps, cfg.min_pts),
                                        backend=NativeShardBackend(0), return_device=True)
        np.save(os.path.join(out_dir, f"r{rank}.npy"), labels.cpu().numpy())
        assert tm.pairs_evaluated > 0
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ranks_sharing_one_gpu_over_gloo(tmp_path, world):
    """The one-process-per-GPU driver with its real device stages and the pairwise
    forest fold, `world` ranks on this box's single GPU (gloo collectives, host-staged
    point-to-point): every rank's labels equal the reference's."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_two_rank_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    g = load_golden("c2.npz")
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"r{r}.npy"), g["labels"]), r
