"""The multi-GPU driver over a real NCCL process group (world size 1 on the one GPU
this run has): run_dbscan_sharded with the device stages must give the same labels
as the single-GPU path and the reference (C1 golden labels)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("cull", [True, False])
def test_sharded_driver_over_nccl_world1(cull):
    import torch
    import torch.distributed as dist

    import paper_1506_02226_b200 as ds
    from paper_1506_02226_b200 import _native
    from paper_1506_02226_b200.distributed import NativeShardBackend, run_dbscan_sharded

    g = load_golden("c1.npz")
    cfg = ds.CONFIGS["C1"]
    pts = cfg.points()
    params = ds.validate_params(cfg.eps, cfg.min_pts)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        backend = NativeShardBackend(0)
        backend.ctx.configure(cull, cull)
        labeling, tm = run_dbscan_sharded(pts, params, formula=_native.FORMULA_ALGEBRAIC,
                                          backend=backend)
        backend.ctx.configure(True, True)
    finally:
        dist.destroy_process_group()
    assert np.array_equal(labeling.labels, g["alg/labels"])
    assert tm.pairs_evaluated > 0
