"""bench.py's multi-GPU launcher on CPU: `bench.py --gpus N` without torchrun spawns N
ranks through bench.spawn_ranks (the same code path the GPU run takes), each rank
sees RANK / LOCAL_RANK / WORLD_SIZE / MASTER_* and joins one process group; here
the group is gloo and the device stages are the numpy stand-in of
tests/test_distributed.py, and every rank must return the reference labels."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np
import torch.distributed as dist

import bench
from oracle import densescan_oracle as oracle
from paper_1506_02226_b200 import distributed as D
from paper_1506_02226_b200.core import validate_params
from paper_1506_02226_b200.datasets import generate_blobs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rank_main(out_dir, eps, min_pts):
    from test_distributed import CpuShardBackend
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    assert int(os.environ["LOCAL_RANK"]) == rank
    assert os.environ["MASTER_ADDR"] == "127.0.0.1"
    dist.init_process_group("gloo")
    try:
        coords = generate_blobs(900, 3, 0.15, 0.2, 4, 2).coords_aos
        labeling, _ = D.run_dbscan_sharded(coords, validate_params(eps, min_pts), formula=1,
                                           backend=CpuShardBackend(1))
        np.save(os.path.join(out_dir, f"rank{rank}_of{world}.npy"), labeling.labels)
    finally:
        dist.destroy_process_group()


def test_spawn_two_ranks_gloo(tmp_path):
    bench.spawn_ranks(2, _rank_main, str(tmp_path), 0.08, 5)
    coords = generate_blobs(900, 3, 0.15, 0.2, 4, 2).coords_aos
    want, _ = oracle.dbscan(coords, 0.08 * 0.08, 5, 1)
    for rank in range(2):
        got = np.load(tmp_path / f"rank{rank}_of2.npy")
        assert np.array_equal(got, want), rank


def test_world_size_mismatch_is_refused():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1",
                        "--steps", "1", "--warmup", "1"], env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode != 0 and "WORLD_SIZE=2" in r.stderr


def test_reference_arm_line_is_full_workload(monkeypatch, capsys):
    """--impl reference at C1: every step a full clustering, labels equal the reference's."""
    class A:
        config, steps, warmup, gpus = "C1", 1, 1, 1
    monkeypatch.setattr(bench.os, "cpu_count", lambda: 2)
    bench.run_reference(A)
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["n_gpus"] == 1
    assert "no sampling" in line["cpu_baseline"]["sample"]
    assert line["parity_vs_reference_labels"] is True
    assert abs(line["ms_per_step"] / 1e3 - 10_000 / line["value"]) < 1e-6
