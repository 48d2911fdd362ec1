"""Full-size parity fixtures for BASELINE configs C3, C4 and C5 — TEST INFRASTRUCTURE.

    python tests/golden/make_golden_big.py [--configs C3,C4,C5] [--threads N]

The reference package cannot run these configurations (a
125 GB / 500 GB bit matrix for C3 / C5, and d=16 is rejected by PointSet,
reference core.py:53-54), so the labels come from the C restatement
(oracle/ds_oracle.c). That oracle is pinned bit-for-bit to fixtures produced
by EXECUTING the reference (C1, C2 at full size, KATs, lattices, random sets;
tests/test_c_oracle.py), and uses the same arithmetic order (reference
kernels.py:383-417, ALGEBRAIC = default_config) and merge contract
(merge.py:116-166, core.py:116-132).

Each fixture (tests/golden/<config>.npz, compressed) holds
  labels        int32 canonical labels (cluster ids < 2^31), all N
  counts_sha    sha256 of the int64 neighbour counts (incl. self)
  counts_sample int32 counts at every 97th point (diagnostics on mismatch)
  clusters, noise, cores, n, d, eps, min_pts, oracle_s, threads
The GPU suite (tests/test_gpu_big.py) compares run_dbscan(default_config())
and the dense schedule against them; nothing there runs the oracle.
"""

from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle import c_oracle  # noqa: E402
from paper_1506_02226_b200.datasets import CONFIGS  # noqa: E402
from paper_1506_02226_b200.core import validate_params  # noqa: E402


def counts_sha(counts: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(counts, dtype=np.int64).tobytes()).hexdigest()


def make(name: str, threads: int) -> None:
    cfg = CONFIGS[name]
    pts = cfg.points()
    params = validate_params(cfg.eps, cfg.min_pts)
    t0 = time.perf_counter()
    labels, counts = c_oracle.dbscan(pts.coords_aos, params.eps_sq, cfg.min_pts, 1, threads)
    secs = time.perf_counter() - t0
    assert labels.max() < 2**31
    out = os.path.join(HERE, f"{name.lower()}.npz")
    np.savez_compressed(
        out, labels=labels.astype(np.int32), counts_sha=np.array(counts_sha(counts)),
        counts_sample=counts[::97].astype(np.int32),
        clusters=np.int64(labels.max() + 1), noise=np.int64((labels < 0).sum()),
        cores=np.int64((counts >= cfg.min_pts).sum()), n=np.int64(pts.n), d=np.int64(pts.d),
        eps=np.float64(cfg.eps), min_pts=np.int64(cfg.min_pts), oracle_s=np.float64(secs),
        threads=np.int64(threads))
    print(f"{name}: n={pts.n} d={pts.d} clusters={labels.max() + 1} "
          f"noise={(labels < 0).sum()} oracle {secs:.1f}s on {threads} threads -> {out} "
          f"({os.path.getsize(out) / 1e6:.2f} MB)", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C3,C4,C5")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    for name in args.configs.split(","):
        make(name, args.threads)


if __name__ == "__main__":
    main()
