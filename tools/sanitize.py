#!/usr/bin/env python
"""Workload for compute-sanitizer runs (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python tools/sanitize.py c1
    compute-sanitizer --tool racecheck python tools/sanitize.py chain

c1:    C1 (10k, 2-D) through run_dbscan (default schedule, graph recorded on the 2nd
       call and replayed on the 3rd), the dense schedule, fused_build with the
       reference-layout export and merge_iterative from those bits.
wide:  20k 16-D blobs through run_dbscan (the d >= 5 pair loop).
chain: a 100k-point serpentine chain + blobs (the C5 generator scaled down): the
       union-find's long-path case, default schedule.
Every result is compared with the C oracle; the script exits 1 on a mismatch.
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_1506_02226_b200 as ds
    from oracle import c_oracle
    which = sys.argv[1] if len(sys.argv) > 1 else "c1"
    if which == "c1":
        cfg = ds.CONFIGS["C1"]
        pts = cfg.points()
        params = ds.validate_params(cfg.eps, cfg.min_pts)
    elif which == "wide":  # 16-D: the paired FFMA2 packing, wide unit batches
        pts = ds.generate_blobs(20_000, 6, 0.3, 0.1, 7, 16)
        params = ds.validate_params(1.5, 8)
    else:
        pts = ds.generate_chain(100_000, 4_000, 8, 2_000, 5)
        params = ds.validate_params(0.3, 8)
    want, wc = c_oracle.dbscan(pts.coords_aos, params.eps_sq, params.min_pts, 1)
    ok = True
    conf = ds.default_config()
    for _ in range(3):  # eager, graph record, graph replay
        lab, _ = ds.run_dbscan(pts, params, conf)
        ok &= bool(np.array_equal(lab.labels, want))
    if which == "c1":
        dense = ds.default_config()
        dense.prune = False
        dense.spatial_order = False
        lab, _ = ds.run_dbscan(pts, params, dense)
        ok &= bool(np.array_equal(lab.labels, want))
        nbr, valid = ds.fused_build_algebraic(pts, params,
                                              ds.KernelVariant(ds.VariantId.FUSED_ALGEBRAIC))
        ok &= bool(np.array_equal(nbr.neighbor_count, wc))
        ok &= bool(np.array_equal(ds.merge_iterative(nbr, valid).labels, want))
    print(f"sanitize workload {which}: n={pts.n} labels_equal_oracle={ok}", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
