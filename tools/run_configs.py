#!/usr/bin/env python
"""Run the BASELINE configurations C1-C5 on one GPU: timings, work counters and
(optionally) parity against the multithreaded C oracle.

    python tools/run_configs.py [--configs C1,C2,C3,C4,C5] [--oracle C3,C4] [--reps 5]

Prints one JSON line per configuration (gpurun_out/configs.jsonl when run by
tools/gpu_configs.sh).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C4,C5")
    ap.add_argument("--oracle", default="")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--dense", action="store_true", help="also time prune=False, order=False")
    args = ap.parse_args()
    import paper_1506_02226_b200 as ds

    for name in args.configs.split(","):
        cfg = ds.CONFIGS[name]
        t0 = time.perf_counter()
        pts = cfg.points()
        gen_s = time.perf_counter() - t0
        params = ds.validate_params(cfg.eps, cfg.min_pts)
        conf = ds.default_config()
        conf.mem_cap = 150 * 1024**3
        labeling, t = ds.run_dbscan(pts, params, conf)  # warm (allocations)
        runs = []
        for _ in range(args.reps):
            labeling, t = ds.run_dbscan(pts, params, conf)
            runs.append(t)
        line = {
            "config": name, "n": pts.n, "d": pts.d, "gen_s": round(gen_s, 2),
            "total_ms": statistics.median(r.total_ms for r in runs),
            "fused_ms": statistics.median(r.fused_ms for r in runs),
            "merge_ms": statistics.median(r.merge_ms for r in runs),
            "tile_ms": statistics.median(r.tile_ms for r in runs),
            "h2d_ms": statistics.median(r.h2d_ms for r in runs),
            "d2h_ms": statistics.median(r.d2h_ms for r in runs),
            "pairs_evaluated": runs[-1].pairs_evaluated,
            "n2": pts.n * pts.n,
            "tiles_kept": runs[-1].tiles_total,
            "words": runs[-1].words_emitted, "clusters": labeling.cluster_count(),
            "noise": labeling.noise_count(), "cores": runs[-1].core_count,
        }
        line["points_per_s"] = pts.n / (line["total_ms"] / 1e3)
        line["gpair_per_s_executed"] = line["pairs_evaluated"] / (line["tile_ms"] / 1e3) / 1e9
        if args.dense:
            dconf = ds.default_config()
            dconf.mem_cap = 150 * 1024**3
            dconf.prune = False
            dconf.spatial_order = False
            dl, dt = ds.run_dbscan(pts, params, dconf)
            dl, dt = ds.run_dbscan(pts, params, dconf)
            line["dense_total_ms"] = dt.total_ms
            line["dense_tile_ms"] = dt.tile_ms
            line["dense_pairs"] = dt.pairs_evaluated
            line["dense_equal"] = bool(np.array_equal(dl.labels, labeling.labels))
        if name in args.oracle.split(","):
            from oracle import c_oracle
            t1 = time.perf_counter()
            want, wc = c_oracle.dbscan(pts.coords_aos, params.eps_sq, cfg.min_pts, 1)
            line["oracle_s"] = round(time.perf_counter() - t1, 1)
            line["oracle_threads"] = c_oracle.threads()
            line["parity_labels"] = bool(np.array_equal(labeling.labels, want))
            ctx = ds._native.context()
            _, counts, _ = ctx.run_dbscan(pts.coords_aos, params.eps_sq, cfg.min_pts, 1,
                                          conf.mem_cap, want_counts=True)
            line["parity_counts"] = bool(np.array_equal(counts, wc))
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
