#!/usr/bin/env python
"""Stage-1 kernel timing across schedules/configs (median of reps) + label parity.

    python tools/tile_bench.py [--configs C2,C4] [--dense C2] [--reps 5]

frac = pairs evaluated x (2d+1) / tile kernel time / (148 SMs x 128 lanes x 1965 MHz).
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1506_02226_b200 as ds  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="C1,C2,C3,C4,C5")
ap.add_argument("--dense", default="C2")
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
PEAK = 148 * 128 * 1965e6


def run(name, dense):
    cfg = ds.CONFIGS[name]
    pts = cfg.points()
    params = ds.validate_params(cfg.eps, cfg.min_pts)
    conf = ds.default_config()
    conf.mem_cap = 150 * 1024**3
    if dense:
        conf.prune = False
        conf.spatial_order = False
    ts = []
    for _ in range(args.reps + 1):
        lab, t = ds.run_dbscan(pts, params, conf)
        ts.append(t)
    ts = ts[1:]
    tile = statistics.median(t.tile_ms for t in ts)
    ops = 2 * pts.d + 1
    pairs = ts[-1].pairs_evaluated
    g = os.path.join(ROOT, "tests", "golden", f"{name.lower()}.npz")
    par = None
    if os.path.exists(g):
        z = np.load(g)
        key = "labels" if "labels" in z.files else "alg/labels"
        par = bool(np.array_equal(lab.labels, z[key]))
    out = {"config": name, "dense": dense, "tile_ms": round(tile, 4),
           "fused_ms": round(statistics.median(t.fused_ms for t in ts), 4),
           "merge_ms": round(statistics.median(t.merge_ms for t in ts), 4),
           "total_ms": round(statistics.median(t.total_ms for t in ts), 4),
           "pairs": pairs, "frac": round(pairs * ops / (tile / 1e3) / PEAK, 4),
           "words": ts[-1].words_emitted, "parity": par, "clusters": lab.cluster_count()}
    print(json.dumps(out), flush=True)


for name in args.configs.split(","):
    run(name, False)
for name in [c for c in args.dense.split(",") if c]:
    run(name, True)
