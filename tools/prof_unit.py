#!/usr/bin/env python
"""One culled and one dense C2 run (for ncu captures of the stage-1 kernels).

    ncu -k regex:eps_unit -c 4 ... python tools/prof_unit.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_02226_b200 as ds  # noqa: E402

cfg = ds.CONFIGS[os.environ.get("DS_CONFIG", "C2")]
pts = cfg.points()
params = ds.validate_params(cfg.eps, cfg.min_pts)
conf = ds.default_config()
conf.mem_cap = 150 * 1024**3
lab, t = ds.run_dbscan(pts, params, conf)
lab, t = ds.run_dbscan(pts, params, conf)
print("culled", t.tile_ms, t.pairs_evaluated)
if os.environ.get("DS_DENSE", "1") == "0":
    sys.exit(0)
conf.prune = False
conf.spatial_order = False
lab2, t2 = ds.run_dbscan(pts, params, conf)
print("dense", t2.tile_ms, t2.pairs_evaluated, bool((lab.labels == lab2.labels).all()))
