#!/usr/bin/env python
"""One clustering of a config through the public API (DS_CONFIG, default C2): for
device-side traces of instrumented builds (tools/build_variant.sh)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_02226_b200 as ds  # noqa: E402

cfg = ds.CONFIGS[os.environ.get("DS_CONFIG", "C2")]
pts = cfg.points()
params = ds.validate_params(cfg.eps, cfg.min_pts)
conf = ds.default_config()
conf.mem_cap = 150 * 1024**3
for _ in range(int(os.environ.get("DS_RUNS", "1"))):
    lab, t = ds.run_dbscan(pts, params, conf)
    print("run", t.fused_ms, t.merge_ms, t.tile_ms, file=sys.stderr)
