#!/usr/bin/env python
"""Large random inputs through the public API (capacity growth, 24-bit keys, 3-D / 8-D):
two calls each, the second must reproduce the first's labels."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1506_02226_b200 as ds
rng = np.random.default_rng(11)
for n, d, eps, mp in [(4_000_000, 2, 0.02, 8), (8_000_000, 2, 0.01, 8), (3_000_000, 3, 0.05, 10), (1_000_000, 8, 0.6, 8)]:
    pts = ds.PointSet(rng.normal(0, 1, (n, d)) * np.array([3.0] + [1.0] * (d - 1)))
    params = ds.validate_params(eps, mp)
    conf = ds.default_config(); conf.mem_cap = 150 * 1024**3
    w0 = time.perf_counter()
    lab, tm = ds.run_dbscan(pts, params, conf)
    w1 = time.perf_counter()
    lab2, tm2 = ds.run_dbscan(pts, params, conf)
    w3 = time.perf_counter()
    ok = bool(np.array_equal(lab.labels, lab2.labels))
    print(f"n={n} d={d} first {1e3*(w1-w0):.1f} ms second {1e3*(w3-w1):.1f} ms clusters {lab.cluster_count()} "
          f"noise {lab.noise_count()} pairs {tm2.pairs_evaluated} words {tm2.words_emitted} repeat_equal {ok}", flush=True)
