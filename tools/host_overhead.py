#!/usr/bin/env python
"""Where the e2e time of run_dbscan goes on the host (C2): wall time of the full
public call vs the bare C call and its device-event parts."""
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_02226_b200 as ds  # noqa: E402
from paper_1506_02226_b200 import _native  # noqa: E402

cfg = ds.CONFIGS[os.environ.get("DS_CONFIG", "C2")]
pts = cfg.points()
params = ds.validate_params(cfg.eps, cfg.min_pts)
conf = ds.default_config()
ctx = _native.context(0)
_native.pin_frozen(pts.coords_aos, pts)
labels = _native.pinned_empty(pts.n)
for _ in range(5):
    ds.run_dbscan(pts, params, conf)


def med(f, k=30):
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        f()
        ts.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(ts)


full = med(lambda: ds.run_dbscan(pts, params, conf))
bare_t = []


def bare():
    import ctypes
    t = _native.Timings()
    st = ctx.lib.ds_run_dbscan(ctx.handle, pts.coords_aos.ctypes.data, pts.n, pts.d,
                               float(params.eps_sq), int(params.min_pts), 1, int(4 << 30),
                               labels.ctypes.data, None, ctypes.byref(t))
    assert st == 0
    bare_t.append(t)


bare_ms = med(bare)
pin_ms = med(lambda: _native.pinned_empty(pts.n), 100)
cfg_ms = med(lambda: ctx.configure(True, True), 100)
t = bare_t[-1]
print({"full_ms": full, "bare_c_call_ms": bare_ms, "pinned_empty_ms": pin_ms, "configure_ms": cfg_ms,
       "h2d": t.h2d_ms, "fused": t.fused_ms, "merge": t.merge_ms, "d2h": t.d2h_ms,
       "device_sum": t.h2d_ms + t.fused_ms + t.merge_ms + t.d2h_ms, "c_total": t.total_ms})
