#!/usr/bin/env python
"""Summarise the stage-3 device traces of variants/trace.so (tools/trace_patch.py).

    python tools/trace_report.py gpurun_out/trace.log   (the last call's lines only)
"""
import sys

import numpy as np

lines = open(sys.argv[1]).read().split("\n")
lt = [list(map(int, l.split()[1:])) for l in lines if l.startswith("LT ")]
dt = [l.split()[1:] for l in lines if l.startswith("DT ")]
# keep the last call: lines after the last big gap in start times
if lt:
    a = np.array(lt, dtype=np.int64)
    ts = a[:, 2]
    cut = ts >= ts.max() - 5_000_000  # the last 5 ms
    a = a[cut]
    blk, w, ts, te, units, uni, full, words, links, skipw = a.T
    t0 = ts.min()
    en = (te - t0) / 1e3
    dur = (te - ts) / 1e3
    print(f"union_links: warps {len(a)} span {en.max():.1f} us; warp end p10/50/90/99/max "
          f"{np.percentile(en, [10, 50, 90, 99, 100]).round(1)}")
    print(f"  units {units.sum()} shortcut {uni.sum()} full {full.sum()} words {words.sum()} "
          f"links {links.sum()} word-skipped blocks {skipw.sum()}")
    for k in np.argsort(-dur)[:8]:
        print(f"  slow warp {blk[k]}.{w[k]} {dur[k]:.1f} us units {units[k]} shortcut {uni[k]} "
              f"full {full[k]} words {words[k]} links {links[k]}")
if dt:
    sub = [list(map(int, x[8:12])) for x in dt]  # t4a..t4d of the tree merge
    rows = [(int(x[0]), *map(int, x[1:8]), x[12], int(x[13]), int(x[14])) for x in dt]
    ts = np.array([r[1] for r in rows])
    keep = ts >= ts.max() - 5_000_000
    rows = [r for r, k in zip(rows, keep) if k]
    t0 = min(r[1] for r in rows)
    st = np.array([(r[1] - t0) / 1e3 for r in rows])
    en = np.array([(r[7] - t0) / 1e3 for r in rows])
    fast = np.array([r[8] == "fast" for r in rows])
    ph = np.array([[(r[2] - r[1]), (r[3] - r[2]), (r[4] - r[3]), (r[7] - r[4]) if f else (r[5] - r[4]),
                    0 if f else r[6] - r[5], 0 if f else r[7] - r[6]] for r, f in zip(rows, fast)]) / 1e3
    print(f"union_diag: tiles {len(rows)} fast {fast.sum()} start p0/50/max {np.percentile(st, [0, 50, 100]).round(1)} "
          f"end p50/max {np.percentile(en, [50, 100]).round(1)}")
    print("  phase us (setup, scatter, column minima, pointer jumping | fast rest, tree merge, final)")
    for nm, sel in (("fast", fast), ("slow", ~fast)):
        if sel.any():
            print(f"    {nm}: median {np.median(ph[sel], axis=0).round(2)} p90 {np.percentile(ph[sel], 90, axis=0).round(2)}")
    sub = [sb for sb, k in zip(sub, keep) if k]
    sl = [(r, sb) for r, sb, f in zip(rows, sub, fast) if not f and sb[0]]
    if sl:
        seg = np.array([[sb[0] - r[5], sb[1] - sb[0], sb[2] - sb[1], sb[3] - sb[2], r[6] - sb[3]]
                        for r, sb in sl]) / 1e3
        print("  tree merge (slots, tree masks, crossing scan, closure, root update) median",
              np.median(seg, axis=0).round(2), "p90", np.percentile(seg, 90, axis=0).round(2))
    ent = np.array([r[9] for r in rows])
    tr = np.array([r[10] for r in rows])
    print(f"  entries p50/max {np.percentile(ent, [50, 100])}, trees (slow) p50/90/max "
          f"{np.percentile(tr[~fast], [50, 90, 100]) if (~fast).any() else '-'}")
ks = [l.split() for l in lines if l.startswith("KS ")]
if ks:
    # the last call: from the last prep_kernel stamp on
    starts = [i for i, x in enumerate(ks) if x[1] == "prep_kernel"]
    call = ks[starts[-1]:] if starts else ks
    t0 = int(call[0][2])
    prev = None
    print("kernel starts of the last call (us after prep start; delta = previous kernel's time):")
    for x in call:
        t = (int(x[2]) - t0) / 1e3
        print(f"  {t:8.2f}  {'' if prev is None else f'+{t - prev:6.2f}'}  {x[1]}")
        prev = t
