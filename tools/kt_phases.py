#!/usr/bin/env python
"""Phase times of union_diag from a DS_KT_PHASES=1 kt build (tools/kt_patch.py):
per CTA, microseconds from its start (after griddep_wait) to each phase mark.

    python tools/kt_phases.py gpurun_out/kt.txt [variants/kt_names.txt]
"""
import statistics
import sys

path = sys.argv[1]
names_path = sys.argv[2] if len(sys.argv) > 2 else "variants/kt_names.txt"
names = dict(l.split() for l in open(names_path) if l.strip())
calls, cur = [], None
for l in open(path):
    if l.startswith("CALL"):
        cur = []
        calls.append(cur)
    elif cur is not None and l.strip():
        cur.append(tuple(map(int, l.split())))
rec = calls[-1]
diag = [k for k, v in names.items() if v == "union_diag_kernel"]
start = {blk: t for f, ln, blk, t in rec if f"{f}:{ln}" in diag}
t0 = min(start.values())
marks = {}
for f, ln, blk, t in rec:
    if 61000 < ln < 62000:
        marks.setdefault(ln, []).append((blk // 32, t))
print(f"union_diag: {len(start)} CTAs; start spread {(max(start.values()) - t0) / 1e3:.2f} us")
for site in sorted(marks):
    rel = [(t - start[b]) / 1e3 for b, t in marks[site] if b in start]
    absol = [(t - t0) / 1e3 for b, t in marks[site]]
    if not rel:
        continue
    rel.sort()
    print(f"site {site}: {len(rel):4d} CTAs  since CTA start p50 {statistics.median(rel):6.2f} "
          f"p90 {rel[int(0.9 * (len(rel) - 1))]:6.2f} max {rel[-1]:6.2f}  | abs max {max(absol):6.2f}")
ends = [t for f, ln, blk, t in rec if ln == 61100]
lk = [k for k, v in names.items() if v == "union_links_kernel"]
lstart = [t for f, ln, blk, t in rec if f"{f}:{ln}" in lk]
if ends and lstart:
    l0 = min(lstart)
    rel = sorted((t - l0) / 1e3 for t in ends)
    q = lambda p: rel[min(len(rel) - 1, int(p * len(rel)))]
    print(f"union_links warp ends (us after its first block): p10 {q(0.1):.1f} p50 {q(0.5):.1f} "
          f"p90 {q(0.9):.1f} p99 {q(0.99):.1f} max {rel[-1]:.1f} ({len(rel)} warps)")
# per-unit durations of union_links (61101 = unit start per warp, 61100 = warp end)
from collections import defaultdict
per = defaultdict(list)
for f, ln, blk, t in rec:
    if ln in (61100, 61101):
        per[blk].append((t, ln))
if per and lstart:
    durs, nunits, tail = [], [], []
    for blk, ev in per.items():
        ev.sort()
        st = [t for t, ln in ev if ln == 61101]
        end = max(t for t, ln in ev)
        nunits.append(len(st))
        for i, t in enumerate(st):
            durs.append(((st[i + 1] if i + 1 < len(st) else end) - t) / 1e3)
        tail.append(((end - l0) / 1e3, len(st), [round(((st[i + 1] if i + 1 < len(st) else end) - t) / 1e3, 1) for i, t in enumerate(st)]))
    durs.sort()
    q = lambda p: durs[min(len(durs) - 1, int(p * len(durs)))]
    print(f"units {len(durs)}; per warp mean {statistics.mean(nunits):.2f} max {max(nunits)}; unit us p50 {q(0.5):.2f} p90 {q(0.9):.2f} p99 {q(0.99):.2f} max {durs[-1]:.2f}")
    tail.sort(reverse=True)
    for e in tail[:8]:
        print("  tail warp end %.1f us, %d units, durations %s" % e)
