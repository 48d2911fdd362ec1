#!/usr/bin/env python
"""Per-kernel timeline of the last call recorded by a tools/kt_patch.py build.

    python tools/kt_report.py gpurun_out/kt.txt [variants/kt_names.txt]

For each kernel (in launch order): first and last block start after griddep_wait
(i.e. after the predecessor completed), and the time until the next kernel's first
block start — the kernel's share of the pipeline including its drain.
"""
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
        f, ln, blk, t = map(int, l.split())
        cur.append((f, ln, blk, t))
rec = calls[-1]
ends = sorted(t for f, ln, blk, t in rec if ln == 60000)  # eps kernel warp ends
rec = [r for r in rec if r[1] != 60000]
# launches in time order: consecutive records of the same kernel site (a kernel's blocks
# stamp after griddepcontrol.wait, i.e. after its predecessor completed)
runs = []
for f, ln, blk, t in sorted(rec, key=lambda r: r[3]):
    if runs and runs[-1][0] == (f, ln):
        runs[-1][1].append(t)
    else:
        runs.append(((f, ln), [t]))
t0 = min(runs[0][1])
print(f"{len(calls)} calls; last call {len(rec)} block records")
print(f"{'kernel':34s} {'blocks':>6s} {'first':>8s} {'last':>8s} {'to next':>8s}")
for i, ((f, ln), ts) in enumerate(runs):
    first, last = (min(ts) - t0) / 1e3, (max(ts) - t0) / 1e3
    nxt = (min(runs[i + 1][1]) - t0) / 1e3 if i + 1 < len(runs) else None
    name = names.get(f"{f}:{ln}", f"{f}:{ln}")
    span = "" if nxt is None else f"{nxt - first:8.2f}"
    print(f"{name[:34]:34s} {len(ts):6d} {first:8.2f} {last:8.2f} {span}")
if ends:
    import statistics
    e0 = min(t for (f, ln), ts in runs if names.get(f"{f}:{ln}") == "eps_unit_kernel" for t in ts)
    rel = [(t - e0) / 1e3 for t in ends]
    q = lambda p: rel[min(len(rel) - 1, int(p * len(rel)))]
    print(f"eps_unit_kernel warp ends (us after its first block): p10 {q(0.1):.1f} p50 {q(0.5):.1f} "
          f"p90 {q(0.9):.1f} p99 {q(0.99):.1f} max {rel[-1]:.1f} ({len(rel)} warps)")
