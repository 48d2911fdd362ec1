#!/usr/bin/env python
"""Mean per-kernel duration of an ncu launch-list CSV: python tools/launch_table.py FILE..."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    d = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > iv and r[im] == "gpu__time_duration.sum":
            d[r[ik][:60]].append(float(r[iv].replace(",", "")))
    print(f"== {path}")
    tot = 0.0
    for k, v in sorted(d.items(), key=lambda x: -sum(x[1]) / len(x[1])):
        m = sum(v) / len(v) / 1000
        if "FillFunctor" not in k:
            tot += m * (2 if "radix_scatter" in k or "digit_scan" in k or "Onesweep" in k else 1)
        print(f"{len(v):3d} {m:8.2f} us  {k}")
    print(f"   sum of per-step kernels ~ {tot:.1f} us")
