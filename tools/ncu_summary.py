#!/usr/bin/env python
"""Summarise ncu output into profiles/ (markdown + csv).

    python tools/ncu_summary.py --launches gpurun_out/launches.csv \
        --report gpurun_out/prof_tile.ncu-rep [--report ...] --out profiles/r01_c2.md

Reads the launch list (gpu__time_duration per launch, cold-cache and serialised)
and full-set reports: speed of light, pipe utilisation, DRAM bytes, occupancy,
top stall reasons and the hottest SASS lines.
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import subprocess

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def ncu_csv(args):
    out = subprocess.run(["ncu", *args], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        name = d["Kernel Name"]
        short = name.split("(")[0].replace("ds::<unnamed>::", "").replace("void ", "")
        agg.setdefault(short[:70], []).append(float(d["Metric Value"]) / 1e3)
    return agg


def report(path):
    raw = ncu_csv(["-i", path, "--page", "raw", "--csv"])
    out = []
    for ki in range(2, len(raw)):
        h, units, v = raw[0], raw[1], raw[ki]
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        vals = {}
        for key, label in METRICS:
            if key in h:
                i = h.index(key)
                vals[label] = f"{v[i]} {units[i]}".strip()
        stalls = []
        for k, x in zip(h, v):
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                try:
                    stalls.append((float(x), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        top = [f"{k} {s / tot * 100:.1f}%" for s, k in sorted(stalls, reverse=True)[:6]]
        out.append((name, vals, top))
    src = ncu_csv(["-i", path, "--page", "source", "--csv", "--print-source", "sass"])
    hot = []
    # one section per profiled kernel, each starting with its own header row
    sections, h = [], None
    for r in src:
        if "Warp Stall Sampling (All Samples)" in r:
            h = r
            sections.append((h, []))
        elif h is not None and len(r) == len(h):
            sections[-1][1].append(r)
    for si, (h, data) in enumerate(sections):
        i_s = h.index("Warp Stall Sampling (All Samples)")
        i_src = h.index("Source")

        def val(r):
            try:
                return float(r[i_s] or 0)
            except ValueError:
                return 0.0

        tot = sum(val(r) for r in data)
        if tot <= 0:
            continue
        if len(sections) > 1:
            hot.append(f"-- kernel {si} --")
        for r in sorted(data, key=lambda r: -val(r))[:12]:
            hot.append(f"{val(r) / tot * 100:5.1f}%  {r[i_src].strip()[:90]}")
    return out, hot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--report", action="append", default=[])
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--note", default="")
    args = ap.parse_args()
    lines = [f"# {args.title}", ""]
    if args.note:
        lines += [args.note, ""]
    if args.launches:
        agg = launches(args.launches)
        lines += ["## Launch list (gpu__time_duration, --clock-control none; cold-cache, serialised)",
                  "", "| kernel | launches | mean us | share of listed % |", "|---|---|---|---|"]
        total = sum(sum(v) for v in agg.values())
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.1f} | {sum(v) / total * 100:.1f} |")
        lines.append("")
    for path in args.report:
        kernels, hot = report(path)
        for name, vals, top in kernels:
            lines += [f"## `{name[:110]}`", "", f"report: `{path.split('/')[-1]}`", ""]
            lines += [f"- {k}: {v}" for k, v in vals.items()]
            lines += ["- top stall reasons: " + ", ".join(top), ""]
        if hot:
            lines += ["hottest SASS (share of warp-stall samples):", "", "```"] + hot + ["```", ""]
    with open(args.out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print(f"wrote {args.out}")


if __name__ == "__main__":
    main()
