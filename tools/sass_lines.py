#!/usr/bin/env python
"""Per-source-line instruction counts and stall samples of one kernel in an ncu report.

    python tools/sass_lines.py REPORT.ncu-rep OBJECT.o MANGLED_KERNEL [top]

Aligns the report's SASS page (instructions executed, warp-stall samples) with the
line table of the same kernel disassembled from the object (nvdisasm -g).
"""
import collections
import csv
import os
import io
import re
import subprocess
import sys
import tempfile

rep, obj, kern = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
isrc, iex = hdr.index("Source"), hdr.index("Instructions Executed")
ist = hdr.index("Warp Stall Sampling (All Samples)")
ins = []
kidx = int(os.environ.get("KIDX", "0"))  # which kernel of the report (each repeats the header)
for r in rows[2:]:
    if len(r) <= iex:
        continue
    if not (r[iex] or "0").isdigit():
        if r[iex] != "Instructions Executed":
            continue
        if kidx == 0:
            break
        kidx -= 1
        ins = []
        continue
    ins.append((r[isrc].strip(), int(r[iex] or 0), int(r[ist] or 0)))
with tempfile.TemporaryDirectory() as d:
    import os
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    import glob
    cub = glob.glob(d + "/*.cubin")[0]
    txt = subprocess.run(["nvdisasm", "-g", cub], capture_output=True, text=True).stdout.split("\n")
start = [i for i, l in enumerate(txt) if l.startswith(".text." + kern + ":")][0]
seq, cur, cfile = [], None, None
for l in txt[start + 1:]:
    if l.startswith(".text.") or l.startswith(".section"):
        break
    m = re.search(r'//## File "(.*?)", line (\d+)', l)
    if m:
        cfile, cur = m.group(1).split("/")[-1], int(m.group(2))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        seq.append((m.group(2).strip(), cfile, cur))
assert len(seq) == len(ins), (len(seq), len(ins))
agg = collections.defaultdict(lambda: [0, 0])
for (op, f, ln), (_, e, s) in zip(seq, ins):
    agg[(f, ln)][0] += e
    agg[(f, ln)][1] += s
tot_e = sum(v[0] for v in agg.values())
tot_s = sum(v[1] for v in agg.values())
srcs = {}
print(f"total warp instructions {tot_e}, stall samples {tot_s}")
for (f, ln), (e, s) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    if f and f not in srcs:
        try:
            srcs[f] = open([p for p in glob.glob("/root/repo/**/" + f, recursive=True)][0]).read().split("\n")
        except Exception:
            srcs[f] = []
    text = srcs.get(f, [])[ln - 1].strip()[:70] if f and ln and srcs.get(f) else ""
    print(f"{f}:{ln:<5} instr {100 * e / tot_e:5.1f}%  stall {100 * s / tot_s:5.1f}%  {text}")
