#!/usr/bin/env python
"""Per-level breakdown of one V-cycle from an ncu launch list of scripts/gamg_profile.py
(cold-cache, serialised per-launch times).  usage: summarize_gamg_launches.py launches.csv"""
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, vi, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
seq = [(re.sub(r"\(.*", "", r[ki]).replace("void ", "").split("<")[0].split("::")[-1], r[gi],
        float(r[vi].replace(",", "")) / 1e3) for r in rows]
ends = [i for i, s in enumerate(seq) if s[0] == "k_gamg_residual"]
c0, c1 = ends[0] + 1, ends[1] + 1
cyc = seq[c0:c1]
tot = sum(s[2] for s in cyc)
print(f"one V-cycle: {len(cyc)} kernels, {tot:.1f} us (sum of serialised cold-cache launches)")
for s in cyc:
    print(f"  {s[0]:22s} grid {s[1]:>12s} {s[2]:9.2f} us")
