#!/usr/bin/env python
"""Summarise gpurun_out/ ncu artefacts into profiles/ (tracked evidence).

usage: python scripts/summarize_ncu.py <round-tag> [launches.csv] [report.ncu-rep ...]
Writes profiles/<tag>_launches.txt (per-kernel share of the launch list),
profiles/<tag>_ncu_<kernel>.txt (key --set full metrics per launch) and, for
k_amul_dot, profiles/ncu_traffic.json (DRAM bytes per launch, read by bench.py).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
WORKLOAD = "C3 cube 200^3 per GPU (weak), gamma=1, tol 1e-6"

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes.sum.per_second",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_static", "smsp__inst_executed.sum"]


def launches(path, tag):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in data:
        if len(r) > vi:
            agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised): "
             f"per-kernel share of the first {sum(len(v) for v in agg.values())} launches",
             f"{'kernel':45s} {'launches':>8s} {'avg_us':>10s} {'share':>7s}"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k:45s} {len(v):8d} {sum(v) / len(v) / 1e3:10.2f} {sum(v) / tot:7.3f}")
    out = os.path.join(PROF, f"{tag}_launches.txt")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def report(path, tag):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, data = rows[0], rows[1], rows[2:]
    by = collections.defaultdict(list)
    for r in data:
        by[r[h.index("Kernel Name")].split("(")[0]].append(r)
    for k, rs in by.items():
        lines = [f"# ncu --set full --clock-control none, {os.path.basename(path)}: {k}"]
        for i, r in enumerate(rs):
            lines.append(f"## launch {i}")
            for key in KEYS:
                if key in h:
                    lines.append(f"{key:60s} {r[h.index(key)]:>20s} {units[h.index(key)]}")
        name = k.replace("void ", "").split("::")[-1].replace("<", "_").replace(">", "").strip()
        open(os.path.join(PROF, f"{tag}_ncu_{name}.txt"), "w").write("\n".join(lines) + "\n")
        print("\n".join(lines))
        if name.startswith("k_amul"):
            def mb(key, r):
                v = float(r[h.index(key)])
                u = units[h.index(key)]
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
            tr = [mb("dram__bytes_read.sum", r) + mb("dram__bytes_write.sum", r) for r in rs]
            json.dump({"workload": WORKLOAD, "kernel": k, "round": tag,
                       "amul_dram_bytes_per_launch": sum(tr) / len(tr),
                       "source": f"profiles/{tag}_ncu_{name}.txt"},
                      open(os.path.join(PROF, "ncu_traffic.json"), "w"), indent=1)


if __name__ == "__main__":
    tag = sys.argv[1]
    for a in sys.argv[2:]:
        if a.endswith(".csv"):
            launches(a, tag)
        else:
            report(a, tag)
