#!/usr/bin/env python
"""Summarise ncu reports / launch lists into profiles/ (committed evidence).
usage: python tools/ncu_summary.py OUT.md [--launches launches.csv] [REPORT.ncu-rep ...]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = dict(zip(h, v))
        u = dict(zip(h, units))
        res.append((d.get("Kernel Name", "?"), {k: (d.get(k, ""), u.get(k, "")) for k in KEYS},
                    sorted(((k.replace("smsp__average_warps_issue_stalled_", "").replace(
                        "_per_issue_active.ratio", ""), float(x or 0)) for k, x in d.items()
                        if "average_warps_issue_stalled" in k and "per_issue_active" in k),
                        key=lambda t: -t[1])[:6]))
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            agg[r[ki]].append(float(r[vi].replace(",", "")))
    return agg


def main():
    out = sys.argv[1]
    args = sys.argv[2:]
    lines = []
    if args and args[0] == "--launches":
        agg = launches(args[1])
        args = args[2:]
        lines.append("## Launch list (ncu gpu__time_duration.sum, cold-cache, serialised)\n")
        lines.append("| launches | avg µs | kernel |\n|---:|---:|---|")
        for k, v in agg.items():
            lines.append(f"| {len(v)} | {sum(v) / len(v) / 1000:.2f} | `{k[:110]}` |")
        lines.append("")
    for p in args:
        for name, m, stalls in report(p):
            lines.append(f"## `{name[:110]}`\n\nfrom `{p}`\n")
            lines.append("| metric | value | unit |\n|---|---:|---|")
            for k, (v, u) in m.items():
                if v:
                    lines.append(f"| {k} | {v} | {u} |")
            lines.append("\ntop stall reasons (cycles per issued instruction): " +
                         ", ".join(f"{k} {v:.2f}" for k, v in stalls) + "\n")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
