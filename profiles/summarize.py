"""Summarise ncu reports / launch lists into the small files committed here.

    python profiles/summarize.py full  <report.ncu-rep> <out.md>
    python profiles/summarize.py launches <launches.csv> <out.md> [regex]

``full`` keeps per-kernel duration, DRAM bytes, hit rates, issue activity,
occupancy and the top stall reasons; ``launches`` keeps every launch of our
kernels with its device time and its share of the listed total.
"""

from __future__ import annotations

import csv
import io
import re
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def full(rep: str, out: str) -> None:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary of `{rep.split('/')[-1]}`", ""]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        lines.append(f"## {name.split('(')[0]}")
        for m in FULL_METRICS:
            if m in hdr:
                lines.append(f"- {m}: {r[hdr.index(m)]} {units[hdr.index(m)]}")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        top = ", ".join(f"{n} {int(v)}" for v, n in sorted(stalls, reverse=True)[:6])
        lines.append(f"- top stall samples: {top}")
        lines.append("")
    with open(out, "w") as f:
        f.write("\n".join(lines))


def launches(path: str, out: str,
             pattern: str = r"translate|plan_kernel|stamp_kernel|exec|shim|stage_table|fifo|ordered|frame|index|"
                            r"encode|map_|pair|classify|identify|cub::|Device") -> None:
    rows = list(csv.reader(open(path)))
    hdr = None
    items = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                items.append((int(d["ID"]), d["Kernel Name"], float(d["Metric Value"]), d["Metric Unit"]))
    mine = [x for x in items if re.search(pattern, x[1])]
    total = sum(x[2] for x in mine) or 1.0
    lines = [f"# launch list (ncu gpu__time_duration.sum, --clock-control none) from `{path.split('/')[-1]}`", "",
             "cold-cache, serialised replay: compare shares, not absolutes", "",
             "| id | kernel | time | share of listed |", "|---|---|---|---|"]
    for i, n, t, u in mine:
        lines.append(f"| {i} | {n.split('(')[0]} | {t:.1f} {u} | {100 * t / total:.1f}% |")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3])
    else:
        launches(sys.argv[2], sys.argv[3], *sys.argv[4:])
