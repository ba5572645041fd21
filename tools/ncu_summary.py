#!/usr/bin/env python
"""Summarise ncu captures for profiles/: per kernel launch, the metrics that
explain an HBM-bound stencil (time, DRAM bytes, throughput, occupancy,
registers, instructions, L2/L1 traffic, top stall reasons).

    python tools/ncu_summary.py gpurun_out/dense_full7.ncu-rep > profiles/r1_dense_step.md
    python tools/ncu_summary.py --launches gpurun_out/launches_dense.csv
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "lts__t_bytes.sum",
    "l1tex__t_bytes.sum",
    "launch__grid_size",
    "launch__block_size",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    header, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": r[header.index("Kernel Name")]}
        for k in KEYS:
            if k in header:
                i = header.index(k)
                d[k] = (r[i], units[i])
        res.append(d)
    return res


def to_float(v, unit):
    x = float(str(v).replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
             "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}.get(unit, 1)
    return x * scale


def summarise(rep):
    lines = [f"# ncu --set full summary: `{rep}`", ""]
    for d in raw(rep):
        lines.append(f"## {d['kernel'][:160]}")
        t = to_float(*d["gpu__time_duration.sum"])
        rd = to_float(*d["dram__bytes_read.sum"])
        wr = to_float(*d["dram__bytes_write.sum"])
        lines.append(f"- duration: {t * 1e3:.4f} ms (cold cache, serialised replay)")
        lines.append(f"- DRAM read {rd / 1e9:.4f} GB, write {wr / 1e9:.4f} GB, "
                     f"traffic {(rd + wr) / 1e9:.4f} GB -> {(rd + wr) / t / 1e9:.1f} GB/s")
        for k in KEYS[3:]:
            if k in d:
                lines.append(f"- {k}: {d[k][0]} {d[k][1]}")
        lines.append("")
    return "\n".join(lines)


def launches(path):
    """Per-kernel mean device time from an ncu --metrics gpu__time_duration.sum CSV log."""
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    agg = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"]
        agg.setdefault(k, []).append(to_float(r["Metric Value"], r["Metric Unit"]))
    total = sum(sum(v) for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append({"kernel": k[:120], "launches": len(v), "mean_ms": round(sum(v) / len(v) * 1e3, 4),
                    "share": round(sum(v) / total, 4)})
    return out


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(json.dumps(launches(sys.argv[2]), indent=1))
    else:
        print(summarise(sys.argv[1]))
