#!/usr/bin/env python
"""Summarise ncu outputs for profiles/: a launch list CSV (gpu__time_duration per launch) into
per-kernel totals and shares, and an ncu-rep (--set full) into the key per-launch counters.

  python tools/ncu_summary.py launches <launches.csv>
  python tools/ncu_summary.py full <report.ncu-rep>
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, 1e-3)
        v *= scale
        name = r[ki].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    print(f"{'kernel':52s} {'launches':>8s} {'total_us':>12s} {'avg_us':>9s} {'share':>6s}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:52]:52s} {n:8d} {t:12.1f} {t / n:9.2f} {100 * t / tot:5.1f}%")
    print(f"{'TOTAL':52s} {sum(n for n, _ in agg.values()):8d} {tot:12.1f}")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, data = rows[0], rows[1], rows[2:]
    for r in data:
        print("---")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {k:64s} {r[i]} {units[i]}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
