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
    ii, ki, mi, vi, ui = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    per = collections.defaultdict(dict)          # launch id -> {metric: value}
    names = {}
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        if r[mi].startswith("gpu__time_duration"):
            v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, 1e-3)
        else:                                    # bytes -> MB
            v *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1e-6)
        per[r[ii]][r[mi]] = v
        names[r[ii]] = r[ki].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for lid, m in per.items():
        a = agg[names[lid]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':44s} {'launches':>8s} {'total_us':>11s} {'avg_us':>9s} {'share':>6s} {'DRAM_MB':>10s} {'GB/s':>7s}")
    for k, (n, t, mb) in sorted(agg.items(), key=lambda x: -x[1][1]):
        gbs = mb / t * 1e3 if t > 0 else 0.0
        print(f"{k[:44]:44s} {n:8d} {t:11.1f} {t / n:9.2f} {100 * t / tot:5.1f}% {mb:10.1f} {gbs:7.0f}")
    print(f"{'TOTAL':44s} {sum(a[0] for a in agg.values()):8d} {tot:11.1f}")


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
