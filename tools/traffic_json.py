#!/usr/bin/env python
"""Write profiles/<round>/ncu_traffic.json from an ncu launch list (dram bytes per launch of the
finest-level colour-SGS phases, the bench's roofline kernel class).

  python tools/traffic_json.py <launches.csv> <source-label> [round, default r02]
"""
import csv
import json
import os
import sys
import collections

path, label = sys.argv[1], sys.argv[2]
rnd = sys.argv[3] if len(sys.argv) > 3 else "r02"
rows = list(csv.reader(open(path)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
ii, ki, mi, vi, ui = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
per = collections.defaultdict(dict)
names = {}
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    if r[mi].startswith("dram__bytes"):
        v *= {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[ui], 1.0)
    per[r[ii]][r[mi]] = v
    names[r[ii]] = r[ki]
sel = [i for i, n in names.items() if any(f"k_stencil<3, 3, 1, {m}," in n for m in (0, 4, 6, 7))]
tot = sum(per[i].get("dram__bytes_read.sum", 0) + per[i].get("dram__bytes_write.sum", 0) for i in sel)
out = {"C5": {"dram_bytes_per_launch": tot / max(1, len(sel)), "launches": len(sel),
              "source": label + ": ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over one fixed-iteration "
                        "C5 solve, finest-level k_stencil<3,3,1,{0,4,6,7}> launches (cold-cache serialised)"}}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
json.dump(out, open(os.path.join(root, "profiles", rnd, "ncu_traffic.json"), "w"), indent=1)
print(json.dumps(out))
