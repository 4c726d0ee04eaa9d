"""the paper's 2D experiment shape (Table 1): quarter annulus on 8x4
patches, p = 2, vertex + edge-average primal constraints, outer PCG to 1e-6, local
Neumann solves by MG-PCG to 1e-10 and 2 V-cycles in M_sD (the paper's MG-MG).
The annulus radii and f are unstated in the paper (R15, R16), so iteration counts are compared
qualitatively with the paper's 9 / 10 / 11 / 11 for m = 64 / 128 / 256 / 512.
Prints one JSON line per m (GPU)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_04531_b200 as lib  # noqa: E402
from workloads import make_workload  # noqa: E402

PAPER = {64: 9, 128: 10, 256: 11, 512: 11, 1024: 13}
# usage: paper_replica.py [--grid 4,8] m ...   (Fig. 1(a)'s 8x4 orientation is not stated: radial x angular)
args = sys.argv[1:]
grid = (4, 8)
if args and args[0] == "--grid":
    grid = tuple(int(v) for v in args[1].split(","))
    args = args[2:]
for m in [int(a) for a in args] or [64, 128, 256, 512]:
    wl = make_workload("E1", m=m, grid=grid)
    t0 = time.perf_counter()
    ie = lib.Ieti.from_workload(wl)
    ts = time.perf_counter() - t0
    rhs = ie.load_builtin(lib.F_SIN2)
    ie.solve(rhs)
    t0 = time.perf_counter()
    u, lam, its, rr, rc = ie.solve(rhs)
    tt = time.perf_counter() - t0
    print(json.dumps({"workload": "E1", "m": m, "p": 2, "patches": "%dx%d (radial x angular)" % grid, "dofs_torn": int(ie.ndofs),
                      "outer_iterations": its, "paper_MG_MG_iterations": PAPER.get(m), "rel_res": rr,
                      "solve_s": tt, "setup_s": ts}), flush=True)
    ie.close()
