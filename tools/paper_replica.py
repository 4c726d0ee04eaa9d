"""the paper's experiment shapes on the GPU, MG-MG variant (Neumann MG-PCG to
1e-10, 2 Dirichlet V-cycles), outer PCG to 1e-6.

  E1: Table 1: 2D quarter annulus on 8x4 patches, p = 2, vertex + edge averages.
  E2: Table 2: 3D annulus on 4x4x8 patches, p = 2, edge averages only; the paper's
      domain is twisted and the twist is undefined, so E2 is the untwisted extrusion.

Annulus radii and f are unstated (R15, R16): iteration counts are compared with the paper's
MG-MG column.  One JSON line per m.

  python tools/paper_replica.py [--workload E1|E2] [--grid a,b[,c]] m ...
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_04531_b200 as lib  # noqa: E402
from workloads import make_workload  # noqa: E402

PAPER = {"E1": {64: 9, 128: 10, 256: 11, 512: 11, 1024: 13},       # Table 1, p = 2, MG-MG
         "E2": {4: 11, 8: 12, 16: 14, 32: 16}}                     # Table 2, p = 2, MG-MG
args = sys.argv[1:]
name, grid = "E1", None
while args and args[0].startswith("--"):
    if args[0] == "--workload":
        name = args[1]
    elif args[0] == "--grid":
        grid = tuple(int(v) for v in args[1].split(","))
    args = args[2:]
ms = [int(a) for a in args] or ([64, 128, 256, 512] if name == "E1" else [4, 8, 16])
for m in ms:
    wl = make_workload(name, m=m, grid=grid)
    t0 = time.perf_counter()
    ie = lib.Ieti.from_workload(wl)
    ts = time.perf_counter() - t0
    rhs = ie.load_builtin(lib.F_SIN2 if wl.dim == 2 else lib.F_SIN3)
    ie.solve(rhs)
    t0 = time.perf_counter()
    u, lam, its, rr, rc = ie.solve(rhs)
    tt = time.perf_counter() - t0
    print(json.dumps({"workload": name, "m": m, "p": wl.p, "patches": "x".join(str(g) for g in wl.grid),
                      "dofs_torn": int(ie.ndofs), "outer_iterations": its,
                      "paper_MG_MG_iterations": PAPER[name].get(m), "rel_res": rr, "solve_s": tt,
                      "setup_s": ts}), flush=True)
    ie.close()
