"""the paper's experiment shapes on the GPU, outer PCG to 1e-6, in the
paper's variants: MG-MG (Neumann MG-PCG to 1e-10, 2 Dirichlet V-cycles),
MG-D (Neumann solves to 1e-12, 2 Dirichlet V-cycles), D-D (both to 1e-12; R27: MG-PCG to
machine accuracy stands in for the paper's direct solvers) and MG-MG-S (BPCG on the
saddle point Eq. (2), K^ = 3 V-cycles, F^ = M_sD).

  E1: Table 1: 2D quarter annulus on 8x4 patches, p = 2, vertex + edge averages.
  E2: Table 2: 3D annulus on 4x4x8 patches, p = 2, edge averages only; the paper's
      domain is twisted and the twist is undefined, so E2 is the untwisted extrusion.

Annulus radii and f are unstated (R15, R16): iteration counts are compared with the paper's
MG-MG column.  One JSON line per m.

  python tools/paper_replica.py [--workload E1|E2] [--grid a,b[,c]] [--p P] [--variant DD,MGD,MGMG,MGMGS,DDX,MGDX|all] m ...
  (DDX / MGDX: D-D / MG-D with the banded-Cholesky direct local solvers instead of R27's MG-PCG)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_04531_b200 as lib  # noqa: E402
from workloads import make_workload  # noqa: E402

# paper iteration counts [variant][(p, m)] (Table 1; Table 2)
PAPER = {"E1": {"DD": {(2, 64): 9, (2, 128): 10, (2, 256): 11, (2, 512): 11,
                       (7, 32): 10, (7, 64): 11, (7, 128): 12, (7, 256): 13},
                "MGD": {(2, 64): 9, (2, 128): 10, (2, 256): 11, (2, 512): 11,
                        (7, 32): 10, (7, 64): 11, (7, 128): 12, (7, 256): 13},
                "MGMG": {(2, 64): 9, (2, 128): 10, (2, 256): 11, (2, 512): 11, (2, 1024): 13,
                         (7, 32): 10, (7, 64): 11, (7, 128): 12, (7, 256): 14, (7, 512): 15},
                "MGMGS": {(2, 64): 14, (2, 128): 15, (2, 256): 16, (2, 512): 15,
                          (7, 32): 14, (7, 64): 15, (7, 128): 17, (7, 256): 18, (7, 512): 20}},
         "E2": {"DD": {(2, 4): 11, (2, 8): 12, (2, 16): 14, (4, 4): 13, (4, 8): 15, (4, 16): 16},
                "MGD": {(2, 4): 11, (2, 8): 12, (2, 16): 14, (2, 32): 16, (4, 4): 13, (4, 8): 15, (4, 16): 17},
                "MGMG": {(2, 4): 11, (2, 8): 12, (2, 16): 14, (2, 32): 16, (4, 4): 13, (4, 8): 15, (4, 16): 17,
                         (4, 32): 19},
                "MGMGS": {(2, 4): 25, (2, 8): 26, (2, 16): 30, (2, 32): 35, (4, 4): 23, (4, 8): 28, (4, 16): 32,
                          (4, 32): 37}}}
# variants (R27): local Neumann / Dirichlet solves
VARIANTS = {"DD": dict(inner_tol=1e-12, dirichlet_mode=lib.DIRICHLET_PCG, dirichlet_tol=1e-12),
            "MGD": dict(inner_tol=1e-12),
            "MGMG": dict(inner_tol=1e-10),
            "MGMGS": dict(outer_mode=lib.OUTER_BPCG, cycles=3),
            # the paper's direct local solvers as batched banded Cholesky factorisations
            "DDX": dict(local_mode=lib.LOCAL_DIRECT, dirichlet_mode=lib.DIRICHLET_DIRECT),
            "MGDX": dict(local_mode=lib.LOCAL_DIRECT)}
PAPER["E1"]["DDX"], PAPER["E1"]["MGDX"] = PAPER["E1"]["DD"], PAPER["E1"]["MGD"]
PAPER["E2"]["DDX"], PAPER["E2"]["MGDX"] = PAPER["E2"]["DD"], PAPER["E2"]["MGD"]
args = sys.argv[1:]
name, grid, p, variants = "E1", None, None, ["MGMG"]
while args and args[0].startswith("--"):
    if args[0] == "--workload":
        name = args[1]
    elif args[0] == "--grid":
        grid = tuple(int(v) for v in args[1].split(","))
    elif args[0] == "--p":
        p = int(args[1])
    elif args[0] == "--variant":
        variants = list(VARIANTS) if args[1] == "all" else args[1].split(",")
    args = args[2:]
ms = [int(a) for a in args] or ([64, 128, 256, 512] if name == "E1" else [4, 8, 16])
for m in ms:
    for var in variants:
        wl = make_workload(name, m=m, grid=grid, p=p)
        kw = dict(VARIANTS[var])
        if var in ("MGMGS", "DDX", "MGDX"):
            wl.local_mode = lib.LOCAL_VCYCLES
        else:
            wl.local_mode, wl.inner_tol = lib.LOCAL_PCG, kw.pop("inner_tol")
        wl.inner_maxit = 500
        t0 = time.perf_counter()
        ie = lib.Ieti.from_workload(wl, **kw)
        ts = time.perf_counter() - t0
        rhs = ie.load_builtin(lib.F_SIN2 if wl.dim == 2 else lib.F_SIN3)
        ie.solve(rhs)
        t0 = time.perf_counter()
        u, lam, its, rr, rc = ie.solve(rhs)
        tt = time.perf_counter() - t0
        print(json.dumps({"workload": name, "variant": var, "m": m, "p": wl.p,
                          "patches": "x".join(str(g) for g in wl.grid), "dofs_torn": int(ie.ndofs),
                          "outer_iterations": its, "paper_iterations": PAPER[name][var].get((wl.p, m)),
                          "rel_res": rr, "solve_s": tt, "setup_s": ts}), flush=True)
        ie.close()
