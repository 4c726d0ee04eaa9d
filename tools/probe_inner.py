"""Probe: inner-PCG counts and per-solve time of a paper-replica variant (dev tool)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1705_04531_b200 as lib
from workloads import make_workload
name, m, p, grid = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), tuple(int(v) for v in sys.argv[4].split(","))
wl = make_workload(name, m=m, grid=grid, p=p)
wl.local_mode, wl.inner_tol, wl.inner_maxit = 1, 1e-10, 500
ie = lib.Ieti.from_workload(wl)
info = ie.info()
rhs = ie.load_builtin(lib.F_SIN2 if wl.dim == 2 else lib.F_SIN3)
ie.solve(rhs)
t0 = time.perf_counter(); u, lam, its, rr, rc = ie.solve(rhs); t = time.perf_counter() - t0
lg = ie.inner_log()
print(json.dumps({"levels": int(info[6]), "outer": its, "solve_s": t, "calls": int(lg.shape[0]),
                  "inner_max_per_call": [int(v) for v in lg.max(axis=1)][:20],
                  "inner_total": int(lg.max(axis=1).sum())}))
