"""Small solves through the C ABI for compute-sanitizer (memcheck / racecheck / initcheck):
every kernel of the hot path and of the setup runs at least once on tiny multi-patch cases."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1705_04531_b200 as lib  # noqa: E402
from workloads import make_workload  # noqa: E402

CASES = [("C1", {}), ("C4", dict(m=4, grid=(3, 2, 2))), ("C5", dict(m=4, grid=(3, 2, 2))),
         ("C2", dict(m=16, grid=(3, 3))), ("C3", dict(m=8, grid=(4, 3)))]
for name, kw in CASES:
    wl = make_workload(name, **kw)
    ie = lib.Ieti.from_workload(wl, basis_tol=1e-12)
    rhs = ie.load_builtin(lib.F_SIN2 if wl.dim == 2 else lib.F_SIN3)
    u, lam, its, rr, rc = ie.solve(rhs)
    for op in (lib.OP_F, lib.OP_MSD):
        ie.apply(op, np.ones(ie.n_lambda))
    ie.apply(lib.OP_NEUMANN, rhs)
    ie.apply(lib.OP_DIRICHLET, rhs)
    print(name, "its", its, "rel_res", rr, flush=True)
    ie.close()
print("sanitize run ok")
