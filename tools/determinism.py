"""Determinism probe: the same solve twice in one process and a digest across processes (dev tool)."""
import sys, os, hashlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1705_04531_b200 as lib
from workloads import make_workload
name = sys.argv[1]
wl = make_workload(name)
ie = lib.Ieti.from_workload(wl)
rhs = ie.load_builtin(lib.F_SIN2 if wl.dim == 2 else lib.F_SIN3)
u1, l1, i1, r1, _ = ie.solve(rhs)
u2, l2, i2, r2, _ = ie.solve(rhs)
Phi = ie.primal_basis(0, int(np.prod([len(t) - wl.p - 1 for t in wl.patches[0].knots])))
print(name, "its", i1, i2, "same-process identical:", bool(np.array_equal(u1, u2)), "max diff", float(np.abs(u1 - u2).max()),
      "u digest", hashlib.sha1(u1.tobytes()).hexdigest()[:12], "phi digest", hashlib.sha1(Phi.tobytes()).hexdigest()[:12],
      "rel_res %.6e" % r1)
