"""Experiment: is C3's lambda deviation from the oracle (full size) the primal basis tolerance?
GPU fixed-iteration solves at basis_tol 1e-12 (product default) and 1e-14 against the committed oracle
dump; prints the relative errors of u and of lambda on range(F)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1705_04531_b200 as lib  # noqa: E402
from tests.test_gpu_full_size import range_projector, rel  # noqa: E402
from workloads import make_workload  # noqa: E402

d = np.load("tests/golden/full/C3.npz")
wl = make_workload("C3")
proj = range_projector(d, None)
for bt in (1e-12, 1e-13, 1e-14):
    ie = lib.Ieti.from_workload(wl, basis_tol=bt)
    uf, lf, rr = ie.solve_fixed(d["f"], int(d["iters"]))
    its = ie.solve(d["f"])[2]
    print(json.dumps({"basis_tol": bt, "iters_gpu": its, "iters_oracle": int(d["iters"]), "err_u": rel(uf, d["u"]),
                      "err_lam_range": rel(proj(lf), proj(d["lam"])), "rel_res": rr}), flush=True)
    ie.close()
