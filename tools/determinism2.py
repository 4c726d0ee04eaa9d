"""Determinism probe 2: digests of every setup product (dev tool)."""
import sys, os, hashlib, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1705_04531_b200 as lib
from workloads import make_workload
name = sys.argv[1]
wl = make_workload(name)
ie = lib.Ieti.from_workload(wl)
H = lambda a: hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()[:10]
nf = int(np.prod([len(t) - wl.p - 1 for t in wl.patches[0].knots]))
out = {"map": H(np.concatenate(ie.multiplier_map()))}
for h in (0, 1):
    out["st%d" % h] = [H(np.concatenate([ie.stencil(h, l, k).ravel() for k in range(ie.n_patches)])) for l in range(ie.levels)]
out["phi"] = H(np.concatenate([ie.primal_basis(k, nf).ravel() for k in range(ie.n_patches)]))
rng = np.random.default_rng(1)
lam = rng.standard_normal(ie.n_lambda)
out["F"] = H(ie.apply(lib.OP_F, lam)); out["M"] = H(ie.apply(lib.OP_MSD, lam))
q = rng.standard_normal(ie.ndofs)
out["N"] = H(ie.apply(lib.OP_NEUMANN, q)); out["V1"] = H(ie.apply(lib.OP_VCYCLE_N, q)); out["D"] = H(ie.apply(lib.OP_DIRICHLET, q))
print(name, json.dumps(out))
