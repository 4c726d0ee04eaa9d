"""Diagnostic (GPU): parity error budget of a small case across building blocks and basis tolerances."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1705_04531_b200 as lib
from oracle.ieti import IetiOracle
from workloads import make_workload
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_parity import act_to_lat, lat_to_act, rel, kernel_basis, lat_offsets

name, kw = sys.argv[1], eval(sys.argv[2])
wl = make_workload(name, **kw)
orc = IetiOracle(wl)
ref = orc.solve(tol=1e-8)
fix = orc.solve(fixed_iters=ref.iters)
Q = kernel_basis(orc)
proj = lambda v: v - Q @ (Q.T @ v)
rhs = act_to_lat(orc, orc.f)
print("oracle iters", ref.iters, "n_lambda", orc.topo.n_lambda, "kernel dim", Q.shape[1])
for btol in (1e-12, 1e-13, 1e-14):
    gpu = lib.Ieti.from_workload(wl, basis_tol=btol)
    e_phi = max(rel(gpu.primal_basis(k, pt.n_full)[:, pt.act_idx].T, orc.Phi[k]) for k, pt in enumerate(orc.topo.ptopo) if orc.Phi[k].shape[1])
    lam = np.random.default_rng(3).standard_normal(orc.topo.n_lambda)
    eF = rel(gpu.apply(lib.OP_F, lam), orc.apply_F(lam))
    eM = rel(gpu.apply(lib.OP_MSD, lam), orc.apply_MsD(lam))
    ed = rel(gpu.apply(lib.OP_D, rhs), orc.rhs_d())
    u, l, its, rr, rc = gpu.solve(rhs)
    uf, lf, _ = gpu.solve_fixed(rhs, ref.iters)
    print(f"basis_tol={btol:g} basis_its={gpu.info()[11]} Phi={e_phi:.2e} F={eF:.2e} M={eM:.2e} d={ed:.2e} its={its} "
          f"u={rel(uf, np.concatenate(fix.u)):.2e} lam={rel(lf, fix.lam):.2e} lam_perp={rel(proj(lf), proj(fix.lam)):.2e}")
    gpu.close()
gpu = lib.Ieti.from_workload(wl, basis_tol=1e-13)
uf, lf, _ = gpu.solve_fixed(rhs, ref.iters)
e = lf - fix.lam
Fe = orc.apply_F(e); Fl = orc.apply_F(fix.lam)
print("F-norm rel diff", np.sqrt(abs(e @ Fe)) / np.sqrt(fix.lam @ Fl), " l2 rel", rel(lf, fix.lam))
# sensitivity of the oracle itself: perturb the rhs by 1e-14 relative and rerun
orc.f = [f * (1 + 1e-14 * np.random.default_rng(9).standard_normal(f.shape)) for f in orc.f]
fix2 = orc.solve(fixed_iters=ref.iters)
print("oracle self-sensitivity (rhs perturbed 1e-14): lam", rel(fix2.lam, fix.lam), "u", rel(np.concatenate(fix2.u), np.concatenate(fix.u)))
