"""Write the CPU oracle's full-size reference results (tests/golden/full/<CONFIG>.npz).

Calls only ``oracle/`` and ``workloads/`` (no CUDA path).  For each
BASELINE.json config at its full size and the product defaults (R2, R7, R19, BASELINE tol 1e-8):

  * the converged dual PCG run (R11): iteration count k, residual history,
    relative residual;
  * u (full patch lattices) and lambda (canonical order, R12) after those k iterations, which is
    the fixed-iteration result of R20 (the same iterate: PCG stops at k either way);
  * the oracle's torn load f (rhs of ieti_solve, full lattices) so the GPU solves the oracle's
    right-hand side;
  * the averaged-entity kernel vectors of F (R14) as sparse rows, so the test can
    compare lambda on range(F);
  * C2 only: the per-call, per-patch inner PCG counts (R19).

usage: python tools/oracle_dump.py C2 C4 C3 [--out tests/golden/full]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.ieti import IetiOracle          # noqa: E402
from workloads import make_workload         # noqa: E402


def kernel_vectors(topo):
    """R14 / App. A.3: per averaged primal entity e and chain link (k_i, k_{i+1}) of its patches,
    lambda_r = w_a on the rows r = (k_i, a) - (k_{i+1}, a).  Returns CSR-like (ptr, rows, vals)."""
    row_of = {(kp, fp, km): r for r, (kp, fp, km, fm) in enumerate(topo.mult)}
    ptr, rows, vals = [0], [], []
    for e in topo.primal:
        if e.kind == "vertex":
            continue
        ks = sorted(e.members)
        for k1, k2 in zip(ks[:-1], ks[1:]):
            for a, w in zip(e.members[k1], e.weights[k1]):
                rows.append(row_of[(k1, int(a), k2)])
                vals.append(w)
            ptr.append(len(rows))
    return (np.array(ptr, dtype=np.int64), np.array(rows, dtype=np.int64), np.array(vals, dtype=np.float64))


def dump(name, out_dir):
    t0 = time.time()
    wl = make_workload(name)
    orc = IetiOracle(wl)
    t1 = time.time()
    res = orc.solve(tol=wl.pcg_tol)
    t2 = time.time()
    T = orc.topo
    f_lat = []
    for k, pt in enumerate(T.ptopo):
        v = np.zeros(pt.n_full)
        v[pt.act_idx] = orc.f[k]
        f_lat.append(v)
    kp, kr, kv = kernel_vectors(T)
    path = os.path.join(out_dir, f"{name}.npz")
    np.savez_compressed(
        path, name=name, iters=res.iters, rel_res=res.rel_res, history=np.array(res.history),
        u=np.concatenate(res.u), lam=res.lam, f=np.concatenate(f_lat),
        n_full=np.array([pt.n_full for pt in T.ptopo]), n_lambda=T.n_lambda, n_pi=T.n_pi, levels=orc.L,
        kernel_ptr=kp, kernel_rows=kr, kernel_vals=kv,
        inner_iters=np.array(res.inner_iters, dtype=np.int32) if res.inner_iters else np.zeros((0, 0), np.int32),
        continuity=orc.continuity_residual(res.u), setup_s=t1 - t0, solve_s=t2 - t1,
        generator="tools/oracle_dump.py (oracle/ only)")
    print(f"{name}: iters={res.iters} rel_res={res.rel_res:.3e} setup {t1 - t0:.1f} s solve {t2 - t1:.1f} s "
          f"-> {path} ({os.path.getsize(path) / 1e6:.1f} MB)", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "full"))
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    for c in a.configs:
        dump(c.upper(), a.out)
