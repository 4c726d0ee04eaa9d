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
  * C2 only: the per-call, per-patch inner PCG counts (R19);
  * the oracle's own sensitivity (R26): the relative change of u and of lambda on range(F) when its
    load is perturbed by 1e-14 (seeded), or the output of every d^ / F^ / M_sD application by 1e-14
    (seeded: a rounding-level change of summation order in each application), and the same k
    iterations are run.

usage: python tools/oracle_dump.py C2 C4 C3 [--out tests/golden/full]
       python tools/oracle_dump.py C5 --workers 12 --mem-gb 13 --sample 16 --n-sens 1   (16-core host)
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


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def range_projector(ptr, rows, vals):
    """Orthogonal projector onto range(F) = (ker F)^perp: the kernel vectors have disjoint supports."""
    seg = np.repeat(np.arange(len(ptr) - 1), np.diff(ptr))
    nrm = np.sqrt(np.bincount(seg, weights=vals * vals, minlength=len(ptr) - 1))
    q = vals / np.where(nrm[seg] > 0, nrm[seg], 1.0)

    def proj(v):
        coef = np.bincount(seg, weights=q * v[rows], minlength=len(ptr) - 1)
        out = v.copy()
        out[rows] -= q * coef[seg]
        return out
    return proj


def dump(name, out_dir, n_sens=2, workers=0, mem_gb=None, sample=0, wl_kw=None):
    """workers > 0: the patch-sharded oracle (oracle/sharded.py; same arithmetic, PCG primal-basis
    route), and with sample > 0 only that many whole patches of u (seeded choice) are stored."""
    t0 = time.time()
    wl = make_workload(name, **(wl_kw or {}))
    if workers:
        from oracle.sharded import ShardedIetiOracle
        orc = ShardedIetiOracle(wl, workers=workers, mem_gb_per_worker=mem_gb)
    else:
        orc = IetiOracle(wl)
    print(f"{name}: setup done in {time.time() - t0:.1f} s", flush=True)
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
    # the oracle's own rounding sensitivity (R26): the same k iterations with the load perturbed by
    # 1e-14 (relative, seeded); relative changes of u and of lambda on range(F)
    proj = range_projector(kp, kr, kv)
    f0 = [v.copy() for v in orc.f]
    sens_u, sens_l = 0.0, 0.0
    for seed in (11, 12)[:n_sens]:
        rng = np.random.default_rng(seed)
        orc.set_load([v * (1.0 + 1e-14 * rng.standard_normal(v.shape)) for v in f0])
        pr = orc.solve(fixed_iters=res.iters)
        sens_u = max(sens_u, rel(np.concatenate(pr.u), np.concatenate(res.u)))
        sens_l = max(sens_l, rel(proj(pr.lam), proj(res.lam)))
    orc.set_load(f0)
    # ... and with every operator application perturbed at rounding level: the outputs of d^, F^ and
    # M_sD multiplied entrywise by (1 + 1e-14 xi), xi ~ N(0, 1) seeded -- a different summation order
    # in each application, as in any other implementation of the same method (R26)
    sens_au, sens_al = 0.0, 0.0
    if n_sens and not workers:
        base = {nm: getattr(orc, nm) for nm in ("apply_F", "apply_MsD", "rhs_d")}
        for seed in (31, 32)[:n_sens]:
            rng = np.random.default_rng(seed)

            def noisy(fn):
                return lambda *a: (lambda v: v * (1.0 + 1e-14 * rng.standard_normal(v.shape)))(fn(*a))
            for nm, fn in base.items():
                setattr(orc, nm, noisy(fn))
            pr = orc.solve(fixed_iters=res.iters)
            sens_au = max(sens_au, rel(np.concatenate(pr.u), np.concatenate(res.u)))
            sens_al = max(sens_al, rel(proj(pr.lam), proj(res.lam)))
        for nm in base:
            delattr(orc, nm)                           # back to the class methods
    t3 = time.time()
    path = os.path.join(out_dir, f"{name}.npz")
    if sample:
        # whole patches of a seeded sample (corner patch 0 and the grid's middle patch included)
        mid = sum(g // 2 * int(np.prod(wl.grid[:d])) for d, g in enumerate(wl.grid))
        pick = np.random.default_rng(2024).choice(T.n_patches, sample - 2, replace=False)
        sel = np.unique(np.concatenate([[0, mid], pick]))
        fields = dict(u_patches=sel, u_sample=np.concatenate([res.u[k] for k in sel]),
                      f_sample=np.concatenate([f_lat[k] for k in sel]))
    else:
        fields = dict(u=np.concatenate(res.u), f=np.concatenate(f_lat))
    np.savez_compressed(
        path, name=name, iters=res.iters, rel_res=res.rel_res, history=np.array(res.history),
        lam=res.lam, **fields,
        n_full=np.array([pt.n_full for pt in T.ptopo]), n_lambda=T.n_lambda, n_pi=T.n_pi, levels=orc.L,
        kernel_ptr=kp, kernel_rows=kr, kernel_vals=kv,
        inner_iters=np.array(res.inner_iters, dtype=np.int32) if res.inner_iters else np.zeros((0, 0), np.int32),
        continuity=orc.continuity_residual(res.u), setup_s=t1 - t0, solve_s=t2 - t1,
        sens_u=max(sens_u, sens_au), sens_lam=max(sens_l, sens_al), sens_u_load=sens_u, sens_lam_load=sens_l,
        sens_u_apply=sens_au, sens_lam_apply=sens_al, n_sens=n_sens, sens_s=t3 - t2,
        generator="tools/oracle_dump.py (oracle/ only)")
    if workers:
        orc.close()
    print(f"{name}: iters={res.iters} rel_res={res.rel_res:.3e} setup {t1 - t0:.1f} s solve {t2 - t1:.1f} s "
          f"sensitivity (load) u {sens_u:.2e} lambda {sens_l:.2e} (per application) u {sens_au:.2e} "
          f"lambda {sens_al:.2e} "
          f"-> {path} ({os.path.getsize(path) / 1e6:.1f} MB)", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "full"))
    ap.add_argument("--workers", type=int, default=0, help="patch-sharded oracle with this many processes")
    ap.add_argument("--mem-gb", type=float, default=None, help="address-space limit per worker")
    ap.add_argument("--sample", type=int, default=0, help="store u on this many whole patches only")
    ap.add_argument("--n-sens", type=int, default=2, help="perturbed re-solves for the sensitivity")
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    for c in a.configs:
        dump(c.upper(), a.out, n_sens=a.n_sens, workers=a.workers, mem_gb=a.mem_gb, sample=a.sample)
