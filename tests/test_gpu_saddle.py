"""MG-MG-S on the GPU (outer_mode BPCG: Bramble-Pasciak CG on the saddle point Eq. (2),
P:249-253; readings R28-R31) against the oracle (oracle/saddle.py).

Building blocks element-wise: K~ (true K on torn vectors, 1e-12), the null-part-free
representative and K^~^-1 (both read the full primal basis iterated to the paper's 1e-12,
P:309: 1e-10 like Phibar), the calibration (theta of K^~_1^-1 K~ from the same counter-based
start vector to 1e-7 -- Ritz values of a 40-step Lanczos process carry the rounding of 40
operator applications -- and s, rounded down to 3 digits by R30, identical).  End to end: +-1 BPCG iteration at tol 1e-8 (north star), u and
lambda (on range F, R14) within 1e-9 after the oracle's iteration count (R20), and the solution
equals the global conforming direct solve (BPCG only preconditions; K~ is exact)."""
import numpy as np
import pytest

from oracle import brute
from oracle.saddle import SaddleOracle
from tests.conftest import parity_log
from workloads import make_workload

pytestmark = pytest.mark.gpu

CASES = {
    "C1": ("C1", dict()),
    "E1s": ("E1", dict(m=8, grid=(2, 4))),
    "C4s": ("C4", dict(m=4, grid=(3, 2, 2))),
    "E2s": ("E2", dict(m=4, grid=(2, 2, 2))),
    "C5s": ("C5", dict(m=4, grid=(3, 2, 2))),
}
_cache = {}


def rel(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def systems(case):
    if case in _cache:
        return _cache[case]
    import paper_1705_04531_b200 as lib
    name, kw = CASES[case]
    wl = make_workload(name, **kw)
    wl.local_mode = 0                     # MG-MG-S: fixed V-cycles only (R29)
    orc = SaddleOracle(wl)                # K^~: 3 V-cycles, M_sD: 2 Dirichlet V-cycles
    orc.calibrate()
    gpu = lib.Ieti.from_workload(wl, cycles=3, outer_mode=lib.OUTER_BPCG)
    _cache[case] = (wl, orc, gpu)
    return _cache[case]


def to_lat(orc, vecs):
    offs = np.cumsum([0] + [pt.n_full for pt in orc.topo.ptopo])
    out = np.zeros(offs[-1])
    for k, v in enumerate(vecs):
        out[offs[k] + orc.topo.ptopo[k].act_idx] = v
    return out


def to_act(orc, lat):
    offs = np.cumsum([0] + [pt.n_full for pt in orc.topo.ptopo])
    return [lat[offs[k] + pt.act_idx] for k, pt in enumerate(orc.topo.ptopo)]


@pytest.mark.parametrize("case", list(CASES))
def test_bpcg_building_blocks(case):
    import paper_1705_04531_b200 as lib
    wl, orc, gpu = systems(case)
    s, tmin, tmax, steps = gpu.bpcg_info()
    parity_log(test="bpcg_calibration", case=case, s_gpu=s, s_oracle=orc.s, theta_min_gpu=tmin,
               theta_min_oracle=orc.theta_min, theta_max_gpu=tmax, theta_max_oracle=orc.theta_max, steps=steps)
    # theta from 40 Lanczos steps carries the rounding of 40 operator applications (~1e-9 here);
    # s is rounded down to 3 significant digits (R30), so both sides use the same s
    assert abs(tmin - orc.theta_min) <= 1e-7 * orc.theta_min and abs(tmax - orc.theta_max) <= 1e-7
    assert s == orc.s, (s, orc.s)
    rng = np.random.default_rng(4)
    r = [rng.standard_normal(len(pt.act_idx)) for pt in orc.topo.ptopo]
    got = to_act(orc, gpu.apply(lib.OP_KT, to_lat(orc, r)))
    assert rel(np.concatenate(got), np.concatenate(orc.apply_Kt(r))) <= 1e-12
    got = to_act(orc, gpu.apply(lib.OP_CAN, to_lat(orc, r)))
    assert rel(np.concatenate(got), np.concatenate(orc.canonical(r))) <= 1e-10
    got = to_act(orc, gpu.apply(lib.OP_KHAT, to_lat(orc, r)))
    assert rel(np.concatenate(got), np.concatenate(orc.apply_Khat_inv(r))) <= 1e-10


@pytest.mark.parametrize("case", list(CASES))
def test_bpcg_solve_parity(case):
    import paper_1705_04531_b200 as lib
    wl, orc, gpu = systems(case)
    rhs = to_lat(orc, orc.f)
    u_ref, lam_ref, k_ref, rr_ref, hist = orc.bpcg(tol=wl.pcg_tol)      # E1/E2: the paper's 1e-6
    assert not orc.breakdown
    u, lam, its, rr, rc = gpu.solve(rhs)
    assert rc == lib.OK and abs(its - k_ref) <= 1, (its, k_ref)
    uf, lf, rrf = gpu.solve_fixed(rhs, k_ref)
    err_u = rel(uf, np.concatenate(u_ref))
    # lambda on range(F) (R14): the averaged-entity kernel vectors, disjoint supports
    T = orc.topo
    row_of = {(kp, fp, km): i for i, (kp, fp, km, fm) in enumerate(T.mult)}
    Q = []
    for e in T.primal:
        if e.kind == "vertex":
            continue
        ks = sorted(e.members)
        for k1, k2 in zip(ks[:-1], ks[1:]):
            v = np.zeros(T.n_lambda)
            for a, w in zip(e.members[k1], e.weights[k1]):
                v[row_of[(k1, int(a), k2)]] = w
            Q.append(v / np.linalg.norm(v))
    Q = np.array(Q).T if Q else np.zeros((T.n_lambda, 0))
    proj = lambda v: v - Q @ (Q.T @ v)
    # lambda is an interface force: where its exact value vanishes (C1 is symmetric, lambda = 0 up to
    # rounding, |lambda| ~ 1e-12 |f|) its error is measured against the load's scale
    err_l = float(np.linalg.norm(proj(lf) - proj(lam_ref)) /
                  max(np.linalg.norm(proj(lam_ref)), np.linalg.norm(np.concatenate(orc.f))))
    parity_log(test="bpcg_solve", case=case, iters_gpu=its, iters_oracle=k_ref, err_u=err_u, err_lam_range=err_l,
               rel_res_gpu=rrf, rel_res_oracle=rr_ref)
    assert err_u <= 1e-9 and err_l <= 1e-9, (err_u, err_l)
    assert abs(rrf - rr_ref) <= 1e-2 * rr_ref
    # BPCG solves Eq. (2) itself: at tol 1e-10 the GPU solution is the Galerkin solution of Eq. (1)
    gpu_tight = lib.Ieti.from_workload(wl, cycles=3, outer_mode=lib.OUTER_BPCG, pcg_tol=1e-10)
    try:
        ut = gpu_tight.solve(rhs)[0]
    finally:
        gpu_tight.close()
    ub, _ = brute.solve_global(orc)
    assert rel(ut, np.concatenate(ub)) <= 1e-8
