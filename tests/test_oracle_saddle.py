"""Pins for oracle/saddle.py (MG-MG-S: BPCG on the saddle point Eq. (2)).

* the generic BPCG equals a dense KKT factorisation on SPEC's toy and on random
  saddle systems with Khat < A (dense augmented-system oracle, 1e-8; here 1e-10)
* a Khat that is NOT below A is detected as a breakdown (negative curvature)
* MG-MG-S reaches the exact Galerkin solution of Eq. (1): the converged u equals the global
  conforming sparse direct solve (brute force) -- BPCG only preconditions, K~ is exact
* the calibration: K^~_1^-1 K~ has spectrum in (0, 1] (App. A.2: N_3 <= (K + alpha Mhat)^-1 and an
  exact coarse block), and s is below every sampled Rayleigh quotient (K^~ < K~, R30)
* the canonical representative (R31) acts on V~_h like the original and kills null functionals
"""
import numpy as np
import pytest

from oracle import brute
from oracle.saddle import SaddleOracle, _dot, bpcg, start_vector
from workloads import make_workload


def test_bpcg_spec_toy():
    """K~ = diag(2,2), B~ = [1 -1], K^ = 0.5 I, F^ = exact Schur -> converges, u1 = u2."""
    A = np.diag([2.0, 2.0])
    Bm = np.array([[1.0, -1.0]])
    f = np.array([1.0, 3.0])
    S = Bm @ np.linalg.solve(A, Bm.T)
    u, lam, k, rel, hist, brk = bpcg(lambda v: A @ v, lambda v: Bm @ v, lambda l: Bm.T @ l,
                                     lambda r: r / 0.5, lambda s: np.linalg.solve(S, s), lambda r: r,
                                     f, 1, 1e-14, 50)
    assert not brk and abs(u[0] - u[1]) <= 1e-13
    kkt = np.block([[A, Bm.T], [Bm, np.zeros((1, 1))]])
    ref = np.linalg.solve(kkt, np.concatenate([f, [0.0]]))
    assert np.allclose(np.concatenate([u, lam]), ref, atol=1e-13)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_bpcg_equals_dense_kkt(seed):
    rng = np.random.default_rng(seed)
    n, m = 40, 12
    Q = rng.standard_normal((n, n))
    A = Q @ Q.T + n * np.eye(n)
    Bm = rng.standard_normal((m, n))
    lam_min = np.linalg.eigvalsh(A)[0]
    Kh = 0.9 * lam_min * np.eye(n) + 0.0        # Khat = 0.9 lambda_min I < A
    Sh = Bm @ np.linalg.solve(A, Bm.T) + 0.3 * np.eye(m)
    f = rng.standard_normal(n)
    u, lam, k, rel, hist, brk = bpcg(lambda v: A @ v, lambda v: Bm @ v, lambda l: Bm.T @ l,
                                     lambda r: np.linalg.solve(Kh, r), lambda s: np.linalg.solve(Sh, s),
                                     lambda r: r, f, m, 1e-13, 500)
    kkt = np.block([[A, Bm.T], [Bm, np.zeros((m, m))]])
    ref = np.linalg.solve(kkt, np.concatenate([f, np.zeros(m)]))
    assert not brk
    assert np.linalg.norm(np.concatenate([u, lam]) - ref) <= 1e-10 * np.linalg.norm(ref)
    # a Khat above A (violating the BPCG condition) is reported, not silently wrong
    Kbad = 2.0 * np.linalg.eigvalsh(A)[-1] * np.eye(n)
    *_, brk2 = bpcg(lambda v: A @ v, lambda v: Bm @ v, lambda l: Bm.T @ l,
                    lambda r: np.linalg.solve(Kbad, r), lambda s: np.linalg.solve(Sh, s),
                    lambda r: r, f, m, 1e-13, 500)
    assert brk2


CASES = [("C1", {}), ("E1", dict(m=8, grid=(2, 4))), ("C4", dict(m=4, grid=(3, 2, 2))),
         ("E2", dict(m=4, grid=(2, 2, 2))), ("C5", dict(m=2, grid=(3, 2, 2)))]


@pytest.mark.parametrize("name,kw", CASES)
def test_mgmgs_reaches_the_galerkin_solution(name, kw):
    wl = make_workload(name, **kw)
    o = SaddleOracle(wl)
    # tol 1e-10: below ~1e-11 the Bramble-Pasciak inner product of the 3D p = 3 case loses its
    # sign to rounding (reported as a breakdown, as it must be); the product runs at 1e-8 / 1e-6
    u, lam, its, rr, hist = o.bpcg(tol=1e-10, maxit=500)
    assert not o.breakdown and rr <= 1e-10
    ub, _ = brute.solve_global(o)
    err = max(np.abs(a - b).max() for a, b in zip(u, ub)) / max(np.abs(b).max() for b in ub)
    assert err <= 1e-8, err
    # spectrum of the unscaled preconditioned operator in (0, 1] (App. A.2) and s below it (R30)
    assert 0.0 < o.theta_min <= o.theta_max <= 1.0 + 1e-10
    rng = np.random.default_rng(3)
    for _ in range(10):
        r = [rng.standard_normal(len(pt.act_idx)) for pt in o.topo.ptopo]
        x = o.apply_Khat_inv(r, scaled=False)
        assert _dot(x, o.apply_Kt(x)) / _dot(x, r) > o.s


def test_canonical_representative():
    wl = make_workload("C4", m=4, grid=(3, 2, 2))
    o = SaddleOracle(wl)
    T = o.topo
    rng = np.random.default_rng(0)
    r = [rng.standard_normal(len(pt.act_idx)) for pt in T.ptopo]
    c = o.canonical(r)
    # same action on V~_h (K^~^-1 outputs span V~_h)
    for _ in range(3):
        v = o.apply_Khat_inv([rng.standard_normal(len(pt.act_idx)) for pt in T.ptopo], scaled=False)
        assert abs(_dot(r, v) - _dot(c, v)) <= 1e-12 * np.sqrt(_dot(r, r) * _dot(v, v))
    # B^T of a kernel vector of F (an averaged entity, R14) is a null functional on V~_h
    e = next(e for e in T.primal if e.kind != "vertex")
    k1, k2 = sorted(e.members)[:2]
    row_of = {(kp, fp, km): i for i, (kp, fp, km, fm) in enumerate(T.mult)}
    lam = np.zeros(T.n_lambda)
    for a, w in zip(e.members[k1], e.weights[k1]):
        lam[row_of[(k1, int(a), k2)]] = w
    null = o.apply_Bt(lam)
    assert np.sqrt(_dot(null, null)) > 0.1
    cn = o.canonical(null)
    assert np.sqrt(_dot(cn, cn)) <= 1e-13
    # idempotent
    cc = o.canonical(c)
    assert max(np.abs(a - b).max() for a, b in zip(cc, c)) <= 1e-13 * max(np.abs(a).max() for a in c)


def test_start_vector_is_the_counter_sequence():
    v = start_vector(5)
    want = [((i * 2654435761) % 2 ** 32) / 2 ** 32 - 0.5 for i in range(1, 6)]
    assert np.array_equal(v, np.array(want))
