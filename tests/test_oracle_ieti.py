"""Pins for oracle/ieti.py (CPU).

* exact IETI-DP == global conforming sparse direct solve (brute force)
* O(h^{p+1}) L2 error of the manufactured solution (north star)
* primal basis: C Phibar = I, K-orthogonality to ker C, sum phi = 1 on floating patches, S = -mu
* F symmetric PSD with the predicted kernel, M_sD SPD, exact vs 2-V-cycle M_sD: +-1 iteration
  (PAPER Tables 1-2: MG-D = D-D)
* fixed-cycle modes: F^, d^, M_sD equal dense textbook matrices (V-cycle from (D+L)^-1, (D+U)^-1,
  Galerkin coarse correction); the converged u equals the dense solve of the inexact dual system;
  k-step PCG residuals equal the Krylov-Galerkin characterisation of CG; C2's inner PCG iterates
  likewise; c -> inf reaches exact
"""
import math

import numpy as np
import pytest

from oracle import assembly, brute
from oracle.ieti import IetiOracle
from workloads import make_workload


def rel_inf(a_list, b_list):
    num = max(float(np.abs(a - b).max()) for a, b in zip(a_list, b_list))
    den = max(float(np.abs(b).max()) for b in b_list)
    return num / den


@pytest.mark.parametrize("name,kw", [("C1", {}), ("STRIP", {}), ("SINGLE", {}), ("C2", dict(m=4)),
                                     ("C3", dict(m=4)), ("C4", dict(m=2)), ("C5", dict(m=2, grid=(2, 2, 2)))])
def test_exact_ieti_equals_global_direct_solve(name, kw):
    wl = make_workload(name, **kw)
    ex = IetiOracle(wl, neumann="exact", dirichlet="exact")
    res = ex.solve(tol=1e-13)
    ub, _ = brute.solve_global(ex)
    assert rel_inf(res.u, ub) <= 1e-10
    assert ex.continuity_residual(res.u) <= 1e-10 * max(np.abs(u).max() for u in ub)


def test_strip_is_pure_feti():
    wl = make_workload("STRIP")
    ex = IetiOracle(wl, neumann="exact", dirichlet="exact")
    assert ex.topo.n_pi == 0
    F = ex.dense(ex.apply_F, ex.topo.n_lambda)
    assert np.allclose(F, F.T, atol=1e-13)
    assert np.all(np.linalg.eigvalsh(F) > 0)


def test_manufactured_solution_rate():
    """L2 error of exact IETI-DP on the C1 geometry converges with order p+1 (>= p + 0.7)."""
    errs = []
    for m in (2, 4, 8):
        wl = make_workload("C1", m=m)
        ex = IetiOracle(wl, neumann="exact", dirichlet="exact")
        res = ex.solve(tol=1e-13)
        e2 = sum(assembly.l2_error(pa, u, wl.u_exact) for pa, u in zip(wl.patches, res.u))
        errs.append(math.sqrt(e2))
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]
    assert min(rates[1:]) >= wl.p + 0.7, rates


def test_manufactured_solution_rate_3d():
    errs = []
    # (3,2,2) patch grid: a mirror-symmetric 2x2x2 split makes d = 0 up to rounding
    for m in (4, 8):
        wl = make_workload("C4", m=m, grid=(3, 2, 2))
        ex = IetiOracle(wl, neumann="exact", dirichlet="exact")
        res = ex.solve(tol=1e-11)
        errs.append(math.sqrt(sum(assembly.l2_error(pa, u, wl.u_exact) for pa, u in zip(wl.patches, res.u))))
    assert math.log2(errs[0] / errs[1]) >= wl.p + 0.7


@pytest.mark.parametrize("name,grid,ms", [("C2", (3, 3), (4, 8, 16)), ("C5", (2, 2, 2), (2, 4, 8))])
def test_manufactured_solution_rate_jittered_maps(name, grid, ms):
    """Curved (non-affine) geometry: the C2 (bilinear, seed 2) and C5 (trilinear, seed 5) jitter
    recipes keep the unit square / cube, so u = prod sin(pi x_d) is the exact solution; exact
    IETI-DP must converge in L2 with order p + 1 (>= p + 0.7; north star O(h^{p+1})).
    This pins the non-affine assembly (J^-T gradhat N): using J^-1 instead gives rate ~0
    (checked by mutation when this test was written)."""
    errs = []
    for m in ms:
        wl = make_workload(name, m=m, grid=grid)
        ex = IetiOracle(wl, neumann="exact", dirichlet="exact")
        res = ex.solve(tol=1e-13)
        errs.append(math.sqrt(sum(assembly.l2_error(pa, u, wl.u_exact) for pa, u in zip(wl.patches, res.u))))
    assert math.log2(errs[-2] / errs[-1]) >= wl.p + 0.7, errs


@pytest.mark.parametrize("name,kw", [("C2", dict(m=4)), ("C3", dict(m=4)), ("C4", dict(m=2)),
                                     ("C5", dict(m=2, grid=(2, 2, 2)))])
def test_primal_basis_properties(name, kw):
    wl = make_workload(name, **kw)
    ex = IetiOracle(wl, neumann="exact", dirichlet="exact")
    T = ex.topo
    rng = np.random.default_rng(0)
    for k in range(T.n_patches):
        Phi, C, K = ex.Phi[k], T.C[k].toarray(), ex.K[k]
        if C.shape[0] == 0:
            continue
        assert np.allclose(C @ Phi, np.eye(C.shape[0]), atol=1e-10)                 # C Phibar = I
        # K-orthogonality to ker C: v in ker C -> Phibar^T K v = 0
        Q, _ = np.linalg.qr(C.T, mode="complete")
        v = Q[:, C.shape[0]:] @ rng.standard_normal(Q.shape[0] - C.shape[0])
        assert np.abs(Phi.T @ (K @ v)).max() <= 1e-9 * np.abs(K @ v).max()
        if T.ptopo[k].floating:
            assert np.abs(Phi.sum(axis=1) - 1.0).max() <= 1e-9                     # sum phi_j = 1
        S = ex.S_loc[k]
        assert np.allclose(S, -ex.mu[k], atol=1e-9 * np.abs(S).max())             # S_PiPi^(k) = -mu
    if T.n_pi:
        assert np.all(np.linalg.eigvalsh(ex.S_PiPi) > 0)


@pytest.mark.parametrize("name,kw", [("C1", {}), ("C4", dict(m=4, grid=(2, 2, 2))), ("C3", dict(m=4, grid=(3, 3)))])
def test_F_and_MsD_spectral_properties(name, kw):
    wl = make_workload(name, **kw)
    ex = IetiOracle(wl)                                   # fixed-cycle mode (inexact F-hat)
    n = ex.topo.n_lambda
    F = ex.dense(ex.apply_F, n)
    M = ex.dense(ex.apply_MsD, n)
    assert np.abs(F - F.T).max() <= 1e-11 * np.abs(F).max()
    assert np.abs(M - M.T).max() <= 1e-11 * np.abs(M).max()
    evF = np.linalg.eigvalsh(0.5 * (F + F.T))
    evM = np.linalg.eigvalsh(0.5 * (M + M.T))
    assert evF.min() >= -1e-10 * evF.max()                # PSD (App. A.2/A.3)
    assert evM.min() >= -1e-12 * evM.max()
    # kernel dimension of F = number of averaged entities' dual pairs ... (App. A.3): with vertex-only
    # primal constraints (C1) F is definite
    if wl.primal == 1:
        assert evF.min() > 1e-8 * evF.max()


@pytest.mark.parametrize("name,kw", [("C1", {}), ("C4", dict(m=4, grid=(2, 2, 2))), ("C2", dict(m=8))])
def test_inexact_preconditioner_changes_iterations_by_at_most_one(name, kw):
    """PAPER Tables 1-2: MG-D (2 V-cycles in M_sD) = D-D iteration counts."""
    wl = make_workload(name, **kw)
    dd = IetiOracle(wl, neumann="exact", dirichlet="exact").solve(tol=1e-8)
    mgd = IetiOracle(wl, neumann="exact", dirichlet="vcycle", dirichlet_cycles=2).solve(tol=1e-8)
    assert abs(dd.iters - mgd.iters) <= 1


def test_fixed_cycle_consistency_and_convergence_to_exact():
    """parity unpinned (fixed-cycle result): internal consistency only."""
    wl = make_workload("C1", m=8)
    ex = IetiOracle(wl, neumann="exact", dirichlet="exact").solve(tol=1e-12)
    prev = None
    for c in (1, 2, 8, 30):
        o = IetiOracle(wl, cycles=c, dirichlet_cycles=c)
        r = o.solve(tol=1e-12)
        assert o.continuity_residual(r.u) <= 1e-9
        err = rel_inf(r.u, ex.u)
        if prev is not None:
            assert err <= prev * 1.01 + 1e-12
        prev = err
    assert prev <= 1e-9


def test_inner_pcg_mode_close_to_exact():
    wl = make_workload("C2", m=8)
    ex = IetiOracle(wl, neumann="exact", dirichlet="exact").solve(tol=1e-10)
    o = IetiOracle(wl)
    assert o.neumann == "pcg"
    r = o.solve(tol=1e-10)
    assert rel_inf(r.u, ex.u) <= 1e-4
    assert all(max(c) <= 200 for c in r.inner_iters)
    assert max(max(c) for c in r.inner_iters) >= 2


def test_zero_rhs_gives_zero_iterations():
    wl = make_workload("C1")
    o = IetiOracle(wl)
    o.set_load([np.zeros_like(f) for f in o.f])
    r = o.solve()
    assert r.iters == 0 and all(np.all(u == 0) for u in r.u)


def test_paper_replica_iteration_band():
    """SURVEY NEXT-4 / S:653: on the shape of the paper's 2D experiment (8x4 quarter-annulus
    patches, p = 2, vertex + edge averages, tol 1e-6, exact local solves) the outer iteration
    count lies in [7, 14] and grows by at most 2 per refinement (paper Table 1: 9, 10, 11, 11
    for m = 64 ... 512)."""
    its = []
    for m in (4, 8):
        wl = make_workload("E1", m=m, grid=(8, 4))
        its.append(IetiOracle(wl, neumann="exact", dirichlet="exact").solve().iters)
    assert all(7 <= k <= 14 for k in its), its
    assert 0 <= its[1] - its[0] <= 2, its


# ---- textbook dense matrices of the fixed-cycle method (pins the fixed-cycle result) ----------
def _dense_vcycle(H, nu_pre=1, nu_post=1):
    """Matrix B_L of one V-cycle from x = 0 on the finest level (O7), built from dense
    textbook factors instead of the oracle's sweeps: forward Gauss-Seidel = (D + L)^{-1} and
    backward = (D + U)^{-1} in colour-major row order (R6), Galerkin coarse correction with the
    hierarchy's P, exact coarsest solve A_0^{-1} (R9):
        X = F + P B_{l-1} P^T (I - A F),   B_l = X + G (I - A X)."""
    A0 = H.A[0].toarray()
    Bm = np.linalg.inv(A0) if A0.shape[0] else A0
    for l in range(1, H.L):
        A = H.A[l].toarray()
        n = A.shape[0]
        perm = np.concatenate(H.colour_rows[l])
        Ap = A[np.ix_(perm, perm)]
        F, G = np.zeros((n, n)), np.zeros((n, n))
        F[np.ix_(perm, perm)] = np.linalg.inv(np.tril(Ap))
        G[np.ix_(perm, perm)] = np.linalg.inv(np.triu(Ap))
        P = H.P[l].toarray()
        Fn = F.copy()                                  # nu_pre forward sweeps from x = 0 (R5)
        for _ in range(nu_pre - 1):
            Fn = Fn + F @ (np.eye(n) - A @ Fn)
        X = Fn + P @ Bm @ P.T @ (np.eye(n) - A @ Fn)
        for _ in range(nu_post):                       # nu_post backward sweeps
            X = X + G @ (np.eye(n) - A @ X)
        Bm = X
    return Bm


def _dense_cycles(H, c):
    """N_c: c steps of x <- x + B (b - A x) from x = 0 (R10)."""
    A = H.A[H.L - 1].toarray()
    B1 = _dense_vcycle(H)
    N = B1.copy()
    for _ in range(c - 1):
        N = N + B1 @ (np.eye(A.shape[0]) - A @ N)
    return N


def _dense_system(o):
    """Ktilde^-1 = Phi S^-1 Phi^T + P N_c P^T (App. A.1, R3), F = B Ktilde^-1 B^T, d = B Ktilde^-1 f
    (Eq. (4)), M_sD = sum B_D (K_GG - K_GI D_c K_IG) B_D^T as dense matrices."""
    T = o.topo
    off = np.cumsum([0] + [K.shape[0] for K in o.K])
    n = off[-1]
    Phi = np.zeros((n, T.n_pi))
    Pm = np.zeros((n, n))
    for k in range(T.n_patches):
        s = slice(off[k], off[k + 1])
        Phi[s, T.R[k]] += o.Phi[k]
        Pm[s, s] = np.eye(off[k + 1] - off[k]) - o.Phi[k] @ T.C[k].toarray()
    S = np.zeros((T.n_pi, T.n_pi))
    for k in range(T.n_patches):
        S[np.ix_(T.R[k], T.R[k])] += o.Phi[k].T @ (o.K[k] @ o.Phi[k])
    N = _dense_cycles(o.HN, o.cycles)
    Kti = (Phi @ np.linalg.solve(S, Phi.T) if T.n_pi else 0.0) + Pm @ N @ Pm.T
    B = np.hstack([T.B[k].toarray() for k in range(T.n_patches)])
    f = np.concatenate(o.f)
    D = _dense_cycles(o.HD, o.dcycles)
    offD = np.cumsum([0] + [K.shape[0] for K in o.K_II])
    M = np.zeros((T.n_lambda, T.n_lambda))
    for k in range(T.n_patches):
        pt = T.ptopo[k]
        Dk = D[offD[k]:offD[k + 1], offD[k]:offD[k + 1]]
        Sk = o.K_GG[k].toarray() - o.K_GI[k].toarray() @ Dk @ o.K_IG[k].toarray()
        BG = T.BD[k].toarray()[:, pt.gamma]
        M += BG @ Sk @ BG.T
    return Kti, B, f, B @ Kti @ B.T, B @ Kti @ f, M, off


@pytest.mark.parametrize("name,kw", [("C1", {}), ("C4", dict(m=4, grid=(2, 2, 2))), ("C2", dict(m=4)),
                                     ("C5", dict(m=2, grid=(2, 2, 2)))])
def test_fixed_cycle_method_equals_textbook_dense_algebra(name, kw):
    """Pins the fixed-cycle (inexact) result: the oracle's F^, d^, M_sD equal the dense textbook
    matrices above; its converged u equals u* = Ktilde^-1 (f - B^T lam*) with F^ lam* = d^ solved
    densely; and after k PCG steps its residual equals the Galerkin (Krylov) characterisation of
    CG (R11): lam_k in K_k(M F, M d) with V^T (d - F lam_k) = 0."""
    wl = make_workload(name, **kw)
    o = IetiOracle(wl, neumann="vcycle")
    Kti, B, f, F, d, M, off = _dense_system(o)
    n = o.topo.n_lambda
    sc = np.abs(F).max()
    assert np.abs(o.dense(o.apply_F, n) - F).max() <= 1e-11 * sc
    assert np.abs(o.dense(o.apply_MsD, n) - M).max() <= 1e-11 * np.abs(M).max()
    assert np.abs(o.rhs_d() - d).max() <= 1e-11 * np.abs(d).max()
    # converged solution = dense solve of the inexact dual system (u is unique, App. A.3)
    lam_s = np.linalg.lstsq(F, d, rcond=1e-13)[0]
    u_s = Kti @ (f - B.T @ lam_s)
    res = o.solve(tol=1e-13, maxit=500)
    u_o = np.concatenate([u[pt.act_idx] for u, pt in zip(res.u, o.topo.ptopo)])
    assert np.abs(u_o - u_s).max() <= 1e-9 * np.abs(u_s).max()
    # k-step PCG iterate: Galerkin condition on the preconditioned Krylov space
    for k in (1, 2, 3, 5):
        Q = _arnoldi(lambda v: M @ (F @ v), M @ d, k)
        lam_k = Q @ np.linalg.lstsq(Q.T @ F @ Q, Q.T @ d, rcond=1e-13)[0]
        fix = o.solve(fixed_iters=k)
        r_o, r_k = d - F @ fix.lam, d - F @ lam_k
        assert np.linalg.norm(r_o - r_k) <= 1e-9 * np.linalg.norm(d), k


def _arnoldi(op, v0, k):
    """Orthonormal basis of the Krylov space span{v0, op v0, ..., op^(k-1) v0} (Gram-Schmidt twice)."""
    Q = [v0 / np.linalg.norm(v0)]
    for _ in range(k - 1):
        w = op(Q[-1])
        for _ in range(2):
            for qv in Q:
                w = w - (qv @ w) * qv
        Q.append(w / np.linalg.norm(w))
    return np.column_stack(Q)


def test_inner_pcg_iterates_equal_krylov_galerkin():
    """Pins C2's inner PCG (R19): per patch, the iterate after its logged count k lies in the
    Krylov space K_k(N_1 K, N_1 q) (N_1 = the dense textbook V-cycle) and satisfies the Galerkin
    condition V^T (q - K x) = 0 (K x compared: unique also on floating patches), and the count is
    the first k with ||q - K x_k|| <= inner_tol ||q||."""
    wl = make_workload("C2", m=4)
    o = IetiOracle(wl)
    assert o.neumann == "pcg"
    rng = np.random.default_rng(11)
    q = []
    for pt, K in zip(o.topo.ptopo, o.K):
        v = rng.standard_normal(K.shape[0])
        q.append(v - v.mean() if pt.floating else v)        # consistent on floating patches
    x = o._inner_pcg(q)
    its = o.inner_log[-1]
    N1 = _dense_cycles(o.HN, 1)
    off = o.offN
    for k, (qk, xk, K) in enumerate(zip(q, x, o.K)):
        Kd = K.toarray()
        Nk = N1[off[k]:off[k + 1], off[k]:off[k + 1]]
        Q = _arnoldi(lambda v: Nk @ (Kd @ v), Nk @ qk, its[k])
        xg = Q @ np.linalg.lstsq(Q.T @ Kd @ Q, Q.T @ qk, rcond=1e-13)[0]
        assert np.linalg.norm(Kd @ xk - Kd @ xg) <= 1e-9 * np.linalg.norm(qk), k
        assert np.linalg.norm(qk - Kd @ xk) <= o.inner_tol * np.linalg.norm(qk)
        if its[k] > 1:                                       # not converged one step earlier
            Q1 = Q[:, :its[k] - 1]
            x1 = Q1 @ np.linalg.lstsq(Q1.T @ Kd @ Q1, Q1.T @ qk, rcond=1e-13)[0]
            assert np.linalg.norm(qk - Kd @ x1) > o.inner_tol * np.linalg.norm(qk)


@pytest.mark.parametrize("name,kw", [("C4", dict(m=4, grid=(2, 2, 2))), ("C2", dict(m=8, grid=(2, 2)))])
def test_vcycle_with_more_smoothing_steps_equals_textbook(name, kw):
    """R5 with nu_pre = nu_post = 2 (the boundary's nu_1, nu_2): one V-cycle of the oracle equals
    the dense textbook V-cycle with two (D+L)^-1 sweeps before and two (D+U)^-1 sweeps after the
    Galerkin coarse correction; it stays symmetric and contracts better than nu = 1."""
    wl = make_workload(name, **kw)
    wl.nu_pre, wl.nu_post = 2, 2
    o = IetiOracle(wl, neumann="vcycle", dirichlet="vcycle")
    A = o.HN.A[o.HN.L - 1].toarray()
    n = A.shape[0]
    V2 = np.column_stack([o.HN.apply_cycles(e, 1) for e in np.eye(n)])
    assert np.abs(V2 - _dense_vcycle(o.HN, 2, 2)).max() <= 1e-10 * np.abs(V2).max()
    assert np.abs(V2 - V2.T).max() <= 1e-10 * np.abs(V2).max()
    wl1 = make_workload(name, **kw)
    o1 = IetiOracle(wl1, neumann="vcycle", dirichlet="vcycle")
    V1 = np.column_stack([o1.HN.apply_cycles(e, 1) for e in np.eye(n)])
    rho = lambda V: max(abs(np.linalg.eigvals(np.eye(n) - V @ A)))
    assert rho(V2) < rho(V1) < 1.0
