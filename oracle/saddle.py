"""MG-MG-S: Bramble-Pasciak CG on the saddle-point problem Eq. (2) -- oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md Sec. 3.3 and Sec. 4: instead of the dual PCG on
F lambda = d, solve

    [K~  B~^T] [u     ]   [f~]
    [B~  0   ] [lambda] = [0 ]                                      Eq. (2)

in V~_h (primal continuity built in) by BPCG, with a preconditioner K^~ for K~ made of "a few MG
V-cycles" (3 V-cycles) of the regularised MG of P:207-211, scaled below K~, and
F^ = the scaled Dirichlet preconditioner M_sD for the Schur complement.

Readings (R28-R31):
  R28 V~_h is represented inside the torn space: u = (u^(k))_k with C^(k) u^(k) = R_k u_Pi for a
      global u_Pi (= Phibar R u_Pi + w, w^(k) in ker C^(k): the K-orthogonal split of App. A.1).
      Functionals on V~_h are torn vectors r = (r^(k))_k acting by sum_k r^(k).u^(k).  Then
      K~ u = (K^(k) u^(k))_k (true K, Dirichlet dofs eliminated), B~ u = sum_k B^(k) u^(k),
      B~^T lambda = (B^(k)T lambda)_k, f~ = (f^(k))_k -- "at each iteration step we only have to
      apply a given matrix".
  R29 K^~^-1 r = (1/s) (Phibar S_PiPi^-1 Phibar^T r + sum_k P N_3 P^T r), P = I - Phibar C: the
      App. A.1 form of K~^-1 with the local solves replaced by 3 V-cycles (N_3) of the Neumann
      hierarchy (K + alpha Mhat on floating patches, R4) -- "the construction of K^~ follows the
      same steps as in the previous section, but we only apply a few MG V-cycles".
      It maps functionals into V~_h and is unchanged by representatives of the same functional.
  R30 "scaled below K~" (required by BPCG): s = (1 - 0.05) theta_min rounded down to 3 significant
      digits (floor_sig3), theta_min the smallest Ritz
      value of 40 Lanczos steps on K^~_1^-1 K~ (unscaled, from 40 PCG steps on K~ x = b0), b0 the
      counter-based sequence of ``start_vector`` on the concatenated active dofs (the GPU library
      computes the same sequence).  Without an exact coarse block theta_min would be tiny; with it
      K^~_1^-1 K~ has spectrum in (0, 1] (N_3 <= (K + alpha Mhat)^-1).
  R31 BPCG (Bramble & Pasciak 1988): preconditioner P = [[K^~, 0], [B~, -M_sD^-1]], CG in the
      inner product H = diag(K~ - K^~, M_sD^-1) on P^-1 A x = P^-1 b, zero initial guess; stop at
      the first k with ||rho_k||_2 <= tol ||rho_0||_2, rho = (f - K~ u - B~^T lambda, -B~ u) the
      unpreconditioned residual of Eq. (2) (both blocks; cf. R11), its first block kept in the
      null-part-free representative of ``canonical`` (a torn vector is only one representative of
      a functional on V~_h).  delta <= 0 or gamma <= 0 (K^~ not below K~) is a breakdown,
      reported.

Recurrences (one K~, one K^~^-1, one M_sD per iteration):
  a = (can(K~ p_u + B~^T p_l), B~ p_u);  w = K^~^-1 a_u;  delta = a_u.w - p.a;  alpha = gamma / delta
  x += alpha p;  rho -= alpha a;  r_u -= alpha w;  Kr = K~ r_u;  s_l = B~ r_u - rho_l;  r_l = M_sD s_l
  gamma' = r_u.(Kr - rho_u) + r_l.s_l;  beta = gamma'/gamma;  p = r + beta p;  Kp = Kr + beta Kp
with gamma = <r, r>_H = r_u.(K~ r_u - rho_u) + r_l.s_l and delta = <P^-1 A p, p>_H.
"""
from __future__ import annotations

from typing import List

import numpy as np
import scipy.linalg as sla

from .ieti import IetiOracle


def start_vector(n: int) -> np.ndarray:
    """Counter-based start vector of the calibration (R30): v_i = ((i+1) * 2654435761 mod 2^32)/2^32 - 1/2
    (exact integer arithmetic, so the GPU library reproduces it bit for bit)."""
    i = np.arange(1, n + 1, dtype=np.uint64)
    return ((i * np.uint64(2654435761)) % np.uint64(2 ** 32)).astype(np.float64) / 2.0 ** 32 - 0.5


def floor_sig3(x: float) -> float:
    """R30: s rounded DOWN to 3 significant digits, m / 10^k (m integer, 10^k exact): s stays below
    theta_min, and two implementations whose Lanczos estimates differ by rounding (~1e-9 relative)
    get the same s unless theta_min sits within ~1e-9 of a 3-digit boundary."""
    import math
    e = math.floor(math.log10(x))
    k = 2 - e                                    # x * 10^k in [100, 1000)
    if k >= 0:
        m = math.floor(x * float(10 ** k))
        return m / float(10 ** k)
    m = math.floor(x / float(10 ** (-k)))
    return m * float(10 ** (-k))


def _dot(a: List[np.ndarray], b: List[np.ndarray]) -> float:
    return float(sum(float(x @ y) for x, y in zip(a, b)))


class SaddleOracle(IetiOracle):
    """MG-MG-S on the IetiOracle's matrices, hierarchies, primal basis and M_sD."""

    def __init__(self, wl, khat_cycles: int = 3, lanczos_steps: int = 40, margin: float = 0.05, **kw):
        kw.setdefault("neumann", "vcycle")
        kw.setdefault("dirichlet", "vcycle")
        super().__init__(wl, cycles=khat_cycles, **kw)
        self.lanczos_steps, self.margin = lanczos_steps, margin
        self.s = None

    # -- operators of Eq. (2) on V~_h (R28) ----------------------------------------------------
    def apply_Kt(self, u):
        return [self.K[k] @ u[k] for k in range(self.topo.n_patches)]

    def apply_B(self, u):
        T = self.topo
        return sum((T.B[k] @ u[k] for k in range(T.n_patches)), np.zeros(T.n_lambda))

    def apply_Bt(self, lam):
        return [self.topo.B[k].T @ lam for k in range(self.topo.n_patches)]

    def canonical(self, r):
        """The representative of the functional r on V~_h without a null part (R31):
        r^_k = P_k^T r_k + C_k^T W_k R_k g,  g = sum_k R_k^T Phibar_k^T r_k,  W_k = 1 / multiplicity of
        each primal entity.  It acts on u = Phibar R u_Pi + w (w in ker C) as g.u_Pi + sum_k r_k.w_k, i.e.
        like r; a torn vector that annihilates V~_h (on each patch some C^T mu, e.g. B^T of a kernel
        vector of F, R14) maps to 0.  The BPCG keeps every functional it updates in this form:
        otherwise the null parts, O(|f|) and not decaying, meet the O(eps) drift of the iterates
        out of V~_h and break the Bramble-Pasciak inner product at ~1e-10 (observed)."""
        T = self.topo
        g = np.zeros(T.n_pi)
        ts = []
        for k in range(T.n_patches):
            t = self.Phi[k].T @ r[k]
            np.add.at(g, T.R[k], t)
            ts.append(t)
        mult = np.zeros(T.n_pi)
        for k in range(T.n_patches):
            np.add.at(mult, T.R[k], 1.0)
        out = []
        for k in range(T.n_patches):
            out.append(r[k] - T.C[k].T @ ts[k] + T.C[k].T @ (g[T.R[k]] / mult[T.R[k]]))
        return out

    def res_norm(self, rho_u, rho_l):
        return float(np.sqrt(_dot(rho_u, rho_u) + float(rho_l @ rho_l)))

    def apply_Khat_inv(self, r, scaled=True):
        """R29: K^~^-1 r = (1/s) Ktilde^-1_{N_3}(r)."""
        y = self.ktilde_inv(r)
        return [v / self.s for v in y] if scaled else y

    # -- calibration (R30) ------------------------------------------------------------------
    def calibrate(self):
        """theta_min of K^~_1^-1 K~ from the Lanczos matrix of PCG (Golub & Van Loan 11.3.5)."""
        T = self.topo
        sizes = [len(pt.act_idx) for pt in T.ptopo]
        off = np.cumsum([0] + sizes)
        b = start_vector(int(off[-1]))
        r = [b[off[k]:off[k + 1]].copy() for k in range(T.n_patches)]
        z = self.apply_Khat_inv(r, scaled=False)
        p = [v.copy() for v in z]
        rho = rho0 = _dot(r, z)
        alphas, betas = [], []
        for _ in range(self.lanczos_steps):
            q = self.apply_Kt(p)
            a = rho / _dot(p, q)
            r = [x - a * y for x, y in zip(r, q)]
            z = self.apply_Khat_inv(r, scaled=False)
            rho_new = _dot(r, z)
            if rho_new <= 1e-24 * rho0:          # Krylov space exhausted (tiny problems)
                alphas.append(a)
                break
            bta = rho_new / rho
            alphas.append(a)
            betas.append(bta)
            rho = rho_new
            p = [x + bta * y for x, y in zip(z, p)]
        m = len(alphas)
        betas = betas[:m - 1] if len(betas) >= m else betas
        diag = np.array([1.0 / alphas[0]] + [1.0 / alphas[j] + betas[j - 1] / alphas[j - 1] for j in range(1, m)])
        offd = np.array([np.sqrt(betas[j]) / alphas[j] for j in range(m - 1)])
        theta = sla.eigvalsh_tridiagonal(diag, offd)
        self.theta_min, self.theta_max = float(theta[0]), float(theta[-1])
        self.s = floor_sig3((1.0 - self.margin) * self.theta_min)
        return self.s

    # -- BPCG (R31) ---------------------------------------------------------------------------
    def bpcg(self, tol=None, maxit=None, fixed_iters=None):
        tol = self.wl.pcg_tol if tol is None else tol
        maxit = self.wl.pcg_maxit if maxit is None else maxit
        if fixed_iters is not None:
            maxit, tol = fixed_iters, -1.0
        if self.s is None:
            self.calibrate()
        T = self.topo
        off = np.cumsum([0] + [len(pt.act_idx) for pt in T.ptopo])

        def split(v):
            return [v[off[k]:off[k + 1]] for k in range(T.n_patches)]

        def flat(f):
            return lambda v: np.concatenate(f(split(v))) if T.n_patches else v
        u, lam, k, rel, hist, self.breakdown = bpcg(
            A=flat(self.apply_Kt), B=lambda v: self.apply_B(split(v)),
            Bt=lambda l: np.concatenate(self.apply_Bt(l)), Khat_inv=flat(self.apply_Khat_inv),
            Shat_inv=self.apply_MsD, can=flat(self.canonical), f=np.concatenate(self.f),
            n_lambda=T.n_lambda, tol=tol, maxit=maxit)
        return self._full(split(u)), lam, k, rel, hist

    def _full(self, u):
        T = self.topo
        out = []
        for k in range(T.n_patches):
            full = np.zeros(T.ptopo[k].n_full)
            full[T.ptopo[k].act_idx] = u[k]
            out.append(full)
        return out


def bpcg(A, B, Bt, Khat_inv, Shat_inv, can, f, n_lambda, tol, maxit):
    """Bramble-Pasciak CG (R31) for [[A, B^T], [B, 0]] [u; l] = [f; 0] with Khat < A (Khat given by
    its inverse) and a Schur-complement preconditioner Shat^-1; ``can`` maps a functional to the
    representative the iteration keeps (identity for plain vectors).  Returns
    (u, l, iterations, relative residual, residual history, breakdown)."""
    u = np.zeros_like(f)
    lam = np.zeros(n_lambda)
    rho_u, rho_l = can(f), np.zeros(n_lambda)
    r0 = float(np.sqrt(rho_u @ rho_u))
    hist = [r0]
    if r0 == 0.0:
        return u, lam, 0, 0.0, hist, False
    r_u = Khat_inv(rho_u)
    Kr = A(r_u)
    s_l = B(r_u) - rho_l
    r_l = Shat_inv(s_l)
    gamma = float(r_u @ (Kr - rho_u)) + float(r_l @ s_l)       # <r, r>_H
    p_u, p_l, Kp = r_u.copy(), r_l.copy(), Kr.copy()
    k, breakdown = 0, False
    for k in range(1, maxit + 1):
        a_u = can(Kp + Bt(p_l))
        a_l = B(p_u)
        w = Khat_inv(a_u)
        delta = float(a_u @ w) - float(p_u @ a_u) - float(p_l @ a_l)   # <P^-1 A p, p>_H
        if not (np.isfinite(delta) and delta > 0.0 and np.isfinite(gamma) and gamma > 0.0):
            breakdown = True                   # Khat not below A (negative curvature)
            k -= 1
            break
        alpha = gamma / delta
        u = u + alpha * p_u
        lam = lam + alpha * p_l
        rho_u = rho_u - alpha * a_u
        rho_l = rho_l - alpha * a_l
        rn = float(np.sqrt(rho_u @ rho_u + rho_l @ rho_l))
        hist.append(rn)
        if rn <= tol * r0 or k == maxit:
            break
        r_u = r_u - alpha * w
        Kr = A(r_u)
        s_l = B(r_u) - rho_l
        r_l = Shat_inv(s_l)
        gamma_new = float(r_u @ (Kr - rho_u)) + float(r_l @ s_l)
        beta = gamma_new / gamma
        gamma = gamma_new
        p_u = r_u + beta * p_u
        p_l = r_l + beta * p_l
        Kp = Kr + beta * Kp
    return u, lam, k, hist[-1] / r0, hist, breakdown
