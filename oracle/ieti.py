"""Inexact IETI-DP (K-level) -- oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows PAPER.md Sec. 2-4 in the K-level form of the north star (reading R1):

  Eq. (6) P:197-201   primal basis  [K C^T; C 0][phibar_j; mu_j] = [0; e_j]   (sparse LU of the KKT matrix)
                      S_PiPi = sum_k R_k^T (Phibar^T K Phibar) R_k, dense Cholesky
  P:163-165, App A.1  Ktilde^{-1} r = Phibar S_PiPi^{-1} Phibar^T r + sum_k P N P^T r,  P = I - Phibar C  (R3)
  Eq. (7) P:219-231   the constrained Neumann solve: x = N(P^T r), projected  (exact mode: KKT solve)
  Eq. (4) P:153-159   F = B Ktilde^{-1} B^T,  d = B Ktilde^{-1} f
  P:161-163           M_sD r = sum_k B_D S^(k) B_D^T r,  S v = K_GG v - K_GI D(K_IG v)
  P:161, P:304-308    CG with M_sD, zero initial guess, stop at ||r_k|| <= tol ||r_0||  (R11)
  App A.1, S:547      recovery u = Ktilde^{-1}(f - B^T lambda)

Local solver modes (R2, R19):
  neumann  = 'vcycle' : N = N_c (c V-cycles of the Neumann hierarchy, K (+alpha Mhat if floating))
             'pcg'    : per-patch PCG on K, preconditioner one Neumann V-cycle, rel. tol inner_tol
             'exact'  : KKT solve of Eq. (7)
  dirichlet= 'vcycle' : D = D_c (c V-cycles of the Dirichlet hierarchy, K_II)
             'exact'  : K_II^{-1} (sparse LU)

Primal basis routes (Eq. (6) has a unique solution, so any accurate method is allowed):
  basis='kkt' : sparse LU of the KKT matrix [K C^T; C 0] (default; 2D and small 3D patches)
  basis='pcg' : A = K + C^T D C (SPD, D = delta I), Z = A^{-1} C^T column by column by PCG with the
                patch's Neumann V-cycle as preconditioner to rel. 1e-13, H = C Z, Phibar = Z H^{-1}
                (used for C5-size 3D patches, whose KKT LU does not fit);
                pinned to the 'kkt' route on small cases (tests/test_oracle_ieti.py).

Patch-local work (assembly, hierarchies, Phibar, and inside every operator the per-patch parts of
Ktilde^{-1} and M_sD) is organised per patch ids (``ids``) behind three hooks -- ``_local_t``,
``_local_w``, ``_local_msd`` -- so that oracle/sharded.py can run the same methods with the patches
spread over processes; the PCG, B, B_D and coarse-solve steps are shared code.

The fixed-cycle result (modes 'vcycle'/'pcg') is pinned in tests/test_oracle_ieti.py to dense
textbook algebra: F^, d^ and M_sD equal the matrices built from (D+L)^-1, (D+U)^-1, the Galerkin
coarse correction and App. A.1's Ktilde^-1; the converged u equals the dense solve of the inexact
dual system; the k-step outer and inner PCG iterates equal their Krylov-Galerkin characterisation.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import assembly, mg
from .topology import Topology

NEUMANN_MODES = ("vcycle", "pcg", "exact")
DIRICHLET_MODES = ("vcycle", "exact")


@dataclasses.dataclass
class SolveResult:
    u: List[np.ndarray]            # per patch, full lattice (Dirichlet entries 0)
    lam: np.ndarray                # canonical multiplier order (R12)
    iters: int
    rel_res: float
    history: List[float]
    inner_iters: List[List[int]]   # C2: per local solve call, per patch inner PCG counts


class IetiOracle:
    def __init__(self, wl, neumann: Optional[str] = None, dirichlet: Optional[str] = None,
                 cycles: Optional[int] = None, dirichlet_cycles: Optional[int] = None,
                 levels: Optional[int] = None, alpha: Optional[float] = None,
                 inner_tol: Optional[float] = None, assemble_load: bool = True, basis: str = "kkt",
                 ids: Optional[List[int]] = None, topo: Optional[Topology] = None, lean: bool = False):
        """ids/topo/lean: internal (oracle/sharded.py) -- build only patches ``ids`` against a given
        global topology; lean drops the matrices the vcycle-mode operators no longer need."""
        self.wl = wl
        self.dim = wl.dim
        self.p = wl.p
        if neumann is None:
            neumann = {0: "vcycle", 1: "pcg", 2: "exact"}[wl.local_mode]
        if dirichlet is None:
            dirichlet = "exact" if neumann == "exact" else "vcycle"
        assert neumann in NEUMANN_MODES and dirichlet in DIRICHLET_MODES
        self.neumann, self.dirichlet = neumann, dirichlet
        self.cycles = wl.cycles if cycles is None else cycles
        self.dcycles = wl.dirichlet_cycles if dirichlet_cycles is None else dirichlet_cycles
        self.alpha = wl.alpha_reg if alpha is None else alpha
        self.inner_tol = wl.inner_tol if inner_tol is None else inner_tol
        self.inner_maxit = wl.inner_maxit
        self.L = mg.num_levels(wl.m) if levels is None else levels
        self.inner_log: List[List[int]] = []
        assert basis in ("kkt", "pcg")
        self.basis = basis
        self.topo = Topology(wl.patches, wl.primal) if topo is None else topo
        n = self.topo.n_patches
        self.ids = list(range(n)) if ids is None else list(ids)
        self.lean = lean
        self._assemble(assemble_load)
        self._local_matrices()
        self._hierarchies()
        self._primal_basis()
        if lean:
            for k in self.ids:                 # vcycle modes never touch these after setup
                self.K_full[k] = self.K[k] = self.K_II[k] = None
            if self.neumann == "vcycle":
                self.kkt = [None] * n

    # -- assembly (Eq. (1)) --------------------------------------------------------------
    def _assemble(self, with_load):
        n = self.topo.n_patches
        self.K_full, self.f_full = [None] * n, [None] * n
        for k in self.ids:
            self.K_full[k], self.f_full[k] = assembly.assemble_patch(self.wl.patches[k],
                                                                     self.wl.f if with_load else None)

    def _local_matrices(self):
        T = self.topo
        n = T.n_patches
        self.K, self.f = [None] * n, [None] * n
        self.K_II, self.K_IG, self.K_GG, self.K_GI = [None] * n, [None] * n, [None] * n, [None] * n
        for k in self.ids:
            pt = T.ptopo[k]
            Ka = self.K_full[k][pt.act_idx][:, pt.act_idx].tocsr()        # Dirichlet elimination
            self.K[k] = Ka
            self.f[k] = self.f_full[k][pt.act_idx].copy()
            if self.lean:
                self.f_full[k] = None
            I, G = pt.interior, pt.gamma
            self.K_II[k] = Ka[I][:, I].tocsc()
            self.K_IG[k] = Ka[I][:, G].tocsr()
            self.K_GG[k] = Ka[G][:, G].tocsr()
            self.K_GI[k] = Ka[G][:, I].tocsr()

    def set_load(self, f_act_list):
        """Replace the (active-dof) patch loads f^(k)."""
        self.f = [np.asarray(v, dtype=np.float64).copy() for v in f_act_list]

    # -- MG hierarchies (R4-R9) ---------------------------------------------------
    def _hierarchies(self):
        T = self.topo
        lvN, lvD, AN, AD = [], [], [], []
        for k in self.ids:
            pa = self.wl.patches[k]
            pt = T.ptopo[k]
            dlo = [(d, 0) in pt.dirichlet_sides for d in range(self.dim)]
            dhi = [(d, 1) in pt.dirichlet_sides for d in range(self.dim)]
            lvN.append(mg.PatchLevels(pa.knots, self.p, self.L, dlo, dhi))
            lvD.append(mg.PatchLevels(pa.knots, self.p, self.L, [True] * self.dim, [True] * self.dim))
            A = self.K[k]
            if pt.floating:                                    # R4: K + alpha*Mhat, floating patches only
                Mh = assembly.parameter_mass(pa)[pt.act_idx][:, pt.act_idx]
                A = (A + self.alpha * Mh).tocsr()
            AN.append(A)
            AD.append(self.K_II[k].tocsr())
        self.levN, self.levD = lvN, lvD        # per patch in ids order
        have = bool(self.ids)                  # a sharded master (oracle/sharded.py) holds no patches
        nu = dict(nu_pre=getattr(self.wl, "nu_pre", 1), nu_post=getattr(self.wl, "nu_post", 1))   # R5
        self.HN = mg.Hierarchy(AN, lvN, lean=self.lean, **nu) if have and self.neumann in ("vcycle", "pcg") else None
        self.HD = mg.Hierarchy(AD, lvD, lean=self.lean, **nu) if have and self.dirichlet == "vcycle" else None
        self.offN = np.cumsum([0] + [self.K[k].shape[0] for k in self.ids])     # offsets in ids order
        self.offD = np.cumsum([0] + [self.K_II[k].shape[0] for k in self.ids])
        if self.dirichlet == "exact":
            self.K_II_lu = [None] * T.n_patches
            for k in self.ids:
                self.K_II_lu[k] = spla.splu(self.K_II[k]) if self.K_II[k].shape[0] else None

    # -- primal basis, Eq. (6) -----------------------------------------------------------
    def _primal_basis(self):
        T = self.topo
        n_p = T.n_patches
        self.Phi, self.mu, self.kkt, self.S_loc = [None] * n_p, [None] * n_p, [None] * n_p, [None] * n_p
        for k in self.ids:
            K, C = self.K[k], T.C[k]
            npk = C.shape[0]
            n = K.shape[0]
            if self.basis == "pcg" and npk:
                self.Phi[k] = self._basis_pcg(k)
                self.mu[k] = None
            else:
                kkt = sp.bmat([[K, C.T], [C, None]], format="csc") if npk else K.tocsc()
                lu = spla.splu(kkt)
                self.kkt[k] = lu
                if npk:
                    rhs = np.zeros((n + npk, npk))
                    rhs[n:, :] = np.eye(npk)
                    sol = lu.solve(rhs)
                    self.Phi[k] = sol[:n, :]
                    self.mu[k] = sol[n:, :]
                else:
                    self.Phi[k] = np.zeros((n, 0))
                    self.mu[k] = np.zeros((0, 0))
            self.S_loc[k] = self.Phi[k].T @ (K @ self.Phi[k])
        if len(self.ids) == n_p:
            self.set_coarse(self.S_loc)

    def set_coarse(self, S_loc):
        """S_PiPi = sum_k R_k^T S_PiPi^(k) R_k, dense Cholesky."""
        T = self.topo
        S = np.zeros((T.n_pi, T.n_pi))
        for k in range(T.n_patches):
            R = T.R[k]
            S[np.ix_(R, R)] += S_loc[k]
        self.S_PiPi = S
        self.S_chol = sla.cho_factor(S, lower=True) if T.n_pi else None

    def _basis_pcg(self, k, tol=1e-13, maxit=2000):
        """Eq. (6) by the A-route of SURVEY O8 (App. A.1): A = K + C^T D C with D = delta I (SPD for
        any delta > 0 since C 1 != 0 on floating patches), Z = A^{-1} C^T by textbook PCG for every
        column (preconditioner: one V-cycle of the patch's Neumann hierarchy; the columns advance
        together, each with its own scalars, and stop at ||r_j|| <= tol ||b_j||), H = C Z,
        Phibar = Z H^{-1}.  Then C Phibar = I and Phibar^T K v = Phibar^T A v = H^{-T} C v = 0 for
        v in ker C, i.e. Eq. (6).  delta = mean diagonal of K (any delta > 0 gives the same Phibar)."""
        T = self.topo
        K, C = self.K[k], T.C[k].tocsr()
        delta = float(K.diagonal().mean())
        A = (K + delta * (C.T @ C)).tocsr()
        pos = self.ids.index(k)
        H1 = _single_patch_view(self.HN, self.offN, pos)
        B = C.T.toarray()                                            # [n, n_Pi^(k)] right-hand sides
        X = np.zeros_like(B)
        R = B.copy()
        Z = H1(R)
        Pv = Z.copy()
        rho = np.einsum("ij,ij->j", R, Z)
        bn = np.linalg.norm(B, axis=0)
        active = np.ones(B.shape[1], dtype=bool)
        for it in range(maxit):
            AP = A @ Pv
            a = np.where(active, rho / np.einsum("ij,ij->j", Pv, AP), 0.0)
            X += a * Pv
            R -= a * AP
            active &= np.linalg.norm(R, axis=0) > tol * bn
            if not active.any():
                break
            Z = H1(R)
            rho_new = np.einsum("ij,ij->j", R, Z)
            beta = np.where(active, rho_new / rho, 0.0)
            Pv = np.where(active, Z + beta * Pv, Pv)
            rho = np.where(active, rho_new, rho)
        else:
            raise RuntimeError(f"primal-basis PCG did not converge on patch {k}")
        H = C @ X
        return np.linalg.solve(H.T, X.T).T                         # Z H^{-1}

    def coarse_solve(self, g):
        return sla.cho_solve(self.S_chol, g) if self.topo.n_pi else np.zeros(0)

    # -- local Neumann solves --------------------------------------------------------------
    def _stack(self, vecs):
        return np.concatenate(vecs) if vecs else np.zeros(0)

    def _split(self, v, off):
        return [v[off[k]:off[k + 1]].copy() for k in range(len(off) - 1)]

    def local_neumann(self, q_list):
        """x^(k) = N^(k)(q^(k)) for every patch of ids (mode-dependent); lists in ids order."""
        if self.neumann == "vcycle":
            x = self.HN.apply_cycles(self._stack(q_list), self.cycles)
            return self._split(x, self.offN)
        if self.neumann == "exact":
            out = []
            for k, q in zip(self.ids, q_list):
                npk = self.topo.C[k].shape[0]
                out.append(self.kkt[k].solve(np.concatenate([q, np.zeros(npk)]))[:len(q)])
            return out
        return self._inner_pcg(q_list)

    def _inner_pcg(self, q_list):
        """R19: independent per-patch PCG on K with one Neumann V-cycle as preconditioner.

        Each patch runs the textbook PCG; all patches advance in lockstep and a patch
        stops at its first iteration with ||res|| <= tol ||q|| (recursive residual).
        """
        npch = len(q_list)
        off = self.offN
        Kblk = sp.block_diag([self.K[k] for k in self.ids], format="csr")
        q = self._stack(q_list)
        x = np.zeros_like(q)
        r = q.copy()
        seg = [slice(off[k], off[k + 1]) for k in range(npch)]
        qn = np.array([np.linalg.norm(q[s]) for s in seg])
        active = qn > 0
        its = np.zeros(npch, dtype=np.int64)

        def dots(a, b):
            return np.array([float(a[s] @ b[s]) for s in seg])

        def bcast(vals):
            return np.concatenate([np.full(off[k + 1] - off[k], vals[k]) for k in range(npch)]) if npch else vals

        z = self.HN.apply_cycles(r, 1)
        pvec = z.copy()
        rho = dots(r, z)
        for it in range(1, self.inner_maxit + 1):
            if not active.any():
                break
            Ap = Kblk @ pvec
            pAp = dots(pvec, Ap)
            alpha = np.where(active, rho / np.where(active, pAp, 1.0), 0.0)
            x = x + bcast(alpha) * pvec
            r = r - bcast(alpha) * Ap
            rn = np.array([np.linalg.norm(r[s]) for s in seg])
            its[active] = it
            done = active & (rn <= self.inner_tol * qn)
            active = active & ~done
            if not active.any():
                break
            z = self.HN.apply_cycles(r, 1)
            rho_new = dots(r, z)
            beta = np.where(active, rho_new / np.where(active, rho, 1.0), 0.0)
            pvec = np.where(bcast(active.astype(float)) > 0, z + bcast(beta) * pvec, pvec)
            rho = np.where(active, rho_new, rho)
        self.inner_log.append([int(i) for i in its])
        return self._split(x, off)

    # -- Ktilde^{-1} (App. A.1, R3) ------------------------------------------------------
    # patch-local hooks (lists over ALL patches, entries of patches outside ids unused)
    def _local_t(self, r_list):
        """t^(k) = Phibar^(k)T r^(k)."""
        out = [None] * self.topo.n_patches
        for k in self.ids:
            out[k] = self.Phi[k].T @ r_list[k]
        return out

    def _local_w(self, r_list, t, uPi):
        """q = r - C^T t (= P^T r); x = N(q); w = x + Phibar (R u_Pi - C x)  (App. A.1, R3)."""
        T = self.topo
        q = [r_list[k] - T.C[k].T @ t[k] for k in self.ids]
        x = self.local_neumann(q)
        w = [None] * T.n_patches
        for k, xk in zip(self.ids, x):
            w[k] = xk + self.Phi[k] @ (uPi[T.R[k]] - T.C[k] @ xk)
        return w

    def _local_msd(self, vG):
        """y_G^(k) = K_GG v_G - K_GI D(K_IG v_G)  (S^(k) of M_sD)."""
        s = [self.K_IG[k] @ vG[k] for k in self.ids]
        zI = self.local_dirichlet(s)
        yG = [None] * self.topo.n_patches
        for k, z in zip(self.ids, zI):
            yG[k] = self.K_GG[k] @ vG[k] - self.K_GI[k] @ z
        return yG

    def ktilde_inv(self, r_list):
        T = self.topo
        t = self._local_t(r_list)
        g = np.zeros(T.n_pi)
        for k in range(T.n_patches):
            np.add.at(g, T.R[k], t[k])
        uPi = self.coarse_solve(g)
        return self._local_w(r_list, t, uPi)

    def apply_F(self, lam):
        T = self.topo
        r = [T.B[k].T @ lam for k in range(T.n_patches)]
        w = self.ktilde_inv(r)
        return sum((T.B[k] @ w[k] for k in range(T.n_patches)), np.zeros(T.n_lambda))

    def rhs_d(self):
        T = self.topo
        w = self.ktilde_inv(self.f)
        return sum((T.B[k] @ w[k] for k in range(T.n_patches)), np.zeros(T.n_lambda))

    # -- scaled Dirichlet preconditioner -------------------------------------------------
    def local_dirichlet(self, s_list):
        """z_I = D(s) per patch of ids (lists in ids order)."""
        if self.dirichlet == "vcycle":
            z = self.HD.apply_cycles(self._stack(s_list), self.dcycles)
            return self._split(z, self.offD)
        return [self.K_II_lu[k].solve(s) if s.size else s for k, s in zip(self.ids, s_list)]

    def apply_MsD(self, r):
        T = self.topo
        v = [T.BD[k].T @ r for k in range(T.n_patches)]
        vG = [v[k][T.ptopo[k].gamma] for k in range(T.n_patches)]
        yG = self._local_msd(vG)
        out = np.zeros(T.n_lambda)
        for k in range(T.n_patches):
            y = np.zeros(len(T.ptopo[k].act_idx))
            y[T.ptopo[k].gamma] = yG[k]
            out += T.BD[k] @ y
        return out

    # -- dual PCG (R11, R20) -------------------------------------------
    def pcg(self, tol=None, maxit=None, fixed_iters=None):
        tol = self.wl.pcg_tol if tol is None else tol
        maxit = self.wl.pcg_maxit if maxit is None else maxit
        self.breakdown = False
        d = self.rhs_d()
        lam = np.zeros_like(d)
        r = d.copy()
        r0 = float(np.linalg.norm(r))
        hist = [r0]
        if fixed_iters is not None:
            maxit, tol = fixed_iters, -1.0
        if r0 == 0.0:
            return lam, 0, 0.0, hist
        z = self.apply_MsD(r)
        pv = z.copy()
        rho = float(r @ z)
        k = 0
        for k in range(1, maxit + 1):
            q = self.apply_F(pv)
            pq = float(pv @ q)
            if not np.isfinite(pq) or pq <= 0.0:
                self.breakdown = True          # reported state, not an exception
                k -= 1
                break
            a = rho / pq
            lam = lam + a * pv
            r = r - a * q
            rn = float(np.linalg.norm(r))
            hist.append(rn)
            if rn <= tol * r0:
                break
            if k == maxit:
                break
            z = self.apply_MsD(r)
            rho_new = float(r @ z)
            beta = rho_new / rho
            rho = rho_new
            pv = z + beta * pv
        return lam, k, hist[-1] / r0, hist

    def recover(self, lam):
        T = self.topo
        r = [self.f[k] - T.B[k].T @ lam for k in range(T.n_patches)]
        w = self.ktilde_inv(r)
        u = []
        for k in range(T.n_patches):
            full = np.zeros(T.ptopo[k].n_full)
            full[T.ptopo[k].act_idx] = w[k]
            u.append(full)
        return u

    def solve(self, tol=None, maxit=None, fixed_iters=None) -> SolveResult:
        self.inner_log = []
        lam, its, rel, hist = self.pcg(tol, maxit, fixed_iters)
        u = self.recover(lam)
        return SolveResult(u, lam, its, rel, hist, list(self.inner_log))

    # -- diagnostics -----------------------------------------------------------------------
    def continuity_residual(self, u):
        T = self.topo
        return float(np.max(np.abs(sum((T.B[k] @ u[k][T.ptopo[k].act_idx] for k in range(T.n_patches)),
                                       np.zeros(T.n_lambda))))) if T.n_lambda else 0.0

    def dense(self, op, n):
        return np.column_stack([op(e) for e in np.eye(n)])


def _single_patch_view(H, off, pos):
    """One V-cycle of the hierarchy restricted to block ``pos`` (a block-diagonal hierarchy's
    V-cycle acts block by block, so applying it to a vector that is zero outside the block and
    reading the block back is the block's own V-cycle)."""
    n = off[-1]

    def apply(r):
        v = np.zeros((n,) + r.shape[1:])
        v[off[pos]:off[pos + 1]] = r
        return H.apply_cycles(v, 1)[off[pos]:off[pos + 1]]
    return apply
