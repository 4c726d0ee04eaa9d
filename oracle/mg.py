"""Geometric multigrid on nested dyadic spline grids -- oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Readings:
  R4  fine operator K (+ alpha*Mhat on floating patches, alpha = 1e-2)
  R5  nu_pre forward colour sweeps before, nu_post backward colour sweeps after the coarse
      correction (default 1 / 1)
  R6  colour(i) = sum_d (i_d mod (p+1)) (p+1)^d on the FULL-lattice multi-index (0-based);
      forward = colours ascending; rows of one colour updated simultaneously
  R7  L = max(2, log2(m/4) + 1) levels (coarsest: 4 elements per direction, C1: 2)
  R8  Galerkin coarse operators A_{l-1} = P_l^T A_l P_l
  R9  exact coarsest solve (dense Cholesky)
  R10 N_c(b): c steps of x <- V_L(x, b) from x = 0

A hierarchy is stored for a *set* of patches as block-diagonal matrices (one block
per patch).  A colour phase on the block-diagonal operator is, by definition,
the simultaneous colour phase of every patch, so this is the same algorithm.
"""
from __future__ import annotations

import math
from typing import List

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from . import bspline
from .topology import unravel


def num_levels(m: int) -> int:
    """R7."""
    return max(2, int(round(math.log2(m / 4))) + 1)


def level_knots(t, p, L):
    """Knot vectors of levels 0..L-1 (0 coarsest) by dyadic coarsening of t."""
    ks = [np.asarray(t, dtype=np.float64)]
    for _ in range(L - 1):
        ks.append(bspline.coarsen_dyadic(ks[-1], p))
    return ks[::-1]


def kron_dirs(mats):
    """Kronecker product with direction 1 fastest (first factor innermost)."""
    out = sp.csr_matrix(mats[0])
    for A in mats[1:]:
        out = sp.kron(sp.csr_matrix(A), out, format="csr")
    return out


def active_box_mask(M, lo, hi):
    """Full-lattice mask of the box prod [lo_d, hi_d)."""
    n = int(np.prod(M))
    mask = np.zeros(n, dtype=bool)
    for flat in range(n):
        idx = unravel(flat, M)
        mask[flat] = all(lo[d] <= idx[d] < hi[d] for d in range(len(M)))
    return mask


def colours_of(M, p):
    """R6 colour of every full-lattice index."""
    n = int(np.prod(M))
    col = np.zeros(n, dtype=np.int64)
    for flat in range(n):
        idx = unravel(flat, M)
        c, s = 0, 1
        for d in range(len(M)):
            c += (idx[d] % (p + 1)) * s
            s *= (p + 1)
        col[flat] = c
    return col


class PatchLevels:
    """One patch's hierarchy data: per level full dims, active mask, P (trimmed), colours."""

    def __init__(self, knots, p, L, dirichlet_lo, dirichlet_hi):
        # dirichlet_lo[d] / dirichlet_hi[d]: True if the side i_d = 0 / i_d = M-1 is eliminated
        self.dim = len(knots)
        self.p = p
        kn = [level_knots(t, p, L) for t in knots]
        self.M, self.mask, self.colour, self.P = [], [], [], []
        for l in range(L):
            M = tuple(len(kn[d][l]) - p - 1 for d in range(self.dim))
            lo = [1 if dirichlet_lo[d] else 0 for d in range(self.dim)]
            hi = [M[d] - 1 if dirichlet_hi[d] else M[d] for d in range(self.dim)]
            self.M.append(M)
            self.mask.append(active_box_mask(M, lo, hi))
            self.colour.append(colours_of(M, p)[self.mask[-1]])
        for l in range(1, L):
            Pd = [bspline.knot_insertion_matrix(kn[d][l - 1], p, kn[d][l]) for d in range(self.dim)]
            Pfull = kron_dirs(Pd)
            # trim: rows of eliminated fine dofs and columns of eliminated coarse dofs (exact for open knots)
            self.P.append(Pfull[self.mask[l]][:, self.mask[l - 1]].tocsr())


class Hierarchy:
    """Block-diagonal MG hierarchy over a list of patches (levels 0..L-1, L-1 finest)."""

    def __init__(self, A_fine_blocks: List[sp.csr_matrix], levels: List[PatchLevels], lean: bool = False,
                 nu_pre: int = 1, nu_post: int = 1):
        """lean: keep each level's rows only once (split by colour, ``rowsets``) and form the residual
        b - A x colour block by colour block from them -- the same row dot products in the same
        order as the CSR product (each colour block holds A's rows unchanged), i.e. bitwise equal;
        it halves the memory of full-size (C5) hierarchies."""
        self.L = len(levels[0].M)
        self.p = levels[0].p
        self.nu_pre, self.nu_post = nu_pre, nu_post         # R5: forward / backward sweeps per level
        self.ncol = (self.p + 1) ** levels[0].dim
        self.sizes = []                        # per level, per patch block size
        self.A = [None] * self.L
        self.P = [None] * self.L               # P[l]: level l-1 -> l
        self.A[self.L - 1] = sp.block_diag(A_fine_blocks, format="csr")
        for l in range(1, self.L):
            self.P[l] = sp.block_diag([lv.P[l - 1] for lv in levels], format="csr")
        for l in range(self.L - 1, 0, -1):
            self.A[l - 1] = (self.P[l].T @ self.A[l] @ self.P[l]).tocsr()   # R8 Galerkin
        self.colour_rows = []
        for l in range(self.L):
            col = np.concatenate([lv.colour[l] for lv in levels])
            self.colour_rows.append([np.nonzero(col == c)[0] for c in range(self.ncol)])
        self.diag = [A.diagonal() for A in self.A]
        self.rowsets = [[self.A[l][rows] for rows in self.colour_rows[l]] for l in range(self.L)]
        self.shape = [A.shape[0] for A in self.A]
        # coarsest: dense Cholesky per patch block (R9)
        sizes0 = [int(lv.mask[0].sum()) for lv in levels]
        self.coarse_slices = []
        off = 0
        A0 = self.A[0].toarray() if self.A[0].shape[0] else np.zeros((0, 0))
        self.coarse_chol = []
        for s in sizes0:
            blk = A0[off:off + s, off:off + s]
            self.coarse_slices.append(slice(off, off + s))
            self.coarse_chol.append(sla.cho_factor(blk, lower=True) if s else None)
            off += s
        if lean:
            self.A = [None] * self.L

    def residual(self, l, x, b):
        """r = b - A_l x."""
        if self.A[l] is not None:
            return b - self.A[l] @ x
        r = np.empty_like(b)
        for rows, Ar in zip(self.colour_rows[l], self.rowsets[l]):
            if rows.size:
                r[rows] = b[rows] - Ar @ x
        return r

    # -- smoother (R5, R6) --------------------------------------------------------------------
    def sweep(self, l, x, b, forward=True):
        order = range(self.ncol) if forward else range(self.ncol - 1, -1, -1)
        for c in order:
            rows = self.colour_rows[l][c]
            if rows.size == 0:
                continue
            r = b[rows] - self.rowsets[l][c] @ x
            d = self.diag[l][rows]
            x[rows] += r / (d if x.ndim == 1 else d[:, None])      # x may hold several columns
        return x

    def coarse_solve(self, b):
        x = np.zeros_like(b)
        for sl, ch in zip(self.coarse_slices, self.coarse_chol):
            if ch is not None:
                x[sl] = sla.cho_solve(ch, b[sl])
        return x

    # -- V-cycle (O7) ---------------------------------------------------------------------
    def vcycle(self, l, x, b):
        if l == 0:
            return self.coarse_solve(b)
        for _ in range(self.nu_pre):
            x = self.sweep(l, x, b, forward=True)
        r = self.residual(l, x, b)
        e = self.vcycle(l - 1, np.zeros((self.shape[l - 1],) + b.shape[1:]), self.P[l].T @ r)
        x = x + self.P[l] @ e
        for _ in range(self.nu_post):
            x = self.sweep(l, x, b, forward=False)
        return x

    def apply_cycles(self, b, c):
        """N_c(b) (R10): c V-cycles on the finest level from x = 0."""
        x = np.zeros_like(b)
        for _ in range(c):
            x = self.vcycle(self.L - 1, x, b)
        return x
