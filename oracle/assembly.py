"""Per-patch Galerkin assembly (Eq. (1)) -- oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

For one patch with open knot vectors t_delta, degrees p_delta and control points
P_i (geometry map G(xi) = sum_i P_i N_i(xi)):

    K_ab = sum_elements sum_q w_q (J^-T grad N_a) . (J^-T grad N_b) |det J|
    f_a  = sum_elements sum_q w_q f(G(xi_q)) N_a |det J|
    Mhat = M_d (x) ... (x) M_1     (parameter-domain mass)

with (p+1)-point Gauss-Legendre per direction per element (north star).  All
matrices are on the FULL lattice (lexicographic, direction 1 fastest); Dirichlet
elimination happens in ``topology``/``ieti`` by row/column selection.
"""
from __future__ import annotations

import itertools

import numpy as np
import scipy.sparse as sp

from . import bspline


def _direction_tables(t, p):
    """Per element e and Gauss point q: span start, point, weight, values, derivatives."""
    el = bspline.spans(t)
    xg, wg = bspline.gauss_legendre01(p + 1)
    ne, nq = len(el), p + 1
    first = np.zeros(ne, dtype=np.int64)
    pts = np.zeros((ne, nq))
    wts = np.zeros((ne, nq))
    val = np.zeros((ne, nq, p + 1))
    der = np.zeros((ne, nq, p + 1))
    for e, (a, b) in enumerate(el):
        for q in range(nq):
            x = a + (b - a) * xg[q]
            mu, d = bspline.basis_funs_ders(t, p, x, 1)
            first[e] = mu - p
            pts[e, q] = x
            wts[e, q] = (b - a) * wg[q]
            val[e, q] = d[0]
            der[e, q] = d[1]
    return first, pts, wts, val, der


def _tensor(arrs):
    """Outer product over directions with direction 1 fastest in the flattened index."""
    out = arrs[0]
    for a in arrs[1:]:
        # out[..., i_prev], a[..., i_new] -> [..., i_new, i_prev] (new direction slower)
        out = (a[..., :, None] * out[..., None, :]).reshape(a.shape[:-1] + (-1,))
    return out


class PatchElements:
    """Basis tables of one patch, evaluated at every Gauss point of every element."""

    def __init__(self, patch):
        self.dim = patch.dim
        self.p = tuple(patch.degree)
        self.knots = tuple(np.asarray(t, dtype=np.float64) for t in patch.knots)
        self.M = tuple(bspline.validate_open_knots(t, p) for t, p in zip(self.knots, self.p))
        self.ctrl = np.asarray(patch.ctrl, dtype=np.float64)
        if self.ctrl.shape != (int(np.prod(self.M)), self.dim):
            raise ValueError("control point array has the wrong shape")
        self.tab = [_direction_tables(t, p) for t, p in zip(self.knots, self.p)]
        self.strides = [int(np.prod(self.M[:d])) for d in range(self.dim)]

    def elements(self):
        ne = [len(tb[0]) for tb in self.tab]
        # element multi-index, direction 1 fastest
        for e_rev in itertools.product(*[range(n) for n in reversed(ne)]):
            yield tuple(reversed(e_rev))

    def element_data(self, e):
        """For element e: local dof ids, quad weights, N, grad-hat N (param), physical x, J."""
        d = self.dim
        firsts, wts, vals, ders, locs = [], [], [], [], []
        for k in range(d):
            first, _, w, v, dv = self.tab[k]
            firsts.append(first[e[k]])
            wts.append(w[e[k]])                    # [nq]
            vals.append(v[e[k]])                   # [nq, p+1]
            ders.append(dv[e[k]])
            locs.append(np.arange(first[e[k]], first[e[k]] + self.p[k] + 1))
        # local dof ids (direction 1 fastest)
        dof = np.zeros(1, dtype=np.int64)
        for k in range(d):
            dof = (locs[k][:, None] * self.strides[k] + dof[None, :]).ravel()
        # quadrature weights, tensor
        wq = _tensor([w[None, :] for w in wts])[0]                     # [nqt]
        # values N[qt, a] = prod_k vals_k[q_k, a_k]
        def tens_qa(tabs):
            # tabs[k]: [nq_k, nloc_k]; returns [nqt, nloct] with q and a direction-1 fastest
            out = tabs[0]
            for tb in tabs[1:]:
                out = (tb[:, None, :, None] * out[None, :, None, :])
                out = out.reshape(tb.shape[0] * out.shape[1], tb.shape[1] * out.shape[3])
            return out
        N = tens_qa(vals)
        dN = []
        for i in range(d):
            dN.append(tens_qa([ders[k] if k == i else vals[k] for k in range(d)]))
        dN = np.stack(dN, axis=-1)                                      # [nqt, nloc, d] (param grad)
        P = self.ctrl[dof]                                              # [nloc, d]
        x = N @ P                                                       # [nqt, d]
        J = np.einsum("qai,aj->qji", dN, P)                             # J[q, j, i] = dG_j/dxi_i
        return dof, wq, N, dN, x, J


def assemble_patch(patch, f=None):
    """K (full-lattice CSR), load f (full lattice) for one patch; raises on det J <= 0."""
    pe = PatchElements(patch)
    n = int(np.prod(pe.M))
    rows, cols, vals = [], [], []
    load = np.zeros(n)
    for e in pe.elements():
        dof, wq, N, dN, x, J = pe.element_data(e)
        det = np.linalg.det(J)
        if np.any(det <= 0.0):
            raise ValueError("non-positive Jacobian determinant at a quadrature point")
        Jinv = np.linalg.inv(J)                                         # [q, i, j]
        # physical gradient: grad N = J^{-T} gradhat N  -> g[q, a, j] = sum_i Jinv[q, i, j] dN[q, a, i]
        g = np.einsum("qij,qai->qaj", Jinv, dN)
        wdet = wq * det
        Kloc = np.einsum("q,qaj,qbj->ab", wdet, g, g)
        rows.append(np.repeat(dof, len(dof)))
        cols.append(np.tile(dof, len(dof)))
        vals.append(Kloc.ravel())
        if f is not None:
            load[dof] += (wdet * f(x)) @ N
    K = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, n)).tocsr()
    K.sum_duplicates()
    return K, load


def parameter_mass(patch):
    """Mhat = kron over directions of 1D masses (direction 1 fastest => last factor)."""
    mats = [bspline.mass_1d(np.asarray(t, dtype=np.float64), p) for t, p in zip(patch.knots, patch.degree)]
    Mh = sp.csr_matrix(mats[0])
    for Md in mats[1:]:
        Mh = sp.kron(sp.csr_matrix(Md), Mh, format="csr")
    return Mh


def quadrature_points(patch):
    """Physical Gauss points and weights*|det J| of a patch (for L2 errors, f sums)."""
    pe = PatchElements(patch)
    xs, ws = [], []
    for e in pe.elements():
        dof, wq, N, dN, x, J = pe.element_data(e)
        xs.append(x)
        ws.append(wq * np.linalg.det(J))
    return np.concatenate(xs), np.concatenate(ws)


def l2_error(patch, coeffs, u_exact):
    """(sum_q w |det J| (u_h - u)^2)  -- squared L2 error contribution of one patch."""
    pe = PatchElements(patch)
    err2 = 0.0
    for e in pe.elements():
        dof, wq, N, dN, x, J = pe.element_data(e)
        uh = N @ coeffs[dof]
        err2 += float(np.sum(wq * np.linalg.det(J) * (uh - u_exact(x)) ** 2))
    return err2
