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
        """Element multi-indices, direction 1 fastest: array [n_el, dim]."""
        ne = [len(tb[0]) for tb in self.tab]
        grids = np.meshgrid(*[np.arange(n) for n in ne], indexing="ij")
        return np.stack([g.transpose(tuple(range(self.dim - 1, -1, -1))).ravel() for g in grids], axis=-1)

    def element_data(self, es):
        """For a batch of elements es [n_e, dim] (the same formulas element by element):
        local dof ids [n_e, nloc], quad weights [n_e, nqt], N [n_e, nqt, nloc],
        param gradients dN [n_e, nqt, nloc, d], physical points x [n_e, nqt, d] and the
        Jacobian J [n_e, nqt, d, d] (J[.., j, i] = dG_j / dxi_i)."""
        d = self.dim
        es = np.atleast_2d(np.asarray(es, dtype=np.int64))
        ne = es.shape[0]
        wts, vals, ders = [], [], []
        dof = np.zeros((ne, 1), dtype=np.int64)
        for k in range(d):
            first, _, w, v, dv = self.tab[k]
            wts.append(w[es[:, k]])                                     # [n_e, nq]
            vals.append(v[es[:, k]])                                    # [n_e, nq, p+1]
            ders.append(dv[es[:, k]])
            loc = first[es[:, k]][:, None] + np.arange(self.p[k] + 1)[None, :]
            # local dof ids, direction 1 fastest
            dof = (loc[:, :, None] * self.strides[k] + dof[:, None, :]).reshape(ne, -1)
        # quadrature weights, tensor (direction 1 fastest)
        wq = wts[0]
        for w in wts[1:]:
            wq = (w[:, :, None] * wq[:, None, :]).reshape(ne, -1)

        def tens_qa(tabs):
            # tabs[k]: [n_e, nq_k, nloc_k] -> [n_e, nqt, nloct], q and a direction-1 fastest
            out = tabs[0]
            for tb in tabs[1:]:
                out = tb[:, :, None, :, None] * out[:, None, :, None, :]
                out = out.reshape(ne, out.shape[1] * out.shape[2], out.shape[3] * out.shape[4])
            return out
        N = tens_qa(vals)
        dN = np.stack([tens_qa([ders[k] if k == i else vals[k] for k in range(d)]) for i in range(d)],
                      axis=-1)                                          # [n_e, nqt, nloc, d]
        P = self.ctrl[dof]                                              # [n_e, nloc, d]
        x = np.matmul(N, P)                                             # [n_e, nqt, d]
        nqt, nl = N.shape[1], N.shape[2]
        # J[e, q, j, i] = dG_j/dxi_i = sum_a P[e, a, j] dN[e, q, a, i]
        Jt = np.matmul(dN.transpose(0, 1, 3, 2).reshape(ne, nqt * d, nl), P).reshape(ne, nqt, d, d)
        J = Jt.transpose(0, 1, 3, 2)
        return dof, wq, N, dN, x, J

    def chunks(self, max_el=2048):
        es = self.elements()
        for a in range(0, len(es), max_el):
            yield es[a:a + max_el]


def assemble_patch(patch, f=None):
    """K (full-lattice CSR), load f (full lattice) for one patch; raises on det J <= 0.

    Element by element (evaluated in batches of elements, the same formula per element):
        K_loc[a, b] = sum_q w_q |det J_q| (J_q^-T gradhat N_a) . (J_q^-T gradhat N_b)
        f_loc[a]    = sum_q w_q |det J_q| f(x_q) N_a(x_q)
    scattered into the patch matrix (duplicates summed)."""
    pe = PatchElements(patch)
    n = int(np.prod(pe.M))
    K = sp.csr_matrix((n, n))
    load = np.zeros(n)
    for es in pe.chunks():
        dof, wq, N, dN, x, J = pe.element_data(es)
        det = np.linalg.det(J)                                          # [n_e, nqt]
        if np.any(det <= 0.0):
            raise ValueError("non-positive Jacobian determinant at a quadrature point")
        Jinv = np.linalg.inv(J)                                         # [e, q, i, j]
        # physical gradient: grad N = J^{-T} gradhat N  -> g[e, q, a, j] = sum_i Jinv[e, q, i, j] dN[e, q, a, i]
        g = np.matmul(dN, Jinv)
        wdet = wq * det
        # K_loc[e, a, b] = sum_{q, j} wdet[e, q] g[e, q, a, j] g[e, q, b, j]  (one batched matmul)
        ne_, nq_, nl, d_ = g.shape
        G = g.transpose(0, 2, 1, 3).reshape(ne_, nl, nq_ * d_)          # [e, a, (q, j)]
        Kloc = np.matmul(G * np.repeat(wdet, d_, axis=1)[:, None, :], G.transpose(0, 2, 1))
        rows = np.repeat(dof, nl, axis=1).ravel().astype(np.int32)
        cols = np.tile(dof, (1, nl)).ravel().astype(np.int32)
        # scatter this batch of elements (duplicates summed) and add it to the patch matrix
        K = K + sp.coo_matrix((Kloc.ravel(), (rows, cols)), shape=(n, n)).tocsr()
        if f is not None:
            floc = np.einsum("eq,eqa->ea", wdet * f(x), N)
            np.add.at(load, dof.ravel(), floc.ravel())
    K = K.tocsr()
    K.sum_duplicates()
    K.sort_indices()
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
    for es in pe.chunks():
        dof, wq, N, dN, x, J = pe.element_data(es)
        xs.append(x.reshape(-1, pe.dim))
        ws.append((wq * np.linalg.det(J)).ravel())
    return np.concatenate(xs), np.concatenate(ws)


def l2_error(patch, coeffs, u_exact):
    """(sum_q w |det J| (u_h - u)^2)  -- squared L2 error contribution of one patch."""
    pe = PatchElements(patch)
    err2 = 0.0
    for es in pe.chunks():
        dof, wq, N, dN, x, J = pe.element_data(es)
        uh = np.einsum("eqa,ea->eq", N, coeffs[dof])
        err2 += float(np.sum(wq * np.linalg.det(J) * (uh - u_exact(x)) ** 2))
    return err2
