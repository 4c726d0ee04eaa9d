"""Univariate B-splines on open knot vectors (Sec. 2) -- oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* ``basis_funs_ders``: Cox-de Boor triangular evaluation of the p+1 nonzero
  basis functions and their derivatives ("via the Cox-De Boor's algorithm",
  P:96).
* ``basis_recursive``: the textbook recursive definition, used only as a
  brute-force pin in tests.
* ``knot_insertion_matrix``: Boehm single-knot insertion composed over the
  midpoints of all spans (the nested dyadic grids of P:287, reading R7/R8).
* ``gauss_legendre01``: (p+1)-point Gauss rule on [0,1] (numpy ``leggauss``).
* ``mass_1d``: 1D parameter-domain mass matrix M_delta.
"""
from __future__ import annotations

import numpy as np


def validate_open_knots(t, p):
    """Open (clamped), non-decreasing, interior multiplicity <= p, M >= p+1."""
    t = np.asarray(t, dtype=np.float64)
    if p < 1:
        raise ValueError("degree must be >= 1")
    if np.any(np.diff(t) < 0):
        raise ValueError("knot vector decreasing")
    if len(t) < 2 * (p + 1):
        raise ValueError("too few knots")
    if not (np.all(t[:p + 1] == t[0]) and np.all(t[-(p + 1):] == t[-1])):
        raise ValueError("knot vector not open")
    inner = t[p + 1:len(t) - p - 1]
    if inner.size:
        _, counts = np.unique(inner, return_counts=True)
        if counts.max() > p:
            raise ValueError("interior knot multiplicity > p")
        if inner.min() <= t[0] or inner.max() >= t[-1]:
            raise ValueError("interior knot on the boundary")
    return len(t) - p - 1


def find_span(t, p, x):
    """Index mu with t[mu] <= x < t[mu+1], p <= mu <= M-1 (x = t[-1] -> last span)."""
    M = len(t) - p - 1
    if x >= t[M]:
        return M - 1
    mu = int(np.searchsorted(t, x, side="right")) - 1
    return max(p, min(mu, M - 1))


def basis_funs_ders(t, p, x, nder=1):
    """Cox-de Boor: values and derivatives of the p+1 nonzero B-splines at x.

    Returns (span, ders) with ders[k, j] = d^k/dx^k N_{span-p+j, p}(x).
    Triangular table of the recursion
        N_{i,0} = 1 on [t_i, t_{i+1}),
        N_{i,q} = (x-t_i)/(t_{i+q}-t_i) N_{i,q-1} + (t_{i+q+1}-x)/(t_{i+q+1}-t_{i+1}) N_{i+1,q-1}
    and its derivative formula (standard, e.g. Piegl-Tiller A2.3).
    """
    t = np.asarray(t, dtype=np.float64)
    mu = find_span(t, p, x)
    ndu = np.zeros((p + 1, p + 1))
    left = np.zeros(p + 1)
    right = np.zeros(p + 1)
    ndu[0, 0] = 1.0
    for j in range(1, p + 1):
        left[j] = x - t[mu + 1 - j]
        right[j] = t[mu + j] - x
        saved = 0.0
        for r in range(j):
            ndu[j, r] = right[r + 1] + left[j - r]           # lower triangle: knot differences
            temp = ndu[r, j - 1] / ndu[j, r]
            ndu[r, j] = saved + right[r + 1] * temp
            saved = left[j - r] * temp
        ndu[j, j] = saved
    ders = np.zeros((nder + 1, p + 1))
    ders[0, :] = ndu[:, p]
    a = np.zeros((2, p + 1))
    for r in range(p + 1):
        s1, s2 = 0, 1
        a[0, 0] = 1.0
        for k in range(1, nder + 1):
            d = 0.0
            rk, pk = r - k, p - k
            if r >= k:
                a[s2, 0] = a[s1, 0] / ndu[pk + 1, rk]
                d = a[s2, 0] * ndu[rk, pk]
            j1 = 1 if rk >= -1 else -rk
            j2 = k - 1 if r - 1 <= pk else p - r
            for j in range(j1, j2 + 1):
                a[s2, j] = (a[s1, j] - a[s1, j - 1]) / ndu[pk + 1, rk + j]
                d += a[s2, j] * ndu[rk + j, pk]
            if r <= pk:
                a[s2, k] = -a[s1, k - 1] / ndu[pk + 1, r]
                d += a[s2, k] * ndu[r, pk]
            ders[k, r] = d
            s1, s2 = s2, s1
    fac = p
    for k in range(1, nder + 1):
        ders[k, :] *= fac
        fac *= (p - k)
    return mu, ders


def basis_recursive(t, p, i, x):
    """Brute force: the recursive Cox-de Boor definition of N_{i,p}(x) (pin only)."""
    t = np.asarray(t, dtype=np.float64)
    M = len(t) - p - 1
    if p == 0:
        if t[i] <= x < t[i + 1]:
            return 1.0
        # right end of the parameter domain belongs to the last nonempty span
        if x == t[-1] and t[i] < t[i + 1] and t[i + 1] == t[-1]:
            return 1.0
        return 0.0
    val = 0.0
    if t[i + p] > t[i]:
        val += (x - t[i]) / (t[i + p] - t[i]) * basis_recursive(t, p - 1, i, x)
    if t[i + p + 1] > t[i + 1]:
        val += (t[i + p + 1] - x) / (t[i + p + 1] - t[i + 1]) * basis_recursive(t, p - 1, i + 1, x)
    del M
    return val


def eval_all(t, p, x, nder=0):
    """Dense row of all M basis functions (and derivatives) at x: shape (nder+1, M)."""
    M = len(t) - p - 1
    mu, d = basis_funs_ders(t, p, x, nder)
    out = np.zeros((nder + 1, M))
    out[:, mu - p:mu + 1] = d
    return out


def gauss_legendre01(n):
    """n-point Gauss-Legendre rule on [0,1] (library routine numpy leggauss)."""
    xg, wg = np.polynomial.legendre.leggauss(n)
    return 0.5 * (xg + 1.0), 0.5 * wg


def spans(t):
    """Nonempty knot spans (a, b)."""
    u = np.unique(np.asarray(t, dtype=np.float64))
    return list(zip(u[:-1], u[1:]))


def insert_knot_matrix(t, p, u):
    """Boehm insertion of one knot u: returns (t_new, A) with c_new = A c (shape (M+1) x M)."""
    t = np.asarray(t, dtype=np.float64)
    M = len(t) - p - 1
    k = find_span(t, p, u)
    A = np.zeros((M + 1, M))
    for i in range(M + 1):
        if i <= k - p:
            A[i, i] = 1.0
        elif i >= k + 1:
            A[i, i - 1] = 1.0
        else:
            a = (u - t[i]) / (t[i + p] - t[i])
            A[i, i] = a
            A[i, i - 1] = 1.0 - a
    t_new = np.sort(np.concatenate([t, [u]]))
    return t_new, A


def midpoint_refine(t):
    """Insert every nonempty span midpoint once (dyadic refinement)."""
    t = np.asarray(t, dtype=np.float64)
    mids = [(a + b) / 2 for a, b in spans(t)]
    return np.sort(np.concatenate([t, mids]))


def knot_insertion_matrix(t_coarse, p, t_fine):
    """Prolongation P_delta (M_f x M_c) from nested knot vectors by repeated Boehm insertion.

    Coarse spline coefficients c represent the same spline as fine coefficients P c.
    """
    t_coarse = np.asarray(t_coarse, dtype=np.float64)
    t_fine = np.asarray(t_fine, dtype=np.float64)
    # multiset difference fine \ coarse
    extra = []
    tc = list(t_coarse)
    for u in t_fine:
        if tc and any(abs(u - v) == 0.0 for v in tc):
            tc.remove(u)
        else:
            extra.append(u)
    if tc:
        raise ValueError("knot vectors are not nested")
    t = t_coarse
    P = np.eye(len(t_coarse) - p - 1)
    for u in extra:
        t, A = insert_knot_matrix(t, p, u)
        P = A @ P
    if not np.array_equal(t, t_fine):
        raise ValueError("knot insertion did not reproduce the fine knot vector")
    return P


def coarsen_dyadic(t, p):
    """Inverse of ``midpoint_refine`` for a dyadically refined open knot vector (R7)."""
    t = np.asarray(t, dtype=np.float64)
    u = np.unique(t)
    if (len(u) - 1) % 2:
        raise ValueError("odd number of spans: cannot coarsen")
    keep = u[::2]
    tc = np.concatenate([[t[0]] * p, keep, [t[-1]] * p])
    if not np.array_equal(midpoint_refine(tc), t):
        raise ValueError("knot vector is not a dyadic refinement")
    return tc


def mass_1d(t, p):
    """1D mass matrix M[i,j] = int_0^1 N_i N_j (p+1 Gauss points per span, exact)."""
    M = len(t) - p - 1
    xg, wg = gauss_legendre01(p + 1)
    out = np.zeros((M, M))
    for a, b in spans(t):
        for xq, wq in zip(xg, wg):
            x = a + (b - a) * xq
            mu, d = basis_funs_ders(t, p, x, 0)
            n = d[0]
            idx = np.arange(mu - p, mu + 1)
            out[np.ix_(idx, idx)] += (b - a) * wq * np.outer(n, n)
    return out
