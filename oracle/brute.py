"""Brute force: the global C^0-conforming Galerkin system of Eq. (1), solved directly -- oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Exact IETI-DP (every local solve exact, tight PCG tolerance) reaches the Galerkin
solution of Eq. (1) in the conforming multipatch spline space
with homogeneous Dirichlet data.  This module builds that
space directly: coinciding active dofs of different patches are identified into
one global dof, the patch stiffness matrices and loads are summed into the
global system (sum_k E_k^T K^(k) E_k), and the system is solved with a sparse
direct solver.  It shares the patch assembly with the oracle but none of the
IETI-DP algebra (no multipliers, constraints, primal basis or Krylov method).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def global_numbering(topo):
    """E_k as index arrays: active dof a of patch k -> global dof id."""
    gid = {}
    n = 0
    maps = []
    for k in range(topo.n_patches):
        pt = topo.ptopo[k]
        mk = np.zeros(len(pt.act_idx), dtype=np.int64)
        for a, flat in enumerate(pt.act_idx):
            key = topo.geo_group_of.get((k, int(flat)), ((k, int(flat)),))
            if key not in gid:
                gid[key] = n
                n += 1
            mk[a] = gid[key]
        maps.append(mk)
    return maps, n


def solve_global(oracle_sys):
    """Returns (u per patch on the full lattice, number of global dofs)."""
    topo = oracle_sys.topo
    maps, n = global_numbering(topo)
    rows, cols, vals = [], [], []
    f = np.zeros(n)
    for k, mk in enumerate(maps):
        K = oracle_sys.K[k].tocoo()
        rows.append(mk[K.row]); cols.append(mk[K.col]); vals.append(K.data)
        np.add.at(f, mk, oracle_sys.f[k])
    A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n)).tocsc()
    ug = spla.spsolve(A, f)
    u = []
    for k, mk in enumerate(maps):
        full = np.zeros(topo.ptopo[k].n_full)
        full[topo.ptopo[k].act_idx] = ug[mk]
        u.append(full)
    return u, n
