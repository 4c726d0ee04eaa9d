"""Pins for oracle/topology.py (CPU): counts vs closed forms and the paper's Dofs column; B, B_D, C."""
import json
import os

import numpy as np
import pytest

from oracle import brute
from oracle.topology import Topology, PRIMAL_EDGE, PRIMAL_FACE, PRIMAL_VERTEX
from workloads import identity_patches, jitter_patches, make_workload

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_dofs.json")))


def n_lambda_closed_form(grid, M, primal):
    """App. A.5 (non-redundant multipliers, primal vertices excluded)."""
    if len(grid) == 2:
        nx, ny = grid
        interfaces = (nx - 1) * ny + nx * (ny - 1)
        n = interfaces * (M - 2)
        if not primal & PRIMAL_VERTEX:
            n += 3 * (nx - 1) * (ny - 1)
        return n
    nx, ny, nz = grid
    faces = (nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1)
    edges = (nx - 1) * (ny - 1) * nz + (nx - 1) * ny * (nz - 1) + nx * (ny - 1) * (nz - 1)
    return faces * (M - 2) ** 2 + 3 * edges * (M - 2)


@pytest.mark.parametrize("name,m", [("C1", 4), ("C2", 4), ("C3", 4), ("C4", 4), ("C5", 2)])
def test_counts(name, m):
    wl = make_workload(name, m=m)
    T = Topology(wl.patches, wl.primal)
    M = m + wl.p
    assert T.n_lambda == n_lambda_closed_form(wl.grid, M, wl.primal)
    expected_pi = {"C1": 1, "C2": 9, "C3": 161, "C4": 135, "C5": 1319}[name]
    assert T.n_pi == expected_pi
    nfloat = sum(pt.floating for pt in T.ptopo)
    assert nfloat == {"C1": 0, "C2": 4, "C3": 36, "C4": 8, "C5": 72}[name]
    # interior-patch Gamma size = M^d - (M-2)^d (App. A.5)
    d = wl.dim
    for pt in T.ptopo:
        if pt.floating:
            assert len(pt.gamma) == M ** d - (M - 2) ** d
    # C^(k) 1 = 1 (each functional reproduces constants) and C rows are independent
    for k in range(T.n_patches):
        C = T.C[k].toarray()
        if C.shape[0]:
            assert np.allclose(C @ np.ones(C.shape[1]), 1.0, atol=1e-14)
            assert np.linalg.matrix_rank(C) == C.shape[0]


@pytest.mark.parametrize("row", [r for r in GOLD["rows"] if r["dofs"] < 200000])
def test_paper_dofs_column(row):
    """PAPER.md Tables 1-2 'Dofs' = number of global conforming dofs of the patch grid (decoded)."""
    grid, p, m = tuple(row["grid"]), row["p"], row["m"]
    pats = identity_patches(grid, p, m)
    T = Topology(pats, PRIMAL_VERTEX)
    _, n = brute.global_numbering(T)
    assert n == row["dofs"], row["cite"]


def test_paper_dofs_formula_all_rows():
    for row in GOLD["rows"]:
        n = 1
        for g in row["grid"]:
            n *= g * (row["m"] + row["p"] - 1) - 1
        assert n == row["dofs"], row["cite"]


@pytest.mark.parametrize("name,m,grid", [("C1", 4, None), ("C4", 2, (3, 2, 2)), ("C5", 2, (3, 3, 2)),
                                         ("C3", 4, (4, 3))])
def test_jump_operators(name, m, grid):
    wl = make_workload(name, m=m, grid=grid)
    T = Topology(wl.patches, wl.primal)
    # rows of B: one +1 and one -1, sign + on the lower patch id; canonical order (R12)
    Bd = [T.B[k].toarray() for k in range(T.n_patches)]
    for i, (kp, fp, km, fm) in enumerate(T.mult):
        assert kp < km
        assert Bd[kp][i, T.ptopo[kp].full_to_act[fp]] == 1.0
        assert Bd[km][i, T.ptopo[km].full_to_act[fm]] == -1.0
        assert sum(np.count_nonzero(B[i]) for B in Bd) == 2
    keys = [min(T.geo_group_of[(kp, fp)]) + (kp,) for kp, fp, _, _ in T.mult]   # (k1, flat in k1, chain pos)
    assert keys == sorted(keys)
    # B w = 0 for a globally continuous function (random global coefficients scattered)
    maps, n = brute.global_numbering(T)
    g = np.random.default_rng(1).standard_normal(n)
    jump = sum(T.B[k] @ g[maps[k]] for k in range(T.n_patches))
    assert np.max(np.abs(jump)) == 0.0
    # B_D^T B restricted to a dof group = I - 1 1^T / m  (App. A.4)
    for mem in T.dual_groups[:50]:
        mlt = len(mem)
        rows = sorted({i for i, mu in enumerate(T.mult) if (mu[0], mu[1]) in mem or (mu[2], mu[3]) in mem})
        Bg = np.zeros((len(rows), mlt))
        BDg = np.zeros((len(rows), mlt))
        for c, (k, fl) in enumerate(mem):
            a = T.ptopo[k].full_to_act[fl]
            Bg[:, c] = T.B[k][rows][:, [a]].toarray().ravel()
            BDg[:, c] = T.BD[k][rows][:, [a]].toarray().ravel()
        assert np.allclose(BDg.T @ Bg, np.eye(mlt) - np.ones((mlt, mlt)) / mlt, atol=1e-14)


def test_dirichlet_sides_and_orientation_free_matching():
    # reversing the control-point order of a patch (a flip) must not change matching
    pats = identity_patches((2, 1), 2, 3)
    T = Topology(pats, PRIMAL_VERTEX)
    assert T.n_pi == 0 and T.n_lambda == 3          # strip: 5 shared dofs minus 2 Dirichlet ends
    assert sorted(T.ptopo[0].dirichlet_sides) == [(0, 0), (1, 0), (1, 1)]
