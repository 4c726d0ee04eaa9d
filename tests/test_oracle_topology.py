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


def test_edge_only_3d_multiplicity_8_groups():
    """Paper's 3D constraint set (edge averages only): the interior vertex of a 2x2x2
    patch grid is a dual dof shared by 8 patches.  Its chain of 7 multipliers (R12) and the scaled
    B_D = (B_g B_g^T)^-1 B_g satisfy B_D^T B = I - 1 1^T / m exactly, and the
    multiplicity-4 edge dofs likewise (the chain with +-1/m would fail both, App. A.4)."""
    wl = make_workload("E2", m=2, grid=(2, 2, 2))
    T = Topology(wl.patches, wl.primal)
    mults = sorted({len(g) for g in T.dual_groups})
    assert mults == [2, 4, 8], mults
    n8 = 0
    for mem in T.dual_groups:
        mlt = len(mem)
        rows = sorted({i for i, mu in enumerate(T.mult) if (mu[0], mu[1]) in mem or (mu[2], mu[3]) in mem})
        assert len(rows) == mlt - 1                       # non-redundant chain
        Bg = np.zeros((len(rows), mlt))
        BDg = np.zeros((len(rows), mlt))
        for c, (k, fl) in enumerate(mem):
            a = T.ptopo[k].full_to_act[fl]
            Bg[:, c] = T.B[k][rows][:, [a]].toarray().ravel()
            BDg[:, c] = T.BD[k][rows][:, [a]].toarray().ravel()
        assert np.allclose(BDg.T @ Bg, np.eye(mlt) - np.ones((mlt, mlt)) / mlt, atol=1e-14)
        if mlt == 8:
            n8 += 1
            # the naive chain scaling +-1/m is NOT a left inverse here (App. A.4: error 0.75 at m = 8)
            naive = Bg / mlt
            assert np.abs(naive.T @ Bg - (np.eye(mlt) - np.ones((mlt, mlt)) / mlt)).max() > 0.5
    assert n8 == 1


@pytest.mark.parametrize("name,kw", [("C3", dict(m=8, grid=(3, 2))), ("C4", dict(m=4, grid=(2, 2, 2))),
                                     ("C5", dict(m=4, grid=(2, 2, 2)))])
def test_average_weights_are_normalised_integrals(name, kw):
    """R13: the weights of an average row are w_a ~ integral of the parameter-domain
    tensor B-spline over the entity's free directions, normalised to 1 -- computed here
    independently by SciPy's BSpline antiderivative (not the closed form the oracle uses).
    Uniform weights would fail: open knots make the end functions' integrals smaller."""
    from scipy.interpolate import BSpline
    from oracle.topology import unravel
    wl = make_workload(name, **kw)
    T = Topology(wl.patches, wl.primal)
    checked = 0
    for gid, e in enumerate(T.primal):
        if e.kind == "vertex":
            continue
        for k, flats in e.members.items():
            pa = wl.patches[k]
            M = pa.n_basis
            w_ref = np.ones(len(flats))
            for j, fl in enumerate(flats):
                idx = unravel(int(fl), M)
                for d in range(wl.dim):
                    if 0 < idx[d] < M[d] - 1:            # a free direction of the open entity
                        t = np.asarray(pa.knots[d])
                        c = np.zeros(M[d])
                        c[idx[d]] = 1.0
                        w_ref[j] *= BSpline(t, c, pa.degree[d]).integrate(t[0], t[-1])
            w_ref /= w_ref.sum()
            row = T.C[k][list(T.R[k]).index(gid)].toarray().ravel()
            got = row[T.ptopo[k].full_to_act[flats]]
            assert np.allclose(got, w_ref, rtol=1e-12, atol=0), (name, e.kind, k)
            assert np.ptp(got) > 1e-3                      # not uniform
            checked += 1
    assert checked > 0
