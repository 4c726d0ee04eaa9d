"""Pins for oracle/mg.py (CPU): GS hand example, colour GS vs sequential GS, V-cycle symmetry,
contraction, bounded MG-preconditioned condition number (north star), N_c -> exact."""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import assembly, mg
from oracle.ieti import IetiOracle
from oracle.topology import unravel
from workloads import identity_patches, jitter_patches, make_workload

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def dirichlet_patch_hierarchy(p, m, dim=2, L=None, jitter=False):
    grid = (1,) * dim
    pa = (jitter_patches((2,) * dim, p, m, seed=3)[0] if jitter else identity_patches(grid, p, m)[0])
    K, _ = assembly.assemble_patch(pa)
    M = pa.n_basis
    lv = mg.PatchLevels(pa.knots, p, L or mg.num_levels(m), [True] * dim, [True] * dim)
    KII = K[lv.mask[-1]][:, lv.mask[-1]].tocsr()
    return mg.Hierarchy([KII], [lv]), KII


class _TinyH(mg.Hierarchy):
    def __init__(self, A, colours):
        self.A = [sp.csr_matrix(A)]
        self.diag = [self.A[0].diagonal()]
        self.ncol = max(colours) + 1
        self.colour_rows = [[np.nonzero(np.array(colours) == c)[0] for c in range(self.ncol)]]
        self.rowsets = [[self.A[0][r] for r in self.colour_rows[0]]]


def test_spec_gauss_seidel_example():
    ex = GOLD["gauss_seidel"]
    H = _TinyH(np.array(ex["A"], float), [0, 1])
    x = H.sweep(0, np.zeros(2), np.array(ex["b"], float), forward=True)
    assert np.allclose(x, ex["x_after_forward_sweep"], atol=1e-16)


@pytest.mark.parametrize("p,dim", [(2, 2), (3, 2), (2, 3)])
def test_colour_sweep_equals_sequential_gs_in_colour_order(p, dim):
    """R6: rows of one colour are decoupled, so the simultaneous colour phase equals a
    sequential point GS over the rows taken in colour-major order (brute force loop)."""
    H, A = dirichlet_patch_hierarchy(p, 8 if dim == 2 else 4, dim)
    l = H.L - 1
    rng = np.random.default_rng(0)
    b = rng.standard_normal(A.shape[0])
    x0 = rng.standard_normal(A.shape[0])
    x = H.sweep(l, x0.copy(), b, forward=True)
    Ad = A.toarray()
    y = x0.copy()
    for c in range(H.ncol):
        for i in H.colour_rows[l][c]:
            y[i] += (b[i] - Ad[i] @ y) / Ad[i, i]
    assert np.max(np.abs(x - y)) <= 1e-13 * np.abs(y).max()
    # within-colour rows are structurally independent: |i_d - j_d| >= p+1 for some d => A_ij = 0
    for c in range(H.ncol):
        rows = H.colour_rows[l][c]
        sub = Ad[np.ix_(rows, rows)]
        assert np.count_nonzero(sub - np.diag(np.diag(sub))) == 0


@pytest.mark.parametrize("p,dim,jit", [(2, 2, False), (3, 2, True), (2, 3, False)])
def test_vcycle_symmetric_and_contracting(p, dim, jit):
    H, A = dirichlet_patch_hierarchy(p, 16 if dim == 2 else 8, dim, jitter=jit)
    n = A.shape[0]
    rng = np.random.default_rng(1)
    x, y = rng.standard_normal(n), rng.standard_normal(n)
    Vx = H.apply_cycles(x, 1)
    Vy = H.apply_cycles(y, 1)
    assert abs(y @ Vx - x @ Vy) <= 1e-12 * abs(y @ Vx)
    # contraction of the stationary iteration x <- V(x,b): rho(I - N_1 A) < 0.5 for 2D p=2
    E = np.column_stack([e - H.apply_cycles(A @ e, 1) for e in np.eye(n)])
    rho = max(abs(np.linalg.eigvals(E)))
    if p == 2 and dim == 2:
        assert rho < 0.5
    assert rho < 1.0
    # N_c -> exact as c grows (c chosen from the measured contraction rate)
    b = rng.standard_normal(n)
    xe = spla.spsolve(A.tocsc(), b)
    c = int(np.ceil(np.log(1e-12) / np.log(rho)))
    assert np.linalg.norm(H.apply_cycles(b, c) - xe) <= 1e-9 * np.linalg.norm(xe)


def test_bounded_condition_number_under_refinement():
    """North star: MG-preconditioned K_II has a bounded condition number under refinement."""
    conds = []
    for m in (8, 16, 32):
        H, A = dirichlet_patch_hierarchy(2, m, 2)
        n = A.shape[0]
        NA = np.column_stack([H.apply_cycles(A @ e, 1) for e in np.eye(n)])
        ev = np.linalg.eigvals(NA).real
        conds.append(ev.max() / ev.min())
    assert max(conds) < 2.0
    assert conds[-1] <= 1.25 * conds[0]


def test_galerkin_and_trimmed_prolongation():
    """Trimmed P equals deleting first/last rows+cols (exact for open knots): the coarse space
    with zero boundary values is mapped into the fine space with zero boundary values."""
    pa = identity_patches((1, 1), 3, 8)[0]
    lv = mg.PatchLevels(pa.knots, 3, 3, [True, False], [True, True])
    for l in range(1, 3):
        P = lv.P[l - 1].toarray()
        assert P.shape == (lv.mask[l].sum(), lv.mask[l - 1].sum())
    H, A = dirichlet_patch_hierarchy(2, 16, 2)
    for l in range(1, H.L):
        ref = (H.P[l].T @ H.A[l] @ H.P[l]).toarray()
        assert np.allclose(H.A[l - 1].toarray(), ref, atol=1e-14)
        assert np.allclose(ref, ref.T, atol=1e-13)


def test_num_levels_rule():
    assert [mg.num_levels(m) for m in (4, 16, 32, 64, 128)] == [2, 3, 4, 5, 6]
