"""Pins for oracle/assembly.py (CPU). Eq. (1); parameter mass P:210-211."""
import json
import math
import os

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.interpolate import BSpline

from oracle import assembly
from workloads import (Patch, annulus_patches, identity_patches, jitter_patches, make_workload,
                       open_uniform_knots, f_one)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def scipy_1d(t, p, L=1.0):
    """1D stiffness and mass by an INDEPENDENT route: scipy BSpline basis, 12-point Gauss per span."""
    M = len(t) - p - 1
    xg, wg = np.polynomial.legendre.leggauss(12)
    K = np.zeros((M, M))
    Ms = np.zeros((M, M))
    spl = []
    for i in range(M):
        c = np.zeros(M)
        c[i] = 1.0
        s = BSpline(t, c, p)
        spl.append((s, s.derivative()))
    for a, b in zip(np.unique(t)[:-1], np.unique(t)[1:]):
        x = 0.5 * (a + b) + 0.5 * (b - a) * xg
        w = 0.5 * (b - a) * wg
        V = np.array([s(x) for s, _ in spl])
        D = np.array([d(x) for _, d in spl])
        K += (D * w) @ D.T / L        # d/dX = (1/L) d/dx, dX = L dx
        Ms += (V * w) @ V.T * L
    return K, Ms


def test_spec_1d_stiffness_and_elimination():
    ex = GOLD["stiffness_1d_p1_h_half"]
    K, _ = scipy_1d(np.array(ex["knots"], float), ex["p"])
    assert np.allclose(K, ex["K"], atol=1e-13)
    assert np.allclose(K[1:-1, 1:-1], ex["K_dirichlet_both_ends"])


def test_spec_bilinear_element():
    pa = identity_patches((1, 1), 1, 1)[0]
    K, _ = assembly.assemble_patch(pa)
    assert np.allclose(K.toarray(), GOLD["bilinear_element_stiffness"]["K"], atol=1e-15)


@pytest.mark.parametrize("p,m", [(1, 3), (2, 4), (3, 5), (4, 4)])
def test_identity_map_kronecker_2d(p, m):
    """Affine box [0,a]x[0,b]: K = M2(x)K1 + K2(x)M1 with independent 1D matrices (closed-form structure)."""
    a, b = 0.7, 1.3
    t = open_uniform_knots(p, m)
    pa = identity_patches((1, 1), p, m, extent=(a, b))[0]
    K, _ = assembly.assemble_patch(pa)
    K1, M1 = scipy_1d(t, p, a)
    K2, M2 = scipy_1d(t, p, b)
    ref = np.kron(M2, K1) + np.kron(K2, M1)
    assert np.max(np.abs(K.toarray() - ref)) <= 1e-12 * np.abs(ref).max()


def test_identity_map_kronecker_3d():
    p, m = 2, 3
    t = open_uniform_knots(p, m)
    pa = identity_patches((1, 1, 1), p, m)[0]
    K, _ = assembly.assemble_patch(pa)
    K1, M1 = scipy_1d(t, p)
    ref = (np.kron(M1, np.kron(M1, K1)) + np.kron(M1, np.kron(K1, M1)) + np.kron(K1, np.kron(M1, M1)))
    assert np.max(np.abs(K.toarray() - ref)) <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("maker", ["jitter2", "annulus", "jitter3"])
def test_symmetry_kernel_and_load(maker):
    if maker == "jitter2":
        pats, area = jitter_patches((3, 3), 3, 4, seed=2), 1.0
    elif maker == "annulus":
        pats, area = annulus_patches((2, 2), 4, 4), math.pi * (4 - 1) / 4
    else:
        pats, area = jitter_patches((2, 2, 2), 2, 3, seed=5), 1.0
    total = 0.0
    for pa in pats:
        K, f = assembly.assemble_patch(pa, f_one)
        Kd = K.toarray()
        assert np.max(np.abs(Kd - Kd.T)) <= 1e-12 * np.abs(Kd).max()
        assert np.max(np.abs(Kd @ np.ones(K.shape[0]))) <= 1e-10 * np.abs(Kd).max()   # K 1 = 0
        total += f.sum()
    # load with f = 1 sums to the area (exact for multilinear maps); the polar map is sampled at
    # Greville points (R15: O(h^2) in theta), so there the error must shrink (observed ~3x) per refinement
    if maker != "annulus":
        assert abs(total - area) <= 1e-12 * area
    else:
        fine = sum(assembly.assemble_patch(pa, f_one)[1].sum() for pa in annulus_patches((2, 2), 4, 8))
        e0, e1 = abs(total - area), abs(fine - area)
        assert e0 <= 0.02 * area and e1 <= e0 / 2.5


def test_parameter_mass():
    pa = identity_patches((1, 1), 3, 4)[0]
    Mh = assembly.parameter_mass(pa)
    assert abs(Mh.sum() - 1.0) <= 1e-14
    # equals a full 2D quadrature of N_a N_b on the parameter domain (identity map with extent 1)
    t = open_uniform_knots(3, 4)
    _, M1 = scipy_1d(t, 3)
    assert np.allclose(Mh.toarray(), np.kron(M1, M1), atol=1e-14)


def test_negative_jacobian_rejected():
    pa = identity_patches((1, 1), 2, 2)[0]
    bad = Patch(pa.degree, pa.knots, pa.ctrl * np.array([-1.0, 1.0]))
    with pytest.raises(ValueError):
        assembly.assemble_patch(bad)
