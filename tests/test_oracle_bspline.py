"""Pins for oracle/bspline.py (CPU). PAPER.md:93-96 (Cox-de Boor), P:287 (nested dyadic grids)."""
import json
import os
from math import comb

import numpy as np
import pytest
from scipy.interpolate import BSpline

from oracle import bspline
from workloads import open_uniform_knots

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def nonuniform(p, m, seed):
    rng = np.random.default_rng(seed)
    inner = np.sort(rng.uniform(0.05, 0.95, m - 1))
    return np.concatenate([[0.0] * (p + 1), inner, [1.0] * (p + 1)])


@pytest.mark.parametrize("p", [1, 2, 3, 4, 7])
def test_partition_of_unity_and_derivative_sum(p):
    for t in (open_uniform_knots(p, 8), nonuniform(p, 6, p)):
        for x in np.linspace(0, 1, 101):
            mu, d = bspline.basis_funs_ders(t, p, x, 1)
            assert abs(d[0].sum() - 1.0) <= 1e-13
            assert abs(d[1].sum()) <= 1e-10
            assert np.all(d[0] >= -1e-15)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_cox_de_boor_vs_recursive_definition(p):
    t = nonuniform(p, 5, 10 + p)
    M = len(t) - p - 1
    for x in np.linspace(0, 1, 37):
        row = bspline.eval_all(t, p, x, 0)[0]
        brute = np.array([bspline.basis_recursive(t, p, i, x) for i in range(M)])
        assert np.max(np.abs(row - brute)) <= 1e-14


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_cox_de_boor_vs_scipy_bspline(p):
    """Library routine scipy.interpolate.BSpline as an independent evaluator (values + 1st derivative)."""
    t = nonuniform(p, 7, 20 + p)
    M = len(t) - p - 1
    xs = np.linspace(0, 1, 53)[:-1]
    for i in range(M):
        c = np.zeros(M)
        c[i] = 1.0
        spl = BSpline(t, c, p)
        dspl = spl.derivative()
        for x in xs:
            row = bspline.eval_all(t, p, x, 1)
            assert abs(row[0, i] - spl(x)) <= 1e-13
            assert abs(row[1, i] - dspl(x)) <= 1e-10 * max(1.0, abs(dspl(x)))


def test_spec_examples_cox_de_boor():
    for ex in GOLD["cox_de_boor"]:
        mu, d = bspline.basis_funs_ders(np.array(ex["knots"], float), ex["p"], ex["x"], 0)
        assert mu - ex["p"] == ex["first_active"]
        assert np.allclose(d[0], ex["values"], atol=1e-15)


def test_spec_prolongation_p1():
    ex = GOLD["prolongation_p1"]
    P = bspline.knot_insertion_matrix(np.array(ex["coarse"], float), ex["p"], np.array(ex["fine"], float))
    assert np.array_equal(P, np.array(ex["P"], float))


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_prolongation_constant_and_subdivision_mask(p):
    """P 1 = 1; interior columns equal the uniform subdivision mask C(p+1, j)/2^p (closed form)."""
    tc = open_uniform_knots(p, 8)
    tf = bspline.midpoint_refine(tc)
    assert np.array_equal(tf, open_uniform_knots(p, 16))
    P = bspline.knot_insertion_matrix(tc, p, tf)
    assert np.allclose(P @ np.ones(P.shape[1]), 1.0, atol=1e-14)
    mask = np.array([comb(p + 1, j) for j in range(p + 2)]) / 2.0 ** p
    # a coarse function far from the boundary: column i with support inside
    for i in range(p + 1, P.shape[1] - p - 1):
        col = P[:, i]
        nz = np.nonzero(np.abs(col) > 1e-15)[0]
        assert len(nz) == p + 2
        assert np.allclose(col[nz], mask, atol=1e-14)


@pytest.mark.parametrize("p", [2, 3])
def test_prolongation_sampled_spline_equality(p):
    tc = nonuniform(p, 5, 3)
    tf = bspline.midpoint_refine(tc)
    P = bspline.knot_insertion_matrix(tc, p, tf)
    c = np.random.default_rng(0).standard_normal(P.shape[1])
    for x in np.linspace(0, 1, 50):
        vc = bspline.eval_all(tc, p, x, 0)[0] @ c
        vf = bspline.eval_all(tf, p, x, 0)[0] @ (P @ c)
        assert abs(vc - vf) <= 1e-12


def test_coarsen_inverts_refine():
    for p in (1, 2, 3):
        t = open_uniform_knots(p, 16)
        assert np.array_equal(bspline.coarsen_dyadic(t, p), open_uniform_knots(p, 8))


def test_mass_1d_and_integrals():
    ex = GOLD["mass_1d_p1_single_span"]
    M = bspline.mass_1d(np.array(ex["knots"], float), ex["p"])
    assert np.allclose(M, ex["M"], atol=1e-15)
    # row sums are int N_a = (t_{a+p+1} - t_a)/(p+1) (the R13 weight), normalised -> S:475
    ex = GOLD["edge_average_p1"]
    t, p = np.array(ex["knots"], float), ex["p"]
    Mm = bspline.mass_1d(t, p)
    w = np.array([(t[a + p + 1] - t[a]) / (p + 1) for a in range(len(t) - p - 1)])
    assert np.allclose(Mm.sum(axis=1), w, atol=1e-15)
    assert np.allclose(w / w.sum(), ex["weights"], atol=1e-15)
    # 1^T M 1 = 1 (measure of the parameter domain)
    for p in (2, 3, 4):
        assert abs(bspline.mass_1d(open_uniform_knots(p, 6), p).sum() - 1.0) <= 1e-14


def test_validation_errors():
    with pytest.raises(ValueError):
        bspline.validate_open_knots([0, 0.5, 1, 1], 1)          # not open
    with pytest.raises(ValueError):
        bspline.validate_open_knots([0, 0, 0.6, 0.4, 1, 1], 1)  # decreasing
    with pytest.raises(ValueError):
        bspline.validate_open_knots([0, 0, 0, 0.5, 0.5, 0.5, 1, 1, 1], 2)  # multiplicity > p
