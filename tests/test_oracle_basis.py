"""Pins of the oracle's 1-D LGL basis (Fig. 1; eq. (7))
against closed forms, the paper's printed values, numpy's independent Legendre routines and
the exactness invariants.  No GPU."""
import os

import numpy as np
import pytest
from numpy.polynomial import legendre as npleg

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_lgl_closed_forms(orc):
    # p=1: +-1, w=1,1; p=2: 0,+-1, w=4/3,1/3; p=3: +-1/sqrt5, w=5/6,1/6; p=4: 0,+-sqrt(3/7)
    x, w = orc.lgl(1)
    np.testing.assert_allclose(x, [-1, 1], atol=0)
    np.testing.assert_allclose(w, [1, 1], rtol=1e-15)
    x, w = orc.lgl(2)
    np.testing.assert_array_equal(x, [-1, 0, 1])
    np.testing.assert_allclose(w, [1 / 3, 4 / 3, 1 / 3], rtol=1e-15)
    x, w = orc.lgl(3)
    np.testing.assert_allclose(x, [-1, -1 / np.sqrt(5), 1 / np.sqrt(5), 1], rtol=1e-15, atol=1e-16)
    np.testing.assert_allclose(w, [1 / 6, 5 / 6, 5 / 6, 1 / 6], rtol=1e-14)
    x, w = orc.lgl(4)
    np.testing.assert_allclose(x, [-1, -np.sqrt(3 / 7), 0, np.sqrt(3 / 7), 1], rtol=1e-15, atol=1e-16)
    np.testing.assert_allclose(w, [1 / 10, 49 / 90, 32 / 45, 49 / 90, 1 / 10], rtol=1e-14)


def test_lgl_fig1_printed_values(orc):
    """Fig. 1 prints the p=4 nodes on [0,1] as 0, 0.1727, 0.5, 0.8273, 1.0."""
    vals = [float(l) for l in open(os.path.join(GOLDEN, "fig1_lgl_p4.txt")) if l.strip() and not l.startswith("#")]
    x, _ = orc.lgl(4)
    np.testing.assert_allclose((x + 1) / 2, vals, atol=0.5e-4)


@pytest.mark.parametrize("p", range(1, 17))
def test_lgl_against_numpy_legendre(orc, p):
    x, w = orc.lgl(p)
    ref = np.sort(np.concatenate([[-1.0, 1.0], npleg.Legendre.basis(p).deriv().roots().real]))
    np.testing.assert_allclose(x, ref, rtol=0, atol=2e-14)
    Pp = npleg.legval(ref, [0] * p + [1])
    np.testing.assert_allclose(w, 2.0 / (p * (p + 1) * Pp ** 2), rtol=1e-12)
    # symmetric, strictly increasing, exact endpoints and exact centre (symmetrise)
    assert x[0] == -1.0 and x[-1] == 1.0
    np.testing.assert_array_equal(x, -x[::-1])
    assert np.all(np.diff(x) > 0)
    if p % 2 == 0:
        assert x[p // 2] == 0.0
    assert abs(w.sum() - 2.0) < 1e-14


@pytest.mark.parametrize("p", [1, 2, 3, 4, 8, 16])
def test_lgl_quadrature_exactness(orc, p):
    """Lobatto rule: exact through degree 2p-1, inexact at degree 2p (R1)."""
    x, w = orc.lgl(p)
    for k in range(0, 2 * p):
        exact = 0.0 if k % 2 else 2.0 / (k + 1)
        assert abs(np.dot(w, x ** k) - exact) < 1e-13, k
    k = 2 * p
    assert abs(np.dot(w, x ** k) - 2.0 / (k + 1)) > 1e-12


def _bary_D(x):
    """Independent derivative matrix from barycentric weights (Berrut-Trefethen form)."""
    n = len(x)
    lam = np.array([1.0 / np.prod([x[j] - x[k] for k in range(n) if k != j]) for j in range(n)])
    D = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            if i != j:
                D[i, j] = (lam[j] / lam[i]) / (x[i] - x[j])
        D[i, i] = -D[i].sum()
    return D


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 8, 12, 16])
def test_derivative_matrix(orc, p):
    x, w = orc.lgl(p)
    D = orc.deriv_matrix(p)
    scale = np.abs(D).max()
    np.testing.assert_allclose(D, _bary_D(x), rtol=0, atol=1e-12 * scale)
    np.testing.assert_allclose(D.sum(axis=1), 0, atol=1e-11 * scale)
    assert abs(D[0, 0] + p * (p + 1) / 4) < 1e-11 * scale
    assert abs(D[p, p] - p * (p + 1) / 4) < 1e-11 * scale
    e = np.zeros(p + 1)
    e[0], e[p] = -1, 1
    np.testing.assert_allclose(w @ D, e, atol=1e-11 * scale)
    for k in range(1, p + 1):   # exact differentiation of polynomials of degree <= p
        np.testing.assert_allclose(D @ x ** k, k * x ** (k - 1), atol=1e-10 * scale)


def test_lagrange_cardinal_and_partition(orc):
    for p in (1, 3, 8, 16):
        x, _ = orc.lgl(p)
        for i, xi in enumerate(x):
            l, dl = orc.lagrange_eval(p, xi)
            np.testing.assert_array_equal(l, np.eye(p + 1)[i])   # exactly delta (no rounding)
        for t in (-0.77, 0.1, 0.5):
            l, dl = orc.lagrange_eval(p, t)
            assert abs(l.sum() - 1) < 1e-12
            assert abs(dl.sum()) < 1e-9
    l, _ = orc.lagrange_eval(1, 0.0)
    np.testing.assert_allclose(l, [0.5, 0.5])


def test_interp_matrix(orc):
    np.testing.assert_allclose(orc.interp_matrix(1, 2), [[1, 0], [0.5, 0.5], [0, 1]], atol=1e-16)
    for pc in (1, 2, 4, 8):
        np.testing.assert_allclose(orc.interp_matrix(pc, pc), np.eye(pc + 1), atol=1e-15)
        I = orc.interp_matrix(pc, 2 * pc)
        np.testing.assert_allclose(I.sum(axis=1), 1, atol=1e-13)
        xc, _ = orc.lgl(pc)
        xf, _ = orc.lgl(2 * pc)
        for k in range(pc + 1):      # polynomial exactness
            np.testing.assert_allclose(I @ xc ** k, xf ** k, atol=1e-12)


def test_splitmix_matches_input_module(orc):
    from paper_1402_5938_b200 import inputs
    z = inputs.splitmix64(12345, 0, 5)
    assert [int(v) for v in z] == [orc.splitmix64(12345, i) for i in range(5)]
    # published first output of splitmix64 seeded with 0 (Vigna's reference generator)
    assert orc.splitmix64(0, 0) == 0xE220A8397B1DCDAF
