"""Pins of the 2-D oracle (NEXT-2; the paper's 2-D problems P:875-890): quadrilateral
elements of order p, isoparametric geometry, collocated LGL or Gauss quadrature.  Pinned against
closed forms and independent numpy constructions, not against the oracle's own formulas:

* affine unit square, mu = 1, LGL: A = K1 (x) W1 + W1 (x) K1 (1-D SEM matrices, numpy);
* constant mu = c0: c0 times the same Kronecker sum;
* Gauss quadrature, p = 1: the exact bilinear stiffness, 9-point stencil (8, -1 x 8) / 3;
* warped mesh, 2d-var / 2d-var' coefficients: brute-force numpy element matrix; symmetry, A 1 = 0,
  SPD after the Dirichlet projection;
* transfers: Kronecker products of the 1-D global prolongations (p and h), adjointness;
* MMS u* = sin(pi x) sin(pi y): algebraic h-convergence (order >= p + 0.5) and spectral p-convergence;
* two-level V-cycle = closed matrix form; Chebyshev error propagator closed form;
* tab:box (2d-const, 32x32): the paper's iteration counts to +-1 where the paper's
  columns and this discretisation agree (Gauss quadrature; see DESIGN.md section 9e for the rest).
No GPU."""
import os

import numpy as np
import pytest

from test_oracle_mg import np_lagrange_matrix
from test_oracle_next1 import np_global_h1
from test_oracle_operator import assembled_1d, np_D, np_lgl

WARPED2 = dict(warp=1, amp=0.1, coeff=1, c0=1.0, c1=3.0)
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "tab_box.txt")


@pytest.mark.parametrize("ne,p", [(1, 1), (3, 2), (2, 4), (2, 7)])
def test_affine_kronecker_sum(orc, ne, p):
    L = orc.Level2(ne, ne, p)
    A = L.assemble_dense(1)
    K1, W1 = assembled_1d(ne, p, 1.0 / ne)
    ref = np.kron(W1, K1) + np.kron(K1, W1)   # index g = I + Mx J: x fastest
    np.testing.assert_allclose(A, ref, rtol=0, atol=1e-12 * np.abs(ref).max())


def test_constant_coefficient_scaling(orc):
    """mu = c0: A = c0 (K1 (x) W1 + W1 (x) K1) on the affine square."""
    ne, p = 2, 3
    L = orc.Level2(ne, ne, p, coeff=0, c0=2.5)
    A = L.assemble_dense(1)
    K1, W1 = assembled_1d(ne, p, 1.0 / ne)
    np.testing.assert_allclose(A, 2.5 * (np.kron(W1, K1) + np.kron(K1, W1)), rtol=0, atol=1e-12 * np.abs(A).max())


def test_gauss_q1_stencil(orc):
    orc.set_quadrature(1)
    try:
        L = orc.Level2(2, 2, 1)
        A = L.assemble_dense(1)
    finally:
        orc.set_quadrature(0)
    row = A[4].reshape(3, 3)   # centre node of the 3x3 lattice
    np.testing.assert_allclose(row, np.array([[-1, -1, -1], [-1, 8, -1], [-1, -1, -1]]) / 3.0, atol=1e-14)
    assert abs(A.sum()) < 1e-13


def np_element_matrix_2d(x, w, X, Y, mu):
    """Brute force: isoparametric map from the nodal coordinates, collocated LGL quadrature."""
    n = len(x)
    D = np_D(x)
    K = np.zeros((n * n, n * n))
    for j in range(n):
        for i in range(n):
            # gradients of every basis function (a, b) at node (i, j): (D[i,a] delta_jb, delta_ia D[j,b])
            dxi = np.zeros((n, n))
            deta = np.zeros((n, n))
            dxi[:, j] = D[i, :]   # [a, b]
            deta[i, :] = D[j, :]
            J = np.array([[np.sum(dxi * X), np.sum(deta * X)], [np.sum(dxi * Y), np.sum(deta * Y)]])
            Ji = np.linalg.inv(J)
            gx = Ji[0, 0] * dxi + Ji[1, 0] * deta
            gy = Ji[0, 1] * dxi + Ji[1, 1] * deta
            gx, gy = gx.T.ravel(), gy.T.ravel()   # l = a + n b
            K += w[i] * w[j] * np.linalg.det(J) * mu(X[i, j], Y[i, j]) * (np.outer(gx, gx) + np.outer(gy, gy))
    return K


@pytest.mark.parametrize("coeff,c0,c1", [(1, 1.0, 3.0), (3, 1.0, 1e6), (4, 1.0, 1e6)])
def test_element_matrix_brute_force_warped(orc, coeff, c0, c1):
    p, ne = 3, 2
    L = orc.Level2(ne, ne, p, warp=1, amp=0.1, coeff=coeff, c0=c0, c1=c1)
    x, w = np_lgl(p)
    mus = {1: lambda X, Y: np.exp(c1 * np.sin(2 * np.pi * X) * np.sin(2 * np.pi * Y)),
           3: lambda X, Y: c0 + c1 * (np.cos(2 * np.pi * X) ** 2 + np.cos(2 * np.pi * Y) ** 2),
           4: lambda X, Y: c0 + c1 * (np.cos(10 * np.pi * X) ** 2 + np.cos(10 * np.pi * Y) ** 2)}
    for e in (0, 3):
        ex, ey = e % ne, e // ne
        Xr = (ex + (x[:, None] + 1) / 2) / ne + 0 * x[None, :]
        Yr = (ey + (x[None, :] + 1) / 2) / ne + 0 * x[:, None]
        s = 0.1 * np.sin(np.pi * Xr) * np.sin(np.pi * Yr)
        K = np_element_matrix_2d(x, w, Xr + s, Yr + s, mus[coeff])
        Ko = L.element_matrix(e)
        np.testing.assert_allclose(Ko, K, rtol=0, atol=1e-10 * np.abs(K).max())


@pytest.mark.parametrize("coeff,c1", [(1, 3.0), (4, 1e6)])
def test_operator_invariants_warped(orc, coeff, c1):
    L = orc.Level2(3, 2, 4, warp=1, amp=0.1, coeff=coeff, c0=1.0, c1=c1)
    A1 = L.assemble_dense(1)
    assert np.abs(A1 - A1.T).max() <= 1e-12 * np.abs(A1).max()
    assert np.abs(A1 @ np.ones(L.N)).max() <= 1e-10 * np.abs(A1).max()
    A0 = L.assemble_dense(0)
    assert np.linalg.eigvalsh(A0).min() > 0
    u = np.random.default_rng(1).uniform(-1, 1, L.N)
    np.testing.assert_allclose(L.apply(u, 0), A0 @ u, rtol=0, atol=1e-12 * np.abs(A0 @ u).max())
    np.testing.assert_allclose(L.diag(0), np.diag(A0), rtol=0, atol=1e-13 * np.abs(np.diag(A0)).max())


def test_transfers_kronecker(orc):
    rng = np.random.default_rng(3)
    # p pair 2 -> 4 on 2x3 elements
    C, F = orc.Level2(2, 3, 2, **WARPED2), orc.Level2(2, 3, 4, **WARPED2)
    xc, _ = np_lgl(2)
    xf, _ = np_lgl(4)
    I = np_lagrange_matrix(xc, xf)

    def glob(ne):
        P = np.zeros((ne * 4 + 1, ne * 2 + 1))
        for e in range(ne):
            P[e * 4:e * 4 + 5, e * 2:e * 2 + 3] = I
        return P
    P = np.kron(glob(3), glob(2))
    P0 = np.diag(1.0 - F.mask()) @ P @ np.diag(1.0 - C.mask())
    uc, rf = rng.uniform(-1, 1, C.N), rng.uniform(-1, 1, F.N)
    np.testing.assert_allclose(orc.prolong2(C, F, uc), P0 @ uc, atol=1e-14)
    np.testing.assert_allclose(orc.restrict2(C, F, rf), P0.T @ rf, atol=1e-13)
    # h pair at p = 3: 2x1 -> 4x2
    C, F = orc.Level2(2, 1, 3, **WARPED2), orc.Level2(4, 2, 3, **WARPED2)
    P = np.kron(np_global_h1(1, 3), np_global_h1(2, 3))
    P0 = np.diag(1.0 - F.mask()) @ P @ np.diag(1.0 - C.mask())
    uc, rf = rng.uniform(-1, 1, C.N), rng.uniform(-1, 1, F.N)
    np.testing.assert_allclose(orc.prolong2(C, F, uc), P0 @ uc, atol=1e-14)
    np.testing.assert_allclose(orc.restrict2(C, F, rf), P0.T @ rf, atol=1e-13)


def test_mms_convergence_2d(orc):
    def err(ne, p):
        H = orc.Hier2(ne, ne, p, nu_pre=2, nu_post=2, degree=4, coarse_rtol=1e-13, **WARPED2)
        lv = H.levels[0]
        r = H.solve(lv.load_vector(1), mode=1, rtol=1e-12, maxit=200)
        assert r["converged"]
        return np.abs(r["x"] - lv.exact_solution()).max()
    for p, nes in ((1, (8, 16, 32)), (2, (4, 8, 16)), (4, (2, 4, 8))):
        e = [err(ne, p) for ne in nes]
        rates = np.log2(np.array(e[:-1]) / np.array(e[1:]))
        assert rates[-1] >= p + 0.5, (p, e, rates)
    ep = [err(4, p) for p in (1, 2, 4, 8)]
    ratios = np.array(ep[:-1]) / np.array(ep[1:])
    assert np.all(ratios > 4) and np.all(np.diff(ratios) > 0), ep


def test_vcycle_two_level_closed_form_2d(orc):
    H = orc.Hier2(4, 2, 2, nu_pre=2, nu_post=2, degree=3, coarse_rtol=1e-15, **WARPED2)   # 2 -> 1
    assert H.nlevels == 2
    F, Cl = H.levels
    A = F.assemble_dense(0)
    Ac = Cl.assemble_dense(0)
    I = np.eye(F.N)
    P0 = np.stack([orc.prolong2(Cl, F, e) for e in np.eye(Cl.N)], axis=1)
    d = np.diag(A)
    lam = H.lam(0)
    lo, hi = 0.1 * lam, 1.1 * lam
    theta, delta = 0.5 * (hi + lo), 0.5 * (hi - lo)
    X = (theta * I - A / d[:, None]) / delta
    T = [I, X]
    for _ in range(2):
        T.append(2 * X @ T[-1] - T[-2])
    E = T[3] / np.cosh(3 * np.arccosh(theta / delta))
    S = E @ E
    Cc = I - P0 @ np.linalg.solve(Ac, P0.T @ A)
    Bref = (I - S @ Cc @ S) @ np.linalg.inv(A)
    B = np.stack([H.vcycle(e) for e in I], axis=1)
    np.testing.assert_allclose(B, Bref, rtol=0, atol=1e-9 * np.abs(Bref).max())


def test_lambda_and_chebyshev_2d(orc):
    L = orc.Level2(3, 3, 3, **WARPED2)
    A = L.assemble_dense(0)
    d = np.diag(A)
    lam_dense = np.linalg.eigvals(A / d[:, None]).real.max()
    lp, la = L.lambda_max(10, 12345), L.lambda_arnoldi(10, 12345)
    assert 0.5 * lam_dense < lp <= la <= lam_dense * (1 + 1e-12)
    x0 = np.random.default_rng(4).uniform(-1, 1, L.N)
    lo, hi = 0.1 * la, 1.1 * la
    x = L.cheb(np.zeros(L.N), x0, 4, lo, hi)
    theta, delta = 0.5 * (hi + lo), 0.5 * (hi - lo)
    Xm = (theta * np.eye(L.N) - A / d[:, None]) / delta
    T = [np.eye(L.N), Xm]
    for _ in range(3):
        T.append(2 * Xm @ T[-1] - T[-2])
    ref = (T[4] / np.cosh(4 * np.arccosh(theta / delta))) @ x0
    np.testing.assert_allclose(x, ref, rtol=0, atol=1e-11 * np.abs(ref).max())


def paper_rows():
    rows = {}
    for line in open(GOLDEN):
        if line.strip() and not line.startswith("#"):
            v = [t for t in line.split()]
            rows[int(v[0])] = [None if t == "-" else int(t) for t in v[1:]]
    return rows


def tab_counts(orc, p, coarsen):
    out = []
    for mode in (0, 1):
        for sm in (1, 0):
            nu = 3 if sm == 1 else 1
            H = orc.Hier2(32, 32, p, nu_pre=nu, nu_post=nu, degree=3, lo_frac=0.25, hi_frac=1.0, power_iters=10,
                          smoother=sm, omega=2.0 / 3.0, lambda_method=1, h_levels=2, coarsen=coarsen)
            r = H.solve(H.levels[0].load_vector(1), mode=mode, rtol=1e-8, maxit=200)
            assert r["converged"]
            out.append(r["iterations"])
    return out


@pytest.mark.parametrize("p", [2, 4])
def test_tab_box_gauss_quadrature(orc, p):
    """tab:box (tests/golden/tab_box.txt): with the paper's settings and Gauss
    quadrature the h-multigrid columns and the Chebyshev columns agree to +-1 for p = 2, 4 (the
    Jacobi p-multigrid columns converge faster here)."""
    orc.set_quadrature(1)
    try:
        h = tab_counts(orc, p, 1)
        pm = tab_counts(orc, p, 0)
    finally:
        orc.set_quadrature(0)
    row = paper_rows()[p]   # MG-J h, p, MG-C h, p, pCG-J h, p, pCG-C h, p
    paper_h = [row[0], row[2], row[4], row[6]]
    paper_p = [row[1], row[3], row[5], row[7]]
    assert np.all(np.abs(np.array(h) - np.array(paper_h)) <= 1), (h, paper_h)
    cheb = [1, 3]   # MG-C, pCG-C
    assert np.all(np.abs(np.array(pm)[cheb] - np.array(paper_p)[cheb]) <= 1), (pm, paper_p)
