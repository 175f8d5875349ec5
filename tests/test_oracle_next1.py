"""Pins of the oracle's NEXT-1 pieces: h-coarsening transfer at one order (eq. (7)
across nested element grids), the lambda_max estimate by Arnoldi iterations
(reading R26), damped point Jacobi (omega = 2/3) and the
paper-style hierarchy p -> ... -> 1 followed by geometric coarsening.  Pinned against
an independent hat-function / Lagrange construction, dense eigenvalues, convergence properties and
the closed two-level matrix form.  No GPU."""
import numpy as np
import pytest

from test_oracle_mg import np_lagrange_matrix
from test_oracle_operator import np_lgl, WARPED


def np_global_h1(nec, p):
    """1-D global h-prolongation at order p from nec coarse elements to 2 nec fine elements: fine node
    positions (two fine elements per coarse element) evaluated in the coarse element's Lagrange basis."""
    x, _ = np_lgl(p)
    # local coordinates in [-1, 1] of the fine nodes of the two halves of one coarse element
    left = -1.0 + 0.5 * (x + 1.0)
    right = 0.5 * (x + 1.0)
    Il = np_lagrange_matrix(x, left)
    Ir = np_lagrange_matrix(x, right)
    P = np.zeros((2 * nec * p + 1, nec * p + 1))
    for e in range(nec):
        P[2 * e * p:2 * e * p + p + 1, e * p:e * p + p + 1] = Il
        P[(2 * e + 1) * p:(2 * e + 1) * p + p + 1, e * p:e * p + p + 1] = Ir
    return P


def np_hat_h1(nec):
    """p = 1: piecewise-linear hats, P[I_f, J_c] = max(0, 1 - |x_f - x_c| / h_c)."""
    xf = np.arange(2 * nec + 1) / (2.0 * nec)
    xc = np.arange(nec + 1) / float(nec)
    return np.maximum(0.0, 1.0 - np.abs(xf[:, None] - xc[None, :]) * nec)


def np_P0_h(shape_c, p, mask_c, mask_f, hat=False):
    f = (lambda n: np_hat_h1(n)) if hat else (lambda n: np_global_h1(n, p))
    P = np.kron(f(shape_c[2]), np.kron(f(shape_c[1]), f(shape_c[0])))
    return np.diag(1.0 - mask_f) @ P @ np.diag(1.0 - mask_c)


@pytest.mark.parametrize("shape_c,p", [((1, 1, 1), 1), ((2, 2, 2), 1), ((2, 1, 3), 1), ((1, 2, 1), 2),
                                       ((1, 1, 2), 3), ((1, 1, 1), 4)])
def test_h_prolong_restrict_against_hats_and_adjoint(orc, shape_c, p):
    C = orc.Level(*shape_c, p, **WARPED)
    F = orc.Level(*[2 * s for s in shape_c], p, **WARPED)
    mc, mf = C.mask().astype(float), F.mask().astype(float)
    P0 = np_P0_h(shape_c, p, mc, mf)
    if p == 1:   # two independent constructions agree
        np.testing.assert_allclose(P0, np_P0_h(shape_c, p, mc, mf, hat=True), atol=1e-15)
    rng = np.random.default_rng(11)
    uc = rng.uniform(-1, 1, C.N)
    rf = rng.uniform(-1, 1, F.N)
    uf = orc.prolong(C, F, uc)
    np.testing.assert_allclose(uf, P0 @ uc, rtol=0, atol=1e-14)
    rc = orc.restrict(C, F, rf)
    np.testing.assert_allclose(rc, P0.T @ rf, rtol=0, atol=1e-13)
    assert abs(uf @ rf - uc @ rc) <= 1e-12 * max(1.0, abs(uf @ rf))


def test_h_pair_rules(orc):
    with pytest.raises(ValueError):   # neither a p pair nor an h pair
        orc.prolong(orc.Level(2, 2, 2, 1), orc.Level(3, 3, 3, 1), np.zeros(27))
    with pytest.raises(ValueError):
        orc.Hier(6, 6, 6, 2, h_levels=2)   # 6 -> 3 -> cannot halve


def interior_dense_lambda(L):
    A = L.assemble_dense(0)
    inner = ~L.mask().astype(bool)
    Ai = A[np.ix_(inner, inner)]
    d = np.diag(Ai)
    return np.linalg.eigvalsh(Ai / np.sqrt(np.outer(d, d)))


def test_lambda_arnoldi_exact_on_small_krylov_space(orc):
    # 1 interior dof: D^{-1} A_D = 1 there
    assert abs(orc.Level(2, 2, 2, 1, **WARPED).lambda_arnoldi(10, 12345) - 1.0) < 1e-14
    # 9 interior dofs <= 10 Arnoldi steps: the Krylov space is the whole interior space, so the
    # largest Ritz value is the largest eigenvalue of the interior D^{-1} A
    L = orc.Level(1, 2, 2, 2, **WARPED)
    ev = interior_dense_lambda(L)
    assert len(ev) == 9
    assert abs(L.lambda_arnoldi(10, 12345) - ev.max()) <= 1e-12 * ev.max()


@pytest.mark.parametrize("p", [1, 2, 4])
def test_lambda_arnoldi_bounds(orc, p):
    """power-iteration Rayleigh quotient (a vector of K_10) <= max Ritz value of K_10 <= lambda_max,
    and the estimate grows with the Krylov dimension."""
    L = orc.Level(3, 3, 3, p, **WARPED)
    lam = interior_dense_lambda(L).max()
    a10 = L.lambda_arnoldi(10, 12345)
    assert L.lambda_max(10, 12345) <= a10 * (1 + 1e-12)
    assert a10 <= lam * (1 + 1e-12)
    assert L.lambda_arnoldi(4, 12345) <= a10 * (1 + 1e-12)
    assert a10 >= 0.9 * lam


def test_jacobi_fixed_point_and_convergence(orc):
    L = orc.Level(2, 2, 2, 2, **WARPED)
    A = L.assemble_dense(0)
    rng = np.random.default_rng(2)
    x = rng.uniform(-1, 1, L.N)
    # an exact solution is a fixed point
    np.testing.assert_allclose(L.jacobi(A @ x, x, 3), x, rtol=0, atol=1e-13)
    # omega = 2/3 < 2 / lambda_max(D^-1 A): the iteration converges to A^{-1} b
    b = rng.uniform(-1, 1, L.N)
    xs = np.linalg.solve(A, b)
    xk = L.jacobi(b, np.zeros(L.N), 600)
    np.testing.assert_allclose(xk, xs, rtol=0, atol=1e-9 * np.abs(xs).max())


def test_vcycle_two_level_h_pair_jacobi(orc):
    """Two-level V(3,3)-cycle with damped Jacobi and an h-coarsened p = 1 coarse grid equals the closed
    form (I - E^3 C E^3) A^{-1}, E = I - omega D^{-1} A, C = I - P0 A_c^{-1} P0^T A."""
    kw = dict(nu_pre=3, nu_post=3, smoother=1, omega=2.0 / 3.0, coarse_rtol=1e-15, geom_tier=2, tier=2,
              h_levels=1)
    H = orc.Hier(2, 2, 4, 1, **WARPED, **kw)
    assert H.nlevels == 2
    F, Cl = H.levels
    A = F.assemble_dense(0)
    Ac = Cl.assemble_dense(0)
    P0 = np_P0_h((1, 1, 2), 1, Cl.mask().astype(float), F.mask().astype(float), hat=True)
    d = np.diag(A)
    E = np.eye(F.N) - (2.0 / 3.0) * A / d[:, None]
    E3 = np.linalg.matrix_power(E, 3)
    Cc = np.eye(F.N) - P0 @ np.linalg.solve(Ac, P0.T @ A)
    Bref = (np.eye(F.N) - E3 @ Cc @ E3) @ np.linalg.inv(A)
    N = F.N
    B = np.stack([H.vcycle(np.eye(N)[i]) for i in range(N)], axis=1)
    s = np.abs(Bref).max()
    np.testing.assert_allclose(B, Bref, rtol=0, atol=1e-10 * s)
    np.testing.assert_allclose(B, B.T, rtol=0, atol=1e-10 * s)


def test_paper_hierarchy_counters(orc):
    """p-coarsening to 1, then geometric coarsening 8^3 -> 4^3 -> 2^3 (here 4^3 -> 2^3
    -> 1^3); Jacobi(3,3) costs one residual and six fine applies per V-cycle."""
    H = orc.Hier(4, 4, 4, 4, nu_pre=3, nu_post=3, smoother=1, lambda_method=1, h_levels=2, **WARPED)
    assert H.nlevels == 5
    assert [lv.N for lv in H.levels] == [17 ** 3, 9 ** 3, 5 ** 3, 3 ** 3, 2 ** 3]
    b = H.levels[0].load_vector(1)
    mg = H.solve(b, mode=0, rtol=1e-8)
    pcg = H.solve(b, mode=1, rtol=1e-8)
    assert mg["converged"] and pcg["converged"]
    assert mg["fine_applies"] == mg["iterations"] * (7 + 1)
    assert pcg["fine_applies"] == pcg["iterations"] * (7 + 1)
    assert pcg["iterations"] <= mg["iterations"]
    r = b - H.levels[0].apply(pcg["x"], 0, tier=3)
    assert np.linalg.norm(r) <= 1.0000001e-8 * np.linalg.norm(b)


# ------------------------------------------------------------------ NEXT-4: high-order h-multigrid


def test_vcycle_two_level_high_order_h_pair(orc):
    """NEXT-4: two-level V(2,2) with degree-3 Chebyshev smoothing at order p = 2 on meshes
    2x2x2 -> 1x1x1 (coarsen = 1 keeps the order) equals the closed form (I - S C S) A^{-1} with
    S = T_3((theta - D^-1 A)/delta) / T_3(theta/delta) squared and C = I - P0 A_c^{-1} P0^T A, P0 from
    the independent global 1-D Lagrange construction."""
    kw = dict(nu_pre=2, nu_post=2, degree=3, coarse_rtol=1e-15, geom_tier=2, tier=2, h_levels=1, coarsen=1)
    H = orc.Hier(2, 2, 2, 2, **WARPED, **kw)
    assert H.nlevels == 2 and [lv.N for lv in H.levels] == [125, 27]
    F, Cl = H.levels
    A = F.assemble_dense(0)
    Ac = Cl.assemble_dense(0)
    P0 = np_P0_h((1, 1, 1), 2, Cl.mask().astype(float), F.mask().astype(float))
    d = np.diag(A)
    lam = H.lam(0)
    lo, hi = 0.1 * lam, 1.1 * lam
    theta, delta = 0.5 * (hi + lo), 0.5 * (hi - lo)
    X = (theta * np.eye(F.N) - A / d[:, None]) / delta
    T = [np.eye(F.N), X]
    for _ in range(2):
        T.append(2 * X @ T[-1] - T[-2])
    s3 = np.cosh(3 * np.arccosh(theta / delta))
    E = T[3] / s3   # degree-3 Chebyshev error propagator (R7)
    S = E @ E
    Cc = np.eye(F.N) - P0 @ np.linalg.solve(Ac, P0.T @ A)
    Bref = (np.eye(F.N) - S @ Cc @ S) @ np.linalg.inv(A)
    B = np.stack([H.vcycle(np.eye(F.N)[i]) for i in range(F.N)], axis=1)
    sc = np.abs(Bref).max()
    np.testing.assert_allclose(B, Bref, rtol=0, atol=1e-9 * sc)


@pytest.mark.parametrize("p", [1, 3])
def test_high_order_h_hierarchy_counters(orc, p):
    """three meshes at one order (odd p allowed, no p-coarsening); Cheb(3,3) costs one
    residual and six fine applies per V-cycle; pCG <= MG-solver iterations."""
    H = orc.Hier(4, 4, 4, p, nu_pre=1, nu_post=1, degree=3, lo_frac=0.25, hi_frac=1.0, lambda_method=1,
                 h_levels=2, coarsen=1, **WARPED)
    assert H.nlevels == 3
    assert [lv.N for lv in H.levels] == [(4 * p + 1) ** 3, (2 * p + 1) ** 3, (p + 1) ** 3]
    b = H.levels[0].load_vector(1)
    mg = H.solve(b, mode=0, rtol=1e-8)
    pcg = H.solve(b, mode=1, rtol=1e-8)
    assert mg["converged"] and pcg["converged"]
    assert mg["fine_applies"] == mg["iterations"] * (7 + 1)
    assert pcg["fine_applies"] == pcg["iterations"] * (7 + 1)
    assert pcg["iterations"] <= mg["iterations"]
    r = b - H.levels[0].apply(pcg["x"], 0, tier=3)
    assert np.linalg.norm(r) <= 1.0000001e-8 * np.linalg.norm(b)
