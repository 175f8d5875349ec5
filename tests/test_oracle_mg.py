"""Pins of the oracle's transfer operators (eq. (7)), lambda_max (R9),
Chebyshev smoother (R7), coarse CG and V-cycle / MG solvers (Algorithm 1,
P:973-991) against closed forms, an independent Kronecker construction and
algebraic invariants.  No GPU."""
import numpy as np
import pytest

from test_oracle_operator import np_lgl, WARPED


def np_lagrange_matrix(xc, xf):
    """I[i][a] = ell_a(xf_i) on nodes xc, by the barycentric formula (independent of the oracle)."""
    n = len(xc)
    lam = np.array([1.0 / np.prod([xc[j] - xc[k] for k in range(n) if k != j]) for j in range(n)])
    I = np.zeros((len(xf), n))
    for i, t in enumerate(xf):
        hit = np.flatnonzero(t == xc)
        if len(hit):
            I[i, hit[0]] = 1.0
            continue
        c = lam / (t - xc)
        I[i] = c / c.sum()
    return I


def np_global_P1(ne, pc):
    """1-D global p-prolongation p/2 -> p on ne elements (unmasked)."""
    pf = 2 * pc
    xc, _ = np_lgl(pc)
    xf, _ = np_lgl(pf)
    I = np_lagrange_matrix(xc, xf)
    P = np.zeros((ne * pf + 1, ne * pc + 1))
    for e in range(ne):
        P[e * pf:e * pf + pf + 1, e * pc:e * pc + pc + 1] = I   # shared nodes: identical rows
    return P


def np_P0(shape, pc, mask_c, mask_f):
    nex, ney, nez = shape
    P = np.kron(np_global_P1(nez, pc), np.kron(np_global_P1(ney, pc), np_global_P1(nex, pc)))
    return np.diag(1.0 - mask_f) @ P @ np.diag(1.0 - mask_c)


@pytest.mark.parametrize("shape,pc", [((2, 2, 2), 1), ((2, 3, 1), 2), ((1, 2, 2), 4)])
def test_prolong_restrict_kronecker_and_adjoint(orc, shape, pc):
    C = orc.Level(*shape, pc, **WARPED)
    F = orc.Level(*shape, 2 * pc, **WARPED)
    P0 = np_P0(shape, pc, C.mask().astype(float), F.mask().astype(float))
    rng = np.random.default_rng(3)
    uc = rng.uniform(-1, 1, C.N)
    rf = rng.uniform(-1, 1, F.N)
    uf = orc.prolong(C, F, uc)
    np.testing.assert_allclose(uf, P0 @ uc, rtol=0, atol=1e-13)
    rc = orc.restrict(C, F, rf)
    np.testing.assert_allclose(rc, P0.T @ rf, rtol=0, atol=1e-12)
    assert abs(uf @ rf - uc @ rc) < 1e-12 * abs(uf @ rf)
    # P 1 = 1 away from the boundary elements (P0 masks coarse boundary values to zero)
    ones = orc.prolong(C, F, np.ones(C.N))
    Mf = [s * 2 * pc + 1 for s in shape]
    ones = ones.reshape(Mf[2], Mf[1], Mf[0])
    inner = ones[2 * pc:-2 * pc, 2 * pc:-2 * pc, 2 * pc:-2 * pc]
    if inner.size:
        np.testing.assert_allclose(inner, 1.0, atol=1e-14)


def test_prolong_polynomial_exactness(orc):
    """A coarse polynomial of degree <= pc per direction that vanishes on the boundary is
    reproduced exactly at the fine nodes."""
    shape, pc = (2, 2, 2), 2
    C = orc.Level(*shape, pc)
    F = orc.Level(*shape, 2 * pc)
    def nodal(L):
        l2g = L.l2g_closed()
        X = np.zeros((3, L.N))
        for e in range(L.E):
            X[:, l2g[e]] = L.geometry(e)[2]
        return X
    f = lambda X: X[0] * (1 - X[0]) * X[1] * (1 - X[1]) * X[2] * (1 - X[2])
    np.testing.assert_allclose(orc.prolong(C, F, f(nodal(C))), f(nodal(F)), atol=1e-15)


def test_transfer_rejects_bad_pairs(orc):
    with pytest.raises(ValueError):
        orc.prolong(orc.Level(2, 2, 2, 2), orc.Level(2, 2, 2, 3), np.zeros(125))


def test_lambda_max_pins(orc):
    # one interior dof: D^{-1} A_D is the identity on it and on the boundary -> lambda = 1
    L = orc.Level(2, 2, 2, 1, **WARPED)
    assert abs(L.lambda_max(10, 12345) - 1.0) < 1e-14
    for p in (1, 2, 4):
        L = orc.Level(3, 3, 3, p, **WARPED)
        A = L.assemble_dense(0)
        d = np.diag(A)
        lam = np.linalg.eigvalsh(A / np.sqrt(np.outer(d, d))).max()
        est = L.lambda_max(10, 12345)
        assert 0.5 * lam < est <= lam * (1 + 1e-12), (p, est, lam)


@pytest.mark.parametrize("p,iters", [(2, 10), (2, 3), (3, 10)])
def test_lambda_max_closed_form(orc, p, iters):
    """R9 / P:576-578: after `iters` power steps on D^{-1}A_D the estimate is the D-Rayleigh
    quotient of the last iterate, lambda = (x^T A x)/(x^T D x) with x proportional to
    (D^{-1}A_D)^(iters-1) x0 -- formed here from a dense matrix power (no iteration, no normalisation),
    with x0 = splitmix64(12345) in [-1,1] and the boundary zeroed (R15).  Pins the preconditioned
    operator (D^{-1}A, not A) and the iteration count (an off-by-one changes the value)."""
    from paper_1402_5938_b200 import inputs
    L = orc.Level(3, 3, 3, p, **WARPED)
    A = L.assemble_dense(0)
    d = np.diag(A).copy()
    x0 = inputs.uniform_pm1(12345, L.N)
    x0[L.mask() == 1] = 0.0
    x = np.linalg.matrix_power(A / d[:, None], iters - 1) @ x0
    ref = (x @ A @ x) / (x @ (d * x))
    est = L.lambda_max(iters, 12345)
    assert abs(est - ref) <= 1e-13 * ref, (est, ref)
    if iters == 10:   # the neighbouring counts and the unpreconditioned iteration all differ by far more
        for k in (iters - 2, iters):
            y = np.linalg.matrix_power(A / d[:, None], k) @ x0
            assert abs((y @ A @ y) / (y @ (d * y)) - ref) > 1e-9 * ref
        y = np.linalg.matrix_power(A, iters - 1) @ x0
        assert abs((y @ A @ y) / (y @ (d * y)) - ref) > 1e-6 * ref


def cheb_error_operator(A, lam_lo, lam_hi, K):
    """T_K((theta I - D^{-1}A)/delta) / T_K(theta/delta): the error propagator of R7."""
    d = np.diag(A)
    theta, delta = (lam_hi + lam_lo) / 2, (lam_hi - lam_lo) / 2
    Z = (theta * np.eye(len(d)) - A / d[:, None]) / delta
    T0, T1 = np.eye(len(d)), Z.copy()
    t0, t1 = 1.0, theta / delta
    for _ in range(K - 1):
        T0, T1 = T1, 2 * Z @ T1 - T0
        t0, t1 = t1, 2 * (theta / delta) * t1 - t0
    return (T1 if K >= 1 else T0) / t1


@pytest.mark.parametrize("K", [1, 2, 3, 4, 6])
def test_chebyshev_closed_form(orc, K):
    L = orc.Level(2, 2, 2, 2, **WARPED)
    A = L.assemble_dense(0)
    rng = np.random.default_rng(K)
    b = rng.uniform(-1, 1, L.N)
    x0 = rng.uniform(-1, 1, L.N)
    lam = L.lambda_max(10, 12345)
    lo, hi = 0.1 * lam, 1.1 * lam
    xs = np.linalg.solve(A, b)
    xk = L.cheb(b, x0, K, lo, hi)
    ek = cheb_error_operator(A, lo, hi, K) @ (x0 - xs)
    np.testing.assert_allclose(xk - xs, ek, rtol=0, atol=1e-12 * np.abs(x0 - xs).max())
    # exact input is a fixed point
    np.testing.assert_allclose(L.cheb(A @ x0, x0, K, lo, hi), x0, rtol=0, atol=1e-13)


def test_cg_dense_pin(orc):
    x, it, rc = orc.cg_dense(np.array([[4.0, 1.0], [1.0, 3.0]]), np.array([1.0, 2.0]))
    assert rc == 0 and it <= 2
    np.testing.assert_allclose(x, [1 / 11, 7 / 11], rtol=1e-14)
    x, it, rc = orc.cg_dense(np.eye(5), np.arange(1.0, 6.0))
    assert it == 1
    _, _, rc = orc.cg_dense(np.array([[1.0, 0.0], [0.0, -1.0]]), np.array([0.0, 1.0]))
    assert rc == 6   # breakdown on (p, Ap) <= 0


def two_level_matrix(orc, H, nu):
    """Closed form of the two-level V-cycle from x=0: B = (I - E^nu C E^nu) A^{-1},
    E = Chebyshev error propagator, C = I - P0 A_c^{-1} R A (exact coarse solve)."""
    F, Cl = H.levels
    A = F.assemble_dense(0)
    Ac = Cl.assemble_dense(0)
    shape = (F.nex, F.ney, F.nez)
    P0 = np_P0(shape, Cl.p, Cl.mask().astype(float), F.mask().astype(float))
    lam = H.lam(0)
    E = cheb_error_operator(A, 0.1 * lam, 1.1 * lam, 3)
    En = np.linalg.matrix_power(E, nu)
    Cc = np.eye(F.N) - P0 @ np.linalg.solve(Ac, P0.T @ A)
    return (np.eye(F.N) - En @ Cc @ En) @ np.linalg.inv(A)


def test_vcycle_two_level_matrix_linear_symmetric(orc):
    kw = dict(nu_pre=2, nu_post=2, degree=3, coarse_rtol=1e-15, geom_tier=2, tier=2)
    H = orc.Hier(2, 2, 2, 2, **WARPED, **kw)
    assert H.nlevels == 2
    # Hier levels carry mesh metadata for the numpy construction
    for lv in H.levels:
        lv.nex = lv.ney = lv.nez = 2
    N = H.N
    B = np.stack([H.vcycle(np.eye(N)[i]) for i in range(N)], axis=1)
    Bref = two_level_matrix(orc, H, 2)
    s = np.abs(Bref).max()
    np.testing.assert_allclose(B, Bref, rtol=0, atol=1e-9 * s)
    np.testing.assert_allclose(B, B.T, rtol=0, atol=1e-9 * s)
    rng = np.random.default_rng(5)
    b1, b2 = rng.uniform(-1, 1, N), rng.uniform(-1, 1, N)
    np.testing.assert_allclose(H.vcycle(2.5 * b1 + b2), 2.5 * H.vcycle(b1) + H.vcycle(b2),
                               rtol=0, atol=1e-9 * s)


def test_solver_counters_and_modes(orc):
    H = orc.Hier(3, 3, 3, 4, nu_pre=2, nu_post=2, degree=4, **WARPED)
    assert H.nlevels == 3
    b = H.levels[0].load_vector(1)
    pcg = H.solve(b, mode=1, rtol=1e-8)
    mg = H.solve(b, mode=0, rtol=1e-8)
    assert pcg["converged"] and mg["converged"]
    assert pcg["r_norm"] <= 1e-8 * pcg["r0_norm"] and mg["r_norm"] <= 1e-8 * mg["r0_norm"]
    per_v = (2 + 2) * 4 + 1                      # (nu_pre + nu_post) K + 1
    it = pcg["iterations"]
    assert pcg["fine_applies"] == it * per_v + it   # it V-cycles + it h = A p
    assert mg["fine_applies"] == mg["iterations"] * (per_v + 1)
    assert pcg["iterations"] <= mg["iterations"]
    assert len(pcg["history"]) == it + 1
    A = H.levels[0]
    r = b - A.apply(pcg["x"], 0, tier=3)
    assert np.linalg.norm(r) <= 1.0000001e-8 * np.linalg.norm(b)


def test_invalid_hierarchy(orc):
    with pytest.raises(ValueError):
        orc.Hier(2, 2, 2, 6)   # 6 -> 3 -> cannot p-coarsen
