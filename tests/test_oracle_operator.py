"""Pins of the oracle's mesh, geometry, operator and diagonal (P:326-385, P:421-462,
P:568-570) against closed forms, independent numpy constructions, invariants and an MMS
convergence study.  No GPU."""
import numpy as np
import pytest
from numpy.polynomial import legendre as npleg

WARPED = dict(warp=1, amp=0.1, coeff=1, c0=1.0, c1=3.0)


# ----------------------------------------------------------------------------- independent numpy basis
def np_lgl(p):
    x = np.sort(np.concatenate([[-1.0, 1.0], npleg.Legendre.basis(p).deriv().roots().real]))
    w = 2.0 / (p * (p + 1) * npleg.legval(x, [0] * p + [1]) ** 2)
    return x, w


def np_D(x):
    n = len(x)
    lam = np.array([1.0 / np.prod([x[j] - x[k] for k in range(n) if k != j]) for j in range(n)])
    D = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            if i != j:
                D[i, j] = (lam[j] / lam[i]) / (x[i] - x[j])
        D[i, i] = -D[i].sum()
    return D


def assembled_1d(ne, p, h, mu=None):
    """1-D assembled stiffness K and (diagonal) mass M on a uniform mesh of ne elements of length h,
    with collocated LGL quadrature and optional coefficient mu(x) sampled at the nodes."""
    x, w = np_lgl(p)
    D = np_D(x)
    M_ = ne * p + 1
    K = np.zeros((M_, M_))
    Mm = np.zeros((M_, M_))
    for e in range(ne):
        xs = e * h + (x + 1) * h / 2
        m = np.ones(p + 1) if mu is None else mu(xs)
        Ke = (2.0 / h) * D.T @ np.diag(w * m) @ D
        Me = (h / 2.0) * np.diag(w * m)
        sl = slice(e * p, e * p + p + 1)
        K[sl, sl] += Ke
        Mm[sl, sl] += Me
    return K, Mm


# ----------------------------------------------------------------------------- mesh
@pytest.mark.parametrize("shape,p", [((1, 1, 1), 3), ((2, 3, 4), 2), ((3, 1, 2), 4), ((4, 4, 4), 1)])
def test_l2g_matching_equals_closed_form_and_lattice(orc, shape, p):
    L = orc.Level(*shape, p)
    a = L.l2g_by_matching()
    b = L.l2g_closed()
    np.testing.assert_array_equal(a, b)
    nex, ney, nez = shape
    Mx, My = nex * p + 1, ney * p + 1
    n = p + 1
    # the lattice formula of SURVEY 8(a) a2, written from the index definitions
    for e in [0, L.E - 1, L.E // 2]:
        ex, ey, ez = e % nex, (e // nex) % ney, e // (nex * ney)
        for (aa, bb, cc) in [(0, 0, 0), (p, 0, 1 % n), (p, p, p)]:
            g = (ex * p + aa) + Mx * ((ey * p + bb) + My * (ez * p + cc))
            assert a[e, aa + n * (bb + n * cc)] == g


@pytest.mark.parametrize("shape,p", [((2, 3, 4), 2), ((3, 3, 3), 3), ((1, 2, 1), 4)])
def test_mesh_counts(orc, shape, p):
    L = orc.Level(*shape, p)
    Mx, My, Mz = [s * p + 1 for s in shape]
    assert L.N == Mx * My * Mz
    mask = L.mask()
    assert mask.sum() == Mx * My * Mz - (Mx - 2) * (My - 2) * (Mz - 2)
    l2g = L.l2g_by_matching()
    mult = np.bincount(l2g.ravel(), minlength=L.N)
    assert mult.sum() == L.E * (p + 1) ** 3
    assert set(np.unique(mult)) <= {1, 2, 4, 8}
    # colouring: no two elements of one colour share a node
    col = L.colors()
    for c in range(8):
        nodes = l2g[col == c].ravel()
        assert len(np.unique(nodes)) == len(nodes)


# ----------------------------------------------------------------------------- geometry
def test_geometry_affine_closed_form(orc):
    nex, ney, nez, p = 2, 3, 4, 3
    L = orc.Level(nex, ney, nez, p)
    x, w = np_lgl(p)
    G, dJ, X = L.geometry(5)
    hx, hy, hz = 1 / nex, 1 / ney, 1 / nez
    np.testing.assert_allclose(dJ, hx * hy * hz / 8, rtol=1e-14)
    W = np.einsum("k,j,i->kji", w, w, w).ravel()
    np.testing.assert_allclose(G[0], W * hy * hz / (2 * hx), rtol=1e-13)
    np.testing.assert_allclose(G[3], W * hx * hz / (2 * hy), rtol=1e-13)
    np.testing.assert_allclose(G[5], W * hx * hy / (2 * hz), rtol=1e-13)
    np.testing.assert_allclose(G[[1, 2, 4]], 0, atol=1e-15)


@pytest.mark.parametrize("p", [1, 2, 4, 5])
def test_geometry_tiers_agree(orc, p):
    A = orc.Level(2, 2, 2, p, geom_tier=2, **WARPED)
    B = orc.Level(2, 2, 2, p, geom_tier=3, **WARPED)
    for e in range(8):
        Ga, da, _ = A.geometry(e)
        Gb, db, _ = B.geometry(e)
        np.testing.assert_allclose(Ga, Gb, rtol=0, atol=1e-13 * np.abs(Ga).max())
        np.testing.assert_allclose(da, db, rtol=1e-13)


def test_geometry_folding_detected(orc):
    L = orc.Level(2, 2, 2, 2, warp=1, amp=2.0)
    assert L.status == 4 and L.min_detj() <= 0
    L = orc.Level(8, 8, 8, 1, **WARPED)
    # det J relative to the affine element's (h/2)^3; the warp keeps it in [0.55, 1.4]
    rel = L.min_detj() / (1 / 16) ** 3
    assert L.status == 0 and 0.5 < rel < 1.0


def np_element_matrix(Xe, p, mu_fn):
    """Brute force, independent of the oracle: isoparametric J by einsum, dense quadrature."""
    x, w = np_lgl(p)
    n = p + 1
    D = np_D(x)
    I = np.eye(n)
    # grad_ref phi_l at q, l = a + n(b + n c), q = i + n(j + n k)
    g0 = np.einsum("ia,jb,kc->kjicba", D, I, I).reshape(n ** 3, n ** 3)
    g1 = np.einsum("ia,jb,kc->kjicba", I, D, I).reshape(n ** 3, n ** 3)
    g2 = np.einsum("ia,jb,kc->kjicba", I, I, D).reshape(n ** 3, n ** 3)
    Gr = np.stack([g0, g1, g2])                      # [beta][q][l]
    J = np.einsum("bql,al->qab", Gr, Xe)            # J[q][alpha][beta]
    det = np.linalg.det(J)
    Ji = np.linalg.inv(J)
    W = np.einsum("k,j,i->kji", w, w, w).ravel()
    mu = mu_fn(Xe[0], Xe[1], Xe[2])
    M = np.einsum("q,qag,qbg->qab", W * mu * det, Ji, Ji)
    return np.einsum("aql,qab,bqm->lm", Gr, M, Gr)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_element_matrix_brute_force(orc, p):
    L = orc.Level(2, 2, 2, p, **WARPED)
    S = lambda x, y, z: np.sin(2 * np.pi * x) * np.sin(2 * np.pi * y) * np.sin(2 * np.pi * z)
    for e in (0, 5):
        _, _, X = L.geometry(e)
        K = L.element_matrix(e)
        Kb = np_element_matrix(X, p, lambda x, y, z: np.exp(3 * S(x, y, z)))
        np.testing.assert_allclose(K, Kb, rtol=0, atol=1e-12 * np.abs(Kb).max())


# coefficient kinds of BASELINE config 4 (mu = 10^(c1 S), contrast 1e4) and of the paper's 3d-var
# (mu = c0 + c1 sum_i cos^2(2 pi x_i)), each against the brute-force numpy element matrix
COEFF_KINDS = [
    (2, 1.0, 2.0, lambda x, y, z: 10.0 ** (2.0 * np.sin(2 * np.pi * x) * np.sin(2 * np.pi * y) * np.sin(2 * np.pi * z))),
    (3, 1.0, 1e6, lambda x, y, z: 1.0 + 1e6 * (np.cos(2 * np.pi * x) ** 2 + np.cos(2 * np.pi * y) ** 2
                                                + np.cos(2 * np.pi * z) ** 2)),
]


@pytest.mark.parametrize("kind,c0,c1,mu", COEFF_KINDS, ids=["pow10", "cos2"])
@pytest.mark.parametrize("p", [1, 2, 3])
def test_element_matrix_brute_force_coeff_kinds(orc, p, kind, c0, c1, mu):
    L = orc.Level(2, 2, 2, p, warp=1, amp=0.1, coeff=kind, c0=c0, c1=c1)
    for e in (0, 3, 6):
        _, _, X = L.geometry(e)
        K = L.element_matrix(e)
        Kb = np_element_matrix(X, p, mu)
        np.testing.assert_allclose(K, Kb, rtol=0, atol=1e-12 * np.abs(Kb).max())


@pytest.mark.parametrize("p", [1, 2, 4])
def test_element_matrix_affine_kronecker(orc, p):
    nex, ney, nez = 2, 3, 1
    L = orc.Level(nex, ney, nez, p)
    x, w = np_lgl(p)
    D = np_D(x)
    Kh = D.T @ np.diag(w) @ D
    W = np.diag(w)
    hx, hy, hz = 1 / nex, 1 / ney, 1 / nez
    Kref = (hy * hz / (2 * hx)) * np.kron(W, np.kron(W, Kh)) \
         + (hx * hz / (2 * hy)) * np.kron(W, np.kron(Kh, W)) \
         + (hx * hy / (2 * hz)) * np.kron(Kh, np.kron(W, W))
    K = L.element_matrix(3)
    np.testing.assert_allclose(K, Kref, rtol=0, atol=1e-13 * np.abs(Kref).max())
    if p == 1:   # 1-D p=1 element stiffness {{1,-1},{-1,1}}/h
        np.testing.assert_allclose((2 / 0.25) * Kh, np.array([[1, -1], [-1, 1]]) / 0.25)


@pytest.mark.parametrize("shape,p,sep", [((2, 3, 2), 2, False), ((3, 2, 2), 3, False), ((2, 2, 3), 2, True)])
def test_global_operator_kronecker_sum(orc, shape, p, sep):
    """Affine mesh, mu = 1 (or separable mu = e^{c x} e^{2c y} e^{3c z}, oracle-only kind 100):
    A = Mz (x) My (x) Kx + Mz (x) Ky (x) Mx + Kz (x) My (x) Mx with 1-D assembled matrices."""
    c1 = 0.7
    L = orc.Level(*shape, p, coeff=100 if sep else 0, c1=c1)
    A = L.assemble_dense(bc=1)
    nex, ney, nez = shape
    mus = [None] * 3
    if sep:
        mus = [lambda t: np.exp(c1 * t), lambda t: np.exp(2 * c1 * t), lambda t: np.exp(3 * c1 * t)]
    Kx, Mx = assembled_1d(nex, p, 1 / nex, mus[0])
    Ky, My = assembled_1d(ney, p, 1 / ney, mus[1])
    Kz, Mz = assembled_1d(nez, p, 1 / nez, mus[2])
    Aref = np.kron(Mz, np.kron(My, Kx)) + np.kron(Mz, np.kron(Ky, Mx)) + np.kron(Kz, np.kron(My, Mx))
    np.testing.assert_allclose(A, Aref, rtol=0, atol=1e-12 * np.abs(Aref).max())


@pytest.mark.parametrize("p", [1, 2, 4])
def test_operator_invariants_warped(orc, p):
    L = orc.Level(2, 2, 2, p, **WARPED)
    A1 = L.assemble_dense(bc=1)
    AD = L.assemble_dense(bc=0)
    s = np.abs(A1).max()
    np.testing.assert_allclose(A1, A1.T, rtol=0, atol=1e-13 * s)          # symmetry
    np.testing.assert_allclose(A1 @ np.ones(L.N), 0, atol=1e-12 * s)      # A 1 = 0, no BC
    assert np.linalg.eigvalsh(AD).min() > 0                               # SPD after projection
    rng = np.random.default_rng(0)
    u, v = rng.standard_normal(L.N), rng.standard_normal(L.N)
    Au, Av = L.apply(u, 0), L.apply(v, 0)
    assert abs(u @ Av - v @ Au) < 1e-12 * abs(u @ Av) + 1e-12
    np.testing.assert_allclose(Au, AD @ u, rtol=0, atol=1e-12 * np.abs(Au).max())
    np.testing.assert_allclose(L.apply(u, 1), A1 @ u, rtol=0, atol=1e-12 * np.abs(Au).max())


@pytest.mark.parametrize("shape,p", [((1, 1, 1), 5), ((2, 1, 1), 8), ((2, 2, 2), 4), ((1, 1, 1), 16)])
def test_apply_tiers_agree(orc, shape, p):
    """O2 (dense direct quadrature) == O3 (sum-factorised) == O1 (assembled) when small."""
    L = orc.Level(*shape, p, **WARPED)
    u = np.random.default_rng(1).uniform(-1, 1, L.N)
    for bc in (0, 1):
        v2 = L.apply(u, bc, tier=2)
        v3 = L.apply(u, bc, tier=3)
        np.testing.assert_allclose(v3, v2, rtol=0, atol=1e-13 * np.abs(v2).max())
        if L.N <= 1000:
            A = L.assemble_dense(bc)
            np.testing.assert_allclose(A @ u, v2, rtol=0, atol=1e-13 * np.abs(v2).max())
    rows = np.array([0, 1, L.N // 2, L.N - 2, 7])
    np.testing.assert_allclose(L.apply_rows(u, rows, 0, tier=2), L.apply(u, 0, tier=2)[rows], rtol=1e-14, atol=1e-14)


def test_patch_test_affine(orc):
    """Affine mesh, constant mu: A x_lin vanishes at interior nodes for any linear function."""
    L = orc.Level(3, 2, 2, 4, coeff=0, c0=2.5)
    # node coordinates on the affine lattice
    l2g = L.l2g_closed()
    X = np.zeros((3, L.N))
    for e in range(L.E):
        _, _, Xe = L.geometry(e)
        X[:, l2g[e]] = Xe
    xl = 0.3 + 1.7 * X[0] - 0.4 * X[1] + 2.2 * X[2]
    v = L.apply(xl, bc=1)
    interior = L.mask() == 0
    assert np.abs(v[interior]).max() < 1e-12 * np.abs(xl).max() * 100


def test_diag_definitions(orc):
    L = orc.Level(2, 2, 1, 3, **WARPED)
    d = L.diag(0)
    A = L.assemble_dense(0)
    np.testing.assert_allclose(d, np.diag(A), rtol=1e-13)
    assert np.all(d > 0)
    np.testing.assert_array_equal(d[L.mask() == 1], 1.0)
    e = np.zeros(L.N)
    g = int(np.flatnonzero(L.mask() == 0)[3])
    e[g] = 1.0
    assert abs(L.apply(e, 0)[g] - d[g]) < 1e-13 * d[g]
    np.testing.assert_allclose(L.diag(1), np.diag(L.assemble_dense(1)), rtol=1e-13)


def test_diag_translation_invariant_affine(orc):
    L = orc.Level(4, 4, 4, 2)
    d = L.diag(0).reshape(9, 9, 9)
    # interior element-vertex nodes at lattice positions 2,4,6 are all equivalent by translation
    v = d[2:7:2, 2:7:2, 2:7:2]
    np.testing.assert_allclose(v, v.flat[0], rtol=1e-14)


@pytest.mark.slow
def test_mms_convergence(orc):
    """Manufactured solution u* = sin(pi x) sin(pi y) sin(pi z), mu = exp(3S), warped mesh:
    nodal max error falls algebraically under h-refinement (order >= p + 0.5) and
    exponentially under p-refinement (SURVEY 8(c) pins, BASELINE north_star)."""
    def solve_err(ne, p):
        H = orc.Hier(ne, ne, ne, p, nu_pre=2, nu_post=2, degree=4, coarse_rtol=1e-13, **WARPED)
        lv = H.levels[0]
        b = lv.load_vector(1)
        res = H.solve(b, mode=1, rtol=1e-12, maxit=200)
        assert res["converged"]
        return np.abs(res["x"] - lv.exact_solution()).max()

    for p, nes in ((1, (4, 8, 16)), (2, (2, 4, 8)), (4, (2, 4, 8))):
        errs = [solve_err(ne, p) for ne in nes]
        rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
        assert rates[-1] >= p + 0.5, (p, errs, rates)
    ep = [solve_err(4, p) for p in (1, 2, 4, 8)]
    ratios = np.array(ep[:-1]) / np.array(ep[1:])
    # spectral convergence: the error ratio per doubling of p itself grows (6x, 25x, 260x here)
    assert np.all(ratios > 4) and np.all(np.diff(ratios) > 0) and ep[3] < 1e-4, ep
