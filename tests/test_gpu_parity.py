"""GPU <-> oracle parity through the C ABI (run on a B200 with -m gpu).

Bars (BASELINE north_star):
  index maps, mask, colours           bit-exact
  geometric factors                   max |dG| <= 1e-12 max |G|
  A u and diag                        max |dv| <= 1e-11 ||A||_inf ||u||_inf (R19: ||A u||_inf when A
                                      is not assembled, which is the stricter normaliser)
  Chebyshev / V-cycle iterates        max |dx| <= 1e-11 ||x_oracle||_inf (R18); V-cycle bar
                                      1e-8 because its coarse CG stops at 1e-10 (R13)
  solves                              iterations +-1, final residual <= rtol
"""
import numpy as np
import pytest

from paper_1402_5938_b200 import inputs

pytestmark = pytest.mark.gpu

WARP = dict(warp=1, amp=0.1, coeff=1, c0=1.0, c1=3.0)


@pytest.fixture(scope="module")
def S():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1402_5938_b200 import sfmg
    return sfmg


def gpu_level(S, d):
    return S.Level(S.Problem.from_dict(d))


def orc_level(orc, d, eager=True, tier=2, geom_tier=2):
    return orc.Level(d["nex"], d["ney"], d["nez"], d["p"], d.get("warp", 0), d.get("amp", 0.0), d.get("coeff", 0),
                     d.get("c0", 1.0), d.get("c1", 0.0), eager=eager, tier=tier, geom_tier=geom_tier)


def to_gpu(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def rel_err(got, ref, scale):
    return float(np.abs(np.asarray(got) - np.asarray(ref)).max() / scale)


SMALL = [inputs.problem(1, p, **WARP) for p in range(1, 17)] + \
        [inputs.problem(2, p, ney=1, nez=1, **WARP) for p in (1, 2, 3, 4, 7, 8, 16)] + \
        [inputs.problem(3, 2, ney=2, nez=4, **WARP), inputs.problem(2, 5, ney=3, nez=2, warp=1, amp=0.05, coeff=2, c1=2.0),
         inputs.problem(4, 1, ney=3, nez=2, coeff=3, c0=1.0, c1=1e6), inputs.problem(4, 4)]


def _id(d):
    return "%dx%dx%d_p%d_w%d_c%d" % (d["nex"], d["ney"], d["nez"], d["p"], d.get("warp", 0), d.get("coeff", 0))


@pytest.mark.parametrize("d", SMALL[::3] + [SMALL[-1]], ids=_id)
def test_index_maps_bit_exact(S, orc, d):
    g = gpu_level(S, d)
    o = orc_level(orc, d)
    np.testing.assert_array_equal(g.export_l2g().cpu().numpy(), o.l2g_by_matching())
    np.testing.assert_array_equal(g.export_mask().cpu().numpy(), o.mask())
    np.testing.assert_array_equal(g.export_colors().cpu().numpy(), o.colors())


@pytest.mark.parametrize("d", SMALL, ids=_id)
def test_geometry_apply_diag_small(S, orc, d):
    g = gpu_level(S, d)
    o = orc_level(orc, d)
    n = d["p"] + 1
    # exported layout [E][k][6][n^2] -> oracle's [6][n^3] with q = (i + n j) + n^2 k
    G = g.export_geometry().cpu().numpy().reshape(o.E, n, 6, n * n).transpose(0, 2, 1, 3).reshape(o.E, 6, n ** 3)
    for e in range(o.E):
        Go, _, _ = o.geometry(e)
        assert rel_err(G[e], Go, np.abs(Go).max()) <= 1e-12
    u = inputs.uniform_pm1(7, o.N)
    for bc in (0, 1):
        A = o.assemble_dense(bc) if (o.N <= 6000 and o.n ** 3 <= 343) else None
        ref = o.apply(u, bc, tier=2 if o.n ** 3 <= 729 else 3)
        normA = np.abs(A).sum(axis=1).max() if A is not None else np.abs(ref).max()
        got = g.apply(to_gpu(u), bc=bc).cpu().numpy()
        assert rel_err(got, ref, normA * np.abs(u).max()) <= 1e-11, bc
        dref = o.diag(bc)
        dgot = g.diag(bc).cpu().numpy()
        assert rel_err(dgot, dref, np.abs(dref).max()) <= 1e-11
    # boundary pass-through (bc 0) is exact; zero in -> zero out
    mask = o.mask().astype(bool)
    got = g.apply(to_gpu(u), bc=0).cpu().numpy()
    np.testing.assert_array_equal(got[mask], u[mask])
    z = g.apply(to_gpu(np.zeros(o.N))).cpu().numpy()
    assert not z.any()


def test_random_meshes_apply(S, orc):
    rng = np.random.default_rng(11)
    for _ in range(6):
        p = int(rng.choice([1, 2, 3, 4, 6, 8]))
        ne = [int(v) for v in rng.integers(2, 5, 3)]
        d = inputs.problem(ne[0], p, ney=ne[1], nez=ne[2], warp=1, amp=float(rng.uniform(0, 0.12)),
                           coeff=int(rng.integers(0, 4)), c0=1.0, c1=float(rng.uniform(0.5, 2.0)))
        g = gpu_level(S, d)
        o = orc_level(orc, d, tier=3, geom_tier=3)
        u = inputs.uniform_pm1(int(rng.integers(0, 1000)), o.N)
        ref = o.apply(u, 0, tier=3)
        got = g.apply(to_gpu(u)).cpu().numpy()
        assert rel_err(got, ref, np.abs(ref).max()) <= 1e-11, d


@pytest.mark.parametrize("p", [2, 4, 5])
def test_apply_unaligned_views(S, orc, p):
    """u and v as 8-byte-offset views (not 16-byte aligned): same result as the oracle."""
    import torch
    d = inputs.problem(2, p, ney=3, nez=2, **WARP)
    g = gpu_level(S, d)
    o = orc_level(orc, d, tier=3, geom_tier=3)
    u = inputs.uniform_pm1(5, o.N)
    ref = o.apply(u, 0, tier=3)
    ub = torch.zeros(o.N + 1, dtype=torch.float64, device="cuda")
    vb = torch.full((o.N + 1,), 7.0, dtype=torch.float64, device="cuda")
    ub[1:] = to_gpu(u)
    g.apply(ub[1:], vb[1:])
    assert float(vb[0]) == 7.0
    assert rel_err(vb[1:].cpu().numpy(), ref, np.abs(ref).max()) <= 1e-11


def test_config1_full_workload(S, orc):
    """Config 1: 4^3 affine, p=4, mu = 1; A u from seed 0, then a degree-3 Chebyshev application
    (b = 0, x0 = u, R16) on [0.1, 1.1] lambda_max with 10 power iterations (seed 12345)."""
    d = inputs.CONFIG1
    g = gpu_level(S, d)
    o = orc_level(orc, d)
    u = inputs.uniform_pm1(0, o.N)
    A = o.assemble_dense(0)
    ref = A @ u
    got = g.apply(to_gpu(u)).cpu().numpy()
    assert rel_err(got, ref, np.abs(A).sum(axis=1).max() * np.abs(u).max()) <= 1e-11
    lam_g, lam_o = g.lambda_max(10, inputs.POWER_SEED), o.lambda_max(10, inputs.POWER_SEED)
    assert abs(lam_g - lam_o) <= 1e-12 * lam_o
    b = np.zeros(o.N)
    xo = o.cheb(b, u, 3, 0.1 * lam_o, 1.1 * lam_o)
    xg = to_gpu(u)
    g.cheb(to_gpu(b), xg, 3, 0.1 * lam_o, 1.1 * lam_o)
    assert rel_err(xg.cpu().numpy(), xo, np.abs(xo).max()) <= 1e-11
    # host-buffer variants give the same numbers
    np.testing.assert_allclose(g.apply_host(u), got, rtol=0, atol=1e-14 * np.abs(got).max())
    xh = u.copy()
    g.cheb_host(b, xh, 3, 0.1 * lam_o, 1.1 * lam_o)
    np.testing.assert_allclose(xh, xg.cpu().numpy(), rtol=0, atol=1e-14 * np.abs(xo).max())


@pytest.mark.parametrize("K", [1, 2, 4, 5])
def test_chebyshev_small_nonzero_rhs(S, orc, K):
    d = inputs.problem(3, 4, ney=2, nez=2, **WARP)
    g = gpu_level(S, d)
    o = orc_level(orc, d)
    lam = o.lambda_max(10, 12345)
    assert abs(g.lambda_max(10, 12345) - lam) <= 1e-12 * lam
    b = inputs.uniform_pm1(3, o.N)
    x0 = inputs.uniform_pm1(4, o.N)
    xo = o.cheb(b, x0, K, 0.1 * lam, 1.1 * lam)
    xg = g.cheb(to_gpu(b), to_gpu(x0), K, 0.1 * lam, 1.1 * lam).cpu().numpy()
    assert rel_err(xg, xo, np.abs(xo).max()) <= 1e-11


@pytest.mark.parametrize("shape,pc", [((2, 2, 2), 1), ((3, 2, 1), 2), ((2, 2, 2), 4), ((1, 2, 1), 8)])
def test_transfer_parity(S, orc, shape, pc):
    dc = inputs.problem(shape[0], pc, ney=shape[1], nez=shape[2], **WARP)
    df = dict(dc, p=2 * pc)
    gc, gf = gpu_level(S, dc), gpu_level(S, df)
    oc, of = orc_level(orc, dc, tier=3, geom_tier=3), orc_level(orc, df, tier=3, geom_tier=3)
    uc = inputs.uniform_pm1(5, oc.N)
    rf = inputs.uniform_pm1(6, of.N)
    uf = S.prolong(gc, gf, to_gpu(uc)).cpu().numpy()
    ref = orc.prolong(oc, of, uc)
    assert rel_err(uf, ref, np.abs(ref).max()) <= 1e-13
    rc = S.restrict(gc, gf, to_gpu(rf)).cpu().numpy()
    ref = orc.restrict(oc, of, rf)
    assert rel_err(rc, ref, np.abs(ref).max()) <= 1e-12


def test_transfer_rejects_odd(S):
    a = gpu_level(S, inputs.problem(2, 3))
    b = gpu_level(S, inputs.problem(2, 5))
    import torch
    with pytest.raises(S.SfmgError) as ei:
        S.prolong(a, b, torch.zeros(a.N, dtype=torch.float64, device="cuda"))
    assert ei.value.status == "SFMG_E_PCOARSEN"


def test_error_paths(S):
    import torch
    with pytest.raises(S.SfmgError) as ei:
        gpu_level(S, inputs.problem(2, 2, warp=1, amp=2.0))
    assert ei.value.status == "SFMG_E_GEOMETRY"
    g = gpu_level(S, inputs.problem(2, 2))
    with pytest.raises(ValueError):
        g.apply(torch.zeros(g.N + 1, dtype=torch.float64, device="cuda"))


def test_vcycle_and_solves_small(S, orc):
    d = inputs.problem(3, 4, ney=3, nez=2, **WARP)
    prob = S.Problem.from_dict(d)
    H = S.Hierarchy(prob, S.MgParams())
    O = orc.Hier(d["nex"], d["ney"], d["nez"], d["p"], 1, 0.1, 1, 1.0, 3.0, geom_tier=3, tier=3)
    assert H.nlevels == O.nlevels == 3
    for l in range(H.nlevels - 1):
        assert abs(H.lam(l) - O.lam(l)) <= 1e-12 * O.lam(l)
    b = O.levels[0].load_vector(1)
    bg = H.levels[0].load_vector(1).cpu().numpy()
    assert rel_err(bg, b, np.abs(b).max()) <= 1e-12
    xo = O.vcycle(b)
    xg = H.vcycle(to_gpu(b)).cpu().numpy()
    assert rel_err(xg, xo, np.abs(xo).max()) <= 1e-8
    for mode in (0, 1):
        ro = O.solve(b, mode=mode, rtol=1e-8)
        xg, rg = H.solve(to_gpu(b), mode=mode, rtol=1e-8)
        assert rg["converged"] and ro["converged"]
        assert abs(rg["iterations"] - ro["iterations"]) <= 1
        assert rg["r_norm"] <= 1e-8 * rg["r0_norm"]
        assert rg["fine_applies"] == ro["fine_applies"] or abs(rg["iterations"] - ro["iterations"]) == 1
        assert rel_err(xg.cpu().numpy(), ro["x"], np.abs(ro["x"]).max()) <= 1e-6


@pytest.mark.parametrize("p", [1, 2, 3, 5, 8, 16])
def test_degenerate_and_bc1_cases(S, orc, p):
    """Edge cases: a single element (p = 1: no interior dof at all, A_D = I), the un-projected operator
    (bc = 1) against the oracle and its any-size property A 1 = 0, and a zero right-hand side."""
    import torch
    d = inputs.problem(1, p, **WARP)
    g = gpu_level(S, d)
    o = orc_level(orc, d, tier=3, geom_tier=3)
    u = inputs.uniform_pm1(3, g.N)
    for bc in (0, 1):
        ref = o.apply(u, bc, tier=3)
        got = g.apply(to_gpu(u), bc=bc).cpu().numpy()
        assert rel_err(got, ref, np.abs(ref).max()) <= 1e-11, (p, bc)
    if p == 1:
        np.testing.assert_array_equal(g.apply(to_gpu(u)).cpu().numpy(), u)   # every node is a boundary node
        with pytest.raises(S.SfmgError):
            g.lambda_max(10, 12345)
    # A 1 = 0 without the boundary projection, on a warped multi-element mesh
    d2 = inputs.problem(2, p, ney=1, nez=2, **WARP)
    g2 = gpu_level(S, d2)
    ones = torch.ones(g2.N, dtype=torch.float64, device="cuda")
    r = g2.apply(ones, bc=1).cpu().numpy()
    dg = g2.diag(bc=1).cpu().numpy()
    assert np.abs(r).max() <= 1e-12 * np.abs(dg).max(), p


def test_zero_rhs_solve(S):
    import torch
    H = S.Hierarchy(S.Problem.from_dict(inputs.problem(2, 4, **WARP)), S.MgParams())
    b = torch.zeros(H.N, dtype=torch.float64, device="cuda")
    for mode in (0, 1):
        x, rep = H.solve(b, mode=mode)
        assert rep["converged"] and rep["iterations"] == 0
        assert float(x.abs().max()) == 0.0


PIPE = [inputs.problem(4, 1, ney=8, nez=5, **WARP), inputs.problem(8, 2, ney=4, nez=3, **WARP),
        inputs.problem(3, 3, ney=2, nez=7, **WARP), inputs.problem(2, 8, ney=3, nez=4, **WARP),
        inputs.problem(2, 4, ney=2, nez=3, warp=0, coeff=0), inputs.problem(1, 16, ney=1, nez=2, **WARP)]


@pytest.mark.parametrize("d", PIPE, ids=_id)
@pytest.mark.parametrize("bc", [0, 1])
def test_apply_host_pipelined_slabs(S, orc, d, bc):
    """sfmg_apply_host split into z-slabs (host_pipeline): every slab count gives the oracle's A u
    (the cut planes are summed by two slabs, the true boundary planes pass u through)."""
    g = gpu_level(S, d)
    o = orc_level(orc, d)
    u = inputs.uniform_pm1(7, o.N)
    ref = o.apply(u, bc, tier=2)
    scale = np.abs(ref).max()
    dev = g.apply(to_gpu(u), bc=bc).cpu().numpy()
    for slabs in (1, 2, 3, d["nez"], 8):
        g.host_pipeline(slabs)
        got = g.apply_host(u, bc=bc)
        assert rel_err(got, ref, scale) <= 1e-11, slabs
        np.testing.assert_allclose(got, dev, rtol=0, atol=1e-14 * scale)
    g.host_pipeline(0)


def test_cheb_rejects_aliased_b_x(S):
    """sfmg_cheb alternates its iterates through x, so b == x would be overwritten mid-recurrence:
    the ABI rejects it (SFMG_E_ARG) and leaves x untouched."""
    import torch
    lv = gpu_level(S, inputs.problem(2, 4, **WARP))
    x = to_gpu(inputs.uniform_pm1(3, lv.N))
    x0 = x.clone()
    with pytest.raises(S.SfmgError):
        lv.cheb(x, x, 4, 0.1, 1.1)
    torch.cuda.synchronize()
    assert torch.equal(x, x0)


def test_repeated_standalone_applies(S, orc):
    """The standalone apply initialises v inside its persistent grid and synchronises the grid on a
    per-level barrier word pair that returns to its initial state after every launch: back-to-back
    applies (stream-ordered, programmatic-dependent launches) into the same and into different outputs
    all match the oracle, for the thread-per-element (p <= 2) and persistent (p >= 3) kernels."""
    import torch
    for p in (1, 2, 4, 8, 16):
        d = inputs.problem(2, p, ney=3, nez=2, **WARP)
        lv = gpu_level(S, d)
        o = orc_level(orc, d, tier=3)
        us = [inputs.uniform_pm1(40 + k, lv.N) for k in range(3)]
        refs = [o.apply(u, 0, 3) for u in us]
        ug = [to_gpu(u) for u in us]
        vs = [torch.full_like(ug[0], 7.0) for _ in range(3)]
        for rep in range(4):
            for k in range(3):
                lv.apply(ug[k], vs[k])
        torch.cuda.synchronize()
        for k in range(3):
            err = rel_err(vs[k].cpu().numpy(), refs[k], np.abs(refs[k]).max())
            assert err <= 1e-11, (p, k, err)
