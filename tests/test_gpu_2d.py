"""GPU <-> oracle parity of the NEXT-2 row: the 2-D quadrilateral variant
through the same C ABI (sfmg_problem.dim = 2): geometry, A u (both boundary modes), diag, load vector,
lambda estimates, Chebyshev and Jacobi, p- and h-transfer, and the p- and h-multigrid hierarchies
(MG solver and MG-PCG), for collocated LGL and Gauss quadrature, against oracle.Level2 / Hier2.

Bars as in 3-D (test_gpu_parity.py, test_gpu_next1.py): A u, diag, load and smoother iterates
1e-11 relative; transfers 1e-14 / 1e-13; lambda 1e-10; V-cycle 1e-8; iteration counts +-1.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
KINDS = [dict(warp=1, amp=0.1, coeff=1, c0=1.0, c1=3.0), dict(warp=1, amp=0.1, coeff=3, c0=1.0, c1=1e6),
         dict(warp=1, amp=0.05, coeff=4, c0=1.0, c1=1e6), dict(warp=0, coeff=0, c0=1.0)]


@pytest.fixture(scope="module")
def S():
    import torch
    assert torch.cuda.is_available()
    from paper_1402_5938_b200 import sfmg
    return sfmg


def to_gpu(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def prob2(nex, ney, p, quad=0, **kw):
    return dict(nex=nex, ney=ney, nez=1, p=p, dim=2, quadrature=quad, **kw)


def levels(S, orc, d):
    orc.set_quadrature(d["quadrature"])
    try:
        o = orc.Level2(d["nex"], d["ney"], d["p"], d.get("warp", 0), d.get("amp", 0.0), d.get("coeff", 0),
                       d.get("c0", 1.0), d.get("c1", 0.0))
    finally:
        orc.set_quadrature(0)
    return S.Level(S.Problem.from_dict(d)), o


CASES = [(3, 2, 1, 0, 0), (4, 3, 2, 1, 0), (2, 3, 3, 0, 1), (3, 3, 4, 2, 1), (2, 2, 8, 1, 0), (2, 1, 8, 0, 1),
         (1, 2, 16, 3, 0), (2, 2, 16, 1, 1), (3, 2, 5, 2, 0)]


@pytest.mark.parametrize("nex,ney,p,kind,quad", CASES)
def test_operator_parity_2d(S, orc, nex, ney, p, kind, quad):
    d = prob2(nex, ney, p, quad, **KINDS[kind])
    g, o = levels(S, orc, d)
    assert g.N == o.N == (nex * p + 1) * (ney * p + 1)
    u = np.random.default_rng(p + 7 * kind).uniform(-1, 1, g.N)
    for bc in (0, 1):
        ref = o.apply(u, bc)
        got = g.apply(to_gpu(u), bc=bc).cpu().numpy()
        assert np.abs(got - ref).max() <= 1e-11 * np.abs(ref).max(), bc
        dref = o.diag(bc)
        dgot = g.diag(bc=bc).cpu().numpy()
        assert np.abs(dgot - dref).max() <= 1e-11 * np.abs(dref).max(), bc
    fref = o.load_vector(1)
    fgot = g.load_vector(1).cpu().numpy()
    assert np.abs(fgot - fref).max() <= 1e-11 * max(np.abs(fref).max(), 1e-300)


@pytest.mark.parametrize("p,quad", [(2, 0), (4, 1), (7, 0), (16, 1)])
def test_smoothers_and_lambda_2d(S, orc, p, quad):
    d = prob2(3, 2, p, quad, **KINDS[0])
    g, o = levels(S, orc, d)
    lo_, la_ = o.lambda_max(10, 12345), o.lambda_arnoldi(10, 12345)
    assert abs(g.lambda_max(10, 12345) - lo_) <= 1e-10 * lo_
    assert abs(g.lambda_arnoldi(10, 12345) - la_) <= 1e-10 * la_
    rng = np.random.default_rng(p)
    b, x0 = rng.uniform(-1, 1, g.N), rng.uniform(-1, 1, g.N)
    xo = o.cheb(b, x0, 4, 0.1 * lo_, 1.1 * lo_)
    xg = to_gpu(x0)
    g.cheb(to_gpu(b), xg, 4, 0.1 * lo_, 1.1 * lo_)
    assert np.abs(xg.cpu().numpy() - xo).max() <= 1e-11 * np.abs(xo).max()
    xo = o.jacobi(b, x0, 3, 2.0 / 3.0)
    xg = to_gpu(x0)
    g.jacobi(to_gpu(b), xg, 3, 2.0 / 3.0)
    assert np.abs(xg.cpu().numpy() - xo).max() <= 1e-11 * np.abs(xo).max()


@pytest.mark.parametrize("pc,pf,cshape,fshape", [(1, 2, (3, 2), (3, 2)), (4, 8, (2, 2), (2, 2)), (8, 16, (1, 2), (1, 2)),
                                                 (1, 1, (2, 3), (4, 6)), (3, 3, (2, 1), (4, 2)), (16, 16, (1, 1), (2, 2))])
def test_transfer_parity_2d(S, orc, pc, pf, cshape, fshape):
    dc, df = prob2(*cshape, pc, **KINDS[0]), prob2(*fshape, pf, **KINDS[0])
    gc, oc = levels(S, orc, dc)
    gf, of = levels(S, orc, df)
    rng = np.random.default_rng(pc + pf)
    uc, rf = rng.uniform(-1, 1, gc.N), rng.uniform(-1, 1, gf.N)
    uf_ref, rc_ref = orc.prolong2(oc, of, uc), orc.restrict2(oc, of, rf)
    uf = S.prolong(gc, gf, to_gpu(uc)).cpu().numpy()
    rc = S.restrict(gc, gf, to_gpu(rf)).cpu().numpy()
    np.testing.assert_allclose(uf, uf_ref, rtol=0, atol=1e-14 * max(1.0, np.abs(uf_ref).max()))
    np.testing.assert_allclose(rc, rc_ref, rtol=0, atol=1e-13 * max(1.0, np.abs(rc_ref).max()))


def orc_hier2(orc, d, mg):
    orc.set_quadrature(d["quadrature"])
    try:
        return orc.Hier2(d["nex"], d["ney"], d["p"], d.get("warp", 0), d.get("amp", 0.0), d.get("coeff", 0),
                         d.get("c0", 1.0), d.get("c1", 0.0), nu_pre=mg.nu_pre, nu_post=mg.nu_post,
                         degree=mg.cheb_degree, lo_frac=mg.eig_lo_frac, hi_frac=mg.eig_hi_frac,
                         power_iters=mg.power_iters, seed=mg.power_seed, coarse_rtol=mg.coarse_rtol,
                         coarse_maxit=mg.coarse_max_iter, smoother=mg.smoother, omega=mg.jacobi_omega,
                         lambda_method=mg.lambda_method, h_levels=mg.h_levels, coarsen=mg.coarsen)
    finally:
        orc.set_quadrature(0)


@pytest.mark.parametrize("p,quad,which", [(4, 0, "baseline"), (8, 1, "paper"), (3, 0, "paper_h"), (4, 1, "paper_h")])
def test_hierarchy_parity_2d(S, orc, p, quad, which):
    import torch
    d = prob2(8, 8, p, quad, **KINDS[0])
    mg = {"baseline": S.MgParams(h_levels=1), "paper": S.MgParams.paper("cheb", 2),
          "paper_h": S.MgParams.paper_h("jacobi", 2)}[which]
    H = S.Hierarchy(S.Problem.from_dict(d), mg)
    O = orc_hier2(orc, d, mg)
    assert H.nlevels == O.nlevels
    assert [lv.N for lv in H.levels] == [lv.N for lv in O.levels]
    for l in range(H.nlevels - 1):
        assert abs(H.lam(l) - O.lam(l)) <= 1e-10 * O.lam(l), l
    b = O.levels[0].load_vector(1)
    xo = O.vcycle(b)
    xg = H.vcycle(to_gpu(b))
    torch.cuda.synchronize()
    np.testing.assert_allclose(xg.cpu().numpy(), xo, rtol=0, atol=1e-8 * np.abs(xo).max())
    for mode in (0, 1):
        ro = O.solve(b, mode=mode, rtol=1e-8, maxit=200)
        _, rg = H.solve(to_gpu(b), mode=mode, rtol=1e-8, max_iter=200)
        assert rg["converged"] == ro["converged"]
        assert abs(rg["iterations"] - ro["iterations"]) <= 1, (mode, rg["iterations"], ro["iterations"])
        assert rg["r_norm"] <= 1e-8 * rg["r0_norm"]


@pytest.mark.parametrize("p", [2, 4])
def test_tab_box_gpu(S, orc, p):
    """tab:box (2d-const 32x32) with Gauss quadrature and the paper's smoothers: GPU
    iteration counts of the h- and p-multigrid columns +-1 of the oracle's."""
    d = prob2(32, 32, p, 1)
    ours, ref = [], []
    for params in (S.MgParams.paper_h, S.MgParams.paper):
        for mode in (0, 1):
            for sm in ("jacobi", "cheb"):
                mg = params(sm, 2)
                H = S.Hierarchy(S.Problem.from_dict(d), mg)
                O = orc_hier2(orc, d, mg)
                b = O.levels[0].load_vector(1)
                _, rg = H.solve(to_gpu(b), mode=mode, rtol=1e-8, max_iter=300)
                ro = O.solve(b, mode=mode, rtol=1e-8, maxit=300)
                assert rg["converged"] and ro["converged"]
                ours.append(rg["iterations"])
                ref.append(ro["iterations"])
    assert np.all(np.abs(np.array(ours) - np.array(ref)) <= 1), (ours, ref)


def test_2d_rejections(S):
    with pytest.raises(S.SfmgError):
        S.Level(S.Problem.from_dict(dict(nex=2, ney=2, nez=3, p=2, dim=2)))
    g = S.Level(S.Problem.from_dict(prob2(2, 2, 2)))
    for f in (g.export_l2g, g.export_mask, g.export_colors, g.export_geometry):
        with pytest.raises(S.SfmgError):
            f()
