"""GPU <-> oracle parity of the NEXT-1 row: h-transfer at p = 1 (eq. (7) across nested
meshes, R25), damped Jacobi, lambda_max by Arnoldi (R26) and the
paper-style hierarchy p -> ... -> 1 -> ne/2 -> ne/4 with Jacobi(3,3) / Cheb(3,3) smoothing
(P:1015-1022), through the C ABI.

Bars: transfers and Jacobi iterates as the p-transfer / Chebyshev bars (test_gpu_parity.py); lambda
1e-10 relative (Arnoldi coefficients are reduced in a different order); V-cycle 1e-8 (coarse-CG
tolerance, R13); solver iteration counts +-1.
"""
import json
import os

import numpy as np
import pytest

from paper_1402_5938_b200 import inputs

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
WARP = dict(warp=1, amp=0.1, coeff=1, c0=1.0, c1=3.0)


@pytest.fixture(scope="module")
def S():
    import torch
    assert torch.cuda.is_available()
    from paper_1402_5938_b200 import sfmg
    return sfmg


def to_gpu(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def pair(S, orc, shape_c, **kw):
    dc = inputs.problem(shape_c[0], 1, ney=shape_c[1], nez=shape_c[2], **kw)
    df = inputs.problem(2 * shape_c[0], 1, ney=2 * shape_c[1], nez=2 * shape_c[2], **kw)
    gc, gf = S.Level(S.Problem.from_dict(dc)), S.Level(S.Problem.from_dict(df))
    oc = orc.Level(dc["nex"], dc["ney"], dc["nez"], 1, dc["warp"], dc["amp"], dc["coeff"], dc["c0"], dc["c1"])
    of = orc.Level(df["nex"], df["ney"], df["nez"], 1, df["warp"], df["amp"], df["coeff"], df["c0"], df["c1"])
    return gc, gf, oc, of


@pytest.mark.parametrize("shape_c", [(1, 1, 1), (2, 2, 2), (3, 1, 2), (4, 4, 4)])
def test_h_transfer_parity(S, orc, shape_c):
    gc, gf, oc, of = pair(S, orc, shape_c, **WARP)
    rng = np.random.default_rng(sum(shape_c))
    uc = rng.uniform(-1, 1, gc.N)
    rf = rng.uniform(-1, 1, gf.N)
    uf_ref = orc.prolong(oc, of, uc)
    rc_ref = orc.restrict(oc, of, rf)
    uf = S.prolong(gc, gf, to_gpu(uc)).cpu().numpy()
    rc = S.restrict(gc, gf, to_gpu(rf)).cpu().numpy()
    np.testing.assert_allclose(uf, uf_ref, rtol=0, atol=1e-15 * max(1.0, np.abs(uf_ref).max()))
    np.testing.assert_allclose(rc, rc_ref, rtol=0, atol=1e-14 * max(1.0, np.abs(rc_ref).max()))


def test_h_transfer_rejects_non_pairs(S):
    a = S.Level(S.Problem.from_dict(inputs.problem(2, 1)))
    b = S.Level(S.Problem.from_dict(inputs.problem(3, 1)))
    c = S.Level(S.Problem.from_dict(inputs.problem(4, 2)))
    import torch
    for lc, lf in ((a, b), (a, c)):
        with pytest.raises(S.SfmgError) as ex:
            S.prolong(lc, lf, torch.zeros(lc.N, dtype=torch.float64, device="cuda"))
        assert ex.value.status == "SFMG_E_PCOARSEN"


@pytest.mark.parametrize("shape,p", [((1, 2, 2), 2), ((3, 3, 3), 1), ((3, 3, 3), 2), ((2, 3, 2), 4), ((2, 2, 2), 8)])
def test_lambda_arnoldi_parity(S, orc, shape, p):
    d = inputs.problem(shape[0], p, ney=shape[1], nez=shape[2], **WARP)
    g = S.Level(S.Problem.from_dict(d))
    o = orc.Level(d["nex"], d["ney"], d["nez"], p, d["warp"], d["amp"], d["coeff"], d["c0"], d["c1"])
    lo = o.lambda_arnoldi(10, inputs.POWER_SEED)
    lg = g.lambda_arnoldi(10, inputs.POWER_SEED)
    assert abs(lg - lo) <= 1e-10 * lo, (lg, lo)


@pytest.mark.parametrize("p,steps", [(1, 1), (3, 3), (4, 2), (8, 3)])
def test_jacobi_parity(S, orc, p, steps):
    d = inputs.problem(2, p, ney=3, nez=2, **WARP)
    g = S.Level(S.Problem.from_dict(d))
    o = orc.Level(d["nex"], d["ney"], d["nez"], p, d["warp"], d["amp"], d["coeff"], d["c0"], d["c1"], tier=3,
                  geom_tier=3)
    rng = np.random.default_rng(p)
    b = rng.uniform(-1, 1, g.N)
    x0 = rng.uniform(-1, 1, g.N)
    xo = o.jacobi(b, x0, steps, 2.0 / 3.0)
    xg = to_gpu(x0)
    g.jacobi(to_gpu(b), xg, steps, 2.0 / 3.0)
    np.testing.assert_allclose(xg.cpu().numpy(), xo, rtol=0, atol=1e-11 * np.abs(xo).max())


def orc_hier(orc, d, mg):
    return orc.Hier(d["nex"], d["ney"], d["nez"], d["p"], d["warp"], d["amp"], d["coeff"], d["c0"], d["c1"],
                    nu_pre=mg.nu_pre, nu_post=mg.nu_post, degree=mg.cheb_degree, lo_frac=mg.eig_lo_frac,
                    hi_frac=mg.eig_hi_frac, power_iters=mg.power_iters, seed=mg.power_seed,
                    coarse_rtol=mg.coarse_rtol, coarse_maxit=mg.coarse_max_iter, smoother=mg.smoother,
                    omega=mg.jacobi_omega, lambda_method=mg.lambda_method, h_levels=mg.h_levels)


@pytest.mark.parametrize("smoother", ["jacobi", "cheb"])
def test_paper_hierarchy_parity(S, orc, smoother):
    import torch
    d = inputs.problem(4, 4, **WARP)
    mg = S.MgParams.paper(smoother, h_levels=2)
    H = S.Hierarchy(S.Problem.from_dict(d), mg)
    O = orc_hier(orc, d, mg)
    assert H.nlevels == O.nlevels == 5
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
        per_v = (3 + 1 + 3) if smoother == "jacobi" else (3 + 1 + 3)
        assert rg["fine_applies"] == rg["iterations"] * (per_v + 1)


def test_paper_hierarchy_invalid(S):
    with pytest.raises(S.SfmgError) as ex:
        S.Hierarchy(S.Problem.from_dict(inputs.problem(6, 2)), S.MgParams.paper("cheb", h_levels=2))
    assert ex.value.status == "SFMG_E_PCOARSEN"


def test_3dconst_paper_settings_against_golden(S):
    """tab:3d-box setting (3d-const, 8^3, p = 2..16, paper hierarchy and smoothers; NEXT-1): GPU iteration
    counts +-1 of the oracle's (tests/golden/next1_3dconst_oracle.json, written from oracle/ only)."""
    import torch
    g = json.load(open(os.path.join(GOLDEN, "next1_3dconst_oracle.json")))
    for p in (2, 4, 8, 16):
        d = inputs.problem(8, p)   # unit cube, mu = 1
        for name in ("jacobi33", "cheb33"):
            H = S.Hierarchy(S.Problem.from_dict(d), S.MgParams.paper("jacobi" if name == "jacobi33" else "cheb", 2))
            b = H.levels[0].load_vector(1)
            for mode, mname in ((0, "mg_solver"), (1, "pcg")):
                ref = g["runs"]["p%d_%s_%s" % (p, mname, name)]
                for l, lam in enumerate(ref["lambda"]):
                    assert abs(H.lam(l) - lam) <= 1e-9 * lam, (p, name, l)
                _, rep = H.solve(b, mode=mode, rtol=1e-8, max_iter=300)
                assert rep["converged"] == ref["converged"]
                assert abs(rep["iterations"] - ref["iterations"]) <= 1, (p, name, mname, rep["iterations"])
                assert rep["r_norm"] <= 1e-8 * rep["r0_norm"]
            del H
            torch.cuda.empty_cache()
