"""GPU <-> oracle parity of the NEXT-4 row: high-order h-multigrid -- the
h-transfer at one order p = 1..16 between nested meshes (eq. (7) across meshes, R25) and the hierarchy
of three meshes ne, ne/2, ne/4 at the fine order, with its general coarse CG (R13),
through the C ABI.

Bars as NEXT-1 (test_gpu_next1.py): transfers 1e-14 relative; lambda 1e-10 relative; V-cycle 1e-8
(coarse-CG tolerance); solver iteration counts +-1.  The tab:3d-box h columns (golden from the paper,
P:1266-1275) are reproduced on the GPU with Gauss quadrature to +-1 of the oracle's counts.
"""
import os

import numpy as np
import pytest

from paper_1402_5938_b200 import inputs

pytestmark = pytest.mark.gpu
GOLDEN_H = os.path.join(os.path.dirname(__file__), "golden", "tab_3d_box_h.txt")
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


@pytest.mark.parametrize("shape_c,p", [((1, 1, 1), 2), ((2, 1, 1), 3), ((1, 2, 1), 4), ((1, 1, 2), 5),
                                       ((1, 1, 1), 8), ((1, 1, 1), 11), ((1, 1, 1), 16)])
def test_h_transfer_any_order_parity(S, orc, shape_c, p):
    dc = inputs.problem(shape_c[0], p, ney=shape_c[1], nez=shape_c[2], **WARP)
    df = inputs.problem(2 * shape_c[0], p, ney=2 * shape_c[1], nez=2 * shape_c[2], **WARP)
    gc, gf = S.Level(S.Problem.from_dict(dc)), S.Level(S.Problem.from_dict(df))
    oc = orc.Level(dc["nex"], dc["ney"], dc["nez"], p, 1, 0.1, 1, 1.0, 3.0, eager=False)
    of = orc.Level(df["nex"], df["ney"], df["nez"], p, 1, 0.1, 1, 1.0, 3.0, eager=False)
    rng = np.random.default_rng(p)
    uc = rng.uniform(-1, 1, gc.N)
    rf = rng.uniform(-1, 1, gf.N)
    uf_ref = orc.prolong(oc, of, uc)
    rc_ref = orc.restrict(oc, of, rf)
    uf = S.prolong(gc, gf, to_gpu(uc)).cpu().numpy()
    rc = S.restrict(gc, gf, to_gpu(rf)).cpu().numpy()
    np.testing.assert_allclose(uf, uf_ref, rtol=0, atol=1e-14 * max(1.0, np.abs(uf_ref).max()))
    np.testing.assert_allclose(rc, rc_ref, rtol=0, atol=1e-13 * max(1.0, np.abs(rc_ref).max()))
    # adjointness on the device results
    assert abs(uf @ rf - uc @ rc) <= 1e-12 * max(1.0, abs(uf @ rf))


def orc_hier(orc, d, mg):
    return orc.Hier(d["nex"], d["ney"], d["nez"], d["p"], d["warp"], d["amp"], d["coeff"], d["c0"], d["c1"],
                    nu_pre=mg.nu_pre, nu_post=mg.nu_post, degree=mg.cheb_degree, lo_frac=mg.eig_lo_frac,
                    hi_frac=mg.eig_hi_frac, power_iters=mg.power_iters, seed=mg.power_seed,
                    coarse_rtol=mg.coarse_rtol, coarse_maxit=mg.coarse_max_iter, smoother=mg.smoother,
                    omega=mg.jacobi_omega, lambda_method=mg.lambda_method, h_levels=mg.h_levels,
                    coarsen=mg.coarsen)


@pytest.mark.parametrize("p,smoother", [(2, "cheb"), (3, "jacobi"), (5, "cheb"), (4, "jacobi")])
def test_h_multigrid_hierarchy_parity(S, orc, p, smoother):
    import torch
    d = inputs.problem(4, p, **WARP)
    mg = S.MgParams.paper_h(smoother, h_levels=2)
    H = S.Hierarchy(S.Problem.from_dict(d), mg)
    O = orc_hier(orc, d, mg)
    assert H.nlevels == O.nlevels == 3
    assert [lv.N for lv in H.levels] == [lv.N for lv in O.levels] == [(4 * p + 1) ** 3, (2 * p + 1) ** 3,
                                                                       (p + 1) ** 3]
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
        assert rg["fine_applies"] == rg["iterations"] * (7 + 1)
        assert rg["r_norm"] <= 1e-8 * rg["r0_norm"]


def test_h_multigrid_invalid(S):
    mg = S.MgParams.paper_h("cheb", h_levels=2)
    with pytest.raises(S.SfmgError) as ex:   # 6 -> 3 -> cannot halve
        S.Hierarchy(S.Problem.from_dict(inputs.problem(6, 3)), mg)
    assert ex.value.status == "SFMG_E_PCOARSEN"
    mg.h_levels = 0
    with pytest.raises(S.SfmgError):
        S.Hierarchy(S.Problem.from_dict(inputs.problem(4, 3)), mg)


def paper_h_rows():
    rows = {}
    for line in open(GOLDEN_H):
        if line.strip() and not line.startswith("#"):
            v = [int(t) for t in line.split()]
            rows[v[0]] = v[1:]
    return rows


@pytest.mark.parametrize("p", [1, 2, 3])
def test_tab_3d_box_h_columns_gpu(S, orc, p):
    """tab:3d-box h columns (3d-const, 8^3 -> 4^3 -> 2^3 at order p, Gauss quadrature, paper smoothers):
    GPU counts +-1 of the oracle's, and +-1 of the printed ones."""
    d = dict(inputs.problem(8, p), quadrature=1)
    ours, ref = [], []
    orc.set_quadrature(1)
    try:
        for mode in (0, 1):
            for sm in ("jacobi", "cheb"):
                mg = S.MgParams.paper_h(sm, h_levels=2)
                H = S.Hierarchy(S.Problem.from_dict(d), mg)
                O = orc_hier(orc, d, mg)
                b = O.levels[0].load_vector(1)
                _, rg = H.solve(to_gpu(b), mode=mode, rtol=1e-8, max_iter=300)
                ro = O.solve(b, mode=mode, rtol=1e-8, maxit=300)
                assert rg["converged"] and ro["converged"]
                ours.append(rg["iterations"])
                ref.append(ro["iterations"])
    finally:
        orc.set_quadrature(0)
    assert np.all(np.abs(np.array(ours) - np.array(ref)) <= 1), (ours, ref)
    assert np.all(np.abs(np.array(ours) - np.array(paper_h_rows()[p])) <= 1), (ours, paper_h_rows()[p])
