"""GPU <-> oracle parity at BASELINE.json's full sizes, through the C ABI, in the launch
configuration bench.py times (the same Level / apply / cheb calls).

At full size the oracle computes sampled rows one by one (`orc_apply_rows`: the <= 8 elements touching
each row, O2 direct quadrature, geometry recomputed per element), plus properties that hold at any
size.  Bars as in test_gpu_parity.py; the normaliser is ||A u||_inf (R19, stricter than ||A|| ||u||).
"""
import json
import os

import numpy as np
import pytest

from paper_1402_5938_b200 import inputs

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def S():
    import torch
    assert torch.cuda.is_available()
    from paper_1402_5938_b200 import sfmg
    return sfmg


def sample_rows(d, count, seed):
    """Seeded sample: random dofs + the lattice corners/edges/faces of an interior element + boundary."""
    N = inputs.ndofs(d)
    p, Mx, My = d["p"], d["nex"] * d["p"] + 1, d["ney"] * d["p"] + 1
    rng = np.random.default_rng(seed)
    rows = list(rng.integers(0, N, count))
    ex = ey = ez = d["nex"] // 2
    for (a, b, c) in [(0, 0, 0), (p, 0, 0), (0, p, p), (1, 0, 0), (p // 2, p // 2, 0), (p // 2, p // 2, p // 2)]:
        rows.append((ex * p + a) + Mx * ((ey * p + b) + My * (ez * p + c)))
    rows += [0, N - 1, Mx + 1]
    return np.unique(np.array(rows, dtype=np.int64))


def orc_lazy(orc, d):
    return orc.Level(d["nex"], d["ney"], d["nez"], d["p"], d["warp"], d["amp"], d["coeff"], d["c0"], d["c1"],
                     eager=False, geom_tier=2, tier=2)


def check_apply_rows(S, orc, d, seed, count):
    import torch
    lv = S.Level(S.Problem.from_dict(d))
    u = inputs.uniform_pm1(seed, lv.N)
    v = lv.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    o = orc_lazy(orc, d)
    rows = sample_rows(d, count, seed + 100)
    ref = o.apply_rows(u, rows, bc=0, tier=2)
    scale = np.abs(v).max()
    err = np.abs(v[rows] - ref).max() / scale
    assert err <= 1e-11, err
    # boundary pass-through is exact everywhere; apply is deterministic up to atomics ordering
    return lv, u, v


def test_config2_apply_sampled(S, orc):
    check_apply_rows(S, orc, inputs.CONFIG2, inputs.SEEDS[2], 300)


@pytest.mark.parametrize("p", [1, 2, 4, 8, 16])
def test_config3_apply_sampled(S, orc, p):
    check_apply_rows(S, orc, inputs.CONFIG3[p], inputs.SEEDS[3], 60 if p < 16 else 20)


def test_config4_apply_sampled(S, orc):
    import torch
    lv, u, v = check_apply_rows(S, orc, inputs.CONFIG4, inputs.SEEDS[4], 120)
    # any-size property: u^T A_D w = w^T A_D u (symmetry) on the full 135 M-dof operator
    w = torch.from_numpy(inputs.uniform_pm1(77, lv.N)).cuda()
    ut = torch.from_numpy(u).cuda()
    Aw = lv.apply(w)
    Au = torch.from_numpy(v).cuda()
    lhs, rhs = float(torch.dot(ut, Aw)), float(torch.dot(w, Au))
    assert abs(lhs - rhs) <= 1e-10 * abs(lhs)


def orc_full(orc, d):
    """O3 sum-factorised apply with the factorised geometry recomputed per element (no stored factors:
    config 4's 9 GB of G never sits in host memory); O3 = O2 = O1 and factorised = dense geometry are
    pinned by tests/test_oracle_operator.py."""
    return orc.Level(d["nex"], d["ney"], d["nez"], d["p"], d["warp"], d["amp"], d["coeff"], d["c0"], d["c1"],
                     eager=False, geom_tier=3, tier=3)


def check_apply_full(S, orc, d, seed):
    """Every row of A_D u at full size, GPU (the bench's launch path) against the oracle's O3 tier."""
    import torch
    lv = S.Level(S.Problem.from_dict(d))
    u = inputs.uniform_pm1(seed, lv.N)
    v = lv.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    del lv
    torch.cuda.empty_cache()
    ref = orc_full(orc, d).apply(u, 0, 3)
    err = np.abs(v - ref).max() / np.abs(ref).max()
    assert err <= 1e-11, err
    return err


def test_config2_apply_full(S, orc):
    check_apply_full(S, orc, inputs.CONFIG2, inputs.SEEDS[2])


@pytest.mark.parametrize("p", [1, 2, 4, 8, 16])
def test_config3_apply_full(S, orc, p):
    check_apply_full(S, orc, inputs.CONFIG3[p], inputs.SEEDS[3])


def test_config4_apply_full(S, orc):
    """135 M dofs: the whole output vector (~35 s of oracle time on 16 host cores)."""
    check_apply_full(S, orc, inputs.CONFIG4, inputs.SEEDS[4])


def test_config2_chebyshev_full(S, orc):
    """The bench's Chebyshev workload at full size: lambda_max (10 power iterations) and one degree-4
    application (b = 0, x0 = u) against the oracle's O3 run (O3 pinned to O1/O2 by the CPU tests)."""
    import torch
    d = inputs.CONFIG2
    lv = S.Level(S.Problem.from_dict(d))
    o = orc.Level(d["nex"], d["ney"], d["nez"], d["p"], d["warp"], d["amp"], d["coeff"], d["c0"], d["c1"],
                  eager=True, geom_tier=3, tier=3)
    lam_o = o.lambda_max(10, inputs.POWER_SEED)
    lam_g = lv.lambda_max(10, inputs.POWER_SEED)
    assert abs(lam_g - lam_o) <= 1e-12 * lam_o
    u = inputs.uniform_pm1(inputs.SEEDS[2], lv.N)
    xo = o.cheb(np.zeros(lv.N), u, 4, 0.1 * lam_o, 1.1 * lam_o)
    xg = torch.from_numpy(u).cuda()
    lv.cheb(torch.zeros_like(xg), xg, 4, 0.1 * lam_o, 1.1 * lam_o)
    err = np.abs(xg.cpu().numpy() - xo).max() / np.abs(xo).max()
    assert err <= 1e-11, err
    dg = lv.diag().cpu().numpy()
    do = o.diag(0)
    assert np.abs(dg - do).max() <= 1e-11 * np.abs(do).max()


def test_config5_solves_against_golden(S):
    """Config 5 p-MG: PCG and MG-solver iteration counts +-1 of the oracle's (tests/golden/
    config5_oracle.json, written by tools/make_golden.py from oracle/ only), residual <= 1e-8."""
    g = json.load(open(os.path.join(GOLDEN, "config5_oracle.json")))
    H = S.Hierarchy(S.Problem.from_dict(inputs.CONFIG5), S.MgParams())
    assert H.nlevels == g["levels"] == 5
    for l, lam in enumerate(g["lambda"]):
        assert abs(H.lam(l) - lam) <= 1e-11 * lam
    b = H.levels[0].load_vector(1)
    assert abs(float(b.norm()) - g["b_norm"]) <= 1e-12 * g["b_norm"]
    for mode, name in ((1, "pcg"), (0, "mg_solver")):
        x, rep = H.solve(b, mode=mode, rtol=1e-8, max_iter=200)
        ref = g[name]
        # the oracle's MG-as-solver run with these settings diverges (stops at ||r|| > 10 ||r0||,
        # S:483); the GPU must reproduce the same outcome and iteration count
        assert rep["converged"] == ref["converged"], name
        assert abs(rep["iterations"] - ref["iterations"]) <= 1, (name, rep["iterations"], ref["iterations"])
        hg, ho = np.array(rep["history"]), np.array(ref["history"])
        k = min(len(hg), len(ho))
        r0 = ref["r0_norm"]
        if mode == 1:
            # every PCG residual norm.  Both sides run the same algorithm; their V-cycles differ by the
            # coarse CG's stopping tolerance (1e-10 relative to its right-hand side, R13), a perturbation
            # that does not shrink with the residual: measured |dh| <= 1.4e-10 = 3e-9 ||r0|| on B200.
            # Bar: 1e-6 relative, or below the solve's own stopping tolerance 1e-8 ||r0||,
            # under which a difference cannot move the iteration count by more than the allowed +-1.
            np.testing.assert_allclose(hg[:k], ho[:k], rtol=1e-6, atol=1e-8 * r0)
        else:
            # MG as a solver diverges on both sides (test_config5_mg_solver_divergence); the first 4
            # cycles, before the growth dominates, agree to the same bar
            np.testing.assert_allclose(hg[:4], ho[:4], rtol=1e-6, atol=1e-8 * r0)
        if ref["converged"]:
            assert rep["r_norm"] <= 1e-8 * rep["r0_norm"]
            xs = x.cpu().numpy()[::99991]
            np.testing.assert_allclose(xs, ref["x_sample"], rtol=0, atol=1e-6 * np.abs(ref["x_sample"]).max())


def test_config5_mg_solver_divergence(S):
    """Why MG-as-solver diverges at config 5 while MG-PCG converges: the 10-step power estimate
    (R9) under-covers lambda_max(D^-1 A_D) on the high-contrast (mu = e^{3S}) levels, so the
    top of the spectrum lies above the Chebyshev interval [0.1, 1.1] lambda_hat, where the smoother
    amplifies instead of damping (|T_K| > 1 outside the interval); CG is robust to a few such modes.
    Evidence: a 200-step estimate exceeds 1.1 lambda_hat on at least one level, and with the 200-step
    estimates (power_iters = 200) the same V(2,2) cycle converges as a solver."""
    H = S.Hierarchy(S.Problem.from_dict(inputs.CONFIG5), S.MgParams())
    ratios = []
    for l in range(H.nlevels - 1):
        lam10 = H.lam(l)
        lam200 = H.levels[l].lambda_max(200, inputs.POWER_SEED)
        assert lam200 >= lam10 * (1 - 1e-12)
        ratios.append(lam200 / lam10)
    print("lambda_200 / lambda_10 per level:", ["%.4f" % r for r in ratios])
    assert max(ratios) > 1.1, ratios
    H2 = S.Hierarchy(S.Problem.from_dict(inputs.CONFIG5), S.MgParams(power_iters=200))
    b = H2.levels[0].load_vector(1)
    _, rep = H2.solve(b, mode=0, rtol=1e-8, max_iter=200)
    assert rep["converged"], rep["iterations"]
    _, rep1 = H2.solve(b, mode=1, rtol=1e-8, max_iter=200)
    assert rep1["converged"] and rep1["iterations"] <= rep["iterations"]
