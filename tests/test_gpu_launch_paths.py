"""Both launch schedules of the apply / Chebyshev kernels against the oracle (run with -m gpu).

For vectors of <= 2^24 dofs the v init, the Chebyshev update and the persistent apply trigger their
programmatic dependents early ("Launch overlap"); larger vectors take the
completion-ordered path.  The in-process GPU tests only reach the early path (their meshes are small),
so this test re-runs an apply and a Chebyshev application in a subprocess with SFMG_EARLY_MAXN=0, which
forces the completion-ordered path, and checks both against the oracle with the section-2 bars.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, %(root)r)
import torch
import oracle
from paper_1402_5938_b200 import inputs, sfmg
oracle.build()
out = {}
for p in (3, 4, 5, 8, 9, 12, 14, 16):
    d = inputs.problem(2, p, ney=2, nez=2, warp=1, amp=0.1, coeff=1, c0=1.0, c1=3.0)
    g = sfmg.Level(sfmg.Problem.from_dict(d))
    o = oracle.Level(d["nex"], d["ney"], d["nez"], p, 1, 0.1, 1, 1.0, 3.0, eager=True, tier=3, geom_tier=2)
    u = inputs.uniform_pm1(5, o.N)
    vo = o.apply(u, 0, 3)
    v = torch.empty(o.N, dtype=torch.float64, device="cuda")
    g.apply(torch.from_numpy(u).cuda(), v)
    ea = float(np.abs(v.cpu().numpy() - vo).max() / np.abs(vo).max())
    lam = o.lambda_max(10, 12345)
    b = inputs.uniform_pm1(6, o.N)
    xo = o.cheb(b, u, 4, 0.1 * lam, 1.1 * lam)
    xg = g.cheb(torch.from_numpy(b).cuda(), torch.from_numpy(u.copy()).cuda(), 4, 0.1 * lam, 1.1 * lam).cpu().numpy()
    ec = float(np.abs(xg - xo).max() / np.abs(xo).max())
    out[p] = [ea, ec]
print(json.dumps(out))
"""


@pytest.mark.parametrize("maxn,ksplit", [("0", "0"), (str(1 << 24), "0"), ("0", "1"), (str(1 << 24), "1"),
                                         ("0", "v6"), (str(1 << 24), "v6")],
                         ids=["completion_ordered", "early_triggers", "ksplit_completion_ordered", "ksplit_early",
                              "v6_completion_ordered", "v6_early"])
def test_launch_schedules_match_oracle(maxn, ksplit):
    """ksplit = 1 routes even p >= 12 to the k-split cluster kernel (k_apply_ks.cuh, opt-in); "v6" to the
    two-blocks-per-SM kernel (k_apply_v6.cuh, opt-in)."""
    env = dict(os.environ, SFMG_EARLY_MAXN=maxn, SFMG_KSPLIT="1" if ksplit == "1" else "0",
               SFMG_V6="1" if ksplit == "v6" else "0")
    r = subprocess.run([sys.executable, "-c", SCRIPT % {"root": ROOT}], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for p, (ea, ec) in res.items():
        assert ea <= 1e-11, (p, ea)   # ||A u||_inf normaliser (R19, stricter than ||A|| ||u||)
        assert ec <= 1e-11, (p, ec)   # R18


COLOR_SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, %(root)r)
import torch
import oracle
from paper_1402_5938_b200 import inputs, sfmg
oracle.build()
out = {}
for (p, nex, ney, nez) in ((8, 2, 2, 2), (8, 3, 2, 5), (7, 4, 3, 3), (8, 1, 1, 1)):
    d = inputs.problem(nex, p, ney=ney, nez=nez, warp=1, amp=0.1, coeff=1, c0=1.0, c1=3.0)
    g = sfmg.Level(sfmg.Problem.from_dict(d))
    o = oracle.Level(nex, ney, nez, p, 1, 0.1, 1, 1.0, 3.0, eager=True, tier=3, geom_tier=3)
    u = inputs.uniform_pm1(5, o.N)
    errs = []
    for bc in (0, 1):
        vo = o.apply(u, bc, 3)
        v = torch.empty(o.N, dtype=torch.float64, device="cuda")
        g.apply(torch.from_numpy(u).cuda(), v, bc=bc)
        errs.append(float(np.abs(v.cpu().numpy() - vo).max() / np.abs(vo).max()))
    lam = o.lambda_max(10, 12345)
    b = inputs.uniform_pm1(6, o.N)
    xo = o.cheb(b, u, 4, 0.1 * lam, 1.1 * lam)
    xg = g.cheb(torch.from_numpy(b).cuda(), torch.from_numpy(u.copy()).cuda(), 4, 0.1 * lam, 1.1 * lam).cpu().numpy()
    errs.append(float(np.abs(xg - xo).max() / np.abs(xo).max()))
    out["%%d_%%dx%%dx%%d" %% (p, nex, ney, nez)] = errs
print(json.dumps(out))
"""


def test_coloured_launches_match_oracle():
    """SFMG_COLOR=1: the eight-colour measurement variant of the p = 7, 8 apply (plain load-add-store
    scatter, one launch per colour; profiles/r02_experiments.md) on meshes with even and odd element counts."""
    env = dict(os.environ, SFMG_COLOR="1")
    r = subprocess.run([sys.executable, "-c", COLOR_SCRIPT % {"root": ROOT}], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert len(res) == 4
    for key, errs in res.items():
        for e in errs:
            assert e <= 1e-11, (key, errs)
