"""The fused Chebyshev step / apply (k_apply_v4<.., FU>, DESIGN.md section 6 "Fused step") against the
oracle (run with -m gpu).

The library takes the fused path for vectors of more than 2^24 dofs (config 4); SFMG_FUSED=1 forces it
wherever the kernel applies (3 <= p <= 8, bc 0, >= 3 element layers, whole groups per layer), so a
subprocess runs small meshes through it -- several element layers, several grid rounds per layer or
several layers per round, odd and even Chebyshev degrees (in-place last step), Jacobi, and the
standalone apply -- and compares every output element with the oracle at the section-2 bars.
The full-size check (config 4 through the default path) is in test_gpu_fullsize.py.
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
cases = %(cases)s
for (p, nex, ney, nez) in cases:
    d = inputs.problem(nex, p, ney=ney, nez=nez, warp=1, amp=0.1, coeff=1, c0=1.0, c1=3.0)
    g = sfmg.Level(sfmg.Problem.from_dict(d))
    o = oracle.Level(nex, ney, nez, p, 1, 0.1, 1, 1.0, 3.0, eager=True, tier=3, geom_tier=3)
    u = inputs.uniform_pm1(5, o.N)
    ug = torch.from_numpy(u).cuda()
    vo = o.apply(u, 0, 3)
    errs = []
    for rep in range(2):   # twice: the ring must be left clean
        v = torch.full((o.N,), 7.0, dtype=torch.float64, device="cuda")
        g.apply(ug, v)
        errs.append(float(np.abs(v.cpu().numpy() - vo).max() / np.abs(vo).max()))
    lam = o.lambda_max(10, 12345)
    lam_g = g.lambda_max(10, 12345)
    errs.append(abs(lam_g - lam) / lam)
    b = inputs.uniform_pm1(6, o.N)
    bg = torch.from_numpy(b).cuda()
    for K in (1, 2, 3, 4, 5):
        xo = o.cheb(b, u, K, 0.1 * lam, 1.1 * lam)
        xg = g.cheb(bg, ug.clone(), K, 0.1 * lam, 1.1 * lam).cpu().numpy()
        errs.append(float(np.abs(xg - xo).max() / np.abs(xo).max()))
    xo = o.jacobi(b, u, 3, 2.0 / 3.0)
    xg = g.jacobi(bg, ug.clone(), 3, 2.0 / 3.0).cpu().numpy()
    errs.append(float(np.abs(xg - xo).max() / np.abs(xo).max()))
    out["%%d_%%dx%%dx%%d" %% (p, nex, ney, nez)] = errs
print(json.dumps(out))
"""

# (p, nex, ney, nez): nex ney is a multiple of the elements per block of every order (12, 6, 3, 2, 1, 1)
SMALL = [(3, 4, 3, 3), (4, 6, 2, 4), (5, 3, 2, 5), (6, 2, 2, 3), (7, 2, 1, 4), (8, 2, 2, 5), (8, 3, 1, 3)]
# more groups per layer than resident blocks (several grid rounds inside one element layer)
WIDE = [(4, 72, 60, 3), (8, 28, 24, 4)]


# SFMG_FUSED_RING_EXTRA: ring planes beyond the default 3 p + 1 (clamped to [2 p + 1, Mz]); -100 gives
# the minimum 2 p + 1, where the pieces cannot lag their layer (shift 0)
@pytest.mark.parametrize("cases,extra", [(SMALL, "0"), (SMALL, "3"), (SMALL, "-100"), (WIDE, "0"), (WIDE, "-100")],
                         ids=["small", "small_ring_plus3", "small_min_ring", "wide_layers", "wide_min_ring"])
def test_fused_step_matches_oracle(cases, extra):
    env = dict(os.environ, SFMG_FUSED="1", SFMG_FUSED_RING_EXTRA=extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT % {"root": ROOT, "cases": repr(cases)}], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert len(res) == len(cases)
    for key, errs in res.items():
        for e in errs:
            assert e <= 1e-11, (key, errs)
