"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck): the persistent apply at
p = 2, 4, 8, 16 (both launch schedules via SFMG_EARLY_MAXN, set by the caller), a degree-4 Chebyshev
application, power iteration, and a short p-MG hierarchy V-cycle + PCG solve.  Usage:
    compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1402_5938_b200 import inputs, sfmg  # noqa: E402

W = dict(warp=1, amp=0.1, coeff=1, c0=1.0, c1=3.0)
for p in (2, 4, 8, 16):
    d = inputs.problem(2, p, ney=2, nez=1, **W)
    lv = sfmg.Level(sfmg.Problem.from_dict(d))
    u = torch.from_numpy(inputs.uniform_pm1(1, lv.N)).cuda()
    v = lv.apply(u)
    lam = lv.lambda_max(10, 12345)
    x = u.clone()
    lv.cheb(torch.zeros_like(u), x, 4, 0.1 * lam, 1.1 * lam)
    torch.cuda.synchronize()
    print("p=%d apply/cheb ok |v|=%.6e |x|=%.6e" % (p, float(v.norm()), float(x.norm())), flush=True)
H = sfmg.Hierarchy(sfmg.Problem.from_dict(inputs.problem(2, 8, **W)), sfmg.MgParams())
b = H.levels[0].load_vector(1)
for _ in range(3):
    H.vcycle(b)
x, rep = H.solve(b, mode=1, rtol=1e-8, max_iter=50)
torch.cuda.synchronize()
print("p-MG PCG iterations", rep["iterations"], "converged", rep["converged"], flush=True)
