"""Developer probe: the 2-D p = 16 h-multigrid PCG solve of the bench (NEXT-2), for an ncu launch list."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1402_5938_b200 import sfmg

prob = sfmg.Problem.from_dict(dict(nex=32, ney=32, nez=1, p=16, dim=2, quadrature=1))
H = sfmg.Hierarchy(prob, sfmg.MgParams.paper_h("cheb", 2))
b = H.levels[0].load_vector(1)
torch.cuda.synchronize()
t0 = time.perf_counter()
x, rep = H.solve(b, mode=1, rtol=1e-8)
torch.cuda.synchronize()
print("solve_ms", (time.perf_counter() - t0) * 1e3, {k: v for k, v in rep.items() if k != "history"})
