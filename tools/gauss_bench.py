"""Developer timing of the Gauss-Legendre (NEXT-3) apply on the config-3 meshes (p = 4, 8, 16)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1402_5938_b200 import inputs, sfmg
from tools.quick_bench import timeit, HBM

flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
for p in (4, 8, 16):
    d = dict(inputs.CONFIG3[p], quadrature=1)
    lv = sfmg.Level(sfmg.Problem.from_dict(d))
    u = torch.from_numpy(inputs.uniform_pm1(3, lv.N)).cuda()
    v = torch.empty_like(u)
    t = timeit(lambda: lv.apply(u, v), flush=flush)
    byts = 48 * lv.E * lv.n ** 3 + 16 * lv.N
    print("gauss p=%2d apply %8.2f us  frac %.3f" % (p, t * 1e6, byts / t / HBM))
