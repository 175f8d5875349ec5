"""Developer probe: one pass over the kernels outside the collocated 3-D apply, for ncu captures
(profiles/r02_*): the Gauss-quadrature apply (NEXT-3) on the config-3 meshes, the 2-D apply and a 2-D
p-MG V-cycle (NEXT-2), a high-order h-MG V-cycle (NEXT-4), and the config-5 p-MG V-cycle.
python tools/kernel_zoo.py [gauss] [2d] [hmg] [vcycle]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1402_5938_b200 import inputs, sfmg

which = sys.argv[1:] or ["gauss", "2d", "hmg", "vcycle"]
reps = 2
if "gauss" in which:
    for p in (4, 8, 16):
        d = dict(inputs.CONFIG3[p], quadrature=1)
        lv = sfmg.Level(sfmg.Problem.from_dict(d))
        u = torch.from_numpy(inputs.uniform_pm1(3, lv.N)).cuda()
        v = torch.empty_like(u)
        for _ in range(reps):
            lv.apply(u, v)
        torch.cuda.synchronize()
        del lv
if "2d" in which:
    for p, ne in ((4, 256), (16, 64)):
        d = inputs.problem(ne, p, ney=ne, nez=1, warp=1, amp=0.1, coeff=1, c0=1.0, c1=3.0)
        pr = sfmg.Problem.from_dict(dict(d, dim=2))
        lv = sfmg.Level(pr)
        u = torch.from_numpy(inputs.uniform_pm1(3, lv.N)).cuda()
        v = torch.empty_like(u)
        for _ in range(reps):
            lv.apply(u, v)
        H = sfmg.Hierarchy(pr, sfmg.MgParams())
        b = H.levels[0].load_vector(1)
        x = torch.empty_like(b)
        for _ in range(reps):
            H.vcycle(b, x)
        torch.cuda.synchronize()
        del H, lv
if "hmg" in which:
    d = inputs.problem(8, 4, ney=8, nez=8, warp=1, amp=0.1, coeff=1, c0=1.0, c1=3.0)
    H = sfmg.Hierarchy(sfmg.Problem.from_dict(d), sfmg.MgParams.paper_h())
    b = H.levels[0].load_vector(1)
    x = torch.empty_like(b)
    for _ in range(reps):
        H.vcycle(b, x)
    torch.cuda.synchronize()
    del H
if "vcycle" in which:
    H = sfmg.Hierarchy(sfmg.Problem.from_dict(inputs.CONFIG5), sfmg.MgParams())
    b = H.levels[0].load_vector(1)
    x = torch.empty_like(b)
    for _ in range(reps + 1):
        H.vcycle(b, x)
    torch.cuda.synchronize()
print("ok")
