"""Developer probe: a few Chebyshev applications (and applies) on one BASELINE config, for ncu
captures of the fused / unfused step kernels.  python tools/fused_probe.py [config] [degree] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1402_5938_b200 import inputs, sfmg

cfg = sys.argv[1] if len(sys.argv) > 1 else "4"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 2
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
d = {"2": inputs.CONFIG2, "4": inputs.CONFIG4}[cfg] if cfg in ("2", "4") else inputs.CONFIG3[int(cfg[2:])]
lv = sfmg.Level(sfmg.Problem.from_dict(d))
u = torch.from_numpy(inputs.uniform_pm1(2, lv.N)).cuda()
b = torch.zeros_like(u)
v = torch.empty_like(u)
x = u.clone()
for _ in range(reps):
    lv.cheb(b, x, K, 0.1, 1.1)
    lv.apply(u, v)
torch.cuda.synchronize()
print("ok", lv.N)
