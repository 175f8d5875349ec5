"""Developer probe: cost of writes (torch zero_ of a 17 MB vector) and of the config-2 apply after
different L2 flush protocols.  Usage: python tools/flush_probe.py"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1402_5938_b200 import inputs, sfmg  # noqa: E402

A = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
B = torch.ones(512 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
flushes = {
    "none": lambda k: None,
    "write": lambda k: A.fill_(float(k)),
    "write+read_same": lambda k: (A.fill_(float(k)), A.sum()),
    "write+read_other": lambda k: (A.fill_(float(k)), B.sum()),
    "read_other": lambda k: B.sum(),
}
lv = sfmg.Level(sfmg.Problem.from_dict(inputs.CONFIG2))
u = torch.from_numpy(inputs.uniform_pm1(1, lv.N)).cuda()
v = torch.empty_like(u)
ops = {"zero_": lambda: v.zero_(), "apply": lambda: lv.apply(u, v),
       "cheb4": lambda: lv.cheb(torch.zeros_like(u), v, 4, 1.0, 11.0)}
for fname, f in flushes.items():
    for oname, op in ops.items():
        ts = []
        for k in range(25):
            f(k)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            op()
            b.record()
            torch.cuda.synchronize()
            if k >= 5:
                ts.append(a.elapsed_time(b) * 1e3)
        ts.sort()
        print("%-18s %-6s median %7.2f us  min %7.2f" % (fname, oname, ts[len(ts) // 2], ts[0]))
