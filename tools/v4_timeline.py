"""Developer probe: per-block globaltimer marks of k_apply_v4 in the standalone apply path (library
variant built with -DSFMG_TIMELINE: python tools/build_variant.py tl -DSFMG_TIMELINE).  Usage: python tools/v4_timeline.py [config: 2 | 3:<p>]"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1402_5938_b200 import inputs, sfmg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
d = inputs.CONFIG2 if cfg == "2" else inputs.CONFIG3[int(cfg.split(":")[1])]
lib = ctypes.CDLL(os.path.join(ROOT, "paper_1402_5938_b200", "libsfmg.so"))
lv = sfmg.Level(sfmg.Problem.from_dict(d))
u = torch.from_numpy(inputs.uniform_pm1(1, lv.N)).cuda()
v = torch.empty_like(u)
flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
t_host = []
for it in range(6):
    flush.fill_(1.0)
    flush.sum()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    lv.apply(u, v)
    b.record()
    torch.cuda.synchronize()
print("event time %.2f us" % (a.elapsed_time(b) * 1e3))
n = 2048 * 4
buf = (ctypes.c_ulonglong * n)()
bi = (ctypes.c_ulonglong * (4096 * 2))()
lib.sfmg_tl_read(bi, 4096 * 2, buf, n)
t = np.frombuffer(buf, dtype=np.uint64).reshape(2048, 4).astype(np.float64)
ok = t[:, 0] > 0
t = t[ok]
t0 = t[:, 0].min()
for s, name in enumerate(["entry", "before first wait", "after first wait", "exit"]):
    c = (t[:, s] - t0) / 1e3
    c = c[t[:, s] > 0]
    print("%-18s n=%4d min %7.2f med %7.2f max %7.2f us" % (name, len(c), c.min(), np.median(c), c.max()))

ti = np.frombuffer(bi, dtype=np.uint64).reshape(4096, 2).astype(np.float64)
ti = ti[ti[:, 0] > 0]
print("k_init: blocks %d, first entry %.2f us before the apply's first entry; last exit %.2f us after it"
      % (len(ti), (t0 - ti[:, 0].min()) / 1e3, (ti[:, 1].max() - t0) / 1e3))
print("k_init span %.2f us; apply span %.2f us; init first entry -> apply last exit %.2f us"
      % ((ti[:, 1].max() - ti[:, 0].min()) / 1e3, (t[:, 3].max() - t0) / 1e3, (t[:, 3].max() - ti[:, 0].min()) / 1e3))
