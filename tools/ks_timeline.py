"""Developer probe: per-phase durations of the k-split apply (library variant built with
-DSFMG_KS_DBG).  Usage: python tools/ks_timeline.py [p]"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1402_5938_b200 import inputs, sfmg  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 16
lib = ctypes.CDLL(os.path.join(ROOT, "paper_1402_5938_b200", "libsfmg.so"))
lv = sfmg.Level(sfmg.Problem.from_dict(inputs.CONFIG3[p]))
u = torch.from_numpy(inputs.uniform_pm1(1, lv.N)).cuda()
v = torch.empty_like(u)
flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
for it in range(5):
    flush.fill_(1.0)
    flush.sum()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    lv.apply(u, v)
    b.record()
    torch.cuda.synchronize()
print("event time %.2f us" % (a.elapsed_time(b) * 1e3))
n = 148 * 16 * 10
buf = (ctypes.c_ulonglong * n)()
lib.sfmg_ksdbg_read(buf, n)
t = np.frombuffer(buf, dtype=np.uint64).reshape(148, 16, 10).astype(np.float64)
t0 = t[:, 0, 0][t[:, 0, 0] > 0].min()
names = ["gather", "P1P2", "clwait", "P3", "P4P5", "rxwait", "P6", "next"]
for h in (0, 1):
    rows = t[h::2]
    d = []
    for el in range(16):
        r = rows[:, el, :]
        ok = r[:, 7] > 0
        if not ok.any():
            continue
        r = r[ok]
        seg = [r[:, s + 1] - r[:, s] for s in range(7)]
        nxt = rows[:, el + 1, 0][ok] - r[:, 7] if el + 1 < 16 else np.zeros(ok.sum())
        d.append([np.median(x) / 1e3 for x in seg] + [np.median(np.where(nxt > 0, nxt, 0)) / 1e3])
    d = np.array(d)
    print("H=%d  per-element phase medians (us), elements %d" % (h, len(d)))
    print("   " + " ".join("%7s" % x for x in names))
    for i, row in enumerate(d):
        print("%2d " % i + " ".join("%7.2f" % x for x in row))
    print("start of element 0 (us after first block): med %.2f" % (np.median(rows[:, 0, 0] - t0) / 1e3))
    print("end (us): med %.2f max %.2f" % (np.median(rows[:, :, 7].max(1) - t0) / 1e3, (rows[:, :, 7].max(1) - t0).max() / 1e3))
s = t[:, 15, :]
ok = s[:, 0] > 0
print("kernel entry (us after first entry): med %.2f max %.2f" % (np.median(s[ok, 0] - s[ok, 0].min()) / 1e3, (s[ok, 0] - s[ok, 0].min()).max() / 1e3))
print("setup (entry -> loop): med %.2f max %.2f" % (np.median(s[ok, 1] - s[ok, 0]) / 1e3, (s[ok, 1] - s[ok, 0]).max() / 1e3))
print("exit (us after first entry): med %.2f max %.2f" % (np.median(s[ok, 2] - s[ok, 0].min()) / 1e3, (s[ok, 2] - s[ok, 0].min()).max() / 1e3))
print("first loop mark after first entry: %.2f" % ((t[:, 0, 0][t[:, 0, 0] > 0].min() - s[ok, 0].min()) / 1e3))
# element-kernel time alone (library events around the launch)
lv.profile(True)
for it in range(5):
    flush.fill_(1.0)
    flush.sum()
    lv.apply(u, v)
torch.cuda.synchronize()
ms, nl = lv.profile_read(reset=True)
print("element kernel alone (events around the launch): %.2f us" % (ms * 1e3 / nl))
