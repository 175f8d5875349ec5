"""Developer timing of the apply / Chebyshev kernels on the BASELINE configs (not the bench
contract; bench.py is).  Prints GDoF/s and the fraction of the HBM roofline per config."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1402_5938_b200 import inputs, sfmg

HBM = 6538.6e9


def timeit(fn, reps=40, warm=3, flush=None):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush is not None:
            mode = os.environ.get("QB_FLUSH", "writeread")
            if mode in ("write", "writeread"):
                flush.fill_(1.0)
            if mode in ("read", "writeread"):
                flush.sum()   # leaves clean lines in L2: no dirty write-back inside the timed region
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    ts.sort()
    k = len(ts) // 5   # trimmed mean: the event clock is coarse, a median of 20 quantises to ~2 us
    return sum(ts[k:len(ts) - k]) / (len(ts) - 2 * k)


def main():
    which = sys.argv[1:] or ["2", "3"]
    flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
    cfgs = []
    if "2" in which:
        cfgs.append(("config2", inputs.CONFIG2, 1))
    if "3" in which:
        cfgs += [("config3_p%d" % p, inputs.CONFIG3[p], 1) for p in (1, 2, 4, 8, 16)]
    for w in which:
        if w.startswith("3:"):
            p = int(w[2:])
            cfgs.append(("config3_p%d" % p, inputs.CONFIG3[p], 1))
    if "4" in which:
        cfgs.append(("config4", inputs.CONFIG4, 2))
    for name, d, seed in cfgs:
        lv = sfmg.Level(sfmg.Problem.from_dict(d))
        N, E, n = lv.N, lv.E, lv.n
        u = torch.from_numpy(inputs.uniform_pm1(seed, N)).cuda()
        v = torch.empty_like(u)
        b = torch.zeros_like(u)
        x = u.clone()
        lam = lv.lambda_max(10, 12345)
        if not (lam == lam and 0 < lam < 1e300):   # developer variants with garbage operators
            lam = 1.0
        t_apply = timeit(lambda: lv.apply(u, v), flush=flush)
        t_cheb = timeit(lambda: lv.cheb(b, x, 4, 0.1 * lam, 1.1 * lam), flush=flush)
        bytes_apply = 48 * E * n ** 3 + 16 * N
        bytes_step = 48 * E * n ** 3 + 40 * N
        flops = E * (12 * n ** 4 + 15 * n ** 3)
        print(json.dumps(dict(cfg=name, N=N, t_apply_us=t_apply * 1e6, gdofs_apply=N / t_apply / 1e9,
                              frac_hbm_apply=bytes_apply / t_apply / HBM, tflops_apply=flops / t_apply / 1e12,
                              t_step_us=t_cheb / 4 * 1e6, gdofs_step=N / (t_cheb / 4) / 1e9,
                              frac_hbm_step=bytes_step / (t_cheb / 4) / HBM)), flush=True)
        del lv


if __name__ == "__main__":
    main()
