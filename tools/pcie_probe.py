"""Developer probe of the host<->device copy rates behind the end-to-end (host-buffer) apply:
H2D alone, D2H alone, both directions at once, and sfmg_apply_host at several slab counts."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1402_5938_b200 import inputs, sfmg


def wall(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def main():
    N = 129 ** 3
    h1 = torch.empty(N, dtype=torch.float64).pin_memory()
    h2 = torch.empty(N, dtype=torch.float64).pin_memory()
    d1 = torch.empty(N, dtype=torch.float64, device="cuda")
    d2 = torch.empty(N, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    B = 8 * N / 1e9
    t = wall(lambda: d1.copy_(h1, non_blocking=True))
    print("H2D  %.1f us  %.1f GB/s" % (t * 1e6, B / t))
    t = wall(lambda: h2.copy_(d2, non_blocking=True))
    print("D2H  %.1f us  %.1f GB/s" % (t * 1e6, B / t))

    def both():
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    t = wall(both)
    print("both %.1f us  %.1f GB/s per direction" % (t * 1e6, B / t))
    lv = sfmg.Level(sfmg.Problem.from_dict(inputs.CONFIG2))
    u = h1.numpy()
    u[:] = inputs.uniform_pm1(1, N)
    v = h2.numpy()
    for S in (1, 2, 4, 8, 16):
        lv.host_pipeline(S)
        t = wall(lambda: lv.apply_host(u, v))
        print("apply_host slabs=%2d  %.1f us  %.2f GDoF/s" % (S, t * 1e6, N / t / 1e9))


if __name__ == "__main__":
    main()
