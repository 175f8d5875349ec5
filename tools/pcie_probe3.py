"""Developer probe: H2D rate of one 17 MB vector copied as k back-to-back chunks on one stream, and
D2H likewise (is the chunked copy of the pipelined host apply slower than one large copy?)."""
import time
import torch

N = 129 ** 3
B = 8 * N / 1e9
h = torch.empty(N, dtype=torch.float64).pin_memory()
d = torch.empty(N, dtype=torch.float64, device="cuda")
h.fill_(1.0)


def wall(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


for k in (1, 2, 4, 8, 16):
    ch = (N + k - 1) // k
    def f():
        for i in range(k):
            d[i * ch:(i + 1) * ch].copy_(h[i * ch:(i + 1) * ch], non_blocking=True)
    def g():
        for i in range(k):
            h[i * ch:(i + 1) * ch].copy_(d[i * ch:(i + 1) * ch], non_blocking=True)
    print("chunks=%2d  H2D %.1f GB/s  D2H %.1f GB/s" % (k, B / wall(f), B / wall(g)))
