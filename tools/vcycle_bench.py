"""Developer timing of the config-5 p-MG V-cycle and PCG solve (per-kernel split via ncu)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1402_5938_b200 import inputs, sfmg


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    H = sfmg.Hierarchy(sfmg.Problem.from_dict(inputs.CONFIG5), sfmg.MgParams())
    b = H.levels[0].load_vector(1)
    x = torch.empty_like(b)
    for _ in range(2):
        H.vcycle(b, x)
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        H.vcycle(b, x)
    e.record()
    torch.cuda.synchronize()
    print("vcycle_ms", a.elapsed_time(e) / reps)
    if len(sys.argv) > 2 and sys.argv[2] == "nosolve":
        return
    t0 = time.perf_counter()
    xs, rep = H.solve(b, mode=1, rtol=1e-8)
    torch.cuda.synchronize()
    print("solve_ms", (time.perf_counter() - t0) * 1e3, {k: v for k, v in rep.items() if k != "history"})


if __name__ == "__main__":
    main()
