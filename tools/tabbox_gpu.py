"""Iteration counts of the paper's settings on 2d-const 32x32 (tab:box) on the GPU (NEXT-2), both
quadratures, h- and p-multigrid columns: python tools/tabbox_gpu.py [orders...].  One JSON line per
(order, quadrature); columns MG-J, MG-C, pCG-J, pCG-C for h then p (p-columns only for powers of two)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1402_5938_b200 import sfmg  # noqa: E402

# tab:box rows: MG-J h, p, MG-C h, p, pCG-J h, p, pCG-C h, p
PAPER = {1: [6, None, 5, None, 5, None, 4, None], 2: [7, 7, 5, 6, 5, 5, 4, 4], 3: [8, None, 6, None, 6, None, 5, None],
         4: [9, 8, 6, 6, 6, 5, 5, 5], 5: [12, None, 8, None, 7, None, 6, None], 6: [12, None, 9, None, 7, None, 6, None],
         7: [16, None, 12, None, 8, None, 7, None], 8: [17, 14, 13, 10, 9, 8, 7, 6], 16: [40, 33, 33, 27, 14, 12, 12, 11]}


def run(d, params):
    its, ms = [], []
    for mode in (0, 1):
        for sm in ("jacobi", "cheb"):
            H = sfmg.Hierarchy(sfmg.Problem.from_dict(d), params(sm, 2))
            b = H.levels[0].load_vector(1)
            H.solve(b, mode=mode, rtol=1e-8, max_iter=300)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, rep = H.solve(b, mode=mode, rtol=1e-8, max_iter=300)
            torch.cuda.synchronize()
            ms.append(round((time.perf_counter() - t0) * 1e3, 2))
            its.append(rep["iterations"])
            del H
    return its, ms


def main():
    orders = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5, 6, 7, 8, 16]
    for quad in (1, 0):
        for p in orders:
            d = dict(nex=32, ney=32, nez=1, p=p, dim=2, quadrature=quad)
            h, hms = run(d, sfmg.MgParams.paper_h)
            pm, pms = run(d, sfmg.MgParams.paper) if (p & (p - 1)) == 0 else (None, None)
            print(json.dumps({"p": p, "quadrature": "gauss" if quad else "lgl", "N": (32 * p + 1) ** 2,
                              "h_mgJ_mgC_pcgJ_pcgC": h, "p_mgJ_mgC_pcgJ_pcgC": pm, "paper_h": PAPER[p][0::2],
                              "paper_p": PAPER[p][1::2], "solve_ms_h": hms, "solve_ms_p": pms}), flush=True)


if __name__ == "__main__":
    main()
