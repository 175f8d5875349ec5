"""Iteration counts of the paper's settings on 3d-const 8^3 (tab:3d-box) on the GPU, for
both quadratures and both hierarchies (p: p-multigrid then two h-coarsenings at p = 1; h: three meshes
8^3, 4^3, 2^3 at the fine order, NEXT-4): python tools/tab3dbox_gpu.py [--h] [orders...].  Prints one
JSON line per (order, quadrature, hierarchy)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1402_5938_b200 import inputs, sfmg  # noqa: E402

PAPER = {1: [6, 4, 5, 4], 2: [8, 5, 6, 4], 4: [10, 7, 7, 5], 8: [19, 15, 10, 8], 16: [42, 34, 14, 13]}
PAPER_H = {1: [6, 4, 5, 4], 2: [8, 4, 6, 4], 3: [10, 7, 6, 5], 4: [11, 8, 7, 6], 5: [14, 10, 8, 7],
           6: [16, 11, 9, 7], 7: [20, 15, 10, 9], 8: [22, 17, 10, 9], 16: [47, 38, 16, 14]}


def main():
    args = sys.argv[1:]
    hmg = "--h" in args
    orders = [int(a) for a in args if a != "--h"] or ([1, 2, 3, 4, 5, 6, 7, 8, 16] if hmg else [1, 2, 4, 8, 16])
    params = sfmg.MgParams.paper_h if hmg else sfmg.MgParams.paper
    for quad in (1, 0):
        for p in orders:
            d = dict(inputs.problem(8, p), quadrature=quad)
            its, ms = [], []
            for mode in (0, 1):
                for sm in ("jacobi", "cheb"):
                    H = sfmg.Hierarchy(sfmg.Problem.from_dict(d), params(sm, h_levels=2))
                    b = H.levels[0].load_vector(1)
                    H.solve(b, mode=mode, rtol=1e-8, max_iter=300)
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    _, rep = H.solve(b, mode=mode, rtol=1e-8, max_iter=300)
                    torch.cuda.synchronize()
                    ms.append((time.perf_counter() - t0) * 1e3)
                    its.append(rep["iterations"])
                    del H
            print(json.dumps({"p": p, "quadrature": "gauss" if quad else "lgl", "hierarchy": "h" if hmg else "p",
                              "N": inputs.ndofs(d), "iterations_mgJ_mgC_pcgJ_pcgC": its,
                              "paper": (PAPER_H if hmg else PAPER).get(p),
                              "solve_ms": [round(x, 2) for x in ms]}), flush=True)


if __name__ == "__main__":
    main()
