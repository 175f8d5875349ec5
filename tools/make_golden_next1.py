"""Writes tests/golden/next1_3dconst_oracle.json: the CPU oracle's (oracle/ only) iteration counts of the
paper's own multigrid settings on the paper's 3d-const problem (unit cube, mu = 1), 8^3
elements, p = 2, 4, 8, 16 (tab:3d-box P:1250-1278):
  hierarchy  p -> p/2 -> ... -> 1 on 8^3, then 4^3 and 2^3 at p = 1 (h_levels = 2)
  smoothers  Jacobi(3,3), omega = 2/3 / Cheb(3,3) = one degree-3 Chebyshev-Jacobi application before
             and after, on [lambda/4, lambda], lambda from 10 Arnoldi iterations (R26)
  solvers    MG as solver / MG-preconditioned CG, ||r|| <= 1e-8 ||r0||, x0 = 0
  rhs        the manufactured load vector (rhs_id 1; the paper does not state its right-hand side)
The GPU test compares iteration counts (+-1).  The paper's own counts (tab:3d-box, p-multigrid
columns) are stored beside them as context only: this build uses collocated LGL quadrature (R1),
the paper does not state its quadrature, so the counts are not expected to coincide.

    python tools/make_golden_next1.py        (minutes on 8 host cores)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

# tab:3d-box, p-multigrid columns: MG-solver Jacobi(3,3), Cheb(3,3); pCG Jacobi, Cheb
PAPER = {2: [8, 5, 6, 4], 4: [10, 7, 7, 5], 8: [19, 15, 10, 8], 16: [42, 34, 14, 13]}


def main(orders=(2, 4, 8, 16)):
    out = {"source": "tools/make_golden_next1.py (oracle only: O3 apply, factorised geometry)",
           "problem": "3d-const (P:892-893): unit cube, mu = 1, affine 8^3 elements, MMS load vector",
           "paper_tab_3d_box_p_columns": {str(k): v for k, v in PAPER.items()},
           "paper_columns": ["mg_solver_jacobi33", "mg_solver_cheb33", "pcg_jacobi33", "pcg_cheb33"],
           "runs": {}}
    for p in orders:
        for sm, name in ((1, "jacobi33"), (0, "cheb33")):
            nu = 3 if sm == 1 else 1
            t0 = time.time()
            H = oracle.Hier(8, 8, 8, p, nu_pre=nu, nu_post=nu, degree=3, lo_frac=0.25, hi_frac=1.0,
                            power_iters=10, seed=12345, coarse_rtol=1e-10, coarse_maxit=10000, geom_tier=3, tier=3,
                            smoother=sm, omega=2.0 / 3.0, lambda_method=1, h_levels=2)
            b = H.levels[0].load_vector(1)
            lams = [H.lam(l) for l in range(H.nlevels - 1)]
            for mode, mname in ((0, "mg_solver"), (1, "pcg")):
                r = H.solve(b, mode=mode, rtol=1e-8, maxit=300)
                out["runs"]["p%d_%s_%s" % (p, mname, name)] = {
                    "p": p, "smoother": name, "mode": mname, "iterations": r["iterations"],
                    "converged": r["converged"], "rel_residual": r["r_norm"] / r["r0_norm"],
                    "history": [float(h) for h in r["history"]], "lambda": lams, "levels": H.nlevels}
                print(p, name, mname, r["iterations"], r["converged"], "%.1fs" % (time.time() - t0), flush=True)
            del H
    path = os.path.join(ROOT, "tests", "golden", "next1_3dconst_oracle.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
