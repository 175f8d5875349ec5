"""Writes tests/golden/config5_oracle.json: the CPU oracle's (oracle/ only) MG-PCG and MG-solver runs on
BASELINE config 5 (8^3 warped hexes, p = 16 -> 8 -> 4 -> 2 -> 1, mu = exp(3S), MMS load vector, V(2,2)
degree-4 Chebyshev on [0.1, 1.1] lambda_max, coarse CG 1e-10, rtol 1e-8).  The GPU test compares the
iteration counts (+-1) and the final residual bar against these stored values.

    python tools/make_golden.py            (minutes on 8 host cores)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1402_5938_b200 import inputs  # noqa: E402


def main():
    d = inputs.CONFIG5
    t0 = time.time()
    H = oracle.Hier(d["nex"], d["ney"], d["nez"], d["p"], d["warp"], d["amp"], d["coeff"], d["c0"], d["c1"],
                    nu_pre=2, nu_post=2, degree=4, lo_frac=0.1, hi_frac=1.1, power_iters=10, seed=inputs.POWER_SEED,
                    coarse_rtol=1e-10, coarse_maxit=10000, geom_tier=3, tier=3)
    t_setup = time.time() - t0
    b = H.levels[0].load_vector(1)
    out = {"source": "tools/make_golden.py (oracle only: O3 sum-factorised apply, factorised geometry, "
                     "pinned against O1/O2 by tests/test_oracle_*.py)",
           "config": "BASELINE config 5", "N": H.N, "levels": H.nlevels,
           "lambda": [H.lam(l) for l in range(H.nlevels - 1)], "setup_s": t_setup,
           "b_norm": float(np.linalg.norm(b)), "b_sum": float(b.sum())}
    for mode, name in ((1, "pcg"), (0, "mg_solver")):
        t0 = time.time()
        r = H.solve(b, mode=mode, rtol=1e-8, maxit=200)
        out[name] = {"iterations": r["iterations"], "converged": r["converged"], "r0_norm": r["r0_norm"],
                     "r_norm": r["r_norm"], "history": [float(h) for h in r["history"]],
                     "fine_applies": r["fine_applies"], "seconds": time.time() - t0,
                     "x_sample": [float(r["x"][i]) for i in range(0, H.N, 99991)]}
        print(name, r["iterations"], r["r_norm"] / r["r0_norm"], time.time() - t0, flush=True)
    path = os.path.join(ROOT, "tests", "golden", "config5_oracle.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
