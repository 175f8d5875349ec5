"""sfmg: B200-native (sm_100a, fp64) matrix-free sum-factorised high-order stiffness operator,
Chebyshev-Jacobi smoother and p-multigrid of arXiv 1402.5938, behind the C ABI include/sfmg.h.

`import paper_1402_5938_b200.sfmg` loads libsfmg.so (fails loudly if it is not built)."""
