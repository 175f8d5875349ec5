"""Seeded synthetic inputs shared by the tests, the oracle runs and bench.py.

This module holds none of the method's arithmetic: only the counter-based splitmix64
generator of DESIGN.md reading R15 ("u uniform in [-1,1] from seed s", BASELINE.json configs)
and the BASELINE.json problem descriptions.  Both the CUDA path and the oracle receive the
arrays it produces; neither computes them.
"""
from __future__ import annotations

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, start: int, count: int) -> np.ndarray:
    """Outputs start..start+count-1 of splitmix64 with initial state `seed` (uint64 array)."""
    with np.errstate(over="ignore"):
        i = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform_pm1(seed: int, n: int, chunk: int = 1 << 24) -> np.ndarray:
    """u_g = 2 * ((z_g >> 11) * 2^-53) - 1 for g = 0..n-1 (R15); all n entries are drawn."""
    out = np.empty(n, dtype=np.float64)
    for s in range(0, n, chunk):
        c = min(chunk, n - s)
        z = splitmix64(seed, s, c)
        out[s:s + c] = 2.0 * ((z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)) - 1.0
    return out


# BASELINE.json configs as problem dicts ("input recipe").
# warp 1: x_i -> x_i + amp sin(pi x) sin(pi y) sin(pi z); coeff 0: c0, 1: exp(c1 S), 2: 10^(c1 S),
# 3: c0 + c1 sum cos^2(2 pi x_i) with S = sin(2 pi x) sin(2 pi y) sin(2 pi z).
def problem(ne, p, warp=0, amp=0.0, coeff=0, c0=1.0, c1=0.0, ney=None, nez=None):
    return dict(nex=ne, ney=ne if ney is None else ney, nez=ne if nez is None else nez, p=p,
                warp=warp, amp=amp, coeff=coeff, c0=c0, c1=c1)


CONFIG1 = problem(4, 4)                                             # affine, mu = 1
CONFIG2 = problem(16, 8, warp=1, amp=0.1, coeff=1, c1=3.0)          # deformed, mu = exp(3S)
CONFIG3 = {p: problem(128 // p, p, warp=1, amp=0.1, coeff=1, c1=3.0) for p in (1, 2, 4, 8, 16)}
CONFIG4 = problem(64, 8, warp=1, amp=0.1, coeff=2, c1=2.0)          # mu = 10^(2S)
CONFIG5 = problem(8, 16, warp=1, amp=0.1, coeff=1, c1=3.0)          # p-MG 16 -> 1
SEEDS = {1: 0, 2: 1, 3: 1, 4: 2}
POWER_SEED = 12345


def ndofs(prob) -> int:
    p = prob["p"]
    return (prob["nex"] * p + 1) * (prob["ney"] * p + 1) * (prob["nez"] * p + 1)
