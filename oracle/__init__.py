"""ctypes binding of the CPU oracle (oracle/sfmg_oracle.cpp).

TEST INFRASTRUCTURE, NOT PRODUCT CODE: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg may import this package.  The product path
(paper_1402_5938_b200) never imports it and shares no code with it.

Every function here only marshals numpy arrays; the arithmetic is in sfmg_oracle.cpp, whose
functions each cite the PAPER.md passage they follow.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sfmg_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with plain g++ (-O2, no FMA contraction: DESIGN.md R23)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call([
            "g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
            _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        d, i, i64, u64, vp = C.c_double, C.c_int, C.c_int64, C.c_uint64, C.c_void_p
        dp = C.POINTER(C.c_double)
        L.orc_level_create.restype = vp
        L.orc_level_create.argtypes = [i, i, i, i, i, d, i, d, d, i, i, i]
        L.orc_level_destroy.argtypes = [vp]
        L.orc_level_status.argtypes = [vp]
        L.orc_level_min_detj.argtypes = [vp]
        L.orc_level_min_detj.restype = d
        L.orc_level_ndofs.argtypes = [vp]
        L.orc_level_ndofs.restype = i64
        L.orc_level_nelem.argtypes = [vp]
        L.orc_level_nelem.restype = i64
        L.orc_level_set_tier.argtypes = [vp, i]
        L.orc_lgl.argtypes = [i, vp, vp]
        L.orc_deriv_matrix.argtypes = [i, vp]
        L.orc_lagrange_eval.argtypes = [i, d, vp, vp]
        L.orc_interp_matrix.argtypes = [i, i, vp]
        L.orc_splitmix64.argtypes = [u64, u64]
        L.orc_splitmix64.restype = u64
        L.orc_coeff.argtypes = [i, d, d, d, d, d]
        L.orc_coeff.restype = d
        L.orc_l2g_by_matching.argtypes = [vp, vp]
        L.orc_l2g_closed.argtypes = [vp, vp]
        L.orc_mask.argtypes = [vp, vp]
        L.orc_colors.argtypes = [vp, vp]
        L.orc_geometry.argtypes = [vp, i64, vp, vp, vp]
        L.orc_element_matrix.argtypes = [vp, i64, vp]
        L.orc_assemble_dense.argtypes = [vp, i, vp]
        L.orc_apply.argtypes = [vp, i, vp, vp, i]
        L.orc_apply_elements.argtypes = [vp, vp, vp, i64, vp, i]
        L.orc_level_cache_elements.argtypes = [vp, i64, vp]
        L.orc_apply_rows.argtypes = [vp, i, vp, i64, vp, vp, i]
        L.orc_diag.argtypes = [vp, i, vp]
        L.orc_lambda_max.argtypes = [vp, i, u64]
        L.orc_lambda_max.restype = d
        L.orc_cheb.argtypes = [vp, vp, vp, i, d, d]
        L.orc_lambda_arnoldi.argtypes = [vp, i, u64]
        L.orc_lambda_arnoldi.restype = d
        L.orc_jacobi.argtypes = [vp, vp, vp, i, d]
        L.orc_pair_kind.argtypes = [vp, vp]
        L.orc_set_quadrature.argtypes = [i]
        L.orc_hier_create2.restype = vp
        L.orc_hier_create2.argtypes = [i, i, i, i, i, d, i, d, d, i, i, i, d, d, i, u64, d, i, i, i,
                                       i, d, i, i, C.POINTER(C.c_int)]
        L.orc_hier_create3.restype = vp
        L.orc_hier_create3.argtypes = [i, i, i, i, i, d, i, d, d, i, i, i, d, d, i, u64, d, i, i, i,
                                       i, d, i, i, i, C.POINTER(C.c_int)]
        L.orc_prolong.argtypes = [vp, vp, vp, vp]
        L.orc_restrict.argtypes = [vp, vp, vp, vp]
        L.orc_load_vector.argtypes = [vp, i, vp]
        L.orc_exact_solution.argtypes = [vp, vp]
        L.orc_cg_dense.argtypes = [i, vp, vp, vp, d, i, C.POINTER(C.c_int)]
        L.orc_hier_create.restype = vp
        L.orc_hier_create.argtypes = [i, i, i, i, i, d, i, d, d, i, i, i, d, d, i, u64, d, i, i, i,
                                      C.POINTER(C.c_int)]
        L.orc_hier_destroy.argtypes = [vp]
        L.orc_hier_nlevels.argtypes = [vp]
        L.orc_hier_level.argtypes = [vp, i]
        L.orc_hier_level.restype = vp
        L.orc_hier_lambda.argtypes = [vp, i]
        L.orc_hier_lambda.restype = d
        L.orc_hier_fine_applies.argtypes = [vp]
        L.orc_hier_fine_applies.restype = i64
        L.orc_hier_coarse_iters.argtypes = [vp]
        L.orc_hier_coarse_iters.restype = i64
        L.orc_vcycle.argtypes = [vp, vp, vp]
        L.orc_solve.argtypes = [vp, i, vp, vp, d, i, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                dp, dp, vp, i, C.POINTER(C.c_int64)]
        # NEXT-2: 2-D levels / hierarchies
        L.orc2_level_create.restype = vp
        L.orc2_level_create.argtypes = [i, i, i, i, d, i, d, d]
        for nm in ("orc2_level_destroy", "orc2_hier_destroy"):
            getattr(L, nm).argtypes = [vp]
        L.orc2_level_status.argtypes = [vp]
        L.orc2_level_ndofs.argtypes = [vp]
        L.orc2_level_ndofs.restype = i64
        L.orc2_mask.argtypes = [vp, vp]
        L.orc2_geometry.argtypes = [vp, i64, vp]
        L.orc2_element_matrix.argtypes = [vp, i64, vp]
        L.orc2_assemble_dense.argtypes = [vp, i, vp]
        L.orc2_apply.argtypes = [vp, i, vp, vp]
        L.orc2_diag.argtypes = [vp, i, vp]
        L.orc2_lambda_max.argtypes = [vp, i, u64]
        L.orc2_lambda_max.restype = d
        L.orc2_lambda_arnoldi.argtypes = [vp, i, u64]
        L.orc2_lambda_arnoldi.restype = d
        L.orc2_cheb.argtypes = [vp, vp, vp, i, d, d]
        L.orc2_jacobi.argtypes = [vp, vp, vp, i, d]
        L.orc2_prolong.argtypes = [vp, vp, vp, vp]
        L.orc2_restrict.argtypes = [vp, vp, vp, vp]
        L.orc2_load_vector.argtypes = [vp, i, vp]
        L.orc2_exact_solution.argtypes = [vp, vp]
        L.orc2_hier_create.restype = vp
        L.orc2_hier_create.argtypes = [i, i, i, i, d, i, d, d, i, i, i, d, d, i, u64, d, i, i, d, i, i, i,
                                       C.POINTER(C.c_int)]
        L.orc2_hier_nlevels.argtypes = [vp]
        L.orc2_hier_level.argtypes = [vp, i]
        L.orc2_hier_level.restype = vp
        L.orc2_hier_lambda.argtypes = [vp, i]
        L.orc2_hier_lambda.restype = d
        L.orc2_vcycle.argtypes = [vp, vp, vp]
        L.orc2_solve.argtypes = [vp, i, vp, vp, d, i, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                 dp, dp, vp, i, C.POINTER(C.c_int64)]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def set_threads(t: int):
    lib().orc_set_threads(int(t))


def set_quadrature(q: int):
    """0: LGL points collocated with the nodes (R1, default); 1: p+1 Gauss-Legendre points per
    direction (NEXT-3).  Applies to levels / hierarchies created afterwards (oracle only)."""
    lib().orc_set_quadrature(int(q))


def get_threads() -> int:
    return int(lib().orc_get_threads())


# ----------------------------------------------------------------------------- basis
def lgl(p: int):
    x = np.zeros(p + 1)
    w = np.zeros(p + 1)
    if lib().orc_lgl(p, _p(x), _p(w)) != 0:
        raise ValueError("invalid order")
    return x, w


def deriv_matrix(p: int):
    D = np.zeros((p + 1, p + 1))
    if lib().orc_deriv_matrix(p, _p(D)) != 0:
        raise ValueError("invalid order")
    return D


def lagrange_eval(p: int, t: float):
    l = np.zeros(p + 1)
    dl = np.zeros(p + 1)
    lib().orc_lagrange_eval(p, float(t), _p(l), _p(dl))
    return l, dl


def interp_matrix(pc: int, pf: int):
    I = np.zeros((pf + 1, pc + 1))
    lib().orc_interp_matrix(pc, pf, _p(I))
    return I


def splitmix64(seed: int, i: int) -> int:
    return int(lib().orc_splitmix64(seed, i))


def coeff(kind, c0, c1, x, y, z):
    return lib().orc_coeff(kind, c0, c1, x, y, z)


# ----------------------------------------------------------------------------- level
class Level:
    """One (mesh, p) discretisation.  problem: dict with nex, ney, nez, p, warp, amp, coeff, c0, c1."""

    def __init__(self, nex, ney, nez, p, warp=0, amp=0.0, coeff=0, c0=1.0, c1=0.0,
                 eager=True, geom_tier=2, tier=2):
        self.h = lib().orc_level_create(nex, ney, nez, p, warp, amp, coeff, c0, c1,
                                        1 if eager else 0, geom_tier, tier)
        if not self.h:
            raise ValueError("invalid level parameters")
        self.nex, self.ney, self.nez, self.p = nex, ney, nez, p
        self.n = p + 1
        self.N = int(lib().orc_level_ndofs(self.h))
        self.E = int(lib().orc_level_nelem(self.h))

    def close(self):
        if self.h:
            lib().orc_level_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def status(self):
        return int(lib().orc_level_status(self.h))

    def min_detj(self):
        return float(lib().orc_level_min_detj(self.h))

    def set_tier(self, tier):
        lib().orc_level_set_tier(self.h, tier)

    def l2g_by_matching(self):
        a = np.zeros((self.E, self.n ** 3), dtype=np.int32)
        rc = lib().orc_l2g_by_matching(self.h, _p(a))
        assert rc == 0
        return a

    def l2g_closed(self):
        a = np.zeros((self.E, self.n ** 3), dtype=np.int32)
        lib().orc_l2g_closed(self.h, _p(a))
        return a

    def mask(self):
        a = np.zeros(self.N, dtype=np.uint8)
        lib().orc_mask(self.h, _p(a))
        return a

    def colors(self):
        a = np.zeros(self.E, dtype=np.uint8)
        lib().orc_colors(self.h, _p(a))
        return a

    def geometry(self, e):
        n3 = self.n ** 3
        G = np.zeros((6, n3))
        dJ = np.zeros(n3)
        X = np.zeros((3, n3))
        lib().orc_geometry(self.h, int(e), _p(G), _p(dJ), _p(X))
        return G, dJ, X

    def element_matrix(self, e):
        n3 = self.n ** 3
        K = np.zeros((n3, n3))
        lib().orc_element_matrix(self.h, int(e), _p(K))
        return K

    def assemble_dense(self, bc=0):
        A = np.zeros((self.N, self.N))
        if lib().orc_assemble_dense(self.h, bc, _p(A)) != 0:
            raise ValueError("mesh too large to assemble densely")
        return A

    def apply(self, u, bc=0, tier=2):
        u = np.ascontiguousarray(u, dtype=np.float64)
        v = np.zeros(self.N)
        lib().orc_apply(self.h, bc, _p(u), _p(v), tier)
        return v

    def apply_elements(self, u, elems, tier=2):
        u = np.ascontiguousarray(u, dtype=np.float64)
        elems = np.ascontiguousarray(elems, dtype=np.int64)
        v = np.zeros(self.N)
        lib().orc_apply_elements(self.h, _p(u), _p(v), len(elems), _p(elems), tier)
        return v

    def cache_elements(self, elems):
        elems = np.ascontiguousarray(elems, dtype=np.int64)
        lib().orc_level_cache_elements(self.h, len(elems), _p(elems))

    def apply_rows(self, u, rows, bc=0, tier=2):
        u = np.ascontiguousarray(u, dtype=np.float64)
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        out = np.zeros(len(rows))
        lib().orc_apply_rows(self.h, bc, _p(u), len(rows), _p(rows), _p(out), tier)
        return out

    def diag(self, bc=0):
        d = np.zeros(self.N)
        lib().orc_diag(self.h, bc, _p(d))
        return d

    def lambda_max(self, iters=10, seed=12345):
        return float(lib().orc_lambda_max(self.h, iters, seed))

    def lambda_arnoldi(self, m=10, seed=12345):
        """lambda_max(D^-1 A_D) from m Arnoldi iterations in the D-inner product (R26)."""
        return float(lib().orc_lambda_arnoldi(self.h, m, seed))

    def jacobi(self, b, x, steps, omega=2.0 / 3.0):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.array(x, dtype=np.float64, copy=True)
        lib().orc_jacobi(self.h, _p(b), _p(x), steps, omega)
        return x

    def cheb(self, b, x, degree, lo, hi):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.array(x, dtype=np.float64, copy=True)
        lib().orc_cheb(self.h, _p(b), _p(x), degree, lo, hi)
        return x

    def load_vector(self, rhs_id=1):
        f = np.zeros(self.N)
        if lib().orc_load_vector(self.h, rhs_id, _p(f)) != 0:
            raise ValueError("unknown rhs")
        return f

    def exact_solution(self):
        u = np.zeros(self.N)
        lib().orc_exact_solution(self.h, _p(u))
        return u


def prolong(coarse: Level, fine: Level, uc):
    uc = np.ascontiguousarray(uc, dtype=np.float64)
    uf = np.zeros(fine.N)
    rc = lib().orc_prolong(coarse.h, fine.h, _p(uc), _p(uf))
    if rc:
        raise ValueError("levels are neither (p/2, p) on one grid nor (ne/2, ne) at one order")
    return uf


def restrict(coarse: Level, fine: Level, rf):
    rf = np.ascontiguousarray(rf, dtype=np.float64)
    rc_ = np.zeros(coarse.N)
    rc = lib().orc_restrict(coarse.h, fine.h, _p(rf), _p(rc_))
    if rc:
        raise ValueError("levels are neither (p/2, p) on one grid nor (ne/2, ne) at one order")
    return rc_


def cg_dense(A, b, rtol=1e-12, maxit=1000):
    A = np.ascontiguousarray(A, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(len(b))
    it = C.c_int(0)
    rc = lib().orc_cg_dense(len(b), _p(A), _p(b), _p(x), rtol, maxit, C.byref(it))
    return x, it.value, rc


class _LevelView(Level):
    def __init__(self, h, owner):
        self.h = h
        self._owner = owner
        self.N = int(lib().orc_level_ndofs(h))
        self.E = int(lib().orc_level_nelem(h))

    def close(self):
        self.h = None


class Hier:
    """p-multigrid hierarchy p, p/2, ..., 1 (+ h_levels geometric coarsenings of the p = 1 mesh);
    coarsen=1: high-order h-multigrid, order p on meshes ne, ne/2, ..., ne/2^h_levels (NEXT-4).
    smoother 0: Chebyshev-Jacobi of `degree`; 1: damped point Jacobi (omega), one step per smoothing
    application.  lambda_method 0: power iteration (R9); 1: Arnoldi (R26)."""

    def __init__(self, nex, ney, nez, p, warp=0, amp=0.0, coeff=0, c0=1.0, c1=0.0,
                 nu_pre=2, nu_post=2, degree=4, lo_frac=0.1, hi_frac=1.1, power_iters=10,
                 seed=12345, coarse_rtol=1e-10, coarse_maxit=10000, geom_tier=3, tier=3,
                 smoother=0, omega=2.0 / 3.0, lambda_method=0, h_levels=0, coarsen=0):
        st = C.c_int(0)
        self.h = lib().orc_hier_create3(nex, ney, nez, p, warp, amp, coeff, c0, c1, nu_pre, nu_post,
                                        degree, lo_frac, hi_frac, power_iters, seed, coarse_rtol,
                                        coarse_maxit, geom_tier, tier, smoother, omega, lambda_method,
                                        h_levels, coarsen, C.byref(st))
        self.status = st.value
        if not self.h:
            raise ValueError("cannot build hierarchy (status %d)" % st.value)
        self.nlevels = int(lib().orc_hier_nlevels(self.h))
        self.levels = [_LevelView(lib().orc_hier_level(self.h, l), self) for l in range(self.nlevels)]
        orders = []
        q = p
        while True:
            orders.append(q)
            if q == 1 or coarsen == 1:
                break
            q //= 2
        orders += [orders[-1]] * h_levels
        for lv, q in zip(self.levels, orders):
            lv.p = q
            lv.n = q + 1
        self.N = self.levels[0].N

    def __del__(self):
        try:
            if self.h:
                lib().orc_hier_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def lam(self, l):
        return float(lib().orc_hier_lambda(self.h, l))

    @property
    def fine_applies(self):
        return int(lib().orc_hier_fine_applies(self.h))

    def vcycle(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros(self.N)
        rc = lib().orc_vcycle(self.h, _p(b), _p(x))
        if rc:
            raise RuntimeError("vcycle status %d" % rc)
        return x

    def solve(self, b, mode=1, rtol=1e-8, maxit=500, hist_cap=1024):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros(self.N)
        it, conv = C.c_int(0), C.c_int(0)
        r0, rn = C.c_double(0), C.c_double(0)
        fa = C.c_int64(0)
        hist = np.zeros(hist_cap)
        st = lib().orc_solve(self.h, mode, _p(b), _p(x), rtol, maxit, C.byref(it), C.byref(conv),
                             C.byref(r0), C.byref(rn), _p(hist), hist_cap, C.byref(fa))
        return dict(x=x, status=st, iterations=it.value, converged=bool(conv.value),
                    r0_norm=r0.value, r_norm=rn.value, history=hist[:min(it.value + 1, hist_cap)],
                    fine_applies=fa.value)


# ----------------------------------------------------------------------------- NEXT-2: 2-D
class Level2:
    """2-D quadrilateral level (NEXT-2): nex x ney elements of order p on the unit square,
    warp 1: x_i += amp sin(pi X) sin(pi Y); coeff 0 const c0, 1 exp(c1 S), 2 10^(c1 S),
    3 c0 + c1 (cos^2 2 pi x + cos^2 2 pi y) (2d-var), 4 the same with 10 pi (2d-var').  The quadrature
    is the one set by set_quadrature() at creation."""

    def __init__(self, nex, ney, p, warp=0, amp=0.0, coeff=0, c0=1.0, c1=0.0, _handle=None, _owner=None):
        if _handle is None:
            self.h = lib().orc2_level_create(nex, ney, p, warp, amp, coeff, c0, c1)
            if not self.h:
                raise ValueError("invalid level parameters")
        else:
            self.h, self._owner = _handle, _owner
        self.nex, self.ney, self.p, self.n = nex, ney, p, p + 1
        self.N = int(lib().orc2_level_ndofs(self.h))
        self.E = nex * ney

    def __del__(self):
        try:
            if self.h and getattr(self, "_owner", None) is None:
                lib().orc2_level_destroy(self.h)
            self.h = None
        except Exception:
            pass

    @property
    def status(self):
        return int(lib().orc2_level_status(self.h))

    def mask(self):
        m = np.zeros(self.N, dtype=np.uint8)
        lib().orc2_mask(self.h, m.ctypes.data_as(C.c_void_p))
        return m

    def geometry(self, e):
        G = np.zeros(3 * self.n * self.n)
        lib().orc2_geometry(self.h, e, _p(G))
        return G.reshape(3, self.n * self.n)

    def element_matrix(self, e):
        K = np.zeros((self.n * self.n, self.n * self.n))
        lib().orc2_element_matrix(self.h, e, _p(K))
        return K

    def assemble_dense(self, bc=0):
        A = np.zeros((self.N, self.N))
        lib().orc2_assemble_dense(self.h, bc, _p(A))
        return A

    def apply(self, u, bc=0):
        u = np.ascontiguousarray(u, dtype=np.float64)
        v = np.zeros(self.N)
        lib().orc2_apply(self.h, bc, _p(u), _p(v))
        return v

    def diag(self, bc=0):
        d = np.zeros(self.N)
        lib().orc2_diag(self.h, bc, _p(d))
        return d

    def lambda_max(self, iters=10, seed=12345):
        return float(lib().orc2_lambda_max(self.h, iters, seed))

    def lambda_arnoldi(self, m=10, seed=12345):
        return float(lib().orc2_lambda_arnoldi(self.h, m, seed))

    def cheb(self, b, x, degree, lo, hi):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.array(x, dtype=np.float64)
        lib().orc2_cheb(self.h, _p(b), _p(x), degree, lo, hi)
        return x

    def jacobi(self, b, x, steps, omega=2.0 / 3.0):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.array(x, dtype=np.float64)
        lib().orc2_jacobi(self.h, _p(b), _p(x), steps, omega)
        return x

    def load_vector(self, rhs_id=1):
        f = np.zeros(self.N)
        if lib().orc2_load_vector(self.h, rhs_id, _p(f)) != 0:
            raise ValueError("unknown rhs")
        return f

    def exact_solution(self):
        u = np.zeros(self.N)
        lib().orc2_exact_solution(self.h, _p(u))
        return u


def prolong2(coarse: Level2, fine: Level2, uc):
    uc = np.ascontiguousarray(uc, dtype=np.float64)
    uf = np.zeros(fine.N)
    if lib().orc2_prolong(coarse.h, fine.h, _p(uc), _p(uf)):
        raise ValueError("levels are neither (p/2, p) on one grid nor (ne/2, ne) at one order")
    return uf


def restrict2(coarse: Level2, fine: Level2, rf):
    rf = np.ascontiguousarray(rf, dtype=np.float64)
    rc = np.zeros(coarse.N)
    if lib().orc2_restrict(coarse.h, fine.h, _p(rf), _p(rc)):
        raise ValueError("levels are neither (p/2, p) on one grid nor (ne/2, ne) at one order")
    return rc


class Hier2:
    """2-D hierarchy (NEXT-2): coarsen 0 p-multigrid p, ..., 1 then h_levels meshes at p = 1; coarsen 1
    high-order h-multigrid at order p (32x32, 16x16, 8x8)."""

    def __init__(self, nex, ney, p, warp=0, amp=0.0, coeff=0, c0=1.0, c1=0.0, nu_pre=2, nu_post=2, degree=4,
                 lo_frac=0.1, hi_frac=1.1, power_iters=10, seed=12345, coarse_rtol=1e-10, coarse_maxit=10000,
                 smoother=0, omega=2.0 / 3.0, lambda_method=0, h_levels=0, coarsen=0):
        st = C.c_int(0)
        self.h = lib().orc2_hier_create(nex, ney, p, warp, amp, coeff, c0, c1, nu_pre, nu_post, degree, lo_frac,
                                        hi_frac, power_iters, seed, coarse_rtol, coarse_maxit, smoother, omega,
                                        lambda_method, h_levels, coarsen, C.byref(st))
        self.status = st.value
        if not self.h:
            raise ValueError("cannot build hierarchy (status %d)" % st.value)
        self.nlevels = int(lib().orc2_hier_nlevels(self.h))
        orders, q = [], p
        while True:
            orders.append(q)
            if q == 1 or coarsen == 1:
                break
            q //= 2
        meshes = [(nex, ney)] * len(orders) + [(nex >> j, ney >> j) for j in range(1, h_levels + 1)]
        orders += [orders[-1]] * h_levels
        self.levels = [Level2(mx, my, q, _handle=lib().orc2_hier_level(self.h, l), _owner=self)
                       for l, ((mx, my), q) in enumerate(zip(meshes, orders))]
        self.N = self.levels[0].N

    def __del__(self):
        try:
            if self.h:
                for lv in self.levels:
                    lv.h = None
                lib().orc2_hier_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def lam(self, l):
        return float(lib().orc2_hier_lambda(self.h, l))

    def vcycle(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros(self.N)
        rc = lib().orc2_vcycle(self.h, _p(b), _p(x))
        if rc:
            raise RuntimeError("vcycle status %d" % rc)
        return x

    def solve(self, b, mode=1, rtol=1e-8, maxit=500, hist_cap=1024):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros(self.N)
        it, conv = C.c_int(0), C.c_int(0)
        r0, rn = C.c_double(0), C.c_double(0)
        fa = C.c_int64(0)
        hist = np.zeros(hist_cap)
        st = lib().orc2_solve(self.h, mode, _p(b), _p(x), rtol, maxit, C.byref(it), C.byref(conv),
                              C.byref(r0), C.byref(rn), _p(hist), hist_cap, C.byref(fa))
        return dict(x=x, status=st, iterations=it.value, converged=bool(conv.value),
                    r0_norm=r0.value, r_norm=rn.value, history=hist[:min(it.value + 1, hist_cap)],
                    fine_applies=fa.value)
