"""Thin Python binding of libsfmg.so (include/sfmg.h).

Argument marshalling only: every step of the method runs in the library's CUDA kernels.  torch
is used for device memory (the caller-owned workspace and vectors) and for the current CUDA
stream.  There is no CPU fallback: if libsfmg.so is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsfmg.so")

if not os.path.exists(LIB_PATH):
    raise ImportError("libsfmg.so not built (run `python -m paper_1402_5938_b200._build` or "
                      "__graft_entry__.build()); there is no CPU fallback")

_lib = C.CDLL(LIB_PATH)

STATUS = {0: "SFMG_OK", 1: "SFMG_E_ARG", 2: "SFMG_E_ORDER", 3: "SFMG_E_MESH", 4: "SFMG_E_GEOMETRY",
          5: "SFMG_E_PCOARSEN", 6: "SFMG_E_BREAKDOWN", 7: "SFMG_E_WORKSPACE", 8: "SFMG_E_CUDA"}


class SfmgError(RuntimeError):
    def __init__(self, code, where):
        self.code = code
        self.status = STATUS.get(code, str(code))
        msg = _lib.sfmg_last_error().decode(errors="replace")
        super().__init__("%s: %s (%s)" % (where, self.status, msg))


class _Problem(C.Structure):
    _fields_ = [("nex", C.c_int32), ("ney", C.c_int32), ("nez", C.c_int32), ("order", C.c_int32),
                ("warp", C.c_int32), ("warp_amp", C.c_double), ("coeff", C.c_int32),
                ("c0", C.c_double), ("c1", C.c_double), ("quadrature", C.c_int32), ("dim", C.c_int32)]


class _MgParams(C.Structure):
    _fields_ = [("nu_pre", C.c_int32), ("nu_post", C.c_int32), ("cheb_degree", C.c_int32),
                ("eig_lo_frac", C.c_double), ("eig_hi_frac", C.c_double), ("power_iters", C.c_int32),
                ("power_seed", C.c_uint64), ("coarse_rtol", C.c_double), ("coarse_max_iter", C.c_int32),
                ("smoother", C.c_int32), ("jacobi_omega", C.c_double), ("lambda_method", C.c_int32),
                ("h_levels", C.c_int32), ("coarsen", C.c_int32)]


class _Report(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("r0_norm", C.c_double),
                ("r_norm", C.c_double), ("fine_applies", C.c_int64), ("vcycles", C.c_int64),
                ("history", C.POINTER(C.c_double)), ("history_cap", C.c_int32)]


_vp, _i32, _i64, _u64, _d = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
_P = C.POINTER
_SIG = {
    "sfmg_version": ([], C.c_char_p),
    "sfmg_last_error": ([], C.c_char_p),
    "sfmg_level_query": ([_P(_Problem), _P(_i64), _P(_i64), _P(C.c_size_t)], C.c_int),
    "sfmg_level_create": ([_P(_Problem), _vp, C.c_size_t, _vp, _P(_vp)], C.c_int),
    "sfmg_level_destroy": ([_vp], C.c_int),
    "sfmg_level_info": ([_vp, _P(_i64), _P(_i64), _P(_i32)], C.c_int),
    "sfmg_export_l2g": ([_vp, _vp, _vp], C.c_int),
    "sfmg_export_mask": ([_vp, _vp, _vp], C.c_int),
    "sfmg_export_colors": ([_vp, _vp, _vp], C.c_int),
    "sfmg_export_geometry": ([_vp, _vp, _vp], C.c_int),
    "sfmg_apply": ([_vp, _i32, _vp, _vp, _i64, _vp], C.c_int),
    "sfmg_diag": ([_vp, _i32, _vp, _i64, _vp], C.c_int),
    "sfmg_lambda_max": ([_vp, _i32, _u64, _P(_d), _vp], C.c_int),
    "sfmg_cheb": ([_vp, _vp, _vp, _i64, _i32, _d, _d, _vp], C.c_int),
    "sfmg_lambda_arnoldi": ([_vp, _i32, _u64, _vp, _P(_d), _vp], C.c_int),
    "sfmg_jacobi": ([_vp, _vp, _vp, _i64, _i32, _d, _vp], C.c_int),
    "sfmg_load_vector": ([_vp, _i32, _vp, _i64, _vp], C.c_int),
    "sfmg_apply_host": ([_vp, _i32, _vp, _vp, _i64, _vp], C.c_int),
    "sfmg_cheb_host": ([_vp, _vp, _vp, _i64, _i32, _d, _d, _vp], C.c_int),
    "sfmg_host_pipeline": ([_vp, _i32], C.c_int),
    "sfmg_profile_enable": ([_vp, _i32], C.c_int),
    "sfmg_profile_read": ([_vp, _P(_d), _P(_i64), _i32], C.c_int),
    "sfmg_prolong": ([_vp, _vp, _vp, _vp, _vp], C.c_int),
    "sfmg_restrict": ([_vp, _vp, _vp, _vp, _vp], C.c_int),
    "sfmg_hier_query": ([_P(_Problem), _P(_MgParams), _P(C.c_size_t)], C.c_int),
    "sfmg_hier_create": ([_P(_Problem), _P(_MgParams), _vp, C.c_size_t, _vp, _P(_vp)], C.c_int),
    "sfmg_hier_destroy": ([_vp], C.c_int),
    "sfmg_hier_info": ([_vp, _P(_i32), _P(_i64)], C.c_int),
    "sfmg_hier_level": ([_vp, _i32, _P(_vp)], C.c_int),
    "sfmg_hier_lambda": ([_vp, _i32, _P(_d)], C.c_int),
    "sfmg_vcycle": ([_vp, _vp, _vp, _vp], C.c_int),
    "sfmg_solve": ([_vp, _i32, _vp, _vp, _d, _i32, _P(_Report), _vp], C.c_int),
}
for _name, (_args, _res) in _SIG.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_SIG)


def _ck(rc, where):
    if rc != 0:
        raise SfmgError(rc, where)


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _dptr(t: torch.Tensor, n=None, dtype=torch.float64):
    if not (t.is_cuda and t.dtype == dtype and t.is_contiguous()):
        raise ValueError("expected a contiguous CUDA %s tensor" % dtype)
    if n is not None and t.numel() != n:
        raise ValueError("expected %d entries, got %d" % (n, t.numel()))
    return C.c_void_p(t.data_ptr())


def _workspace(nbytes: int, device) -> torch.Tensor:
    ws = torch.empty(nbytes + 256, dtype=torch.uint8, device=device)
    return ws


def _aligned(ws: torch.Tensor) -> int:
    p = ws.data_ptr()
    return (p + 255) & ~255


@dataclass
class Problem:
    """Problem statement: nex x ney x nez hexes on [0,1]^3, order p, warp
    (0 identity, 1 sine bump of amplitude amp), coefficient kind (0: c0, 1: exp(c1 S),
    2: 10^(c1 S), 3: c0 + c1 sum cos^2(2 pi x_i))."""
    nex: int
    ney: int
    nez: int
    p: int
    warp: int = 0
    amp: float = 0.0
    coeff: int = 0
    c0: float = 1.0
    c1: float = 0.0
    quadrature: int = 0     # 0 collocated LGL (R1), 1 Gauss-Legendre (NEXT-3)
    dim: int = 3            # 2: quadrilaterals on [0,1]^2 (NEXT-2; nez = 1, coeff 4 = 2d-var')

    @classmethod
    def from_dict(cls, d):
        return cls(d["nex"], d["ney"], d["nez"], d["p"], d.get("warp", 0), d.get("amp", 0.0),
                   d.get("coeff", 0), d.get("c0", 1.0), d.get("c1", 0.0), d.get("quadrature", 0), d.get("dim", 3))

    def _c(self):
        return _Problem(self.nex, self.ney, self.nez, self.p, self.warp, self.amp, self.coeff, self.c0, self.c1,
                        self.quadrature, self.dim)


def version() -> str:
    return _lib.sfmg_version().decode()


def level_query(prob: Problem):
    n, e, ws = _i64(), _i64(), C.c_size_t()
    _ck(_lib.sfmg_level_query(C.byref(prob._c()), C.byref(n), C.byref(e), C.byref(ws)), "sfmg_level_query")
    return n.value, e.value, ws.value


class Level:
    """One (mesh, p) level: geometric factors, diag(A_D) and scratch inside a torch workspace."""

    def __init__(self, prob: Problem, device="cuda", stream=None, _handle=None, _owner=None):
        self.prob = prob
        self._owner = _owner
        if _handle is not None:
            self.h = _handle
            self.ws = None
        else:
            self.N, self.E, nbytes = level_query(prob)
            self.ws = _workspace(nbytes, device)
            h = _vp()
            _ck(_lib.sfmg_level_create(C.byref(prob._c()), C.c_void_p(_aligned(self.ws)), nbytes,
                                       _stream(stream), C.byref(h)), "sfmg_level_create")
            self.h = h
        n, e, p = _i64(), _i64(), _i32()
        _ck(_lib.sfmg_level_info(self.h, C.byref(n), C.byref(e), C.byref(p)), "sfmg_level_info")
        self.N, self.E, self.p = n.value, e.value, p.value
        self.n = self.p + 1
        self.device = device

    def close(self):
        if self._owner is None and getattr(self, "h", None):
            _lib.sfmg_level_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _vec(self, like=None):
        return torch.empty(self.N, dtype=torch.float64, device=self.device)

    def apply(self, u, v=None, bc=0, stream=None):
        v = self._vec() if v is None else v
        _ck(_lib.sfmg_apply(self.h, bc, _dptr(u, self.N), _dptr(v, self.N), self.N, _stream(stream)), "sfmg_apply")
        return v

    def diag(self, bc=0, out=None, stream=None):
        d = self._vec() if out is None else out
        _ck(_lib.sfmg_diag(self.h, bc, _dptr(d, self.N), self.N, _stream(stream)), "sfmg_diag")
        return d

    def lambda_max(self, iters=10, seed=12345, stream=None):
        lam = _d()
        _ck(_lib.sfmg_lambda_max(self.h, iters, seed, C.byref(lam), _stream(stream)), "sfmg_lambda_max")
        return lam.value

    def lambda_arnoldi(self, steps=10, seed=12345, stream=None):
        """lambda_max(D^-1 A_D) by `steps` Arnoldi iterations in the D-inner product (R26)."""
        work = torch.empty((steps + 2) * self.N, dtype=torch.float64, device=self.device)
        lam = _d()
        _ck(_lib.sfmg_lambda_arnoldi(self.h, steps, seed, C.c_void_p(work.data_ptr()), C.byref(lam),
                                     _stream(stream)), "sfmg_lambda_arnoldi")
        return lam.value

    def jacobi(self, b, x, steps, omega=2.0 / 3.0, stream=None):
        """In place on x: `steps` damped point-Jacobi steps."""
        _ck(_lib.sfmg_jacobi(self.h, _dptr(b, self.N), _dptr(x, self.N), self.N, steps, omega, _stream(stream)),
            "sfmg_jacobi")
        return x

    def cheb(self, b, x, degree, lam_lo, lam_hi, stream=None):
        """In place on x (initial guess in, smoothed iterate out)."""
        _ck(_lib.sfmg_cheb(self.h, _dptr(b, self.N), _dptr(x, self.N), self.N, degree, lam_lo, lam_hi,
                           _stream(stream)), "sfmg_cheb")
        return x

    def load_vector(self, rhs_id=1, out=None, stream=None):
        f = self._vec() if out is None else out
        _ck(_lib.sfmg_load_vector(self.h, rhs_id, _dptr(f, self.N), self.N, _stream(stream)), "sfmg_load_vector")
        return f

    def export_l2g(self, stream=None):
        a = torch.empty((self.E, self.n ** 3), dtype=torch.int32, device=self.device)
        _ck(_lib.sfmg_export_l2g(self.h, _dptr(a, dtype=torch.int32), _stream(stream)), "sfmg_export_l2g")
        return a

    def export_mask(self, stream=None):
        a = torch.empty(self.N, dtype=torch.uint8, device=self.device)
        _ck(_lib.sfmg_export_mask(self.h, _dptr(a, dtype=torch.uint8), _stream(stream)), "sfmg_export_mask")
        return a

    def export_colors(self, stream=None):
        a = torch.empty(self.E, dtype=torch.uint8, device=self.device)
        _ck(_lib.sfmg_export_colors(self.h, _dptr(a, dtype=torch.uint8), _stream(stream)), "sfmg_export_colors")
        return a

    def export_geometry(self, stream=None):
        a = torch.empty((self.E, self.n, 6, self.n ** 2), dtype=torch.float64, device=self.device)
        _ck(_lib.sfmg_export_geometry(self.h, _dptr(a), _stream(stream)), "sfmg_export_geometry")
        return a

    def profile(self, enable=True):
        _ck(_lib.sfmg_profile_enable(self.h, 1 if enable else 0), "sfmg_profile_enable")

    def profile_read(self, reset=True):
        ms, n = _d(), _i64()
        _ck(_lib.sfmg_profile_read(self.h, C.byref(ms), C.byref(n), 1 if reset else 0), "sfmg_profile_read")
        return ms.value, n.value

    # host-buffer (end-to-end) variants; numpy in, numpy out
    def apply_host(self, u: np.ndarray, v: np.ndarray = None, bc=0, stream=None):
        u = np.ascontiguousarray(u, dtype=np.float64)
        v = np.empty(self.N) if v is None else v
        _ck(_lib.sfmg_apply_host(self.h, bc, u.ctypes.data_as(_vp), v.ctypes.data_as(_vp), self.N,
                                 _stream(stream)), "sfmg_apply_host")
        return v

    def host_pipeline(self, slabs: int = 0):
        """Slab count of the pipelined apply_host (0 = automatic)."""
        _ck(_lib.sfmg_host_pipeline(self.h, slabs), "sfmg_host_pipeline")

    def cheb_host(self, b: np.ndarray, x: np.ndarray, degree, lam_lo, lam_hi, stream=None):
        """In place on the host array x."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        assert x.flags.c_contiguous and x.dtype == np.float64
        _ck(_lib.sfmg_cheb_host(self.h, b.ctypes.data_as(_vp), x.ctypes.data_as(_vp), self.N, degree, lam_lo,
                                lam_hi, _stream(stream)), "sfmg_cheb_host")
        return x


def prolong(coarse: Level, fine: Level, uc, uf=None, stream=None):
    uf = fine._vec() if uf is None else uf
    _ck(_lib.sfmg_prolong(coarse.h, fine.h, _dptr(uc, coarse.N), _dptr(uf, fine.N), _stream(stream)), "sfmg_prolong")
    return uf


def restrict(coarse: Level, fine: Level, rf, rc=None, stream=None):
    rc = coarse._vec() if rc is None else rc
    _ck(_lib.sfmg_restrict(coarse.h, fine.h, _dptr(rf, fine.N), _dptr(rc, coarse.N), _stream(stream)),
        "sfmg_restrict")
    return rc


@dataclass
class MgParams:
    """p-MG parameters (BASELINE config 5 defaults; R7-R11, R13).  smoother 1 = damped Jacobi
    (jacobi_omega), lambda_method 1 = Arnoldi, h_levels = geometric coarsenings after p = 1: the
    paper's own settings (see MgParams.paper())."""
    nu_pre: int = 2
    nu_post: int = 2
    cheb_degree: int = 4
    eig_lo_frac: float = 0.1
    eig_hi_frac: float = 1.1
    power_iters: int = 10
    power_seed: int = 12345
    coarse_rtol: float = 1e-10
    coarse_max_iter: int = 10000
    smoother: int = 0
    jacobi_omega: float = 2.0 / 3.0
    lambda_method: int = 0
    h_levels: int = 0
    coarsen: int = 0   # 1: high-order h-multigrid at fixed p (NEXT-4)

    @staticmethod
    def paper(smoother="cheb", h_levels=2):
        """Jacobi(3,3) with omega = 2/3, or Cheb(3,3) = one degree-3
        Chebyshev application before and after, on [lambda/4, lambda] with lambda from 10 Arnoldi
        iterations; p-coarsening to 1, then `h_levels` geometric coarsenings."""
        if smoother == "jacobi":
            return MgParams(nu_pre=3, nu_post=3, smoother=1, lambda_method=1, h_levels=h_levels,
                            eig_lo_frac=0.25, eig_hi_frac=1.0)
        return MgParams(nu_pre=1, nu_post=1, cheb_degree=3, eig_lo_frac=0.25, eig_hi_frac=1.0, lambda_method=1,
                        h_levels=h_levels)

    @staticmethod
    def paper_h(smoother="cheb", h_levels=2):
        """The paper's h-multigrid columns: the same smoothers on three meshes
        ne, ne/2, ne/4 at the fine order (NEXT-4)."""
        mg = MgParams.paper(smoother, h_levels)
        mg.coarsen = 1
        return mg

    def _c(self):
        return _MgParams(self.nu_pre, self.nu_post, self.cheb_degree, self.eig_lo_frac, self.eig_hi_frac,
                         self.power_iters, self.power_seed, self.coarse_rtol, self.coarse_max_iter,
                         self.smoother, self.jacobi_omega, self.lambda_method, self.h_levels, self.coarsen)


class Hierarchy:
    """p-multigrid hierarchy p, p/2, ..., 1 on one element grid."""

    def __init__(self, prob: Problem, mg: MgParams = None, device="cuda", stream=None):
        self.prob = prob
        self.mg = mg or MgParams()
        nbytes = C.c_size_t()
        _ck(_lib.sfmg_hier_query(C.byref(prob._c()), C.byref(self.mg._c()), C.byref(nbytes)), "sfmg_hier_query")
        self.ws = _workspace(nbytes.value, device)
        h = _vp()
        _ck(_lib.sfmg_hier_create(C.byref(prob._c()), C.byref(self.mg._c()), C.c_void_p(_aligned(self.ws)),
                                  nbytes.value, _stream(stream), C.byref(h)), "sfmg_hier_create")
        self.h = h
        nl, nf = _i32(), _i64()
        _ck(_lib.sfmg_hier_info(self.h, C.byref(nl), C.byref(nf)), "sfmg_hier_info")
        self.nlevels, self.N = nl.value, nf.value
        self.device = device
        self.levels = []
        for l in range(self.nlevels):
            lh = _vp()
            _ck(_lib.sfmg_hier_level(self.h, l, C.byref(lh)), "sfmg_hier_level")
            self.levels.append(Level(prob, device, _handle=lh, _owner=self))

    def __del__(self):
        try:
            if getattr(self, "h", None):
                for lv in self.levels:
                    lv.h = None
                _lib.sfmg_hier_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def lam(self, l):
        v = _d()
        _ck(_lib.sfmg_hier_lambda(self.h, l, C.byref(v)), "sfmg_hier_lambda")
        return v.value

    def vcycle(self, b, x=None, stream=None):
        x = torch.empty_like(b) if x is None else x
        _ck(_lib.sfmg_vcycle(self.h, _dptr(b, self.N), _dptr(x, self.N), _stream(stream)), "sfmg_vcycle")
        return x

    def solve(self, b, x=None, mode=1, rtol=1e-8, max_iter=500, history_cap=1024, stream=None):
        x = torch.empty_like(b) if x is None else x
        hist = (C.c_double * history_cap)()
        rep = _Report(0, 0, 0.0, 0.0, 0, 0, C.cast(hist, C.POINTER(C.c_double)), history_cap)
        rc = _lib.sfmg_solve(self.h, mode, _dptr(b, self.N), _dptr(x, self.N), rtol, max_iter, C.byref(rep),
                             _stream(stream))
        if rc not in (0, 6):
            _ck(rc, "sfmg_solve")
        n = min(rep.iterations + 1, history_cap)
        return x, dict(status=STATUS[rc], iterations=rep.iterations, converged=bool(rep.converged),
                       r0_norm=rep.r0_norm, r_norm=rep.r_norm, fine_applies=rep.fine_applies,
                       vcycles=rep.vcycles, history=list(hist[:n]))
