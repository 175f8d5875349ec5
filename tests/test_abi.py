"""CPU checks of the C-ABI library: it loads, exports every symbol include/sfmg.h declares, and
the synchronous argument checks / size queries (no GPU needed) behave as documented."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1402_5938_b200 import _build
    _build.build()
    from paper_1402_5938_b200 import sfmg
    return sfmg


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "sfmg.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(sfmg_[a-z0-9_]+)\s*\(", hdr)))


def test_header_symbols_exported(lib):
    so = C.CDLL(lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(so, s), s
    assert set(syms) == set(lib.EXPORTED)


def test_version_and_query(lib):
    assert "sm_100a" in lib.version()
    from paper_1402_5938_b200 import inputs
    N, E, ws = lib.level_query(lib.Problem.from_dict(inputs.CONFIG2))
    assert N == 129 ** 3 and E == 16 ** 3
    assert ws >= 48 * E * 9 ** 3 + 5 * 8 * N        # G plus the level's vectors
    N, E, ws = lib.level_query(lib.Problem.from_dict(inputs.CONFIG4))
    assert N == 513 ** 3 and E == 64 ** 3 and ws < 16 * 2 ** 30


@pytest.mark.parametrize("bad,code", [
    (dict(nex=2, ney=2, nez=2, p=0), "SFMG_E_ORDER"),
    (dict(nex=2, ney=2, nez=2, p=17), "SFMG_E_ORDER"),
    (dict(nex=0, ney=2, nez=2, p=2), "SFMG_E_MESH"),
    (dict(nex=2000, ney=2000, nez=2000, p=2), "SFMG_E_MESH"),
    (dict(nex=2, ney=2, nez=2, p=2, warp=3), "SFMG_E_ARG"),
    (dict(nex=2, ney=2, nez=2, p=2, coeff=9), "SFMG_E_ARG"),
])
def test_query_rejects_bad_problems(lib, bad, code):
    with pytest.raises(lib.SfmgError) as ei:
        lib.level_query(lib.Problem.from_dict(bad))
    assert ei.value.status == code


def test_hier_query_pcoarsen(lib):
    nb = C.c_size_t()
    prob = lib.Problem(2, 2, 2, 6)._c()
    rc = lib._lib.sfmg_hier_query(C.byref(prob), C.byref(lib.MgParams()._c()), C.byref(nb))
    assert lib.STATUS[rc] == "SFMG_E_PCOARSEN"
    prob = lib.Problem(8, 8, 8, 16)._c()
    assert lib._lib.sfmg_hier_query(C.byref(prob), C.byref(lib.MgParams()._c()), C.byref(nb)) == 0
    bad = lib.MgParams(cheb_degree=0)._c()
    assert lib.STATUS[lib._lib.sfmg_hier_query(C.byref(prob), C.byref(bad), C.byref(nb))] == "SFMG_E_ARG"


def test_null_handles_rejected(lib):
    assert lib.STATUS[lib._lib.sfmg_apply(None, 0, None, None, 0, None)] == "SFMG_E_ARG"
    assert lib.STATUS[lib._lib.sfmg_vcycle(None, None, None, None)] == "SFMG_E_ARG"
