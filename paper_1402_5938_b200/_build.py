"""In-tree build of libsfmg.so for sm_100a (nvcc, no JIT cache): the .so lands next to this file
so it travels with the repo snapshot to the GPU box."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libsfmg.so")
SOURCES = ["basis.cu", "k_operator.cu", "k_gauss.cu", "k_2d.cu", "k_blas.cu", "k_transfer.cu", "sfmg_api.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I" + INCLUDE, "-I" + CSRC]


def _stale(out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str) -> str:
    obj = os.path.join(BUILD, os.path.splitext(src)[0] + ".o")
    # every header of csrc/ and include/ (conservative: a header edit rebuilds every object)
    deps = [os.path.join(CSRC, src), __file__] + [os.path.join(d, f) for d in (CSRC, INCLUDE)
                                                  for f in os.listdir(d) if f.endswith((".h", ".cuh"))]
    if _stale(obj, deps):
        log = obj + ".log"
        cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        with open(log, "w") as fh:
            r = subprocess.run(cmd, stdout=fh, stderr=subprocess.STDOUT)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed for %s:\n%s" % (src, open(log).read()[-6000:]))
    return obj


def build(force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    if force:
        for f in os.listdir(BUILD):
            if f.endswith(".o"):
                os.remove(os.path.join(BUILD, f))
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    if _stale(LIB, objs):
        tmp = LIB + ".tmp%d" % os.getpid()
        subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-ldl",
                               "-lpthread"])
        os.replace(tmp, LIB)
    return LIB


def build_tools() -> str:
    """Measurement tools (not the library): tools/fp64_peak, the DFMA-chain FP64 peak benchmark."""
    src = os.path.join(ROOT, "tools", "fp64_peak.cu")
    exe = os.path.join(ROOT, "tools", "fp64_peak")
    if _stale(exe, [src]):
        subprocess.check_call([NVCC, *ARCH, "-O3", "-o", exe, src])
    return exe


if __name__ == "__main__":
    print(build())
