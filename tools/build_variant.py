"""Developer A/B helper: build a variant of libsfmg.so with extra preprocessor defines into
abvar/<name>.so (git-ignored, travels with gpurun) (only k_operator.cu is recompiled; the other objects come from the in-tree build).
Usage: python tools/build_variant.py NAME -DSFMG_X=1 [-DSFMG_Y=2 ...]"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1402_5938_b200 import _build as B  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    B.build()
    out_dir = os.path.join(B.ROOT, "abvar")
    os.makedirs(out_dir, exist_ok=True)
    obj = os.path.join(out_dir, name + "_k_operator.o")
    subprocess.check_call([B.NVCC, *B.ARCH, *[f for f in B.FLAGS if f != "-v" and f != "-Xptxas"], *defs, "-c",
                           os.path.join(B.CSRC, "k_operator.cu"), "-o", obj])
    objs = [os.path.join(B.BUILD, os.path.splitext(s)[0] + ".o") for s in B.SOURCES if s != "k_operator.cu"]
    lib = os.path.join(out_dir, name + ".so")
    subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-o", lib, obj, *objs, "-lcudart_static", "-lrt", "-ldl",
                           "-lpthread"])
    os.remove(obj)
    print(lib)


if __name__ == "__main__":
    main()
