"""Build libagatha.so (the sm_100a CUDA library behind include/agatha.h) in-tree."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC = os.path.join(PKG, "csrc", "agatha.cu")
HDR = os.path.join(ROOT, "include", "agatha.h")
LIB = os.path.join(PKG, "libagatha.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2", "-shared",
    "-Xptxas", "-warn-spills",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in (SRC, HDR, __file__))


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Compile SRC into ``out``.  ``defines`` (e.g. ["AGATHA_FMA_ADD=0"]) build A/B
    variants of the kernels for tools/ab_bench.sh; the default build uses none."""
    if force or out != LIB or defines or stale():
        cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"),
               "-o", out + ".tmp", SRC]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if a != "--force"]
    defs = [a[2:] for a in args if a.startswith("-D")]
    outs = [a[len("--out="):] for a in args if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose=True, out=outs[0] if outs else LIB, defines=defs))
