"""Compile the sm_100a extension (librd.so) in-tree with nvcc.

No JIT cache, no torch extension machinery: a plain shared library with the
C ABI of include/rd.h, built for `-gencode arch=compute_100a,code=sm_100a`.
"""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "librd.so")
SOURCES = [os.path.join(HERE, "csrc", "rd_runtime.cu")]
DEPS = sorted(glob.glob(os.path.join(HERE, "csrc", "*")) + [os.path.join(ROOT, "include", "rd.h")])

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    # numerics: IEEE division/sqrt, no FTZ, no FMA contraction in host code
    # (device FP math also uses explicit __f*_rn/__d*_rn intrinsics, never contracted)
    "-prec-div=true", "-ftz=false", "-fmad=false", "-Xcompiler", "-ffp-contract=off",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def build(force: bool = False, verbose: bool = False) -> str:
    newest = max(os.path.getmtime(p) for p in DEPS)
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= newest:
        return LIB
    cmd = [nvcc(), *NVCC_FLAGS, "-o", LIB, *SOURCES, "-lcudart"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
