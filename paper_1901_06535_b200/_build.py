"""Compile the sm_100a extension (librd.so) in-tree with nvcc.

No JIT cache, no torch extension machinery: a plain shared library with the
C ABI of include/rd.h, built for `-gencode arch=compute_100a,code=sm_100a`.
"""
from __future__ import annotations

import glob
import os
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "librd.so")
# the runtime and the kernel-instantiation units (rd_launch.h), compiled in
# parallel and linked into one shared library
SOURCES = [os.path.join(HERE, "csrc", f) for f in
           ("rd_runtime.cu", "rd_launch_tb_f32.cu", "rd_launch_tb_f64.cu", "rd_launch_cr.cu")]
DEPS = sorted(glob.glob(os.path.join(HERE, "csrc", "*")) + [os.path.join(ROOT, "include", "rd.h")])

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xfatbin", "-compress-all",
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
    with tempfile.TemporaryDirectory() as tmp:
        objs, procs = [], []
        for src in SOURCES:
            obj = os.path.join(tmp, os.path.basename(src) + ".o")
            cmd = [nvcc(), *NVCC_FLAGS, "-c", "-o", obj, src]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            procs.append((subprocess.Popen(cmd), cmd))
            objs.append(obj)
        for p, cmd in procs:
            if p.wait() != 0:
                raise subprocess.CalledProcessError(p.returncode, cmd)
        subprocess.run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB, *objs,
                        "-lcudart"], check=True)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
