"""Compile the sm_100a extension (librd.so) in-tree with nvcc.

No JIT cache, no torch extension machinery: a plain shared library with the
C ABI of include/rd.h, built for `-gencode arch=compute_100a,code=sm_100a`.
Object files are kept under build/ (git-ignored) and rebuilt only when their
source or a header they include changed.
"""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "librd.so")
OBJDIR = os.path.join(HERE, "build")
CSRC = os.path.join(HERE, "csrc")
RD_H = os.path.join(ROOT, "include", "rd.h")
KERNELS = [os.path.join(CSRC, f) for f in ("rd_kernels.cuh", "rd_launch.h", "rd_gz.cuh")]
# the runtime and the kernel-instantiation units (rd_launch.h), compiled in
# parallel and linked into one shared library: source -> headers it includes
UNITS = {
    "rd_runtime.cu": KERNELS + [RD_H, os.path.join(CSRC, "rd_dist.cuh")],
    "rd_launch_tb_f32.cu": KERNELS + [os.path.join(CSRC, "rd_launch_tb.cuh")],
    "rd_launch_tb_f64.cu": KERNELS + [os.path.join(CSRC, "rd_launch_tb.cuh")],
    "rd_launch_cr.cu": KERNELS,
    "rd_launch_gz.cu": KERNELS,
}
SOURCES = [os.path.join(CSRC, f) for f in UNITS]

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


def _mtime(p: str) -> float:
    return os.path.getmtime(p) if os.path.exists(p) else -1.0


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    objs, procs = [], []
    for name, deps in UNITS.items():
        src = os.path.join(CSRC, name)
        obj = os.path.join(OBJDIR, name + ".o")
        objs.append(obj)
        newest = max(_mtime(p) for p in [src, *deps, __file__])
        if force or _mtime(obj) < newest:
            # RD_NVCC_DEFS: extra -D flags for A/B builds of kernel variants
            cmd = [nvcc(), *NVCC_FLAGS, *os.environ.get("RD_NVCC_DEFS", "").split(), "-c", "-o", obj, src]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            procs.append((subprocess.Popen(cmd), cmd, obj))
    failed = None
    for p, cmd, obj in procs:
        if p.wait() != 0:
            if os.path.exists(obj):
                os.remove(obj)
            failed = failed or subprocess.CalledProcessError(p.returncode, cmd)
    if failed:
        raise failed
    if procs or force or _mtime(LIB) < max(_mtime(o) for o in objs):
        subprocess.run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB, *objs,
                        "-lcudart", "-ldl"], check=True)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
