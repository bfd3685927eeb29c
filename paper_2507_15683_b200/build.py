"""Build libgs.so (the C-ABI library of include/gs.h) for sm_100a with nvcc.

gs_project.cu is compiled with -fmad=false (no FMA contraction) so its
pinned fp32 expressions round exactly as written; every
translation unit uses IEEE division / square root and keeps denormals
(no --use_fast_math).  The library is built in-tree so it travels to the GPU
box with the repository snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libgs.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", INCLUDE,
          "-ftz=false", "-prec-div=true", "-prec-sqrt=true", "--expt-relaxed-constexpr"]
SOURCES = {
    "gs_api.cu": [],
    "gs_project.cu": ["-fmad=false"],
    "gs_bin_sort.cu": [],
    "gs_rasterize.cu": [],
    "gs_backproject.cu": [],
    "gs_visibility.cu": [],
    "gs_match.cu": [],
    "gs_pose.cu": [],
    "gs_ssim.cu": [],
}
HEADERS = [os.path.join(INCLUDE, "gs.h"), os.path.join(CSRC, "gs_common.cuh"), os.path.join(CSRC, "gs_tc.cuh")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    for src, extra in SOURCES.items():
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s, *HEADERS, __file__]):
            cmd = [NVCC, *ARCH, *COMMON, *extra, "-c", s, "-o", o]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
                print(" ".join(cmd), file=sys.stderr)
            subprocess.check_call(cmd)
    if force or _stale(LIB, objs):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"])
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
