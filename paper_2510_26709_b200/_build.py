"""Compile ``libarctopk.so`` (sm_100a) in-tree with nvcc.

Called by ``__graft_entry__.build()``; also usable as
``python -m paper_2510_26709_b200._build``.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libarctopk.so")
SOURCES = [os.path.join(CSRC, "arc_kernels.cu"), os.path.join(CSRC, "arc_sketch.cu"),
           os.path.join(CSRC, "arc_select.cu"), os.path.join(CSRC, "arc_lsa.cu"),
           os.path.join(CSRC, "arc_optim.cu"), os.path.join(CSRC, "arc_loopback.cu"),
           os.path.join(CSRC, "arc_api.cu")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # IEEE binary32 exactly as written: no FMA contraction, no flush-to-zero,
    # correctly rounded division and square root (R9, R10).
    "-fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
]


def _nccl_include() -> str:
    import nvidia.nccl  # the NCCL torch links against (types only; symbols resolved at run time)
    for base in list(getattr(nvidia.nccl, "__path__", [])):
        inc = os.path.join(base, "include")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc
    raise RuntimeError("nccl.h from the nvidia-nccl wheel not found")


def _nvcc() -> str:
    for c in [os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"]:
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = SOURCES + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        [os.path.join(ROOT, "include", "arc_topk.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [_nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-I", _nccl_include(),
           *SOURCES, "-o", tmp, "-ldl"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
