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
SOURCES = [os.path.join(CSRC, "arc_kernels.cu"), os.path.join(CSRC, "arc_sketch.cu"), os.path.join(CSRC, "arc_sketch_tma.cu"),
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


def build(force: bool = False, verbose: bool = False, extra: list[str] | None = None, out: str | None = None) -> str:
    """extra / out: additional nvcc flags and another output path (A/B variants, tools/build_variant.sh)."""
    target = out or LIB
    if out is None and not force and not needs_build():
        return LIB
    tmp = target + f".tmp{os.getpid()}"
    inc = ["-I", os.path.join(ROOT, "include"), "-I", _nccl_include()]
    compile_flags = [f for f in NVCC_FLAGS if f not in ("-shared", "-cudart", "static")]
    objdir = os.path.join(PKG, "build_obj", str(os.getpid()))
    os.makedirs(objdir, exist_ok=True)
    # one nvcc per source, in parallel (the kernel files take minutes each), then one link
    jobs = []
    for src in SOURCES:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [_nvcc(), *compile_flags, *(extra or []), *(["-Xptxas=-v"] if verbose else []), *inc, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        jobs.append((obj, subprocess.Popen(cmd)))
    failed = [obj for obj, pr in jobs if pr.wait() != 0]
    try:
        if failed:
            raise subprocess.CalledProcessError(1, f"nvcc ({len(failed)} source(s) failed)")
        subprocess.run([_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
                        "-Xcompiler", "-fPIC", *[obj for obj, _ in jobs], "-o", tmp, "-ldl"], check=True)
    finally:
        for obj, _ in jobs:
            if os.path.exists(obj):
                os.remove(obj)
        try:
            os.rmdir(objdir)
        except OSError:
            pass
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    if "--out" in sys.argv:   # python -m paper_2510_26709_b200._build --out PATH [nvcc flags ...]
        i = sys.argv.index("--out")
        print(build(extra=sys.argv[i + 2:], out=os.path.abspath(sys.argv[i + 1])))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
