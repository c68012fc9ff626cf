"""Builds paper_1405_0562_b200/_lib/libsfa.so (the C-ABI of include/sfa.h).

nvcc for sm_100a only (``-gencode arch=compute_100a,code=sm_100a``), in-tree,
``-lineinfo`` so ncu's source page maps to csrc/.  Cross-compiles on a box
without a GPU.  Rebuilds only when a source is newer than the library.
"""
from __future__ import annotations

import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIBDIR, "libsfa.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["api.cpp", "compile.cpp", "kernels.cu", "kernels_private.cu", "kernels_shared.cu", "kernels_global.cu",
           "kernels_hot.cu", "kernels_private_seg.cu", "kernels_shared_seg.cu", "kernels_global_seg.cu",
           "kernels_hot_seg.cu", "kernels_spec.cu", "kernels_lazy.cu", "lazy.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden", "--expt-relaxed-constexpr"]


def _inputs():
    return ([os.path.join(CSRC, s) for s in SOURCES] + glob.glob(os.path.join(CSRC, "*.hpp"))
            + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "sfa.h"), __file__])


DIAG_LIB = os.path.join(LIBDIR, "libsfa_diag.so")


def build(force: bool = False, verbose: bool = False, diag: bool = False, counters: bool = False) -> str:
    """diag: the diagnostic library (-DSFA_STAMPS: per-CTA phase stamps of the
    TMA scan, sfa_diag_stamps) -- never loaded by the product, tests or bench."""
    os.makedirs(LIBDIR, exist_ok=True)
    LIB = DIAG_LIB if diag else globals()["LIB"]
    if not force and os.path.exists(LIB):
        newest = max(os.path.getmtime(p) for p in _inputs())
        if os.path.getmtime(LIB) >= newest:
            return LIB
    objs, cmds = [], []
    for src_name in SOURCES:
        src = os.path.join(CSRC, src_name)
        obj = os.path.join(LIBDIR, src_name + f".{os.getpid()}{'.diag' if diag else ''}.o")
        extra = (["-DSFA_STAMPS"] if diag else []) + (["-DSFA_COUNTERS"] if diag and counters else [])
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", src, "-o", obj]
        if src_name.endswith(".cu") and verbose:
            cmd[1:1] = ["-Xptxas", "-v"]
        if verbose:
            print(" ".join(cmd))
        cmds.append(cmd)
        objs.append(obj)
    # one nvcc per translation unit, in parallel (the kernels are split by step policy)
    try:
        with ThreadPoolExecutor(max_workers=len(cmds)) as ex:
            for f in [ex.submit(subprocess.check_call, c) for c in cmds]:
                f.result()
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-ldl", "-lrt",
                               "-lpthread"])
        os.replace(tmp, LIB)
    finally:  # an interrupted or failed build leaves no objects behind
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
    return LIB


if __name__ == "__main__":
    import sys
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, diag="--diag" in sys.argv,
                counters="--counters" in sys.argv))
