"""Builds liblpsim.so in-tree for sm_100a (nvcc), so it travels to the GPU box."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRCS = [os.path.join(HERE, "csrc", f) for f in ("lpsim_capi.cu", "lpsim_step.cu", "lpsim_partition.cpp")]
DEPS = SRCS + [os.path.join(HERE, "csrc", f) for f in ("lpsim_dev.h", "lpsim_kernels.h")] + [
    os.path.join(ROOT, "include", "lpsim.h")]
OUT = os.path.join(HERE, "liblpsim.so")

NVCC_FLAGS = [
    "-shared", "-Xcompiler", "-fPIC", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
    "--fmad=false",  # fixed fp32 operation order, no FMA contraction
    "-std=c++17", "-diag-suppress", "550,177",
]


def nvcc() -> str:
    for p in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if p and (os.path.exists(p) or p == "nvcc"):
            return p
    return "nvcc"


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= max(os.path.getmtime(d) for d in DEPS):
        return OUT
    tmp = OUT + ".tmp%d" % os.getpid()
    extra = os.environ.get("LPSIM_NVCC_EXTRA", "").split()  # experiments, e.g. -DLPSIM_MINB=4
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I" + os.path.join(ROOT, "include"), *SRCS, "-o", tmp]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
