"""Build liboocgb.so in-tree for sm_100a (nvcc, -gencode arch=compute_100a,code=sm_100a).

Flags: -O3 -lineinfo (ncu source view), -fmad=false and host -ffp-contract=off (no FMA
contraction anywhere in the split/sampling arithmetic, DESIGN.md §3 R14).  NCCL (multi-GPU
histogram all-reduce) is dlopen'ed at run time, not linked.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = [os.path.join(HERE, "csrc", f) for f in ("api.cu", "quantise.cu", "sample.cu", "tree.cu")]
HDR = [os.path.join(HERE, "csrc", f) for f in ("internal.cuh", "philox.cuh", "stream.cuh")] + [
    os.path.join(HERE, "..", "include", "oocgb.h")]
OUT = os.path.join(HERE, "liboocgb.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-fmad=false", "-Xcompiler", "-fPIC,-ffp-contract=off", "-shared", "-diag-suppress", "177,550"]


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(f) <= t for f in SRC + HDR)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    tmp = OUT + f".tmp{os.getpid()}"
    extra = os.environ.get("OOCGB_EXTRA_NVCC", "").split()  # tuning experiments (-D...)
    flags = [f for f in FLAGS if not (f == "-fmad=false" and os.environ.get("OOCGB_FMAD") == "1")]
    cmd = [NVCC, *flags, *extra, "-o", tmp, *SRC, "-ldl"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
