"""Builds libalphax_b200.so (hand-written CUDA, sm_100a) in-tree with nvcc.

    python -m paper_1908_05944_b200.build [--force]

nvcc cross-compiles without a GPU.  ``-fmad=false`` is part of the numerical
contract (csrc/predicates.cuh): the device arithmetic must round exactly like
the reference's numpy expressions.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libalphax_b200.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-std=c++17", "-lineinfo",
    "-fmad=false",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math",
    "-shared",
]


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh"))) + [
        os.path.join(os.path.dirname(HERE), "include", "alphax_b200.h")]


def is_stale() -> bool:
    if not os.path.exists(LIB):
        return True
    built = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > built for s in _sources())


def build_native(force: bool = False, verbose: bool = False) -> str:
    if not force and not is_stale():
        return LIB
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        raise RuntimeError("nvcc not found; cannot build libalphax_b200.so")
    extra = os.environ.get("AXB_NVCC_EXTRA", "").split()       # e.g. -DAXB_AC2_VARIANT=2 for A/B builds
    cmd = [nvcc, *NVCC_FLAGS, *extra, "-o", LIB, os.path.join(CSRC, "alphax_b200.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build_native(force="--force" in sys.argv, verbose="-v" in sys.argv))
