"""Compile libdilu.so for sm_100a in-tree (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libdilu.so")
SOURCES = [os.path.join(HERE, "csrc", n) for n in ("dilu_api.cu", "sim_kernel.cuh", "state.cuh", "sim_lanes.cuh", "profile.cuh")]
HEADER = os.path.join(ROOT, "include", "dilu.h")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xptxas", "-v", "-shared", "-Xcompiler", "-fPIC"]


def nvcc() -> str:
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.sep not in c or os.path.exists(c):
            return c
    return "nvcc"


def build(force: bool = False, verbose: bool = False) -> str:
    newest = max(os.path.getmtime(p) for p in SOURCES + [HEADER])
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= newest:
        return LIB
    cmd = [nvcc()] + NVCC_FLAGS + ["-o", LIB, SOURCES[0]]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + out.stderr)
    if verbose:
        print(out.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
