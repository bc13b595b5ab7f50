"""Compile libdilu.so for sm_100a in-tree (nvcc cross-compiles without a GPU).

Nine translation units compile in parallel: dilu_api.cu (C-ABI, init / snapshot /
profiler kernels) and run_variants.cu eight times (DILU_VGROUP = 0..3, two of the
eight kernel variants each, x DILU_HOT_SMEM = 1 for the shared-memory kernels / 0 for the
global-memory and cluster kernels); one nvcc link makes the shared library.
`python _build.py -DNAME[=v] ...` builds a side library libdilu_<name>.so with extra
defines (e.g. -DDILU_PHASE_TIMING) for experiments."""
from __future__ import annotations

import os
import subprocess
import tempfile
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libdilu.so")
CSRC = os.path.join(HERE, "csrc")
SOURCES = [os.path.join(CSRC, n) for n in ("dilu_api.cu", "run_variants.cu", "sim_kernel.cuh",
                                           "state.cuh", "profile.cuh",
                                           "variants.h")]
HEADER = os.path.join(ROOT, "include", "dilu.h")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xptxas", "-v", "-Xcompiler", "-fPIC"]


def nvcc() -> str:
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.sep not in c or os.path.exists(c):
            return c
    return "nvcc"


def build(force: bool = False, verbose: bool = False, extra=(), out: str = LIB) -> str:
    newest = max(os.path.getmtime(p) for p in SOURCES + [HEADER])
    if not force and not extra and os.path.exists(out) and os.path.getmtime(out) >= newest:
        return out
    with tempfile.TemporaryDirectory(prefix="dilu_build_") as tmp:
        units = [(os.path.join(CSRC, "dilu_api.cu"), [], "api.o")]
        units += [(os.path.join(CSRC, "run_variants.cu"), [f"-DDILU_VGROUP={g}", f"-DDILU_HOT_SMEM={h}"],
                   f"v{g}h{h}.o") for g in range(4) for h in (0, 1)]

        def compile_one(u):
            src, defs, obj = u
            cmd = [nvcc()] + NVCC_FLAGS + list(extra) + defs + ["-c", src, "-o", os.path.join(tmp, obj)]
            return subprocess.run(cmd, capture_output=True, text=True)

        with ThreadPoolExecutor(max_workers=len(units)) as ex:
            results = list(ex.map(compile_one, units))
        log = "".join(r.stderr for r in results)
        for r in results:
            if r.returncode != 0:
                raise RuntimeError("nvcc failed:\n" + r.stderr)
        link = [nvcc()] + ARCH + ["-shared", "-o", out] + [os.path.join(tmp, u[2]) for u in units]
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc link failed:\n" + r.stderr)
    if verbose:
        print(log)
    return out


if __name__ == "__main__":
    import sys
    verbose = "verbose" in sys.argv or "-v" in sys.argv
    extra = [a for a in sys.argv[1:] if a.startswith("-D")]
    out = LIB if not extra else os.path.join(HERE, "libdilu_" + "_".join(
        e[2:].lower().replace("=", "_") for e in extra) + ".so")
    print(build(force=True, verbose=verbose, extra=extra, out=out))
