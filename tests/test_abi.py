"""CPU-side checks of the boundary: libdilu.so builds for sm_100a, loads, and exports
every function include/dilu.h declares; the ABI struct sizes match the generator's
field lists; the product package never imports the oracle."""
import ast
import os
import re

import numpy as np
import pytest

import dilu_inputs as di

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "dilu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(dilu_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2503_05130_b200 import _build
    import ctypes
    path = _build.build()
    L = ctypes.CDLL(path)
    names = header_functions()
    assert "dilu_sim_create" in names and "dilu_scale_step" in names
    for n in names:
        assert hasattr(L, n), n
    import paper_2503_05130_b200 as pkg
    assert sorted(pkg.EXPORTED) == names


def test_struct_field_counts_match_header():
    src = open(os.path.join(ROOT, "include", "dilu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)

    def fields(name):
        body = re.search(r"typedef struct \{([^{}]*)\}\s*" + name + ";", src).group(1)
        return sum(len(d.split(",")) for d in re.findall(r"int32_t\s+([^;]+);", body))
    assert fields("dilu_config") == len(di.CONFIG_FIELDS)
    assert fields("dilu_func") == len(di.FUNC_FIELDS)
    assert fields("dilu_scenario") == len(di.SCEN_FIELDS)


def test_workspace_bytes_and_validation_without_gpu():
    import numpy as np
    import paper_2503_05130_b200 as pkg
    wl = di.c4(n_scenarios=8, T=100)
    n = pkg.dilu_workspace_bytes(wl.cfg_array())
    assert n > 0 and n % 256 == 0
    bad = wl.cfg_array().copy()
    bad[di.CONFIG_FIELDS.index("q_pm")] = 999
    assert pkg.dilu_workspace_bytes(bad) == 0


def test_product_package_does_not_touch_oracle():
    pkg_dir = os.path.join(ROOT, "paper_2503_05130_b200")
    for dp, _, files in os.walk(pkg_dir):
        for fn in files:
            p = os.path.join(dp, fn)
            if fn.endswith(".py"):
                tree = ast.parse(open(p).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert all(not a.name.startswith("oracle") for a in node.names), p
                    if isinstance(node, ast.ImportFrom):
                        assert not (node.module or "").startswith("oracle"), p
            if fn.endswith((".cu", ".cuh", ".h")):
                assert "dilu_ref" not in open(p).read(), p


def test_profiler_struct_layouts_match_header():
    """dilu_prof_session / dilu_prof_out (include/dilu.h) and the generator's dtypes have
    the same fields in the same order and size (both sides read the same bytes)."""
    src = open(os.path.join(ROOT, "include", "dilu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)

    def names(struct):
        body = re.search(r"typedef struct \{([^{}]*)\}\s*" + struct + ";", src).group(1)
        out = []
        for typ, decl in re.findall(r"(int32_t|double)\s+([^;]+);", body):
            out += [(typ, n.strip()) for n in decl.split(",")]
        return out
    for struct, dt in (("dilu_prof_session", di.PROF_SESSION), ("dilu_prof_out", di.PROF_OUT)):
        fs = names(struct)
        assert [n for _, n in fs] == list(dt.names), struct
        for (typ, n) in fs:
            assert dt[n] == (np.dtype("<i4") if typ == "int32_t" else np.dtype("<f8")), (struct, n)


def test_abi_argument_errors_without_gpu():
    """Argument validation that needs no device: dilu_profile rejects n < 0 and null or
    misaligned pointers; the latency / Alg.2 flags are validated with the config."""
    import ctypes
    import paper_2503_05130_b200 as pkg
    L = pkg.lib()
    assert L.dilu_profile(None, -1, None, None) == 1
    assert L.dilu_profile(None, 5, None, None) == 1
    assert L.dilu_profile(ctypes.c_void_p(8), 1, ctypes.c_void_p(12), None) == 1
    assert L.dilu_profile(None, 0, None, None) == 0
    wl = di.c1()
    cfg = wl.cfg_array().copy()
    cfg[di.CONFIG_FIELDS.index("flags")] |= 4 | 8
    assert pkg.dilu_workspace_bytes(cfg) > 0                     # 1 s slots: fine
    cfg[di.CONFIG_FIELDS.index("slot_ms")] = 8                   # not a multiple of 5
    assert pkg.dilu_workspace_bytes(cfg) == 0


def test_bench_refuses_more_gpus_than_visible():
    """bench.py --gpus N outside torchrun spawns N ranks itself, and refuses clearly (exit
    2, message) when fewer than N GPUs are visible (a 1-GPU --gpus 2 run must
    not silently time one GPU)."""
    import subprocess, sys, os, torch
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    n = torch.cuda.device_count()
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", str(n + 1)],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 2
    assert "visible GPUs" in r.stderr
