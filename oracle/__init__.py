"""ctypes binding to the CPU oracle ``liboracle_dilu.so`` (oracle/dilu_ref.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
bench.py's cpu_baseline / ``--impl reference`` legs, never by the product package
``paper_2503_05130_b200``.  It shares no code with the CUDA path; both consume the
same integer tables from ``dilu_inputs``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle_dilu.so")
NT = 17


def build(force: bool = False) -> str:
    srcs = [os.path.join(_HERE, n) for n in ("dilu_ref.c", "dilu_ref_profile.c", "dilu_ref_load.c")]
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
            [os.path.getmtime(x) for x in srcs] + [os.path.getmtime(os.path.join(_HERE, "dilu_ref.h"))]):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-Wall", "-shared",
                               "-fPIC", "-pthread"] + srcs + ["-lm", "-o", LIB_PATH])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        P32 = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
        P64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
        L.dilu_ref_create.restype = C.c_int32
        L.dilu_ref_create.argtypes = [P32, C.c_void_p, P32, C.c_void_p, C.POINTER(C.c_void_p)]
        L.dilu_ref_place_batch.restype = C.c_int32
        L.dilu_ref_place_batch.argtypes = [C.c_void_p, C.c_int32, P32, P32, P32, P32]
        L.dilu_ref_scale_step.restype = C.c_int32
        L.dilu_ref_scale_step.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
        L.dilu_ref_metrics.restype = C.c_int32
        L.dilu_ref_metrics.argtypes = [C.c_void_p, P64, P64]
        L.dilu_ref_snapshot.restype = C.c_int32
        L.dilu_ref_snapshot.argtypes = [C.c_void_p, C.c_int32, P32, P32]
        L.dilu_ref_slot.restype = C.c_int32
        L.dilu_ref_slot.argtypes = [C.c_void_p]
        L.dilu_ref_slot_detail.restype = C.c_int32
        L.dilu_ref_slot_detail.argtypes = [C.c_void_p, C.c_int32, C.c_int32, P64, P32, P64]
        L.dilu_ref_last_error.restype = C.c_char_p
        L.dilu_ref_last_error.argtypes = [C.c_void_p]
        L.dilu_ref_destroy.restype = None
        L.dilu_ref_destroy.argtypes = [C.c_void_p]
        L.dilu_ref_mix.restype = C.c_uint64
        L.dilu_ref_mix.argtypes = [C.c_uint64] * 5
        L.dilu_ref_cap1.restype = C.c_int64
        L.dilu_ref_cap1.argtypes = [C.c_int32] * 4
        L.dilu_ref_select_opt_gpu.restype = C.c_int32
        L.dilu_ref_select_opt_gpu.argtypes = [C.c_int32, P32, P32, P32, P32, P32] + [C.c_int32] * 9
        L.dilu_ref_vertical_row.restype = None
        L.dilu_ref_vertical_row.argtypes = [C.c_int32, P32, P32, P64, P64, P64, C.c_int64, P64]
        L.dilu_ref_scaling_decision.restype = C.c_int32
        L.dilu_ref_scaling_decision.argtypes = [C.c_int32, P32, C.c_int32, C.c_int64, C.c_int32,
                                                C.c_int32, C.c_int32, C.POINTER(C.c_int32)]
        L.dilu_ref_llm_split.restype = C.c_int32
        L.dilu_ref_llm_split.argtypes = [C.c_int32, P32, P32, P32, P32, P32, P32] + [C.c_int32] * 7 + [P32, P32]
        L.dilu_ref_latency.restype = C.c_int32
        L.dilu_ref_latency.argtypes = [C.c_void_p, P64, P64]
        L.dilu_ref_lat_bucket.restype = C.c_int32
        L.dilu_ref_lat_bucket.argtypes = [C.c_int64]
        L.dilu_ref_instance_latency.restype = None
        L.dilu_ref_instance_latency.argtypes = [C.c_int64] * 6 + [P64]
        L.dilu_ref_load_batch.restype = None
        L.dilu_ref_load_batch.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]
        L.dilu_ref_profile_batch.restype = None
        L.dilu_ref_profile_batch.argtypes = [C.c_int32, C.c_void_p, C.c_void_p]
        L.dilu_ref_infer_exec_ms.restype = C.c_double
        L.dilu_ref_infer_exec_ms.argtypes = [C.c_void_p, C.c_int32, C.c_double]
        L.dilu_ref_train_tput.restype = C.c_double
        L.dilu_ref_train_tput.argtypes = [C.c_void_p, C.c_double]
        L.dilu_ref_alg2_row.restype = None
        L.dilu_ref_alg2_row.argtypes = [C.c_int32, P32, P32, P32, P32, P64, P32, C.c_int32,
                                        C.c_int32, P32, P32, P64, P32]
        _lib = L
    return _lib


A2_STATES = {0: "NONE", 1: "EMERGENCY", 2: "RECOVERY", 3: "CONTENTION"}


def alg2_row(prio, ids, req_p, lim_p, d, cst, NP, p0=0, res_state=None, gpu_state=None):
    """NP periods of literal Algorithm 2 on one GPU row (dilu_ref_alg2_row).
    res_state: int32 [n][4] (t_cur, t_min, r_last, last_exec), updated in place;
    gpu_state: int32 [3] (state, owner, owner_dt), updated in place.
    Returns (exec [n] int64, grants [NP][n] int32)."""
    n = len(prio)
    a = lambda x, t=np.int32: np.ascontiguousarray(np.asarray(x, dtype=t).reshape(-1))
    if res_state is None:
        res_state = np.tile(np.array([0, 0, 0, -(1 << 30)], np.int32), (n, 1))
    if gpu_state is None:
        gpu_state = np.array([0, -1, 0], np.int32)
    rs = a(res_state)
    gs = a(gpu_state)
    ex = np.zeros(max(n, 1), np.int64)
    gr = np.zeros(max(NP * n, 1), np.int32)
    lib().dilu_ref_alg2_row(n, a(prio), a(ids), a(req_p), a(lim_p), a(d, np.int64), a(cst), NP,
                            p0, rs, gs, ex, gr)
    res_state[...] = rs.reshape(np.shape(res_state))
    gpu_state[...] = gs.reshape(np.shape(gpu_state))
    return ex[:n], gr[:NP * n].reshape(NP, n)


NLAT = 82


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


class RefSim:
    """One oracle handle over a ``dilu_inputs.Workload`` (all scenarios)."""

    def __init__(self, wl, flags: Optional[int] = None):
        self.wl = wl
        cfg = dict(wl.cfg)
        if flags is not None:
            cfg["flags"] = flags
        from dilu_inputs import CONFIG_FIELDS
        self._cfg = np.array([cfg[k] for k in CONFIG_FIELDS], dtype=np.int32)
        self._scen = np.ascontiguousarray(wl.scen, dtype=np.int32)
        self._funcs = np.ascontiguousarray(wl.funcs, dtype=np.int32)
        self._pat = np.ascontiguousarray(wl.patterns, dtype=np.int32)
        h = C.c_void_p()
        rc = lib().dilu_ref_create(self._cfg, self._scen.ctypes.data, self._funcs,
                                   self._pat.ctypes.data, C.byref(h))
        if rc != 0:
            raise OracleError(rc, "create failed (see stderr)")
        self.h = h

    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(rc, lib().dilu_ref_last_error(self.h).decode())

    def place_batch(self, req_scenario, req_func) -> Tuple[np.ndarray, np.ndarray]:
        rs = np.ascontiguousarray(req_scenario, dtype=np.int32)
        rf = np.ascontiguousarray(req_func, dtype=np.int32)
        og = np.full(rs.size, -2, dtype=np.int32)
        oi = np.full(rs.size, -2, dtype=np.int32)
        self._check(lib().dilu_ref_place_batch(self.h, rs.size, rs, rf, og, oi))
        return og, oi

    def scale_step(self, n_slots: int, threads: int = 1):
        self._check(lib().dilu_ref_scale_step(self.h, n_slots, threads))

    def metrics(self) -> Tuple[np.ndarray, np.ndarray]:
        per = np.zeros((self.wl.S, NT), dtype=np.int64)
        tot = np.zeros(NT, dtype=np.int64)
        self._check(lib().dilu_ref_metrics(self.h, per.reshape(-1), tot))
        return per, tot

    def latency(self) -> Tuple[np.ndarray, np.ndarray]:
        """Request-level latency vectors [S][82] and their sum (cfg.flags bit3)."""
        per = np.zeros((self.wl.S, NLAT), dtype=np.int64)
        tot = np.zeros(NLAT, dtype=np.int64)
        self._check(lib().dilu_ref_latency(self.h, per.reshape(-1), tot))
        return per, tot

    def snapshot(self, id_cap: int) -> Tuple[np.ndarray, np.ndarray]:
        gpu = np.zeros((self.wl.S, self.wl.G, 4), dtype=np.int32)
        inst = np.zeros((self.wl.S, id_cap, 12), dtype=np.int32)
        self._check(lib().dilu_ref_snapshot(self.h, id_cap, gpu.reshape(-1), inst.reshape(-1)))
        return gpu, inst

    def slot_detail(self, scenario: int, id_cap: int):
        a = np.zeros((id_cap, 4), dtype=np.int64)
        r = np.zeros(id_cap, dtype=np.int32)
        ex = np.zeros(self.wl.G, dtype=np.int64)
        self._check(lib().dilu_ref_slot_detail(self.h, scenario, id_cap, a.reshape(-1), r, ex))
        return a, r, ex

    @property
    def slot(self) -> int:
        return lib().dilu_ref_slot(self.h)

    def close(self):
        if getattr(self, "h", None):
            lib().dilu_ref_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run(wl, n_slots: Optional[int] = None, threads: int = 1, flags: Optional[int] = None):
    """Run a workload for n_slots (default: its whole trace); return (per, sum)."""
    s = RefSim(wl, flags=flags)
    s.scale_step(wl.n_slots if n_slots is None else n_slots, threads)
    out = s.metrics()
    s.close()
    return out


def profile_batch(sessions):
    """The profiler oracle over a ``dilu_inputs.PROF_SESSION`` array; returns a
    ``dilu_inputs.PROF_OUT`` array."""
    import dilu_inputs as di
    ses = np.ascontiguousarray(sessions, dtype=di.PROF_SESSION)
    out = np.zeros(len(ses), dtype=di.PROF_OUT)
    lib().dilu_ref_profile_batch(len(ses), ses.ctypes.data, out.ctypes.data)
    return out


def infer_exec_ms(session, ibs: int, smr: float) -> float:
    import dilu_inputs as di
    s = np.ascontiguousarray(np.asarray(session, dtype=di.PROF_SESSION).reshape(1))
    return lib().dilu_ref_infer_exec_ms(s.ctypes.data, ibs, smr)


def train_tput(session, smr: float) -> float:
    import dilu_inputs as di
    s = np.ascontiguousarray(np.asarray(session, dtype=di.PROF_SESSION).reshape(1))
    return lib().dilu_ref_train_tput(s.ctypes.data, smr)


def lat_bucket(L: int) -> int:
    return int(lib().dilu_ref_lat_bucket(int(L)))


def instance_latency(r, ibs, b, e, slo_us, T_us):
    lat = np.zeros(NLAT, dtype=np.int64)
    lib().dilu_ref_instance_latency(int(r), int(ibs), int(b), int(e), int(slo_us), int(T_us), lat)
    return lat


def load_profiles(catalog, prof_out, slot_ms: int):
    """The a0 loader oracle: ``dilu_inputs.CATALOG_ROW`` rows + ``PROF_OUT`` rows ->
    (int32 [n, 16] function rows, int32 [n] status)."""
    cat = np.ascontiguousarray(catalog)
    pr = np.ascontiguousarray(prof_out)
    n = len(cat)
    assert len(pr) == n
    rows = np.zeros((n, 16), dtype=np.int32)
    st = np.zeros(n, dtype=np.int32)
    lib().dilu_ref_load_batch(n, cat.ctypes.data, pr.ctypes.data, int(slot_ms), rows.ctypes.data,
                              st.ctypes.data)
    return rows, st
