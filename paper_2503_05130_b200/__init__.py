"""B200-native batched Dilu provisioning loop (arXiv 2503.05130).

A thin ctypes binding over ``libdilu.so`` (include/dilu.h): argument marshalling
only.  Every step of the provisioning loop runs in the CUDA kernels of
``csrc/``; PyTorch supplies device memory (the workspace and request/output
tensors), the CUDA stream, and the NCCL process group (``dist.py``).  There is no
CPU fallback: importing works without a GPU, but creating a simulation raises if
the extension or the device is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DILU_LIB", os.path.join(HERE, "libdilu.so"))  # override: experiments
NT = 17
DILU_OK, DILU_E_USAGE, DILU_E_INVARIANT, DILU_E_IO, DILU_E_CUDA, DILU_E_STATE, DILU_E_CAPACITY = range(7)

_lib = None


class DiluError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"dilu status {code}: {msg}")
        self.code = code


def lib():
    """Load libdilu.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() "
                              "(no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64p = C.c_void_p, C.c_int32, C.POINTER(C.c_int64)
        L.dilu_workspace_bytes.restype = C.c_size_t
        L.dilu_workspace_bytes.argtypes = [vp]
        L.dilu_sim_create.restype = i32
        L.dilu_sim_create.argtypes = [vp, vp, vp, vp, vp, C.c_size_t, vp, C.POINTER(vp)]
        L.dilu_sim_reset.restype = i32
        L.dilu_sim_reset.argtypes = [vp]
        L.dilu_place_batch.restype = i32
        L.dilu_place_batch.argtypes = [vp, i32, vp, vp, vp, vp]
        L.dilu_scale_step.restype = i32
        L.dilu_scale_step.argtypes = [vp, i32]
        L.dilu_metrics.restype = i32
        L.dilu_metrics.argtypes = [vp, vp, vp]
        L.dilu_snapshot.restype = i32
        L.dilu_snapshot.argtypes = [vp, i32, vp, vp]
        L.dilu_kernel_stats.restype = i32
        L.dilu_kernel_stats.argtypes = [vp, vp, vp]
        L.dilu_current_slot.restype = i32
        L.dilu_current_slot.argtypes = [vp]
        L.dilu_last_error.restype = C.c_char_p
        L.dilu_last_error.argtypes = [vp]
        L.dilu_sim_destroy.restype = None
        L.dilu_sim_destroy.argtypes = [vp]
        L.dilu_latency.restype = i32
        L.dilu_latency.argtypes = [vp, vp, vp]
        L.dilu_profile.restype = i32
        L.dilu_profile.argtypes = [vp, i32, vp, vp]
        if hasattr(L, "dilu_load_profiles"):   # (older side libraries in A/B runs lack it)
            L.dilu_load_profiles.restype = i32
            L.dilu_load_profiles.argtypes = [vp, vp, i32, i32, vp, vp, vp]
        _lib = L
    return _lib


EXPORTED = ["dilu_workspace_bytes", "dilu_sim_create", "dilu_sim_reset", "dilu_place_batch",
            "dilu_scale_step", "dilu_metrics", "dilu_snapshot", "dilu_kernel_stats",
            "dilu_current_slot",
            "dilu_last_error", "dilu_sim_destroy", "dilu_profile", "dilu_latency",
            "dilu_load_profiles"]


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def dilu_workspace_bytes(cfg: np.ndarray) -> int:
    cfg = _i32(cfg)
    return int(lib().dilu_workspace_bytes(cfg.ctypes.data))


class DiluSim:
    """One handle over all scenarios of a workload on one device.

    cfg/scen/funcs/patterns are the flat int32 host tables of include/dilu.h (the
    ``dilu_inputs`` generator writes them).  All device buffers are torch tensors."""

    def __init__(self, cfg: np.ndarray, scen: Optional[np.ndarray], funcs: np.ndarray,
                 patterns: np.ndarray, device="cuda", stream=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("DiluSim needs a CUDA device (no CPU fallback)")
        self.torch = torch
        self.device = torch.device(device)
        self._cfg = _i32(cfg)
        self.S = int(self._cfg[0])
        self.G = int(self._cfg[1])
        self._scen = None if scen is None else _i32(scen)
        self._funcs = _i32(funcs)
        self._pat = _i32(patterns)
        nbytes = dilu_workspace_bytes(self._cfg)
        if nbytes == 0:
            raise DiluError(DILU_E_USAGE, "invalid config")
        with torch.cuda.device(self.device):
            self.stream = stream or torch.cuda.current_stream(self.device)
            self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            h = C.c_void_p()
            rc = lib().dilu_sim_create(self._cfg.ctypes.data,
                                       None if self._scen is None else self._scen.ctypes.data,
                                       self._funcs.ctypes.data, self._pat.ctypes.data,
                                       self.workspace.data_ptr(), nbytes,
                                       self.stream.cuda_stream, C.byref(h))
        if rc != DILU_OK:
            raise DiluError(rc, "dilu_sim_create failed (see stderr)")
        self.h = h

    @classmethod
    def from_workload(cls, wl, device="cuda", stream=None) -> "DiluSim":
        return cls(wl.cfg_array(), wl.scen, wl.funcs, wl.patterns, device=device, stream=stream)

    def _check(self, rc: int):
        if rc != DILU_OK:
            raise DiluError(rc, lib().dilu_last_error(self.h).decode())

    def reset(self):
        self._check(lib().dilu_sim_reset(self.h))

    def place_batch(self, req_scenario, req_func):
        """Explicit deployment requests (device int32 tensors or array-likes)."""
        t = self.torch
        rs = t.as_tensor(req_scenario, dtype=t.int32, device=self.device).contiguous()
        rf = t.as_tensor(req_func, dtype=t.int32, device=self.device).contiguous()
        og = t.full_like(rs, -2)
        oi = t.full_like(rs, -2)
        self._check(lib().dilu_place_batch(self.h, rs.numel(), rs.data_ptr(), rf.data_ptr(),
                                           og.data_ptr(), oi.data_ptr()))
        return og, oi

    def scale_step(self, n_slots: int):
        self._check(lib().dilu_scale_step(self.h, int(n_slots)))

    def metrics(self, per_scenario: bool = True, host: bool = False):
        """(per-scenario int64 [S,17] or None, scenario-sum int64 [17])."""
        t = self.torch
        dev = "cpu" if host else self.device
        per = t.zeros((self.S, NT), dtype=t.int64, device=dev) if per_scenario else None
        tot = t.zeros(NT, dtype=t.int64, device=dev)
        if host:
            tot = tot.pin_memory()
            per = per.pin_memory() if per is not None else None
        self._check(lib().dilu_metrics(self.h, None if per is None else per.data_ptr(),
                                       tot.data_ptr()))
        return per, tot

    def snapshot(self, id_cap: int):
        t = self.torch
        gpu = t.zeros((self.S, self.G, 4), dtype=t.int32, device=self.device)
        inst = t.zeros((self.S, max(id_cap, 1), 12), dtype=t.int32, device=self.device)
        self._check(lib().dilu_snapshot(self.h, int(id_cap), gpu.data_ptr(), inst.data_ptr()))
        return gpu, inst[:, :id_cap]

    STAT_NAMES = ["attempts", "retry_checks", "row_repacks", "boundary_events", "queue_scans",
                  "slots", "resident_slots", "function_slots", "cyc_pre_boundary", "cyc_boundary",
                  "cyc_repack", "cyc_p0", "cyc_p1", "cyc_p2", "cyc_b3", "cyc_terminate",
                  "cyc_enqueue", "cyc_next_attempt", "cyc_place", "t19", "t20", "t21", "t22", "t23"]

    def kernel_stats(self):
        """Diagnostics: dict of summed kernel counters (dilu_kernel_stats); the cyc_*
        phase timers are filled only by a -DDILU_PHASE_TIMING build."""
        tot = np.zeros(24, dtype=np.int64)
        self._check(lib().dilu_kernel_stats(self.h, None, tot.ctypes.data))
        return dict(zip(self.STAT_NAMES, tot.tolist()))

    NLAT = 82

    def latency(self):
        """Request-level latency vectors (dilu_latency; cfg.flags bit3): (per-scenario
        [S][82] int64 numpy, sum [82])."""
        per = np.zeros((self.S, self.NLAT), dtype=np.int64)
        tot = np.zeros(self.NLAT, dtype=np.int64)
        self._check(lib().dilu_latency(self.h, per.ctypes.data, tot.ctypes.data))
        return per, tot

    @property
    def slot(self) -> int:
        return int(lib().dilu_current_slot(self.h))

    def close(self):
        if getattr(self, "h", None):
            lib().dilu_sim_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


PROF_SESSION_BYTES, PROF_OUT_BYTES = 104, 48


def dilu_profile(sessions, out=None, stream=None):
    """Batched profiler (dilu_profile).  ``sessions``: a uint8 CUDA tensor
    of n * 104 bytes (rows laid out as dilu_prof_session, e.g. a dilu_inputs.PROF_SESSION
    array copied to the device); returns (or fills) a uint8 CUDA tensor of n * 48 bytes
    (dilu_prof_out rows).  Asynchronous on ``stream`` (default: the current stream)."""
    import torch
    if not (isinstance(sessions, torch.Tensor) and sessions.is_cuda and sessions.dtype == torch.uint8):
        raise TypeError("sessions must be a uint8 CUDA tensor of dilu_prof_session rows")
    n = sessions.numel() // PROF_SESSION_BYTES
    if sessions.numel() != n * PROF_SESSION_BYTES:
        raise ValueError("sessions size is not a multiple of 104 bytes")
    if out is None:
        out = torch.empty(n * PROF_OUT_BYTES, dtype=torch.uint8, device=sessions.device)
    if stream is None:
        stream = torch.cuda.current_stream(sessions.device)
    rc = lib().dilu_profile(sessions.data_ptr(), n, out.data_ptr(), stream.cuda_stream)
    if rc:
        raise DiluError(rc, "dilu_profile failed")
    return out


CATALOG_ROW_BYTES, FUNC_ROW_BYTES = 72, 64


def dilu_load_profiles(catalog, prof_out, slot_ms: int, stream=None):
    """Profile-table loader (dilu_load_profiles): ``catalog`` a uint8 CUDA
    tensor of n * 72 bytes (dilu_catalog_row rows), ``prof_out`` the n * 48-byte
    dilu_profile output of their sessions.  Returns (rows: int32 CUDA tensor [n, 16] =
    dilu_func rows, status: int32 CUDA tensor [n]).  Asynchronous on ``stream``."""
    import torch
    for t, w in ((catalog, CATALOG_ROW_BYTES), (prof_out, PROF_OUT_BYTES)):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.uint8):
            raise TypeError("catalog / prof_out must be uint8 CUDA tensors")
    n = catalog.numel() // CATALOG_ROW_BYTES
    if catalog.numel() != n * CATALOG_ROW_BYTES or prof_out.numel() != n * PROF_OUT_BYTES:
        raise ValueError("catalog / prof_out sizes do not describe the same n rows")
    rows = torch.empty((n, 16), dtype=torch.int32, device=catalog.device)
    st = torch.empty(n, dtype=torch.int32, device=catalog.device)
    if stream is None:
        stream = torch.cuda.current_stream(catalog.device)
    rc = lib().dilu_load_profiles(catalog.data_ptr(), prof_out.data_ptr(), n, int(slot_ms),
                                  rows.data_ptr(), st.data_ptr(), stream.cuda_stream)
    if rc:
        raise DiluError(rc, "dilu_load_profiles failed")
    return rows, st


def lat_bucket_bounds(b: int):
    """[lo, hi) in microseconds of latency bucket b (D10), hi = inf for 79."""
    if b >= 79:
        return float("inf"), float("inf")
    if b < 4:
        return float(b), float(b + 1)
    h, sub = (b + 4) // 4, (b + 4) % 4
    lo = (1 << h) + sub * (1 << (h - 2))
    return float(lo), float(lo + (1 << (h - 2)))


def latency_summary(lat) -> dict:
    """p50 / p95 / p99 (upper bucket bounds, ms), mean served latency and latency SVR
    from a dilu_latency vector (reporting only: the histogram itself is the GPU's)."""
    lat = np.asarray(lat, dtype=np.int64)
    hist = lat[:80]
    n = int(hist.sum())
    served = int(hist[:79].sum())
    out = {"requests": n, "served": served,
           "latency_svr": float(lat[80]) / n if n else 0.0,
           "mean_ms": float(lat[81]) / served / 1000.0 if served else None}
    cum = np.cumsum(hist)
    cum_s = np.cumsum(hist[:79])
    for q in (50, 95, 99):
        # over all requests: an unserved request (capacity, bucket 79) has infinite latency,
        # so the percentile is undefined (None) once more than (100 - q) % are unserved
        if n == 0:
            out[f"p{q}_ms"] = None
        else:
            b = int(np.searchsorted(cum, q / 100.0 * n, side="left"))
            hi = lat_bucket_bounds(b)[1]
            out[f"p{q}_ms"] = hi / 1000.0 if hi != float("inf") else None
        # over the served requests only (always defined when any request was served)
        if served == 0:
            out[f"p{q}_served_ms"] = None
        else:
            b = int(np.searchsorted(cum_s, q / 100.0 * served, side="left"))
            out[f"p{q}_served_ms"] = lat_bucket_bounds(b)[1] / 1000.0
    out["unserved_fraction"] = float(lat[79]) / n if n else 0.0
    return out
