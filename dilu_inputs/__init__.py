"""Seeded synthetic inputs shared by the CUDA path and the CPU oracle.

This module holds NONE of the method's arithmetic (no placement, no token
allocation, no scaling rule, no capacity formula).  It only writes the integer
input tables both sides consume:

* a config row (20 int32, field order ``CONFIG_FIELDS``),
* per-scenario rows (4 int32: global scenario id, Omega, gamma, baseline mode),
* the quantised profile table (16 int32 per function row, ``FUNC_FIELDS``),
* the per-slot arrival pattern table (int32 ``[n_patterns][pattern_len]``).

The recipes follow SURVEY.md s8(d) ("Synthetic model catalogue", "Fleet
generator", "Pattern tables", "Configs restated") and are restated in DESIGN.md
s4.  Configs: C1 (Appendix A worked example), C2 (64 GPUs), C3 (1,024 GPUs),
C4 (4,096 x 64-GPU sweep), C5 (16,384 GPUs at 100 ms slots).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional

import numpy as np

CONFIG_FIELDS = [
    "n_scenarios", "gpus_per_scenario", "max_funcs", "max_instances",
    "q_pm", "mem_mib", "omega_pm", "gamma_pm", "alpha_w", "beta_w", "slot_ms",
    "window_s", "phi_out", "phi_in", "min_instances", "max_residents", "max_llm_stages",
    "n_patterns", "pattern_len", "flags",
]
FUNC_FIELDS = [
    "kind", "prio", "ibs", "req_pm", "lim_pm", "mem_mib", "work_per_batch", "n_workers",
    "duty_pm", "cold_slots", "affinity_class", "arrive_sec", "depart_sec",
    "pattern", "scale_q10", "phase_slots",
]
SCEN_FIELDS = ["scenario_id", "omega_pm", "gamma_pm", "mode"]
MODES = {"dilu": 0, "exclusive": 1, "static_limit": 2, "static_request": 3, "eager_horizontal": 4}
FI = {n: i for i, n in enumerate(FUNC_FIELDS)}

NEVER = 2**31 - 1          # depart_sec for "never departs"
K_UNUSED, K_INF, K_LLM, K_TRAIN = -1, 0, 1, 2
TALLY_NAMES = [
    "gpu_slots_active", "sm_unused_tokens", "mem_unused_mib_slots", "req_total",
    "req_served", "req_violated", "inf_exec_tokens", "train_progress_tokens",
    "placements_ok", "placement_failures", "cold_starts", "scale_out_events",
    "scale_in_events", "llm_split_placements", "alloc_hash", "gpu_row_slots", "max_active",
]


def default_config(**kw) -> Dict[str, int]:
    """Defaults: Omega=1, gamma=1.5, alpha=beta, W=40, phi_out=20,
    phi_in=30, min 1 instance, 32 residents, <=4 LLM stages
    (P:1188), A100-40GB memory."""
    c = dict(n_scenarios=1, gpus_per_scenario=4, max_funcs=1, max_instances=64,
             q_pm=1000, mem_mib=40960, omega_pm=1000, gamma_pm=1500, alpha_w=1, beta_w=1,
             slot_ms=1000, window_s=40, phi_out=20, phi_in=30, min_instances=1,
             max_residents=32, max_llm_stages=4, n_patterns=0, pattern_len=1, flags=1)
    c.update(kw)
    return c


@dataclasses.dataclass
class Workload:
    name: str
    cfg: Dict[str, int]
    scen: np.ndarray          # int32 [S, 4]
    funcs: np.ndarray         # int32 [S, F, 16]
    patterns: np.ndarray      # int32 [P, T_pat]
    n_slots: int              # trace length in slots
    note: str = ""

    @property
    def S(self) -> int:
        return int(self.cfg["n_scenarios"])

    @property
    def G(self) -> int:
        return int(self.cfg["gpus_per_scenario"])

    def cfg_array(self) -> np.ndarray:
        return np.array([self.cfg[k] for k in CONFIG_FIELDS], dtype=np.int32)

    def shard(self, rank: int, world: int) -> "Workload":
        """Contiguous scenario block [r*S/P, (r+1)*S/P)."""
        lo = self.S * rank // world
        hi = self.S * (rank + 1) // world
        cfg = dict(self.cfg)
        cfg["n_scenarios"] = hi - lo
        return Workload(self.name, cfg, self.scen[lo:hi].copy(), self.funcs[lo:hi].copy(),
                        self.patterns, self.n_slots, self.note)

    def subset(self, idx) -> "Workload":
        idx = np.asarray(idx)
        cfg = dict(self.cfg)
        cfg["n_scenarios"] = int(idx.size)
        return Workload(self.name, cfg, self.scen[idx].copy(), self.funcs[idx].copy(),
                        self.patterns, self.n_slots, self.note)


def _rng(seed: int, stream: str) -> np.random.Generator:
    """Named sub-streams from one seed."""
    h = 0
    for ch in stream:
        h = (h * 131 + ord(ch)) % (2**31)
    return np.random.default_rng([seed, h])


# ------------------------------------------------ profiler sessions (s8(f) #3)
# Flat layouts shared by the profiler oracle (oracle/dilu_ref.h ref_prof_session /
# ref_prof_out) and the C-ABI (include/dilu.h dilu_prof_session / dilu_prof_out).
PROF_SESSION = np.dtype([("kind", "<i4"), ("workers", "<i4"), ("ibs_max", "<i4"),
                         ("reserved", "<i4"), ("a_ms", "<f8"), ("b_ms", "<f8"),
                         ("knee_c", "<f8"), ("knee_t", "<f8"), ("t_max", "<f8"),
                         ("idle", "<f8"), ("slo_ms", "<f8"), ("smr_step", "<f8"),
                         ("p_req", "<f8"), ("p_lim", "<f8"), ("tol", "<f8")])
PROF_OUT = np.dtype([("request_smr", "<f8"), ("limit_smr", "<f8"), ("t_exec_ms", "<f8"),
                     ("ibs", "<i4"), ("trials", "<i4"), ("req_pm", "<i4"), ("lim_pm", "<i4"),
                     ("status", "<i4"), ("reserved", "<i4")])
assert PROF_SESSION.itemsize == 104 and PROF_OUT.itemsize == 48

# SPEC's four built-in inference profiles ("resnet152-like", "roberta-large-like",
# "gpt2-large-like", "llama2-7b-like") = Figure 4 / Table 2 models (a)-(d).  Calibration
# constants ("calibration constants live in a versioned JSON asset, not code" --
# here a versioned table): a (ms), b (ms per sample), knee coefficient c, SLO (ms).
# roberta-large-like has knee(IBS=4) = 51 % -> a 2 % throughput gain from SMR 50 to 100
# ("merely a 2% throughput boost").  Calibration v1 (D9): the constants
# nearest a first guess for which the search takes Table 2's Dilu trial counts 8 / 6 / 6 / 9
# and returns the exhaustive-grid TE maximum.
PROFILE_MODELS_V1 = [
    # name, a_ms, b_ms, knee_c, slo_ms
    ("resnet152-like", 5.0, 1.5, 30.0, 60.0),
    ("roberta-large-like", 6.0, 2.0, 25.5, 120.0),
    ("gpt2-large-like", 10.0, 4.5, 35.0, 120.0),
    ("llama2-7b-like", 30.0, 6.0, 32.0, 250.0),
]
# training models: knee_t (saturation SMR), T_max samples/s at 100 %, comm idle
PROFILE_TRAIN_V1 = [
    ("bert-base", 55.0, 400.0, 0.2),
    ("roberta-large", 70.0, 150.0, 0.3),
    ("gpt2-large", 85.0, 60.0, 0.4),
    ("resnet152", 60.0, 250.0, 0.1),
]


def prof_inference(a_ms, b_ms, knee_c, slo_ms, ibs_max=32, smr_step=10.0):
    s = np.zeros(1, PROF_SESSION)
    s["kind"], s["ibs_max"], s["a_ms"], s["b_ms"], s["knee_c"] = 0, ibs_max, a_ms, b_ms, knee_c
    s["slo_ms"], s["smr_step"] = slo_ms, smr_step
    return s[0]


def prof_training(knee_t, t_max, idle, workers=1, p_req=0.8, p_lim=1.0, tol=0.02):
    s = np.zeros(1, PROF_SESSION)
    s["kind"], s["workers"], s["knee_t"], s["t_max"], s["idle"] = 2, workers, knee_t, t_max, idle
    s["p_req"], s["p_lim"], s["tol"] = p_req, p_lim, tol
    return s[0]


def profile_sessions(n: int, seed: int = 0) -> np.ndarray:
    """n profiling sessions shaped like the C4 sweep's function table: 3/4 inference
    sessions on the four built-in profiles with per-session jitter of the latency model
    and SLO (x U[0.8, 1.25]), 1/4 training sessions with jittered knee, T_max and idle."""
    rng = _rng(seed, "profile")
    out = np.zeros(n, PROF_SESSION)
    kind = np.where(rng.random(n) < 0.75, 0, 2)
    mi = rng.integers(0, 4, n)
    j = lambda: rng.uniform(0.8, 1.25, n)
    A = np.array([m[1:] for m in PROFILE_MODELS_V1])
    Tr = np.array([m[1:] for m in PROFILE_TRAIN_V1])
    out["kind"] = kind
    out["workers"] = rng.choice([1, 2, 4], n)
    out["ibs_max"] = 32
    out["a_ms"], out["b_ms"] = A[mi, 0] * j(), A[mi, 1] * j()
    out["knee_c"], out["slo_ms"] = A[mi, 2] * j(), A[mi, 3] * j()
    out["smr_step"] = 10.0
    out["knee_t"] = np.minimum(100.0, Tr[mi, 0] * j())
    out["t_max"], out["idle"] = Tr[mi, 1] * j(), np.minimum(0.6, Tr[mi, 2] * j())
    out["p_req"], out["p_lim"], out["tol"] = 0.8, 1.0, 0.02
    return out


# ------------------------------------------------- catalogue rows for the a0 loader

# One catalogue row per function before quantisation (include/dilu.h dilu_catalog_row):
# the profiled quotas come from the function's profiling session; memory (GB), cold start
# (ms) and SLO (ms) are real-valued model facts.  Input data only: the quantisation (Q25,
# R4) is the loader's (oracle/dilu_ref_load.c, csrc/profile.cuh k_load).
CATALOG_ROW = np.dtype([("kind", "<i4"), ("prio", "<i4"), ("n_workers", "<i4"), ("duty_pm", "<i4"),
                        ("affinity_class", "<i4"), ("arrive_sec", "<i4"), ("depart_sec", "<i4"),
                        ("pattern", "<i4"), ("scale_q10", "<i4"), ("phase_slots", "<i4"),
                        ("reserved", "<i4", (2,)), ("mem_gb", "<f8"), ("cold_ms", "<f8"),
                        ("slo_ms", "<f8")])
assert CATALOG_ROW.itemsize == 72


def profiled_fleet(seed: int = 0, T: int = 900, n_inf: int = 120, n_llm: int = 40, n_train: int = 40):
    """A C2-shaped fleet described before profiling (SURVEY s8(a) a0 input): per function
    a profiling session (``PROF_SESSION``, the built-in latency / throughput models with
    jitter) and a catalogue row (``CATALOG_ROW``: memory in GB, cold start in ms, SLO in ms,
    lifecycle, arrival pattern).  Returns (sessions, catalogue, patterns); the loader turns
    profiling results + catalogue into the function table (profile -> load -> simulate)."""
    rng = _rng(seed, "catalog")
    pats = make_patterns(T, 1000, 1300 + seed, diurnal=False)
    pat_mean = pats.mean(axis=1)
    n = n_inf + n_llm + n_train
    ses = np.zeros(n, PROF_SESSION)
    cat = np.zeros(n, CATALOG_ROW)
    A = np.array([m[1:] for m in PROFILE_MODELS_V1])
    Tr = np.array([m[1:] for m in PROFILE_TRAIN_V1])
    for i in range(n):
        j = lambda: rng.uniform(0.9, 1.1)
        if i < n_inf + n_llm:
            llm = i >= n_inf
            mi = 3 if llm else int(rng.integers(0, 3))         # llama2-7b-like for LLMs
            ses[i]["kind"], ses[i]["workers"], ses[i]["ibs_max"] = 0, 1, 32
            ses[i]["a_ms"], ses[i]["b_ms"] = A[mi, 0] * j(), A[mi, 1] * j()
            ses[i]["knee_c"], ses[i]["slo_ms"] = A[mi, 2] * j(), A[mi, 3]
            ses[i]["smr_step"] = 10.0
            pat = int(BURSTY_FAMILY[rng.integers(len(BURSTY_FAMILY))])
            nominal_rps = 4 * 1000.0 / (A[mi, 3] / 2.0)          # a nominal IBS-4 server
            u = rng.uniform(0.2, 0.8)
            cat[i]["kind"] = K_LLM if llm else K_INF
            cat[i]["prio"] = 0
            cat[i]["n_workers"] = 1
            cat[i]["mem_gb"] = rng.choice([14.0, 16.0]) if llm else rng.choice([1.0, 2.0, 4.0, 6.0, 1.5])
            cat[i]["cold_ms"] = 10000.0 if llm else rng.choice([2000.0, 2500.0, 3000.0])
            cat[i]["slo_ms"] = A[mi, 3]
            cat[i]["pattern"] = pat
            cat[i]["scale_q10"] = int(round(1024.0 * u * nominal_rps / max(pat_mean[pat], 1e-3)))
            cat[i]["phase_slots"] = int(rng.integers(0, T))
            cat[i]["affinity_class"] = int(cat[i]["kind"]) * 1000 + pat
            cat[i]["arrive_sec"], cat[i]["depart_sec"] = 0, NEVER
        else:
            mi = int(rng.integers(0, 4))
            w = int(rng.choice([1, 2, 4], p=[0.5, 0.3, 0.2]))
            ses[i]["kind"], ses[i]["workers"] = 2, w
            ses[i]["knee_t"] = min(100.0, Tr[mi, 0] * j())
            ses[i]["t_max"], ses[i]["idle"] = Tr[mi, 1] * j(), min(0.6, Tr[mi, 2] * j())
            ses[i]["p_req"], ses[i]["p_lim"], ses[i]["tol"] = 0.8, 1.0, 0.02
            arr = int(rng.integers(0, T))
            cat[i]["kind"], cat[i]["prio"], cat[i]["n_workers"] = K_TRAIN, 1, w
            cat[i]["duty_pm"] = int(rng.integers(600, 1001))
            cat[i]["mem_gb"] = rng.choice([8.0, 10.0, 12.0, 20.0])
            cat[i]["cold_ms"] = 5000.0
            cat[i]["pattern"] = -1
            cat[i]["affinity_class"] = 2000 + i
            cat[i]["arrive_sec"] = arr
            cat[i]["depart_sec"] = arr + int(rng.integers(600, 2400))
    return ses, cat, pats


def workload_from_rows(name: str, rows: np.ndarray, patterns: np.ndarray, T: int,
                       gpus: int = 64, max_instances: int = 512) -> Workload:
    """One scenario over already-loaded function rows (int32 [F, 16])."""
    funcs = np.ascontiguousarray(rows, dtype=np.int32)[None]
    cfg = default_config(n_scenarios=1, gpus_per_scenario=gpus, max_funcs=funcs.shape[1],
                         max_instances=max_instances, n_patterns=patterns.shape[0],
                         pattern_len=patterns.shape[1])
    scen = np.array([[0, 1000, 1500, 0]], dtype=np.int32)
    return Workload(name, cfg, scen, funcs, patterns, T, "loaded from profiles")


# ------------------------------------------------------- model catalogue (s8(d))
# kind, mem MiB, req per-mille, lim per-mille, IBS, SLO ms, cold s.  Inference limit
# = 2 x request; c_b = req * SLO/2 (R4); training request ~80% and
# limit ~100% throughput points.
INF_MODELS = [  # name, mem, req, lim, ibs, slo_ms, cold_s
    ("resnet152", 2048, 150, 300, 8, 100, 2),
    ("vgg19", 2048, 150, 300, 8, 100, 2),
    ("bert-base", 1024, 100, 200, 8, 50, 2),
    ("roberta-large", 4096, 300, 600, 4, 100, 2),
    ("gpt2-large", 6144, 300, 600, 4, 200, 3),
]
LLM_MODELS = [
    ("llama2-7b", 16384, 400, 800, 1, 100, 10),
    ("chatglm3-6b", 14336, 350, 700, 1, 100, 10),
]
TRAIN_MODELS = [  # name, mem, req, lim, cold_s
    ("bert-base", 8192, 300, 500, 5),
    ("roberta-large", 12288, 400, 700, 5),
    ("gpt2-large", 20480, 500, 800, 5),
    ("resnet152", 10240, 350, 600, 5),
    ("vgg19", 10240, 300, 500, 5),
]


# ----------------------------------------------------------------- patterns

def make_patterns(T: int, slot_ms: int, seed: int, diurnal: bool) -> np.ndarray:
    """64 per-slot arrival patterns (SURVEY s8(d) "Pattern tables"): 12 Poisson,
    12 Gamma(CV 1..6), 16 Bursty (x4/x6 bursts), 8 Periodic, 8 Sporadic, 8 Diurnal.
    Values are requests per slot; generated once with double math, shipped as data."""
    rng = _rng(seed, "pattern")
    dt = slot_ms / 1000.0
    sec = np.arange(T, dtype=np.float64) * dt
    out = np.zeros((64, T), dtype=np.int64)
    p = 0
    for j in range(12):                         # Poisson(mu), mu in [1, 200] RPS
        mu = float(np.exp(rng.uniform(0.0, np.log(200.0))))
        out[p] = rng.poisson(mu * dt, T); p += 1
    for j in range(12):                         # Gamma(mu, CV)
        mu = float(np.exp(rng.uniform(np.log(5.0), np.log(150.0))))
        cv = 1 + (j % 6)
        lam = rng.gamma(1.0 / cv**2, mu * cv**2, T)
        out[p] = rng.poisson(lam * dt); p += 1
    for j in range(16):                         # Bursty (burst scale 4/6)
        base = float(np.exp(rng.uniform(np.log(5.0), np.log(100.0))))
        scale = 4.0 if j % 2 == 0 else 6.0
        period = rng.uniform(120, 600)
        length = rng.uniform(10, 60)
        off = rng.uniform(0, period)
        rate = np.where(((sec + off) % period) < length, base * scale, base)
        out[p] = rng.poisson(rate * dt); p += 1
    for j in range(8):                          # Periodic, 5-60 min sinusoid
        base = float(np.exp(rng.uniform(np.log(5.0), np.log(100.0))))
        per = rng.uniform(300, 3600)
        ph = rng.uniform(0, 2 * np.pi)
        rate = base * (1.0 + 0.8 * np.sin(2 * np.pi * sec / per + ph))
        out[p] = rng.poisson(np.maximum(rate, 0) * dt); p += 1
    for j in range(8):                          # Sporadic: mostly off
        base = float(np.exp(rng.uniform(np.log(5.0), np.log(60.0))))
        minute = (sec // 60).astype(np.int64)
        on_min = rng.random(int(minute.max()) + 1) < rng.uniform(0.1, 0.5)
        rate = np.where(on_min[minute], base, 0.0)
        out[p] = rng.poisson(rate * dt); p += 1
    for j in range(8):                          # Diurnal: 24 h, trough:peak 1:5
        base = float(np.exp(rng.uniform(np.log(5.0), np.log(100.0))))
        ph = rng.uniform(0, 86400)
        rate = base * (3.0 + 2.0 * np.sin(2 * np.pi * (sec + ph) / 86400.0)) / 3.0
        out[p] = rng.poisson(rate * dt); p += 1
    assert p == 64
    return out.astype(np.int32)


BURSTY_FAMILY = list(range(24, 56))     # Bursty + Periodic + Sporadic
MIXED_FAMILY = list(range(0, 24)) + list(range(56, 64))  # Poisson/Gamma + Diurnal


# ------------------------------------------------------------ fleet builder

def _func_row(kind, prio, ibs, req, lim, mem, cb, workers, duty, cold, cls, arr, dep,
              pat, scale, phase):
    return [kind, prio, ibs, req, lim, mem, cb, workers, duty, cold, cls, arr, dep, pat, scale,
            phase]


def _fleet(rng: np.random.Generator, n_train_jobs: int, n_llm: int, n_inf: int, slot_ms: int,
           T: int, patterns: np.ndarray, pat_family: List[int], inf_arrive_frac0: float,
           inf_life_s: tuple, train_arrive_max_s: int, train_len_s: tuple,
           horizon_s: int, load=(0.2, 0.8)) -> np.ndarray:
    """Build one scenario's profile table (training : LLM : non-LLM inference)."""
    sps = 1000 // slot_ms
    pat_mean = patterns.mean(axis=1) * sps  # mean RPS of each pattern
    kinds = np.array([K_TRAIN] * n_train_jobs + [K_LLM] * n_llm + [K_INF] * n_inf)
    rng.shuffle(kinds)
    rows = []
    for f, kind in enumerate(kinds):
        if kind == K_TRAIN:
            name, mem, req, lim, cold_s = TRAIN_MODELS[rng.integers(len(TRAIN_MODELS))]
            workers = int(rng.choice([1, 2, 4], p=[0.5, 0.3, 0.2]))
            duty = int(rng.integers(600, 1001))          # comm idle up to 40%
            arr = int(rng.integers(0, max(1, train_arrive_max_s)))
            dep = arr + int(rng.integers(train_len_s[0], train_len_s[1] + 1))
            rows.append(_func_row(K_TRAIN, 1, 0, req, lim, mem, 0, workers, duty,
                                  -(-cold_s * 1000 // slot_ms), 100000 + f, arr, dep, -1, 0, 0))
        else:
            models = LLM_MODELS if kind == K_LLM else INF_MODELS
            name, mem, req, lim, ibs, slo, cold_s = models[rng.integers(len(models))]
            cb = req * slo // 2                              # c_b = req * SLO/2 (R4)
            pat = int(pat_family[rng.integers(len(pat_family))])
            u = rng.uniform(*load)                           # load factor
            nominal_rps = ibs * 1000.0 / (slo / 2.0)         # IBS / t_exec
            scale = int(round(1024.0 * u * nominal_rps / max(pat_mean[pat], 1e-3)))
            phase = int(rng.integers(0, T))
            if rng.random() < inf_arrive_frac0:
                arr = 0
            else:
                arr = int(rng.integers(1, max(2, horizon_s)))
            dep = NEVER
            if arr > 0:                                      # staggered lifecycle
                dep = arr + int(rng.integers(inf_life_s[0], inf_life_s[1] + 1))
            cls = int(kind) * 1000 + pat                     # shared pattern tag
            rows.append(_func_row(int(kind), 0, ibs, req, lim, mem, cb, 1, 0,
                                  -(-cold_s * 1000 // slot_ms), cls, arr, dep, pat, scale, phase))
    return np.array(rows, dtype=np.int32)


def _pad_funcs(rows: List[np.ndarray]) -> np.ndarray:
    F = max(r.shape[0] for r in rows)
    out = np.zeros((len(rows), F, 16), dtype=np.int32)
    out[:, :, FI["kind"]] = K_UNUSED
    out[:, :, FI["depart_sec"]] = NEVER
    out[:, :, FI["pattern"]] = -1
    for i, r in enumerate(rows):
        out[i, : r.shape[0]] = r
    return out


# -------------------------------------------------------------------- configs

def c1() -> Workload:
    """Appendix A: 4 GPUs, 6 functions, 100 one-second slots."""
    T = 100
    s = np.arange(T)
    pats = np.zeros((4, T), dtype=np.int32)
    pats[0] = np.where(s < 20, 40, np.where(s < 60, 200, 40))
    pats[1] = 100
    pats[2] = 30
    pats[3] = np.where((s >= 70) & (s < 75), 4, 2)
    rows = [
        # kind prio ibs req lim mem c_b workers duty cold cls arr dep pat scale phase
        _func_row(K_INF, 0, 4, 200, 400, 4096, 10000, 1, 0, 2, 0, 0, NEVER, 0, 1024, 0),
        _func_row(K_INF, 0, 8, 150, 300, 2048, 3750, 1, 0, 2, 1, 0, NEVER, 1, 1024, 0),
        _func_row(K_INF, 0, 4, 300, 600, 6144, 30000, 1, 0, 2, 2, 0, NEVER, 2, 1024, 0),
        _func_row(K_LLM, 0, 1, 250, 500, 14336, 125000, 1, 0, 10, 3, 0, NEVER, 3, 1024, 0),
        _func_row(K_TRAIN, 1, 0, 400, 500, 10240, 0, 2, 1000, 5, 4, 0, NEVER, -1, 0, 0),
        _func_row(K_TRAIN, 1, 0, 300, 400, 8192, 0, 1, 1000, 5, 5, 0, NEVER, -1, 0, 0),
    ]
    funcs = np.array([rows], dtype=np.int32)
    cfg = default_config(n_scenarios=1, gpus_per_scenario=4, max_funcs=6, max_instances=16,
                         n_patterns=4, pattern_len=T)
    scen = np.array([[0, 1000, 1500, 0]], dtype=np.int32)
    return Workload("C1", cfg, scen, funcs, pats, T, "SURVEY Appendix A worked example")


def c2(seed: int = 0, T: int = 3600, max_instances: int = 512) -> Workload:
    """64 GPUs, 200 functions (40 training jobs, 40 LLM, 120 non-LLM), bursty family,
    1 h at 1 s slots."""
    pats = make_patterns(T, 1000, 1000 + seed, diurnal=False)
    rows = _fleet(_rng(seed, "fleet"), 40, 40, 120, 1000, T, pats, BURSTY_FAMILY,
                  inf_arrive_frac0=1.0, inf_life_s=(0, 0), train_arrive_max_s=T,
                  train_len_s=(600, 2400), horizon_s=T)
    funcs = _pad_funcs([rows])
    cfg = default_config(n_scenarios=1, gpus_per_scenario=64, max_funcs=funcs.shape[1],
                         max_instances=max_instances, n_patterns=64, pattern_len=T)
    scen = np.array([[0, 1000, 1500, 0]], dtype=np.int32)
    return Workload("C2", cfg, scen, funcs, pats, T, f"seed {seed}")


C4_RHO = [0.6, 0.7, 0.8, 0.9, 1.0, 1.1, 1.2, 1.3]
C4_LAMBDA = [1.0, 1.25, 1.5, 1.75, 2.0, 2.25, 2.5, 3.0]
C4_GAMMA = [1.0, 1.125, 1.25, 1.375, 1.5, 1.75, 2.0, 2.5]


def c4(n_scenarios: int = 4096, T: int = 3600, max_instances: int = 512,
       first: int = 0, replica: int = 0) -> Workload:
    """4,096 C2-shaped scenarios: sweep rho x lambda x gamma x seed = 8^4.
    Scenario id = seed + 8*(gamma_i + 8*(lambda_i + 8*rho_i)).  ``first``/``n_scenarios``
    select a contiguous id range of the full grid.  ``replica`` r > 0 draws the 8 fleet
    seeds from 8r..8r+7 and offsets ids by 4096r (weak-scaling copies of the sweep, one
    per rank)."""
    pats = make_patterns(T, 1000, 4000, diurnal=False)
    bases = []
    for seed in range(8 * replica, 8 * replica + 8):
        bases.append(_fleet(_rng(seed, "fleet"), 40, 40, 120, 1000, T, pats, BURSTY_FAMILY,
                            inf_arrive_frac0=1.0, inf_life_s=(0, 0),
                            train_arrive_max_s=T, train_len_s=(600, 2400),
                            horizon_s=T))
    base = _pad_funcs(bases)                                   # [8, F, 16]
    ids = np.arange(first, first + n_scenarios)
    seed_i = ids % 8
    gam_i = (ids // 8) % 8
    lam_i = (ids // 64) % 8
    rho_i = (ids // 512) % 8
    funcs = base[seed_i].copy()                                # [S, F, 16]
    kind = funcs[:, :, FI["kind"]]
    rho = np.array(C4_RHO)[rho_i][:, None]
    lam = np.array(C4_LAMBDA)[lam_i][:, None]
    used = kind != K_UNUSED
    req = funcs[:, :, FI["req_pm"]].astype(np.float64)
    req2 = np.where(used, np.ceil(req * rho - 1e-9), req).astype(np.int64)
    inf = (kind == K_INF) | (kind == K_LLM)
    lim_inf = np.minimum(1000, np.ceil(req2 * lam - 1e-9)).astype(np.int64)
    lim2 = np.where(inf, lim_inf, np.maximum(funcs[:, :, FI["lim_pm"]], req2))
    funcs[:, :, FI["req_pm"]] = np.where(used, req2, funcs[:, :, FI["req_pm"]])
    funcs[:, :, FI["lim_pm"]] = np.where(used, lim2, funcs[:, :, FI["lim_pm"]])
    gam = (np.array(C4_GAMMA)[gam_i] * 1000 + 0.5).astype(np.int32)
    scen = np.stack([ids + 4096 * replica, np.full_like(ids, 1000), gam, np.zeros_like(ids)],
                    axis=1).astype(np.int32)
    cfg = default_config(n_scenarios=int(n_scenarios), gpus_per_scenario=64,
                         max_funcs=funcs.shape[1], max_instances=max_instances, n_patterns=64,
                         pattern_len=T)
    return Workload("C4", cfg, scen, funcs.astype(np.int32), pats, T,
                    f"scenarios [{first}, {first + n_scenarios}) of the 8^4 sweep")


def _large(name: str, G: int, n_jobs: int, n_llm: int, n_inf: int, slot_ms: int, T_slots: int,
           seeds: List[int], horizon_s: int, max_instances: int, pattern_seed: int,
           base_frac: float) -> Workload:
    """Staggered lifecycle: a base fraction of inference functions lives all
    day from s=0; the rest arrive uniformly over the day and live U[1, 8] h; training
    jobs arrive uniformly and run U[1, 6] h.  base_frac is calibrated so the peak
    request sum is ~80-90% of the gamma-bound packing capacity."""
    pats = make_patterns(T_slots, slot_ms, pattern_seed, diurnal=True)
    rows = []
    for sd in seeds:
        rows.append(_fleet(_rng(sd, "fleet"), n_jobs, n_llm, n_inf, slot_ms, T_slots, pats,
                           MIXED_FAMILY, inf_arrive_frac0=base_frac, inf_life_s=(3600, 8 * 3600),
                           train_arrive_max_s=horizon_s, train_len_s=(3600, 6 * 3600),
                           horizon_s=horizon_s))
    funcs = _pad_funcs(rows)
    cfg = default_config(n_scenarios=len(seeds), gpus_per_scenario=G, max_funcs=funcs.shape[1],
                         max_instances=max_instances, n_patterns=64, pattern_len=T_slots,
                         slot_ms=slot_ms)
    scen = np.array([[i, 1000, 1500, 0] for i in range(len(seeds))], dtype=np.int32)
    return Workload(name, cfg, scen, funcs, pats, T_slots, f"seeds {seeds}")


def c3(seed: int = 0, T: int = 86400, max_instances: int = 16384) -> Workload:
    """1,024 GPUs, ~5,000 initial-deployment instances (526 training jobs, 1,000 LLM,
    3,000 non-LLM), diurnal/Poisson/Gamma mix, 24 h at 1 s."""
    return _large("C3", 1024, 526, 1000, 3000, 1000, T, [seed], 86400, max_instances, 3000 + seed,
                  base_frac=0.5)


def c5(n_scenarios: int = 8, T: int = 864000, max_instances: int = 262144,
       first_seed: int = 50) -> Workload:
    """16,384 GPUs, ~100,000 instances (10,526 training jobs, 20,000 LLM, 60,000
    non-LLM), 24 h at 100 ms slots; seeds 50-57.  ``T`` may be cut
    to the timed window (36,000 slots)."""
    return _large("C5", 16384, 10526, 20000, 60000, 100, T,
                  list(range(first_seed, first_seed + n_scenarios)), 86400, max_instances, 5000,
                  base_frac=0.35)


def scaled(name: str, G: int, n_jobs: int, n_llm: int, n_inf: int, slot_ms: int, T: int,
           seeds: List[int], max_instances: int) -> Workload:
    """A large-config-shaped workload at a reduced size (parity tests)."""
    return _large(name, G, n_jobs, n_llm, n_inf, slot_ms, T, seeds, T * slot_ms // 1000,
                  max_instances, 777, base_frac=0.5)


def with_modes(wl: Workload, modes) -> Workload:
    """The same fleet under baseline modes: scenario i gets modes[i]."""
    scen = wl.scen.copy()
    scen[:, 3] = np.asarray(modes, dtype=np.int32)
    return Workload(wl.name, wl.cfg, scen, wl.funcs, wl.patterns, wl.n_slots, wl.note)


def replicate(wl: Workload, n: int) -> Workload:
    """n copies of scenario 0 (for running one fleet under several modes)."""
    cfg = dict(wl.cfg)
    cfg["n_scenarios"] = n
    scen = np.repeat(wl.scen[:1], n, axis=0)
    return Workload(wl.name, cfg, scen, np.repeat(wl.funcs[:1], n, axis=0), wl.patterns,
                    wl.n_slots, wl.note)


def by_name(name: str, **kw) -> Workload:
    return {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}[name.upper()](**kw)
