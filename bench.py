#!/usr/bin/env python
"""bench.py -- simulated GPU-slot decisions/s of the batched Dilu provisioning loop.

Workload (default): C4 of BASELINE.json -- 4,096 independent 64-GPU scenarios (the
rho x lambda x gamma x seed = 8^4 request/limit/oversubscription sweep), 200 functions
each, one hour of 1 s slots, "sharded across 8 GPUs".  One step = one full pass of the
hot path over that batch: reset to slot 0 (inputs resident in HBM), 3,600 slots of
boundary work (window push, departures, lazy scaling, arrivals, Alg.1 placement pass)
and per-slot arrivals, dispatch, token allocation, gang minima and metric fold, then the
device tally reduce and the one NCCL all-reduce of the int64 tally vector.  Decisions =
sum over scenarios of G * slots (tally gpu_row_slots).

Multi-GPU: one process per GPU.  Launched by torchrun (RANK/WORLD_SIZE/LOCAL_RANK in the
environment) or, with --gpus N > 1 and no torchrun environment, bench.py re-executes
itself under torch.distributed.run (it refuses if fewer than N GPUs are visible).
--scaling strong (default, BASELINE's definition): the 4,096 scenarios (C5: 8) are split
into contiguous blocks, one per rank; --scaling weak: every rank runs its own replica.
Time = max over ranks of the summed CUDA-event step times; value = all ranks' decisions /
that time.  L2 is flushed (256 MiB write) between timed steps.

--impl reference times the CPU oracle (oracle/, plain C, all host cores) on the same
bounded sample the product line's cpu_baseline uses; only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "simulated GPU-slot decisions/sec"
UNIT = "decisions/s"
# Algorithmic bytes per unit (SURVEY s8(d) "Which roofline bounds the path"):
BYTES_PER_ACTIVE_ROW_SLOT = 8        # vertical + fold: nres and U of an active GPU row
BYTES_PER_RESIDENT_SLOT = 16         # id, req, lim, function and ready of a warm resident
BYTES_PER_FUNCTION_SLOT = 8          # arrivals / dispatch: rps_acc read + write
BYTES_PER_FUNCTION_SECOND = 24       # hscaler: ring slot RW + incremental up/down counters
BYTES_PER_GPU_SCORED = 12            # placement: R, L, U of a candidate row ...
BYTES_PER_RESIDENT_SCORED = 2        # ... + 2 B per resident (affinity test)
PAPER_PLACEMENTS = (3200, 1.12)      # "3,200 instances ... within 1.12 seconds" (context)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="dilu", choices=["dilu", "reference"])
    ap.add_argument("--workload", default="C4", choices=["C4", "C2", "C3", "C5", "PROFILE"],
                    help="PROFILE: the batched profiler (SURVEY 8(f) #3) over the C4 sweep's "
                         "4,096 x 200 function rows, metric profiling sessions/s")
    ap.add_argument("--prof-sessions", type=int, default=4096 * 200)
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"])
    ap.add_argument("--slots", type=int, default=0, help="slots per step (0: workload default)")
    ap.add_argument("--scenarios", type=int, default=0,
                    help="C5: scenarios in the batch (0: the 8 of BASELINE's C5; 1 = one 8-GPU strong shard)")
    ap.add_argument("--cpu-sample", type=int, default=0, help="oracle sample scenarios (0: auto)")
    ap.add_argument("--cpu-slots", type=int, default=0, help="oracle sample slots (0: the step's)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the isolated place_batch (placements/s) measurement")
    ap.add_argument("--latency", action="store_true",
                    help="request-level latency (cfg.flags bit3, DESIGN.md D10): adds p50/p95 "
                         "and the latency SVR to the line")
    ap.add_argument("--vertical", default="slot", choices=["slot", "alg2"],
                    help="slot: slot-level grant (default); alg2: literal Algorithm 2 at 5 ms "
                         "periods (cfg.flags bit2, DESIGN.md D8)")
    return ap.parse_args()


# ------------------------------------------------------------------ process launch

def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def maybe_spawn(args) -> None:
    """--gpus N > 1 outside torchrun: re-execute under torch.distributed.run, one rank per
    GPU; refuse clearly when fewer than N GPUs are visible."""
    if "WORLD_SIZE" in os.environ or args.gpus <= 1:
        return
    if args.impl == "dilu" or args.workload == "PROFILE":
        import torch
        n = torch.cuda.device_count()
        if n < args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, "
                             f"found {n}\n")
            sys.exit(2)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def world_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# ------------------------------------------------------------------ workloads

def build_workload(name: str, rank: int, world: int, scaling: str, slots: int,
                   vertical: str = "slot", latency: bool = False, n_c5: int = 0):
    import dilu_inputs as di
    wl, desc, n = _build_workload(name, rank, world, scaling, slots, n_c5)
    extra = (4 if vertical == "alg2" else 0) | (8 if latency else 0)
    if extra:
        cfg = dict(wl.cfg, flags=wl.cfg["flags"] | extra)
        wl = di.Workload(wl.name, cfg, wl.scen, wl.funcs, wl.patterns, wl.n_slots, wl.note)
    if vertical == "alg2":
        desc += "; literal Alg.2, %d x 5 ms periods per slot" % (wl.cfg["slot_ms"] // 5)
    if latency:
        desc += "; request-level latency"
    return wl, desc, n


def _build_workload(name: str, rank: int, world: int, scaling: str, slots: int, n_c5: int = 0):
    import dilu_inputs as di
    if name == "C4":
        if scaling == "weak":
            wl = di.c4(n_scenarios=4096, T=slots or 3600, replica=rank)
            desc = "C4 replica %d: 4096 x 64-GPU scenarios (rho x lambda x gamma x seed sweep)" % rank
        else:
            lo, hi = 4096 * rank // world, 4096 * (rank + 1) // world
            wl = di.c4(n_scenarios=hi - lo, first=lo, T=slots or 3600)
            desc = "C4: scenarios [%d, %d) of the 4096 x 64-GPU sweep" % (lo, hi)
        return wl, desc, wl.n_slots
    if name == "C2":
        wl = di.c2(seed=rank, T=slots or 3600)
        return wl, "C2: one 64-GPU cluster, 200 functions, bursty (replica per rank)", wl.n_slots
    if name == "C3":
        wl = di.c3(seed=rank, T=86400)
        return wl, "C3: one 1,024-GPU cluster, ~4,500 functions, diurnal (replica per rank)", slots or 3600
    if name == "C5":
        T = slots or 36000
        tot = n_c5 or 8
        if scaling == "weak":
            n, first = tot, 50 + tot * rank
        else:
            lo, hi = tot * rank // world, tot * (rank + 1) // world
            n, first = max(1, hi - lo), 50 + lo
        wl = di.c5(n_scenarios=n, T=T, first_seed=first)
        return wl, "C5: %d x 16,384-GPU clusters (seeds %d..%d), 100 ms slots, timed window" % (
            n, first, first + n - 1), T
    raise ValueError(name)


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_sample(args, wl, n_slots):
    """The bounded oracle sample both the cpu_baseline field and --impl reference time:
    C4 64 scenarios spread over the sweep x the full hour; single-scenario configs the
    scenario itself; C5 min(8, cores) scenarios x the full timed window."""
    import numpy as np
    cores = len(os.sched_getaffinity(0))
    if args.workload == "C4":
        k = args.cpu_sample or 64
    elif args.workload == "C5":
        k = args.cpu_sample or min(8, cores)
    else:
        k = args.cpu_sample or 1
    k = max(1, min(wl.S, k))
    idx = np.linspace(0, wl.S - 1, k).round().astype(int)
    sub = wl.subset(idx) if wl.S > 1 else wl
    slots = args.cpu_slots or n_slots
    return sub, slots, min(cores, k)


def time_oracle(sub, slots, threads):
    import oracle
    s = oracle.RefSim(sub)
    t0 = time.perf_counter()
    s.scale_step(slots, threads)
    dt = time.perf_counter() - t0
    _, tot = s.metrics()
    s.close()
    return int(tot[15]), dt


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: NVML polled every
    2 ms on a thread (so even sub-millisecond regions get samples), else nvidia-smi."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.rows = []          # (sm_mhz, max_mhz, [reason flags])
        self.proc = None
        self.nvml = None
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            bits = [N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                    N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap]
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)

            def poll():
                while True:
                    sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                    r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append((float(sm), float(mx), [bool(r & b) for b in bits]))
                    if self.stop.wait(0.002):
                        break
            self.nvml = N
            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nvml = None
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7 and parts[0].replace(".", "").isdigit():
                self.rows.append((float(parts[0]), float(parts[1]) if parts[1].replace(".", "").isdigit() else None,
                                  [parts[3 + i] == "Active" for i in range(4)]))

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml is not None:
            self.thread.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        import statistics
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [r[0] for r in self.rows]
        mx = [r[1] for r in self.rows if r[1] is not None]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4) if r[2][i]})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), \
            "MEASURED_PEAKS.json hbm_gbs (copy, burst)"
    except Exception:
        return 7700.0, "B200_PROFILING.md fallback"


def ncu_evidence(workload: str):
    """ncu counters of the bench kernel captured from the same build (profiles/
    r2_ncu_summary.json, written by tools/ncu_summary.py from an `ncu --set full` report):
    dram bytes per launch, ALU-pipe %, issue-active %.  None if absent."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r2_ncu_summary.json")))
        return d.get(workload)
    except Exception:
        return None


# ------------------------------------------------------------------ reference arm

def run_reference(args):
    rank, world, _ = world_env()
    if rank != 0:
        return
    wl, desc, n_slots = build_workload(args.workload, 0, 1, args.scaling, args.slots, args.vertical,
                                       args.latency, args.scenarios)
    sub, slots, threads = oracle_sample(args, wl, n_slots)
    vals = []
    for k in range(args.warmup + args.steps):
        D, dt = time_oracle(sub, slots, threads)
        if k >= args.warmup:
            vals.append((D, dt))
    tot_D = sum(x[0] for x in vals)
    tot_t = sum(x[1] for x in vals)
    value = tot_D / tot_t
    smp = (f"{sub.S} of {wl.S} scenarios x {slots} slots per step ({desc}); one pthread per "
           f"scenario on {threads} of {len(os.sched_getaffinity(0))} host threads; {cpu_model()}")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * tot_t / len(vals), "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "int32",
            "data": "synthetic", "config": {"workload": desc, "slots": slots,
                                            "oracle_sample_scenarios": sub.S,
                                            "note": "CPU oracle; rank 0 only"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": smp, "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ product arm

def initial_fleet_requests(wl):
    """dilu_place_batch requests of the initial fleet: every function arriving at second 0,
    one request each (inference: min_instances single-instance requests; training: one
    gang of n_workers), scenario-major in function order."""
    import numpy as np
    import dilu_inputs as di
    kind = wl.funcs[:, :, di.FI["kind"]]
    arr = wl.funcs[:, :, di.FI["arrive_sec"]]
    s_idx, f_idx = np.nonzero((kind != di.K_UNUSED) & (arr == 0))
    reps = np.where(kind[s_idx, f_idx] == di.K_TRAIN, 1, wl.cfg["min_instances"])
    return (np.repeat(s_idx, reps).astype(np.int32), np.repeat(f_idx, reps).astype(np.int32))


def run_dilu(args):
    import numpy as np
    import torch
    rank, world, local = world_env()
    if world > torch.cuda.device_count():
        sys.stderr.write(f"bench.py: world size {world} > {torch.cuda.device_count()} visible GPUs\n")
        sys.exit(2)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2503_05130_b200 import DiluSim, dist as ddist
    ddist.init("nccl", device=dev)
    wl, desc, n_slots = build_workload(args.workload, rank, world, args.scaling, args.slots,
                                       args.vertical, args.latency, args.scenarios)
    sim = DiluSim.from_workload(wl, device=dev)
    stream = sim.stream
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    tally = torch.zeros(17, dtype=torch.int64, device=dev)

    def step(ev=None):
        sim.reset()
        if ev:
            ev[0].record(stream)
        sim.scale_step(n_slots)
        if ev:
            ev[1].record(stream)
        _, tot = sim.metrics(per_scenario=False)
        tally.copy_(tot)
        ddist.allreduce_tallies(tally)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    step_ms, kern_ms = [], []
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.fill_(k & 0xFF)                       # L2 flush between timed steps
            torch.cuda.synchronize()
            ddist.barrier()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            e[0].record(stream)
            step(ev=(e[2], e[3]))
            e[1].record(stream)
            torch.cuda.synchronize()
            step_ms.append(e[0].elapsed_time(e[1]))
            kern_ms.append(e[2].elapsed_time(e[3]))
        ddist.barrier()
    local_ms = sum(step_ms)
    max_ms = ddist.allreduce_max(local_ms)
    _, tot_local = sim.metrics(per_scenario=False)
    tot_local = tot_local.cpu().numpy()
    D_all = int(tally[15].item())                        # all ranks (after the all-reduce)
    value = D_all * args.steps / (max_ms / 1000.0)
    stats = sim.kernel_stats()
    lat_line = None
    if args.latency:
        from paper_2503_05130_b200 import latency_summary
        _, lat = sim.latency()
        lat_t = torch.from_numpy(lat).to(dev)
        ddist.allreduce_tallies(lat_t)                  # int64 SUM over ranks
        lat_line = latency_summary(lat_t.cpu().numpy())

    # roofline of the dominant kernel (k_run, the scale_step launch): SURVEY s8(d)'s
    # algorithmic bytes per unit x this launch's unit counts (kernel counters and tallies)
    sps = 1000 // wl.cfg["slot_ms"]
    act = int(tot_local[0])
    rho = stats["resident_slots"] / max(act, 1)
    units = {"active_row_slots": act, "warm_resident_slots": stats["resident_slots"],
             "inference_function_slots": stats["function_slots"],
             "inference_function_seconds": stats["function_slots"] // sps,
             "placement_attempts": stats["attempts"]}
    alg_bytes = (BYTES_PER_ACTIVE_ROW_SLOT * act
                 + BYTES_PER_RESIDENT_SLOT * stats["resident_slots"]
                 + BYTES_PER_FUNCTION_SLOT * stats["function_slots"]
                 + BYTES_PER_FUNCTION_SECOND * (stats["function_slots"] // sps)
                 + stats["attempts"] * wl.G * (BYTES_PER_GPU_SCORED + BYTES_PER_RESIDENT_SCORED * rho))
    k_s = sum(kern_ms) / len(kern_ms) / 1000.0
    peak, peak_src = hbm_peak()
    achieved = alg_bytes / k_s / 1e9
    ev = ncu_evidence(args.workload) if (args.vertical == "slot" and not args.latency) else None
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": ev.get("dram_bytes_per_launch") if ev else None,
            "kernel": "k_run (one scale_step launch per step)", "kernel_ms": 1000 * k_s,
            "algorithmic_bytes_per_launch": int(alg_bytes), "units_per_launch": units,
            "peak_source": peak_src,
            "regime": ("R-SMEM: hot state staged in shared memory, latency/issue-bound; HBM "
                       "roofline per north_star" if wl.G <= 256 else
                       "R-HBM/L2: state in HBM/L2 (cluster engine)")}
    if ev:
        roof["ncu"] = {k: ev[k] for k in ev if k != "dram_bytes_per_launch"}

    # secondary metrics (SURVEY s8(d) "Also reported")
    secondary = {"resident_slot_allocations_per_s": stats["resident_slots"] / k_s,
                 "scaling_decisions_per_s": (stats["function_slots"] // sps) / k_s,
                 "placement_attempts_per_s": stats["attempts"] / k_s}
    if not args.no_secondary and args.vertical == "slot" and not args.latency:
        rs, rf = initial_fleet_requests(wl)
        times, placed = [], 0
        for k in range(3):
            s3 = DiluSim.from_workload(wl, device=dev)
            d_rs = torch.from_numpy(rs).to(dev)
            d_rf = torch.from_numpy(rf).to(dev)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            og, _ = s3.place_batch(d_rs, d_rf)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
            _, t3 = s3.metrics(per_scenario=False)
            placed = int(t3[8].item())
            s3.close()
            del s3
        tb = sorted(times)[1]
        placed_all = int(ddist.allreduce_tallies(torch.tensor([placed], dtype=torch.int64, device=dev))[0].item())
        tb_max = ddist.allreduce_max(tb)
        secondary.update({
            "placements_per_s": placed_all / tb_max,
            "place_batch": {"instances_placed": placed_all, "requests": int(len(rs)) * world,
                            "call_ms": 1000 * tb_max,
                            "what": "one dilu_place_batch call per rank over the initial fleet "
                                    "(every function arriving at second 0), median of 3, wall "
                                    "clock around the call incl. its one host validation sync",
                            "paper_context": "%d instances in %.2f s on the paper's host (P:1363)" % PAPER_PLACEMENTS}})

    # end to end through the public API: pinned host inputs -> create (H2D) -> slots ->
    # tallies D2H into pinned host memory, every step
    e2e_val, h2d, d2h = None, 0, 0
    if args.e2e_steps > 0:
        pin = {k: torch.from_numpy(np.ascontiguousarray(getattr(wl, k))).pin_memory()
               for k in ("scen", "funcs", "patterns")}
        h2d = sum(t.numel() * t.element_size() for t in pin.values())
        d2h = 17 * 8
        times = []
        for k in range(args.e2e_steps):
            torch.cuda.synchronize()
            ddist.barrier()
            t0 = time.perf_counter()
            s2 = DiluSim(wl.cfg_array(), pin["scen"].numpy(), pin["funcs"].numpy(),
                         pin["patterns"].numpy(), device=dev)
            s2.scale_step(n_slots)
            _, tot = s2.metrics(per_scenario=False, host=True)
            times.append(time.perf_counter() - t0)
            s2.close()
            del s2
        e2e_s = ddist.allreduce_max(sum(times))
        e2e_val = D_all * len(times) / e2e_s

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sub, slots, threads = oracle_sample(args, wl, n_slots)
        D, dt = time_oracle(sub, slots, threads)
        cpu = {"value": D / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
               "cpu_model": cpu_model(),
               "sample": f"{sub.S} of {wl.S} scenarios x {slots} slots, one pthread per scenario "
                         f"on {threads} of {len(os.sched_getaffinity(0))} host threads, {dt:.1f} s "
                         "(the same sample --impl reference times)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": desc, "scenarios_per_gpu": wl.S, "gpus_per_scenario": wl.G,
                       "slots": n_slots, "slot_ms": wl.cfg["slot_ms"], "decisions_per_step": D_all,
                       "l2": "flushed between timed steps (256 MiB write)",
                       "parallelism": f"scenario shards x{world} ({args.scaling})",
                       "vertical": args.vertical, "latency": bool(args.latency)},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": 3 * args.steps,
            "clocks": clk.summary(),
            "secondary": secondary,
            "kernel_stats_per_step": stats,
        }
        if lat_line is not None:
            line["latency"] = lat_line
        print(json.dumps(line), flush=True)
    ddist.barrier()
    ddist.finalize()


PROF_METRIC, PROF_UNIT = "profiling sessions/sec", "sessions/s"
PROF_BYTES_PER_SESSION = 104 + 48       # one dilu_prof_session read + one dilu_prof_out written


def run_profile(args):
    """The batched profiler: one dilu_profile launch per step over the C4 sweep's function
    rows (weak scaling: every rank profiles its own replica)."""
    import numpy as np
    import dilu_inputs as di
    rank, world, local = world_env()
    n = args.prof_sessions
    ses = di.profile_sessions(n, seed=1000 + rank)
    if args.impl == "reference":
        if rank != 0:
            return
        import oracle
        sub = ses[: min(n, 2_000_000)]
        times = []
        for k in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            oracle.profile_batch(sub)
            if k >= args.warmup:
                times.append(time.perf_counter() - t0)
        v = len(sub) * len(times) / sum(times)
        line = {"impl": "reference", "metric": PROF_METRIC, "value": v, "unit": PROF_UNIT,
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1000 * sum(times) / len(times), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": "profiler over %d C4-sweep function rows" % len(sub)},
                "cpu_baseline": {"value": v, "unit": PROF_UNIT, "cores": 1, "kind": "oracle",
                                 "sample": "%d sessions, one thread" % len(sub), "cpu_model": cpu_model()},
                "e2e": {"value": v, "unit": PROF_UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    import torch
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2503_05130_b200 import dilu_profile, dist as ddist
    ddist.init("nccl", device=dev)
    stream = torch.cuda.current_stream(dev)
    host = torch.from_numpy(np.ascontiguousarray(ses).view(np.uint8)).pin_memory()
    d_in = host.to(dev)
    d_out = torch.empty(n * 48, dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        dilu_profile(d_in, d_out)
    torch.cuda.synchronize()
    ms = []
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            torch.cuda.synchronize()
            ddist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dilu_profile(d_in, d_out)
            e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        ddist.barrier()
    max_ms = ddist.allreduce_max(sum(ms))
    value = n * world * args.steps / (max_ms / 1000.0)
    k_s = sum(ms) / len(ms) / 1000.0
    achieved = n * PROF_BYTES_PER_SESSION / k_s / 1e9
    peak, src = hbm_peak()
    # end to end: pinned host sessions -> device -> profile -> outputs back to pinned host
    h_out = torch.empty(n * 48, dtype=torch.uint8).pin_memory()
    times = []
    for k in range(max(1, args.e2e_steps)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d2 = host.to(dev, non_blocking=True)
        o2 = dilu_profile(d2)
        h_out.copy_(o2, non_blocking=True)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    e2e_s = ddist.allreduce_max(sum(times))
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        sub = ses[: min(n, 1_000_000)]
        t0 = time.perf_counter()
        oracle.profile_batch(sub)
        dt = time.perf_counter() - t0
        cpu = {"value": len(sub) / dt, "unit": PROF_UNIT, "cores": 1, "kind": "oracle",
               "cpu_model": cpu_model(), "sample": "%d sessions, one thread, %.2f s" % (len(sub), dt)}
    if rank == 0:
        line = {"metric": PROF_METRIC, "value": value, "unit": PROF_UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": "profiler (SURVEY 8(f) #3) over %d C4-sweep function rows "
                                       "per GPU (3/4 inference HGS, 1/4 training bisection)" % n,
                           "sessions_per_gpu": n, "l2": "flushed between timed steps (256 MiB write)",
                           "parallelism": f"session shards x{world}"},
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "traffic": None, "kernel": "k_profile",
                             "kernel_ms": 1000 * k_s, "bytes_per_session": PROF_BYTES_PER_SESSION,
                             "peak_source": src},
                "cpu_baseline": cpu,
                "e2e": {"value": n * world * len(times) / e2e_s, "unit": PROF_UNIT,
                        "h2d_bytes_per_step": n * 104, "d2h_bytes_per_step": n * 48},
                "gpu_launches": args.steps, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    ddist.barrier()
    ddist.finalize()


def main():
    args = parse()
    maybe_spawn(args)
    if args.workload == "PROFILE":
        run_profile(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_dilu(args)


if __name__ == "__main__":
    main()
