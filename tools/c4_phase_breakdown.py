"""Per-phase cycle breakdown of the C4 sweep from a -DDILU_PHASE_TIMING build
(`python paper_2503_05130_b200/_build.py -DDILU_PHASE_TIMING`, then
`DILU_LIB=paper_2503_05130_b200/libdilu_dilu_phase_timing.so python tools/c4_phase_breakdown.py`).
Timers are the leader thread's clock64 deltas (barrier waits included), summed per
scenario; printed as mean cycles per scenario-slot, plus the event counters per slot."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dilu_inputs as di
from paper_2503_05130_b200 import DiluSim, lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
slots = int(sys.argv[2]) if len(sys.argv) > 2 else 3600
wl = di.c4(n_scenarios=n)
sim = DiluSim.from_workload(wl)
s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
s0.record(); sim.scale_step(slots); s1.record(); torch.cuda.synchronize()
per = np.zeros((n, 24), dtype=np.int64)
lib().dilu_kernel_stats(sim.h, per.ctypes.data, None)
# timers 8..13 are the leader's TICK(0..5); in the pipelined (overlapped) C4 path:
# 9 = prologue B1 + B3a + barrier, 10 = repack, 11 = B3b + placement pass + fold,
# 12 = wait for P0 + B1 of the next boundary (warp 0), 13 = join wait;
# 19..21 = the first worker thread's P0 / P1 / P2 (each incl. its barrier wait),
# 23 = the slowest worker's finish since the arm start (summed per slot)
names = ["attempts", "retry_checks", "row_repacks", "boundary_events", "queue_scans", "slots",
         "resident_slots", "function_slots", "tick0_pre", "tick1_b3a", "tick2_repack",
         "tick3_ctl_place", "tick4_ctl_b1", "tick5_join",
         "b3", "terminate", "enqueue", "next_attempt", "place", "w_p0", "w_p1", "w_p2", "scratch",
         "worker_arm_max"]
tot = per.sum(0)
ss = tot[5]
out = {"ms": s0.elapsed_time(s1), "scenario_slots": int(ss)}
for k, nm in enumerate(names):
    out[nm + "_per_slot"] = float(tot[k]) / ss
print(json.dumps(out, indent=1))
