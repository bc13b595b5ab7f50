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
names = ["attempts", "retry_checks", "row_repacks", "boundary_events", "queue_scans", "slots",
         "resident_slots", "function_slots", "pre_boundary", "boundary", "repack", "p0", "p1", "p2",
         "b3", "terminate", "enqueue", "next_attempt", "place", "w_p0", "w_p1", "w_p2", "b1_count_scan", "t23"]
tot = per.sum(0)
ss = tot[5]
out = {"ms": s0.elapsed_time(s1), "scenario_slots": int(ss)}
for k, nm in enumerate(names):
    out[nm + "_per_slot"] = float(tot[k]) / ss
print(json.dumps(out, indent=1))
