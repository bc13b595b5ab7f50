"""Per-phase cycle breakdown of the C5 bench shape (8 x 16,384-GPU scenarios, 100 ms
slots, cluster engine, fused 1 s batches) from a -DDILU_PHASE_TIMING build:
  DILU_LIB=paper_2503_05130_b200/libdilu_dilu_phase_timing.so python tools/c5_phase_breakdown.py [slots]
Leader (cluster CTA 0, thread 0) clock64 deltas summed per scenario, printed per fused
batch (second): 8 pre-boundary, 9 boundary (B1 + B3 + placement), 10 repack, 11 P0b + fold,
12 P1b, 13 P2b; 14 B3 ... 18 place; plus the event counters."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dilu_inputs as di  # noqa: E402
from paper_2503_05130_b200 import DiluSim, lib  # noqa: E402

slots = int(sys.argv[1]) if len(sys.argv) > 1 else 3600
burst = len(sys.argv) > 2 and sys.argv[2] == "burst"   # time the first 600 slots instead
wl = di.c5(n_scenarios=8, T=slots, first_seed=50)
sim = DiluSim.from_workload(wl)
if burst:
    slots = 1200
else:
    sim.scale_step(600)                  # past the initial fleet burst
torch.cuda.synchronize()
lib().dilu_sim_reset  # noqa
per0 = np.zeros((8, 24), dtype=np.int64)
lib().dilu_kernel_stats(sim.h, per0.ctypes.data, None)
s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
s0.record(); sim.scale_step(slots - 600); s1.record(); torch.cuda.synchronize()   # (burst: slots 0..599)
per = np.zeros((8, 24), dtype=np.int64)
lib().dilu_kernel_stats(sim.h, per.ctypes.data, None)
d = (per - per0).sum(0)
names = ["attempts", "retry_checks", "row_repacks", "boundary_events", "queue_scans", "slots",
         "resident_slots", "function_slots", "tick0_pre", "tick1_boundary", "tick2_repack",
         "tick3_p0b", "tick4_p1b", "tick5_p2b", "b3", "terminate", "enqueue", "next_attempt",
         "place", "t19", "t20", "t21", "t22", "t23"]
secs = (slots - 600) / 10.0 * 8
out = {"ms_steady": s0.elapsed_time(s1), "seconds_x_scenarios": secs}
for k, n in enumerate(names):
    out[n + "_per_second"] = float(d[k]) / secs
print(json.dumps(out, indent=1))
