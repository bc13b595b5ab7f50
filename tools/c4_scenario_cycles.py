"""Per-scenario cycle counts of the C4 sweep (a -DDILU_PHASE_TIMING build via DILU_LIB),
for the scheduling analysis in DESIGN.md s7: python tools/c4_scenario_cycles.py."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dilu_inputs as di
from paper_2503_05130_b200 import DiluSim, lib
wl = di.c4(n_scenarios=4096)
sim = DiluSim.from_workload(wl)
sim.scale_step(3600); torch.cuda.synchronize()
per = np.zeros((4096, 24), dtype=np.int64)
lib().dilu_kernel_stats(sim.h, per.ctypes.data, None)
cyc = per[:, 8:14].sum(1)
np.save("gpurun_out/c4_cycles.npy", cyc)
np.save("gpurun_out/c4_stats.npy", per)
print("cycles per scenario: mean %.3g min %.3g max %.3g cv %.3f" % (cyc.mean(), cyc.min(), cyc.max(), cyc.std() / cyc.mean()))
