"""Freeze the oracle's C5 tallies over the bench's timed window (8 x 16,384-GPU scenarios,
seeds 50..57, 36,000 x 100 ms slots) into tests/golden/c5_window_tallies.json.  Calls only
oracle/ (plain C, one pthread per scenario); the GPU test compares against this file
("a hash frozen by a committed script that calls only oracle/")."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import dilu_inputs as di  # noqa: E402
import oracle  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 36000
wl = di.c5(n_scenarios=8, T=T, first_seed=50)
s = oracle.RefSim(wl)
t0 = time.time()
s.scale_step(T, threads=8)
per, tot = s.metrics()
out = {"source": "tools/freeze_c5_golden.py (oracle only)", "workload": "di.c5(n_scenarios=8, T=%d, first_seed=50)" % T,
       "slots": T, "oracle_seconds": round(time.time() - t0, 1),
       "tally_names": di.TALLY_NAMES, "per_scenario": per.tolist(), "sum": tot.tolist()}
path = os.path.join(ROOT, "tests", "golden", "c5_window_tallies.json" if T == 36000 else "c5_window_%d.json" % T)
json.dump(out, open(path, "w"), indent=1)
print(path, out["oracle_seconds"], "s")
