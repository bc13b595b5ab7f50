"""Baseline-mode report over the C4 sweep on the GPU (PAPER.md:1149-1169,
Table 3, s5.5 P:1417): every sweep point runs under Dilu, Exclusive, StaticLimit
(MPS-l, "INFless+-l"), StaticRequest (MPS-r) and EagerHorizontal (FaST-GS+-like); the
report gives, from the integer tallies, the GPU saving of Dilu against Exclusive and MPS-l
(the paper: -30 % / -23 % at 3,200 instances), SVR, cold-start count (CSC) and saved GPU
time (SGT: a baseline's active GPU-seconds minus Dilu's, Table 3) per mode.

  python tools/modes_report.py [--scenarios 4096] [--slots 3600] [--out profiles/r2_modes_report.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import dilu_inputs as di  # noqa: E402

MODES = ["dilu", "exclusive", "static_limit", "static_request", "eager_horizontal"]


def summarise(tot, slot_ms, n_scen, T):
    t = {n: int(tot[i]) for i, n in enumerate(di.TALLY_NAMES)}
    act = max(t["gpu_slots_active"], 1)
    return {"avg_active_gpus_per_scenario": t["gpu_slots_active"] / (n_scen * T),
            "gpu_seconds": t["gpu_slots_active"] * slot_ms / 1000.0,
            "svr": t["req_violated"] / max(t["req_total"], 1),
            "csc": t["cold_starts"],
            "sm_frag": t["sm_unused_tokens"] / (act * 1000.0 * slot_ms),
            "mem_frag": t["mem_unused_mib_slots"] / (act * 40960.0),
            "placement_failures": t["placement_failures"],
            "scale_out_events": t["scale_out_events"], "scale_in_events": t["scale_in_events"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scenarios", type=int, default=4096)
    ap.add_argument("--slots", type=int, default=3600)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_modes_report.json"))
    a = ap.parse_args()
    from paper_2503_05130_b200 import DiluSim
    full = di.c4(n_scenarios=a.scenarios, T=a.slots)
    slot_ms = full.cfg["slot_ms"]
    res = {}
    for m, name in enumerate(MODES):
        wl = di.with_modes(full, [m] * full.S)
        sim = DiluSim.from_workload(wl)
        sim.scale_step(a.slots)
        _, tot = sim.metrics(per_scenario=False)
        res[name] = summarise(tot.cpu().numpy(), slot_ms, full.S, a.slots)
        sim.close()
    d = res["dilu"]
    rep = {"workload": f"C4 sweep, {full.S} scenarios x {a.slots} slots (every point under every mode)",
           "modes": res,
           "gpu_saving_vs_exclusive": 1 - d["gpu_seconds"] / res["exclusive"]["gpu_seconds"],
           "gpu_saving_vs_static_limit": 1 - d["gpu_seconds"] / res["static_limit"]["gpu_seconds"],
           "paper_context": "Dilu vs Exclusive -30 %, vs INFless+-l -23 % (P:1417, 3,200 instances, A100s)",
           "svr_reduction_vs_eager": res["eager_horizontal"]["svr"] - d["svr"],
           "csc_ratio_eager_over_dilu": res["eager_horizontal"]["csc"] / max(d["csc"], 1),
           "sgt_seconds_per_scenario_hour": {k: (res[k]["gpu_seconds"] - d["gpu_seconds"]) / full.S * 3600.0 / (a.slots * slot_ms / 1000.0)
                                             for k in MODES if k != "dilu"},
           "sgt_note": "SGT of a baseline = its active GPU-seconds minus Dilu's on the same fleet (Table 3 'saved GPU time', P:1295)"}
    print(json.dumps(rep, indent=1))
    if a.out:
        json.dump(rep, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
