"""Run one workload through the C-ABI (the library DILU_LIB names) and, unless --no-check,
compare the tallies with the oracle.  Used under compute-sanitizer and for layout /
bounds-check variants.  Prints one line: PASS/FAIL <workload> <detail>.

  python tools/san_run.py c2 [--slots N] [--seed S]
  python tools/san_run.py c4slice [--slots N] [--every K]
  python tools/san_run.py c5win [--slots N]
  python tools/san_run.py c1
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import dilu_inputs as di  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", choices=["c1", "c2", "c4slice", "c5win", "c3win"])
    ap.add_argument("--slots", type=int, default=0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--every", type=int, default=91)
    ap.add_argument("--chunks", type=int, default=1)
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--flags", type=int, default=0, help="extra cfg.flags bits (4 alg2, 8 latency)")
    a = ap.parse_args()
    if a.workload == "c1":
        wl = di.c1()
    elif a.workload == "c2":
        wl = di.c2(seed=a.seed, T=a.slots or 3600)
    elif a.workload == "c4slice":
        full = di.c4(n_scenarios=4096, T=a.slots or 600)
        wl = full.subset(np.arange(5, 4096, a.every))
    elif a.workload == "c3win":
        wl = di.c3(seed=a.seed, T=a.slots or 600)
    else:
        wl = di.c5(n_scenarios=1, T=a.slots or 300, first_seed=50)
    if a.flags:
        cfg = dict(wl.cfg, flags=wl.cfg["flags"] | a.flags)
        wl = di.Workload(wl.name, cfg, wl.scen, wl.funcs, wl.patterns, wl.n_slots, wl.note)
    from paper_2503_05130_b200 import DiluSim
    import torch
    gs = DiluSim.from_workload(wl)
    n = wl.n_slots
    step = max(1, n // a.chunks)
    done = 0
    while done < n:
        k = min(step, n - done)
        gs.scale_step(k)
        done += k
    torch.cuda.synchronize()
    _, tot = gs.metrics()
    tot = tot.cpu().numpy()
    if a.no_check:
        print("DONE", wl.name, tot.tolist())
        return
    import oracle
    rs = oracle.RefSim(wl)
    rs.scale_step(n, threads=8)
    ref = rs.metrics()[1]
    ok = np.array_equal(tot, ref)
    print("PASS" if ok else "FAIL", wl.name, "" if ok else f"gpu {tot.tolist()} ref {ref.tolist()}")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
