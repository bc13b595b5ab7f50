"""Summarise `ncu --set full` reports of the bench kernel: duration, DRAM bytes, issue
active, ALU-pipe %, warps active, occupancy limits, stall breakdown, instructions; and the
source-level split of instructions / stall samples by kernel function.

  python tools/ncu_summary.py REPORT.ncu-rep [--json OUT.json --key C4 --source NOTE]

With --json the per-launch numbers are merged into OUT.json under KEY (the file bench.py
reads as profiles/r2_ncu_summary.json: dram_bytes_per_launch -> roofline.traffic)."""
import argparse
import csv
import io
import json
import re
import subprocess
from collections import defaultdict

METRICS = {
    "gpu__time_duration.sum": "duration_ms",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "launch__occupancy_limit_shared_mem": "occ_limit_smem_blocks",
    "launch__occupancy_limit_registers": "occ_limit_regs_blocks",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__block_size": "block_size",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__cycles_elapsed.avg": "sm_cycles",
    # regime reporting: L2 and DRAM throughput as % of peak
    "lts__throughput.sum.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "lts__t_sectors.sum.pct_of_peak_sustained_elapsed": "l2_sectors_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "memory_throughput_pct",
}
STALLS = ["barrier", "long_scoreboard", "short_scoreboard", "wait", "no_instruction", "selected",
          "not_selected", "math_pipe_throttle", "mio_throttle", "branch_resolving", "lg_throttle",
          "dispatch_stall", "membar", "sleeping", "drain", "misc", "tex_throttle"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    d = {}
    for i, n in enumerate(h):
        if n in METRICS:
            x = v[i].replace(",", "")
            try:
                val = float(x)
            except ValueError:
                continue
            if u[i] == "Mbyte":
                val *= 1e6
            elif u[i] == "Gbyte":
                val *= 1e9
            elif u[i] == "Kbyte":
                val *= 1e3
            elif u[i] in ("usecond", "us"):
                val /= 1e3
            elif u[i] in ("nsecond", "ns"):
                val /= 1e6
            elif u[i] in ("second", "s"):
                val *= 1e3
            elif u[i] == "Tbyte":
                val *= 1e12
            d[METRICS[n]] = val
        m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio", n)
        if m and m.group(1) in STALLS:
            try:
                d.setdefault("stall_per_issue", {})[m.group(1)] = float(v[i])
            except ValueError:
                pass
    d["dram_bytes_per_launch"] = d.get("dram_read_bytes", 0) + d.get("dram_write_bytes", 0)
    if d.get("duration_ms"):
        d["dram_gbs"] = d["dram_bytes_per_launch"] / d["duration_ms"] / 1e6   # achieved DRAM GB/s
    st = d.get("stall_per_issue", {})
    tot = sum(st.values()) or 1.0
    d["stall_share_pct"] = {k: round(100 * x / tot, 1) for k, x in sorted(st.items(), key=lambda kv: -kv[1]) if x > 0}
    return d


def by_function(rep, src_file):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, f = None, None
    inst, samp = defaultdict(float), defaultdict(float)
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if len(r) > 5 and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0].strip():
            k = (f, int(r[0]))
            inst[k] += float(r[hdr.index("Instructions Executed")] or 0)
            samp[k] += float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    src = open(src_file).read().split("\n")
    funcs = []
    for i, l in enumerate(src, 1):
        m = re.match(r"^(?:static |template|__global__|inline ).*?(\w+)\(", l)
        if m and not l.strip().endswith(";"):
            funcs.append((i, m.group(1)))

    def fn(line):
        name = "?"
        for a, n in funcs:
            if a <= line:
                name = n
        return name
    T, S = sum(inst.values()) or 1, sum(samp.values()) or 1
    agg = defaultdict(lambda: [0.0, 0.0])
    for (fl, l), x in inst.items():
        key = fn(l) if fl == src_file.split("/")[-1] else fl
        agg[key][0] += x
        agg[key][1] += samp[(fl, l)]
    top = sorted(agg.items(), key=lambda kv: -kv[1][0])[:20]
    lines = sorted(samp.items(), key=lambda kv: -kv[1])[:15]
    return ({k: {"inst_pct": round(100 * a / T, 1), "samples_pct": round(100 * b / S, 1)} for k, (a, b) in top},
            [{"line": l, "samples_pct": round(100 * x / S, 2),
              "src": src[l - 1].strip()[:100] if fl == src_file.split("/")[-1] else fl} for (fl, l), x in lines])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--src", default="paper_2503_05130_b200/csrc/sim_kernel.cuh")
    ap.add_argument("--json")
    ap.add_argument("--key", default="C4")
    ap.add_argument("--source", default="")
    ap.add_argument("--no-source-page", action="store_true")
    a = ap.parse_args()
    d = raw(a.report)
    if not a.no_source_page:
        d["by_function"], d["top_stall_lines"] = by_function(a.report, a.src)
    d["report"] = a.report
    if a.source:
        d["source"] = a.source
    print(json.dumps(d, indent=1))
    if a.json:
        try:
            allj = json.load(open(a.json))
        except Exception:
            allj = {}
        allj[a.key] = {k: d[k] for k in d if k not in ("by_function", "top_stall_lines")}
        json.dump(allj, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
