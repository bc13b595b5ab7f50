"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, element by
element on the same seeded inputs.  Integer tallies, the uint64 allocation hash,
placements (GPU state + every instance's GPUs/shares/ready slot) must be bit-exact.
Float ratios are derived on the host from identical integers (tol 1e-9 rel)."""
import os

import numpy as np
import pytest

import dilu_inputs as di
import oracle

pytestmark = pytest.mark.gpu
T = {n: i for i, n in enumerate(di.TALLY_NAMES)}


def gpu_sim(wl):
    from paper_2503_05130_b200 import DiluSim
    return DiluSim.from_workload(wl)


def compare_snapshots(gs, rs, id_cap, where=""):
    gg, gi = gs.snapshot(id_cap)
    rg, ri = rs.snapshot(id_cap)
    gg = gg.cpu().numpy(); gi = gi.cpu().numpy()
    bad = np.argwhere(gg != rg)
    assert bad.size == 0, f"{where}: GPU state differs at {bad[:5].tolist()}"
    badi = np.argwhere(gi != ri)
    assert badi.size == 0, (f"{where}: instance table differs at {badi[:5].tolist()}: "
                            f"gpu {gi[tuple(badi[0][:2])].tolist()} ref {ri[tuple(badi[0][:2])].tolist()}")


def compare_metrics(gs, rs, where=""):
    gper, gtot = gs.metrics()
    rper, rtot = rs.metrics()
    gper = gper.cpu().numpy(); gtot = gtot.cpu().numpy()
    if not np.array_equal(gper, rper):
        bad = np.argwhere(gper != rper)
        s, k = bad[0]
        raise AssertionError(f"{where}: tally {di.TALLY_NAMES[k]} of scenario {s}: "
                             f"gpu {gper[s, k]} ref {rper[s, k]} ({len(bad)} mismatches)")
    assert np.array_equal(gtot, rtot)
    return gtot


def ratios(t):
    """Final ratios (SURVEY s8(c) 'Final ratios'), host double from integers."""
    act = max(int(t[T["gpu_slots_active"]]), 1)
    return np.array([t[T["req_violated"]] / max(int(t[T["req_total"]]), 1),
                     t[T["sm_unused_tokens"]] / act, t[T["mem_unused_mib_slots"]] / act])


def run_pair(wl, chunks, id_cap=None, snap=True):
    gs, rs = gpu_sim(wl), oracle.RefSim(wl)
    id_cap = id_cap or 4 * wl.cfg["max_instances"]
    done = 0
    for n in chunks:
        gs.scale_step(n)
        rs.scale_step(n, threads=8)
        done += n
        if snap:
            compare_snapshots(gs, rs, id_cap, f"{wl.name} slot {done}")
    tot = compare_metrics(gs, rs, f"{wl.name} slot {done}")
    np.testing.assert_allclose(ratios(tot), ratios(rs.metrics()[1]), rtol=1e-9)
    return gs, rs, tot


def test_c1_appendix_a():
    wl = di.c1()
    gs, rs, tot = run_pair(wl, [1, 4, 20, 15, 1, 1, 49, 1, 1, 7], id_cap=16)
    assert tot[T["req_total"]] == 23610 and tot[T["req_violated"]] == 1250
    assert tot[T["train_progress_tokens"]] == 114500000


def test_c1_call_split_invariance():
    wl = di.c1()
    a = gpu_sim(wl); a.scale_step(100)
    b = gpu_sim(wl)
    for _ in range(100):
        b.scale_step(1)
    assert np.array_equal(a.metrics()[1].cpu().numpy(), b.metrics()[1].cpu().numpy())


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_c2_full_hour(seed):
    wl = di.c2(seed=seed)
    run_pair(wl, [1, 59, 540, 3000], id_cap=4096)


def test_c4_sample_full_hour():
    """C4 at full trace length on 48 scenarios spread over the 8^4 grid."""
    full = di.c4(n_scenarios=4096)
    wl = full.subset(np.arange(0, 4096, 87))
    run_pair(wl, [3600], snap=False)


@pytest.mark.parametrize("mode", ["cta_threads64", "cta_threads1024", "cta_no_smem", "cta_no_ovl",
                                  "cta_threads96", "cluster_k1", "cluster_k3"])
def test_launch_shape_invariance(mode, monkeypatch):
    """Both engines and several launch shapes give bit-identical results (45 scenarios)."""
    full = di.c4(n_scenarios=4096, T=600)
    wl = full.subset(np.arange(5, 4096, 91))
    engine, _, shape = mode.partition("_")
    monkeypatch.setenv("DILU_ENGINE", engine)
    if shape == "threads96":
        monkeypatch.setenv("DILU_THREADS", "96")
    if shape == "threads64":
        monkeypatch.setenv("DILU_THREADS", "64")
    elif shape == "threads1024":
        monkeypatch.setenv("DILU_THREADS", "1024")
    elif shape == "no_smem":
        monkeypatch.setenv("DILU_NO_SMEM", "1")
    elif shape == "no_ovl":          # placement pass not overlapped with P0/P1/P2
        monkeypatch.setenv("DILU_NO_OVL", "1")
    elif shape.startswith("k"):
        monkeypatch.setenv("DILU_CLUSTER", shape[1:])
    run_pair(wl, [1, 599], id_cap=2048)


@pytest.mark.parametrize("engine", ["cta", "cluster"])
def test_engines_on_c1_c2(engine, monkeypatch):
    monkeypatch.setenv("DILU_ENGINE", engine)
    run_pair(di.c1(), [1, 39, 1, 59], id_cap=16)
    run_pair(di.c2(seed=5, T=900), [1, 299, 600], id_cap=4096)


def test_c3_window():
    """C3 (1,024 GPUs, ~4,500 functions, state in HBM) for the first 30 minutes."""
    wl = di.c3(T=86400)
    run_pair(wl, [1, 299, 1500], id_cap=8192)


def test_c5_shaped_reduced():
    """C5-shaped (100 ms slots, diurnal mix) at reduced G for a full-trace parity."""
    wl = di.scaled("C5r", 2048, 1300, 2500, 7500, 100, 3000, [50, 51], max_instances=32768)
    run_pair(wl, [1, 9, 990, 2000], id_cap=20000)


def test_place_batch_matches_oracle():
    wl = di.c2(seed=3, T=300)
    F = wl.cfg["max_funcs"]
    rng = np.random.default_rng(0)
    req_f = rng.integers(0, F, 150)
    gs, rs = gpu_sim(wl), oracle.RefSim(wl)
    g_gpu, g_iid = gs.place_batch(np.zeros(150, np.int32), req_f)
    r_gpu, r_iid = rs.place_batch(np.zeros(150, np.int32), req_f)
    assert np.array_equal(g_iid.cpu().numpy(), r_iid)
    assert np.array_equal(g_gpu.cpu().numpy(), r_gpu)
    compare_snapshots(gs, rs, 2048, "after place_batch")
    gs.scale_step(300); rs.scale_step(300)
    compare_snapshots(gs, rs, 4096, "after place_batch + 300 slots")
    compare_metrics(gs, rs)


def test_llm_split_heavy():
    """Many LLM functions with big memory on few GPUs force worst-fit splits."""
    wl = di.c4(n_scenarios=4096, T=900).subset(np.arange(0, 640, 61))
    gs, rs, tot = run_pair(wl, [900], snap=False)
    assert tot[T["llm_split_placements"]] > 0


def test_capacity_error_matches():
    wl = di.c2(seed=0, T=200, max_instances=100)
    from paper_2503_05130_b200 import DiluError
    gs = gpu_sim(wl)
    gs.scale_step(200)
    with pytest.raises(DiluError) as e:
        gs.metrics()
    assert e.value.code == 6
    with pytest.raises(oracle.OracleError) as e2:
        rs = oracle.RefSim(wl)
        rs.scale_step(200)
    assert e2.value.code == 6


def test_degenerate_inputs():
    """All rows unused; a single GPU; zero arrivals."""
    wl = di.c1()
    funcs = wl.funcs.copy()
    funcs[:, :, 0] = -1
    empty = di.Workload("empty", wl.cfg, wl.scen, funcs, wl.patterns, 100)
    run_pair(empty, [100], id_cap=16)
    one = di.c2(seed=4, T=120)
    f1 = one.funcs.copy()
    f1[:, :, di.FI["n_workers"]] = np.minimum(f1[:, :, di.FI["n_workers"]], 1)
    one = di.Workload("G1", dict(one.cfg, gpus_per_scenario=1), one.scen, f1, one.patterns, 120)
    run_pair(one, [120], id_cap=1024)
    zero = di.c2(seed=5, T=120)
    zero = di.Workload("zero", zero.cfg, zero.scen, zero.funcs, np.zeros_like(zero.patterns), 120)
    run_pair(zero, [120], id_cap=1024)


# ------------------------------------------------------------------ full sizes
# BASELINE.json's full sizes in the launch configuration bench.py times; the oracle
# computes a sample of the outputs one by one (task contract).

def test_c4_full_size_sampled():
    """All 4,096 C4 scenarios for the full hour on the GPU (bench launch shape); 24
    scenarios spread over the sweep recomputed by the oracle, per-scenario bit-exact."""
    wl = di.c4(n_scenarios=4096)
    gs = gpu_sim(wl)
    gs.scale_step(wl.n_slots)
    per, tot = gs.metrics()
    per = per.cpu().numpy()
    idx = np.linspace(0, 4095, 24).round().astype(int)
    rper, _ = oracle.run(wl.subset(idx), threads=8)
    assert np.array_equal(per[idx], rper)
    assert tot.cpu().numpy()[T["gpu_row_slots"]] == 4096 * 64 * 3600


def test_c5_full_size_window():
    """One C5 scenario at full size (16,384 GPUs, ~90,500 functions, 100 ms slots, cluster
    engine) for the first 30 s, including the initial fleet placement: full state and
    tallies bit-exact against the oracle."""
    wl = di.c5(n_scenarios=1, T=36000)
    run_pair(wl, [10, 290], id_cap=160000)


@pytest.mark.slow
def test_c3_full_day():
    """C3 (1,024 GPUs, 24 h at 1 s slots): every tally of the whole day."""
    wl = di.c3(T=86400)
    run_pair(wl, [86400], snap=False)


# ------------------------------------------------------ baseline modes (s8(f) #1)

@pytest.mark.parametrize("mode", [1, 2, 3, 4])
def test_baseline_mode_c2(mode):
    wl = di.with_modes(di.c2(seed=6, T=900), [mode])
    run_pair(wl, [1, 299, 600], id_cap=4096)


@pytest.mark.parametrize("engine", ["cta", "cluster"])
def test_mixed_modes_c4_slice(engine, monkeypatch):
    """40 C4 sweep points, scenario i under mode i % 5, every engine."""
    monkeypatch.setenv("DILU_ENGINE", engine)
    wl = di.c4(n_scenarios=4096, T=600).subset(np.arange(3, 4096, 102))
    wl = di.with_modes(wl, np.arange(wl.S) % 5)
    run_pair(wl, [1, 599], id_cap=2048)


# ------------------------------------------- fused sub-second batches

@pytest.mark.parametrize("shape", ["cluster_b10", "cluster_b3", "cluster_b1", "cta_b10",
                                   "cta_b4"])
def test_fused_batches(shape, monkeypatch):
    """100 ms slots: the slots between two second boundaries run as one fused batch
    (DILU_BATCH = batch cap).  Cold starts shifted by 3 slots end mid-batch, calls start
    and end mid-window, and the five scenarios run modes 0..4."""
    engine, _, b = shape.partition("_")
    monkeypatch.setenv("DILU_ENGINE", engine)
    monkeypatch.setenv("DILU_BATCH", b[1:])
    wl = di.scaled("C5b", 512, 60, 120, 360, 100, 600, [53, 54, 55, 56, 57], max_instances=8192)
    funcs = wl.funcs.copy()
    live = funcs[:, :, di.FI["kind"]] >= 0
    funcs[:, :, di.FI["cold_slots"]] += 3 * live
    wl = di.with_modes(di.Workload("C5b", wl.cfg, wl.scen, funcs, wl.patterns, wl.n_slots),
                       [0, 1, 2, 3, 4])
    run_pair(wl, [1, 13, 7, 279, 300], id_cap=16384)


# ------------------------------- literal Algorithm 2 at 5 ms periods (s8(f) #2, D8)

def with_alg2(wl):
    cfg = dict(wl.cfg, flags=wl.cfg["flags"] | 4)
    return di.Workload(wl.name + "+alg2", cfg, wl.scen, wl.funcs, wl.patterns, wl.n_slots, wl.note)


@pytest.mark.parametrize("seed", [0, 3])
def test_alg2_c2(seed):
    """C2 with 200 Alg.2 periods per 1 s slot (CTA engine, state in shared memory)."""
    run_pair(with_alg2(di.c2(seed=seed, T=300)), [1, 119, 180], id_cap=4096)


@pytest.mark.parametrize("engine", ["cta", "cluster"])
def test_alg2_mixed_modes_c4_slice(engine, monkeypatch):
    """40 C4 sweep points under Alg.2, scenario i in baseline mode i % 5."""
    monkeypatch.setenv("DILU_ENGINE", engine)
    wl = di.c4(n_scenarios=4096, T=240).subset(np.arange(3, 4096, 102))
    wl = with_alg2(di.with_modes(wl, np.arange(wl.S) % 5))
    run_pair(wl, [1, 239], id_cap=2048)


def test_alg2_llm_split():
    """Alg.2 rows of split LLM instances (stage state per GPU, stage minima in P2)."""
    wl = with_alg2(di.c4(n_scenarios=4096, T=300).subset(np.arange(0, 640, 61)))
    gs, rs, tot = run_pair(wl, [300], snap=False)
    assert tot[T["llm_split_placements"]] > 0


@pytest.mark.parametrize("shape", ["cluster_b10", "cta_b10", "cta_b1"])
def test_alg2_fused_100ms(shape, monkeypatch):
    """100 ms slots (20 periods each) in fused batches, cold starts ending mid-batch."""
    engine, _, b = shape.partition("_")
    monkeypatch.setenv("DILU_ENGINE", engine)
    monkeypatch.setenv("DILU_BATCH", b[1:])
    wl = di.scaled("C5b", 512, 60, 120, 360, 100, 400, [53, 54], max_instances=8192)
    funcs = wl.funcs.copy()
    live = funcs[:, :, di.FI["kind"]] >= 0
    funcs[:, :, di.FI["cold_slots"]] += 3 * live
    wl = with_alg2(di.Workload("C5b", wl.cfg, wl.scen, funcs, wl.patterns, wl.n_slots))
    run_pair(wl, [1, 13, 186, 200], id_cap=16384)


# ------------------------------------------- request-level latency (s8(f) #4, D10)

def with_flags(wl, extra):
    cfg = dict(wl.cfg, flags=wl.cfg["flags"] | extra)
    return di.Workload(wl.name, cfg, wl.scen, wl.funcs, wl.patterns, wl.n_slots, wl.note)


def latency_pair(wl, chunks, id_cap=None):
    gs, rs, tot = run_pair(wl, chunks, id_cap=id_cap)
    gl, gsum = gs.latency()
    rl, rsum = rs.latency()
    assert np.array_equal(gl, rl), f"latency differs at {np.argwhere(gl != rl)[:5].tolist()}"
    assert gsum[:79].sum() == tot[T["req_served"]] and gsum[79] == tot[T["req_violated"]]
    return gsum


@pytest.mark.parametrize("seed", [0, 2])
def test_latency_c2(seed):
    lat = latency_pair(with_flags(di.c2(seed=seed, T=600), 8), [1, 299, 300], id_cap=4096)
    assert lat[81] > 0


@pytest.mark.parametrize("engine", ["cta", "cluster"])
def test_latency_modes_c4_slice(engine, monkeypatch):
    monkeypatch.setenv("DILU_ENGINE", engine)
    wl = di.c4(n_scenarios=4096, T=300).subset(np.arange(7, 4096, 102))
    latency_pair(with_flags(di.with_modes(wl, np.arange(wl.S) % 5), 8), [1, 299], id_cap=2048)


def test_latency_llm_split_and_alg2():
    wl = di.c4(n_scenarios=4096, T=240).subset(np.arange(0, 640, 61))
    latency_pair(with_flags(wl, 8), [240])
    latency_pair(with_flags(wl, 8 | 4), [240])


@pytest.mark.parametrize("shape", ["cluster_b10", "cta_b10"])
def test_latency_fused_100ms(shape, monkeypatch):
    engine, _, b = shape.partition("_")
    monkeypatch.setenv("DILU_ENGINE", engine)
    monkeypatch.setenv("DILU_BATCH", b[1:])
    wl = di.scaled("C5b", 512, 60, 120, 360, 100, 400, [53, 54], max_instances=8192)
    latency_pair(with_flags(wl, 8), [1, 13, 386], id_cap=16384)
    latency_pair(with_flags(wl, 8 | 4), [1, 13, 386], id_cap=16384)


def test_latency_requires_flag():
    from paper_2503_05130_b200 import DiluError
    gs = gpu_sim(di.c1())
    gs.scale_step(5)
    with pytest.raises(DiluError) as e:
        gs.latency()
    assert e.value.code == 1


# ------------------------------------------- round-2 parity gaps (VERDICT r1 "next" #2)

@pytest.mark.parametrize("engine", ["cta", "cluster"])
def test_place_batch_engines(engine, monkeypatch):
    """dilu_place_batch on both engines, several scenarios, the initial fleet as requests
    (what bench.py's placements/s times), then slots."""
    monkeypatch.setenv("DILU_ENGINE", engine)
    wl = di.c4(n_scenarios=4096, T=300).subset(np.arange(11, 4096, 409))
    kind = wl.funcs[:, :, di.FI["kind"]]
    arr = wl.funcs[:, :, di.FI["arrive_sec"]]
    s_idx, f_idx = np.nonzero((kind != di.K_UNUSED) & (arr == 0))
    rs_, rf_ = s_idx.astype(np.int32), f_idx.astype(np.int32)
    gs, rs = gpu_sim(wl), oracle.RefSim(wl)
    g_gpu, g_iid = gs.place_batch(rs_, rf_)
    r_gpu, r_iid = rs.place_batch(rs_, rf_)
    assert np.array_equal(g_iid.cpu().numpy(), r_iid)
    assert np.array_equal(g_gpu.cpu().numpy(), r_gpu)
    compare_snapshots(gs, rs, 2048, "after place_batch")
    gs.scale_step(300); rs.scale_step(300, threads=8)
    compare_snapshots(gs, rs, 4096, "after place_batch + 300 slots")
    compare_metrics(gs, rs)


def test_same_slot_warm_cold0():
    """cold_slots = 0: an instance placed at a boundary serves in that same slot, so the
    overlapped-slot schedule is off (host check) and the serial path runs."""
    wl = di.c4(n_scenarios=4096, T=600).subset(np.arange(2, 4096, 127))
    funcs = wl.funcs.copy()
    live = funcs[:, :, di.FI["kind"]] >= 0
    funcs[:, :, di.FI["cold_slots"]] = np.where(live, 0, funcs[:, :, di.FI["cold_slots"]])
    wl = di.Workload("C4cold0", wl.cfg, wl.scen, funcs, wl.patterns, wl.n_slots)
    run_pair(wl, [1, 99, 500], id_cap=2048)


def test_mixed_cold_zero_and_positive():
    """Half the functions with cold_slots = 0 (one zero anywhere turns the overlap off)."""
    wl = di.c2(seed=4, T=900)
    funcs = wl.funcs.copy()
    f = np.arange(funcs.shape[1])
    funcs[:, f % 2 == 0, di.FI["cold_slots"]] = 0
    wl = di.Workload("C2cold0", wl.cfg, wl.scen, funcs, wl.patterns, wl.n_slots)
    run_pair(wl, [1, 299, 600], id_cap=4096)


@pytest.mark.parametrize("parts", [2, 3, 5])
def test_shard_invariance_gpu(parts):
    """P handles on one GPU over contiguous scenario blocks sum to the 1-handle tallies
    bit-exactly (the multi-GPU aggregate); per-scenario rows match too."""
    wl = di.c4(n_scenarios=4096, T=400).subset(np.arange(1, 4096, 157))
    full = gpu_sim(wl)
    full.scale_step(400)
    fper, ftot = full.metrics()
    acc = np.zeros(17, dtype=np.int64)
    rows = []
    for r in range(parts):
        sh = gpu_sim(wl.shard(r, parts))
        sh.scale_step(400)
        per, tot = sh.metrics()
        acc = (acc.view(np.uint64) + tot.cpu().numpy().view(np.uint64)).view(np.int64)
        rows.append(per.cpu().numpy())
    assert np.array_equal(acc, ftot.cpu().numpy())
    assert np.array_equal(np.concatenate(rows), fper.cpu().numpy())


def _two_rank_worker(rank, world, port, out):
    import torch
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK="0",
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    from paper_2503_05130_b200 import DiluSim, dist as ddist
    ddist.init("gloo")
    wl = di.c4(n_scenarios=4096, T=300).subset(np.arange(7, 4096, 211))
    sim = DiluSim.from_workload(wl.shard(rank, world), device="cuda:0")
    sim.scale_step(300)
    _, tot = sim.metrics(per_scenario=False)
    ddist.allreduce_tallies(tot)
    out[rank] = tot.cpu().numpy().tolist()
    ddist.barrier()
    ddist.finalize()


def test_two_ranks_one_gpu_reproduce_one_rank():
    """Two processes (two handles) on one GPU, the scenario sharder's all-reduce over a
    process group (gloo: NCCL refuses two ranks on one device), reproduce the 1-rank
    tallies bit-exactly."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_two_rank_worker, args=(2, port, out), nprocs=2, join=True)
    wl = di.c4(n_scenarios=4096, T=300).subset(np.arange(7, 4096, 211))
    one = gpu_sim(wl)
    one.scale_step(300)
    _, tot = one.metrics(per_scenario=False)
    ref = tot.cpu().numpy()
    for r in range(2):
        assert np.array_equal(np.array(out[r], dtype=np.int64), ref)


def test_c5_bench_shape_window():
    """C5 in the bench launch shape (8 x 16,384-GPU scenarios, 100 ms slots, cluster engine
    at its bench cluster size) against the oracle over the first 600 slots (incl. the
    initial ~28k-instance fleet placement per scenario)."""
    wl = di.c5(n_scenarios=8, T=600, first_seed=50)
    run_pair(wl, [600], snap=False)


def test_c5_timed_window_vs_frozen_oracle():
    """C5 at the bench's full timed window (8 x 16,384 GPUs, 36,000 x 100 ms slots, the bench
    launch shape) against the oracle's per-scenario tallies frozen by
    tools/freeze_c5_golden.py (a committed script that calls only oracle/)."""
    import json
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c5_window_tallies.json")))
    wl = di.c5(n_scenarios=8, T=36000, first_seed=50)
    gs = gpu_sim(wl)
    gs.scale_step(36000)
    per, tot = gs.metrics()
    assert np.array_equal(per.cpu().numpy(), np.array(gold["per_scenario"], dtype=np.int64))
    assert np.array_equal(tot.cpu().numpy(), np.array(gold["sum"], dtype=np.int64))


def test_modes_directional_c4_slice():
    """SURVEY s8(f) #1 directional claims on the GPU path (paper-level, absolute values
    unpinned; Table 3): on the same C4 sweep points Dilu occupies no more GPU-slots
    than StaticLimit (MPS-l) or Exclusive, and the lazy window starts no more instances cold
    than eager (FaST-GS+-like) scaling."""
    base = di.c4(n_scenarios=4096, T=900).subset(np.arange(9, 4096, 137))
    tot = {}
    for m in (0, 1, 2, 4):
        gs = gpu_sim(di.with_modes(base, [m] * base.S))
        gs.scale_step(900)
        tot[m] = gs.metrics(per_scenario=False)[1].cpu().numpy()
    act = {m: tot[m][T["gpu_slots_active"]] for m in tot}
    assert act[0] <= act[2] and act[0] <= act[1], act
    assert tot[0][T["cold_starts"]] <= tot[4][T["cold_starts"]]


@pytest.mark.parametrize("shape", ["g8c2", "g6c3", "g4c1", "g8c2serial"])
def test_multicluster_groups(shape, monkeypatch):
    """Scenario groups of several hardware clusters (scenario-wide barriers in global
    memory, placement inside the leader's cluster): C2, a C5-shaped reduced
    trace and fused 100 ms batches, bit-exact against the oracle -- with the placement pass
    overlapped with the batch (the default when every cold start is >= one batch) and, for
    `serial`, without."""
    if shape.endswith("serial"):
        monkeypatch.setenv("DILU_NO_OVL", "1")
        shape = shape[:-len("serial")]
    k, kc = shape[1:].split("c")
    monkeypatch.setenv("DILU_ENGINE", "cluster")
    monkeypatch.setenv("DILU_GROUP", k)
    monkeypatch.setenv("DILU_CLUSTER", kc)
    run_pair(di.c2(seed=7, T=600), [1, 299, 300], id_cap=4096)
    wl = di.scaled("C5g", 2048, 200, 400, 1200, 100, 900, [52, 53], max_instances=8192)
    run_pair(wl, [1, 13, 886], id_cap=8192, snap=False)


# ---- device state invariants (cfg.flags bit1) ---------------

@pytest.mark.parametrize("case", ["c1", "c2", "c4slice_modes", "c5r", "llm_split", "alg2"])
def test_invariant_checks_clean(case, monkeypatch):
    """With cfg.flags bit1 the device checks I1-I3 and I7 after every call and dilu_metrics
    checks I6; on the paper's loop none may fire, and the tallies stay those of the oracle
    (which runs its own per-slot checks with the same bit)."""
    if case == "c1":
        wl, chunks = di.c1(), [1] * 30 + [70]
    elif case == "c2":
        wl, chunks = di.c2(seed=2, T=600), [1, 1, 98, 500]
    elif case == "c4slice_modes":
        base = di.c4(n_scenarios=4096, T=300).subset(np.arange(3, 4096, 257))
        wl, chunks = di.with_modes(base, np.arange(base.S) % 5), [1, 299]
    elif case == "c5r":
        monkeypatch.setenv("DILU_ENGINE", "cluster")
        wl, chunks = di.scaled("C5i", 2048, 200, 400, 1200, 100, 600, [54], max_instances=8192), [1, 9, 590]
    elif case == "llm_split":     # the C4 sweep points with worst-fit splits (test_llm_split_heavy)
        wl, chunks = di.c4(n_scenarios=4096, T=300).subset(np.arange(0, 640, 61)), [1, 299]
    else:
        wl, chunks = with_flags(di.c2(seed=4, T=300), 4), [1, 299]
    run_pair(with_flags(wl, 2), chunks, snap=False)


def test_invariant_violation_detected():
    """A corrupted GPU row (R_g one above the sum over its residents) is reported as
    DILU_E_INVARIANT by the next call's device check (I3)."""
    from paper_2503_05130_b200 import DiluError
    wl = with_flags(di.c2(seed=1, T=200), 2)
    gs = gpu_sim(wl)
    gs.scale_step(100)
    gs.metrics()                                          # clean so far
    gg, _ = gs.snapshot(1)
    R = gg.cpu().numpy()[0, :, 0].astype(np.int32)        # this scenario's R_g row
    g = int(np.argmax(R))
    assert R[g] > 0
    import torch
    ws = gs.workspace.view(torch.int32)
    W = ws.cpu().numpy()
    hits = np.flatnonzero(np.all(np.lib.stride_tricks.sliding_window_view(W, R.size) == R, axis=1))
    assert hits.size >= 1                                 # the gR array of the state block
    ws[int(hits[0]) + g] += 1
    gs.scale_step(1)
    with pytest.raises(DiluError) as e:
        gs.metrics()
    assert e.value.code == 2                              # DILU_E_INVARIANT
