"""Baseline modes pinned in the
oracle: Exclusive uses exactly one GPU per instance, limit-quota packing never
uses fewer GPUs than request-quota packing (per seed), a lone training worker
at full duty gets the same grants under Dilu and StaticLimit (S:554 reduction), and
eager scaling reacts to a burst the lazy window absorbs (S:463 vs S:490)."""
import numpy as np
import pytest

import dilu_inputs as di
import oracle
from test_oracle_sim import tiny, IDLE

T = {n: i for i, n in enumerate(di.TALLY_NAMES)}


def run_mode(wl, mode, n_slots=None, flags=3):
    return oracle.run(di.with_modes(wl, [mode] * wl.S), n_slots=n_slots, flags=flags)[1]


def test_exclusive_one_gpu_per_instance():
    """Exclusive GPU count equals the number of instances (here 7 on 8 GPUs)."""
    funcs = [dict(kind=0, req_pm=100, lim_pm=200, mem_mib=1024, affinity_class=1),
             dict(kind=2, prio=1, n_workers=3, req_pm=300, lim_pm=400, mem_mib=4096),
             dict(kind=1, req_pm=200, lim_pm=400, mem_mib=8192, work_per_batch=1),
             dict(kind=0, req_pm=100, lim_pm=200, mem_mib=1024, affinity_class=1)]
    wl = tiny(funcs, G=8)
    for mode, want in ((1, 6), (0, None)):
        s = oracle.RefSim(di.with_modes(wl, [mode]), flags=3)
        s.place_batch([0, 0, 0, 0], [0, 1, 2, 3])
        gpu, _ = s.snapshot(16)
        active = int((gpu[0, :, 3] > 0).sum())
        if want is not None:
            assert active == want and gpu[0, :, 3].max() == 1
        else:
            assert active < 6          # Dilu packs


@pytest.mark.parametrize("seed", range(4))
def test_request_packing_never_worse_than_limit_packing(seed):
    """S:549 (directional, per seed): Dilu's active GPU-slots <= StaticLimit's."""
    wl = di.c2(seed=seed, T=400)
    dilu = run_mode(wl, 0)
    slim = run_mode(wl, 2)
    assert dilu[T["gpu_slots_active"]] <= slim[T["gpu_slots_active"]]


def test_lone_training_worker_dilu_equals_static_limit():
    """with a single resident at full duty (demand = limit), Dilu's grant is the
    limit every slot (Alg.2 NONE) -- identical allocations and tallies to
    StaticLimit."""
    wl = tiny([dict(kind=2, prio=1, n_workers=1, req_pm=300, lim_pm=600, mem_mib=4096,
                    duty_pm=1000, arrive_sec=0, depart_sec=IDLE[1], cold_slots=2)], G=2,
              T_pat=50)
    a = run_mode(wl, 0, 50)
    b = run_mode(wl, 2, 50)
    assert np.array_equal(a, b)
    assert a[T["train_progress_tokens"]] == 48 * 600_000


def test_static_request_grants_request_only():
    """MPS-r: a lone worker at full duty executes only its request quota."""
    wl = tiny([dict(kind=2, prio=1, n_workers=1, req_pm=300, lim_pm=600, mem_mib=4096,
                    duty_pm=1000, arrive_sec=0, depart_sec=IDLE[1], cold_slots=0)], G=2,
              T_pat=20)
    t = run_mode(wl, 3, 20)
    assert t[T["train_progress_tokens"]] == 20 * 300_000


def test_exclusive_owns_whole_gpu():
    """Exclusive (pass-through): a lone inference instance whose demand exceeds
    its limit may use the whole GPU; under Dilu it is capped at the limit."""
    pat = np.full((1, 30), 200, np.int32)      # 200 req/s, IBS 1, c_b 5,000 -> d = 1e6
    f = dict(kind=0, req_pm=100, lim_pm=200, mem_mib=1024, ibs=1, work_per_batch=5000,
             arrive_sec=0, depart_sec=IDLE[1], scale_q10=1024, cold_slots=0)
    wl = tiny([f], G=2, patterns=pat)
    ex = run_mode(wl, 1, 30)
    dl = run_mode(wl, 0, 30)
    assert ex[T["inf_exec_tokens"]] == 30 * 1_000_000
    assert dl[T["inf_exec_tokens"]] == 30 * 200_000


def test_eager_scales_on_first_sample_lazy_absorbs():
    """A 5 s burst: EagerHorizontal scales out at the first second above capacity and
    back in afterwards (FaST-GS+ P:1158); Dilu's 40 s window absorbs it."""
    Tn = 120
    s_ = np.arange(Tn)
    pat = np.where((s_ >= 60) & (s_ < 65), 2000, 10).astype(np.int32)[None, :]
    f = dict(kind=0, req_pm=200, lim_pm=400, mem_mib=4096, work_per_batch=10000, ibs=4,
             cold_slots=2, arrive_sec=0, depart_sec=IDLE[1], scale_q10=1024)
    wl = tiny([f], G=8, patterns=pat)
    dilu = run_mode(wl, 0)
    eager = run_mode(wl, 4)
    assert dilu[T["scale_out_events"]] == 0 and dilu[T["cold_starts"]] == 1
    assert eager[T["scale_out_events"]] >= 1 and eager[T["scale_in_events"]] >= 1
    assert eager[T["cold_starts"]] > dilu[T["cold_starts"]]


def test_exclusive_training_runs_at_duty_of_whole_gpu():
    """Exclusive pass-through (D7): a lone worker with duty 0.8 owns the GPU, so
    its demand and grant are 0.8 * T_slot per slot (P:351 comm idle), not 0.8 * limit."""
    wl = tiny([dict(kind=2, prio=1, n_workers=1, req_pm=300, lim_pm=600, mem_mib=4096,
                    duty_pm=800, arrive_sec=0, depart_sec=IDLE[1], cold_slots=0)], G=2,
              T_pat=20)
    assert run_mode(wl, 1, 20)[T["train_progress_tokens"]] == 20 * 800_000
    assert run_mode(wl, 0, 20)[T["train_progress_tokens"]] == 20 * 480_000
