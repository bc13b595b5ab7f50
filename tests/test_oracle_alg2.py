"""Pins for the oracle's literal Algorithm 2 at 5 ms periods (
PAPER.md:975-1039 Alg. 2, P:885-902 workflow; SPEC S:322-414 vscaler; readings D8).

Each pin is a value fixed by the paper / SPEC text or derived by hand from it, not a
re-run of the oracle's own expressions:
  - the Algorithm 2 branch table (SPEC examples S:383-386);
  - the KLC arithmetic of a lone SLO resident, derived by hand period by period;
  - the drain's physical capacity clamp;
  - EMERGENCY ownership;
  - properties that hold for any row (grant ceiling S:401, work conservation).
"""
import numpy as np
import pytest

import dilu_inputs as di
import oracle
from test_oracle_sim import tiny, IDLE

T = {n: i for i, n in enumerate(di.TALLY_NAMES)}
NEVER = -(1 << 30)


def fresh(n):
    return np.tile(np.array([0, 0, 0, NEVER], np.int32), (n, 1))


def test_lone_best_effort_gets_limit():
    """Alg.2 line 29 'Without collocation instances': R_issue = MaxTokens * limit."""
    ex, gr = oracle.alg2_row([1], [7], [1500], [3000], [10 ** 6], [0], 200)
    assert (gr == 3000).all()
    assert ex[0] == 200 * 3000


def test_emergency_scales_best_effort_down():
    """SLO dT = 1.0 > eta_violation; collocated BE with R_last = 1000 and
    MaxTokens*request = 600 gets min(600, 1000) / 1 = 600; the SLO gets MaxTokens*limit.
    The KLC doubles 25 ms -> 50 ms as in P:899 ('from 25ms to 50ms')."""
    rs = fresh(2)
    rs[0, :2] = (50_000, 25_000)         # SLO: T_current 50 ms, T_min 25 ms -> dT = 1000
    rs[0, 3] = 0                         # executed recently
    rs[1, 2:] = (1000, 0)                # BE: R_last 1000
    gs = np.array([0, -1, 0], np.int32)
    _, gr = oracle.alg2_row([0, 1], [4, 9], [2000, 600], [4000, 2500], [10 ** 6, 10 ** 6],
                            [10 ** 6, 0], 1, p0=5, res_state=rs, gpu_state=gs)
    assert gr[0].tolist() == [4000, 600]
    assert gs.tolist() == [1, 4, 1000]      # EMERGENCY, owner id 4, dT 1000


@pytest.mark.parametrize("t_cur,want", [(37_500, 600), (75_000, 300), (125_000, 150)])
def test_emergency_divisor_clamp(t_cur, want):
    """Line 26 divides by dT; SPEC's clamp max(dT, 1) keeps 0.3 < dT < 1 from
    raising the BE grant: dT = 0.5 -> 600, dT = 2 -> 300, dT = 4 -> 150."""
    rs = fresh(2)
    rs[0, :2] = (t_cur, 25_000)
    rs[0, 3] = 0
    rs[1, 2:] = (1000, 0)
    _, gr = oracle.alg2_row([0, 1], [4, 9], [2000, 600], [4000, 2500], [10 ** 6, 10 ** 6],
                            [10 ** 6, 0], 1, p0=5, res_state=rs)
    assert gr[0, 1] == want


def test_idle_slo_lets_best_effort_ramp_to_limit():
    """an idle SLO resident (no kernels in RW, line 16) gets MaxTokens*request
    and state RECOVERY; the BE resident grows by eta_increase = 1.25 per period (ceil)
    until MaxTokens*limit (line 33)."""
    rs = fresh(2)
    rs[1, 2:] = (1000, 0)
    _, gr = oracle.alg2_row([0, 1], [4, 9], [2000, 600], [4000, 4000], [0, 10 ** 6], [3000, 0],
                            10, p0=1, res_state=rs)
    assert (gr[:, 0] == 2000).all()
    assert gr[:, 1].tolist() == [1250, 1563, 1954, 2443, 3054, 3818, 4000, 4000, 4000, 4000]


def test_capacity_clamp():
    """two instances granted 3000 + 3000 on a 5000-token period execute 3000 and
    2000 (in (prio, id) order); the BE-only row stays NONE."""
    ex, gr = oracle.alg2_row([1, 1], [2, 5], [1000, 1000], [3000, 3000], [10 ** 6, 10 ** 6],
                             [0, 0], 4)
    assert (gr == 3000).all()
    assert ex.tolist() == [4 * 3000, 4 * 2000]


def test_klc_hand_derived():
    """A lone SLO resident, request 2500, limit 5000, batches of 2500 tokens.  By hand
    (blocks run at the period's rate y, 1 token = 1 us of the whole GPU):
      p0: idle -> R = 2500 (line 17); batch 0 takes the whole 5 ms: T = 5000 us
      p1: RW busy, others idle -> R = ceil(2500*1.25) = 3125 (line 19); batch 1 runs
          2500 tokens at 3125/5 ms: T = 4000 us
      p2: R = ceil(3125*1.25) = 3907; batch 2 started at 9000 us, ends at
          10000 + ceil(1875*5000/3907) = 12400: T = 3400 us
      p3: R = 4884; batch 3 ends at 15480 (start 12399): 3081 us; batch 4 runs
          15479 -> 18039: T = 2560 us."""
    want_tmin = {1: 5000, 2: 4000, 3: 3400, 4: 2560}
    for NP, tmin in want_tmin.items():
        rs = fresh(1)
        ex, gr = oracle.alg2_row([0], [3], [2500], [5000], [25_000], [2500], NP, res_state=rs)
        assert rs[0, 1] == tmin and rs[0, 0] == tmin
    assert gr[:, 0].tolist() == [2500, 3125, 3907, 4884]
    assert ex[0] == 2500 + 3125 + 3907 + 4884


def test_emergency_ownership():
    """P:1003 'Only the current instance can reset or modify the EMERGENCY state';
    S:398: with two SLO residents tripping line 14, the larger dT owns it."""
    def run(dt_b, b_idle=False):
        rs = fresh(2)
        rs[0, :2] = (37_500, 25_000)                    # A: dT 500
        rs[1, :2] = (25_000 + dt_b * 25, 25_000)        # B: dT dt_b
        rs[:, 3] = 0
        if b_idle:
            rs[1, :2] = (25_000, 25_000)
            rs[1, 3] = NEVER
        gs = np.array([0, -1, 0], np.int32)
        oracle.alg2_row([0, 0], [1, 2], [1000, 1000], [3000, 3000], [10 ** 6, 10 ** 6],
                        [100, 100], 1, p0=3, res_state=rs, gpu_state=gs)
        return gs.tolist()
    assert run(400) == [1, 1, 500]
    assert run(600) == [1, 2, 600]
    assert run(0, b_idle=True) == [1, 1, 500]            # idle non-owner leaves it in place


def test_lost_owner_resets_state():
    """An EMERGENCY whose owner left the GPU does not bind the others (D8): the row
    behaves as from NONE, the SLO resident's own branch sets the state."""
    rs = fresh(2)
    rs[1, 2:] = (1000, 0)
    gs = np.array([1, 99, 4000], np.int32)
    _, gr = oracle.alg2_row([0, 1], [4, 9], [2000, 600], [4000, 2500], [0, 10 ** 6], [3000, 0],
                            1, p0=2, res_state=rs, gpu_state=gs)
    assert gs[0] == 2 and gr[0].tolist() == [2000, 1250]   # RECOVERY, BE ramps


def test_random_rows_properties():
    """Any row: grants within [0, MaxTokens*limit], executed <= demand, executed
    <= sum of grants, row total <= NP * MaxTokens."""
    rng = np.random.default_rng(7)
    for _ in range(300):
        n = int(rng.integers(1, 7))
        NP = int(rng.integers(1, 60))
        prio = rng.integers(0, 2, n)
        req = rng.integers(50, 600, n) * 5
        lim = np.minimum(req * rng.integers(1, 4, n), 5000)
        d = rng.integers(0, 200_000, n)
        cst = np.where(prio == 0, rng.integers(100, 20_000, n), 0)
        rs = fresh(n)
        rs[:, 0] = rng.integers(0, 40_000, n)
        rs[:, 1] = np.where(rng.random(n) < 0.5, 0, rng.integers(1, 20_000, n))
        rs[:, 2] = rng.integers(0, lim + 1)          # reachable: R_last <= limit
        rs[:, 3] = np.where(rng.random(n) < 0.5, NEVER, rng.integers(0, 30, n))
        gs = np.array([rng.integers(0, 4), -1, 0], np.int32)
        ex, gr = oracle.alg2_row(prio, np.arange(n) * 3 + 1, req, lim, d, cst, NP, p0=30,
                                 res_state=rs, gpu_state=gs)
        assert (gr >= 0).all() and (gr <= lim[None, :]).all()
        assert (ex <= d).all() and (ex <= gr.sum(0)).all()
        assert ex.sum() <= NP * 5000


def test_loop_lone_training_worker_matches_closed_form():
    """A lone training worker: Alg.2 NONE grants the limit every period, so it executes
    min(d, lim_tok) per slot -- the closed form's grant for a lone instance (Q13 (iii))."""
    wl = tiny([dict(kind=2, prio=1, n_workers=1, req_pm=300, lim_pm=600, mem_mib=4096,
                    duty_pm=800, arrive_sec=0, depart_sec=IDLE[1], cold_slots=2)], G=2,
              T_pat=30)
    a = oracle.run(wl, 30, flags=3)[1]
    b = oracle.run(wl, 30, flags=7)[1]
    assert b[T["train_progress_tokens"]] == a[T["train_progress_tokens"]] == 28 * 480_000


@pytest.mark.parametrize("seed", [0, 1])
def test_loop_invariants_c2(seed):
    """C2 at 100 ms slots (20 periods per slot) under Alg.2 with the invariant checks on
    (flags bit1: I1-I7 with I4 relaxed to 0 <= a <= limit, I5 per GPU-slot)."""
    wl = di.scaled("C2a", 64, 12, 20, 60, 100, 600, [seed], max_instances=2048)
    per, tot = oracle.run(wl, flags=7)
    assert tot[T["gpu_row_slots"]] == 64 * 600
    assert tot[T["req_served"]] + tot[T["req_violated"]] == tot[T["req_total"]]
    assert tot[T["sm_unused_tokens"]] >= 0


def test_alg2_needs_5ms_periods():
    wl = di.c1()
    cfg = dict(wl.cfg, slot_ms=8)
    bad = di.Workload("bad", cfg, wl.scen, wl.funcs, wl.patterns, 10)
    with pytest.raises(oracle.OracleError):
        oracle.RefSim(bad, flags=5)
