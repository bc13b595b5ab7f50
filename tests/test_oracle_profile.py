"""Pins for the profiler oracle (PAPER.md s3.2 P:604-639; SPEC S:96-233;
readings D9).  Values come from the paper (Table 2 trial counts P:669, "2% throughput
boost" P:631, limit = 2 x request P:637), from SPEC's worked examples (S:107, S:117-118,
S:192-193), from hand derivation, or from brute force over the 6 x 10 grid.
"""
import math

import numpy as np
import pytest

import dilu_inputs as di
import oracle


def prof(*sessions):
    if len(sessions) == 1 and isinstance(sessions[0], np.ndarray) and sessions[0].ndim == 1:
        arr = sessions[0]
    else:
        arr = np.zeros(len(sessions), di.PROF_SESSION)
        for k, x in enumerate(sessions):
            arr[k] = x
    return oracle.profile_batch(arr)


def test_perfmodel_spec_examples():
    """a = 5, b = 5, c = 50, IBS 4: 25 ms at SMR 100, 50 ms at SMR 50; flat beyond
    the knee."""
    m = di.prof_inference(5.0, 5.0, 50.0, 100.0)
    assert oracle.infer_exec_ms(m, 4, 100.0) == 25.0
    assert oracle.infer_exec_ms(m, 4, 50.0) == 50.0
    m2 = di.prof_inference(5.0, 5.0, 20.0, 100.0)          # knee(4) = 40
    assert oracle.infer_exec_ms(m2, 4, 60.0) == oracle.infer_exec_ms(m2, 4, 80.0)


def test_train_throughput_spec_examples():
    """SMR 100 -> workers * T_max * (1 - idle) exactly; a linear model at SMR
    80 -> 0.8 T_max; idle 0.4 -> 60 % of the compute-bound value (Figure 2a)."""
    m = di.prof_training(100.0, 250.0, 0.0, workers=3)
    assert oracle.train_tput(m, 100.0) == 750.0
    assert oracle.train_tput(di.prof_training(100.0, 250.0, 0.0), 80.0) == 200.0
    assert oracle.train_tput(di.prof_training(60.0, 100.0, 0.4), 100.0) == pytest.approx(60.0)


def test_training_bisection_linear_hand_derived():
    """T(smr) = smr, p = 0.8, +-2 %: probes 100 -> 50 -> 75 -> 87.5 -> 81.25, request
    81.25 in 5 trials.  Limit (p = 1.0, by hand): 50, 75, 87.5, 93.75, 96.875, 98.4375
    (|98.4375 - 100| <= 2) -> 6 more trials.  Q25: 81.25 % -> 813 per-mille."""
    o = prof(di.prof_training(100.0, 100.0, 0.0))[0]
    assert o["request_smr"] == 81.25 and o["limit_smr"] == 98.4375
    assert o["trials"] == 5 + 6 and o["status"] == 0
    assert o["req_pm"] == 813 and o["lim_pm"] == 985


def test_training_literal_stop_rule_flat_model():
    """P:631 'ends until the T_i satisfies T1*p +- 2%': with throughput flat above a knee
    at 60 the limit search (p = 1.0) stops at the first probe inside the band: 50 (0.833
    T1, below) then 75 (= T1) -> 75 (D9; SPEC's [58.8, 61.2] example assumes another rule)."""
    o = prof(di.prof_training(60.0, 100.0, 0.0))[0]
    assert o["limit_smr"] == 75.0


def test_training_bounds_and_order():
    """S:193 depth bound (<= 7 probes per p after T1 -> <= 15 trials), request <= limit
    (S:215), non-monotone oracle flagged."""
    ses = di.profile_sessions(20000, seed=3)
    ses = ses[ses["kind"] == 2]
    out = prof(ses)
    assert (out["trials"] <= 15).all() and (out["status"] == 0).all()
    assert (out["request_smr"] <= out["limit_smr"]).all()
    bad = prof(di.prof_training(100.0, 100.0, 1.5))[0]       # throughput falls with SMR
    assert bad["status"] == 2


def test_table2_trial_counts():
    """Table 2: Dilu profiles models (a)-(d) in 8 / 6 / 6 / 9 iterations."""
    out = prof(*[di.prof_inference(*m[1:]) for m in di.PROFILE_MODELS_V1])
    assert out["trials"].tolist() == [8, 6, 6, 9]
    assert (out["status"] == 0).all()


def test_roberta_marginal_effect():
    """'merely a 2% throughput boost for RoBERTa-large model with IBS=4, while
    increasing SMR doublely from 50% to 100%' (S:109 tolerance +-3 pp)."""
    m = di.prof_inference(*dict((x[0], x[1:]) for x in di.PROFILE_MODELS_V1)["roberta-large-like"])
    gain = oracle.infer_exec_ms(m, 4, 50.0) / oracle.infer_exec_ms(m, 4, 100.0) - 1.0
    assert 0.0 <= gain <= 0.05


def brute_force(m):
    """Exhaustive 6 x 10 grid (Table 2 'Traversal 60'): TE = IBS / (t_exec * SMR) over the
    feasible points t_exec <= SLO/2."""
    best = None
    for ibs in (1, 2, 4, 8, 16, 32):
        for s in range(10, 101, 10):
            t = oracle.infer_exec_ms(m, ibs, float(s))
            if t <= m["slo_ms"] / 2:
                te = ibs / (t * s)
                if best is None or te > best[0]:
                    best = (te, ibs, float(s))
    return best


def test_search_matches_traversal_on_builtin_profiles():
    """the exhaustive-grid TE maximizer equals the search result; limit = 2 x
    request."""
    for m in di.PROFILE_MODELS_V1:
        s = di.prof_inference(*m[1:])
        o = prof(s)[0]
        te, ibs, smr = brute_force(s)
        assert (o["ibs"], o["request_smr"]) == (ibs, smr)
        assert o["limit_smr"] == min(100.0, 2 * smr)
        assert o["trials"] < 60


def test_search_feasible_and_dominated_by_traversal():
    """Any profile: the returned point meets the SLO and its TE never exceeds the
    traversal maximum; an SLO below t_exec(1, 100) is unattainable."""
    ses = di.profile_sessions(3000, seed=5)
    ses = ses[ses["kind"] == 0][:600]
    out = prof(ses)
    for s, o in zip(ses, out):
        b = brute_force(s)
        if o["status"] == 1:
            assert b is None
            continue
        t = oracle.infer_exec_ms(s, int(o["ibs"]), float(o["request_smr"]))
        assert t <= s["slo_ms"] / 2 and t == o["t_exec_ms"]
        assert o["ibs"] / (t * o["request_smr"]) <= b[0] * (1 + 1e-12)
    m = di.prof_inference(5.0, 5.0, 50.0, 9.0)                    # t(1, 100) = 10 ms > 4.5
    assert prof(m)[0]["status"] == 1
