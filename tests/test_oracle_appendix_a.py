"""Pin the oracle to SURVEY.md Appendix A (C1 worked example, hand-derived).

Every expected number comes from tests/golden/c1_appendix_a.json, which cites the
appendix row it restates.  A dropped term (e.g. the gang minimum, Q22), a wrong
order (SLO-first spare sharing), a wrong window comparison or a wrong tie-break
each moves at least one of these values.
"""
import json
import os

import numpy as np
import pytest

import dilu_inputs as di
import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c1_appendix_a.json")))
T = {n: i for i, n in enumerate(di.TALLY_NAMES)}


def test_totals():
    per, tot = oracle.run(di.c1(), flags=3)
    for k, v in GOLD["totals"].items():
        if k.startswith("_"):
            continue
        assert tot[T[k]] == v, k
    # I6 conservation
    assert tot[T["req_total"]] == tot[T["req_served"]] + tot[T["req_violated"]]


def test_placement_at_s0():
    s = oracle.RefSim(di.c1(), flags=3)
    s.scale_step(1)
    gpu, inst = s.snapshot(16)
    g = GOLD["placement_s0"]
    assert list(inst[0, :7, 4]) == g["instance_gpu"]
    assert gpu[0, :, :3].tolist() == g["gpu_RLU"]
    assert inst[0, 7, 1] == -1   # no further ids issued at s=0


def test_select_key_i6():
    """The R6 fit key for I6 on G1/G2 (Appendix A) and the paper's float score order."""
    k = GOLD["placement_s0"]["key_I6"]
    M, Q = 40960, 1000
    assert 950 * M + 32768 * Q == k["G1"]
    assert 700 * M + 18432 * Q == k["G2"]
    # oracle SelectOptGPU over {G1, G2} with the pre-I6 state picks G1
    R = np.array([650, 650, 400, 0], np.int32)
    L = np.array([1300, 1000, 500, 0], np.int32)
    U = np.array([12288, 24576, 10240, 0], np.int32)
    n = np.array([3, 2, 1, 0], np.int32)
    cand = np.array([0, 1, 2], np.int32)
    assert oracle.lib().dilu_ref_select_opt_gpu(3, cand, R, L, U, n, 300, 400, 8192, 1000, 1500,
                                                M, Q, 1, 1) == 1


def test_scale_events():
    s = oracle.RefSim(di.c1(), flags=3)
    s.scale_step(41)                       # slots 0..40 -> boundary s=40 done
    gpu, inst = s.snapshot(16)
    e = GOLD["scale_events"]
    assert inst[0, 7, 4] == e["s40"]["I7"] and inst[0, 8, 4] == e["s40"]["I8"]
    assert inst[0, 7, 3] == e["s40"]["ready"] and inst[0, 8, 3] == e["s40"]["ready"]
    assert gpu[0, 2, :3].tolist() == e["s40"]["G2_RLU_after"]
    s.scale_step(91 - 41)                  # through slot 90: still held
    gpu, inst = s.snapshot(16)
    assert inst[0, 8, 1] == 1
    s.scale_step(1)                        # slot 91: ScaleIn removes I8
    gpu, inst = s.snapshot(16)
    assert inst[0, 8, 1] == 2 and inst[0, 7, 1] == 1
    assert gpu[0, 2, :3].tolist() == e["s91_G2_RLU"]
    s.scale_step(1)                        # slot 92: ScaleIn removes I7
    gpu, inst = s.snapshot(16)
    assert inst[0, 7, 1] == 2
    assert gpu[0, 2, :3].tolist() == e["s92_G2_RLU"]
    s.scale_step(8)
    per, tot = s.metrics()
    assert tot[T["scale_in_events"]] == 2


@pytest.mark.parametrize("key", [k for k in GOLD["slots"] if not k.startswith("_")])
def test_slot_allocations(key):
    spec = GOLD["slots"][key]
    slot = int(key[1:key.index("_")])
    g = int(key[key.index("G") + 1:])
    s = oracle.RefSim(di.c1(), flags=3)
    s.scale_step(slot + 1)
    a, r, ex = s.slot_detail(0, 16)
    for name, v in spec.get("a", {}).items():
        i = int(name[1:])
        assert a[i, 0] == v, (key, name)
    for name, v in spec.get("r", {}).items():
        assert r[int(name[1:])] == v, (key, name)
    assert 1_000_000 - ex[g] == spec["unused"], key
