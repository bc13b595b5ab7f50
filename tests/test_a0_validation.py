"""a0 reject-path parity (SURVEY s8(a) a0, s8(b) "validate_spec -> ok | violations"):
one invalid input per validation rule; the CUDA library's dilu_sim_create and the oracle's
dilu_ref_create must both reject it with DILU_E_USAGE and name the same scenario, function
and rule.  Validation runs on the host before any device work, so this needs no GPU."""
import ctypes as C
import re

import numpy as np
import pytest

import dilu_inputs as di
import oracle

CF, FF = di.CONFIG_FIELDS, di.FI


def base():
    wl = di.c2(seed=1, T=60)
    return wl.cfg_array().copy(), wl.scen.copy(), wl.funcs.copy(), wl.patterns.copy()


def first_used(funcs, kind):
    k = funcs[0, :, FF["kind"]]
    return int(np.nonzero(k == kind)[0][0])


def cfg_set(name, v):
    def m(cfg, scen, funcs, pats):
        cfg[CF.index(name)] = v
    return m


def func_set(kind, field, v, also=None):
    def m(cfg, scen, funcs, pats):
        f = first_used(funcs, kind)
        funcs[0, f, FF[field]] = v
        for k2, v2 in (also or {}).items():
            funcs[0, f, FF[k2]] = v2
        return f
    return m


def scen_set(col, v):
    def m(cfg, scen, funcs, pats):
        scen[0, col] = v
    return m


# (mutation, tag words either side's message must contain, expects a (scenario, func) name)
CASES = [
    ("q_pm", cfg_set("q_pm", 999), ["q_pm"], False),
    ("mem_mib", cfg_set("mem_mib", 0), ["mem_mib"], False),
    ("alpha_beta", lambda c, s, f, p: (cfg_set("alpha_w", 0)(c, s, f, p), cfg_set("beta_w", 0)(c, s, f, p)),
     ["alpha"], False),
    ("slot_ms", cfg_set("slot_ms", 7), ["slot_ms"], False),
    ("window", cfg_set("phi_in", 5), ["phi_out"], False),
    ("min_instances", cfg_set("min_instances", 0), ["min_instances"], False),
    ("max_residents", cfg_set("max_residents", 16), ["max_residents"], False),
    ("max_llm_stages", cfg_set("max_llm_stages", 5), ["max_llm_stages"], False),
    ("omega", scen_set(1, 1200), ["omega"], False),
    ("gamma_lt_omega", scen_set(2, 900), ["gamma"], False),
    ("mode", scen_set(3, 9), ["mode"], False),
    ("kind", func_set(di.K_INF, "kind", 5), ["kind"], True),
    ("prio", func_set(di.K_INF, "prio", 2), ["prio"], True),
    ("req_gt_lim", func_set(di.K_INF, "req_pm", 700, {"lim_pm": 600}), ["req_pm"], True),
    ("q23", func_set(di.K_INF, "req_pm", 20, {"lim_pm": 40, "work_per_batch": 10}), ["Q23"], True),
    ("quota_above_omega", lambda c, s, f, p: (scen_set(1, 800)(c, s, f, p),
                                              func_set(di.K_INF, "req_pm", 900, {"lim_pm": 900})(c, s, f, p))[1],
     ["Omega"], True),
    ("mem", func_set(di.K_INF, "mem_mib", 50000), ["mem_mib"], True),
    ("cold", func_set(di.K_INF, "cold_slots", -1), ["cold_slots"], True),
    ("lifecycle", func_set(di.K_INF, "depart_sec", 0), ["lifecycle"], True),
    ("n_workers", func_set(di.K_TRAIN, "n_workers", 65), ["n_workers"], True),
    ("duty", func_set(di.K_TRAIN, "duty_pm", 1001), ["duty_pm"], True),
    ("ibs", func_set(di.K_INF, "ibs", 0), ["ibs"], True),
    ("r4_cb", func_set(di.K_INF, "work_per_batch", 10**7), ["R4"], True),
    ("pattern", func_set(di.K_INF, "pattern", 64), ["pattern"], True),
    ("scale", func_set(di.K_INF, "scale_q10", -1), ["scale"], True),
]


def gpu_create(cfg, scen, funcs, pats, capfd):
    import paper_2503_05130_b200 as pkg
    h = C.c_void_p()
    rc = pkg.lib().dilu_sim_create(cfg.ctypes.data, scen.ctypes.data, funcs.ctypes.data,
                                   pats.ctypes.data, None, 0, None, C.byref(h))
    return rc, capfd.readouterr().err


def ref_create(cfg, scen, funcs, pats, capfd):
    L = oracle.lib()
    h = C.c_void_p()
    rc = L.dilu_ref_create(cfg, scen.ctypes.data, funcs, pats.ctypes.data, C.byref(h))
    msg = capfd.readouterr().err                    # dilu_ref_create reports on stderr
    if h.value:
        L.dilu_ref_destroy(h)
    return rc, msg


def test_base_inputs_pass_both_validations(capfd):
    cfg, scen, funcs, pats = base()
    rc, msg = ref_create(cfg, scen, funcs, pats, capfd)
    assert rc == 0, msg
    rc_g, err = gpu_create(cfg, scen, funcs, pats, capfd)
    assert rc_g == 1 and "workspace" in err        # validation passed; only the workspace is missing


@pytest.mark.parametrize("name,mut,tags,named", CASES, ids=[c[0] for c in CASES])
def test_reject_same_rule(name, mut, tags, named, capfd):
    cfg, scen, funcs, pats = base()
    f = mut(cfg, scen, funcs, pats)
    rc_r, msg_r = ref_create(cfg, scen, funcs, pats, capfd)
    rc_g, msg_g = gpu_create(cfg, scen, funcs, pats, capfd)
    assert rc_r == 1 and rc_g == 1, (rc_r, rc_g, msg_r, msg_g)
    for tag in tags:
        assert tag in msg_r and tag in msg_g, (tag, msg_r, msg_g)
    if named:
        want = f"scenario 0 func {f}"
        assert want in msg_r and want in msg_g, (msg_r, msg_g)
