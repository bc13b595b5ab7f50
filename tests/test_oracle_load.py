"""Oracle pins of the a0 profile-table loader (oracle/dilu_ref_load.c; SURVEY s8(a) a0,
PAPER.md:606-610, 628, 634-637; readings Q25 and R4): values fixed by the SURVEY's model
catalogue (s8(d)) and by the rounding rule itself, not by re-running the oracle."""
import numpy as np

import dilu_inputs as di
import oracle


def _row(kind=0, mem_gb=2.0, cold_ms=2000.0, slo_ms=100.0, **kw):
    c = np.zeros(1, di.CATALOG_ROW)
    c["kind"], c["mem_gb"], c["cold_ms"], c["slo_ms"] = kind, mem_gb, cold_ms, slo_ms
    c["n_workers"], c["duty_pm"], c["depart_sec"] = 1, 1000, di.NEVER
    for k, v in kw.items():
        c[k] = v
    return c


def _prof(req_pm, lim_pm, ibs, status=0):
    p = np.zeros(1, di.PROF_OUT)
    p["req_pm"], p["lim_pm"], p["ibs"], p["status"] = req_pm, lim_pm, ibs, status
    return p


F = di.FI


def test_r4_work_per_batch_matches_survey_catalogue():
    # SURVEY s8(d) catalogue: c_b = req * SLO / 2 (P:634 footnote)
    for req, slo, cb in [(150, 100, 7500), (100, 50, 2500), (300, 200, 30000), (400, 100, 20000),
                         (350, 100, 17500), (300, 100, 15000)]:
        rows, st = oracle.load_profiles(_row(slo_ms=slo), _prof(req, 2 * req, 8), 1000)
        assert st[0] == 0 and rows[0, F["work_per_batch"]] == cb
        assert rows[0, F["req_pm"]] == req and rows[0, F["lim_pm"]] == 2 * req   # limit = 2 x request
    rows, _ = oracle.load_profiles(_row(slo_ms=125.0), _prof(7, 14, 1), 1000)
    assert rows[0, F["work_per_batch"]] == 437                                  # floor(437.5)


def test_q25_memory_and_cold_start():
    cases = [(2.0, 2048), (1.5, 1536), (0.2, 205), (14.0, 14336), (12.6, 12903), (40.0, 40960)]
    for gb, mib in cases:
        rows, _ = oracle.load_profiles(_row(mem_gb=gb), _prof(150, 300, 8), 1000)
        assert rows[0, F["mem_mib"]] == mib, (gb, rows[0, F["mem_mib"]])
    for cold, slot, slots in [(2000.0, 1000, 2), (2500.0, 1000, 3), (2000.0, 100, 20), (250.0, 100, 3),
                              (10000.0, 100, 100), (0.0, 1000, 0), (1.0, 1000, 1)]:
        rows, _ = oracle.load_profiles(_row(cold_ms=cold), _prof(150, 300, 8), slot)
        assert rows[0, F["cold_slots"]] == slots, (cold, slot)


def test_training_rows_and_copied_fields():
    c = _row(kind=2, mem_gb=10.0, cold_ms=5000.0, n_workers=4, duty_pm=750, affinity_class=77,
             arrive_sec=12, depart_sec=900, pattern=-1)
    rows, st = oracle.load_profiles(c, _prof(400, 500, 0), 1000)
    r = rows[0]
    assert st[0] == 0
    assert (r[F["kind"]], r[F["ibs"]], r[F["work_per_batch"]], r[F["n_workers"]], r[F["duty_pm"]]) == (2, 0, 0, 4, 750)
    assert (r[F["req_pm"]], r[F["lim_pm"]], r[F["mem_mib"]], r[F["cold_slots"]]) == (400, 500, 10240, 5)
    assert (r[F["affinity_class"]], r[F["arrive_sec"]], r[F["depart_sec"]]) == (77, 12, 900)


def test_failed_profiles_and_invalid_rows_are_unused():
    rows, st = oracle.load_profiles(_row(), _prof(0, 0, 0, status=1), 1000)      # SLO unattainable
    assert st[0] == 1 and rows[0, F["kind"]] == -1
    rows, st = oracle.load_profiles(_row(kind=2), _prof(300, 400, 4), 1000)      # inference session
    assert st[0] == 2 and rows[0, F["kind"]] == -1
    rows, st = oracle.load_profiles(_row(mem_gb=-1.0), _prof(150, 300, 8), 1000)
    assert st[0] == 2
    rows, st = oracle.load_profiles(_row(kind=5), _prof(150, 300, 8), 1000)
    assert st[0] == 2
    rows, st = oracle.load_profiles(_row(slo_ms=float("nan")), _prof(150, 300, 8), 1000)
    assert st[0] == 2


def test_profile_load_simulate_pipeline_validates():
    """profile -> load -> simulate on the oracle: every loaded row passes dilu_ref_create's
    validation (R1, R4, Q12, Q23) and the loop runs."""
    ses, cat, pats = di.profiled_fleet(seed=3, T=300)
    prof = oracle.profile_batch(ses)
    rows, st = oracle.load_profiles(cat, prof, 1000)
    assert (st == 0).all()
    wl = di.workload_from_rows("loaded", rows, pats, 300)
    rs = oracle.RefSim(wl)
    rs.scale_step(300)
    _, tot = rs.metrics()
    T = {n: i for i, n in enumerate(di.TALLY_NAMES)}
    assert tot[T["placements_ok"]] > 0 and tot[T["req_total"]] > 0
