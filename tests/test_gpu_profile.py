"""GPU parity of the batched profiler (dilu_profile) against the oracle:
every output byte (fp64 quotas and t_exec, IBS, trials, per-mille quotas, status)
identical -- both sides run the same IEEE operations without contraction (D9)."""
import numpy as np
import pytest

import dilu_inputs as di
import oracle

pytestmark = pytest.mark.gpu


def gpu_profile(ses):
    import torch
    from paper_2503_05130_b200 import dilu_profile
    d = torch.from_numpy(np.ascontiguousarray(ses).view(np.uint8)).cuda()
    out = dilu_profile(d)
    torch.cuda.synchronize()
    return out.cpu().numpy().view(di.PROF_OUT)


def check(ses):
    g = gpu_profile(ses)
    r = oracle.profile_batch(ses)
    for name in di.PROF_OUT.names:
        if not np.array_equal(g[name], r[name]):
            k = int(np.nonzero(g[name] != r[name])[0][0])
            raise AssertionError(f"{name} differs at session {k}: gpu {g[k]} ref {r[k]} in {ses[k]}")
    assert g.tobytes() == r.tobytes()
    return g


def test_profile_builtins_and_edges():
    rows = [di.prof_inference(*m[1:]) for m in di.PROFILE_MODELS_V1]
    rows += [di.prof_training(100.0, 100.0, 0.0), di.prof_training(60.0, 100.0, 0.0),
             di.prof_training(100.0, 100.0, 1.5), di.prof_inference(5.0, 5.0, 50.0, 9.0),
             di.prof_inference(5.0, 5.0, 50.0, 100.0, ibs_max=1)]
    ses = np.zeros(len(rows), di.PROF_SESSION)
    for k, x in enumerate(rows):
        ses[k] = x
    g = check(ses)
    assert g["trials"][:4].tolist() == [8, 6, 6, 9]          # Table 2
    assert g["status"].tolist()[4:8] == [0, 0, 2, 1]


@pytest.mark.parametrize("n,seed", [(1, 0), (257, 1), (200_003, 2)])
def test_profile_random_sessions(n, seed):
    check(di.profile_sessions(n, seed=seed))


def test_profile_c4_sweep_size():
    """The C4 sweep's 4,096 x 200 function rows, every session compared."""
    check(di.profile_sessions(4096 * 200, seed=7))


def test_profile_load_simulate_pipeline():
    """SURVEY s8(a) a0 end to end on the GPU: profiling sessions -> dilu_profile ->
    dilu_load_profiles -> dilu_sim_create -> slots, every stage bit-exact against the
    oracle's profile -> load -> simulate on the same inputs."""
    import torch
    from paper_2503_05130_b200 import dilu_profile, dilu_load_profiles, DiluSim
    ses, cat, pats = di.profiled_fleet(seed=5, T=900)
    d_ses = torch.from_numpy(np.ascontiguousarray(ses).view(np.uint8)).cuda()
    d_cat = torch.from_numpy(np.ascontiguousarray(cat).view(np.uint8)).cuda()
    d_prof = dilu_profile(d_ses)
    rows, st = dilu_load_profiles(d_cat, d_prof, 1000)
    torch.cuda.synchronize()
    r_prof = oracle.profile_batch(ses)
    r_rows, r_st = oracle.load_profiles(cat, r_prof, 1000)
    assert d_prof.cpu().numpy().tobytes() == r_prof.tobytes()
    assert np.array_equal(st.cpu().numpy(), r_st) and (r_st == 0).all()
    assert np.array_equal(rows.cpu().numpy(), r_rows)
    wl = di.workload_from_rows("loaded", rows.cpu().numpy(), pats, 900)
    gs, rs = DiluSim.from_workload(wl), oracle.RefSim(wl)
    gs.scale_step(900)
    rs.scale_step(900)
    assert np.array_equal(gs.metrics()[1].cpu().numpy(), rs.metrics()[1])


def test_load_profiles_status_paths():
    import torch
    from paper_2503_05130_b200 import dilu_load_profiles
    cat = np.zeros(4, di.CATALOG_ROW)
    cat["kind"] = [0, 2, 0, 7]
    cat["mem_gb"] = [2.0, 10.0, -1.0, 1.0]
    cat["cold_ms"], cat["slo_ms"], cat["n_workers"] = 2000.0, 100.0, 1
    pr = np.zeros(4, di.PROF_OUT)
    pr["status"] = [1, 0, 0, 0]
    pr["ibs"] = [0, 4, 8, 8]                     # row 1: an inference result on a training row
    pr["req_pm"], pr["lim_pm"] = 300, 600
    rows, st = dilu_load_profiles(torch.from_numpy(cat.view(np.uint8)).cuda(),
                                  torch.from_numpy(pr.view(np.uint8)).cuda(), 1000)
    r_rows, r_st = oracle.load_profiles(cat, pr, 1000)
    assert st.cpu().tolist() == r_st.tolist() == [1, 2, 2, 2]
    assert np.array_equal(rows.cpu().numpy(), r_rows)
