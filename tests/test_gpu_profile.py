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
