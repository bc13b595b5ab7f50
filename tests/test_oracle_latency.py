"""Pins for the request-level latency model (P:1147 p50/p95 and SVR;
SPEC S:511-519; reading D10): hand-derived batch schedules, the closed form of
a backlogged server, the bucket geometry, and identities with the capacity tallies
(served requests = histogram mass, unserved = capacity-violated requests)."""
import numpy as np
import pytest

import dilu_inputs as di
import oracle

T = {n: i for i, n in enumerate(di.TALLY_NAMES)}


def test_bucket_geometry():
    """Four buckets per octave, monotone, exact at powers of two (D10)."""
    assert [oracle.lat_bucket(x) for x in (0, 1, 2, 3)] == [0, 1, 2, 3]
    for h in range(2, 19):
        assert oracle.lat_bucket(1 << h) == 4 * h - 4
        assert oracle.lat_bucket((1 << h) + (1 << (h - 2))) == 4 * h - 3
        assert oracle.lat_bucket((1 << (h + 1)) - 1) == 4 * h - 1
    prev = 0
    for x in range(0, 5000):
        b = oracle.lat_bucket(x)
        assert prev <= b <= prev + 1
        prev = b
    assert oracle.lat_bucket(10 ** 12) == 78


def test_two_batches_by_hand():
    """r = 8 over T = 1000 us (arrivals every 125 us), IBS 4, e = 100 us: batch 0 ready at
    375 done 475, latencies 475/350/225/100; batch 1 ready 875 done 975, the same four."""
    lat = oracle.instance_latency(8, 4, 2, 100, 1000, 1000)
    assert lat[81] == 2 * (475 + 350 + 225 + 100)
    assert lat[80] == 0 and lat[79] == 0
    want = np.zeros(82, np.int64)
    for L in (475, 350, 225, 100):
        want[oracle.lat_bucket(L)] += 2
    assert (lat[:79] == want[:79]).all()


def test_unserved_and_slo_violations_by_hand():
    """Only b = 1 batch executes: 4 served (475 > SLO 400 violates), 4 unserved (count as
    violations).  With e = 300 both batches run, the second waits for nothing
    (ready 875 > 675): 3 of 4 latencies per batch exceed 400."""
    lat = oracle.instance_latency(8, 4, 1, 100, 400, 1000)
    assert (lat[79], lat[80], lat[81]) == (4, 5, 1150)
    lat = oracle.instance_latency(8, 4, 2, 300, 400, 1000)
    assert (lat[79], lat[80], lat[81]) == (0, 6, 2 * (675 + 550 + 425 + 300))


def test_backlogged_server_closed_form():
    """Arrivals every 25 us, IBS 4 (a batch ready every 100 us at 100k + 75), e = 150 us >
    100: the queue grows, batch k completes at 75 + 150 (k + 1) and its members wait
    150 + 50 k + {75, 50, 25, 0} us."""
    r, ibs, e, Tus = 40, 4, 150, 1000
    lat = oracle.instance_latency(r, ibs, r // ibs, e, 10 ** 9, Tus)
    want = sum(4 * (150 + 50 * k) + 75 + 50 + 25 for k in range(10))
    assert lat[81] == want


def test_latency_observes_without_changing_tallies():
    """flags bit3 only observes: the 17 tallies are unchanged; the histogram holds every
    served request and bucket 79 every capacity-violated one."""
    wl = di.c2(seed=1, T=600)
    a = oracle.run(wl, flags=3)[1]
    s = oracle.RefSim(wl, flags=3 | 8)
    s.scale_step(600, threads=1)
    _, b = s.metrics()
    _, lat = s.latency()
    assert np.array_equal(a, b)
    assert lat[:79].sum() == b[T["req_served"]]
    assert lat[79] == b[T["req_violated"]]
    assert lat[80] >= lat[79]


def test_latency_under_alg2_and_modes():
    """Also defined under literal Alg.2 (a = executed tokens) and every baseline mode:
    the same identities hold."""
    wl = di.with_modes(di.replicate(di.c2(seed=2, T=300), 5), [0, 1, 2, 3, 4])
    for flags in (3 | 8, 3 | 4 | 8):
        s = oracle.RefSim(wl, flags=flags)
        s.scale_step(300, threads=5)
        per, tot = s.metrics()
        lper, lat = s.latency()
        assert (lper[:, :79].sum(1) == per[:, T["req_served"]]).all()
        assert (lper[:, 79] == per[:, T["req_violated"]]).all()


def test_host_percentile_bounds_match_buckets():
    """The host's bucket bounds (percentile reporting) contain every latency the oracle's
    bucket function maps there; percentiles of a known histogram."""
    from paper_2503_05130_b200 import lat_bucket_bounds, latency_summary
    for L in list(range(0, 3000)) + [10 ** k + d for k in range(3, 9) for d in (-1, 0, 1)]:
        lo, hi = lat_bucket_bounds(oracle.lat_bucket(L))
        assert lo <= L < hi or oracle.lat_bucket(L) == 78
    lat = np.zeros(82, np.int64)
    lat[oracle.lat_bucket(1000)] = 50          # 50 requests at ~1 ms
    lat[oracle.lat_bucket(20000)] = 45         # 45 at ~20 ms
    lat[79] = 5                                # 5 unserved
    lat[80] = 5
    lat[81] = 50 * 1000 + 45 * 20000
    s = latency_summary(lat)
    assert s["p50_ms"] == lat_bucket_bounds(oracle.lat_bucket(1000))[1] / 1000
    assert s["p95_ms"] == lat_bucket_bounds(oracle.lat_bucket(20000))[1] / 1000
    assert s["p99_ms"] is None and s["latency_svr"] == 0.05
