"""Pins of the oracle's unit steps against the paper's definitions, closed forms,
textbook reductions and brute force -- never against the oracle's own formula.

* SelectOptGPU: the paper's real-valued score evaluated with
  exact rationals, argmin with strict '<' over ascending ids, vs the oracle.
* Vertical allocator: brute force over every integer spare vector: the oracle's
  allocation must be the lexicographic maximum in (prio, id) order of
  0 <= s_i <= want_i, sum s <= S_g (SURVEY s8(c) pins, vertical (ii)); plus the
  closed form sum a = sum req + min(S_g, sum want) and Alg.2 special cases.
* hscaler: SPEC S:448-460 examples; lazy-out property.
* LLM split: SPEC S:287-288 examples; brute force over <=6 GPUs.
* splitmix64: the published first output of splitmix64 seeded with 0.
"""
import itertools
from fractions import Fraction

import numpy as np
import pytest

import oracle

L = oracle.lib()


def i32(x):
    return np.ascontiguousarray(x, dtype=np.int32)


def i64(x):
    return np.ascontiguousarray(x, dtype=np.int64)


# ------------------------------------------------------------------ mix (R8)

def test_splitmix64_test_vector():
    # splitmix64 seeded with 0 first returns 0xE220A8397B1DCDAF (Steele et al. / Vigna's
    # reference generator); sm64(0) is exactly that first output.  mix(0,...) begins
    # with sm64(0), so check the chain's first link through a degenerate input:
    # mix(scn, t, i, g, a) = sm64(sm64(sm64(sm64(scn)^t)^i)^((g<<32)|a)).
    def sm64(z):
        M = (1 << 64) - 1
        z = (z + 0x9E3779B97F4A7C15) & M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)
    assert sm64(0) == 0xE220A8397B1DCDAF
    rng = np.random.default_rng(1)
    for _ in range(200):
        scn, t, i, g, a = (int(x) for x in rng.integers(0, 2**31 - 1, 5))
        want = sm64(sm64(sm64(sm64(scn) ^ t) ^ i) ^ ((g << 32) | a))
        assert L.dilu_ref_mix(scn, t, i, g, a) == want


# ------------------------------------------------------- SelectOptGPU (Alg.1)

def paper_select(cand, R, Lm, U, nres, req, lim, mem, om, ga, M, Q, alpha, beta):
    """Alg.1 SelectOptGPU verbatim with exact rationals."""
    best, bi = None, -1
    for i in cand:
        nr, nl, nm = R[i] + req, Lm[i] + lim, U[i] + mem
        score = alpha * (1 - Fraction(nr, Q)) + beta * (1 - Fraction(nm, M))
        if nr <= om and nl <= ga and nm <= M and nres[i] < 32 and (best is None or score < best):
            best, bi = score, i
    return bi


def test_select_matches_exact_rational_score():
    rng = np.random.default_rng(7)
    M, Q = 40960, 1000
    n_ok = 0
    for trial in range(20000):
        G = int(rng.integers(1, 9))
        R = rng.integers(0, 1001, G); Lm = R + rng.integers(0, 600, G)
        U = rng.integers(0, M + 1, G); nres = rng.integers(0, 33, G)
        # coarse grids create many exact ties
        if trial % 2:
            R = (R // 100) * 100; U = (U // 4096) * 4096
        req = int(rng.integers(1, 600)); lim = req + int(rng.integers(0, 600))
        mem = int(rng.integers(1, 20000))
        a, b = (int(x) for x in rng.integers(0, 4, 2))
        if a + b == 0:
            a = 1
        cand = sorted(rng.choice(G, size=int(rng.integers(0, G + 1)), replace=False).tolist())
        want = paper_select(cand, R, Lm, U, nres, req, lim, mem, 1000, 1500, M, Q,
                            Fraction(a, a + b), Fraction(b, a + b))
        got = L.dilu_ref_select_opt_gpu(len(cand), i32(cand), i32(R), i32(Lm), i32(U), i32(nres),
                                        req, lim, mem, 1000, 1500, M, Q, a, b)
        assert got == want, (trial, cand)
        n_ok += want >= 0
    assert n_ok > 5000


def test_select_spec_examples():
    M, Q = 40960, 1000
    # req_sum 0.6 under Omega=1 rejects a 0.5 request
    assert L.dilu_ref_select_opt_gpu(1, i32([0]), i32([600]), i32([600]), i32([0]), i32([1]),
                                     500, 500, 1, 1000, 1500, M, Q, 1, 1) == -1
    # fuller in both dimensions wins
    assert L.dilu_ref_select_opt_gpu(2, i32([0, 1]), i32([100, 400]), i32([100, 400]),
                                     i32([1000, 9000]), i32([1, 1]), 100, 100, 100, 1000, 1500,
                                     M, Q, 1, 1) == 1
    # memory-only violation excludes regardless of score
    assert L.dilu_ref_select_opt_gpu(2, i32([0, 1]), i32([100, 900]), i32([100, 900]),
                                     i32([1000, 40000]), i32([1, 1]), 50, 50, 2000, 1000, 1500,
                                     M, Q, 1, 1) == 0


def test_select_alpha1_beta0_is_1d_best_fit():
    """alpha=1, beta=0 reduces to textbook 1-D best fit (tightest remaining
    capacity, first on ties) -- written here independently."""
    rng = np.random.default_rng(3)
    M, Q = 40960, 1000
    for _ in range(5000):
        G = int(rng.integers(1, 10))
        R = rng.integers(0, 1001, G); Lm = R.copy(); U = np.zeros(G, int); n = np.zeros(G, int)
        req = int(rng.integers(1, 500))
        best, bi = None, -1
        for g in range(G):
            rem = 1000 - (R[g] + req)
            if rem >= 0 and (best is None or rem < best):
                best, bi = rem, g
        got = L.dilu_ref_select_opt_gpu(G, i32(range(G)), i32(R), i32(Lm), i32(U), i32(n), req,
                                        req, 1, 1000, 10**6, M, Q, 1, 0)
        assert got == bi


# ------------------------------------------------------- vertical allocator

def vertical(prio, ids, rq, lm, d, T):
    n = len(prio)
    a = np.zeros(n, np.int64)
    L.dilu_ref_vertical_row(n, i32(prio), i32(ids), i64(rq), i64(lm), i64(d), T, a)
    return a


def lexmax_bruteforce(prio, ids, rq, lm, d, T):
    """Enumerate every integer spare vector s with 0 <= s_i <= want_i and sum s <= S_g;
    return the lexicographically largest in (prio, id) order."""
    n = len(prio)
    want = [max(0, min(d[i], lm[i]) - rq[i]) for i in range(n)]
    S = T - sum(rq)
    order = sorted(range(n), key=lambda i: (prio[i], ids[i]))
    best = None
    for s in itertools.product(*[range(want[i] + 1) for i in range(n)]):
        if sum(s) > S:
            continue
        key = tuple(s[i] for i in order)
        if best is None or key > best[0]:
            best = (key, s)
    return [rq[i] + best[1][i] for i in range(n)]


def test_vertical_is_lexicographic_max():
    rng = np.random.default_rng(11)
    for _ in range(600):
        n = int(rng.integers(1, 5))
        rq = rng.integers(0, 5, n); lm = rq + rng.integers(0, 5, n)
        d = rng.integers(0, 10, n); prio = rng.integers(0, 2, n)
        ids = rng.permutation(20)[:n]
        T = int(rq.sum() + rng.integers(0, 12))
        got = vertical(prio, ids, rq, lm, d, T)
        assert got.tolist() == lexmax_bruteforce(prio, ids, rq, lm, d, T)


def test_vertical_closed_form_and_bounds():
    rng = np.random.default_rng(12)
    for _ in range(3000):
        n = int(rng.integers(1, 33))
        rq = rng.integers(30_000, 200_000, n); lm = rq + rng.integers(0, 400_000, n)
        while rq.sum() > 1_000_000:
            rq = rq // 2; lm = lm // 2 + rq
        d = rng.integers(0, 900_000, n); prio = rng.integers(0, 2, n); ids = rng.permutation(1000)[:n]
        a = vertical(prio, ids, rq, lm, d, 1_000_000)
        want = np.maximum(0, np.minimum(d, lm) - rq)
        S = 1_000_000 - rq.sum()
        assert a.sum() == rq.sum() + min(S, want.sum())          # closed form
        assert np.all(a >= rq) and np.all(a <= lm)               # I4: floor and ceiling
        assert a.sum() <= 1_000_000                              # I5


def test_vertical_alg2_special_cases():
    # Alg.2 NONE: a lone instance gets min(d, limit), floored at request
    assert vertical([1], [0], [300], [500], [450], 1000).tolist() == [450]
    assert vertical([1], [0], [300], [500], [900], 1000).tolist() == [500]
    assert vertical([1], [0], [300], [500], [100], 1000).tolist() == [300]
    # Alg.2 RECOVERY scale-down: idle SLO instance keeps request only;
    # its neighbour takes the whole spare up to its limit (PAPER.md:1003-1004 reading)
    assert vertical([0, 1], [0, 1], [200, 300], [400, 700], [0, 700], 1000).tolist() == [200, 700]
    # EMERGENCY reading: an SLO instance with demand above request is served first
    assert vertical([1, 0], [0, 1], [300, 200], [700, 600], [700, 600], 1000).tolist() == [400, 600]


# ----------------------------------------------------------------- hscaler

def decide(window, n, cap1, min_inst=1):
    k = np.zeros(1, np.int32)
    import ctypes
    kk = ctypes.c_int32(0)
    d = L.dilu_ref_scaling_decision(len(window), i32(window), n, cap1, 20, 30, min_inst,
                                    ctypes.byref(kk))
    return d, kk.value


def test_capacity_of_examples():
    # ibs=4, t_exec=25 ms -> 160 RPS (1 s slot: req 200 per-mille, c_b = 5,000 tokens)
    assert L.dilu_ref_cap1(1000, 200, 5000, 4) == 160
    # C1 F0: 80 RPS (Appendix A); same function at 100 ms slots has the same capacity
    assert L.dilu_ref_cap1(1000, 200, 10000, 4) == 80
    assert L.dilu_ref_cap1(100, 200, 10000, 4) == 80


def test_scaling_decision_spec_examples():
    # 20 of 40 samples above capacity -> ScaleOut
    w = [100] * 20 + [10] * 20
    d, k = decide(w, 1, 80)
    assert d == 1 and k == 1
    # all-zero window at n = min = 1 -> Hold
    assert decide([0] * 40, 1, 80)[0] == 0
    # 31 of 40 below capacity(n-1), n=3 -> ScaleIn(1)
    w = [10] * 31 + [500] * 9
    assert decide(w, 3, 80)[0] == 2
    # exactly phi_in (30) below is not "more than" -> Hold
    w = [10] * 30 + [170] * 10
    assert decide(w, 3, 80)[0] == 0
    # 19 above is not "at least 20" -> Hold (lazy-out)
    w = [1000] * 19 + [10] * 21
    assert decide(w, 1, 80)[0] == 0
    # k sized to the window max: ceil(1000/80) - 2 = 11
    w = [1000] * 25 + [10] * 15
    assert decide(w, 2, 80) == (1, 11)


def test_scaling_decision_mutually_exclusive():
    rng = np.random.default_rng(5)
    for _ in range(20000):
        w = rng.integers(0, 400, 40)
        n = int(rng.integers(1, 6))
        d, k = decide(w, n, 80)
        up = int((w > n * 80).sum()); down = int((w < (n - 1) * 80).sum())
        assert not (up >= 20 and down > 30)
        if d == 1:
            assert up >= 20 and k == -(-int(w.max()) // 80) - n and k >= 1
        elif d == 2:
            assert down > 30 and n > 1


# --------------------------------------------------------------- LLM split

def split(free, active=None, req=100, lim=100, mem=0, R=None, Lm=None, n=None, stages=4):
    G = len(free)
    M = 40960
    U = [M - f for f in free]
    active = [1] * G if active is None else active
    R = [0] * G if R is None else R
    Lm = [0] * G if Lm is None else Lm
    n = [1] * G if n is None else n
    og = np.zeros(4, np.int32); osh = np.zeros(4, np.int32)
    k = L.dilu_ref_llm_split(G, i32(active), i32(R), i32(Lm), i32(U), i32(n), i32([0] * G), req,
                             lim, mem, 1000, 1500, M, stages, og, osh)
    return k, og[:k].tolist(), osh[:k].tolist()


def test_llm_split_spec_examples():
    GB = 1024
    # 12.6 GB over free {30, 8, 6} GB -> single GPU (the 30 GB one)
    k, g, sh = split([30 * GB, 8 * GB, 6 * GB], mem=int(12.6 * GB))
    assert k == 1 and g == [0]
    # 50 GB over {30, 20, 10} -> two GPUs {30, 20}
    k, g, sh = split([10 * GB, 30 * GB, 20 * GB], mem=50 * GB)
    assert k == 2 and g == [1, 2] and sh == [30 * GB, 20 * GB]
    # more than 4 stages needed -> no split
    assert split([5 * GB] * 8, mem=21 * GB)[0] == 0


def test_llm_split_bruteforce():
    """Fewest stages; among those, the largest free memories (worst-fit)."""
    rng = np.random.default_rng(9)
    for _ in range(2000):
        G = int(rng.integers(1, 7))
        free = rng.integers(0, 9, G) * 1024
        mem = int(rng.integers(1, 30)) * 512
        act = rng.integers(0, 2, G).tolist()
        k, g, sh = split(free.tolist(), active=act, mem=mem)
        cands = [i for i in range(G) if act[i] and free[i] > 0]
        best = None
        for m in range(1, 5):
            for sub in itertools.combinations(cands, m):
                if sum(free[list(sub)]) >= mem:
                    key = sorted((-int(free[i]), i) for i in sub)
                    if best is None or key < best:
                        best = key
            if best is not None:
                break
        if best is None:
            assert k == 0
        else:
            assert k == len(best) and g == [i for _, i in best]
            assert sum(sh) == mem and all(s > 0 for s in sh)
