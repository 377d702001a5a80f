"""Pins of the oracle's leverage score sampling (SURVEY.md §8(c) P-10..P-13,
P-15c-e).  CPU only."""
import itertools
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import bitsplit, gemm, lss

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TWO32 = 1 << 32


def test_p10_waterfill_golden_cases():
    g = json.load(open(os.path.join(GOLD, "waterfill.json")))
    for case in g["cases"]:
        p = lss.probabilities(case["w"], case["budget"])
        assert p == [Fraction(x) for x in case["p"]], case["name"]
        if "clamped" in case:
            S, R, W, _ = lss.waterfill_a2(case["w"], case["budget"])
            assert (S, R, W) == (case["clamped"], case["R"], case["W"])
            for pi, d in zip(p, case["dyadic"]):
                assert list(lss.dyadic_thresholds(pi, 24)) == d
    f = g["floor_case"]
    assert list(lss.dyadic_thresholds(Fraction(f["p"]), f["e_max"])) == [f["e"], f["T1"], f["T2"]]


def test_p10_a2_loop_equals_closed_form_and_invariants():
    rng = np.random.default_rng(7)
    max_rounds = 0
    for trial in range(300):
        n = int(rng.integers(2, 80))
        budget = int(rng.integers(1, n))
        w = (rng.pareto(1.2, n) * 1000).astype(np.int64)
        w[rng.random(n) < 0.2] = 0
        S1, R1, W1, rounds = lss.waterfill_a2(w, budget)
        S2, R2, W2 = lss.waterfill_sorted(w, budget)
        assert (S1, R1, W1) == (S2, R2, W2)
        max_rounds = max(max_rounds, rounds)
        assert rounds <= n + 1                             # A.2 halts in O(N) rounds
        p = lss.probabilities(w, budget)
        assert all(0 <= x <= 1 for x in p)
        npos = int((w > 0).sum())
        if npos > budget:
            assert sum(p) == budget                        # sum p = N
        else:
            assert sum(p) == npos                          # Z-16
        # p proportional to w on the unclamped items (optimality)
        un = [i for i in range(n) if 0 < p[i] < 1]
        if len(un) >= 2:
            ratios = {p[i] / int(w[i]) for i in un}
            assert len(ratios) == 1
    assert max_rounds >= 2


def test_p11_dyadic_rule_exactly_unbiased():
    rng = np.random.default_rng(3)
    cases = [Fraction(1), Fraction(1, 2), Fraction(1, 3), Fraction(2, 3), Fraction(1, 20),
             Fraction(1, 16), Fraction(3, 17), Fraction(999, 1000), Fraction(1, 2 ** 30)]
    for _ in range(2000):
        W = int(rng.integers(1, 2 ** 58))
        Rw = int(rng.integers(1, W + 1))
        cases.append(Fraction(Rw, W))
    for p in cases:
        for e_max in (4, 24):
            e, T1, T2 = lss.dyadic_thresholds(p, e_max)
            assert 0 <= T1 <= T2 <= TWO32
            ew = Fraction(T1 * 2 ** e + (T2 - T1) * 2 ** (e + 1), TWO32)
            assert ew == 1                                 # E[weight * keep] = 1 exactly
            if p > Fraction(1, 2 ** e_max):
                assert 0 <= p - Fraction(T2, TWO32) < Fraction(1, TWO32)
                assert e < e_max
            else:
                assert T2 == TWO32 >> e_max and e == e_max


def _enumerate_expectation(w, budget, e_max, items_fn):
    """Exact expectation over the keep/weight outcomes of all items, obtained
    by feeding representative uniforms of each outcome interval to lss.sample."""
    n2 = w.size
    p = lss.probabilities(w.reshape(-1), budget)
    per_item = []
    for i in range(n2):
        e, T1, T2 = lss.dyadic_thresholds(p[i], e_max)
        outs = []
        for lo_u, hi_u in ((0, T1), (T1, T2), (T2, TWO32)):
            if hi_u > lo_u:
                outs.append((lo_u, Fraction(hi_u - lo_u, TWO32)))
        per_item.append(outs)
    mean = None
    second = None
    for combo in itertools.product(*per_item):
        u = np.array([c[0] for c in combo], dtype=np.uint64).reshape(w.shape)
        prob = Fraction(1)
        for c in combo:
            prob *= c[1]
        s = lss.sample(w, budget, u, lss.MODE_BERNOULLI, e_max)
        val = items_fn(s["items"], s["wexp"])
        contrib = np.array([[prob * int(v) for v in row] for row in val], dtype=object)
        sq = np.array([[prob * int(v) * int(v) for v in row] for row in val], dtype=object)
        mean = contrib if mean is None else mean + contrib
        second = sq if second is None else second + sq
    return mean, second, p


@pytest.mark.parametrize("e_max", [lss.E_MAX_W, lss.E_MAX_X])
def test_p12_p13_exhaustive_unbiased_and_variance(e_max):
    # PAPER.md:277-285 (unbiased), :289-294 (Prop. 1): brute force over all
    # 3^{2N} outcomes (drop / 2^e / 2^{e+1}) of a tiny instance, exact rationals.
    rng = np.random.default_rng(4)
    N, C, D = 3, 3, 2
    hi = rng.integers(-7, 8, (N, C)); lo = rng.integers(-8, 8, (N, C))
    hi[2] = 0
    xq = rng.integers(-7, 8, (N, D))
    bs = dict(hi=hi.astype(np.int8), lo=lo.astype(np.int8))
    a_sq = np.stack([(hi ** 2).sum(1), (lo ** 2).sum(1)])
    b_sq = (xq ** 2).sum(1)
    w = lss.weight_scores(a_sq, b_sq)
    budget = 2

    def acc_w(items, wexp):
        h = items // N; t = items % N
        codes = np.where((h == 0)[:, None], hi[t], lo[t])
        A = codes * (1 << wexp)[:, None]
        B = xq[t] * np.where(h == 0, 16, 1)[:, None]
        return gemm.int_matmul_abt(A.T, B.T) if len(items) else np.zeros((C, D), dtype=np.int64)

    mean, second, p = _enumerate_expectation(w, budget, e_max, acc_w)
    q = 16 * hi + lo
    exact = gemm.int_matmul_abt(q.T, xq.T)                  # the unsampled BS product (Eq. 6)
    assert np.array_equal(mean.astype(np.int64), exact) and all(
        m == int(e) for m, e in zip(mean.reshape(-1), exact.reshape(-1)))
    # variance = sum_i (E[w_i^2 keep_i] - 1) ||term_i||_F^2 (Prop. 1 with random weights)
    var = sum((second - mean * mean).reshape(-1))
    pred = Fraction(0)
    for i in range(2 * N):
        h, t = divmod(i, N)
        code = hi[t] if h == 0 else lo[t]
        term = (int((code ** 2).sum()) * int((xq[t] ** 2).sum()) * (256 if h == 0 else 1))
        e, T1, T2 = lss.dyadic_thresholds(p[i], e_max)
        ew2 = Fraction(T1 * 4 ** e + (T2 - T1) * 4 ** (e + 1), TWO32)
        if p[i] > 0:
            assert ew2 >= 1 / p[i] or e == e_max            # never below exact 1/p weights...
            assert ew2 <= Fraction(9, 8) / p[i] or e == e_max  # ...and at most +12.5 %
            pred += (ew2 - 1) * term
    assert var == pred


def test_p12_all_p_one_is_deterministic_exact():
    # Z <= N: every positive item kept with weight 1 -> exact BS product.
    w = np.array([[5, 0, 3], [0, 0, 1]], dtype=np.uint64)
    s = lss.sample(w, 3, np.zeros((2, 3), dtype=np.uint64), lss.MODE_BERNOULLI, 4)
    assert s["items"].tolist() == [0, 2, 5] and s["wexp"].tolist() == [0, 0, 0]


def test_p10_budget_monte_carlo():
    # E[#kept] = N when the budget binds; floor adds at most 1/16 per item.
    rng = np.random.default_rng(9)
    N = 64
    w = (rng.pareto(1.0, (2, N)) * 1e6).astype(np.uint64) + 1
    p = lss.probabilities(w.reshape(-1), N)
    assert sum(p) == N
    counts = []
    for seed in range(400):
        u = rng.integers(0, TWO32, (2, N), dtype=np.uint64)
        counts.append(lss.sample(w, N, u, lss.MODE_BERNOULLI, 24)["count"])
    assert abs(np.mean(counts) - N) < 4 * np.std(counts) / np.sqrt(len(counts)) + 0.5


def test_scores_integer_exact():
    a = np.array([[49 * 4096, 0, 1], [0, 25, 2]])
    b = np.array([49 * 1024, 7, 0])
    w = lss.weight_scores(a, b)
    # hi row: floor(sqrt(a b) 2^20); lo row: floor(sqrt(a b) 2^16)
    assert int(w[0, 0]) == int(np.floor(np.sqrt(49 * 4096 * 49 * 1024) * 2 ** 20))
    assert int(w[0, 0]) == 49 * 2048 * 2 ** 20
    assert w[0, 1] == 0 and w[0, 2] == 0 and w[1, 2] == 0
    assert int(w[1, 1]) == int(np.floor(np.sqrt(175.0) * 2 ** 16))
    wx = lss.activation_scores(a)
    assert int(wx[1, 1]) == 5 * 2 ** 16 and int(wx[0, 2]) == 2 ** 20
