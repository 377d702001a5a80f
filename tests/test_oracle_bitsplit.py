"""Pins of the oracle's bit splitting.  CPU only."""
import json
import os

import numpy as np

from oracle import bitsplit

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_p7_exhaustive_split_reconstruction():
    # BS is an INT8 representation whose high/low 4 bits are the halves.
    q = np.arange(-119, 120)
    hi, lo = bitsplit.split(q)
    assert np.array_equal(16 * hi.astype(np.int64) + lo, q)
    assert hi.min() == -7 and hi.max() == 7
    assert lo.min() == -8 and lo.max() == 7
    # uniqueness: the map q -> (hi, lo) is injective on [-119, 119]
    assert len(set(zip(hi.tolist(), lo.tolist()))) == q.size


def test_p15b_golden():
    g = json.load(open(os.path.join(GOLD, "bitsplit.json")))
    amax, s_down, r8 = bitsplit.scales(np.array([g["amax"], -1.0], dtype=np.float32))
    assert amax == np.float32(g["amax"]) and r8 == np.float32(g["r8"]) and s_down == np.float32(g["s_down"])
    for gv, q, hi, lo in g["deterministic"]:
        v = np.float32(gv) * r8
        qq = bitsplit.stochastic_round(np.array([v]), np.array([0]))[0]
        assert qq == q
        h, l = bitsplit.split(np.array([qq]))
        assert (int(h[0]), int(l[0])) == (hi, lo)
    for gv, v_expect, A, u_thr, q_below, q_at in g["stochastic"]:
        v = np.float32(gv) * r8
        assert v == np.float32(v_expect)
        assert np.ceil(np.float64(v) * 2.0 ** 32) == A
        # u just below the threshold keeps floor(v), u = threshold rounds up
        assert bitsplit.stochastic_round(np.array([v]), np.array([u_thr - 1]))[0] == q_below
        assert bitsplit.stochastic_round(np.array([v]), np.array([u_thr]))[0] == q_at
    for q, hi, lo in g["split_ties"]:
        h, l = bitsplit.split(np.array([q]))
        assert (int(h[0]), int(l[0])) == (hi, lo)


def test_sr_threshold_is_exact_fraction():
    # Z-10 floor form: P(q = floor(v) + 1) = ceil(frac(v) 2^32) / 2^32, i.e. the
    # fraction exactly when it has <= 32 bits; a tiny negative v (frac(v) within
    # 2^-32 of 1) rounds to 0 for every u, a tiny positive one up only for the
    # largest u.
    v = np.array([-1e-10, 1e-10, -118.75, 0.0, 119.0, -119.0], dtype=np.float32)
    q0 = bitsplit.stochastic_round(v, np.zeros(6, dtype=np.uint64))
    assert q0.tolist() == [0, 0, -119, 0, 119, -119]
    q1 = bitsplit.stochastic_round(v, np.full(6, 2 ** 32 - 1, dtype=np.uint64))
    assert q1.tolist() == [0, 1, -118, 0, 119, -119]
    # the count of u in [0, 2^32) rounding up is T = ceil(frac(v) 2^32), from the
    # threshold u >= 2^32 - T: check both sides of it for a spread of fractions
    rng = np.random.default_rng(3)
    vs = (rng.integers(-119 * 2 ** 16, 119 * 2 ** 16, 200) / 2.0 ** 16).astype(np.float32)
    for x in vs:
        fl = int(np.floor(np.float64(x)))
        T = int(np.ceil((np.float64(x) - fl) * 2.0 ** 32))
        if T == 0:
            assert bitsplit.stochastic_round(np.array([x]), np.array([2 ** 32 - 1]))[0] == fl
            continue
        thr = 2 ** 32 - T
        assert bitsplit.stochastic_round(np.array([x]), np.array([thr - 1]))[0] == fl
        assert bitsplit.stochastic_round(np.array([x]), np.array([thr]))[0] == fl + 1


def test_p8_sr_unbiased_over_seeds():
    # E[s_down q] = g elementwise (unbiased SR, north star); |s_down q - g| < s_down.
    rng = np.random.default_rng(11)
    g = (rng.standard_normal((4, 16)) * np.array([[1.0], [0.3], [1e-3], [0]])).astype(np.float32)
    g[0, 0] = 2.5                                     # amax element
    trials = 10000
    acc = np.zeros_like(g, dtype=np.float64)
    acc2 = np.zeros_like(g, dtype=np.float64)
    s_down = None
    for seed in range(trials):
        out = bitsplit.bit_split(g, seed, 0)
        s_down = np.float64(out["s_down"])
        val = s_down * out["q"]
        assert np.all(np.abs(val - g) < s_down)
        acc += val
        acc2 += val * val
    mean = acc / trials
    se = np.sqrt(np.maximum(acc2 / trials - mean ** 2, 0) / trials) + 1e-300
    # elements with SR noise: bias within 4 standard errors; exact ones exact
    z = np.abs(mean - g) / se
    noisy = se > 1e-12
    assert np.all(z[noisy] < 4.5)
    # deterministic elements (integer v) are off only by the fp32 scale rounding
    assert np.allclose(mean[~noisy], g[~noisy], rtol=1e-6, atol=0)


def test_zero_gradient_degenerate():
    out = bitsplit.bit_split(np.zeros((3, 8), dtype=np.float32), 1, 2)
    assert out["s_down"] == 0 and not out["q"].any() and not out["a_sq"].any()
