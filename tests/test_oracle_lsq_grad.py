"""Pins of the A.3 / A.4 oracle pieces (LSQ step-size gradients, cold start).
CPU only.  None of these compares the oracle with itself: worked values from
the definitions (golden), the derivative of the STE surrogate by central
differences, brute-force loops over the bit-split planes (Eq. 5) and the
unbiasedness of the sampled estimate (Monte Carlo over Philox seeds)."""
import json
import os

import numpy as np

from oracle import hadamard, hq, linear, lsq_grad, lss

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "lsq_grad.json")))


def test_delta_worked_values():
    v = np.array(GOLD["v"], dtype=np.float32)
    got = lsq_grad.delta(v)
    assert np.allclose(got, np.array(GOLD["delta"]), rtol=0, atol=1e-6)
    # in range: |delta| <= 1/2; clamped: delta is the clamp code itself
    vv = np.linspace(-12, 12, 4801).astype(np.float32)
    d = lsq_grad.delta(vv)
    inside = np.abs(vv) <= 7
    assert np.all(np.abs(d[inside]) <= 0.5)
    assert np.array_equal(d[~inside], np.sign(vv[~inside]) * 7.0)


def test_grad_scale_and_cold_start_closed_forms():
    for n, g in zip(GOLD["g_n"], GOLD["g"]):
        assert abs(lsq_grad.grad_scale(n) - g) < 1e-15
    step = lsq_grad.cold_start_step(np.array(GOLD["cold_x"]))
    assert step == np.float32(GOLD["cold_step"])
    c = np.full((5, 7), -0.75)
    assert lsq_grad.cold_start_step(c) == np.float32(1.5 / np.sqrt(7.0))


def test_delta_is_the_derivative_of_the_ste_surrogate():
    # LSQ: q(s) = s <X/s>; with round' = 1 (STE), the surrogate
    # q~(s) = s (clamp(X/s) + c0), c0 = round(clamp(v0)) - clamp(v0) frozen at s0,
    # has d/ds sum(G o q~) = sum(G o delta(v0)) -- central differences, float64.
    rng = np.random.default_rng(3)
    D, k = 16, 2
    x = rng.standard_normal((6, D)) * 2.0
    x[:, 3] *= 6.0                                    # some clamped elements
    Hn = hadamard.block_diag_hadamard(D, k)           # normalised H
    t = x @ Hn
    s0 = 0.4
    v0 = t / s0
    assert np.any(np.abs(v0) > 7) and np.all(np.abs(np.abs(v0) - 7) > 1e-3)
    c0 = np.rint(np.clip(v0, -7, 7)) - np.clip(v0, -7, 7)
    G = rng.standard_normal(t.shape)

    def L(s):
        return float(np.sum(G * s * (np.clip(t / s, -7, 7) + c0)))

    h = 1e-6
    fd = (L(s0 + h) - L(s0 - h)) / (2 * h)
    assert abs(fd - float(np.sum(G * lsq_grad.delta(v0)))) < 1e-6 * max(1.0, abs(fd))


def _setup(N=8, C=8, D=16, k=2, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((N, D)).astype(np.float32)
    x[:, 1] *= 8.0
    w = (rng.standard_normal((C, D)) * 0.5).astype(np.float32)
    fwd = linear.forward(x, w, k, 0.35, 0.2)
    g = (rng.standard_normal((N, C)) * 0.1).astype(np.float32)
    return x, w, g, fwd


def test_step_grads_brute_force_exact_product():
    # mode NONE: the products are the exact bit-split ones, grad_Y^ = s_up hi + s_down lo
    # (Eq. 5).  Loops straight from A.3 and Eq. 5.
    x, w, g, fwd = _setup()
    N, D = x.shape
    C = w.shape[0]
    out = linear.backward(g, fwd, seed=11, call_id=2, mode=lss.MODE_NONE)
    gs_x, gs_w = linear.step_size_grads(x, w, fwd, out)
    b = out["bs"]
    sd = float(b["s_down"])
    gy = 16.0 * sd * b["hi"].astype(np.float64) + sd * b["lo"].astype(np.float64)
    vx = hq.transformed_scaled(x, fwd["k"], fwd["s_x"]).astype(np.float64)
    vw = hq.transformed_scaled(w, fwd["k"], fwd["s_w"]).astype(np.float64)
    sx, sw = float(fwd["s_x"]), float(fwd["s_w"])
    ref_x = 0.0
    for t in range(N):
        for d in range(D):
            prod = sum(gy[t, c] * sw * float(fwd["wq"][c, d]) for c in range(C))
            code = min(7.0, max(-7.0, float(np.rint(vx[t, d]))))
            dlt = code - (vx[t, d] if abs(vx[t, d]) <= 7 else 0.0)
            ref_x += prod * dlt
    ref_w = 0.0
    for c in range(C):
        for d in range(D):
            prod = sum(gy[t, c] * sx * float(fwd["xq"][t, d]) for t in range(N))
            code = min(7.0, max(-7.0, float(np.rint(vw[c, d]))))
            dlt = code - (vw[c, d] if abs(vw[c, d]) <= 7 else 0.0)
            ref_w += prod * dlt
    ref_x /= np.sqrt(7.0 * N * D)
    ref_w /= np.sqrt(7.0 * C * D)
    assert abs(gs_x - ref_x) <= 1e-10 * max(1.0, abs(ref_x))
    assert abs(gs_w - ref_w) <= 1e-10 * max(1.0, abs(ref_w))
    # the dense chain rule (unquantized grad_Y) is close: BS error is ~1/119 of amax
    dense_x = np.sum(sw * (g.astype(np.float64) @ fwd["wq"].astype(np.float64)) *
                     lsq_grad.delta(hq.transformed_scaled(x, fwd["k"], fwd["s_x"]))) / np.sqrt(7.0 * N * D)
    assert abs(gs_x - dense_x) <= 0.05 * abs(dense_x) + 1e-6


def test_step_grads_sampled_estimate_is_unbiased():
    # Bernoulli LSS with dyadic weights is unbiased for the bit-split product
    # (reading Z-17); the step gradients are linear in it.
    x, w, g, fwd = _setup(N=6, C=4, D=8, k=1, seed=4)
    exact = linear.backward(g, fwd, seed=1, call_id=0, mode=lss.MODE_NONE)
    ex_x, ex_w = linear.step_size_grads(x, w, fwd, exact)
    xs, ws = [], []
    for seed in range(600):
        out = _resample(g, fwd, exact["bs"], seed)
        a, b = linear.step_size_grads(x, w, fwd, out)
        xs.append(a)
        ws.append(b)
    for est, ex in ((np.array(xs), ex_x), (np.array(ws), ex_w)):
        se = est.std(ddof=1) / np.sqrt(len(est)) + 1e-12
        assert abs(est.mean() - ex) < 4.5 * se, (est.mean(), ex, se)


def _resample(g, fwd, bs, seed):
    """Backward with a fixed bit split (fixed SR draw) and fresh Bernoulli masks:
    isolates the sampling step whose unbiasedness the test checks."""
    k = fwd["k"]
    mw = lss.sample_weight_mask(bs["a_sq"], fwd["x_sq"], seed + 1000, 0, 0, lss.MODE_BERNOULLI)
    mx = lss.sample_activation_mask(bs["a_sq"], seed + 1000, 0, 0, lss.MODE_BERNOULLI)
    _, acc_w = linear.grad_w_from_items(bs, mw["items"], mw["wexp"], fwd["xq"], fwd["w_mask"], k, fwd["s_x"])
    return dict(bs=bs, mask_w=mw, mask_x=mx, acc_w=acc_w)
