"""Pins of the composed oracle backward and of the
chain-rule reference it is measured against.  CPU only."""
import numpy as np

from oracle import hadamard, linear, lss


def _setup(N=8, C=8, D=8, k=2, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((N, D)).astype(np.float32)
    x[:, 1] *= 8.0                                          # an outlier column
    w = (rng.standard_normal((C, D)) * 0.5).astype(np.float32)
    fwd = linear.forward(x, w, k, 0.35, 0.2)
    assert 0 < fwd["x_mask"].mean() < 1                     # some clamping present
    return rng, x, w, fwd


def test_p14_exact_bs_product_on_the_8bit_grid():
    # grad_Y = s_down q exactly (amax = 119/32 -> r8 = 32, s_down = 2^-5), mode NONE:
    # grad_X = [I_X o (s_W s_down q W_hat)] H,  grad_W = s_X s_down [(q^T X_hat) o I_W] H.
    rng, x, w, fwd = _setup()
    N, D = x.shape
    C = w.shape[0]
    q = rng.integers(-119, 120, (N, C))
    q[0, 0] = 119
    q[3] = 0
    g = (q / 32.0).astype(np.float32)
    out = linear.backward(g, fwd, seed=5, call_id=1, mode=lss.MODE_NONE)
    assert np.array_equal(out["bs"]["q"], q)
    H = hadamard.block_diag_hadamard(D, fwd["k"])
    sd = 2.0 ** -5
    dx = (fwd["x_mask"] * (np.float64(fwd["s_w"]) * sd * (q @ fwd["wq"].astype(np.float64)))) @ H
    dw = np.float64(fwd["s_x"]) * sd * ((q.T @ fwd["xq"].astype(np.float64)) * fwd["w_mask"]) @ H
    assert np.allclose(out["dx"], dx, rtol=0, atol=1e-12)
    assert np.allclose(out["dw"], dw, rtol=0, atol=1e-12)
    rdx, rdw = linear.backward_dense_reference(g, fwd)
    assert np.allclose(rdx, dx, atol=1e-12) and np.allclose(rdw, dw, atol=1e-12)
    # KEEP_POSITIVE drops only zero rows -> the same product here
    out2 = linear.backward(g, fwd, seed=5, call_id=1, mode=lss.MODE_KEEP_POSITIVE)
    assert np.allclose(out2["dx"], dx, atol=1e-12) and np.allclose(out2["dw"], dw, atol=1e-12)


def test_p14_ste_finite_differences():
    # The chain-rule reference (Eq. 4) is the derivative of the
    # STE surrogate where round' = 1: Y~ = s_W clamp(XH, +-7 s_X) W_hat^T, and
    # Y~ = s_X X_hat clamp(WH, +-7 s_W)^T.  Central differences off the kinks.
    rng, x, w, fwd = _setup(seed=1)
    k, sx, sw = fwd["k"], np.float64(fwd["s_x"]), np.float64(fwd["s_w"])
    N, D = x.shape
    H = hadamard.block_diag_hadamard(D, k)
    G = rng.standard_normal((N, w.shape[0]))
    dx_ref, dw_ref = linear.backward_dense_reference(G, fwd)
    x64, w64 = x.astype(np.float64), w.astype(np.float64)

    def Lx(X):
        return (G * (sw * np.clip(X @ H, -7 * sx, 7 * sx) @ fwd["wq"].T.astype(np.float64))).sum()

    def Lw(W):
        return (G * (sx * fwd["xq"].astype(np.float64) @ np.clip(W @ H, -7 * sw, 7 * sw).T)).sum()

    eps = 1e-6
    vx = np.abs(x64 @ H) / sx
    vw = np.abs(w64 @ H) / sw
    checked = 0
    for (i, j) in [(a, b) for a in range(N) for b in range(D)]:
        blk = slice((j >> k) << k, ((j >> k) + 1) << k)
        if np.any(np.abs(vx[i, blk] - 7) < 1e-3):
            continue
        e = np.zeros_like(x64); e[i, j] = eps
        fd = (Lx(x64 + e) - Lx(x64 - e)) / (2 * eps)
        assert abs(fd - dx_ref[i, j]) <= 1e-4 * (1 + abs(dx_ref[i, j]))
        checked += 1
    for (i, j) in [(a, b) for a in range(w.shape[0]) for b in range(D)]:
        blk = slice((j >> k) << k, ((j >> k) + 1) << k)
        if np.any(np.abs(vw[i, blk] - 7) < 1e-3):
            continue
        e = np.zeros_like(w64); e[i, j] = eps
        fd = (Lw(w64 + e) - Lw(w64 - e)) / (2 * eps)
        assert abs(fd - dw_ref[i, j]) <= 1e-4 * (1 + abs(dw_ref[i, j]))
        checked += 1
    assert checked > 60


def test_p16_whole_backward_unbiased_monte_carlo():
    # E over Philox seeds of the sampled backward = Eq. 4 with the unquantized
    # grad_Y (SR unbiased per element, LSS unbiased given the codes).
    rng, x, w, fwd = _setup(seed=2)
    N, C = 8, 8
    r = np.array([1, 1, 0.05, 0.02, 0, 0.3, 0.01, 0.2])[:, None]
    g = (rng.standard_normal((N, C)) * r).astype(np.float32)
    ref_dx, ref_dw = linear.backward_dense_reference(g, fwd)
    T = 3000
    sx = np.zeros_like(ref_dx); sx2 = np.zeros_like(ref_dx)
    sw = np.zeros_like(ref_dw); sw2 = np.zeros_like(ref_dw)
    kept = []
    for seed in range(T):
        out = linear.backward(g, fwd, seed=seed, call_id=7)
        sx += out["dx"]; sx2 += out["dx"] ** 2
        sw += out["dw"]; sw2 += out["dw"] ** 2
        kept.append(out["mask_w"]["count"])
    for s1, s2, ref in ((sx, sx2, ref_dx), (sw, sw2, ref_dw)):
        mean = s1 / T
        se = np.sqrt(np.maximum(s2 / T - mean ** 2, 0) / T)
        z = np.abs(mean - ref) / np.maximum(se, 1e-12 * (1 + np.abs(ref)))
        assert np.all(z < 5.0), z.max()
        # and the estimate is not trivially noisy: relative Frobenius bias small
        assert np.linalg.norm(mean - ref) < 0.05 * np.linalg.norm(ref)
    assert np.mean(kept) <= N + 1            # budget N (plus the 1/16 floor)


def test_o12_grad_w_folding_matches_the_paper_form_per_sample():
    """the oracle's grad_W folds the item weight into the A
    operand (2^wexp code, |.| <= 128) and s_up = 16 s_down into the B operand
    (16 X_hat on high-half rows).  For single mask draws (not in expectation) the
    folded accumulator times s_down must equal, exactly in rationals, the paper's
    form sum_kept (m_i / p_i) s_h code_i (x) X_hat_t (Eq. 5:
    s_h = s_up for the high half, s_down for the low), with the drawn weight
    2^wexp in the role of m_i / p_i; and the finished grad_W must equal
    s_X [P o I_W] H with P summed item by item in float64."""
    from fractions import Fraction

    weighted = False
    for seed in range(4):
        rng, x, w, fwd = _setup(N=24, C=16, D=32, k=3, seed=seed)
        g = rng.standard_normal((24, 16)).astype(np.float32) * np.where(rng.random(24) < 0.3, 1.0, 0.02)[:, None]
        g = g.astype(np.float32)
        out = linear.backward(g, fwd, seed=seed, call_id=2)
        bs, mw = out["bs"], out["mask_w"]
        assert mw["count"] > 0
        weighted |= bool(np.any(mw["wexp"] > 0))            # the draw up-weighted some items
        N = g.shape[0]
        s_down = Fraction(float(bs["s_down"]))
        xq = fwd["xq"].astype(np.int64)
        P = np.zeros((16, 32))
        entries = [(0, 0), (3, 7), (15, 31), (8, 16)]
        exact = {e: Fraction(0) for e in entries}
        for i, e in zip(mw["items"], mw["wexp"]):
            h, t = int(i) // N, int(i) % N
            code = (bs["hi"] if h == 0 else bs["lo"])[t].astype(np.int64)
            s_h = 16 * s_down if h == 0 else s_down
            weight = Fraction(2) ** int(e)
            P += float(weight) * float(s_h) * np.outer(code, xq[t])
            for (c, d) in entries:
                exact[(c, d)] += weight * s_h * int(code[c]) * int(xq[t, d])
        for (c, d) in entries:
            assert Fraction(int(out["acc_w"][c, d])) * s_down == exact[(c, d)]
        H = hadamard.block_diag_hadamard(32, fwd["k"])
        dw_paper = np.float64(fwd["s_x"]) * (P * fwd["w_mask"]) @ H
        assert np.allclose(out["dw"], dw_paper, rtol=1e-12, atol=1e-12 * np.abs(dw_paper).max())
    assert weighted
