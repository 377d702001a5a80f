"""Pins of the A.1 BMM oracle.  CPU only.  Checked against
numpy einsum forms of the BMM definition and of the per-batch chain rule, not
against linear.py."""
import numpy as np

from oracle import bmm, lss


def test_lossless_bmm_is_exact():
    # Q, K on their LSQ grids and k = 0: T = Q K^T exactly
    rng = np.random.default_rng(0)
    B, N, P, M = 3, 8, 16, 32
    s_q = np.array([0.5, 0.25, 1.0], dtype=np.float32)
    s_k = np.array([0.125, 0.5, 0.25], dtype=np.float32)
    q = (rng.integers(-7, 8, (B, N, M)) * s_q[:, None, None]).astype(np.float32)
    k_ = (rng.integers(-7, 8, (B, P, M)) * s_k[:, None, None]).astype(np.float32)
    fwds, T = bmm.forward(q, k_, 0, s_q, s_k)
    assert np.array_equal(T, np.einsum("bnm,bpm->bnp", q.astype(np.float64), k_.astype(np.float64)))
    # each batch is quantized with its own step sizes
    assert all(f["s_x"] == s_q[b] and f["s_w"] == s_k[b] for b, f in enumerate(fwds))


def test_bmm_backward_exact_bit_split_chain_rule():
    # dT on each batch's 8-bit grid (amax = 119/32 -> exact BS product), mode NONE:
    # dQ_b = [I_Q o (s_K dT_b K_hat_b)] H, dK_b = s_Q [(dT_b^T Q_hat_b) o I_K] H (Eq. 4 per batch)
    rng = np.random.default_rng(1)
    B, N, P, M, kh = 2, 6, 8, 16, 2
    q = rng.standard_normal((B, N, M)).astype(np.float32)
    k_ = (rng.standard_normal((B, P, M)) * 0.5).astype(np.float32)
    s_q = np.array([0.3, 0.4], dtype=np.float32)
    s_k = np.array([0.2, 0.15], dtype=np.float32)
    fwds, _ = bmm.forward(q, k_, kh, s_q, s_k)
    qi = rng.integers(-119, 120, (B, N, P))
    qi[:, 0, 0] = 119
    dt = (qi / 32.0).astype(np.float32)
    dQ, dK, _ = bmm.backward(dt, fwds, seed=3, call_id=1, mode=lss.MODE_NONE)
    b_ = 1 << kh
    H = np.zeros((M, M))
    for i in range(M):
        for j in range(M):
            if i // b_ == j // b_:
                H[i, j] = (-1) ** bin((i % b_) & (j % b_)).count("1") / np.sqrt(b_)
    for b in range(B):
        f = fwds[b]
        g = qi[b].astype(np.float64) / 32.0
        ref_q = (f["x_mask"] * (np.float64(s_k[b]) * np.einsum("np,pm->nm", g, f["wq"].astype(np.float64)))) @ H
        ref_k = np.float64(s_q[b]) * (np.einsum("np,nm->pm", g, f["xq"].astype(np.float64)) * f["w_mask"]) @ H
        assert np.allclose(dQ[b], ref_q, rtol=0, atol=1e-12)
        assert np.allclose(dK[b], ref_k, rtol=0, atol=1e-12)


def test_bmm_batches_draw_distinct_streams():
    # token index b N + t (reading Z-31): two identical batches get different SR draws
    rng = np.random.default_rng(2)
    B, N, P, M = 2, 16, 8, 16
    q1 = rng.standard_normal((1, N, M)).astype(np.float32)
    k1 = rng.standard_normal((1, P, M)).astype(np.float32)
    q = np.concatenate([q1, q1])
    k_ = np.concatenate([k1, k1])
    s = np.array([0.3, 0.3], dtype=np.float32)
    fwds, T = bmm.forward(q, k_, 2, s, s)
    assert np.array_equal(T[0], T[1])
    dt = (rng.standard_normal((1, N, P)) * 0.37).astype(np.float32)
    dt = np.concatenate([dt, dt])
    _, _, outs = bmm.backward(dt, fwds, seed=9, call_id=0, mode=lss.MODE_NONE)
    assert not np.array_equal(outs[0]["bs"]["q"], outs[1]["bs"]["q"])
