"""Pins of the oracle's Philox generator and integer GEMM (SURVEY.md §8(c) P-9,
P-6, P-5).  CPU only."""
import numpy as np

from oracle import gemm, hadamard, linear, philox


def test_p9_philox_known_answers():
    # Random123 philox4x32-10 known-answer vectors (Salmon et al. 2011).
    kat = [
        ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
        ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
        ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
         [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
    ]
    for ctr, key, out in kat:
        assert philox.philox4x32_10(ctr, key).tolist() == out
    # vectorised evaluation equals element-wise evaluation
    ctrs = np.array([k[0] for k in kat], dtype=np.uint64)
    keys = np.array([k[1] for k in kat], dtype=np.uint64)
    assert philox.philox4x32_10(ctrs, keys).tolist() == [k[2] for k in kat]


def test_philox_stream_layout_is_shard_invariant():
    # Z-20: words depend on the global token index only.
    full = philox.sr_uniforms(7, 3, 0, 10, 12)
    shard = philox.sr_uniforms(7, 3, 4, 6, 12)
    assert np.array_equal(full[4:], shard)
    mw = philox.mask_uniforms(7, 3, 0, 10, philox.PURPOSE_MASK_W)
    assert np.array_equal(mw[:, 4:], philox.mask_uniforms(7, 3, 4, 6, philox.PURPOSE_MASK_W))
    # distinct purposes give distinct streams
    mx = philox.mask_uniforms(7, 3, 0, 10, philox.PURPOSE_MASK_X)
    assert not np.array_equal(mw, mx)
    # uniformity sanity: mean of 2^16 words near 2^31
    u = philox.sr_uniforms(1, 0, 0, 256, 256).astype(np.float64) / 2 ** 32
    assert abs(u.mean() - 0.5) < 0.01 and u.min() >= 0 and u.max() < 1


def test_sr_uniform_halves_layout():
    # Z-20: element L's uniform is (16-bit half L % 8 of block L // 8, purpose 1) << 16
    # plus the same half of purpose 4; halves are independent and uniform.
    n_rows, n_cols, t0 = 3, 40, 2
    u = philox.sr_uniforms(9, 5, t0, n_rows, n_cols)
    key = [9, 0]
    for (t, c) in [(0, 0), (0, 7), (1, 13), (2, 39)]:
        L = (t0 + t) * n_cols + c
        b1 = philox.philox4x32_10([L // 8, 0, philox.PURPOSE_SR, 5], key).tolist()
        b4 = philox.philox4x32_10([L // 8, 0, philox.PURPOSE_SR_LOW, 5], key).tolist()
        j = L % 8
        h1 = (b1[j // 2] >> (16 * (j % 2))) & 0xFFFF
        h4 = (b4[j // 2] >> (16 * (j % 2))) & 0xFFFF
        assert int(u[t, c]) == (h1 << 16) | h4
    big = philox.sr_uniforms(2, 0, 0, 256, 256)
    lo, hi = (big & 0xFFFF).astype(np.float64), (big >> 16).astype(np.float64)
    assert abs(lo.mean() / 65536 - 0.5) < 0.01 and abs(hi.mean() / 65536 - 0.5) < 0.01
    assert abs(np.corrcoef(lo.ravel(), hi.ravel())[0, 1]) < 0.02


def test_p6_int_gemm_brute_force():
    assert gemm.int_matmul_abt([[1, 2]], [[3, 4]]).tolist() == [[11]]
    rng = np.random.default_rng(0)
    for (m, n, k) in [(1, 1, 1), (7, 5, 3), (16, 16, 64), (33, 17, 64)]:
        a = rng.integers(-8, 8, (m, k))
        b = rng.integers(-128, 128, (n, k))
        assert np.array_equal(gemm.int_matmul_abt(a, b), gemm.int_matmul_bruteforce(a, b))


def test_int_gemm_overflow_guard():
    a = np.full((1, 200000), 112, dtype=np.int64)
    b = np.full((1, 200000), 112, dtype=np.int64)
    try:
        gemm.int_matmul_abt(a, b)
    except OverflowError:
        return
    raise AssertionError("int32 bound not enforced")


def test_p5_hadamard_cancellation_and_lossless_case():
    rng = np.random.default_rng(5)
    N, D, C, k = 16, 64, 8, 3
    x = rng.standard_normal((N, D))
    w = rng.standard_normal((C, D))
    H = hadamard.block_diag_hadamard(D, k)
    # (XH)(WH)^T = X W^T when nothing is quantized
    assert np.allclose((x @ H) @ (w @ H).T, x @ w.T, atol=1e-10)
    # lossless case k = 0, X = s_X * ints, W = s_W * ints -> Y = X W^T exactly
    sx, sw = 0.5, 0.25
    xi = rng.integers(-7, 8, (N, D))
    wi = rng.integers(-7, 8, (C, D))
    f = linear.forward((xi * sx).astype(np.float32), (wi * sw).astype(np.float32), 0, sx, sw)
    assert np.array_equal(f["xq"], xi) and np.array_equal(f["wq"], wi)
    assert np.array_equal(f["y"], (xi * sx) @ (wi * sw).T)
