"""Pins of the A.5 adaptive-k oracle.  CPU only."""
import numpy as np

from oracle import adaptive_k, lsq


def _popcount_h(D, k):
    """Normalised block-diagonal Hadamard written entry by entry from the
    popcount form of the Sylvester order (reading Z-5), not from hadamard.py."""
    b = 1 << k
    H = np.zeros((D, D))
    for i in range(D):
        for j in range(D):
            if i // b == j // b:
                H[i, j] = (-1) ** bin((i % b) & (j % b)).count("1") / np.sqrt(b)
    return H


def test_k0_is_plain_lsq_error():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((9, 32)).astype(np.float32)
    s = np.float32(0.3)
    codes, _ = lsq.lsq_quantize_real(x, s)
    ref = np.mean((np.float64(s) * codes - x.astype(np.float64)) ** 2)
    assert abs(adaptive_k.mse(x, 0, s) - ref) < 1e-15


def test_reconstruction_brute_force():
    rng = np.random.default_rng(1)
    D, k, s = 16, 3, np.float32(0.25)
    x = rng.standard_normal((5, D)).astype(np.float32)
    H = _popcount_h(D, k)
    t = x.astype(np.float64) @ H
    codes = np.rint(np.clip(t / np.float64(s), -7, 7))
    ref = np.float64(s) * codes @ H.T
    got = adaptive_k.reconstruct(x, k, s)
    # codes may differ only where t/s sits within fp32 rounding of a tie (Z-7)
    assert np.abs(got - ref).max() < 1e-12 or np.mean(np.abs(got - ref) > 1e-12) < 0.02


def test_exactly_representable_input_selects_its_k():
    # x = s c H^T with integer c in [-7, 7]: X_bar_{k0} = x exactly,
    # so the error product is 0 at k0 and positive elsewhere.
    rng = np.random.default_rng(2)
    D, k0 = 64, 4
    s = np.float32(0.5)
    H = _popcount_h(D, k0)
    cx = rng.integers(-7, 8, (12, D)).astype(np.float64)
    cw = rng.integers(-7, 8, (8, D)).astype(np.float64)
    x = (np.float64(s) * cx @ H.T).astype(np.float32)
    w = (np.float64(s) * cw @ H.T).astype(np.float32)
    assert np.array_equal(x.astype(np.float64), np.float64(s) * cx @ H.T)   # exact in fp32
    best, table = adaptive_k.select_k(x, w, s, s, list(range(0, 7)))
    assert best == k0
    assert table[k0][0] < 1e-20 and table[k0][1] < 1e-20          # exact up to the 1/sqrt(2) products of H
    assert all(table[k][0] * table[k][1] > 1e-6 for k in table if k != k0)


def test_hadamard_helps_with_outlier_columns():
    # the paper's motivation: outlier columns inflate the
    # k = 0 error; spreading them over a block reduces it
    rng = np.random.default_rng(3)
    x = rng.standard_normal((64, 128)).astype(np.float32)
    x[:, 5] *= 40.0
    x[:, 77] *= 40.0
    w = (rng.standard_normal((32, 128)) * 0.02).astype(np.float32)
    sx = np.float32(2 * np.abs(x).mean() / np.sqrt(7))
    sw = np.float32(2 * np.abs(w).mean() / np.sqrt(7))
    e0 = adaptive_k.mse(x, 0, sx)
    assert adaptive_k.mse(x, 5, sx) < 0.5 * e0
    best, _ = adaptive_k.select_k(x, w, sx, sw, list(range(0, 8)))
    assert best > 0
