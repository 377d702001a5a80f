"""Pins of the oracle's Hadamard transform, LSQ quantizer and hadamard_quant
(SURVEY.md §8(c) P-1..P-4, P-15a).  CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import hadamard, hq, lsq

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("k", range(0, 8))
def test_p1_orthogonal_symmetric(k):
    # PAPER.md:128 "H_k = H_k^T = H_k^{-1}, so H_k H_k = I"; north star: H H^T = nI.
    H = hadamard.hadamard_normalized(k)
    S = hadamard.sylvester_pm1(k)
    n = 1 << k
    assert np.allclose(H, H.T, atol=0)
    assert np.allclose(H @ H, np.eye(n), atol=1e-12)
    assert np.array_equal(S @ S.T, n * np.eye(n))
    assert set(np.unique(S)) <= {-1.0, 1.0}
    # Natural (Sylvester) order, reading Z-5: S[i][j] = (-1)^popcount(i & j)
    ref = np.array([[(-1) ** bin(i & j).count("1") for j in range(n)] for i in range(n)])
    assert np.array_equal(S, ref)
    # the two constructions agree up to the 2^{-k/2} factor (reading Z-4)
    assert np.allclose(S * 2.0 ** (-k / 2), H, atol=1e-15)


@pytest.mark.parametrize("k", range(1, 8))
def test_p2_one_hot_spreads_to_constant(k):
    # e_i^T H_k = 2^{-k/2} 1.  Literally true for i = 0 only; for
    # every i it holds in magnitude (each entry is +-2^{-k/2}) -- reading Z-26.
    n = 1 << k
    M = 37.0
    for i in range(n):
        x = np.zeros((1, 2 * n))
        x[0, n + i] = M                      # second block; first block all zero
        t = hadamard.block_transform_pm1(x, k) * 2.0 ** (-k / 2)
        assert np.array_equal(t[0, :n], np.zeros(n))
        assert np.allclose(np.abs(t[0, n:]), M * 2.0 ** (-k / 2) * np.ones(n), rtol=0, atol=1e-12)
        if i == 0:
            assert np.allclose(t[0, n:], M * 2.0 ** (-k / 2) * np.ones(n), rtol=0, atol=1e-12)


def test_p3_round_trip_and_block_structure():
    # X = (XH)H^T; block-diagonal with blocks H_k (:130-132).
    rng = np.random.default_rng(0)
    for k in (0, 2, 5, 7):
        D = 256
        x = rng.standard_normal((9, D))
        H = hadamard.block_diag_hadamard(D, k)
        assert np.allclose((x @ H) @ H.T, x, atol=1e-12)
        # the per-block transform equals the explicit D x D matrix product
        assert np.allclose(hadamard.block_transform_pm1(x, k) * 2.0 ** (-k / 2), x @ H, atol=1e-12)
        # off-block entries are zero
        b = 1 << k
        mask = np.kron(np.eye(D // b), np.ones((b, b)))
        assert np.array_equal(H * (1 - mask), np.zeros((D, D)))
    with pytest.raises(ValueError):
        hadamard.block_transform_pm1(np.zeros((1, 12)), 3)


def test_p4_lsq_worked_example_and_ties():
    g = json.load(open(os.path.join(GOLD, "lsq_spec.json")))
    codes, mask = lsq.lsq_quantize_real(g["x"], g["s"])
    assert codes.tolist() == g["codes"]
    assert mask.astype(int).tolist() == g["mask"]
    codes, mask = lsq.lsq_quantize(np.array(g["ties_v"], dtype=np.float32))
    assert codes.tolist() == g["ties_codes"]
    assert mask.astype(int).tolist() == g["ties_mask"]
    # fixed points x = j s -> j, mask 1
    s = 0.37
    j = np.arange(-7, 8)
    c, m = lsq.lsq_quantize_real(j * s, s)
    assert np.array_equal(c, j) and m.all()
    # dequantize error <= s/2 on in-range entries (SPEC.md lsq dequantize property)
    x = np.random.default_rng(1).uniform(-3, 3, 1000)
    c, m = lsq.lsq_quantize_real(x, s)
    assert np.all(np.abs(lsq.dequantize(c, s) - x)[m] <= s / 2 + 1e-12)


def test_p15a_hadamard_quant_golden():
    g = json.load(open(os.path.join(GOLD, "hadamard_quant_k2.json")))
    x = np.array(g["x"], dtype=np.float32)
    assert hq.step_reciprocal(g["k"], g["s"]) == np.float32(g["r"])
    t = hadamard.block_transform_pm1(x, g["k"])
    assert t.tolist() == g["t_pm1"]
    assert hq.transformed_scaled(x, g["k"], g["s"]).tolist() == g["v"]
    codes, mask, sq = hq.hadamard_quant(x, g["k"], g["s"])
    assert codes.tolist() == g["codes"]
    assert mask.astype(int).tolist() == g["mask"]
    assert sq.tolist() == g["sqnorm"]


def test_hadamard_quant_matches_explicit_matrix_definition():
    # Independent restatement: codes = clamp(rint((x H_normalized)/s)) computed
    # with the explicit D x D block matrix in float64; the fp32 path may differ
    # only where v is within 1 ulp of a .5 tie (reading Z-7) -- count them.
    rng = np.random.default_rng(3)
    x = rng.standard_normal((64, 128)).astype(np.float32)
    for k in (0, 3, 5, 7):
        s = 0.3
        codes, mask, sq = hq.hadamard_quant(x, k, s)
        v64 = (x.astype(np.float64) @ hadamard.block_diag_hadamard(128, k)) / s
        ref = np.rint(np.clip(v64, -7, 7))
        near_tie = np.abs(np.abs(v64 - np.floor(v64)) - 0.5) < 1e-5
        bad = (codes != ref) & ~near_tie
        assert not bad.any()
        assert np.array_equal(sq, (codes.astype(np.int64) ** 2).sum(1))
        assert np.array_equal(mask[~near_tie], (np.abs(v64) <= 7)[~near_tie])
