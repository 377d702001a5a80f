"""Hadamard matrices and the block-diagonal transform of HQ.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:118-128 (§3.3): H_0 = [1], H_k = 2^{-1/2} [[H_{k-1}, H_{k-1}],
[H_{k-1}, -H_{k-1}]]; H_k = H_k^T = H_k^{-1}.
PAPER.md:130-132: H = BlockDiag(H_k, ..., H_k) in R^{D x D}, D a multiple of 2^k.

Readings: Z-4 the 2^{-k/2} normalisation is carried separately,
the transform itself uses the unnormalised +-1 Sylvester matrix; Z-5 natural
(Sylvester) order; Z-6 contiguous blocks from column 0.
"""
import numpy as np


def sylvester_pm1(k):
    """Unnormalised +-1 Sylvester matrix of order 2^k, built by the paper's
    recursion without the 1/sqrt(2) factors."""
    if not (0 <= k <= 12):
        raise ValueError("k out of range")
    H = np.ones((1, 1), dtype=np.float64)
    for _ in range(k):
        H = np.block([[H, H], [H, -H]])
    return H


def hadamard_normalized(k):
    """H_k exactly as PAPER.md:123 (1/sqrt(2) per level), in float64."""
    H = np.ones((1, 1), dtype=np.float64)
    for _ in range(k):
        H = np.block([[H, H], [H, -H]]) / np.sqrt(2.0)
    return H


def block_diag_hadamard(D, k, normalized=True):
    """H = BlockDiag(H_k, ..., H_k) in R^{D x D}."""
    b = 1 << k
    if D % b:
        raise ValueError("D must be a multiple of 2^k (PAPER.md:132)")
    Hk = hadamard_normalized(k) if normalized else sylvester_pm1(k)
    H = np.zeros((D, D), dtype=np.float64)
    for j in range(D // b):
        H[j * b:(j + 1) * b, j * b:(j + 1) * b] = Hk
    return H


def block_transform_pm1(x, k):
    """t = x . BlockDiag(S_k) with S_k the +-1 Sylvester matrix, per b-block of
    each row (PAPER.md:130-136 with reading Z-4).  float64, one library matmul
    per block position; exact for bf16 inputs whose block spans < 45-k binades.
    """
    x = np.asarray(x, dtype=np.float64)
    rows, D = x.shape
    b = 1 << k
    if D % b:
        raise ValueError("D must be a multiple of 2^k (PAPER.md:132)")
    S = sylvester_pm1(k)
    xb = x.reshape(rows, D // b, b)
    return (xb @ S).reshape(rows, D)        # S symmetric: x.S == x.S^T
