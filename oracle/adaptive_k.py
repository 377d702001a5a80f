"""Adaptive Hadamard block size (Appendix A.5).
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:654-661 (A.5, "Choose hadamard matrix size"):
    X_bar_k = s_X <X H>_{s_X} H^T,   W_bar_k = s_W <W H>_{s_W} H^T,
    quantization error  MSE(X_bar, X) x MSE(W_bar, W),
    "We search for the optimal k that can minimize this quantization error."
H = BlockDiag(H_k, ..., H_k), normalised.

Readings:
  Z-30  every candidate k is evaluated with the caller's step sizes s_X, s_W (H is
        orthonormal, so the scale of XH does not change with k); MSE is the mean
        over all elements; ties go to the smallest k.  The quantizer is the one of
        the forward path (hq.hadamard_quant, readings Z-4, Z-7).
"""
import numpy as np

from .hadamard import block_diag_hadamard
from .hq import hadamard_quant


def reconstruct(x, k, s):
    """X_bar_k = s <XH>_s H^T, float64."""
    x = np.asarray(x)
    codes, _, _ = hadamard_quant(x, k, s)
    H = block_diag_hadamard(x.shape[1], k)                   # normalised, symmetric
    return np.float64(np.float32(s)) * (codes.astype(np.float64) @ H.T)


def mse(x, k, s):
    """MSE(X_bar_k, X), mean over the elements."""
    x64 = np.asarray(x, dtype=np.float64)
    return float(np.mean((reconstruct(x, k, s) - x64) ** 2))


def quant_error(x, w, k, s_x, s_w):
    """MSE(X_bar, X) x MSE(W_bar, W)."""
    return mse(x, k, s_x) * mse(w, k, s_w)


def select_k(x, w, s_x, s_w, ks):
    """argmin over the candidate k (first on ties).  Returns (k*, {k: (mse_x, mse_w)})."""
    table = {k: (mse(x, k, s_x), mse(w, k, s_w)) for k in ks}
    best = min(ks, key=lambda k: (table[k][0] * table[k][1], k))
    return best, table
