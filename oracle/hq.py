"""hadamard_quant: steps 1-2 of Procedure HQ-MM for one matrix.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:150-153 (Procedure HQ-MM): "Compute XH and H^T W^T ...  Quantize the
resultant matrices to INT4 by LSQ."  PAPER.md:204-205: X_hat = <XH>_{s_X},
I_X = 1(-Q_N <= XH/s_X <= Q_P) (reading Z-8: the indicator is taken on the
transformed, scaled value, which is what the chain rule through Eq. 3 gives).

Arithmetic (readings Z-4, Z-7):
  t   = x . BlockDiag(S_k)               exact, float64, S_k the +-1 Sylvester matrix
  t32 = fl32(t)
  r   = fl32(2^{-k/2} / s)               computed in float64, rounded once
  v   = fl32(t32 * r)                    one IEEE fp32 multiply
  code = clamp(round_half_even(v), -7, 7);  mask = (-7 <= v <= 7)
  sqnorm_row = sum_j code_j^2            (the ||X_hat_i|| of the leverage score,
                                          PAPER.md:296, from INT data, :680)
"""
import numpy as np

from .hadamard import block_transform_pm1
from .lsq import lsq_quantize


def step_reciprocal(k, s):
    """r = fl32(2^{-k/2} / s), s given as an fp32 value (Z-4)."""
    s = np.float64(np.float32(s))
    if not (s > 0 and np.isfinite(s)):
        raise ValueError("step size must be positive and finite (SPEC lsq pre)")
    return np.float32(2.0 ** (-k / 2.0) / s)


def hadamard_quant(x, k, s):
    """x: [rows, cols] array of bf16 values (any float dtype holding them exactly).

    Returns (codes int8 [rows, cols], mask bool [rows, cols], sqnorm int64 [rows]).
    """
    t32 = block_transform_pm1(x, k).astype(np.float32)
    v = t32 * step_reciprocal(k, s)                      # float32 * float32 -> float32
    assert v.dtype == np.float32
    codes, mask = lsq_quantize(v)
    sqnorm = (codes.astype(np.int64) ** 2).sum(axis=1)
    return codes, mask, sqnorm


def transformed_scaled(x, k, s):
    """v = fl32(fl32(xH_pm1) * r) -- exposed so tests can locate rounding ties."""
    return block_transform_pm1(x, k).astype(np.float32) * step_reciprocal(k, s)
