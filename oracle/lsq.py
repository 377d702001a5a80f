"""LSQ quantizer (Esser et al.) as used by the paper.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:78-83 (§3.1, Eq. 2):  <X>_s = round(clamp(X / s, -Q_N, Q_P)),
Q_N = Q_P = 7.  PAPER.md:84-85: dequantize s . <X>_s.
PAPER.md:205 (§4): clamp indicator I = 1(-Q_N <= X/s <= Q_P) (inclusive).

Readings: Z-1 round = round-half-to-even; Z-2 clamp(round(v)) == round(clamp(v))
for integer bounds; Z-3 codes in [-7, 7].
"""
import numpy as np

Q_N = 7
Q_P = 7


def lsq_quantize(v):
    """Codes and clamp mask for already-scaled values v = X/s (any float dtype).

    Returns (codes int8, mask bool).
    """
    v = np.asarray(v)
    codes = np.rint(np.clip(v, -Q_N, Q_P)).astype(np.int8)   # rint: half-to-even
    mask = (v >= -Q_N) & (v <= Q_P)
    return codes, mask


def lsq_quantize_real(x, s):
    """Eq. 2 evaluated in float64 on a real matrix x with step s (used by the
    worked-example pins, where k = 0 and no transform is involved)."""
    return lsq_quantize(np.asarray(x, dtype=np.float64) / np.float64(s))


def dequantize(codes, s):
    """s . <X>_s."""
    return np.float64(s) * np.asarray(codes, dtype=np.float64)
