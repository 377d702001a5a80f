"""Bit splitting (BS) of the output gradient.  TEST INFRASTRUCTURE ONLY.

PAPER.md:234-239 (§4.2, Eq. 5): grad_Y ~= s_up grad_up + s_down grad_down, the
two INT4 matrices being "the higher and lower 4 bits of the INT8
representation"; grad_Y is quantized dynamically for each MM.

Readings (listed in DESIGN.md):
  Z-9  one per-tensor dynamic 8-bit code q in [-119, 119] with
       s_down = fl32(amax / 119), s_up = 16 s_down, r8 = fl32(119 / amax).
  Z-10 unbiased stochastic rounding with 32-bit uniforms u, floor form:
       v = clamp(fl32(g * r8), -119, 119); A = ceil(v * 2^32) (an exact integer);
       q = floor((A + u) / 2^32), i.e. q = floor(v) + 1 with probability
       ceil(frac(v) 2^32) / 2^32 and floor(v) otherwise ("round up with
       probability x - floor(x)", Gupta et al. 2015, on a 2^-32 grid).
  Z-11 balanced base-16 split: hi = floor((q + 8) / 16), lo = q - 16 hi,
       hi in [-7, 7], lo in [-8, 7].
amax == 0 is the degenerate case (SPEC bit_split errors): s_down = 0, q = 0.
"""
import numpy as np

from .philox import sr_uniforms

Q8 = 119          # 16 * 7 + 7
TWO32 = 2.0 ** 32


def scales(g):
    """(amax, s_down, r8) as fp32 values from the bf16 gradient g (Z-9)."""
    amax = np.float32(np.abs(np.asarray(g, dtype=np.float64)).max()) if np.size(g) else np.float32(0)
    if amax == 0:
        return np.float32(0), np.float32(0), np.float32(0)
    s_down = np.float32(amax) / np.float32(Q8)
    r8 = np.float32(Q8) / np.float32(amax)
    return np.float32(amax), np.float32(s_down), np.float32(r8)


def stochastic_round(v, u):
    """Floor-form SR of fp32 values v in [-119, 119] with uint32 words u (Z-10).

    Element-wise q = floor((ceil(v 2^32) + u) / 2^32): P(q = floor(v) + 1) =
    T / 2^32 with T = ceil(frac(v) 2^32), the event u >= 2^32 - T.
    """
    v = np.asarray(v, dtype=np.float32)
    # exact: v 2^32 has <= 24 significant bits and |A| < 2^39, so A + u fits int64
    A = np.ceil(v.astype(np.float64) * TWO32).astype(np.int64)
    u = np.asarray(u, dtype=np.uint64).astype(np.int64)
    return np.floor_divide(A + u, np.int64(1) << 32)


def split(q):
    """q = 16 hi + lo with hi = floor((q+8)/16), lo in [-8, 7] (Z-11)."""
    q = np.asarray(q, dtype=np.int64)
    hi = np.floor_divide(q + 8, 16)
    lo = q - 16 * hi
    return hi.astype(np.int8), lo.astype(np.int8)


def bit_split(g, seed, call_id, token_offset=0):
    """BS of g [N, C] (bf16 values).

    Returns dict with q (int64 8-bit codes), hi, lo (int8), s_down, amax,
    a_sq [2, N] = (sum hi^2, sum lo^2) per token (the INT data the leverage
    score is computed from).
    """
    g = np.asarray(g, dtype=np.float32)
    N, C = g.shape
    amax, s_down, r8 = scales(g)
    if amax == 0:
        q = np.zeros((N, C), dtype=np.int64)
    else:
        v = np.clip(g * r8, np.float32(-Q8), np.float32(Q8))   # fp32 multiply, clamp (Z-10)
        assert v.dtype == np.float32
        u = sr_uniforms(seed, call_id, token_offset, N, C)
        q = stochastic_round(v, u)
    hi, lo = split(q)
    a_sq = np.stack([(hi.astype(np.int64) ** 2).sum(axis=1),
                     (lo.astype(np.int64) ** 2).sum(axis=1)])
    return dict(q=q, hi=hi, lo=lo, s_down=np.float32(s_down), amax=amax, a_sq=a_sq)
