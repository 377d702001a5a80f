"""LSQ step-size gradients (A.3) and the cold-start step rule (A.4).
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:636-646 (A.3, "Learning Quantizer Parameters"):
    grad_{s_W} = g(s_W) grad_Y^T X_hat o delta_W(s_W),
    grad_{s_X} = g(s_X) grad_Y W_hat  o delta_X(s_X),
    g(s) = 1 / sqrt(Q_P N_elem),
    delta_X(s_X) = <X>_{s_X} - I_X o (X / s_X)      (and the same for W).
PAPER.md:647-648: the products grad_Y^T X_hat and grad_Y W_hat are the ones the
backward already computes, so only the elementwise
multiplication with delta is added.
PAPER.md:650-652 (A.4, cold start): in the first iterations the step of each
tensor X is set to 2 mean(X) / sqrt(Q_P) instead of being learned.

Readings:
  Z-27  The quantizer of HQ-MM acts on the transformed, scaled value
        v = fl32(fl32(x H_pm1) * fl32(2^{-k/2}/s)) (hq.py), so delta is taken on v:
        delta = clamp(rint(v), -7, 7) - 1(|v| <= 7) v  (exact in fp32).
  Z-28  "grad_Y W_hat o delta_X" is summed over all elements to the scalar
        gradient, and the partner step size is included (the chain rule through
        Eq. 3: Y = (s_X X_hat)(s_W W_hat)^T):
            grad_{s_X} = g(s_X) sum_{t,d} [s_W grad_Y W_hat]_{t,d} delta_X[t,d]
            grad_{s_W} = g(s_W) sum_{c,d} [s_X grad_Y^T X_hat]_{c,d} delta_W[c,d]
        with the backward's estimates of the two products (the sampled bit-split
        products of LSS-MM, before the mask and the inverse transform).
  Z-29  N_elem = the element count of the quantized tensor (N D for X, C D for W);
        under token sharding the caller passes the global count.
  Z-25  (existing) cold start: s = 2 mean|X| / sqrt(Q_P) on the untransformed
        tensor, rounded once to fp32.
"""
import numpy as np

from .lsq import Q_P, lsq_quantize


def delta(v):
    """delta = <v> - I o v for already-scaled quantizer inputs v (PAPER.md:641-642,
    reading Z-27).  float64 result (exact for fp32 v)."""
    v = np.asarray(v)
    codes, mask = lsq_quantize(v)
    return codes.astype(np.float64) - np.where(mask, v.astype(np.float64), 0.0)


def grad_scale(n_elem):
    """g = 1 / sqrt(Q_P N_elem)."""
    return 1.0 / np.sqrt(np.float64(Q_P) * np.float64(n_elem))


def step_size_grad(product, delta_t, n_elem):
    """g(s) sum(product o delta) (reading Z-28)."""
    return grad_scale(n_elem) * float(np.sum(np.asarray(product, dtype=np.float64) *
                                             np.asarray(delta_t, dtype=np.float64)))


def cold_start_step(x):
    """A.4: 2 mean|X| / sqrt(Q_P), float64 then one rounding to fp32."""
    x = np.asarray(x, dtype=np.float64)
    return np.float32(2.0 * np.abs(x).mean() / np.sqrt(np.float64(Q_P)))
