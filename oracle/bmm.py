"""BMM in attention (Appendix A.1).  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:570-604 (A.1): T = BMM(Q, K^T), Q in R^{B x N x M}, K in R^{B x P x M};
H_hat = Repeat_B(BlockDiag(H_k, ...));
T ~ BMM(BMM(Q, H_hat), BMM(K, H_hat)^T), "batch step size"
s_Q, s_K in R^B; LSS with per-batch leverage scores c_{b,i}
(PAPER.md:598-603).

Reading:
  Z-31  a BMM is B independent instances of the linear operator: batch b is
        HQ-MM / LSS-MM with X = Q_b (N tokens x M features), W = K_b (P rows x M),
        steps s_Q[b], s_K[b], so T_b = s_Q[b] s_K[b] Q_hat_b K_hat_b^T.  The backward
        is Eq. 4 per batch (the chain rule; the A.1 gradient formulas at
        PAPER.md:589-592 are garbled in operand order and step names); each batch
        samples with its own per-tensor amax and budget N; the Philox token index
        of token t of batch b is b N + t (reading Z-20 with token_offset = b N).
"""
import numpy as np

from . import linear
from . import lss as lss_mod


def forward(q, k_, kh, s_q, s_k):
    """Per-batch HQ-MM.  q [B, N, M], k_ [B, P, M]; s_q, s_k length-B.  Returns the
    list of per-batch forward dicts and T [B, N, P] (float64)."""
    fwds = [linear.forward(q[b], k_[b], kh, s_q[b], s_k[b]) for b in range(q.shape[0])]
    return fwds, np.stack([f["y"] for f in fwds])


def backward(dt, fwds, seed, call_id, mode=lss_mod.MODE_BERNOULLI):
    """Per-batch LSS-MM.  dt [B, N, P].  Returns (dQ [B, N, M], dK [B, P, M], outs)."""
    N = dt.shape[1]
    outs = [linear.backward(dt[b], fwds[b], seed, call_id, token_offset=b * N, mode=mode)
            for b in range(dt.shape[0])]
    return np.stack([o["dx"] for o in outs]), np.stack([o["dw"] for o in outs]), outs
