"""Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11, "Parallel random numbers:
as easy as 1, 2, 3") -- the counter-based generator the reading Z-20 fixes for
the paper's random draws (SR of grad_Y and the LSS masks m_i ~ Bern(p_i),
PAPER.md:270 §4.2).  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Round function, literally:
    (hi0, lo0) = mulhilo32(0xD2511F53, c0);  (hi1, lo1) = mulhilo32(0xCD9E8D57, c2)
    c = (hi1 ^ c1 ^ k0,  lo1,  hi0 ^ c3 ^ k1,  lo0)
key schedule between rounds: k0 += 0x9E3779B9, k1 += 0xBB67AE85 (mod 2^32).
Ten rounds.  Pinned by the Random123 known-answer vectors in
tests/test_oracle_philox.py.

Stream layout (reading Z-20; shard-invariant because indices are global):
    key     = (seed & 0xffffffff, seed >> 32)
    counter = (idx & 0xffffffff, idx >> 32, purpose, call_id)
  purposes 1 and 4: stochastic rounding of grad_Y.  Element L = (token_offset+t)*C + c
             takes the 16-bit half j = L % 8 (word j // 2; low half for even j) of
             the block with idx = L // 8 from both streams; its 32-bit uniform is
             (half of purpose 1) * 2^16 + (half of purpose 4).
  purpose 2: Bernoulli mask of the weight-gradient LSS; item (h, t) uses word 0
             of idx = 2*(token_offset+t) + h   (h = 0 high half, 1 low half).
  purpose 3: same for the activation-gradient LSS.
"""
import numpy as np

M0 = 0xD2511F53
M1 = 0xCD9E8D57
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK32 = 0xFFFFFFFF

PURPOSE_SR = 1
PURPOSE_MASK_W = 2
PURPOSE_MASK_X = 3
PURPOSE_SR_LOW = 4


def philox4x32_10(ctr, key):
    """Vectorised Philox4x32-10.

    ctr: uint32-compatible array [..., 4]; key: [..., 2] (broadcastable).
    Returns uint32 array [..., 4].
    """
    c = np.asarray(ctr, dtype=np.uint64) & MASK32
    k = np.asarray(key, dtype=np.uint64) & MASK32
    c0, c1, c2, c3 = c[..., 0], c[..., 1], c[..., 2], c[..., 3]
    k0 = np.broadcast_to(k[..., 0], c0.shape).copy()
    k1 = np.broadcast_to(k[..., 1], c0.shape).copy()
    for r in range(10):
        if r > 0:
            k0 = (k0 + W0) & MASK32
            k1 = (k1 + W1) & MASK32
        p0 = np.uint64(M0) * c0          # < 2^64, exact in uint64
        p1 = np.uint64(M1) * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0), lo1, (hi0 ^ c3 ^ k1), lo0
    return np.stack([c0, c1, c2, c3], axis=-1).astype(np.uint32)


def _key(seed):
    seed = int(seed)
    return np.array([seed & MASK32, (seed >> 32) & MASK32], dtype=np.uint64)


def _counter(idx, purpose, call_id):
    idx = np.asarray(idx, dtype=np.uint64)
    ctr = np.empty(idx.shape + (4,), dtype=np.uint64)
    ctr[..., 0] = idx & MASK32
    ctr[..., 1] = idx >> np.uint64(32)
    ctr[..., 2] = purpose
    ctr[..., 3] = int(call_id) & MASK32
    return ctr


def sr_uniforms(seed, call_id, token_offset, n_rows, n_cols):
    """32-bit uniform for every grad_Y element (purposes 1 and 4, Z-20).

    Returns uint64 array [n_rows, n_cols] with values in [0, 2^32).
    """
    t = np.arange(n_rows, dtype=np.uint64)[:, None] + np.uint64(token_offset)
    c = np.arange(n_cols, dtype=np.uint64)[None, :]
    L = t * np.uint64(n_cols) + c
    j = (L & np.uint64(7)).astype(np.int64)
    halves = []
    for purpose in (PURPOSE_SR, PURPOSE_SR_LOW):
        blocks = philox4x32_10(_counter(L >> np.uint64(3), purpose, call_id), _key(seed))
        word = np.take_along_axis(blocks, (j // 2)[..., None], axis=-1)[..., 0].astype(np.uint64)
        halves.append(np.where(j % 2 == 0, word & np.uint64(0xFFFF), word >> np.uint64(16)))
    return halves[0] * np.uint64(65536) + halves[1]


def mask_uniforms(seed, call_id, token_offset, n_tokens, purpose):
    """32-bit uniform for each LSS item (h, t), h in {0: high, 1: low}.

    Returns uint64 array [2, n_tokens] (row h).
    """
    t = np.arange(n_tokens, dtype=np.uint64)[None, :] + np.uint64(token_offset)
    h = np.arange(2, dtype=np.uint64)[:, None]
    idx = np.uint64(2) * t + h
    blocks = philox4x32_10(_counter(idx, purpose, call_id), _key(seed))
    return blocks[..., 0].astype(np.uint64)
