"""Leverage score sampling (LSS).  TEST INFRASTRUCTURE ONLY.

PAPER.md:258-287 (§4.2, Eq. 7): the BS product is a sum of 2N rank-1 terms;
each gets p_i in [0, 1] with sum_i p_i = N, m_i ~ Bern(p_i), and the estimator
sum_i (m_i / p_i) term_i is unbiased.  PAPER.md:289-305 (Prop. 1): variance
sum_i (1-p_i)/p_i c_i^2, minimised by p_i proportional to the leverage score
c_i = ||grad_updown_i|| ||X_updown_i|| (weight gradient, :296) or
c_i = ||grad_updown_i|| (activation gradient, :365, B.2 :758-777).
PAPER.md:606-610 (A.2): clamp to [0, 1], rescale the rest to sum N, repeat.
PAPER.md:682 (A.6): the authors' timed implementation keeps every row with
score > 0 (mode KEEP_POSITIVE here).

Readings: Z-12 items (h, t) with id h*N + t, h = 0 high / 1 low;
Z-13 integer-exact scores; Z-14 the A.2 loop run to its fixed point; Z-15
zero-score items never kept; Z-16 if at most N items are positive all of them
get p = 1; Z-17 dyadic two-threshold Bernoulli rule with weights in
{2^e, 2^{e+1}} (exactly unbiased), with a floor weight 2^E_MAX; Z-18 separate
masks for grad_W and grad_X; Z-19 budget N per mask.
"""
from fractions import Fraction

import numpy as np

from .philox import PURPOSE_MASK_W, PURPOSE_MASK_X, mask_uniforms

TWO32 = 1 << 32
FIX_BITS = 16          # fixed-point fraction bits of the integer score (Z-13)
HI_SHIFT = 4           # s_up / s_down = 16 = 2^4 (Z-9)
E_MAX_W = 4            # grad_W weights fold into int8 codes: weight <= 16 (Z-17)
E_MAX_X = 24           # grad_X weights are applied in fp32: floor 2^-24 (Z-17)

MODE_BERNOULLI = 0
MODE_KEEP_POSITIVE = 1
MODE_NONE = 2


def _fixed_point(x64, h):
    """floor(x * 2^(16 + 4[h = high])) with x a float64 array (exact scaling)."""
    shift = FIX_BITS + HI_SHIFT * (1 - np.asarray(h))
    return np.floor(np.ldexp(x64, shift)).astype(np.uint64)


def weight_scores(a_sq, b_sq):
    """Integer leverage scores for the weight-gradient LSS.

    c_(h,t) = s_h ||code_(h,t)|| ||X_hat_t||; the common factor s_down s_X
    cancels in p (Z-13), so w = floor(sqrt(a_h,t b_t) 2^(16 + 4[h=up])) with
    a = sum code^2 (exact int), b = sum X_hat^2 (exact int), one IEEE sqrt.
    a_sq: [2, N] ints, b_sq: [N] ints.  Returns uint64 [2, N].
    """
    a = np.asarray(a_sq, dtype=np.int64)
    b = np.asarray(b_sq, dtype=np.int64)[None, :]
    prod = a * b
    assert prod.max(initial=0) < 2 ** 53
    h = np.arange(2)[:, None]
    return _fixed_point(np.sqrt(prod.astype(np.float64)), h)


def activation_scores(a_sq):
    """Integer leverage scores for the activation-gradient LSS:
    c_(h,t) = s_h ||code_(h,t)||  ->  w = floor(sqrt(a_h,t) 2^(16 + 4[h=up]))."""
    a = np.asarray(a_sq, dtype=np.int64)
    h = np.arange(2)[:, None]
    return _fixed_point(np.sqrt(a.astype(np.float64)), h)


def waterfill_a2(w, budget):
    """The A.2 loop, literally, in exact integers.

    p^0 = budget c / sum c; clamp at 1; rescale the unclamped items to sum to
    (budget - #clamped); repeat until nothing new exceeds 1.  With integer
    scores w, "p_i >= 1" is the exact test R w_i >= W (R = budget - |S|,
    W = sum of unclamped positive scores).

    Returns (S sorted list, R, W, rounds); if at most `budget` items are
    positive (Z-16) S is the positive set and R = W = None.
    """
    w = [int(x) for x in w]
    Z = [i for i, x in enumerate(w) if x > 0]
    if len(Z) <= budget:
        return Z, None, None, 0
    S = set()
    rounds = 0
    while True:
        rounds += 1
        R = budget - len(S)
        W = sum(w[i] for i in Z if i not in S)
        new = [i for i in Z if i not in S and R * w[i] >= W]
        if not new:
            return sorted(S), R, W, rounds
        S.update(new)
        assert rounds <= len(w) + 1            # A.2: halts after O(N) rounds


def waterfill_sorted(w, budget):
    """Second, independent algorithm (SURVEY.md §8(c) O-8'): the closed-form
    water level.  Sort descending; the clamped set is the top s* items with
    s* = min{ s : (budget - s) w_(s+1) < sum_{j > s} w_(j) }."""
    w = [int(x) for x in w]
    Z = [i for i, x in enumerate(w) if x > 0]
    if len(Z) <= budget:
        return Z, None, None
    order = sorted(Z, key=lambda i: -w[i])
    suffix = [0] * (len(order) + 1)
    for j in range(len(order) - 1, -1, -1):
        suffix[j] = suffix[j + 1] + w[order[j]]
    for s in range(len(order)):
        R = budget - s
        if R * w[order[s]] < suffix[s]:
            return sorted(order[:s]), R, suffix[s]
    raise AssertionError("unreachable: budget < #positive")


def probabilities(w, budget):
    """Exact rational p_i after A.2 (Fractions)."""
    S, R, W, _ = waterfill_a2(w, budget)
    S = set(S)
    p = []
    for i, x in enumerate(w):
        x = int(x)
        if x == 0:
            p.append(Fraction(0))
        elif i in S:
            p.append(Fraction(1))
        else:
            p.append(Fraction(R * x, W))
    return p


def dyadic_thresholds(p, e_max):
    """Two-threshold Bernoulli rule for one probability p (reading Z-17).

    e = floor(log2(1/p)); T2 = floor(p 2^32); T1 = 2 T2 - 2^(32-e).
    With a 32-bit uniform u: keep iff u < T2, weight 2^e if u < T1 else 2^(e+1).
    Then P(keep) = T2 / 2^32 and E[weight * keep] = 1 exactly.
    If e >= e_max (floor): keep iff u < 2^(32-e_max) with weight 2^e_max.
    Returns (e, T1, T2) as Python ints; p = 0 -> (0, 0, 0).
    """
    p = Fraction(p)
    if p == 0:
        return 0, 0, 0
    assert 0 < p <= 1
    e = 0
    while p * (1 << (e + 1)) <= 1:     # largest e with p 2^e <= 1
        e += 1
    if e >= e_max:
        t = TWO32 >> e_max
        return e_max, t, t
    T2 = (p.numerator * TWO32) // p.denominator
    T1 = 2 * T2 - (TWO32 >> e)
    assert 0 <= T1 <= T2 <= TWO32
    return e, T1, T2


def sample(w, budget, u, mode, e_max):
    """Masks m_i and weights for all 2N items, compacted in ascending item order
    (ids h*N + t).  The estimator is a sum over the kept
    items and does not depend on their order (a kernel may store them in any
    order; parity compares the (item, weight) pairs as sets).

    w: uint64 [2, N] scores, u: uint64 [2, N] Philox words (row h).
    Returns dict(items int64 [K], wexp int64 [K], count K, p list, e, T1, T2).
    """
    w = np.asarray(w)
    two, N = w.shape
    wf = [int(x) for x in w.reshape(-1)]          # item id i = h*N + t
    uf = [int(x) for x in np.asarray(u).reshape(-1)]
    if mode == MODE_NONE:
        items = list(range(2 * N))
        return dict(items=np.array(items, dtype=np.int64),
                    wexp=np.zeros(2 * N, dtype=np.int64), count=2 * N)
    if mode == MODE_KEEP_POSITIVE:
        items = [i for i in range(2 * N) if wf[i] > 0]
        return dict(items=np.array(items, dtype=np.int64),
                    wexp=np.zeros(len(items), dtype=np.int64), count=len(items))
    assert mode == MODE_BERNOULLI
    p = probabilities(wf, budget)
    items, wexp = [], []
    E, T1s, T2s = [], [], []
    for i in range(2 * N):
        e, T1, T2 = dyadic_thresholds(p[i], e_max)
        E.append(e); T1s.append(T1); T2s.append(T2)
        if uf[i] < T2:
            items.append(i)
            wexp.append(e if uf[i] < T1 else e + 1)
    return dict(items=np.array(items, dtype=np.int64), wexp=np.array(wexp, dtype=np.int64),
                count=len(items), p=p, e=E, T1=T1s, T2=T2s)


def sample_weight_mask(a_sq, b_sq, seed, call_id, token_offset, mode=MODE_BERNOULLI):
    """LSS mask of the weight gradient, purpose-2 Philox stream."""
    N = np.asarray(a_sq).shape[1]
    w = weight_scores(a_sq, b_sq)
    u = mask_uniforms(seed, call_id, token_offset, N, PURPOSE_MASK_W)
    out = sample(w, N, u, mode, E_MAX_W)
    out["w"] = w
    return out


def sample_activation_mask(a_sq, seed, call_id, token_offset, mode=MODE_BERNOULLI):
    """LSS mask of the activation gradient, purpose-3 stream."""
    N = np.asarray(a_sq).shape[1]
    w = activation_scores(a_sq)
    u = mask_uniforms(seed, call_id, token_offset, N, PURPOSE_MASK_X)
    out = sample(w, N, u, mode, E_MAX_X)
    out["w"] = w
    return out
