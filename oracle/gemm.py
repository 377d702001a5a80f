"""Exact integer matrix products.  TEST INFRASTRUCTURE ONLY.

PAPER.md:154 (HQ-MM step 3, "Multiply the two INT4 matrices"), :328 and
:370-371 (the INT4 MMs of LSS-MM).  The accumulator is INT32;
reading Z-21 requires every |partial sum| < 2^31, which is asserted.

The product is computed with one float64 library matmul.  For integer inputs
every partial sum is an integer of magnitude < 2^53, so the float64 result is
exact and independent of summation order; `int_matmul_bruteforce` is the
triple loop the pins compare it with.
"""
import numpy as np

INT32_LIMIT = 2 ** 31


def int_matmul_abt(a, b):
    """acc[m, n] = sum_k a[m, k] * b[n, k]  (A . B^T), exact, returned as int64."""
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape[1] == b.shape[1]
    if a.size and b.size:
        amax = int(np.abs(a.astype(np.int64)).max())
        bmax = int(np.abs(b.astype(np.int64)).max())
        if amax * bmax * a.shape[1] >= INT32_LIMIT:       # cheap bound failed: exact one
            bound = np.abs(a.astype(np.float64)) @ np.abs(b.astype(np.float64)).T
            assert bound.max() < 2.0 ** 53
            if bound.max() >= INT32_LIMIT:
                raise OverflowError("INT32 accumulator bound exceeded (Z-21)")
    acc = a.astype(np.float64) @ b.astype(np.float64).T
    return acc.astype(np.int64)


def int_matmul_bruteforce(a, b):
    """The same product as a literal Python triple loop (tiny shapes only)."""
    a = [[int(v) for v in row] for row in np.asarray(a)]
    b = [[int(v) for v in row] for row in np.asarray(b)]
    out = np.zeros((len(a), len(b)), dtype=np.int64)
    for m in range(len(a)):
        for n in range(len(b)):
            s = 0
            for k in range(len(a[m])):
                s += a[m][k] * b[n][k]
            out[m, n] = s
    return out
