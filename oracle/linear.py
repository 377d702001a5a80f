"""HQ-MM forward and LSS-MM backward of one INT4 linear layer, composed from
the step functions.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Forward  (Eq. 3, Procedure HQ-MM):
    X_hat = <XH>_{s_X},  W_hat = <WH>_{s_W},  Y = s_X s_W X_hat W_hat^T.
Backward (Eq. 4, with LSS-MM for the "type 3" MMs):
    grad_W = s_X ((grad_Y^T X_hat) o I_W) H^T
    grad_X = (I_X o (s_W grad_Y W_hat)) H^T
    with grad_Y replaced by the sampled bit-split estimate:
      grad_W:  sum over kept items i=(h,t) of w_i s_h code_i (x) X_hat_t
      grad_X:  row t += w_i s_h code_i W_hat            (w_i = the Z-17 weight ~ m_i/p_i)
    Mask then inverse transform (reading Z-23); H symmetric so H^T = H.
"""
import numpy as np

from . import bitsplit as bs_mod
from . import lss as lss_mod
from .gemm import int_matmul_abt
from .hadamard import block_diag_hadamard
from .hq import hadamard_quant


def forward(x, w, k, s_x, s_w):
    """Procedure HQ-MM.  x [N, D], w [C, D] bf16 values; returns a dict with the
    quantized operands (the forward cache the backward reuses)
    and Y = s_X s_W acc in float64."""
    xq, x_mask, x_sq = hadamard_quant(x, k, s_x)
    wq, w_mask, w_sq = hadamard_quant(w, k, s_w)
    acc = int_matmul_abt(xq, wq)
    y = acc.astype(np.float64) * (np.float64(np.float32(s_x)) * np.float64(np.float32(s_w)))
    return dict(xq=xq, x_mask=x_mask, x_sq=x_sq, wq=wq, w_mask=w_mask, acc=acc, y=y,
                k=k, s_x=np.float32(s_x), s_w=np.float32(s_w))


def _item_rows(bs, items):
    """Code rows, token index and high/low flag of items i = h*N + t (Z-12)."""
    hi, lo = bs["hi"], bs["lo"]
    N = hi.shape[0]
    items = np.asarray(items, dtype=np.int64)
    h = items // N
    t = items % N
    codes = np.where((h == 0)[:, None], hi[t], lo[t]).astype(np.int64)
    return codes, t, h


def grad_x_product(bs, items, wexp, wq, s_w):
    """The sampled estimate of s_W grad_Y W_hat (before the mask
    and the inverse transform): row t = s_W sum_{kept i = (h, t)} w_i s_h code_i W_hat.
    Returns (G float64 [N, D], acc int64 [K, D])."""
    N, C = bs["hi"].shape
    D = wq.shape[1]
    codes, t, h = _item_rows(bs, items)
    acc = int_matmul_abt(codes, np.asarray(wq).T)                   # [K, D] exact
    s_down = np.float64(bs["s_down"])
    s_h = np.where(h == 0, 16.0 * s_down, s_down)                   # s_up = 16 s_down (Z-9)
    scale = np.float64(np.float32(s_w)) * s_h * np.ldexp(1.0, np.asarray(wexp, dtype=np.int64))
    G = np.zeros((N, D), dtype=np.float64)
    np.add.at(G, t, acc.astype(np.float64) * scale[:, None])
    return G, acc


def grad_x_from_items(bs, items, wexp, wq, x_mask, k, s_w):
    """grad_X = [I_X o (s_W sum_i w_i s_h code_i W_hat)] H."""
    D = wq.shape[1]
    G, acc = grad_x_product(bs, items, wexp, wq, s_w)
    G = G * x_mask                                                  # mask first (Z-23)
    return G @ block_diag_hadamard(D, k), acc


def grad_w_from_items(bs, items, wexp, xq, w_mask, k, s_x):
    """grad_W = s_X [(sum_i w_i s_h code_i (x) X_hat_t) o I_W] H.

    The INT GEMM folds the weights into the int8 operands (Z-17):
    A_i = 2^wexp_i code_i  (|A| <= 128),  B_i = 16^[h=up] X_hat_t  (|B| <= 112),
    acc = sum_i A_i^T B_i, grad_W = s_X s_down acc.
    """
    C = bs["hi"].shape[1]
    D = np.asarray(xq).shape[1]
    codes, t, h = _item_rows(bs, items)
    A = codes * (np.int64(1) << np.asarray(wexp, dtype=np.int64))[:, None]
    B = np.asarray(xq, dtype=np.int64)[t] * np.where(h == 0, 16, 1)[:, None]
    assert np.abs(A).max(initial=0) <= 128 and np.abs(B).max(initial=0) <= 112
    acc = int_matmul_abt(A.T, B.T)                                  # [C, D] exact
    G = acc.astype(np.float64) * (np.float64(np.float32(s_x)) * np.float64(bs["s_down"]))
    G = G * w_mask
    return G @ block_diag_hadamard(D, k), acc


def step_size_grads(x, w, fwd, bwd, n_elem_x=None, n_elem_w=None):
    """A.3 step-size gradients (readings Z-27, Z-28, Z-29) from
    the forward cache and the backward's sampled products.  Returns (gs_x, gs_w)."""
    from . import lsq_grad
    from .hq import transformed_scaled
    k = fwd["k"]
    N, D = np.asarray(x).shape
    C = np.asarray(w).shape[0]
    bs = bwd["bs"]
    mx, mw = bwd["mask_x"], bwd["mask_w"]
    Gx, _ = grad_x_product(bs, mx["items"], mx["wexp"], fwd["wq"], fwd["s_w"])
    Gw = bwd["acc_w"].astype(np.float64) * (np.float64(fwd["s_x"]) * np.float64(bs["s_down"]))
    dx = lsq_grad.delta(transformed_scaled(x, k, fwd["s_x"]))
    dw = lsq_grad.delta(transformed_scaled(w, k, fwd["s_w"]))
    gs_x = lsq_grad.step_size_grad(Gx, dx, N * D if n_elem_x is None else n_elem_x)
    gs_w = lsq_grad.step_size_grad(Gw, dw, C * D if n_elem_w is None else n_elem_w)
    return gs_x, gs_w


def backward(g, fwd, seed, call_id, token_offset=0, mode=lss_mod.MODE_BERNOULLI):
    """Procedure LSS-MM for both gradients.

    g: grad_Y [N, C] (bf16 values).  Returns dict with the BS state, both masks
    and grad_X [N, D], grad_W [C, D] in float64.
    """
    k = fwd["k"]
    bs = bs_mod.bit_split(g, seed, call_id, token_offset)
    mw = lss_mod.sample_weight_mask(bs["a_sq"], fwd["x_sq"], seed, call_id, token_offset, mode)
    mx = lss_mod.sample_activation_mask(bs["a_sq"], seed, call_id, token_offset, mode)
    dx, acc_x = grad_x_from_items(bs, mx["items"], mx["wexp"], fwd["wq"], fwd["x_mask"], k, fwd["s_w"])
    dw, acc_w = grad_w_from_items(bs, mw["items"], mw["wexp"], fwd["xq"], fwd["w_mask"], k, fwd["s_x"])
    return dict(bs=bs, mask_w=mw, mask_x=mx, dx=dx, dw=dw, acc_x=acc_x, acc_w=acc_w)


def backward_dense_reference(g, fwd):
    """Eq. 4 with the unquantized grad_Y: the target whose
    expectation the whole sampled backward must equal."""
    g = np.asarray(g, dtype=np.float64)
    k = fwd["k"]
    D = fwd["xq"].shape[1]
    H = block_diag_hadamard(D, k)
    dw = np.float64(fwd["s_x"]) * ((g.T @ fwd["xq"].astype(np.float64)) * fwd["w_mask"]) @ H
    dx = (fwd["x_mask"] * (np.float64(fwd["s_w"]) * (g @ fwd["wq"].astype(np.float64)))) @ H
    return dx, dw
