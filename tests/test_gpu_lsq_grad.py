"""GPU parity of the NEXT row (f1): LSQ step-size gradients (A.3) and the
cold-start step (A.4) against the oracle, through the C ABI."""
import numpy as np
import pytest
import torch

import synth
from oracle.lsq_grad import cold_start_step
from oracle import hq as o_hq
from oracle import linear as o_lin
from oracle import lsq_grad as o_lg
from oracle import lss as o_lss

from gpu_helpers import to_bf16_cuda, unpack_bits

pytestmark = pytest.mark.gpu


def p():
    import paper_2306_11987_b200 as mod
    return mod


def _case(N, D, C, k, mode, dense=False, seed=0, call_id=3, token_offset=0):
    x = synth.activations(N, D, seed=seed)
    w = synth.weights(C, D, seed=seed)
    g = synth.grad_output(N, C, seed=seed, dense=dense)
    s_x, s_w = cold_start_step(x), cold_start_step(w)
    layer = p().Int4Linear(N, D, C, k, step_grads=True)
    Y = torch.empty(N, C, dtype=torch.float32, device="cuda")
    layer.forward(to_bf16_cuda(x), to_bf16_cuda(w), s_x, s_w, Y)
    dX = torch.empty(N, D, dtype=torch.float32, device="cuda")
    dW = torch.empty(C, D, dtype=torch.float32, device="cuda")
    layer.backward(to_bf16_cuda(g), dX, dW, synth.PHILOX_SEED, call_id, token_offset, mode)
    torch.cuda.synchronize()
    return x, w, g, s_x, s_w, layer, dX, dW


def _oracle(x, w, g, s_x, s_w, k, layer, mode, call_id=3, token_offset=0):
    fwd = dict(xq=layer.xq.cpu().numpy(), wq=layer.wq.cpu().numpy(),
               x_mask=unpack_bits(layer.x_mask, layer.D), w_mask=unpack_bits(layer.w_mask, layer.D),
               x_sq=layer.x_sqnorm.cpu().numpy().astype(np.int64), k=k,
               s_x=np.float32(s_x), s_w=np.float32(s_w))
    bwd = o_lin.backward(g, fwd, synth.PHILOX_SEED, call_id, token_offset, mode)
    gs_x, gs_w = o_lin.step_size_grads(x, w, fwd, bwd)
    # magnitude scale of the sums, for the fp32 chunk-sum tolerance
    Gx, _ = o_lin.grad_x_product(bwd["bs"], bwd["mask_x"]["items"], bwd["mask_x"]["wexp"], fwd["wq"], fwd["s_w"])
    Gw = bwd["acc_w"].astype(np.float64) * (np.float64(fwd["s_x"]) * np.float64(bwd["bs"]["s_down"]))
    dx = o_lg.delta(o_hq.transformed_scaled(x, k, s_x))
    dw = o_lg.delta(o_hq.transformed_scaled(w, k, s_w))
    ax = o_lg.grad_scale(x.size) * np.abs(Gx * dx).sum()
    aw = o_lg.grad_scale(w.size) * np.abs(Gw * dw).sum()
    return gs_x, gs_w, ax, aw


def _tol(abs_sum, ref):
    # fp32 products and 32-term fp32 chunk sums (<= 32 * 2^-24 relative to the
    # absolute sum), fp64 beyond, one final fp32 rounding of the result
    return 64 * 2.0 ** -24 * abs_sum + 2.0 ** -23 * abs(ref) + 1e-30


def test_deltas_are_exact():
    N, D, C, k = 200, 256, 128, 5
    x, w, g, s_x, s_w, layer, dX, dW = _case(N, D, C, k, o_lss.MODE_BERNOULLI)
    for t, s, got in ((x, s_x, layer.x_delta), (w, s_w, layer.w_delta)):
        ref = o_lg.delta(o_hq.transformed_scaled(t, k, s))
        got = got.cpu().numpy().astype(np.float64)
        # delta = code - v is exact in fp32 on both sides; v itself differs by the
        # rounding of the staged fp32 FWHT vs the oracle's single rounding of the
        # exact transform (a few ulp of |v| <= 7.5, reading Z-7); where that moves
        # a code across a tie, delta differs by one level
        diff = np.abs(got - ref)
        assert np.mean(diff > 8 * 2.0 ** -21) <= 1e-5
        assert diff.max() <= 1.0 + 1e-6


@pytest.mark.parametrize("mode", [o_lss.MODE_BERNOULLI, o_lss.MODE_KEEP_POSITIVE, o_lss.MODE_NONE])
@pytest.mark.parametrize("N,D,C,k,dense", [(128, 64, 64, 4, False), (1000, 256, 192, 5, True),
                                           (640, 192, 320, 3, False), (256, 128, 256, 6, True)])
def test_step_size_grads_parity(N, D, C, k, dense, mode):
    x, w, g, s_x, s_w, layer, dX, dW = _case(N, D, C, k, mode, dense=dense)
    got = layer.grad_s().cpu().numpy().astype(np.float64)
    gs_x, gs_w, ax, aw = _oracle(x, w, g, s_x, s_w, k, layer, mode)
    assert abs(got[0] - gs_x) <= _tol(ax, gs_x), (got[0], gs_x, ax)
    assert abs(got[1] - gs_w) <= _tol(aw, gs_w), (got[1], gs_w, aw)
    assert abs(gs_x) > 0 and abs(gs_w) > 0


def test_step_grads_leave_dx_dw_unchanged_and_are_deterministic():
    N, D, C, k = 512, 256, 512, 5
    x, w, g, s_x, s_w, layer, dX, dW = _case(N, D, C, k, o_lss.MODE_BERNOULLI)
    first = layer.grad_s().clone()
    plain = p().Int4Linear(N, D, C, k)
    Y = torch.empty(N, C, dtype=torch.float32, device="cuda")
    plain.forward(to_bf16_cuda(x), to_bf16_cuda(w), s_x, s_w, Y)
    dX2 = torch.empty_like(dX)
    dW2 = torch.empty_like(dW)
    plain.backward(to_bf16_cuda(g), dX2, dW2, synth.PHILOX_SEED, 3, 0, o_lss.MODE_BERNOULLI)
    layer.backward(to_bf16_cuda(g), dX, dW, synth.PHILOX_SEED, 3, 0, o_lss.MODE_BERNOULLI)
    torch.cuda.synchronize()
    assert torch.equal(dX, dX2) and torch.equal(dW, dW2)
    assert torch.equal(first, layer.grad_s())


def test_step_grads_need_the_deltas():
    N, D, C, k = 128, 64, 64, 4
    layer = p().Int4Linear(N, D, C, k, step_grads=True)
    x = synth.activations(N, D)
    w = synth.weights(C, D)
    Y = torch.empty(N, C, dtype=torch.float32, device="cuda")
    layer.forward(to_bf16_cuda(x), to_bf16_cuda(w), 0.1, 0.01, Y)
    layer.cache.x_delta = None
    dX = torch.empty(N, D, dtype=torch.float32, device="cuda")
    dW = torch.empty(C, D, dtype=torch.float32, device="cuda")
    with pytest.raises(p().I4Error):
        layer.backward(to_bf16_cuda(synth.grad_output(N, C)), dX, dW, 1)


@pytest.mark.parametrize("n", [1, 7, 4096, 12345, 4096 * 768, 50432 * 3072 // 8])
def test_cold_start_step(n):
    rng = np.random.default_rng(n)
    x = (rng.standard_normal(n) * 0.7).astype(np.float32)
    xb = to_bf16_cuda(x)
    xv = xb.float().cpu().numpy()                      # the bf16 values the kernel reads
    ref = o_lg.cold_start_step(xv)
    step = torch.zeros(1, dtype=torch.float32, device="cuda")
    ws = torch.zeros(p().lsq_cold_start_workspace_size(), dtype=torch.uint8, device="cuda")
    for _ in range(2):                                 # twice: the ticket must come back zeroed
        p().lsq_cold_start_step(xb, step, ws)
        torch.cuda.synchronize()
        got = step.cpu().numpy()[0]
        assert abs(int(np.float32(got).view(np.int32)) - int(np.float32(ref).view(np.int32))) <= 1
    assert not ws.any()
