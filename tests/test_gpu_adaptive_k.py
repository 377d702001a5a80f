"""GPU parity of the NEXT row (f3): adaptive Hadamard size (A.5) against the
oracle, through the C ABI."""
import numpy as np
import pytest
import torch

import synth
from oracle.lsq_grad import cold_start_step
from oracle import adaptive_k as o_ak
from oracle import hadamard as o_had

from gpu_helpers import to_bf16_cuda

pytestmark = pytest.mark.gpu


def p():
    import paper_2306_11987_b200 as mod
    return mod


def _run(x, w, s_x, s_w, k_min, k_max):
    xb, wb = to_bf16_cuda(x), to_bf16_cuda(w)
    k_best = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    mse = torch.zeros(16, dtype=torch.float64, device="cuda")
    ws = torch.zeros(p().hq_select_k_workspace_size(), dtype=torch.uint8, device="cuda")
    p().hq_select_k(xb, wb, s_x, s_w, k_min, k_max, k_best, mse, ws)
    torch.cuda.synchronize()
    assert not ws.any()                                   # scratch left zeroed
    return int(k_best.item()), mse.cpu().numpy(), xb.float().cpu().numpy(), wb.float().cpu().numpy()


@pytest.mark.parametrize("N,D,C,k_min,k_max", [(512, 256, 128, 0, 7), (200, 128, 64, 0, 5), (96, 1024, 192, 2, 6)])
def test_select_k_parity(N, D, C, k_min, k_max):
    x = synth.activations(N, D, seed=N)
    w = synth.weights(C, D, seed=N)
    s_x, s_w = cold_start_step(x), cold_start_step(w)
    k_best, mse, xv, wv = _run(x, w, s_x, s_w, k_min, k_max)
    ks = list(range(k_min, k_max + 1))
    ref_k, table = o_ak.select_k(xv, wv, s_x, s_w, ks)
    for k in ks:
        for got, ref in ((mse[2 * k], table[k][0]), (mse[2 * k + 1], table[k][1])):
            # codes may differ from the oracle's at near-ties (reading Z-7); the
            # reconstruction and the error are fp64 on both sides
            assert abs(got - ref) <= 1e-5 * ref + 1e-30, (k, got, ref)
    prods = {k: table[k][0] * table[k][1] for k in ks}
    runner_up = sorted(prods.values())[1] if len(ks) > 1 else np.inf
    if runner_up > prods[ref_k] * (1 + 1e-4):            # a clear winner: must agree
        assert k_best == ref_k


def test_select_k_exact_input_and_determinism():
    rng = np.random.default_rng(7)
    D, k0 = 128, 4
    s = np.float32(0.5)
    H = o_had.block_diag_hadamard(D, k0)
    x = (np.float64(s) * rng.integers(-7, 8, (64, D)) @ H.T).astype(np.float32)
    w = (np.float64(s) * rng.integers(-7, 8, (32, D)) @ H.T).astype(np.float32)
    k_best, mse, _, _ = _run(x, w, s, s, 0, 7)
    assert k_best == k0 and mse[2 * k0] < 1e-20 and mse[2 * k0 + 1] < 1e-20   # exact up to H's 1/sqrt(2) products
    k2, mse2, _, _ = _run(x, w, s, s, 0, 7)
    assert k2 == k_best and np.array_equal(mse, mse2)


def test_select_k_argument_errors():
    x = to_bf16_cuda(synth.activations(64, 96))
    w = to_bf16_cuda(synth.weights(32, 96))
    k_best = torch.zeros(1, dtype=torch.int32, device="cuda")
    mse = torch.zeros(16, dtype=torch.float64, device="cuda")
    ws = torch.zeros(p().hq_select_k_workspace_size(), dtype=torch.uint8, device="cuda")
    with pytest.raises(p().I4Error):                      # 96 is not a multiple of 64
        p().hq_select_k(x, w, 0.1, 0.1, 0, 3, k_best, mse, ws)
    x = to_bf16_cuda(synth.activations(64, 192))
    w = to_bf16_cuda(synth.weights(32, 192))
    with pytest.raises(p().I4Error):                      # 192 % 2^7 != 0
        p().hq_select_k(x, w, 0.1, 0.1, 0, 7, k_best, mse, ws)
