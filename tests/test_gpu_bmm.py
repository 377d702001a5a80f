"""GPU parity of the NEXT row (f2): BMM in attention (A.1) against the oracle,
through the C ABI, with the batch dimension inside the kernels (3 forward + 4
backward launches for all B batches).  Per batch: T from the exact integer
product of the GPU codes; the SR codes, per-batch s_down and both sampled lists
bit-exact against the oracle's LSS-MM of that batch (token_offset = b N, its own
amax, reading Z-31); dQ / dK against the oracle on the same codes."""
import numpy as np
import pytest
import torch

import synth
from oracle.lsq_grad import cold_start_step
from oracle import bmm as o_bmm
from oracle import gemm as o_gemm
from oracle import lss as o_lss

from gpu_helpers import code_mismatch, rel_frob, same_item_set, to_bf16_cuda, unpack_bits

pytestmark = pytest.mark.gpu

FROB_TOL = 1e-5


def p():
    import paper_2306_11987_b200 as mod
    return mod


def _inputs(B, N, P, M, seed0=10, dense_every=2):
    q = np.stack([synth.activations(N, M, seed=seed0 + b) for b in range(B)])
    kk = np.stack([synth.activations(P, M, seed=seed0 + 100 + b) for b in range(B)])
    dt = np.stack([synth.grad_output(N, P, seed=seed0 + 200 + b, dense=(b % dense_every == 0)) for b in range(B)])
    # per-batch magnitude spread (exact power-of-two scales of bf16 values): every batch
    # has its own amax, so a shared amax would change the codes
    dt = dt * (2.0 ** (np.arange(B) % 3 - 1))[:, None, None]
    s_q = np.array([cold_start_step(q[b]) for b in range(B)], dtype=np.float32)
    s_k = np.array([cold_start_step(kk[b]) for b in range(B)], dtype=np.float32)
    return q, kk, dt, s_q, s_k


def _run(B, N, P, M, k, q, kk, dt, s_q, s_k, mode, call_id=4, dq_dtype=torch.float32, t_dtype=torch.float32):
    op = p().Int4BMM(B, N, P, M, k)
    T = torch.empty(B, N, P, dtype=t_dtype, device="cuda")
    op.forward(to_bf16_cuda(q), to_bf16_cuda(kk), s_q, s_k, T)
    dQ = torch.empty(B, N, M, dtype=dq_dtype, device="cuda")
    dK = torch.empty(B, P, M, dtype=torch.float32, device="cuda")
    op.backward(to_bf16_cuda(dt), dQ, dK, synth.PHILOX_SEED, call_id=call_id, mode=mode)
    torch.cuda.synchronize()
    return op, T, dQ, dK


def _check_against_oracle(op, T, dQ, dK, B, N, P, M, k, q, kk, dt, s_q, s_k, mode, call_id=4, tol=FROB_TOL):
    fwds_o, _ = o_bmm.forward(q, kk, k, s_q, s_k)
    qq, kq = op.qq.cpu().numpy(), op.kq.cpu().numpy()
    fwds = []
    for b in range(B):
        for g, o in ((qq[b], fwds_o[b]["xq"]), (kq[b], fwds_o[b]["wq"])):
            nbad, maxdiff = code_mismatch(g, o)
            assert maxdiff <= 1 and nbad <= 1e-6 * o.size
        acc = o_gemm.int_matmul_abt(qq[b], kq[b])
        t_ref = acc.astype(np.float64) * (np.float64(s_q[b]) * np.float64(s_k[b]))
        assert rel_frob(T[b].float().cpu().numpy(), t_ref) < (tol if T.dtype == torch.float32 else 8e-3)
        fwds.append(dict(xq=qq[b], wq=kq[b], x_mask=unpack_bits(op.q_mask[b], M), w_mask=unpack_bits(op.k_mask[b], M),
                         x_sq=op.q_sqnorm[b].cpu().numpy().astype(np.int64), k=k, s_x=s_q[b], s_w=s_k[b]))
    dq_ref, dk_ref, outs = o_bmm.backward(dt, fwds, synth.PHILOX_SEED, call_id, mode)
    # per-batch intermediates, bit-exact: SR codes, s_down, both kept lists
    q8 = op.ws_view(7).cpu().numpy()
    s_down = op.ws_view(0).cpu().numpy()
    counts = op.ws_view(2).cpu().numpy()
    iw, ew = op.ws_view(3).cpu().numpy(), op.ws_view(4).cpu().numpy()
    ix, ex = op.ws_view(5).cpu().numpy(), op.ws_view(6).cpu().numpy()
    assert not q8[B * N].any()                                  # the pad row
    for b in range(B):
        o = outs[b]
        assert np.array_equal(q8[b * N:(b + 1) * N].astype(np.int64), o["bs"]["q"])
        assert s_down[b] == o["bs"]["s_down"]
        cw, cx = int(counts[0, b]), int(counts[1, b])
        assert (cw, cx) == (o["mask_w"]["count"], o["mask_x"]["count"])
        assert same_item_set(iw[b, :cw], ew[b, :cw], o["mask_w"])
        assert same_item_set(ix[b, :cx], ex[b, :cx], o["mask_x"])
        assert (iw[b, cw:(cw + 127) // 128 * 128] == 2 * N).all()   # sentinel padding
    got_q, got_k = dQ.float().cpu().numpy(), dK.cpu().numpy()
    qtol = tol if dQ.dtype == torch.float32 else 8e-3
    for b in range(B):
        assert rel_frob(got_q[b], dq_ref[b]) < qtol
        assert rel_frob(got_k[b], dk_ref[b]) < tol


@pytest.mark.parametrize("mode", [o_lss.MODE_BERNOULLI, o_lss.MODE_NONE])
@pytest.mark.parametrize("B,N,P,M,k", [(3, 128, 128, 64, 4), (2, 200, 192, 128, 5), (6, 64, 128, 64, 3),
                                       (5, 256, 256, 64, 6), (4, 96, 320, 128, 7)])
def test_bmm_parity(B, N, P, M, k, mode):
    q, kk, dt, s_q, s_k = _inputs(B, N, P, M)
    op, T, dQ, dK = _run(B, N, P, M, k, q, kk, dt, s_q, s_k, mode)
    _check_against_oracle(op, T, dQ, dK, B, N, P, M, k, q, kk, dt, s_q, s_k, mode)


@pytest.mark.parametrize("B,N,P,M,k", [(12, 512, 512, 64, 5), (48, 128, 128, 64, 5)])
def test_bmm_parity_bench_shapes(B, N, P, M, k):
    """The two BASELINE attention shapes bench.py / tools/bench_bmm.py time, in full."""
    q, kk, dt, s_q, s_k = _inputs(B, N, P, M, seed0=300, dense_every=3)
    op, T, dQ, dK = _run(B, N, P, M, k, q, kk, dt, s_q, s_k, o_lss.MODE_BERNOULLI, call_id=9)
    _check_against_oracle(op, T, dQ, dK, B, N, P, M, k, q, kk, dt, s_q, s_k, o_lss.MODE_BERNOULLI, call_id=9)


def test_bmm_bf16_outputs():
    B, N, P, M, k = 3, 128, 256, 64, 5
    q, kk, dt, s_q, s_k = _inputs(B, N, P, M, seed0=40)
    op, T, dQ, dK = _run(B, N, P, M, k, q, kk, dt, s_q, s_k, o_lss.MODE_BERNOULLI, dq_dtype=torch.bfloat16,
                         t_dtype=torch.bfloat16)
    _check_against_oracle(op, T, dQ, dK, B, N, P, M, k, q, kk, dt, s_q, s_k, o_lss.MODE_BERNOULLI)


def test_bmm_zero_batch_and_status():
    """One all-zero batch among normal ones: its codes, lists and gradients are zero,
    bit 1 of the status word is set, the other batches are unaffected."""
    B, N, P, M, k = 4, 128, 128, 64, 4
    q, kk, dt, s_q, s_k = _inputs(B, N, P, M, seed0=60)
    dt[2] = 0.0
    op, T, dQ, dK = _run(B, N, P, M, k, q, kk, dt, s_q, s_k, o_lss.MODE_BERNOULLI)
    assert op.status() & p().STATUS_ZERO_GRAD
    assert not dQ[2].any() and not dK[2].any()
    _check_against_oracle(op, T, dQ, dK, B, N, P, M, k, q, kk, dt, s_q, s_k, o_lss.MODE_BERNOULLI)


def test_bmm_deterministic_and_graph_capturable():
    """Two eager calls and one CUDA-graph replay give byte-identical results (the
    workspace's amax words are left zero by every call)."""
    B, N, P, M, k = 7, 128, 128, 64, 4
    q, kk, dt, s_q, s_k = _inputs(B, N, P, M, seed0=50, dense_every=3)
    op = p().Int4BMM(B, N, P, M, k)
    Qd, Kd, dTd = to_bf16_cuda(q), to_bf16_cuda(kk), to_bf16_cuda(dt)
    T = torch.empty(B, N, P, dtype=torch.float32, device="cuda")
    dQ = torch.empty(B, N, M, dtype=torch.bfloat16, device="cuda")
    dK = torch.empty(B, P, M, dtype=torch.float32, device="cuda")

    def step(stream=None):
        op.forward(Qd, Kd, s_q, s_k, T, stream)
        op.backward(dTd, dQ, dK, synth.PHILOX_SEED, call_id=2, stream=stream)

    outs = []
    for _ in range(2):
        step()
        torch.cuda.synchronize()
        outs.append([t.view(torch.uint8).clone() for t in (T, dQ, dK)])
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        step(s)                                    # warm-up on the capture stream
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step(s)
    for t in (T, dQ, dK):
        t.zero_()
    g.replay()
    torch.cuda.synchronize()
    outs.append([t.view(torch.uint8).clone() for t in (T, dQ, dK)])
    for a, b, c in zip(*outs):
        assert torch.equal(a, b) and torch.equal(a, c)
    assert not op.ws[:256].any()                   # per-batch amax words returned to zero


def test_bmm_bad_shape():
    op = p().Int4BMM(1, 64, 96, 64, 4)                    # P = 96 is not a multiple of 64
    T = torch.empty(1, 64, 96, dtype=torch.float32, device="cuda")
    with pytest.raises(p().I4Error):
        op.forward(to_bf16_cuda(synth.activations(64, 64)[None]), to_bf16_cuda(synth.activations(96, 64)[None]),
                   np.ones(1, np.float32), np.ones(1, np.float32), T)


@pytest.mark.parametrize("B", [200, 2100])
def test_bmm_many_batches_sampled(B):
    """B > 128 (the step table needs its own launch) and B > 2048 (the backward runs in
    chunks of 2048 batches with token offsets b0 N): every batch's T, dQ, dK against the
    oracle on a sample of batches spread over the chunks."""
    N, P, M, k = 64, 64, 64, 3
    q, kk, dt, s_q, s_k = _inputs(B, N, P, M, seed0=1000, dense_every=2)
    op, T, dQ, dK = _run(B, N, P, M, k, q, kk, dt, s_q, s_k, o_lss.MODE_BERNOULLI, call_id=11)
    assert torch.allclose(op.steps[:, 5].cpu(), torch.from_numpy(s_q)) and torch.allclose(op.steps[:, 6].cpu(), torch.from_numpy(s_k))
    qq, kq = op.qq.cpu().numpy(), op.kq.cpu().numpy()
    sample = sorted({0, 1, 127, 128, B // 2, 2047 % B, min(2048, B - 1), B - 1})
    for b in sample:
        fo = o_bmm.forward(q[b:b + 1], kk[b:b + 1], k, s_q[b:b + 1], s_k[b:b + 1])[0][0]
        for g, o in ((qq[b], fo["xq"]), (kq[b], fo["wq"])):
            nbad, maxdiff = code_mismatch(g, o)
            assert maxdiff <= 1 and nbad <= 1e-6 * o.size
        t_ref = o_gemm.int_matmul_abt(qq[b], kq[b]).astype(np.float64) * (np.float64(s_q[b]) * np.float64(s_k[b]))
        assert rel_frob(T[b].cpu().numpy(), t_ref) < FROB_TOL
        fwd = dict(xq=qq[b], wq=kq[b], x_mask=unpack_bits(op.q_mask[b], M), w_mask=unpack_bits(op.k_mask[b], M),
                   x_sq=op.q_sqnorm[b].cpu().numpy().astype(np.int64), k=k, s_x=s_q[b], s_w=s_k[b])
        from oracle import linear as o_lin
        o = o_lin.backward(dt[b], fwd, synth.PHILOX_SEED, 11, token_offset=b * N, mode=o_lss.MODE_BERNOULLI)
        assert rel_frob(dQ[b].cpu().numpy(), o["dx"]) < FROB_TOL
        assert rel_frob(dK[b].cpu().numpy(), o["dw"]) < FROB_TOL
