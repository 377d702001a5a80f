"""GPU parity of the NEXT row (f2): BMM in attention (A.1) against the oracle,
through the C ABI.  Per batch: T from the exact integer product of the GPU codes,
dQ / dK from the oracle's per-batch LSS-MM on the same codes (reading Z-31)."""
import numpy as np
import pytest
import torch

import synth
from oracle.lsq_grad import cold_start_step
from oracle import bmm as o_bmm
from oracle import gemm as o_gemm
from oracle import lss as o_lss

from gpu_helpers import code_mismatch, rel_frob, to_bf16_cuda, unpack_bits

pytestmark = pytest.mark.gpu

FROB_TOL = 1e-5


def p():
    import paper_2306_11987_b200 as mod
    return mod


@pytest.mark.parametrize("mode", [o_lss.MODE_BERNOULLI, o_lss.MODE_NONE])
@pytest.mark.parametrize("B,N,P,M,k", [(3, 128, 128, 64, 4), (2, 200, 192, 128, 5), (6, 64, 128, 64, 3)])
def test_bmm_parity(B, N, P, M, k, mode):
    q = np.stack([synth.activations(N, M, seed=10 + b) for b in range(B)])
    kk = np.stack([synth.activations(P, M, seed=20 + b) for b in range(B)])
    dt = np.stack([synth.grad_output(N, P, seed=30 + b, dense=(b % 2 == 0)) for b in range(B)])
    s_q = np.array([cold_start_step(q[b]) for b in range(B)], dtype=np.float32)
    s_k = np.array([cold_start_step(kk[b]) for b in range(B)], dtype=np.float32)
    op = p().Int4BMM(B, N, P, M, k)
    T = torch.empty(B, N, P, dtype=torch.float32, device="cuda")
    op.forward(to_bf16_cuda(q), to_bf16_cuda(kk), s_q, s_k, T)
    dQ = torch.empty(B, N, M, dtype=torch.float32, device="cuda")
    dK = torch.empty(B, P, M, dtype=torch.float32, device="cuda")
    op.backward(to_bf16_cuda(dt), dQ, dK, synth.PHILOX_SEED, call_id=4, mode=mode)
    torch.cuda.synchronize()

    fwds_o, _ = o_bmm.forward(q, kk, k, s_q, s_k)
    qq, kq = op.qq.cpu().numpy(), op.kq.cpu().numpy()
    fwds = []
    for b in range(B):
        for g, o in ((qq[b], fwds_o[b]["xq"]), (kq[b], fwds_o[b]["wq"])):
            nbad, maxdiff = code_mismatch(g, o)
            assert maxdiff <= 1 and nbad <= 1e-6 * o.size
        acc = o_gemm.int_matmul_abt(qq[b], kq[b])
        t_ref = acc.astype(np.float64) * (np.float64(s_q[b]) * np.float64(s_k[b]))
        assert rel_frob(T[b].cpu().numpy(), t_ref) < FROB_TOL
        fwds.append(dict(xq=qq[b], wq=kq[b], x_mask=unpack_bits(op.q_mask[b], M), w_mask=unpack_bits(op.k_mask[b], M),
                         x_sq=op.q_sqnorm[b].cpu().numpy().astype(np.int64), k=k, s_x=s_q[b], s_w=s_k[b]))
    dq_ref, dk_ref, _ = o_bmm.backward(dt, fwds, synth.PHILOX_SEED, 4, mode)
    got_q, got_k = dQ.cpu().numpy(), dK.cpu().numpy()
    for b in range(B):
        assert rel_frob(got_q[b], dq_ref[b]) < FROB_TOL
        assert rel_frob(got_k[b], dk_ref[b]) < FROB_TOL


def test_bmm_bad_shape():
    op = p().Int4BMM(1, 64, 96, 64, 4)                    # P = 96 is not a multiple of 64
    T = torch.empty(1, 64, 96, dtype=torch.float32, device="cuda")
    with pytest.raises(p().I4Error):
        op.forward(to_bf16_cuda(synth.activations(64, 64)[None]), to_bf16_cuda(synth.activations(96, 64)[None]),
                   np.ones(1, np.float32), np.ones(1, np.float32), T)


def test_bmm_chains_bitwise_independent_of_stream_count(monkeypatch):
    """Batches run as up to 16 concurrent chains (own plan, workspace slice, stream):
    the results are byte-identical to one chain on the caller's stream."""
    B, N, P, M, k = 7, 128, 128, 64, 4
    q = np.stack([synth.activations(N, M, seed=50 + b) for b in range(B)])
    kk = np.stack([synth.activations(P, M, seed=60 + b) for b in range(B)])
    dt = np.stack([synth.grad_output(N, P, seed=70 + b, dense=(b % 3 == 0)) for b in range(B)])
    s_q = np.array([cold_start_step(q[b]) for b in range(B)], dtype=np.float32)
    s_k = np.array([cold_start_step(kk[b]) for b in range(B)], dtype=np.float32)
    outs = []
    for streams in ("1", "16"):
        monkeypatch.setenv("I4_BMM_STREAMS", streams)
        op = p().Int4BMM(B, N, P, M, k)
        T = torch.empty(B, N, P, dtype=torch.float32, device="cuda")
        dQ = torch.empty(B, N, M, dtype=torch.bfloat16, device="cuda")
        dK = torch.empty(B, P, M, dtype=torch.float32, device="cuda")
        op.forward(to_bf16_cuda(q), to_bf16_cuda(kk), s_q, s_k, T)
        op.backward(to_bf16_cuda(dt), dQ, dK, synth.PHILOX_SEED, call_id=2)
        torch.cuda.synchronize()
        outs.append([t.view(torch.uint8).cpu().numpy() if t.dtype == torch.bfloat16 else t.cpu().numpy().view(np.uint32)
                     for t in (T, dQ, dK)])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
