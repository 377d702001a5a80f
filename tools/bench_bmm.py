"""Step time of the attention BMM path (A.1; T = BMM(Q, K^T) fwd + bwd) vs cuBLAS
bf16 batched matmuls (T = Q K^T, dQ = dT K, dK = dT^T Q), CUDA-graph replays with
an L2 flush before each timed step.  Prints one JSON line.

    python tools/bench_bmm.py [B N P M k]
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2306_11987_b200 as i4  # noqa: E402


def main():
    B, N, P, M, k = [int(v) for v in sys.argv[1:6]] if len(sys.argv) > 5 else (12, 512, 512, 64, 5)
    steps, warmup = 20, 3
    bf = lambda a: torch.from_numpy(synth.bf16_bits(a).view(np.int16).copy()).view(torch.bfloat16).cuda()
    q = bf(np.stack([synth.activations(N, M, seed=b) for b in range(B)]))
    kk = bf(np.stack([synth.activations(P, M, seed=100 + b) for b in range(B)]))
    dt = bf(np.stack([synth.grad_output(N, P, seed=200 + b, dense=(b % 2 == 0)) for b in range(B)]))
    s_q = np.full(B, 0.3, np.float32)
    s_k = np.full(B, 0.3, np.float32)
    op = i4.Int4BMM(B, N, P, M, k)
    T = torch.empty(B, N, P, dtype=torch.bfloat16, device="cuda")
    dQ = torch.empty(B, N, M, dtype=torch.bfloat16, device="cuda")
    dK = torch.empty(B, P, M, dtype=torch.float32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def ours():
        op.forward(q, kk, s_q, s_k, T)
        op.backward(dt, dQ, dK, synth.PHILOX_SEED, 0)

    Tb = torch.empty(B, N, P, dtype=torch.bfloat16, device="cuda")
    dQb = torch.empty(B, N, M, dtype=torch.bfloat16, device="cuda")
    dKb = torch.empty(B, P, M, dtype=torch.bfloat16, device="cuda")

    def blas():
        torch.bmm(q, kk.transpose(1, 2), out=Tb)
        torch.bmm(dt, kk, out=dQb)
        torch.bmm(dt.transpose(1, 2), q, out=dKb)

    def time_graph(fn):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn(); fn()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = []
        for i in range(warmup + steps):
            flush.zero_()
            e0.record(); g.replay(); e1.record()
            torch.cuda.synchronize()
            if i >= warmup:
                ms.append(e0.elapsed_time(e1))
        return statistics.mean(ms)

    t_ours = time_graph(ours)
    t_fwd = time_graph(lambda: op.forward(q, kk, s_q, s_k, T))
    t_blas = time_graph(blas)
    work = 6.0 * B * N * P * M
    print(json.dumps({"metric": "attention BMM fwd+bwd (A.1) effective TOPS", "config": dict(B=B, N=N, P=P, M=M, k=k),
                      "ms_per_step": t_ours, "fwd_ms": t_fwd, "value": work / (t_ours * 1e-3) / 1e12, "unit": "TOPS",
                      "bf16_cublas_ms_per_step": t_blas, "speedup_vs_bf16_cublas": t_blas / t_ours,
                      "launches_per_step": 7 + (B - 1) // 128,
                      "note": "batch dimension inside the kernels: step table, hadamard_quant, batched GEMM "
                      "(3-D tensor maps); grad_split (per-batch amax), sampler (one cluster per mask and "
                      "batch), compact, one GEMM launch over every batch's grad_Q / grad_K tiles"}))


if __name__ == "__main__":
    main()
