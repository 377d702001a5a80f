"""One attention BMM fwd+bwd step, repeated (for ncu launch lists).
    python tools/bmm_step.py [B N P M k] [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import synth  # noqa: E402
import paper_2306_11987_b200 as i4  # noqa: E402

B, N, P, M, k = [int(v) for v in sys.argv[1:6]] if len(sys.argv) > 5 else (12, 512, 512, 64, 5)
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
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
for _ in range(reps):
    op.forward(q, kk, s_q, s_k, T)
    op.backward(dt, dQ, dK, synth.PHILOX_SEED, 0)
    torch.cuda.synchronize()
print("counts", op.ws_view(2).cpu().numpy().tolist())
