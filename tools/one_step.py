"""One layer's forward + backward a few times (for ncu captures of single kernels):
    python tools/one_step.py cfg3_bert_large_ffn_up [sparse|dense] [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2306_11987_b200 as i4  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3_bert_large_ffn_up"]
dense = len(sys.argv) > 2 and sys.argv[2] == "dense"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
N, D, C, k = cfg["N"], cfg["D"], cfg["C"], cfg["k"]


def up(a):
    return torch.from_numpy(synth.bf16_bits(a).view(np.int16).copy()).view(torch.bfloat16).cuda()


X, W, G = up(synth.activations(N, D)), up(synth.weights(C, D)), up(synth.grad_output(N, C, dense=dense))
s_x, s_w = i4.cold_start_step(X), i4.cold_start_step(W)
layer = i4.Int4Linear(N, D, C, k)
Y = torch.empty(N, C, dtype=torch.bfloat16, device="cuda")
dX = torch.empty(N, D, dtype=torch.bfloat16, device="cuda")
dW = torch.empty(C, D, dtype=torch.float32, device="cuda")
i4.int4_set_pdl(False)
for _ in range(reps):
    layer.forward(X, W, s_x, s_w, Y)
    layer.backward(G, dX, dW, synth.PHILOX_SEED, call_id=0)
torch.cuda.synchronize()
print("kept", layer.counts().cpu().tolist(), "dense", layer.dense_flags().cpu().tolist())
