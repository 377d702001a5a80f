import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_2306_11987_b200 as i4
for (N, D, C, k, reps) in [(4096, 1024, 320, 5, 30), (2048, 512, 192, 5, 30), (4096, 1024, 1024, 7, 10)]:
    up = lambda a: torch.from_numpy(synth.bf16_bits(a).view(np.int16).copy()).view(torch.bfloat16).cuda()
    X, W = up(synth.activations(N, D)), up(synth.weights(C, D))
    G = up(synth.grad_output(N, C))
    L = i4.Int4Linear(N, D, C, k)
    Y = torch.empty(N, C, dtype=torch.bfloat16, device="cuda")
    dX = torch.empty(N, D, dtype=torch.bfloat16, device="cuda"); dW = torch.empty(C, D, dtype=torch.float32, device="cuda")
    for r in range(reps):
        L.forward(X, W, 0.05, 0.01, Y)
        if k == 7: L.backward(G, dX, dW, 1, call_id=r)
    torch.cuda.synchronize()
    print("ok", N, D, C, k, flush=True)
