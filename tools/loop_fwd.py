"""Back-to-back forwards of one shape (hang check): python tools/loop_fwd.py N D C reps pdl"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_2306_11987_b200 as i4
N, D, C, reps, pdl = [int(v) for v in sys.argv[1:6]]
i4.int4_set_pdl(bool(pdl))
up = lambda a: torch.from_numpy(synth.bf16_bits(a).view(np.int16).copy()).view(torch.bfloat16).cuda()
X, W = up(synth.activations(N, D)), up(synth.weights(C, D))
L = i4.Int4Linear(N, D, C, 5)
Y = torch.empty(N, C, dtype=torch.bfloat16, device="cuda")
for r in range(reps):
    L.forward(X, W, 0.05, 0.01, Y)
    if r % int(os.environ.get("SYNC_EVERY", "5")) == 0:
        torch.cuda.synchronize(); print("rep", r, flush=True)
torch.cuda.synchronize()
print("ok", flush=True)
