"""Forward GEMM device time per config (CUPTI; the library is the default or I4_LIB_OVERRIDE)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
import synth
import paper_2306_11987_b200 as i4

for name in sys.argv[1:]:
    c = synth.CONFIGS[name]
    N, D, C, k = c["N"], c["D"], c["C"], c["k"]
    up = lambda a: torch.from_numpy(synth.bf16_bits(a).view(np.int16).copy()).view(torch.bfloat16).cuda()
    X, W = up(synth.activations(N, D)), up(synth.weights(C, D))
    L = i4.Int4Linear(N, D, C, k)
    Y = torch.empty(N, C, dtype=torch.bfloat16, device="cuda")
    for _ in range(3): L.forward(X, W, 0.05, 0.01, Y)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(20): L.forward(X, W, 0.05, 0.01, Y)
        torch.cuda.synchronize()
    ts = [e.device_time_total for e in prof.events() if "gemm_i8" in e.name]
    lib = os.path.basename(os.environ.get("I4_LIB_OVERRIDE", "default"))
    print(f"{lib:12s} {name:28s} gemm_fwd {np.median(ts):6.1f} us  {2*N*C*D/np.median(ts)/1e6:7.0f} TOPS")
