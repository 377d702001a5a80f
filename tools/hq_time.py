"""hadamard_quant (X and W in one launch) device time per config (CUPTI, L2 flushed
between forwards); the library is the default or I4_LIB_OVERRIDE."""
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
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3): L.forward(X, W, 0.05, 0.01, Y)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(10):
            flush.zero_()
            L.forward(X, W, 0.05, 0.01, Y)
        torch.cuda.synchronize()
    ts = [e.device_time_total for e in prof.events() if "hadamard_quant" in e.name]
    gb = ((N + C) * D * (2 + 1 + 1 / 8) + 4 * N) / 1e9
    t = float(np.median(ts))
    print(f"{os.path.basename(os.environ.get('I4_LIB_OVERRIDE', 'default')):12s} {name:28s} hq {t:6.1f} us  {gb / (t * 1e-6):7.0f} GB/s")
