"""Per-kernel CUPTI times of one fwd + bwd step for the library and its compile
variants (build_variants/*.so), each in its own process (I4_LIB_OVERRIDE).

    python tools/exp_bwd.py cfg4_vit_b16_ffn_down
"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(cfg_name):
    import numpy as np
    import torch
    from torch.profiler import ProfilerActivity, profile

    import synth
    import paper_2306_11987_b200 as i4
    from bench import short_kernel_name
    cfg = synth.CONFIGS[cfg_name]
    N, D, C, k = cfg["N"], cfg["D"], cfg["C"], cfg["k"]
    rng = np.random.default_rng(1)
    bf = lambda a: torch.from_numpy(synth.bf16_bits(a).view(np.int16).copy()).view(torch.bfloat16).cuda()
    X, W, G = bf(synth.activations(N, D)), bf(synth.weights(C, D)), bf(synth.grad_output(N, C))
    i4.int4_set_pdl(False)                    # per-kernel durations without early-launch waits
    L = i4.Int4Linear(N, D, C, k)
    Y = torch.empty(N, C, dtype=torch.bfloat16, device="cuda")
    dX = torch.empty(N, D, dtype=torch.bfloat16, device="cuda")
    dW = torch.empty(C, D, dtype=torch.float32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step():
        L.forward(X, W, 0.05, 0.004, Y)
        L.backward(G, dX, dW, seed=7)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(10):
            flush.zero_()
            step()
        torch.cuda.synchronize()
    per = {}
    for e in prof.events():
        nm = short_kernel_name(e.name)
        if nm:
            per.setdefault(nm, []).append(e.device_time_total)
    lib = os.path.basename(os.environ.get("I4_LIB_OVERRIDE", "default"))
    print(f"{lib:22s} " + "  ".join(f"{k} {np.median(v):6.1f}" for k, v in per.items() if not k.startswith("memset")))


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4_vit_b16_ffn_down"
    if os.environ.get("I4_EXP_CHILD"):
        return child(cfg)
    libs = [None] + sorted(glob.glob(os.path.join(ROOT, "build_variants", "*.so")))
    for lib in libs:
        env = dict(os.environ, I4_EXP_CHILD="1")
        if lib:
            env["I4_LIB_OVERRIDE"] = lib
        subprocess.run([sys.executable, __file__, cfg], env=env, timeout=300)


if __name__ == "__main__":
    main()
