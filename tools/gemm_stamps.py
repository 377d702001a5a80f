"""GEMM phase timing from globaltimer stamps (-DI4_STAMPS=1 build via I4_LIB_OVERRIDE):
CTA 0's entry, setup, PDL wait, first TMA, first full stage, last commit, first
accumulator, epilogue done, exit; plus the earliest CTA entry / latest CTA exit.
    python tools/gemm_stamps.py bmm B N P M k | linear CFG"""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import synth  # noqa: E402
import paper_2306_11987_b200 as i4  # noqa: E402

NAMES = ["setup", "pdl_wait", "first_tma", "first_full", "last_commit", "first_acc", "epi_done", "exit", "sizes",
         "sched", "seg0"]
bf = lambda a: torch.from_numpy(synth.bf16_bits(a).view(np.int16).copy()).view(torch.bfloat16).cuda()


def read():
    buf = (ctypes.c_ulonglong * 16)()
    assert i4.lib.int4_debug_gemm_stamps(buf) == 0
    a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
    t0 = a[0]
    rel = np.concatenate([(a[1:9] - t0), (a[11:14] - t0)]) / 1e3
    span = (a[10] - a[9]) / 1e3
    first = (a[0] - a[9]) / 1e3
    return rel, span, first


def report(tag, runs):
    rel = np.median(np.array([r[0] for r in runs]), 0)
    span = np.median([r[1] for r in runs])
    first = np.median([r[2] for r in runs])
    print(tag, "CTA0 us since entry:", " ".join(f"{n}={v:.2f}" for n, v in zip(NAMES, rel)),
          f"| all-CTA span {span:.2f} us, CTA0 entry after first {first:.2f} us")


mode = sys.argv[1] if len(sys.argv) > 1 else "bmm"
if mode == "bmm":
    B, N, P, M, k = [int(v) for v in sys.argv[2:7]] if len(sys.argv) > 6 else (12, 512, 512, 64, 5)
    q = bf(np.stack([synth.activations(N, M, seed=b) for b in range(B)]))
    kk = bf(np.stack([synth.activations(P, M, seed=100 + b) for b in range(B)]))
    dt = bf(np.stack([synth.grad_output(N, P, seed=200 + b, dense=(b % 2 == 0)) for b in range(B)]))
    s_q = np.full(B, 0.3, np.float32)
    s_k = np.full(B, 0.3, np.float32)
    op = i4.Int4BMM(B, N, P, M, k)
    T = torch.empty(B, N, P, dtype=torch.bfloat16, device="cuda")
    dQ = torch.empty(B, N, M, dtype=torch.bfloat16, device="cuda")
    dK = torch.empty(B, P, M, dtype=torch.float32, device="cuda")
    fw, bw = [], []
    for it in range(8):
        torch.cuda.synchronize(); read()
        op.forward(q, kk, s_q, s_k, T); torch.cuda.synchronize(); fw.append(read())
        op.backward(dt, dQ, dK, synth.PHILOX_SEED, 0); torch.cuda.synchronize(); bw.append(read())
    report(f"bmm{B}x{N}x{P} fwd", fw[3:])
    report(f"bmm{B}x{N}x{P} bwd", bw[3:])
else:
    name = sys.argv[2] if len(sys.argv) > 2 else "cfg3_bert_large_ffn_up"
    cfg = synth.CONFIGS[name]
    N, D, C, k = cfg["N"], cfg["D"], cfg["C"], cfg["k"]
    X, W, G = bf(synth.activations(N, D)), bf(synth.weights(C, D)), bf(synth.grad_output(N, C))
    L = i4.Int4Linear(N, D, C, k)
    Y = torch.empty(N, C, dtype=torch.bfloat16, device="cuda")
    dX = torch.empty(N, D, dtype=torch.bfloat16, device="cuda")
    dW = torch.empty(C, D, dtype=torch.float32, device="cuda")
    fw, bw = [], []
    for it in range(8):
        torch.cuda.synchronize(); read()
        L.forward(X, W, 0.05, 0.01, Y); torch.cuda.synchronize(); fw.append(read())
        L.backward(G, dX, dW, synth.PHILOX_SEED, 0); torch.cuda.synchronize(); bw.append(read())
    report(f"{name} fwd", fw[3:])
    report(f"{name} bwd", bw[3:])
