"""Microbenchmark: our tcgen05 int8 GEMM (int32 out) vs cuBLASLt int8 (torch._int_mm)
and cuBLAS bf16 on the same shapes.  Graph-replayed, CUDA events, L2 warm."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2306_11987_b200 as i4

def tgraph(fn, n=50):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(n):
        a.record(); g.replay(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return statistics.median(ts) * 1e3

shapes = [(4096, 4096, 8192), (8192, 8192, 2048), (4096, 3072, 768), (8192, 4096, 1024), (16384, 16384, 4096)]
for M, N, K in shapes:
    A = torch.randint(-8, 8, (M, K), dtype=torch.int8, device="cuda")
    B = torch.randint(-8, 8, (N, K), dtype=torch.int8, device="cuda")
    C = torch.empty(M, N, dtype=torch.int32, device="cuda")
    ops = 2.0 * M * N * K
    t_ours = tgraph(lambda: i4.int4_gemm_s8s8s32(A, B, C))
    try:
        t_lt = tgraph(lambda: torch._int_mm(A, B.t()))
    except Exception as e:
        t_lt = float("nan")
    Ab, Bb = A.bfloat16(), B.bfloat16()
    t_bf = tgraph(lambda: torch.matmul(Ab, Bb.t()))
    print(f"{M}x{N}x{K}: ours {t_ours:8.1f} us {ops/t_ours/1e6:7.0f} TOPS | cublasLt int8 {t_lt:8.1f} us {ops/t_lt/1e6:7.0f} TOPS | bf16 {t_bf:8.1f} us {ops/t_bf/1e6:7.0f} TFLOPS")
