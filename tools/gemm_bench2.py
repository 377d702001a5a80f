"""GEMM microbenchmark on the operator's GEMM shapes (int32 epilogue), with and
without split-K workspace, vs cuBLASLt int8 and bf16 on equivalent shapes."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2306_11987_b200 as i4

def tgraph(fn, n=30):
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

cases = [  # name, M, N, K, a_mn, b_mn
    ("fwd cfg2", 4096, 3072, 768, False, False),
    ("dgrad cfg2", 4096, 768, 3072, False, True),
    ("wgrad cfg2", 3072, 768, 4096, True, True),
    ("fwd cfg3up", 8192, 4096, 1024, False, False),
    ("dgrad cfg3up", 8192, 1024, 4096, False, True),
    ("wgrad cfg3up", 4096, 1024, 8192, True, True),
]
for name, M, N, K, a_mn, b_mn in cases:
    A = torch.randint(-8, 8, (K, M) if a_mn else (M, K), dtype=torch.int8, device="cuda")
    B = torch.randint(-8, 8, (K, N) if b_mn else (N, K), dtype=torch.int8, device="cuda")
    C = torch.empty(M, N, dtype=torch.int32, device="cuda")
    ops = 2.0 * M * N * K
    t0 = tgraph(lambda: i4.int4_gemm_s8s8s32(A, B, C, a_mn, b_mn))
    t1 = tgraph(lambda: i4.int4_gemm_s8s8s32(A, B, C, a_mn, b_mn))
    Ak = (A.t() if a_mn else A).contiguous(); Bk = (B.t() if b_mn else B).contiguous()
    t_lt = tgraph(lambda: torch._int_mm(Ak, Bk.t()))
    Ab, Bb = Ak.bfloat16(), Bk.bfloat16()
    t_bf = tgraph(lambda: torch.matmul(Ab, Bb.t()))
    print(f"{name:13s} {M}x{N}x{K}: ours {t0:6.1f} us ({ops/t0/1e6:5.0f}) split {t1:6.1f} us ({ops/t1/1e6:5.0f}) | "
          f"cublasLt-i8 {t_lt:6.1f} ({ops/t_lt/1e6:5.0f}) | bf16 {t_bf:6.1f} ({ops/t_bf/1e6:5.0f}) TOPS")
