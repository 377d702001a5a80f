"""INT32 GEMM timing for a few shapes (tile-width experiments): M N K a_mn b_mn ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
import paper_2306_11987_b200 as i4
shapes = [(8192, 1024, 1024, 0, 0), (8192, 1152, 1024, 0, 0), (8192, 896, 1024, 0, 0), (8192, 1024, 4096, 0, 1),
          (8192, 1024, 4096, 0, 0), (8192, 1152, 4096, 0, 0)]
for (M, N, K, a_mn, b_mn) in shapes:
    A = torch.randint(-8, 8, (K, M) if a_mn else (M, K), dtype=torch.int8, device="cuda")
    B = torch.randint(-8, 8, (K, N) if b_mn else (N, K), dtype=torch.int8, device="cuda")
    C = torch.empty(M, N, dtype=torch.int32, device="cuda")
    for _ in range(3): i4.int4_gemm_s8s8s32(A, B, C, bool(a_mn), bool(b_mn))
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(10): i4.int4_gemm_s8s8s32(A, B, C, bool(a_mn), bool(b_mn))
        torch.cuda.synchronize()
    ts = [e.device_time_total for e in prof.events() if "gemm_i8" in e.name]
    t = float(np.median(ts))
    print(f"{M}x{N}x{K} a_mn={a_mn} b_mn={b_mn}: {t:7.1f} us  {2*M*N*K/t/1e6:6.0f} TOPS")
