"""Run one GEMM shape a few times (for ncu). args: M N K a_mn b_mn split"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2306_11987_b200 as i4
M, N, K, a_mn, b_mn, split = [int(x) for x in sys.argv[1:7]]
A = torch.randint(-8, 8, (K, M) if a_mn else (M, K), dtype=torch.int8, device="cuda")
B = torch.randint(-8, 8, (K, N) if b_mn else (N, K), dtype=torch.int8, device="cuda")
C = torch.empty(M, N, dtype=torch.int32, device="cuda")
ws = torch.zeros(i4.int4_gemm_workspace_size(), dtype=torch.uint8, device="cuda") if split else None
for _ in range(3):
    i4.int4_gemm_s8s8s32(A, B, C, bool(a_mn), bool(b_mn), ws=ws)
torch.cuda.synchronize()
