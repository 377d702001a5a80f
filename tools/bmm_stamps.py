"""lss_sampler phase timing (globaltimer stamps, -DI4_STAMPS=1 build via I4_LIB_OVERRIDE)
inside the batched BMM backward: batch 0 (dense dT: binding budget), grad_W mask."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes  # noqa: E402
import numpy as np  # noqa: E402
import torch  # noqa: E402
import synth  # noqa: E402
import paper_2306_11987_b200 as i4  # noqa: E402

B, N, P, M, k = [int(v) for v in sys.argv[1:6]] if len(sys.argv) > 5 else (12, 512, 512, 64, 5)
bf = lambda a: torch.from_numpy(synth.bf16_bits(a).view(np.int16).copy()).view(torch.bfloat16).cuda()
q = bf(np.stack([synth.activations(N, M, seed=b) for b in range(B)]))
kk = bf(np.stack([synth.activations(P, M, seed=100 + b) for b in range(B)]))
dt = bf(np.stack([synth.grad_output(N, P, seed=200 + b, dense=(b % 2 == 0)) for b in range(B)]))
s_q = np.full(B, 0.3, np.float32)
s_k = np.full(B, 0.3, np.float32)
op = i4.Int4BMM(B, N, P, M, k)
T = torch.empty(B, N, P, dtype=torch.bfloat16, device="cuda")
dQ = torch.empty(B, N, M, dtype=torch.bfloat16, device="cuda")
dK = torch.empty(B, P, M, dtype=torch.float32, device="cuda")
op.forward(q, kk, s_q, s_k, T)
i4.lib.int4_debug_sampler_stamps(None, 1)
res = []
for it in range(6):
    op.backward(dt, dQ, dK, synth.PHILOX_SEED, 0)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 32)()
    i4.lib.int4_debug_sampler_stamps(buf, 1)
    a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
    n = int(a[31])
    res.append(np.diff(a[:n]) / 1e3)
i4.lib.int4_debug_sampler_stamps(None, 0)
print("bmm", B, N, P, "stamps", n, "intervals us:", np.round(np.median(np.array(res[2:]), 0), 2),
      "total", round(float(np.median([r.sum() for r in res[2:]])), 2))
