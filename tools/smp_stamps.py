"""lss_sampler phase timing from globaltimer stamps (CTA rank 0 of the grad_W
mask): start, scores summed, each A.2 round, Bernoulli done, compaction done, end."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from oracle.lsq_grad import cold_start_step  # tools only (test infrastructure)
import paper_2306_11987_b200 as i4

for arg in sys.argv[1:] or ["cfg2_bert_base_ffn1"]:
    name, _, kind = arg.partition(":")
    cfg = synth.CONFIGS[name]
    N, D, C, k = cfg["N"], cfg["D"], cfg["C"], cfg["k"]
    up = lambda a: torch.from_numpy(synth.bf16_bits(a).view(np.int16).copy()).view(torch.bfloat16).cuda()
    X, W, G = up(synth.activations(N, D)), up(synth.weights(C, D)), up(synth.grad_output(N, C, dense=(kind == "dense")))
    s_x, s_w = cold_start_step(synth.activations(N, D)), cold_start_step(synth.weights(C, D))
    L = i4.Int4Linear(N, D, C, k)
    Y = torch.empty(N, C, dtype=torch.bfloat16, device="cuda")
    L.forward(X, W, s_x, s_w, Y)
    xsq = L.x_sqnorm
    i4.lib.int4_debug_sampler_stamps(None, 1)
    fn = i4.lib.bitsplit_lss
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    res, rnd = [], []
    for it in range(6):
        st = fn(ctypes.c_void_p(G.data_ptr()), N, C, ctypes.c_void_p(xsq.data_ptr()), 1, 0, 0, 0,
                ctypes.byref(L.plan), stream)
        assert st == 0
        torch.cuda.synchronize()
        buf = (ctypes.c_ulonglong * 32)()
        i4.lib.int4_debug_sampler_stamps(buf, 1)
        a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
        n = int(a[31])
        res.append(np.diff(a[:n]) / 1e3)
        rnd.append(np.diff(a[24:30]) / 1e3)
    i4.lib.int4_debug_sampler_stamps(None, 0)
    print(arg, "stamps", n, "intervals us:", np.round(np.median(np.array(res[2:]), 0), 2),
          "| round 2: items, warp sums, send, wait, final sums:", np.round(np.median(np.array(rnd[2:]), 0), 3))
