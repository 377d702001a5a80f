"""grad_split phase timing from per-CTA globaltimer stamps (a -DI4_STAMPS=1 build,
loaded through I4_LIB_OVERRIDE): prints, in us from the earliest CTA start, the min / median / max
over CTAs of: phase 1 done, barrier passed, amax known, phase 2 done."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_2306_11987_b200 as i4

for name in sys.argv[1:] or ["cfg2_bert_base_ffn1"]:
    cfg = synth.CONFIGS[name]
    N, C = cfg["N"], cfg["C"]
    G = torch.from_numpy(synth.bf16_bits(synth.grad_output(N, C)).view(np.int16).copy()).view(torch.bfloat16).cuda()
    L = i4.Int4Linear(N, cfg["D"], C, cfg["k"])
    xsq = torch.ones(N, dtype=torch.int32, device="cuda")
    fn = i4.lib.bitsplit_lss
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rows = []
    for it in range(8):
        flush.zero_()
        st = fn(ctypes.c_void_p(G.data_ptr()), N, C, ctypes.c_void_p(xsq.data_ptr()), 1, 0, 0, 0,
                ctypes.byref(L.plan), stream)
        assert st == 0, st
        torch.cuda.synchronize()
        buf = (ctypes.c_ulonglong * (5 * 2048))()
        n = i4.lib.int4_debug_grad_split_stamps(buf, 2048)
        a = np.frombuffer(buf, dtype=np.uint64).reshape(5, n).astype(np.int64)
        used = a[0] > 0
        a = a[:, used]
        if it >= 3:
            rows.append((a - a[0].min()) / 1e3)
    print(f"== {name}: {rows[0].shape[1]} CTAs")
    labels = ["start", "phase1 done", "barrier passed", "amax known", "phase2 done"]
    for r, lab in enumerate(labels):
        v = np.array([x[r] for x in rows])
        print(f"  {lab:15s} min {np.median(v.min(1)):6.2f}  med {np.median(np.median(v, 1)):6.2f}  max {np.median(v.max(1)):6.2f} us")
