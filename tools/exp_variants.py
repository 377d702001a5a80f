"""Time grad_split in several compile variants of the library (CUPTI kernel durations)."""
import ctypes, glob, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_2306_11987_b200 as i4
from torch.profiler import profile, ProfilerActivity

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3_bert_large_ffn_up"]
N, C = cfg["N"], cfg["C"]
G = torch.from_numpy(synth.bf16_bits(synth.grad_output(N, C)).view(np.int16).copy()).view(torch.bfloat16).cuda()
L = i4.Int4Linear(N, cfg["D"], C, cfg["k"])
xsq = torch.ones(N, dtype=torch.int32, device="cuda")
libs = [i4.LIB_PATH] + sorted(glob.glob(os.path.join(os.path.dirname(i4.LIB_PATH), "..", "build_variants", "*.so")))
for path in libs:
    lib = ctypes.CDLL(path)
    fn = lib.bitsplit_lss
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32,
                   ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(i4.I4LssPlan), ctypes.c_void_p]
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    def call():
        st = fn(ctypes.c_void_p(G.data_ptr()), N, C, ctypes.c_void_p(xsq.data_ptr()), 1, 0, 0, 0, ctypes.byref(L.plan), stream)
        assert st == 0, st
    for _ in range(3): call()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(10): call()
        torch.cuda.synchronize()
    ts = [e.device_time_total for e in prof.events() if "grad_split" in e.name]
    print(f"{os.path.basename(path):20s} grad_split {np.median(ts):7.1f} us  (n={len(ts)})")
