"""Experiment: overhead of launch-trace events inside the captured graph."""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from oracle.lsq_grad import cold_start_step  # tools only (test infrastructure), paper_2306_11987_b200 as i4

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2_bert_base_ffn1"]
N, D, C, k = cfg["N"], cfg["D"], cfg["C"], cfg["k"]
def up(a): return torch.from_numpy(synth.bf16_bits(a).view(np.int16).copy()).view(torch.bfloat16).cuda()
X, W, G = up(synth.activations(N, D)), up(synth.weights(C, D)), up(synth.grad_output(N, C))
s_x, s_w = cold_start_step(synth.activations(N, D)), cold_start_step(synth.weights(C, D))
layer = i4.Int4Linear(N, D, C, k)
Y = torch.empty(N, C, dtype=torch.bfloat16, device="cuda")
dX = torch.empty(N, D, device="cuda"); dW = torch.empty(C, D, device="cuda")
fw = torch.empty(256 << 20, dtype=torch.uint8, device="cuda"); fr = torch.ones(32 << 20, dtype=torch.int64, device="cuda")
def flush(): fw.zero_(); torch.sum(fr)
def body():
    layer.forward(X, W, s_x, s_w, Y)
    layer.backward(G, dX, dW, synth.PHILOX_SEED, 0, 0, 0)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    body(); body()
torch.cuda.synchronize()
def time_graph(g, n=30, do_flush=True):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for i in range(n + 3):
        if do_flush: flush()
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        if i >= 3: ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)
g1 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g1): body()
print("graph no trace, flushed: %.1f us" % time_graph(g1))
print("graph no trace, warm L2: %.1f us" % time_graph(g1, do_flush=False))
events = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(40)]
tr = i4.LaunchTrace(events)
g2 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g2):
    with tr: body()
print("graph with trace, flushed: %.1f us" % time_graph(g2))
# single-kernel graphs for each stage, measured separately (no trace)
def stage_graph(fn):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g): fn()
    return g
print("memset dX alone: %.1f us" % time_graph(stage_graph(lambda: dX.zero_())))
print("fwd only: %.1f us" % time_graph(stage_graph(lambda: layer.forward(X, W, s_x, s_w, Y))))
# eager (no graph) with trace
flush(); torch.cuda.synchronize()
with tr: body()
torch.cuda.synchronize()
print("eager trace:", [(n, round(ms * 1e3, 1)) for n, ms in tr.durations_ms()])
