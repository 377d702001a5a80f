"""One bench step of a workload (default: the cfg5 stack) between
cudaProfilerStart/Stop, for ncu launch lists of exactly one step:
    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \\
        --csv --log-file gpurun_out/x.csv python tools/stack_step.py [config]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

args = bench.parse(["--config", sys.argv[1] if len(sys.argv) > 1 else bench.DEFAULT_CONFIG])
lins, n_layers = bench.workload(args.config)
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
st = bench.Stack(lins, n_layers, args, dev, 0, 1)
for _ in range(2):                                  # warm: lazy library state, caches
    st.fwd_body()
    for layer in reversed(range(n_layers)):
        st.bwd_body(layer)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
st.fwd_body()
for layer in reversed(range(n_layers)):
    st.bwd_body(layer)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("one step:", len(lins), "linears")
