#!/usr/bin/env python
"""Benchmark of the B200 INT4 linear operator (arXiv 2306.11987, HQ-MM + LSS-MM).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg5_bert_large_stack] [--grad sparse|dense] [--mode bernoulli]

Workload (default): BASELINE.json configs[4], the 24-layer BERT-large linear
stack (QKV 1024->3072, FFN-up 1024->4096, FFN-down 4096->1024 per layer) at
8192 tokens per GPU -- the largest configuration, and the one the paper's
data-parallel throughput setting uses.  `--config` also
takes every single-linear BASELINE shape (synth.CONFIGS) and the cfgT stack.

One step = one training pass of the whole hot path over one batch of
synthetic input:
  forward  : every linear in layer order: hadamard_quant(X, W), INT GEMM + dequant
  backward : every linear in reverse order: amax + bit split, LSS sampler (both
             masks), compaction, grad_X GEMM, grad_W GEMM
  N > 1    : + the NCCL all-reduce of each layer's grad_W bucket, launched
             asynchronously right after that layer's backward so it overlaps
             the next (lower) layer's backward (token-sharded data parallelism,
             SURVEY.md §8(e)); the step ends when every all-reduce is done.
The forward and each layer's backward are CUDA graphs (captured once, replayed).

Metric (BASELINE.json): INT4 linear fwd+bwd speedup vs BF16 cuBLAS; eff. TOPS
and % of INT8 peak.  `value` = effective TOPS = sum over linears of 6 N C D /
t_step, summed over ranks (whole job).  The cuBLAS BF16 stack (Y = X W^T,
dX = dY W, dW = dY^T X, bf16 in / out, its bf16 grad_W all-reduced the same
way) is timed beside it; `per_linear` reports the BERT-large shapes alone in
both grad_Y regimes with the realized kept counts.

`--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (127.0.0.1 rendezvous).  `--impl
reference` times the CPU oracle (test infrastructure) on a bounded sample of
the same workload on the host cores.  `--dry-run` exercises the rank
launcher, sharding and the overlapped all-reduce plumbing on CPU (gloo), with
no operator compute (tests/test_bench_dry.py).
"""
import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "INT4 linear fwd+bwd speedup vs BF16 cuBLAS; eff. TOPS and % of INT8 peak"
UNIT = "TOPS"
DEFAULT_CONFIG = "cfg5_bert_large_stack"   # BASELINE.json configs[4] (largest; the DP throughput setting)
INT8_OVER_BF16 = 2.0                       # nominal dense INT8 : BF16 tensor ratio on B200 (4.5 : 2.25 P)
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
ORACLE_REF_TOKENS = 256                    # tokens per linear per --impl reference step (bounded sample)
MODES = {"bernoulli": 0, "keep_positive": 1, "none": 2}
PER_LINEAR = ["cfg3_bert_large_qkv", "cfg3_bert_large_ffn_up", "cfg3_bert_large_ffn_down"]
GROUP = "gemm_i8_dgrad||gemm_i8_wgrad"     # the library's trace name of the concurrent pair


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return dict(hbm_gbs=float(d["hbm_gbs"]), bf16_tflops=float(d["bf16_tflops"]),
                    bf16_tflops_sustained=float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                    source="measured (MEASURED_PEAKS.json)")
    return dict(hbm_gbs=FALLBACK_PEAKS["hbm_gbs"], bf16_tflops=FALLBACK_PEAKS["bf16_tflops"],
                bf16_tflops_sustained=FALLBACK_PEAKS["bf16_tflops"], source="fallback (B200_PROFILING.md)")


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(synth.CONFIGS) + sorted(synth.STACKS))
    ap.add_argument("--grad", choices=["sparse", "dense"], default="sparse")
    ap.add_argument("--mode", choices=list(MODES), default="bernoulli")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--layer-graphs", action="store_true",
                    help="N > 1 step structure (per-layer graphs + async all-reduce) on a one-rank NCCL group")
    ap.add_argument("--no-per-linear", action="store_true")
    ap.add_argument("--no-gate", action="store_true", help="skip the pre-timing oracle parity gate")
    ap.add_argument("--dry-run", action="store_true", help="CPU/gloo plumbing check, no operator compute")
    ap.add_argument("--wgrad-reduce", choices=["nccl", "nvls"], default="nccl",
                    help="N > 1: grad_W all-reduce by NCCL per layer (overlapped), or inside the grad_W GEMM "
                         "epilogue through an NVLS multicast buffer (SURVEY.md §8(f4); opt-in, unmeasured)")
    return ap.parse_args(argv)


# ---------------------------------------------------------------------------- workload
def workload(config):
    """[(name, N, D, C, k, layer, call_id)] in forward order, and the layer count."""
    if config in synth.STACKS:
        st = synth.STACKS[config]
        out = []
        for layer in range(st["layers"]):
            for j, (nm, D, C) in enumerate(st["linears"]):
                out.append((nm, st["N"], D, C, st["k"], layer, 4 * layer + j))   # call_id = 4 layer + linear
        return out, st["layers"]
    c = synth.CONFIGS[config]
    return [(config, c["N"], c["D"], c["C"], c["k"], 0, 0)], 1


def work_ops(lins):
    return sum(6.0 * N * C * D for (_, N, D, C, *_r) in lins)


def workload_config(args, lins, world):
    N = lins[0][1]
    shapes = sorted({(nm, D, C) for (nm, _, D, C, *_r) in lins})
    stack = args.config in synth.STACKS
    desc = (f"{args.config}: {len(lins)} INT4 linears ({len(lins) // len(shapes)} layers x "
            + ", ".join(f"{nm} {D}->{C}" for nm, D, C in shapes) + f"), {N} tokens per GPU, fwd+bwd") if stack else \
        f"{args.config}: {N} tokens x {lins[0][2]}->{lins[0][3]} INT4 linear fwd+bwd"
    return {"workload": desc, "tokens_per_gpu": N, "global_tokens": N * world, "k": lins[0][4],
            "linears_per_step": len(lins), "grad_y": args.grad, "lss_mode": args.mode,
            "parallelism": f"dp{world} (token-sharded)",
            "l2": "a step's inputs (GBs for the stack) exceed the 126 MB L2; L2 is also flushed before every timed "
                  "step (256 MiB write + 256 MiB read of another buffer)",
            "graph": ("the whole step captured as one CUDA graph" if world == 1 else
                      "forward and each layer's backward captured as CUDA graphs (the all-reduces between them)")
                     + ", kernels chained by programmatic dependent launch; per-kernel breakdown from PDL-off captures"}


# ---------------------------------------------------------------------------- launcher
def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def maybe_spawn(args, argv):
    """--gpus N > 1 outside torchrun: re-launch this script with N ranks."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + list(argv)
    return subprocess.call(cmd)


def env_world():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ---------------------------------------------------------------------------- oracle arms
def oracle_linear_step(N, D, C, k, grad, mode):
    """One oracle fwd+bwd of one linear on N tokens; returns seconds."""
    from oracle import linear
    from oracle.lsq_grad import cold_start_step
    x = synth.activations(N, D)
    w = synth.weights(C, D)
    g = synth.grad_output(N, C, dense=(grad == "dense"))
    s_x, s_w = cold_start_step(x), cold_start_step(w)
    t0 = time.perf_counter()
    f = linear.forward(x, w, k, s_x, s_w)
    linear.backward(g, f, synth.PHILOX_SEED, 0, 0, MODES[mode])
    return time.perf_counter() - t0


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count() or 1


def oracle_sample(lins, n_tokens, grad, mode):
    """The oracle on every distinct linear shape of the workload at n_tokens
    tokens: (ops done, seconds, shapes)."""
    shapes = sorted({(D, C, k) for (_, _, D, C, k, *_r) in lins})
    ops, secs = 0.0, 0.0
    for (D, C, k) in shapes:
        secs += oracle_linear_step(n_tokens, D, C, k, grad, mode)
        ops += 6.0 * n_tokens * C * D
    return ops, secs, shapes


def cpu_baseline(lins, grad, mode, budget_s=20.0):
    """The oracle as it stands, on the host cores, on a bounded sample: one
    layer's distinct linear shapes at up to 1024 tokens (~10-30 s of CPU work)."""
    n = min(1024, lins[0][1])
    ops, secs, shapes = oracle_sample(lins, n, grad, mode)
    reps = 1
    while secs < 0.5 * budget_s and reps < 4:
        o2, s2, _ = oracle_sample(lins, n, grad, mode)
        ops, secs, reps = ops + o2, secs + s2, reps + 1
    return {"value": ops / secs / 1e12, "unit": UNIT, "cores": blas_threads(), "kind": "oracle",
            "sample": f"{reps} x one fwd+bwd of each distinct linear shape "
                      f"({', '.join(f'{D}->{C}' for D, C, _ in shapes)}) at {n} tokens ({secs:.1f} s in total); "
                      f"numpy/OpenBLAS fp64 + Python loops; TOPS = 6 n C D / t"}


def run_reference(args):
    rank, world, _ = env_world()
    if rank != 0:
        return 0
    lins, _ = workload(args.config)
    n = min(ORACLE_REF_TOKENS, lins[0][1])
    for _ in range(args.warmup):
        oracle_sample(lins, n, args.grad, args.mode)
    times, ops, shapes = [], 0.0, []
    for _ in range(args.steps):
        o, t, shapes = oracle_sample(lins, n, args.grad, args.mode)
        times.append(t)
        ops = o
    t = statistics.mean(times)
    value = ops / t / 1e12
    sample = (f"one fwd+bwd of each distinct linear shape ({', '.join(f'{D}->{C}' for D, C, _ in shapes)}) at "
              f"{n} of {lins[0][1]} tokens per step")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, lins, 1),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": blas_threads(), "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv:
            self.t.join()
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            except Exception:
                pass

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------- algorithmic work
def algorithmic_work(name, N, D, C, kx, kw, dense, moved=None):
    """(kind, amount) per launch: kind 'ops' (tensor) or 'bytes' (HBM); the
    per-unit figures are stated in DESIGN.md §6.  dense = (grad_W mask, grad_X
    mask) deterministic: that GEMM ran over the N token rows of Q (reading Z-32)
    and compact moved none of its operands.  moved: compact's actual bytes."""
    dw, dx = dense
    rx = N if dx else kx                      # rows of the grad_X GEMM
    rw = N if dw else kw                      # K of the grad_W GEMM
    if name == "gemm_i8_fwd":
        return "ops", 2.0 * N * C * D
    if name == "gemm_i8_dgrad":
        return "ops", 2.0 * rx * C * D
    if name == "gemm_i8_wgrad":
        return "ops", 2.0 * rw * C * D
    if name in (GROUP, "gemm_i8_bwd"):       # grad_X and grad_W GEMMs in one launch
        return "ops", 2.0 * (rx + rw) * C * D
    if name == "hadamard_quant":              # X and W: read bf16, write int8 codes + 1-bit mask (+ int32 norm)
        return "bytes", (N + C) * D * (2 + 1 + 1 / 8) + 4 * N
    if name == "grad_split":                  # read bf16 grad_Y once (the amax pass's re-read is an
        return "bytes", N * C * (2 + 1) + 8 * N  # implementation cost), write the 8-bit code plane Q + norms
    if name == "compact":
        return "bytes", float(moved or 0.0)
    if name == "lss_sampler":
        return "latency", 0.0
    return "bytes", 0.0


def compact_bytes(layer, N, D, C, kx, kw, form):
    """Bytes compact actually moves (read + write), from the last backward's lists:
    a sampled grad_X mask reads its tokens' Q rows once (a token's second half hits
    L2), writes K_X half-rows of A_X and zeroes the bf16 grad_X rows of untouched
    tokens; a sampled grad_W mask reads the Q and X_hat rows of its tokens and
    writes K_W rows of A_W (C) and B_W (D).  Operand form 2: only the correction rows
    (grad_W) and the sampled tokens' item rows (grad_X), read + written."""
    fw, fx = form
    dw, dx = fw != 0, fx != 0
    b = 0.0
    if fw == 2 or fx == 2:
        cw, cx = [int(v) for v in layer.form2_counts().cpu().numpy()]
        if fw == 2:
            b += 2.0 * cw * (C + D)
        if fx == 2:
            b += 2.0 * cx * C
    if not dx:
        toks = np.unique(layer.items_x[:kx].cpu().numpy() % N).size
        b += toks * C + kx * C + (N - toks) * D * 2
    if not dw:
        toks = np.unique(layer.items_w[:kw].cpu().numpy() % N).size
        b += toks * (C + D) + kw * (C + D)
    return b


# ---------------------------------------------------------------------------- our arm
class Stack:
    """Device buffers and the step of a list of linears (one process = one rank)."""

    def __init__(self, lins, n_layers, args, dev, rank, world):
        import torch

        import paper_2306_11987_b200 as i4
        self.lins, self.n_layers, self.args, self.dev = lins, n_layers, args, dev
        self.world, self.rank = world, rank
        N = lins[0][1]
        self.N = N
        self.token_offset = rank * N                       # global index of this shard's first token (Z-20)
        D_max = max(ln[2] for ln in lins)
        C_max = max(ln[3] for ln in lins)
        self.scratch = i4.BwdScratch(N, D_max, C_max, dev)   # transient backward buffers, shared by all linears
        dense_g = args.grad == "dense"

        def up(a):
            return torch.from_numpy(synth.bf16_bits(a).view(np.int16).copy()).view(torch.bfloat16).to(dev)

        # seeded synthetic data: one base tensor per linear role; layer l's copy is
        # rolled along rows and columns (same distribution, distinct buffers)
        base, self.host = {}, {}
        for (nm, _, D, C, k, layer, cid) in lins:
            if nm not in base:
                x = synth.activations(N, D, seed=synth.DATA_SEED + 7919 * rank)
                w = synth.weights(C, D)
                g = synth.grad_output(N, C, seed=synth.DATA_SEED + 7919 * rank, dense=dense_g)
                base[nm] = (up(x), up(w), up(g))
                self.host[nm] = (x, w, g)
        self.per_layer = {}
        for i, ln in enumerate(lins):
            self.per_layer.setdefault(ln[5], []).append(i)
        # grad_W of one layer = one flat fp32 bucket (the all-reduce unit)
        self.dW_bucket = [torch.zeros(sum(lins[i][3] * lins[i][2] for i in self.per_layer[layer]),
                                      dtype=torch.float32, device=dev) for layer in range(n_layers)]
        self.X, self.W, self.G, self.Y, self.dX, self.dW, self.layers, self.s = [], [], [], [], [], [], [], []
        offs = {layer: 0 for layer in range(n_layers)}
        for i, (nm, _, D, C, k, layer, cid) in enumerate(lins):
            bx, bw, bg = base[nm]
            sh = (131 * layer) % N
            self.X.append(torch.roll(bx, shifts=(sh, 7 * layer), dims=(0, 1)).contiguous() if layer else bx)
            self.W.append(torch.roll(bw, shifts=(3 * layer, 5 * layer), dims=(0, 1)).contiguous() if layer else bw)
            self.G.append(torch.roll(bg, shifts=(sh, 11 * layer), dims=(0, 1)).contiguous() if layer else bg)
            self.Y.append(torch.empty(N, C, dtype=torch.bfloat16, device=dev))     # perf mode: bf16 Y, grad_X (Z-24)
            self.dX.append(torch.empty(N, D, dtype=torch.bfloat16, device=dev))
            o = offs[layer]
            self.dW.append(self.dW_bucket[layer][o:o + C * D].view(C, D))         # fp32 grad_W (all-reduce operand)
            offs[layer] = o + C * D
            self.layers.append(i4.Int4Linear(N, D, C, k, device=dev, scratch=self.scratch))
            self.s.append((i4.cold_start_step(self.X[-1]), i4.cold_start_step(self.W[-1])))   # A.4, library kernel
        self.mode = MODES[args.mode]
        self.mc = [None] * len(lins)              # NVLS multicast grad_W addresses (--wgrad-reduce nvls)
        self.sym = None

    def enable_nvls(self):
        """grad_W buckets in symmetric memory; each linear's grad_W GEMM reduces into its
        bucket's multicast address.  False when no multicast object is available."""
        from paper_2306_11987_b200 import dist as pdist
        self.sym = [pdist.SymmetricGradW(b.numel(), self.dev) for b in self.dW_bucket]
        if not all(s.available for s in self.sym):
            self.sym = None
            return False
        offs = {layer: 0 for layer in range(self.n_layers)}
        for i, (nm, _, D, C, k, layer, cid) in enumerate(self.lins):
            self.mc[i] = self.sym[layer].multicast(offs[layer])
            offs[layer] += C * D
        return True

    def fwd_one(self, i):
        s_x, s_w = self.s[i]
        self.layers[i].forward(self.X[i], self.W[i], s_x, s_w, self.Y[i])

    def bwd_one(self, i):
        self.layers[i].backward(self.G[i], self.dX[i], self.dW[i], synth.PHILOX_SEED, call_id=self.lins[i][6],
                                token_offset=self.token_offset, mode=self.mode, dw_multicast=self.mc[i])

    # the two halves of a step (graph bodies)
    def fwd_body(self):
        for i in range(len(self.lins)):
            self.fwd_one(i)

    def bwd_body(self, layer):
        for i in reversed(self.per_layer[layer]):
            self.bwd_one(i)

    def bytes_h2d(self):
        return sum(t.numel() * t.element_size() for t in self.X + self.W + self.G)


def capture(fn):
    import torch
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2306_11987_b200 as i4

    rank, world, local = env_world()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # --layer-graphs: the N > 1 step structure (per-layer backward graphs, an async NCCL
    # all-reduce per layer) on a one-rank group -- exercises that path on one GPU
    multi = world > 1 or args.layer_graphs
    if multi and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        with stdout_to_stderr():          # NCCL may print its version line: stdout carries only the JSON line
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
            dist.barrier()
    lins, n_layers = workload(args.config)
    peaks = load_peaks()
    int8_peak = peaks["bf16_tflops"] * INT8_OVER_BF16

    st = Stack(lins, n_layers, args, dev, rank, world)
    st.fwd_body()                              # eager once: lazy library state (side streams, attributes)
    for layer in reversed(range(n_layers)):
        st.bwd_body(layer)
    torch.cuda.synchronize()
    gate = parity_gate(st) if (rank == 0 and not args.no_gate) else None
    st.scratch.status_buf.zero_()
    nvls = world > 1 and args.wgrad_reduce == "nvls" and st.enable_nvls()

    flush_w = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    flush_r = torch.ones(32 * 1024 * 1024, dtype=torch.int64, device=dev)

    def flush():
        """256 MiB write (> 126 MB L2) then a 256 MiB read of another buffer, so the
        step starts with a cold, clean L2 (outside the timed events)."""
        flush_w.zero_()
        torch.sum(flush_r)

    def whole_step():
        st.fwd_body()
        for layer in reversed(range(n_layers)):
            st.bwd_body(layer)

    if not multi:       # no exchange: the whole step is one graph (no gaps between graph launches)
        g_fwd, g_bwd = capture(whole_step), [None] * n_layers
    else:               # the all-reduces go between the per-layer backward graphs
        g_fwd = capture(st.fwd_body)
        g_bwd = [capture(lambda l=l: st.bwd_body(l)) for l in range(n_layers)]
    ev_a, ev_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def one_step(gf, gb, buckets, fused=False):
        if fused:           # NVLS: every rank zeroes its copy; the grad_W GEMMs reduce into all copies
            for sym in st.sym:
                sym.zero_()
        gf.replay()
        handles = []
        for layer in reversed(range(n_layers)):
            if gb[layer] is not None:
                gb[layer].replay()
            if multi and not fused:       # async on NCCL's stream: overlaps the next (lower) layer's backward
                handles.append(dist.all_reduce(buckets[layer], op=dist.ReduceOp.SUM, async_op=True))
        for h in handles:
            h.wait()        # the compute stream waits for every all-reduce before the step ends
        if fused:
            st.sym[0].barrier()           # every rank's reductions have landed

    def timed(gf, gb, buckets, n, fused=False):
        out = []
        for _ in range(n):
            flush()
            torch.cuda.synchronize()
            ev_a.record()
            one_step(gf, gb, buckets, fused)
            ev_b.record()
            torch.cuda.synchronize()
            out.append(ev_a.elapsed_time(ev_b))
        return out

    timed(g_fwd, g_bwd, st.dW_bucket, args.warmup, nvls)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        step_ms = timed(g_fwd, g_bwd, st.dW_bucket, args.steps, nvls)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = statistics.mean(step_ms)
    ms_max = max_over_ranks(ms, dev, world)
    ops = work_ops(lins)
    value = ops * world / (ms_max * 1e-3) / 1e12
    status_word = int(st.scratch.status_buf.item())

    # ---- cuBLAS BF16 stack, same protocol (bf16 grad_W buckets all-reduced the same way)
    bf_bucket = [torch.zeros(b.numel(), dtype=torch.bfloat16, device=dev) for b in st.dW_bucket]
    bf_dW, offs = [], {layer: 0 for layer in range(n_layers)}
    for i, (nm, N, D, C, k, layer, cid) in enumerate(lins):
        bf_dW.append(bf_bucket[layer][offs[layer]:offs[layer] + C * D].view(C, D))
        offs[layer] += C * D
    Yb = [torch.empty_like(y) for y in st.Y]
    dXb = [torch.empty_like(x) for x in st.dX]

    def bf_fwd():
        for i in range(len(lins)):
            torch.matmul(st.X[i], st.W[i].t(), out=Yb[i])

    def bf_bwd(layer):
        for i in reversed(st.per_layer[layer]):
            torch.matmul(st.G[i], st.W[i], out=dXb[i])
            torch.matmul(st.G[i].t(), st.X[i], out=bf_dW[i])

    def bf_step():
        bf_fwd()
        for layer in reversed(range(n_layers)):
            bf_bwd(layer)

    bf_step()
    torch.cuda.synchronize()
    if not multi:
        gb_fwd, gb_bwd = capture(bf_step), [None] * n_layers
    else:
        gb_fwd = capture(bf_fwd)
        gb_bwd = [capture(lambda l=l: bf_bwd(l)) for l in range(n_layers)]
    timed(gb_fwd, gb_bwd, bf_bucket, args.warmup)
    bf16_ms = max_over_ranks(statistics.mean(timed(gb_fwd, gb_bwd, bf_bucket, args.steps)), dev, world)
    del gb_fwd, gb_bwd, Yb, dXb, bf_bucket, bf_dW

    # ---- per-kernel breakdown: CUPTI records over PDL-off replays of the same step
    prev_pdl = i4.int4_set_pdl(False)
    s_fwd = capture(st.fwd_body)
    s_bwd = [capture(lambda l=l: st.bwd_body(l)) for l in range(n_layers)]
    cupti, n_launch = cupti_kernel_times(lambda: (flush(), one_step(s_fwd, s_bwd, st.dW_bucket)), min(args.steps, 5))
    i4.int4_set_pdl(prev_pdl)
    del s_fwd, s_bwd
    # realized kept counts / dense flags / compact bytes of each distinct linear shape (one
    # more eager backward of its first instance: the same inputs and streams as in the step)
    shape_stats = {}
    for i, (nm, N, D, C, k, layer, cid) in enumerate(lins):
        if nm in shape_stats:
            continue
        st.bwd_one(i)
        torch.cuda.synchronize()
        kw, kx = [int(v) for v in st.layers[i].counts().cpu().numpy()]
        form = tuple(int(v) for v in st.layers[i].dense_flags().cpu().numpy())
        dense = tuple(f == 1 for f in form)
        shape_stats[nm] = dict(N=N, D=D, C=C, kw=kw, kx=kx, dense=dense, form=form,
                               compact_bytes=compact_bytes(st.layers[i], N, D, C, kx, kw, form))
    step_us = ms * 1e3
    kernels = {nm: {"us_per_step": tot, "launches_per_step": n_launch.get(nm, 0), "share": tot / step_us}
               for nm, tot in cupti.items()}
    for nm in kernels:                        # achieved rate over the step: sum of work / sum of time
        work, kind = 0.0, None
        for ln in lins:
            s_ = shape_stats[ln[0]]
            kind, amt = algorithmic_work(nm, s_["N"], s_["D"], s_["C"], s_["kx"], s_["kw"], s_["dense"],
                                         s_["compact_bytes"])
            work += amt
        t = kernels[nm]["us_per_step"] * 1e-6
        if kind == "ops" and t > 0:
            kernels[nm].update(achieved_tops=work / t / 1e12, frac_int8_peak=work / t / 1e12 / int8_peak)
        elif kind == "bytes" and t > 0 and work > 0:
            kernels[nm].update(achieved_gbs=work / t / 1e9, frac_hbm=work / t / 1e9 / peaks["hbm_gbs"])

    roof = dominant_roofline(st, kernels, shape_stats, args, flush, int8_peak, peaks)

    per_linear = None
    if rank == 0 and not args.no_per_linear and args.config == DEFAULT_CONFIG:
        per_linear = {cfg: {g: time_single(cfg, g, args, dev, flush) for g in ("sparse", "dense")}
                      for cfg in PER_LINEAR}
    attention_bmm = None
    if rank == 0 and not args.no_per_linear and args.config == DEFAULT_CONFIG:
        attention_bmm = {f"B{b}_N{n}_P{p}_M{m}": time_bmm(b, n, p, m, 5, args, dev, flush) for b, n, p, m in BMM_SHAPES}

    e2e = None if args.no_e2e else run_e2e(st, args, dev, world, ops, flush)

    if rank == 0:
        gemm_names = ("gemm_i8_fwd", "gemm_i8_dgrad", "gemm_i8_wgrad", "gemm_i8_bwd")
        gemm_us = sum(kernels[nm]["us_per_step"] for nm in gemm_names if nm in kernels)
        if GROUP in kernels:                  # concurrent pairs: count their union, not both kernels
            gemm_us = kernels.get("gemm_i8_fwd", {}).get("us_per_step", 0.0) + kernels[GROUP]["us_per_step"]
        gemm_ops = 0.0
        for ln in lins:
            s_ = shape_stats[ln[0]]
            gemm_ops += 2.0 * s_["C"] * s_["D"] * (s_["N"] + (s_["N"] if s_["dense"][1] else s_["kx"]) +
                                                   (s_["N"] if s_["dense"][0] else s_["kw"]))
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "s8", "data": "synthetic",
                "config": workload_config(args, lins, world),
                "speedup_vs_bf16_cublas": bf16_ms / ms_max, "bf16_cublas_ms_per_step": bf16_ms,
                "gemm_int8_peak_frac": gemm_ops / (gemm_us * 1e-6) / 1e12 / int8_peak if gemm_us else None,
                "kept_items": {nm: {"grad_W": v["kw"], "grad_X": v["kx"], "budget": v["N"],
                                    "operand_form": {"grad_W": v["form"][0], "grad_X": v["form"][1],
                                                     "legend": "0 compacted kept items, 1 dense Q/X_hat (Z-32), "
                                                               "2 dense + correction rows (Z-33)"}}
                               for nm, v in shape_stats.items()},
                "roofline": roof, "kernels": kernels,
                "kernels_timing": "CUPTI kernel records (torch.profiler) over extra flushed PDL-off replays; per step",
                "gpu_launches": sum(n_launch.values()) * args.steps,
                "clocks": clocks.summary(), "e2e": e2e, "parity_gate": gate, "status_word": status_word,
                "per_linear": per_linear,
                "attention_bmm": attention_bmm,
                "allreduce": (("grad_W reduced inside the grad_W GEMM epilogue into NVLS multicast buffers "
                               "(multimem.red.add; symmetric-memory barrier at the step's end)") if nvls else
                              ("per layer grad_W bucket (fp32), async on NCCL's stream after the layer's backward "
                               "graph, overlapping the next layer's backward; waited before the step's end event"))
                if multi else None}
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(lins, args.grad, args.mode)
        print(json.dumps(line), flush=True)
    if multi:
        dist.barrier()
        dist.destroy_process_group()
    return 0


class stdout_to_stderr:
    """File-descriptor-level redirect of stdout to stderr (native libraries print with printf)."""
    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)
        return False


def max_over_ranks(value, device, world):
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _bits(words, rows, cols):
    w = words.cpu().numpy().view(np.uint32)
    return ((w[..., None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(rows, -1)[:, :cols].astype(bool)


def parity_gate(st):
    """Before timing: one linear of the step (the first FFN-up,
    or the only linear) against the oracle -- codes and forward rows, the bit split
    on sampled rows (bit-exact, with the tensor's global amax), both sampler lists
    in full from the verified norms, grad_X on sampled tokens and grad_W on sampled
    channels within 1e-5.  Part of the harness around the timed region (the
    cpu_baseline side of bench.py), never inside it; fp32 outputs into scratch."""
    import torch

    from oracle import bitsplit as o_bs
    from oracle import gemm as o_gemm
    from oracle import hq as o_hq
    from oracle import linear as o_lin
    from oracle import lss as o_lss
    idx = next((i for i, ln in enumerate(st.lins) if ln[0] == "ffn_up"), 0)
    nm, N, D, C, k, layer, cid = st.lins[idx]
    lay = st.layers[idx]
    s_x, s_w = st.s[idx]
    Y = torch.empty(N, C, dtype=torch.float32, device=st.dev)
    dX = torch.empty(N, D, dtype=torch.float32, device=st.dev)
    dW = torch.empty(C, D, dtype=torch.float32, device=st.dev)
    lay.forward(st.X[idx], st.W[idx], s_x, s_w, Y)
    lay.backward(st.G[idx], dX, dW, synth.PHILOX_SEED, call_id=cid, token_offset=st.token_offset, mode=st.mode)
    torch.cuda.synchronize()
    rows = np.sort(np.random.default_rng(4).choice(N, 32, replace=False))

    def host(t):
        return (t.view(torch.int16).cpu().numpy().view(np.uint16).astype(np.uint32) << 16).view(np.float32)

    x, w, g = host(st.X[idx]), host(st.W[idx]), host(st.G[idx])
    xq, wq = lay.xq.cpu().numpy(), lay.wq.cpu().numpy()
    oc, _, _ = o_hq.hadamard_quant(x[rows], k, s_x)
    ow, _, _ = o_hq.hadamard_quant(w, k, s_w)
    nbad = int((xq[rows] != oc).sum()) + int((wq != ow).sum())
    assert max(int(np.abs(xq[rows].astype(int) - oc).max()), int(np.abs(wq.astype(int) - ow).max())) <= 1
    assert nbad <= 1e-6 * (oc.size + ow.size), "code parity"
    y_ref = o_gemm.int_matmul_abt(xq[rows], wq) * (np.float64(s_x) * np.float64(s_w))
    y_err = float(np.linalg.norm(Y.cpu().numpy()[rows] - y_ref) / np.linalg.norm(y_ref))
    assert y_err < 1e-5, f"forward parity {y_err}"
    # bit split on sampled rows: the oracle per row, the tensor's global amax planted in a second row
    amax_val = np.float32(np.abs(g).max())
    q8 = lay.q8_codes().cpu().numpy()
    a_sq = lay.a_sq.cpu().numpy().reshape(2, N)
    for t in rows[:8]:
        gt = np.zeros((2, C), np.float32)
        gt[0] = g[t]
        gt[1, 0] = amax_val
        b = o_bs.bit_split(gt, synth.PHILOX_SEED, cid, st.token_offset + int(t))
        assert np.array_equal(q8[t].astype(np.int64), b["q"][0]), "bit split parity"
        assert a_sq[0, t] == b["a_sq"][0, 0] and a_sq[1, t] == b["a_sq"][1, 0], "norm parity"
    x_sq = lay.x_sqnorm.cpu().numpy().astype(np.int64)
    assert np.array_equal(x_sq, (xq.astype(np.int64) ** 2).sum(1))
    mw = o_lss.sample_weight_mask(a_sq, x_sq, synth.PHILOX_SEED, cid, st.token_offset, st.mode)
    mx = o_lss.sample_activation_mask(a_sq, synth.PHILOX_SEED, cid, st.token_offset, st.mode)
    cw, cx = [int(v) for v in lay.counts().cpu().numpy()]
    assert (cw, cx) == (mw["count"], mx["count"]), "kept counts"

    def pairs(it, we):
        o = np.argsort(it, kind="stable")
        return np.stack([np.asarray(it, np.int64)[o], np.asarray(we, np.int64)[o]])

    assert np.array_equal(pairs(lay.items_w[:cw].cpu().numpy(), lay.wexp_w[:cw].cpu().numpy()),
                          pairs(mw["items"], mw["wexp"])), "grad_W list"
    assert np.array_equal(pairs(lay.items_x[:cx].cpu().numpy(), lay.wexp_x[:cx].cpu().numpy()),
                          pairs(mx["items"], mx["wexp"])), "grad_X list"
    # gradients from the (sample-verified) code plane
    qq = q8[:N].astype(np.int64)
    hi = np.floor_divide(qq + 8, 16)
    bs = dict(hi=hi.astype(np.int8), lo=(qq - 16 * hi).astype(np.int8), s_down=np.float32(amax_val) / np.float32(119))
    x_mask, w_mask = _bits(lay.x_mask, N, D), _bits(lay.w_mask, C, D)
    sel = np.isin(mx["items"] % N, rows)
    dx_ref, _ = o_lin.grad_x_from_items(bs, mx["items"][sel], mx["wexp"][sel], wq, x_mask, k, np.float32(s_w))
    dx_err = float(np.linalg.norm(dX.cpu().numpy()[rows] - dx_ref[rows]) / max(np.linalg.norm(dx_ref[rows]), 1e-30))
    ch = np.sort(np.random.default_rng(5).choice(C, 16, replace=False))
    bs_c = dict(bs, hi=bs["hi"][:, ch], lo=bs["lo"][:, ch])
    dw_ref, _ = o_lin.grad_w_from_items(bs_c, mw["items"], mw["wexp"], xq, w_mask[ch], k, np.float32(s_x))
    dw_err = float(np.linalg.norm(dW.cpu().numpy()[ch] - dw_ref) / max(np.linalg.norm(dw_ref), 1e-30))
    assert dx_err < 1e-5 and dw_err < 1e-5, f"gradient parity {dx_err} {dw_err}"
    return {"linear": f"layer {layer} {nm}", "y_rel_err": y_err, "dx_rel_err": dx_err, "dw_rel_err": dw_err,
            "kept": [cw, cx], "checked": "codes (32 rows + all of W), Y rows, bit split rows (bit-exact), both "
                                         "sampler lists in full, grad_X on 32 tokens, grad_W on 16 channels vs oracle/"}


def cupti_kernel_times(step, n):
    """Per-step device time (us) summed per kernel name, and launches per step, from
    the CUPTI activity records torch.profiler collects (kernels inside graphs too).
    Concurrent grad_X || grad_W pairs are also reported as GROUP: the summed union
    of the two GEMMs' [start, end) intervals."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    acc, cnt = {}, {}
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(n):
            step()
            torch.cuda.synchronize()
    for ev in prof.events():
        if ev.device_type.name != "CUDA":
            continue
        nm = short_kernel_name(ev.name)
        if nm is None:
            continue
        acc[nm] = acc.get(nm, 0.0) + ev.device_time_total
        cnt[nm] = cnt.get(nm, 0) + 1
    out = {nm: v / n for nm, v in acc.items()}
    launches = {nm: c // n for nm, c in cnt.items()}
    try:
        d, w = [], []
        for ev in prof.profiler.kineto_results.events():
            nm = short_kernel_name(ev.name())
            if nm == "gemm_i8_dgrad":
                d.append((ev.start_ns(), ev.start_ns() + ev.duration_ns()))
            elif nm == "gemm_i8_wgrad":
                w.append((ev.start_ns(), ev.start_ns() + ev.duration_ns()))
        d.sort()
        w.sort()
        if d and len(d) == len(w):            # the i-th grad_X GEMM and the i-th grad_W GEMM are one linear's pair
            union, conc = 0, 0
            for a, b in zip(d, w):
                ov = min(a[1], b[1]) - max(a[0], b[0])
                union += max(a[1], b[1]) - min(a[0], b[0])
                conc += ov > 0.2 * min(a[1] - a[0], b[1] - b[0])
            if conc > len(d) // 2:            # the library ran them concurrently (its work model chose to)
                out[GROUP] = union / n / 1e3
    except Exception:
        pass
    return out, launches


KERNEL_NAMES = [("hadamard_quant_kernel", "hadamard_quant"), ("grad_split_kernel", "grad_split"),
                ("lss_sampler_kernel", "lss_sampler"), ("compact_kernel", "compact")]
GEMM_EPI = {"0": "gemm_i8_int32", "1": "gemm_i8_fwd", "2": "gemm_i8_dgrad", "3": "gemm_i8_wgrad",
            "4": "gemm_i8_bwd"}


def short_kernel_name(full):
    if "gemm_i8_kernel<" in full:
        epi = full.split("gemm_i8_kernel<", 1)[1].split(",")[1].strip()
        return GEMM_EPI.get(epi, "gemm_i8")
    for key, short in KERNEL_NAMES:
        if key in full:
            return short
    return None                          # not ours (L2 flush, NCCL, cuBLAS)


def dominant_roofline(st, kernels, shape_stats, args, flush, int8_peak, peaks):
    """roofline entry of the dominant kernel (largest share of the step): CUDA events
    recorded on the launch stream around its launch inside one linear (the shape
    with the most work for that kernel), replayed within the full step graphs and
    averaged over the timed steps."""
    import torch

    import paper_2306_11987_b200 as i4
    cands = [nm for nm in kernels if nm != GROUP]
    if GROUP in kernels:                      # the concurrent pair is one unit: drop its members
        cands = [nm for nm in cands if nm not in ("gemm_i8_dgrad", "gemm_i8_wgrad")] + [GROUP]
    if not cands:
        return None
    dom = max(cands, key=lambda nm: kernels[nm]["us_per_step"])
    best_i, best_amt, seen = 0, -1.0, set()
    for i, ln in enumerate(st.lins):
        if ln[0] in seen:
            continue
        seen.add(ln[0])
        s_ = shape_stats[ln[0]]
        _, amt = algorithmic_work(dom, s_["N"], s_["D"], s_["C"], s_["kx"], s_["kw"], s_["dense"], s_["compact_bytes"])
        if amt > best_amt:
            best_i, best_amt = i, amt
    nm_l, N, D, C, k, layer, cid = st.lins[best_i]
    s_ = shape_stats[nm_l]
    namer = i4.LaunchTrace([torch.cuda.Event(enable_timing=True) for _ in range(2)], first_launch=10 ** 6)
    with namer:
        st.fwd_one(best_i)
    n_fwd = len(namer.names)
    with namer:
        st.bwd_one(best_i)
    names_b = namer.names
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(2)]
    if dom in ("hadamard_quant", "gemm_i8_fwd"):
        in_fwd, pos = True, ["hadamard_quant", "gemm_i8_fwd"].index(dom)
        if pos >= n_fwd:
            return None
    elif dom in names_b:
        in_fwd, pos = False, names_b.index(dom)
    else:
        return None

    tracer = i4.LaunchTrace(ev, first_launch=pos)     # created (events materialised) outside any capture

    def fwd_traced():
        for i in range(len(st.lins)):
            if i == best_i and in_fwd:
                with tracer:
                    st.fwd_one(i)
            else:
                st.fwd_one(i)

    def bwd_traced(layer):
        for i in reversed(st.per_layer[layer]):
            if i == best_i and not in_fwd:
                with tracer:
                    st.bwd_one(i)
            else:
                st.bwd_one(i)

    gf = capture(fwd_traced)
    gb = [capture(lambda l=l: bwd_traced(l)) for l in range(st.n_layers)]
    durs = []
    for it in range(args.warmup + args.steps):
        flush()
        gf.replay()
        for layer in reversed(range(st.n_layers)):
            gb[layer].replay()
        torch.cuda.synchronize()
        if it >= args.warmup:
            durs.append(ev[0].elapsed_time(ev[1]))
    del gf, gb
    avg_s = statistics.mean(durs) * 1e-3
    kind, amount = algorithmic_work(dom, N, D, C, s_["kx"], s_["kw"], s_["dense"], s_["compact_bytes"])
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(f"{args.config}:{nm_l}", {}).get(dom)
    if kind == "ops":
        achieved = amount / avg_s / 1e12
        roof = {"kernel": dom, "bound": "tensor", "achieved": achieved, "peak": int8_peak, "unit": "TFLOP/s",
                "frac": achieved / int8_peak, "traffic": traffic,
                "peak_source": f"{peaks['source']}: bf16 {peaks['bf16_tflops']} TF/s (burst) x nominal INT8:BF16 = 2 "
                               f"(int8 TOPS); the burst figure because the step runs at full clocks (see clocks)",
                "peak_sustained": 2 * peaks["bf16_tflops_sustained"],
                "frac_vs_sustained": achieved / (2 * peaks["bf16_tflops_sustained"]),
                "work_per_launch": f"2*M*N*K = {amount:.4g} int ops"}
    else:
        achieved = amount / avg_s / 1e9
        roof = {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": traffic, "peak_source": peaks["source"],
                "work_per_launch": f"{amount:.4g} algorithmic bytes"}
    roof["linear"] = f"layer {layer} {nm_l} ({N} x {D} -> {C})"
    roof["avg_launch_us_events"] = avg_s * 1e6
    roof["share_of_step"] = kernels[dom]["share"]
    roof["timing"] = ("CUDA events recorded on the launch stream immediately before/after this kernel's node in "
                      "that linear's captured graph, replayed inside the full step, averaged over the timed steps")
    return roof


def time_single(config, grad, args, dev, flush):
    """One BERT-large linear alone (fwd + bwd graph, flushed L2) and cuBLAS BF16 beside it."""
    import torch

    import paper_2306_11987_b200 as i4
    c = synth.CONFIGS[config]
    N, D, C, k = c["N"], c["D"], c["C"], c["k"]

    def up(a):
        return torch.from_numpy(synth.bf16_bits(a).view(np.int16).copy()).view(torch.bfloat16).to(dev)

    X, W = up(synth.activations(N, D)), up(synth.weights(C, D))
    G = up(synth.grad_output(N, C, dense=(grad == "dense")))
    s_x, s_w = i4.cold_start_step(X), i4.cold_start_step(W)
    lay = i4.Int4Linear(N, D, C, k, device=dev)
    Y = torch.empty(N, C, dtype=torch.bfloat16, device=dev)
    dX = torch.empty(N, D, dtype=torch.bfloat16, device=dev)
    dW = torch.empty(C, D, dtype=torch.float32, device=dev)
    dWb = torch.empty(C, D, dtype=torch.bfloat16, device=dev)
    mode = MODES[args.mode]

    def body():
        lay.forward(X, W, s_x, s_w, Y)
        lay.backward(G, dX, dW, synth.PHILOX_SEED, call_id=1, mode=mode)

    def bf_body():
        torch.matmul(X, W.t(), out=Y)
        torch.matmul(G, W, out=dX)
        torch.matmul(G.t(), X, out=dWb)

    out = {}
    for nm, fn in (("int4", body), ("bf16", bf_body)):
        fn()
        torch.cuda.synchronize()
        g = capture(fn)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for it in range(3 + max(10, args.steps)):
            flush()
            torch.cuda.synchronize()
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            if it >= 3:
                ts.append(a.elapsed_time(b) * 1e3)
        out[nm] = statistics.mean(ts)
    kw, kx = [int(v) for v in lay.counts().cpu().numpy()]
    dense = [bool(v) for v in lay.dense_flags().cpu().numpy()]
    return {"int4_us": out["int4"], "bf16_cublas_us": out["bf16"], "speedup": out["bf16"] / out["int4"],
            "eff_tops": 6.0 * N * C * D / (out["int4"] * 1e-6) / 1e12,
            "kept": {"grad_W": kw, "grad_X": kx, "budget": N}, "dense_masks": {"grad_W": dense[0], "grad_X": dense[1]}}


# attention BMM shapes (A.1; BERT-base heads: 12 heads x 512 tokens x 64, and 48 x 128)
BMM_SHAPES = [(12, 512, 512, 64), (48, 128, 128, 64)]


def time_bmm(B, N, P, M, k, args, dev, flush):
    """T = BMM(Q, K^T) fwd + bwd (A.1, batched inside the kernels: 7 launches) and cuBLAS
    BF16 torch.bmm (T = Q K^T, dQ = dT K, dK = dT^T Q) beside it; graphs, flushed L2."""
    import torch

    import paper_2306_11987_b200 as i4

    def up(a):
        return torch.from_numpy(synth.bf16_bits(a).view(np.int16).copy()).view(torch.bfloat16).to(dev)

    q = up(np.stack([synth.activations(N, M, seed=b) for b in range(B)]))
    kk = up(np.stack([synth.activations(P, M, seed=100 + b) for b in range(B)]))
    dt = up(np.stack([synth.grad_output(N, P, seed=200 + b, dense=(b % 2 == 0)) for b in range(B)]))
    s_q = np.array([float(i4.cold_start_step(q[b])) for b in range(B)], np.float32)
    s_k = np.array([float(i4.cold_start_step(kk[b])) for b in range(B)], np.float32)
    op = i4.Int4BMM(B, N, P, M, k, device=dev)
    T = torch.empty(B, N, P, dtype=torch.bfloat16, device=dev)
    dQ = torch.empty(B, N, M, dtype=torch.bfloat16, device=dev)
    dK = torch.empty(B, P, M, dtype=torch.float32, device=dev)
    Tb, dQb, dKb = torch.empty_like(T), torch.empty_like(dQ), torch.empty(B, P, M, dtype=torch.bfloat16, device=dev)

    def body():
        op.forward(q, kk, s_q, s_k, T)
        op.backward(dt, dQ, dK, synth.PHILOX_SEED, call_id=1, mode=MODES[args.mode])

    def bf_body():
        torch.bmm(q, kk.transpose(1, 2), out=Tb)
        torch.bmm(dt, kk, out=dQb)
        torch.bmm(dt.transpose(1, 2), q, out=dKb)

    out = {}
    for nm, fn in (("int4", body), ("bf16", bf_body)):
        fn()
        torch.cuda.synchronize()
        g = capture(fn)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for it in range(3 + max(10, args.steps)):
            flush()
            torch.cuda.synchronize()
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            if it >= 3:
                ts.append(a.elapsed_time(b) * 1e3)
        out[nm] = statistics.mean(ts)
    return {"int4_us": out["int4"], "bf16_cublas_us": out["bf16"], "speedup": out["bf16"] / out["int4"],
            "eff_tops": 6.0 * B * N * P * M / (out["int4"] * 1e-6) / 1e12, "launches_per_step": 7,
            "status_word": op.status()}


def run_e2e(st, args, dev, world, ops, flush):
    """The same step through the public API (Int4Linear.forward / backward over the C
    ABI, eager launches) with host buffers: every step copies every linear's X, W and
    grad_Y from pinned host memory to the device and reads every grad_W bucket back
    (the step's result: the weight gradients an optimizer consumes).  The copies are
    pipelined with the compute as a training loop would stream them: one copy
    stream brings X and W in forward order, then grad_Y in backward order, and the
    compute stream waits for each linear's own inputs only; a second copy stream
    (the other PCIe direction) reads each layer's grad_W bucket back as soon as its
    backward (and, for N > 1, its all-reduce) is done.  The timed region runs from
    the first copy to the last read-back."""
    import torch
    import torch.distributed as dist
    host_in = {nm: [torch.from_numpy(synth.bf16_bits(a).view(np.int16).copy()).view(torch.bfloat16).pin_memory()
                    for a in xwg] for nm, xwg in st.host.items()}
    host_out = [torch.empty(b.numel(), dtype=torch.float32).pin_memory() for b in st.dW_bucket]
    main = torch.cuda.current_stream()
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    n = len(st.lins)
    ev_xw = [torch.cuda.Event() for _ in range(n)]
    ev_g = [torch.cuda.Event() for _ in range(n)]
    ev_layer = [torch.cuda.Event() for _ in range(st.n_layers)]
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    bwd_order = [i for layer in reversed(range(st.n_layers)) for i in reversed(st.per_layer[layer])]
    times = []
    for it in range(args.warmup + min(args.steps, 10)):
        flush()
        torch.cuda.synchronize()
        a0.record(main)
        h2d.wait_stream(main)
        d2h.wait_stream(main)
        with torch.cuda.stream(h2d):
            for i, ln in enumerate(st.lins):
                hx, hw, _ = host_in[ln[0]]
                st.X[i].copy_(hx, non_blocking=True)
                st.W[i].copy_(hw, non_blocking=True)
                ev_xw[i].record(h2d)
            for i in bwd_order:
                st.G[i].copy_(host_in[st.lins[i][0]][2], non_blocking=True)
                ev_g[i].record(h2d)
        for i in range(n):
            main.wait_event(ev_xw[i])
            st.fwd_one(i)
        for layer in reversed(range(st.n_layers)):
            for i in reversed(st.per_layer[layer]):
                main.wait_event(ev_g[i])
                st.bwd_one(i)
            h = dist.all_reduce(st.dW_bucket[layer], op=dist.ReduceOp.SUM, async_op=True) if world > 1 else None
            ev_layer[layer].record(main)
            with torch.cuda.stream(d2h):
                d2h.wait_event(ev_layer[layer])
                if h is not None:
                    h.wait()                      # the read-back waits for this bucket's all-reduce
                host_out[layer].copy_(st.dW_bucket[layer], non_blocking=True)
        main.wait_stream(d2h)
        main.wait_stream(h2d)
        a1.record(main)
        torch.cuda.synchronize()
        if it >= args.warmup:
            times.append(a0.elapsed_time(a1))
    t = max_over_ranks(statistics.mean(times), dev, world)
    return {"value": ops * world / (t * 1e-3) / 1e12, "unit": UNIT, "h2d_bytes_per_step": int(st.bytes_h2d()),
            "d2h_bytes_per_step": int(sum(b.numel() * 4 for b in st.dW_bucket)), "ms_per_step": t,
            "path": "pinned host X, W, grad_Y of every linear -> device on a copy stream (forward order, then "
                    "grad_Y in backward order), each linear's Int4Linear.forward / backward (C ABI, eager "
                    "launches) waiting for its own inputs only; every layer's grad_W bucket -> pinned host on a "
                    "second copy stream as soon as the layer's backward is done"}


# ---------------------------------------------------------------------------- dry run (CPU)
def run_dry(args):
    """Launcher / sharding / overlapped all-reduce plumbing on CPU with gloo: each
    layer's grad_W bucket is filled with a rank-dependent pattern, all-reduced
    asynchronously layer by layer in backward order, waited and checked; rank 0
    prints one JSON line.  No operator compute (there is no GPU)."""
    import torch
    import torch.distributed as dist
    rank, world, _ = env_world()
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("gloo", rank=rank, world_size=world)
    lins, n_layers = workload(args.config)
    N = lins[0][1]
    buckets = [torch.full((4096,), float(rank + 1) * (layer + 1)) for layer in range(n_layers)]
    t0 = time.perf_counter()
    handles = []
    for layer in reversed(range(n_layers)):
        if world > 1:
            handles.append(dist.all_reduce(buckets[layer], op=dist.ReduceOp.SUM, async_op=True))
    for h in handles:
        h.wait()
    secs = time.perf_counter() - t0
    expect = [sum(r + 1 for r in range(world)) * (layer + 1) for layer in range(n_layers)]
    ok = all(bool(torch.all(b == e)) for b, e in zip(buckets, expect))
    t = torch.tensor([secs], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "allreduce_ok": ok,
                          "token_offsets": [r * N for r in range(world)], "layers": n_layers, "linears": len(lins),
                          "config": workload_config(args, lins, world), "max_rank_s": float(t.item())}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0 if ok else 1


def main(argv=None):
    argv = sys.argv[1:] if argv is None else list(argv)
    args = parse(argv)
    rc = maybe_spawn(args, argv)
    if rc is not None:
        return rc
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
