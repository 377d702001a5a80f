#!/usr/bin/env python
"""Benchmark of the B200 INT4 linear operator (arXiv 2306.11987, HQ-MM + LSS-MM).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg2_bert_base_ffn1] [--grad sparse|dense] [--mode bernoulli]

One step = one pass of the whole hot path over one batch of synthetic input:
  forward  : hadamard_quant(X), hadamard_quant(W) (+ W_hat^T), INT GEMM + dequant
  backward : amax, bit split, LSS sampler (both masks), compaction, grad_X GEMM,
             grad_W GEMM
  N > 1    : + NCCL all-reduce of grad_W (token-sharded data parallelism, §8(e))
The step is captured once in a CUDA graph and replayed; L2 is flushed (a
256 MiB write, outside the timed window) before every timed step.  Step time =
device time between CUDA events bracketing the step's launches on its stream.

Metric (BASELINE.json): INT4 linear fwd+bwd speedup vs BF16 cuBLAS; eff. TOPS
and % of INT8 peak.  `value` = effective TOPS = 6 N C D / t_step summed over
ranks (whole job).  `--impl reference` times the CPU oracle (test
infrastructure) on a bounded sample of the same workload on the host cores.
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "INT4 linear fwd+bwd speedup vs BF16 cuBLAS; eff. TOPS and % of INT8 peak"
UNIT = "TOPS"
DEFAULT_CONFIG = "cfg2_bert_base_ffn1"      # BASELINE.json configs[1]
INT8_OVER_BF16 = 2.0                        # nominal dense INT8 : BF16 tensor ratio on B200
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
ORACLE_REF_TOKENS = 512                     # tokens per --impl reference step (bounded sample)


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return dict(hbm_gbs=float(d["hbm_gbs"]), bf16_tflops=float(d["bf16_tflops"]),
                    bf16_tflops_sustained=float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                    source="measured (MEASURED_PEAKS.json)")
    return dict(hbm_gbs=FALLBACK_PEAKS["hbm_gbs"], bf16_tflops=FALLBACK_PEAKS["bf16_tflops"],
                bf16_tflops_sustained=FALLBACK_PEAKS["bf16_tflops"], source="fallback (B200_PROFILING.md)")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(synth.CONFIGS))
    ap.add_argument("--grad", choices=["sparse", "dense"], default="sparse")
    ap.add_argument("--mode", choices=["bernoulli", "keep_positive", "none"], default="bernoulli")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


MODES = {"bernoulli": 0, "keep_positive": 1, "none": 2}


# ---------------------------------------------------------------------------- oracle arms
def oracle_step(cfg, n_tokens, grad, mode):
    """One oracle fwd+bwd on `n_tokens` tokens of the workload; returns seconds."""
    from oracle import linear
    x = synth.activations(n_tokens, cfg["D"])
    w = synth.weights(cfg["C"], cfg["D"])
    g = synth.grad_output(n_tokens, cfg["C"], dense=(grad == "dense"))
    from oracle.lsq_grad import cold_start_step
    s_x, s_w = cold_start_step(x), cold_start_step(w)
    t0 = time.perf_counter()
    f = linear.forward(x, w, cfg["k"], s_x, s_w)
    linear.backward(g, f, synth.PHILOX_SEED, 0, 0, MODES[mode])
    return time.perf_counter() - t0


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(cfg, grad, mode, budget_s=20.0):
    """The oracle as it stands, on the host cores, on a bounded sample: whole
    workload steps (all tokens) repeated until ~budget_s of CPU work."""
    n = cfg["N"]
    times = []
    t_start = time.perf_counter()
    while True:
        times.append(oracle_step(cfg, n, grad, mode))
        if time.perf_counter() - t_start > budget_s * 0.5 or len(times) >= 4:
            break
    t = statistics.mean(times)
    return {"value": 6.0 * n * cfg["C"] * cfg["D"] / t / 1e12, "unit": UNIT, "cores": blas_threads(),
            "kind": "oracle",
            "sample": f"{len(times)} full fwd+bwd step(s) of the workload ({n} tokens, D={cfg['D']}, C={cfg['C']}),"
                      f" {t:.2f} s each; numpy/OpenBLAS fp64 + Python loops"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = synth.CONFIGS[args.config]
    n = min(ORACLE_REF_TOKENS, cfg["N"])
    for _ in range(args.warmup):
        oracle_step(cfg, n, args.grad, args.mode)
    times = [oracle_step(cfg, n, args.grad, args.mode) for _ in range(args.steps)]
    t = statistics.mean(times)
    value = 6.0 * n * cfg["C"] * cfg["D"] / t / 1e12
    sample = f"{n} of {cfg['N']} tokens per step (full D={cfg['D']}, C={cfg['C']}), fwd+bwd"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, cfg),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": blas_threads(), "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(args, cfg, world=1):
    return {"workload": f"{args.config}: {cfg['N']} tokens x {cfg['D']}->{cfg['C']} INT4 linear fwd+bwd, k={cfg['k']}",
            "tokens_per_gpu": cfg["N"], "global_tokens": cfg["N"] * world, "D": cfg["D"], "C": cfg["C"],
            "k": cfg["k"], "grad_y": args.grad, "lss_mode": args.mode, "parallelism": f"dp{world} (token-sharded)",
            "l2": "flushed before every timed step: 256 MiB write + 256 MiB read of another buffer (cold, clean L2)",
            "graph": "step captured once in a CUDA graph, replayed; kernels chained by programmatic dependent launch (per-kernel breakdown from a PDL-off capture)"}


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
            try:                                  # one more sample at the end of the timed region
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            except Exception:
                pass

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------- our arm
def algorithmic_work(name, N, D, C, kx, kw, dense=(False, False)):
    """(kind, amount) per launch: kind 'ops' (tensor) or 'bytes' (HBM); the
    per-unit figures are stated in DESIGN.md "Rooflines".  dense = (grad_W mask,
    grad_X mask) deterministic: that GEMM ran over the N token rows of Q (reading
    Z-32) and compact moved none of its operands."""
    dw, dx = dense
    rx = N if dx else kx                      # rows of the grad_X GEMM
    rw = N if dw else kw                      # K of the grad_W GEMM
    if name == "gemm_i8_fwd":
        return "ops", 2.0 * N * C * D
    if name == "gemm_i8_dgrad":
        return "ops", 2.0 * rx * C * D
    if name == "gemm_i8_wgrad":
        return "ops", 2.0 * rw * C * D
    if name == GROUP:                         # grad_X and grad_W GEMMs run concurrently: one unit
        return "ops", 2.0 * (rx + rw) * C * D
    if name == "hadamard_quant":              # X and W: read bf16, write int8 codes + 1-bit mask (+ int32 norm)
        return "bytes", (N + C) * D * (2 + 1 + 1 / 8) + 4 * N
    if name == "grad_split":                  # amax + SR: read bf16 grad_Y once (the amax pass's re-read is an
        return "bytes", N * C * (2 + 1) + 8 * N  # implementation cost), write the 8-bit code plane Q + norms
    if name == "compact":                     # half-rows of the sampled masks' items (+ B_W rows): read + write
        return "bytes", 2.0 * ((0 if dx else kx * C) + (0 if dw else kw * (C + D)))
    if name == "lss_sampler":
        return "latency", 0.0
    return "bytes", 0.0


def dominant_roofline(dom, names, step_body, timed_replays, args, N, D, C, kx, kw, int8_peak, peaks, kernels,
                      dense=(False, False)):
    """roofline entry of the dominant kernel: CUDA events around its node in the step graph."""
    import torch

    import paper_2306_11987_b200 as i4

    # ---- dominant kernel: CUDA events bracketing its launch inside the step graph
    dom_idx = names.index(dom)
    dom_ev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(2)]
    dom_tr = i4.LaunchTrace(dom_ev, first_launch=dom_idx)
    g_dom = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_dom):
        with dom_tr:
            step_body()
    dom_ms = []
    timed_replays(g_dom, args.warmup)
    timed_replays(g_dom, args.steps, on_step=lambda: dom_ms.append(dom_ev[0].elapsed_time(dom_ev[1])))
    avg_s = statistics.mean(dom_ms) * 1e-3
    kind, amount = algorithmic_work(dom, N, D, C, kx, kw, dense)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        tt = json.load(open(tpath)).get(args.config, {})
        traffic = tt.get(dom)
        if dom == GROUP and "gemm_i8_dgrad" in tt and "gemm_i8_wgrad" in tt:   # the pair: both kernels' bytes
            traffic = tt["gemm_i8_dgrad"] + tt["gemm_i8_wgrad"]
    if kind == "ops":
        achieved = amount / avg_s / 1e12
        roof = {"kernel": dom, "bound": "tensor", "achieved": achieved, "peak": int8_peak, "unit": "TFLOP/s",
                "frac": achieved / int8_peak, "traffic": traffic,
                "peak_source": f"{peaks['source']}: bf16 {peaks['bf16_tflops']} TF/s x nominal INT8:BF16 = 2 (int8 TOPS)",
                "work_per_launch": f"2*M*N*K = {amount:.4g} int ops"}
    else:
        achieved = amount / avg_s / 1e9
        roof = {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": traffic, "peak_source": peaks["source"],
                "work_per_launch": f"{amount:.4g} algorithmic bytes"}
    roof["avg_launch_us_events"] = avg_s * 1e6
    roof["avg_launch_us_cupti"] = kernels[dom]["avg_us"]
    roof["timing"] = ("CUDA events recorded on the launch stream immediately before/after this kernel's "
                      "node inside the captured step graph, averaged over the timed steps")
    return roof


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2306_11987_b200 as i4
    from paper_2306_11987_b200 import dist as pdist

    rank, world, local = pdist.env_world()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pdist.init("nccl", device=dev)
    cfg = synth.CONFIGS[args.config]
    N, D, C, k = cfg["N"], cfg["D"], cfg["C"], cfg["k"]
    mode = MODES[args.mode]
    peaks = load_peaks()
    int8_peak = peaks["bf16_tflops"] * INT8_OVER_BF16

    # ---- inputs (seeded, synthetic), resident in HBM before timing
    x = synth.activations(N, D, seed=synth.DATA_SEED + rank)
    w = synth.weights(C, D)
    g = synth.grad_output(N, C, seed=synth.DATA_SEED + rank, dense=(args.grad == "dense"))

    def up(a):
        return torch.from_numpy(synth.bf16_bits(a).view(np.int16).copy()).view(torch.bfloat16).to(dev)

    X, W, G = up(x), up(w), up(g)
    s_x, s_w = i4.cold_start_step(X), i4.cold_start_step(W)   # A.4 rule, the library's kernel
    layer = i4.Int4Linear(N, D, C, k, device=dev)
    Y = torch.empty(N, C, dtype=torch.bfloat16, device=dev)
    dX = torch.empty(N, D, dtype=torch.bfloat16, device=dev)   # perf mode: bf16 Y and grad_X (Z-24)
    dW = torch.empty(C, D, dtype=torch.float32, device=dev)    # fp32 grad_W (all-reduce operand)
    token_offset = pdist.token_offset(rank, N)           # global token index of this shard
    flush_w = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    flush_r = torch.ones(32 * 1024 * 1024, dtype=torch.int64, device=dev)

    class _Flush:
        """L2 flush before every timed step: write 256 MiB (> 126 MB L2), then read
        another 256 MiB so the dirty lines are written back before the step
        starts (the step begins with a cold but clean L2)."""

        def zero_(self):
            flush_w.zero_()
            torch.sum(flush_r)

    flush = _Flush()

    def step_body():
        layer.forward(X, W, s_x, s_w, Y)
        layer.backward(G, dX, dW, synth.PHILOX_SEED, call_id=0, token_offset=token_offset, mode=mode)

    # ---- parity gate before timing (sampled rows of Y vs the oracle's exact int product)
    step_body()
    torch.cuda.synchronize()
    rows = np.arange(0, N, max(1, N // 16))
    from oracle import gemm as o_gemm
    acc = o_gemm.int_matmul_abt(layer.xq[rows].cpu().numpy(), layer.wq.cpu().numpy())
    y_ref = acc * (np.float64(s_x) * np.float64(s_w))
    y_got = Y[rows].float().cpu().numpy()
    err = np.linalg.norm(y_got - y_ref) / np.linalg.norm(y_ref)
    assert err < 4e-3, f"parity gate failed: rel err {err}"

    # ---- capture one step in a CUDA graph (no instrumentation inside)
    stream = torch.cuda.Stream(device=dev)
    stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(stream):
        for _ in range(2):
            step_body()
    torch.cuda.current_stream().wait_stream(stream)
    torch.cuda.synchronize()
    namer = i4.LaunchTrace([torch.cuda.Event(enable_timing=True) for _ in range(2)], first_launch=10 ** 6)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        with namer:                       # window never reached: only records launch names
            step_body()
    names = namer.names
    ev_a = torch.cuda.Event(enable_timing=True)
    ev_b = torch.cuda.Event(enable_timing=True)

    def timed_replays(g, n_steps, other_dw=None, on_step=None):
        """Per step: L2 flush (untimed), then CUDA events on the stream around
        the graph replay (+ the grad_W all-reduce when N > 1)."""
        out = []
        for i in range(n_steps):
            flush.zero_()
            ev_a.record()
            g.replay()
            if world > 1:                                 # the one exchange: sum of grad_W partials
                pdist.allreduce_grad_w(dW if other_dw is None else other_dw)
            ev_b.record()
            torch.cuda.synchronize()
            out.append(ev_a.elapsed_time(ev_b))
            if on_step:
                on_step()
        return out

    timed_replays(graph, args.warmup)

    # ---- timed region (headline)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        step_ms = timed_replays(graph, args.steps)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = statistics.mean(step_ms)
    ms_max = pdist.max_over_ranks(ms, dev)
    value = 6.0 * N * C * D * world / (ms_max * 1e-3) / 1e12

    # ---- cuBLAS BF16 baseline (same protocol): Y = X W^T, dX = dY W, dW = dY^T X
    Yb = torch.empty(N, C, dtype=torch.bfloat16, device=dev)
    dXb = torch.empty(N, D, dtype=torch.bfloat16, device=dev)
    dWb = torch.empty(C, D, dtype=torch.bfloat16, device=dev)

    def bf16_body():
        torch.matmul(X, W.t(), out=Yb)
        torch.matmul(G, W, out=dXb)
        torch.matmul(G.t(), X, out=dWb)

    with torch.cuda.stream(stream):
        for _ in range(2):
            bf16_body()
    torch.cuda.synchronize()
    g_bf16 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_bf16):
        bf16_body()
    timed_replays(g_bf16, args.warmup, other_dw=dWb)
    bf16 = statistics.mean(timed_replays(g_bf16, args.steps, other_dw=dWb))

    # ---- kernel breakdown: CUPTI kernel records (torch.profiler) over extra replays
    kx, kw = [int(v) for v in layer.counts().cpu().numpy()]
    dense = tuple(bool(v) for v in layer.dense_flags().cpu().numpy())   # (grad_W, grad_X) masks, Z-32
    # per-kernel numbers come from a PDL-off capture of the same step: with PDL a
    # kernel launches early and its duration would include the wait on its predecessor
    prev_pdl = i4.int4_set_pdl(False)
    graph_serial = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph_serial):
        step_body()
    cupti = cupti_kernel_times(graph_serial, flush, min(args.steps, 20))
    kernels = {}
    for nm, avg_us in cupti.items():
        kind, amount = algorithmic_work(nm, N, D, C, kx, kw, dense)
        ent = {"avg_us": avg_us, "share": avg_us * 1e-3 / ms if ms else 0.0}
        if kind == "ops" and avg_us > 0:
            ent.update(achieved_tops=amount / (avg_us * 1e-6) / 1e12, frac_int8_peak=amount / (avg_us * 1e-6) / 1e12 / int8_peak)
        elif kind == "bytes" and avg_us > 0 and amount > 0:
            ent.update(achieved_gbs=amount / (avg_us * 1e-6) / 1e9, frac_hbm=amount / (avg_us * 1e-6) / 1e9 / peaks["hbm_gbs"])
        kernels[nm] = ent
    # with the concurrent pair, the pair (not either GEMM alone, which shares the GPU) is the unit
    cands = [nm for nm in kernels if not nm.startswith("memset") and
             not (GROUP in kernels and GROUP in names and nm in ("gemm_i8_dgrad", "gemm_i8_wgrad"))]
    if GROUP in kernels and GROUP not in names:
        cands.remove(GROUP)
    dom = max(cands, key=lambda nm: kernels[nm]["avg_us"],
              default=None)   # None when CUPTI is unavailable (e.g. the run is under ncu)
    roof = None
    if dom is not None:
        roof = dominant_roofline(dom, names, step_body, timed_replays, args, N, D, C, kx, kw, int8_peak, peaks, kernels,
                                 dense)
    i4.int4_set_pdl(prev_pdl)
    gemm_ops = 2.0 * C * D * (N + (N if dense[1] else kx) + (N if dense[0] else kw))
    bwd_gemms = (GROUP,) if (GROUP in kernels and GROUP in names) else ("gemm_i8_dgrad", "gemm_i8_wgrad")
    gemm_us = sum(kernels[nm]["avg_us"] for nm in ("gemm_i8_fwd",) + bwd_gemms if nm in kernels)

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        hx = torch.from_numpy(synth.bf16_bits(x).view(np.int16).copy()).view(torch.bfloat16).pin_memory()
        hw = torch.from_numpy(synth.bf16_bits(w).view(np.int16).copy()).view(torch.bfloat16).pin_memory()
        hg = torch.from_numpy(synth.bf16_bits(g).view(np.int16).copy()).view(torch.bfloat16).pin_memory()
        hY = torch.empty(N, C, dtype=torch.bfloat16).pin_memory()
        hdX = torch.empty(N, D, dtype=torch.bfloat16).pin_memory()
        hdW = torch.empty(C, D, dtype=torch.float32).pin_memory()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2e_ms = []
        for i in range(args.warmup + min(args.steps, 20)):
            flush.zero_()
            torch.cuda.synchronize()
            a0.record()
            X.copy_(hx, non_blocking=True); W.copy_(hw, non_blocking=True); G.copy_(hg, non_blocking=True)
            step_body()
            if world > 1:
                pdist.allreduce_grad_w(dW)
            hY.copy_(Y, non_blocking=True); hdX.copy_(dX, non_blocking=True); hdW.copy_(dW, non_blocking=True)
            a1.record()
            torch.cuda.synchronize()
            if i >= args.warmup:
                e2e_ms.append(a0.elapsed_time(a1))
        t_e2e = pdist.max_over_ranks(statistics.mean(e2e_ms), dev)
        e2e = {"value": 6.0 * N * C * D * world / (t_e2e * 1e-3) / 1e12, "unit": UNIT,
               "h2d_bytes_per_step": int(hx.numel() * 2 + hw.numel() * 2 + hg.numel() * 2),
               "d2h_bytes_per_step": int(hY.numel() * 2 + hdX.numel() * 2 + hdW.numel() * 4),
               "ms_per_step": t_e2e,
               "path": "pinned host X, W, grad_Y -> device; Int4Linear.forward/backward (C ABI); Y, grad_X, grad_W -> pinned host"}

    line = None
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "s8", "data": "synthetic",
                "config": workload_config(args, cfg, world),
                "speedup_vs_bf16_cublas": bf16 / ms, "bf16_cublas_ms_per_step": bf16,
                "gemm_int8_peak_frac": gemm_ops / (gemm_us * 1e-6) / 1e12 / int8_peak if gemm_us else None,
                "kept_items": {"grad_W": kw, "grad_X": kx, "budget": N},
                "dense_masks": {"grad_W": dense[0], "grad_X": dense[1],
                                "note": "deterministic mask: its GEMM ran on the code plane Q (DESIGN.md Z-32)"},
                "roofline": roof, "kernels": kernels, "kernels_timing": "CUPTI kernel records (torch.profiler) over extra flushed replays",
                "gpu_launches": n_launch_ours(names) * args.steps,
                "clocks": clocks.summary(), "e2e": e2e}
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(cfg, args.grad, args.mode)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


KERNEL_NAMES = [("hadamard_quant_kernel", "hadamard_quant"), ("grad_split_kernel", "grad_split"),
                ("lss_sampler_kernel", "lss_sampler"),
                ("compact_kernel", "compact")]
GEMM_EPI = {"0": "gemm_i8_int32", "1": "gemm_i8_fwd", "2": "gemm_i8_dgrad", "3": "gemm_i8_wgrad"}


def short_kernel_name(full):
    if "gemm_i8_kernel<" in full:
        epi = full.split("gemm_i8_kernel<", 1)[1].split(",")[1].strip()
        return GEMM_EPI.get(epi, "gemm_i8")
    for key, short in KERNEL_NAMES:
        if key in full:
            return short
    return None                          # not ours (e.g. the L2-flush memset between timed steps)


def cupti_kernel_times(graph, flush, n):
    """Average device duration (us) of each of our kernels per replay, from the
    CUPTI activity records torch.profiler collects (kernels inside graphs too).
    A concurrent grad_X || grad_W pair also gets the entry GROUP: the average
    per replay of the union of the two kernels' [start, end) intervals."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    acc = {}
    spans = []                                          # (name, start_ns, end_ns) of the two bwd GEMMs
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(n):
            flush.zero_()
            graph.replay()
            torch.cuda.synchronize()
    for ev in prof.events():
        if ev.device_type.name != "CUDA":
            continue
        nm = short_kernel_name(ev.name)
        if nm is None:
            continue
        acc.setdefault(nm, []).append(ev.device_time_total)
    out = {nm: sum(v) / n for nm, v in acc.items()}
    try:
        for ev in prof.profiler.kineto_results.events():
            nm = short_kernel_name(ev.name())
            if nm in ("gemm_i8_dgrad", "gemm_i8_wgrad"):
                spans.append((nm, ev.start_ns(), ev.start_ns() + ev.duration_ns()))
    except Exception:                                   # older profiler API: no group entry
        spans = []
    d = sorted(x for x in spans if x[0] == "gemm_i8_dgrad")
    w = sorted(x for x in spans if x[0] == "gemm_i8_wgrad")
    if d and len(d) == len(w):
        unions = [max(a[2], b[2]) - min(a[1], b[1]) for a, b in zip(d, w)]
        overlap = [min(a[2], b[2]) - max(a[1], b[1]) for a, b in zip(d, w)]
        if min(o / min(a[2] - a[1], b[2] - b[1]) for o, a, b in zip(overlap, d, w)) > 0.2:   # ran concurrently
            out[GROUP] = sum(unions) / len(unions) / 1e3
    return out


GROUP = "gemm_i8_dgrad||gemm_i8_wgrad"                 # the library's trace name of the concurrent pair


def n_launch_ours(names):
    return sum(2 if nm == GROUP else 1 for nm in names if not nm.startswith("memset"))


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
