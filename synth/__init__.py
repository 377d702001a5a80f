"""Seeded synthetic inputs shared by the oracle-side tests, the CUDA-side tests
and bench.py.  This module holds NONE of the method's arithmetic (no
Hadamard, quantization, splitting or sampling): only random tensors with the
structure of the paper's workloads, as stated in DESIGN.md "Input recipe".

  X      bf16 N(0,1) with ceil(0.005 D) seeded outlier columns scaled x30:
         "only a few columns of X are significantly larger" (Fig. 1).
  W      bf16 N(0, 0.02^2) (BERT initialisation scale).
  grad_Y bf16, "few rows large, most close to zero" (Fig. 2):
         per-token scale r_t = 1 for 5 % of tokens, 1e-3 for 90 %, 0 for 5 %
         (padding), times lognormal(0, 0.5) jitter; entries r_t N(0,1).
         dense variant: r_t = 1 for every token.
  steps  not generated here: they are operator inputs set by the A.4 cold-start
         rule, which is method arithmetic -- tests take it from
         oracle.lsq_grad.cold_start_step, bench.py from the library's
         lsq_cold_start_step kernel (bit-identical, tests/test_gpu_lsq_grad.py).

Arrays are numpy float32 holding exactly-representable bf16 values, so the
same bytes can be handed to the oracle (as float64) and to the GPU (as bf16).
"""
import numpy as np

DATA_SEED = 2306
PHILOX_SEED = 0x0000000230611987


def _to_bf16_values(a):
    """Round-to-nearest-even float32 -> bf16, returned as float32 values."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    u = ((u + rounding) >> 16) << 16
    return (u.astype(np.uint32)).view(np.float32)


def bf16_bits(a):
    """uint16 bit patterns of bf16-representable float32 values (for upload)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    return (a.view(np.uint32) >> 16).astype(np.uint16)


def activations(N, D, seed=DATA_SEED, outlier_frac=0.005, outlier_scale=30.0):
    rng = np.random.default_rng([seed, 1, N, D])
    x = rng.standard_normal((N, D), dtype=np.float32)
    n_out = int(np.ceil(outlier_frac * D)) if outlier_scale != 1.0 else 0
    if n_out:
        cols = rng.choice(D, size=n_out, replace=False)
        x[:, cols] *= np.float32(outlier_scale)
    return _to_bf16_values(x)


def weights(C, D, seed=DATA_SEED, std=0.02):
    rng = np.random.default_rng([seed, 2, C, D])
    return _to_bf16_values(rng.standard_normal((C, D), dtype=np.float32) * np.float32(std))


def grad_output(N, C, seed=DATA_SEED, dense=False):
    rng = np.random.default_rng([seed, 3, N, C, int(dense)])
    if dense:
        r = np.ones(N, dtype=np.float32)
    else:
        kind = rng.random(N)
        r = np.where(kind < 0.05, 1.0, np.where(kind < 0.95, 1e-3, 0.0)).astype(np.float32)
    r = r * rng.lognormal(0.0, 0.5, N).astype(np.float32)
    g = rng.standard_normal((N, C), dtype=np.float32) * r[:, None]
    return _to_bf16_values(g)


# BASELINE.json configs (shapes only; k per SURVEY.md §8(d)).  cfgT: the
# translation layers north_star names (Transformer-base d = 512, FFN 2048, a
# 4096-token batch ~ fairseq max-tokens) and the
# 16384-token variant SURVEY.md §8(d) asks for.
CONFIGS = {
    "cfg1": dict(N=128, D=64, C=64, k=4),
    "cfg2_bert_base_ffn1": dict(N=4096, D=768, C=3072, k=5),
    "cfg3_bert_large_qkv": dict(N=8192, D=1024, C=3072, k=5),
    "cfg3_bert_large_ffn_up": dict(N=8192, D=1024, C=4096, k=5),
    "cfg3_bert_large_ffn_down": dict(N=8192, D=4096, C=1024, k=5),
    "cfg4_vit_b16_ffn_up": dict(N=50432, D=768, C=3072, k=5),
    "cfg4_vit_b16_ffn_down": dict(N=50432, D=3072, C=768, k=5),
    "cfgT_transformer_base_qkv": dict(N=4096, D=512, C=1536, k=5),
    "cfgT_transformer_base_ffn_up": dict(N=4096, D=512, C=2048, k=5),
    "cfgT_transformer_base_ffn_down": dict(N=4096, D=2048, C=512, k=5),
    "cfgT16k_transformer_base_qkv": dict(N=16384, D=512, C=1536, k=5),
    "cfgT16k_transformer_base_ffn_up": dict(N=16384, D=512, C=2048, k=5),
    "cfgT16k_transformer_base_ffn_down": dict(N=16384, D=2048, C=512, k=5),
}

# Stacks of linears (one training step = every linear's forward, then every
# backward in reverse layer order).  cfg5 = BASELINE configs[4]: the 24-layer
# BERT-large linear stack (QKV, FFN-up, FFN-down per layer),
# N tokens per GPU (token-sharded data parallelism, weak scaling).
STACKS = {
    "cfg5_bert_large_stack": dict(layers=24, N=8192, k=5,
                                  linears=[("qkv", 1024, 3072), ("ffn_up", 1024, 4096), ("ffn_down", 4096, 1024)]),
    "cfgT_transformer_base_stack": dict(layers=6, N=4096, k=5,
                                        linears=[("qkv", 512, 1536), ("ffn_up", 512, 2048), ("ffn_down", 2048, 512)]),
}
