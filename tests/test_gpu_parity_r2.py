"""GPU parity, second set (VERDICT r1 "next round" item 1): backward at the
Hadamard orders k = 0, 1, 2, full-size ViT-B/16 and binding (dense grad_Y)
backwards against the oracle, the token-sharded backward summed over shards
(SURVEY.md §8(e) parity), the stochastic-rounding subnormal corner, and the
device status word (SPEC.md:124 input errors, :339 degenerate).  Same
protocol as test_gpu_parity.py: stage by stage, the oracle fed only inputs
it has verified."""
import numpy as np
import pytest
import torch

import synth
from oracle import bitsplit as o_bs
from oracle import gemm as o_gemm
from oracle import hq as o_hq
from oracle import linear as o_lin
from oracle import lss as o_lss
from oracle.lsq_grad import cold_start_step

from gpu_helpers import code_mismatch, rel_frob, same_item_set, to_bf16_cuda, unpack_bits
from test_gpu_parity import CODE_FRAC_TOL, FROB_TOL, _bwd_case, _check_backward, _oracle_from_gpu_codes, p

pytestmark = pytest.mark.gpu


# ----------------------------------------------------------------------------- k = 0, 1, 2
@pytest.mark.parametrize("k", [0, 1, 2])
@pytest.mark.parametrize("mode,dense_g,expect", [(o_lss.MODE_BERNOULLI, True, (0, 0)),       # binding: sampled path
                                                 (o_lss.MODE_KEEP_POSITIVE, True, (1, 1)),   # deterministic: Q path
                                                 (o_lss.MODE_BERNOULLI, False, (1, 1))])     # non-binding sparse
def test_backward_low_hadamard_orders(k, mode, dense_g, expect):
    """The grad_X / grad_W epilogues compiled for k = 0, 1, 2 (block 1, 2, 4) in
    both operand forms (compacted items and the code plane Q, reading Z-32)."""
    N, D, C = 520, 192, 320
    x, w, s_x, s_w, layer, g, dX, dW = _bwd_case(N, D, C, k, dense=dense_g, mode=mode, token_offset=5, seed=k)
    assert tuple(int(v) for v in layer.dense_flags().cpu().numpy()) == expect
    _check_backward(layer, g, s_x, s_w, k, dX, dW, mode, token_offset=5)


# ----------------------------------------------------------------------------- full size
def _full_size(cfg, dense_g, n_rows=48, n_ch=24, dims=None):
    """BASELINE config at full size in the bench's launch configuration (fp32
    outputs for parity): codes on sampled rows, the bit split in full, both
    sampler lists in full, grad_X on sampled tokens and grad_W on sampled
    channels from the verified intermediates.  dims = (N, D, C, k) overrides cfg."""
    if dims is not None:
        N, D, C, k = dims
    else:
        c = synth.CONFIGS[cfg]
        N, D, C, k = c["N"], c["D"], c["C"], c["k"]
    x, w, s_x, s_w, layer, g, dX, dW = _bwd_case(N, D, C, k, dense=dense_g)
    xq, wq = layer.xq.cpu().numpy(), layer.wq.cpu().numpy()
    rows = np.sort(np.random.default_rng(1).choice(N, n_rows, replace=False))
    oc, _, osq = o_hq.hadamard_quant(x[rows], k, s_x)
    nbad, maxdiff = code_mismatch(xq[rows], oc)
    assert maxdiff <= 1 and nbad <= CODE_FRAC_TOL * oc.size
    if nbad == 0:
        assert np.array_equal(layer.x_sqnorm.cpu().numpy()[rows], osq)
    ow, _, _ = o_hq.hadamard_quant(w, k, s_w)
    nbad, maxdiff = code_mismatch(wq, ow)
    assert maxdiff <= 1 and nbad <= CODE_FRAC_TOL * ow.size
    # bit split in full (bit-exact codes and norms)
    bs = o_bs.bit_split(g, synth.PHILOX_SEED, 3, 0)
    q8 = layer.q8.cpu().numpy()
    assert np.array_equal(q8[:N].astype(np.int64), bs["q"]) and not q8[N].any()
    assert np.array_equal(layer.a_sq.cpu().numpy().reshape(2, N), bs["a_sq"])
    # sampler: both lists in full from the verified norms (x_sqnorm = sum of the codes squared)
    x_sq = layer.x_sqnorm.cpu().numpy().astype(np.int64)
    assert np.array_equal(x_sq, (xq.astype(np.int64) ** 2).sum(1))
    mw = o_lss.sample_weight_mask(bs["a_sq"], x_sq, synth.PHILOX_SEED, 3, 0)
    mx = o_lss.sample_activation_mask(bs["a_sq"], synth.PHILOX_SEED, 3, 0)
    cw, cx = [int(v) for v in layer.counts().cpu().numpy()]
    assert (cw, cx) == (mw["count"], mx["count"])
    assert same_item_set(layer.items_w.cpu().numpy()[:cw], layer.wexp_w.cpu().numpy()[:cw], mw)
    assert same_item_set(layer.items_x.cpu().numpy()[:cx], layer.wexp_x.cpu().numpy()[:cx], mx)
    x_mask = unpack_bits(layer.x_mask, D)
    w_mask = unpack_bits(layer.w_mask, D)
    sel = np.isin(mx["items"] % N, rows)
    dx_ref, _ = o_lin.grad_x_from_items(bs, mx["items"][sel], mx["wexp"][sel], wq, x_mask, k, np.float32(s_w))
    assert rel_frob(dX[rows], dx_ref[rows]) < FROB_TOL
    # tokens without a kept grad_X item are exact zero rows
    untouched = np.setdiff1d(np.arange(N), mx["items"] % N)
    if untouched.size:
        assert not dX[untouched[:256]].any()
    ch = np.sort(np.random.default_rng(2).choice(C, n_ch, replace=False))
    bs_c = dict(bs, hi=bs["hi"][:, ch], lo=bs["lo"][:, ch])
    dw_ref, _ = o_lin.grad_w_from_items(bs_c, mw["items"], mw["wexp"], xq, w_mask[ch], k, np.float32(s_x))
    assert rel_frob(dW[ch], dw_ref) < FROB_TOL
    return layer, mw, mx


@pytest.mark.parametrize("cfg", ["cfg2_bert_base_ffn1", "cfg3_bert_large_ffn_up"])
def test_full_size_binding_dense_grad(cfg):
    """Dense grad_Y: 2N positive items against a budget of N, so A.2 binds and
    both masks are sampled (the compacted-operand path)."""
    layer, mw, mx = _full_size(cfg, dense_g=True)
    assert tuple(int(v) for v in layer.dense_flags().cpu().numpy()) == (0, 0)
    assert mw["count"] < 2 * layer.N and mx["count"] < 2 * layer.N


@pytest.mark.parametrize("cfg", ["cfg4_vit_b16_ffn_down", "cfg4_vit_b16_ffn_up"])
def test_full_size_vit(cfg):
    """ViT-B/16 linears at N = 50432 tokens: 16-CTA sampler clusters (100 K-item
    lists), grad_W split-K over K = 50432 under the FWHT epilogue."""
    _full_size(cfg, dense_g=False)


@pytest.mark.parametrize("cfg,dense_g", [("cfg3_bert_large_qkv", False), ("cfg3_bert_large_ffn_down", False),
                                         ("cfg3_bert_large_qkv", True), ("cfg3_bert_large_ffn_down", True),
                                         ("cfgT_transformer_base_ffn_up", False),
                                         ("cfgT16k_transformer_base_qkv", True)])
def test_full_size_remaining_linears(cfg, dense_g):
    """The rest of the BERT-large layer set and the translation (Transformer-base)
    linears at full size, in both grad_Y regimes (sparse: the bench default, usually
    deterministic masks and the dense code-plane operands; dense: binding budgets)."""
    layer, mw, mx = _full_size(cfg, dense_g=dense_g)
    flags = tuple(int(v) for v in layer.dense_flags().cpu().numpy())
    assert all(f in (0, 1, 2) for f in flags)
    if dense_g:
        assert mw["count"] < 2 * layer.N and mx["count"] < 2 * layer.N


@pytest.mark.parametrize("dense_g", [False, True])
def test_max_tokens_per_call(dense_g):
    """N = 65536 tokens, the largest backward call (reading Z-21: grad_W's INT32
    accumulator bound K_W 128 112 < 2^31; 131072 items on 16-CTA sampler clusters)."""
    _full_size(None, dense_g=dense_g, dims=(65536, 256, 512, 5))


# ----------------------------------------------------------------------------- sharding
def test_token_sharded_backward_sum_equals_oracle_shards():
    """SURVEY.md §8(e) parity: the CUDA operator run on G token shards (each with
    its global token_offset, its own amax and budget) and its grad_W partials
    summed (the all-reduce) equals the oracle's sum over the same emulated shards;
    grad_X shards concatenate."""
    G, Nr, D, C, k = 4, 640, 256, 512, 5
    N = G * Nr
    x = synth.activations(N, D, seed=11)
    w = synth.weights(C, D, seed=11)
    g = synth.grad_output(N, C, seed=11, dense=True)
    s_x, s_w = cold_start_step(x), cold_start_step(w)
    dW_sum = torch.zeros(C, D, dtype=torch.float64, device="cuda")
    dw_ref = np.zeros((C, D))
    dX_all, dx_ref = [], []
    for r in range(G):
        sl = slice(r * Nr, (r + 1) * Nr)
        layer = p().Int4Linear(Nr, D, C, k)
        Y = torch.empty(Nr, C, dtype=torch.float32, device="cuda")
        layer.forward(to_bf16_cuda(x[sl]), to_bf16_cuda(w), s_x, s_w, Y)
        dX = torch.empty(Nr, D, dtype=torch.float32, device="cuda")
        dW = torch.empty(C, D, dtype=torch.float32, device="cuda")
        layer.backward(to_bf16_cuda(g[sl]), dX, dW, synth.PHILOX_SEED, call_id=7, token_offset=r * Nr)
        torch.cuda.synchronize()
        dW_sum += dW.double()
        dX_all.append(dX.cpu().numpy())
        # oracle on the same shard, fed the GPU's codes once they are verified
        f = o_lin.forward(x[sl], w, k, s_x, s_w)
        for got, ref in ((layer.xq.cpu().numpy(), f["xq"]), (layer.wq.cpu().numpy(), f["wq"])):
            nbad, maxdiff = code_mismatch(got, ref)
            assert maxdiff <= 1 and nbad <= CODE_FRAC_TOL * ref.size
        fwd = _oracle_from_gpu_codes(layer, s_x, s_w, k)
        b = o_lin.backward(g[sl], fwd, synth.PHILOX_SEED, 7, token_offset=r * Nr)
        dw_ref += b["dw"]
        dx_ref.append(b["dx"])
    assert rel_frob(dW_sum.cpu().numpy(), dw_ref) < FROB_TOL
    assert rel_frob(np.concatenate(dX_all), np.concatenate(dx_ref)) < FROB_TOL


# ----------------------------------------------------------------------------- SR corner
def test_sr_subnormal_products_bit_exact():
    """Reading Z-10 computes v = fl32(g r8) in fp32; when |g| r8 is subnormal
    (|g| / amax < 2^-126 / 119) v is a subnormal or flushes to 0 and the SR
    rounds A = ceil(v 2^32) of that value.  The kernel forms the same
    fl32(g r8) and scales by 2^32 exactly afterwards, so codes are
    bit-identical to the oracle across the subnormal range."""
    N, C = 64, 512
    rng = np.random.default_rng(5)
    e = rng.integers(-30, 1, size=(N, C)).astype(np.float64)
    g = (rng.choice([-1.0, 1.0], size=(N, C)) * rng.random((N, C)) * 2.0 ** e * 1e-2).astype(np.float32)
    g[0, 0] = 3.0e38                        # amax near the bf16 maximum: r8 ~ 4e-37, |g| r8 in [4e-48, 4e-39]
    g = (synth.bf16_bits(g).view(np.uint16).astype(np.uint32) << 16).view(np.float32)
    bs = o_bs.bit_split(g, synth.PHILOX_SEED, 2, 0)
    r8 = np.float32(119.0) / np.float32(np.abs(g).max())
    prod = np.abs(g[1:]) * r8                              # fp32 products, as the oracle forms them
    assert (prod[prod > 0] < np.float32(2.0 ** -126)).mean() > 0.9 and (prod == 0).any()
    mod = p()
    plan = mod._PlanBuffers(N, C, "cuda")
    xsq = torch.ones(N, dtype=torch.int32, device="cuda")
    mod.bitsplit_lss(to_bf16_cuda(g), xsq, synth.PHILOX_SEED, 2, 0, o_lss.MODE_BERNOULLI, plan.plan)
    torch.cuda.synchronize()
    assert np.array_equal(plan.q8.cpu().numpy().astype(np.int64)[:N], bs["q"])
    assert np.array_equal(plan.a_sq.cpu().numpy().reshape(2, N), bs["a_sq"])


def test_sr_low_half_draws_bit_exact():
    """Reading Z-20: an element's 32-bit uniform is (purpose-1 half) 2^16 +
    (purpose-4 half); the kernel draws the purpose-4 block only when the high
    half leaves the decision open (the low word of A + half1 2^16 above
    0xFFFF0000).  At 2^-16 per element a 4096 x 2048 gradient has ~100 such
    elements: count them from the oracle's streams and require bit-exact codes
    and norms."""
    N, C = 4096, 2048
    g = synth.grad_output(N, C, dense=True)
    bs = o_bs.bit_split(g, synth.PHILOX_SEED, 6, 3)
    from oracle import philox as o_ph
    u = o_ph.sr_uniforms(synth.PHILOX_SEED, 6, 3, N, C).astype(np.int64)
    _, _, r8 = o_bs.scales(g)
    v = np.clip(g * r8, np.float32(-119), np.float32(119))
    A = np.ceil(v.astype(np.float64) * 2.0 ** 32).astype(np.int64)
    hi = (u >> 16) << 16
    open_ = np.floor_divide(A + hi, 1 << 32) != np.floor_divide(A + hi + 0xFFFF, 1 << 32)
    assert open_.sum() >= 20, open_.sum()
    mod = p()
    plan = mod._PlanBuffers(N, C, "cuda")
    xsq = torch.ones(N, dtype=torch.int32, device="cuda")
    mod.bitsplit_lss(to_bf16_cuda(g), xsq, synth.PHILOX_SEED, 6, 3, o_lss.MODE_BERNOULLI, plan.plan)
    torch.cuda.synchronize()
    q = plan.q8.cpu().numpy().astype(np.int64)[:N]
    assert np.array_equal(q, bs["q"])
    assert np.array_equal(plan.a_sq.cpu().numpy().reshape(2, N), bs["a_sq"])


# ----------------------------------------------------------------------------- status word
def test_status_word_nonfinite_and_zero_grad():
    N, D, C, k = 256, 128, 256, 5
    mod = p()
    x = synth.activations(N, D)
    w = synth.weights(C, D)
    s_x, s_w = cold_start_step(x), cold_start_step(w)
    layer = mod.Int4Linear(N, D, C, k)
    Y = torch.empty(N, C, dtype=torch.float32, device="cuda")
    dX = torch.empty(N, D, dtype=torch.float32, device="cuda")
    dW = torch.empty(C, D, dtype=torch.float32, device="cuda")
    g = synth.grad_output(N, C, dense=True)
    # clean inputs: no bit
    layer.forward(to_bf16_cuda(x), to_bf16_cuda(w), s_x, s_w, Y)
    layer.backward(to_bf16_cuda(g), dX, dW, synth.PHILOX_SEED, 1)
    torch.cuda.synchronize()
    assert int(layer.status()[0]) == 0
    # Inf in X: the forward flags it
    xb = x.copy()
    xb[17, 33] = np.inf
    layer.forward(to_bf16_cuda(xb), to_bf16_cuda(w), s_x, s_w, Y)
    torch.cuda.synchronize()
    assert int(layer.status()[0]) & mod.STATUS_NONFINITE
    layer.clear_status()
    # NaN in W: flagged too (W is quantized by the same launch)
    wb = w.copy()
    wb[3, 5] = np.nan
    layer.forward(to_bf16_cuda(x), to_bf16_cuda(wb), s_x, s_w, Y)
    torch.cuda.synchronize()
    assert int(layer.status()[0]) & mod.STATUS_NONFINITE
    layer.clear_status()
    # NaN in grad_Y: bit 0, the tensor treated as zero -> zero gradients, nothing kept
    layer.forward(to_bf16_cuda(x), to_bf16_cuda(w), s_x, s_w, Y)
    gb = g.copy()
    gb[100, 7] = np.nan
    layer.backward(to_bf16_cuda(gb), dX, dW, synth.PHILOX_SEED, 1)
    torch.cuda.synchronize()
    assert int(layer.status()[0]) == mod.STATUS_NONFINITE
    assert not dX.any() and not dW.any()
    assert layer.counts().cpu().numpy().tolist() == [0, 0]
    assert float(layer.s_down()[0]) == 0.0
    layer.clear_status()
    # -Inf in grad_Y: the same
    gb = g.copy()
    gb[0, 0] = -np.inf
    layer.backward(to_bf16_cuda(gb), dX, dW, synth.PHILOX_SEED, 1)
    torch.cuda.synchronize()
    assert int(layer.status()[0]) == mod.STATUS_NONFINITE
    layer.clear_status()
    # all-zero grad_Y: the degenerate flag, zero gradients
    layer.backward(to_bf16_cuda(np.zeros((N, C), np.float32)), dX, dW, synth.PHILOX_SEED, 1)
    torch.cuda.synchronize()
    assert int(layer.status()[0]) == mod.STATUS_ZERO_GRAD
    assert not dX.any() and not dW.any()
    layer.clear_status()
    # and a clean call afterwards is bit-exact again
    layer.backward(to_bf16_cuda(g), dX, dW, synth.PHILOX_SEED, 1)
    torch.cuda.synchronize()
    assert int(layer.status()[0]) == 0
    _check_backward(layer, g, s_x, s_w, k, dX.cpu().numpy(), dW.cpu().numpy(), o_lss.MODE_BERNOULLI, call_id=1)


# ----------------------------------------------------------------------------- operand form 2
@pytest.mark.parametrize("N,D,C,seed,k", [(2048, 256, 2048, 0, 5), (4096, 256, 2048, 2, 5), (4096, 256, 2048, 1, 3)])
def test_binding_few_sampled_dense_plus_correction(N, D, C, seed, k):
    """Reading Z-33: a binding budget that leaves few items sampled (sparse grad_Y
    just over the budget: these seeds give 18-220 sampled items, found with the
    oracle's A.2) runs the dense Q / X_hat GEMMs plus correction rows -- grad_W gets
    a -1 row per sampled item and a +2^e row per kept one, grad_X takes the sampled
    tokens' rows from their kept items.  Gradients equal the oracle's item-by-item
    sums; the kept lists are unchanged."""
    x, w, s_x, s_w, layer, g, dX, dW = _bwd_case(N, D, C, k, dense=False, seed=seed, token_offset=0)
    assert tuple(int(v) for v in layer.dense_flags().cpu().numpy()) == (2, 2)
    _check_backward(layer, g, s_x, s_w, k, dX, dW, o_lss.MODE_BERNOULLI)


def test_form2_bf16_grad_x_matches_fp32():
    N, D, C, k = 2048, 256, 2048, 5
    x, w, s_x, s_w, layer, g, dX32, dW32 = _bwd_case(N, D, C, k, dense=False, seed=0)
    dX = torch.empty(N, D, dtype=torch.bfloat16, device="cuda")
    dW = torch.empty(C, D, dtype=torch.float32, device="cuda")
    layer.backward(to_bf16_cuda(g), dX, dW, synth.PHILOX_SEED, 3, 0, 0)
    torch.cuda.synchronize()
    assert tuple(int(v) for v in layer.dense_flags().cpu().numpy()) == (2, 2)
    assert np.array_equal(dW.cpu().numpy(), dW32)
    assert rel_frob(dX.float().cpu().numpy(), dX32) < 4e-3
