"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, stage
by stage on identical seeded inputs (SURVEY.md §8(c) parity protocol):
  (i)   codes   X_hat / W_hat: <= 1e-6 of codes differ, none by more than 1
                (reading Z-7); grad_Y hi/lo planes bit-exact
  (ii)  sampler index sets, weight exponents, counts bit-exact
  (iii) INT32 accumulators bit-exact given identical codes
  (iv)  Y, grad_X, grad_W within 1e-5 relative Frobenius of the oracle fed the
        GPU's intermediates
Tolerances are written in each test."""
import numpy as np
import pytest
import torch

import synth
from oracle.lsq_grad import cold_start_step
from oracle import bitsplit as o_bs
from oracle import gemm as o_gemm
from oracle import hadamard as o_had
from oracle import hq as o_hq
from oracle import linear as o_lin
from oracle import lss as o_lss

from gpu_helpers import code_mismatch, rel_frob, same_item_set, to_bf16_cuda, unpack_bits

pytestmark = pytest.mark.gpu

FROB_TOL = 1e-5          # north star: dequantized outputs within 1e-5 rel. Frobenius
CODE_FRAC_TOL = 1e-6     # north star: <= 1e-6 of INT4 codes differ, by at most one level


def p():
    import paper_2306_11987_b200 as mod
    return mod


# ----------------------------------------------------------------------------- (iii)
GEMM_SHAPES = [(128, 64, 64), (300, 256, 1024), (1000, 192, 128), (77, 512, 4096), (129, 128, 48),
               (4096, 3072, 768), (256, 384, 256)]


@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, True)])
@pytest.mark.parametrize("M,N,K", GEMM_SHAPES + [(128, 64, 8192), (512, 256, 3008), (300, 256, 12288),
                                     (1024, 512, 4096)])
def test_gemm_int32_bit_exact(M, N, K, a_mn, b_mn):
    if a_mn and M % 16:
        pytest.skip("MN-major A needs 16-byte rows")
    rng = np.random.default_rng(M * 7 + N + K)
    a = rng.integers(-8, 8, (M, K), dtype=np.int8)
    b = rng.integers(-128, 128, (N, K), dtype=np.int8)
    b[:, :K // 2] = np.clip(b[:, :K // 2], -112, 112)
    A = torch.from_numpy(np.ascontiguousarray(a.T) if a_mn else a).cuda()
    B = torch.from_numpy(np.ascontiguousarray(b.T) if b_mn else b).cuda()
    if K % 16:
        pytest.skip("K must be a multiple of 16")
    acc = torch.full((M, N), -1, dtype=torch.int32, device="cuda")
    p().int4_gemm_s8s8s32(A, B, acc, a_mn_major=a_mn, b_mn_major=b_mn)
    torch.cuda.synchronize()
    ref = o_gemm.int_matmul_abt(a, b)
    assert np.array_equal(acc.cpu().numpy().astype(np.int64), ref)


# ----------------------------------------------------------------------------- (i)
@pytest.mark.parametrize("k", list(range(0, 8)))
@pytest.mark.parametrize("rows,cols", [(200, 256), (64, 1024)])
def test_hadamard_quant_codes(k, rows, cols):
    x = synth.activations(rows, cols, seed=k)
    s = cold_start_step(x)
    X = to_bf16_cuda(x)
    codes = torch.empty(rows, cols, dtype=torch.int8, device="cuda")
    bits = torch.empty(rows, cols // 32, dtype=torch.int32, device="cuda")
    sq = torch.empty(rows, dtype=torch.int32, device="cuda")
    p().hadamard_quant(X, k, s, codes, bits, sq)
    torch.cuda.synchronize()
    oc, om, osq = o_hq.hadamard_quant(x, k, s)
    gc = codes.cpu().numpy()
    nbad, maxdiff = code_mismatch(gc, oc)
    assert maxdiff <= 1 and nbad <= max(CODE_FRAC_TOL * oc.size, 0)
    gm = unpack_bits(bits, cols)
    if nbad == 0:
        assert np.array_equal(gm, om)
        assert np.array_equal(sq.cpu().numpy(), osq)
    else:
        assert (gm != om).sum() <= nbad


def test_hadamard_quant_no_fma_contraction_at_ties():
    # exact .5 ties must round half-to-even identically (Z-1): x chosen so that
    # v = t r is exactly j + 0.5 for a power-of-two r
    k = 2
    s = 0.25                         # r = 2^-1 / 0.25 = 2
    x = np.zeros((4, 64), dtype=np.float32)
    x[:, 0] = np.array([0.75, 1.25, -0.75, 3.25], dtype=np.float32)   # v = 1.5, 2.5, -1.5, 6.5
    X = to_bf16_cuda(x)
    codes = torch.empty(4, 64, dtype=torch.int8, device="cuda")
    p().hadamard_quant(X, k, s, codes)
    oc, _, _ = o_hq.hadamard_quant(x, k, s)
    assert np.array_equal(codes.cpu().numpy(), oc)
    assert codes.cpu().numpy()[:, 0].tolist() == [2, 2, -2, 6]


# ----------------------------------------------------------------------------- forward
def _run_forward(N, D, C, k, y_dtype=torch.float32, seed=0):
    x = synth.activations(N, D, seed=seed)
    w = synth.weights(C, D, seed=seed)
    s_x, s_w = cold_start_step(x), cold_start_step(w)
    layer = p().Int4Linear(N, D, C, k)
    Y = torch.empty(N, C, dtype=y_dtype, device="cuda")
    layer.forward(to_bf16_cuda(x), to_bf16_cuda(w), s_x, s_w, Y)
    torch.cuda.synchronize()
    return x, w, s_x, s_w, layer, Y


@pytest.mark.parametrize("N,D,C,k", [(128, 64, 64, 4), (333, 256, 192, 5), (512, 768, 3072, 5), (256, 1024, 128, 7),
                                     (130, 128, 256, 0)])
def test_forward_parity(N, D, C, k):
    x, w, s_x, s_w, layer, Y = _run_forward(N, D, C, k)
    f = o_lin.forward(x, w, k, s_x, s_w)
    gx, gw = layer.xq.cpu().numpy(), layer.wq.cpu().numpy()
    for g, o in ((gx, f["xq"]), (gw, f["wq"])):
        nbad, maxdiff = code_mismatch(g, o)
        assert maxdiff <= 1 and nbad <= CODE_FRAC_TOL * o.size
    # (iii)+(iv): Y from the GPU codes, exact int acc then fp32 scale
    acc = o_gemm.int_matmul_abt(gx, gw)
    y_ref = acc.astype(np.float64) * (np.float64(np.float32(s_x)) * np.float64(np.float32(s_w)))
    y = Y.cpu().numpy()
    assert rel_frob(y, y_ref) < FROB_TOL
    assert np.array_equal(y, (acc.astype(np.float32) * np.float32(np.float32(s_x) * np.float32(s_w))))
    if np.array_equal(gx, f["xq"]) and np.array_equal(gw, f["wq"]):
        assert rel_frob(y, f["y"]) < FROB_TOL                                # (v) end to end


def test_forward_bf16_output():
    x, w, s_x, s_w, layer, Y = _run_forward(256, 512, 512, 5, torch.bfloat16)
    acc = o_gemm.int_matmul_abt(layer.xq.cpu().numpy(), layer.wq.cpu().numpy())
    y_ref = acc * (np.float64(s_x) * np.float64(s_w))
    assert rel_frob(Y.float().cpu().numpy(), y_ref) < 4e-3          # bf16 output rounding (2^-9)


# ----------------------------------------------------------------------------- backward
def _bwd_case(N, D, C, k, dense=False, mode=0, seed=0, call_id=3, token_offset=0, g=None):
    x, w, s_x, s_w, layer, Y = _run_forward(N, D, C, k, seed=seed)
    if g is None:
        g = synth.grad_output(N, C, seed=seed, dense=dense)
    dX = torch.empty(N, D, dtype=torch.float32, device="cuda")
    dW = torch.empty(C, D, dtype=torch.float32, device="cuda")
    layer.backward(to_bf16_cuda(g), dX, dW, synth.PHILOX_SEED, call_id, token_offset, mode)
    torch.cuda.synchronize()
    return x, w, s_x, s_w, layer, g, dX.cpu().numpy(), dW.cpu().numpy()


def _oracle_from_gpu_codes(layer, s_x, s_w, k):
    return dict(xq=layer.xq.cpu().numpy(), wq=layer.wq.cpu().numpy(),
                x_mask=unpack_bits(layer.x_mask, layer.D), w_mask=unpack_bits(layer.w_mask, layer.D),
                x_sq=layer.x_sqnorm.cpu().numpy().astype(np.int64), k=k,
                s_x=np.float32(s_x), s_w=np.float32(s_w))


def _check_backward(layer, g, s_x, s_w, k, dX, dW, mode, call_id=3, token_offset=0):
    fwd = _oracle_from_gpu_codes(layer, s_x, s_w, k)
    N, C = g.shape
    # (i) bit split: bit-exact planes and norms
    bs = o_bs.bit_split(g, synth.PHILOX_SEED, call_id, token_offset)
    q8 = layer.q8.cpu().numpy().astype(np.int64)
    assert np.array_equal(q8[:N], bs["q"]) and not q8[N].any()             # 8-bit codes; pad row
    assert np.array_equal(16 * bs["hi"].astype(np.int64) + bs["lo"], bs["q"])
    assert np.array_equal(layer.a_sq.cpu().numpy().reshape(2, N), bs["a_sq"])
    assert layer.s_down().cpu().numpy()[0] == bs["s_down"]
    assert np.array_equal(fwd["x_sq"], (fwd["xq"].astype(np.int64) ** 2).sum(1))
    # (ii) sampler: index sets, weight exponents, counts bit-exact
    mw = o_lss.sample_weight_mask(bs["a_sq"], fwd["x_sq"], synth.PHILOX_SEED, call_id, token_offset, mode)
    mx = o_lss.sample_activation_mask(bs["a_sq"], synth.PHILOX_SEED, call_id, token_offset, mode)
    cw, cx = [int(v) for v in layer.counts().cpu().numpy()]
    assert cw == mw["count"] and cx == mx["count"]
    assert same_item_set(layer.items_w.cpu().numpy()[:cw], layer.wexp_w.cpu().numpy()[:cw], mw)
    assert same_item_set(layer.items_x.cpu().numpy()[:cx], layer.wexp_x.cpu().numpy()[:cx], mx)
    pad_w = layer.items_w.cpu().numpy()[cw:(cw + 127) // 128 * 128]
    assert np.all(pad_w == 2 * N)
    # (iv) outputs from identical codes and lists
    dx_ref, _ = o_lin.grad_x_from_items(bs, mx["items"], mx["wexp"], fwd["wq"], fwd["x_mask"], k, fwd["s_w"])
    dw_ref, _ = o_lin.grad_w_from_items(bs, mw["items"], mw["wexp"], fwd["xq"], fwd["w_mask"], k, fwd["s_x"])
    assert rel_frob(dX, dx_ref) < FROB_TOL
    assert rel_frob(dW, dw_ref) < FROB_TOL
    return mw, mx


@pytest.mark.parametrize("mode", [o_lss.MODE_BERNOULLI, o_lss.MODE_KEEP_POSITIVE, o_lss.MODE_NONE])
@pytest.mark.parametrize("dense", [False, True])
def test_backward_parity_cfg1(mode, dense):
    N, D, C, k = 128, 64, 64, 4                                     # BASELINE configs[0]
    x, w, s_x, s_w, layer, g, dX, dW = _bwd_case(N, D, C, k, dense=dense, mode=mode)
    _check_backward(layer, g, s_x, s_w, k, dX, dW, mode)


@pytest.mark.parametrize("N,D,C,k,dense", [(333, 256, 192, 5, True), (1000, 512, 768, 5, False),
                                           (512, 256, 512, 7, True), (256, 128, 256, 6, False),
                                           (640, 192, 320, 3, True)])
def test_backward_parity_shapes(N, D, C, k, dense):
    x, w, s_x, s_w, layer, g, dX, dW = _bwd_case(N, D, C, k, dense=dense, token_offset=17)
    _check_backward(layer, g, s_x, s_w, k, dX, dW, o_lss.MODE_BERNOULLI, token_offset=17)


def test_backward_degenerate_zero_and_single_row():
    N, D, C, k = 256, 128, 128, 5
    g = np.zeros((N, C), dtype=np.float32)
    x, w, s_x, s_w, layer, g, dX, dW = _bwd_case(N, D, C, k, g=g)
    assert not dX.any() and not dW.any()
    assert layer.counts().cpu().numpy().tolist() == [0, 0]
    g = np.zeros((N, C), dtype=np.float32)
    g[37] = synth.grad_output(1, C, dense=True)[0]
    x, w, s_x, s_w, layer, g, dX, dW = _bwd_case(N, D, C, k, g=g)
    _check_backward(layer, g, s_x, s_w, k, dX, dW, o_lss.MODE_BERNOULLI)
    assert not np.delete(dX, 37, axis=0).any()


def test_backward_bf16_grad_x():
    # perf mode (reading Z-24): bf16 grad_X equals the fp32 result rounded once
    N, D, C, k = 512, 256, 512, 5
    x, w, s_x, s_w, layer, g, dX32, dW32 = _bwd_case(N, D, C, k, dense=True)
    dX = torch.empty(N, D, dtype=torch.bfloat16, device="cuda")
    dW = torch.empty(C, D, dtype=torch.float32, device="cuda")
    layer.backward(to_bf16_cuda(g), dX, dW, synth.PHILOX_SEED, 3, 0, 0)
    torch.cuda.synchronize()
    assert np.array_equal(dW.cpu().numpy(), dW32)
    assert rel_frob(dX.float().cpu().numpy(), dX32) < 4e-3


def test_backward_deterministic_bytes():
    N, D, C, k = 512, 256, 512, 5
    runs = [_bwd_case(N, D, C, k, dense=True) for _ in range(2)]
    assert np.array_equal(runs[0][6], runs[1][6]) and np.array_equal(runs[0][7], runs[1][7])


def test_shard_invariance_of_random_streams():
    # Z-20: token t of a shard starting at token_offset draws the same Philox
    # words as global token token_offset + t: the hi/lo planes of the second
    # half of a batch equal those of the full batch computed with offset 0.
    N, D, C, k = 256, 128, 128, 5
    g = synth.grad_output(N, C, dense=True)
    g[0, 0] = np.abs(g).max() * 2          # same amax in both halves' runs below
    g_half = g[N // 2:].copy()
    g_half[0, 0] = g[0, 0]
    _, _, _, _, full, _, _, _ = _bwd_case(N, D, C, k, g=g)
    _, _, _, _, half, _, _, _ = _bwd_case(N // 2, D, C, k, g=g_half, token_offset=N // 2)
    hf = full.q8.cpu().numpy()
    hh = half.q8.cpu().numpy()
    assert np.array_equal(hf[N // 2 + 1:N], hh[1:N // 2])


def test_api_errors_are_loud():
    mod = p()
    X = torch.zeros(128, 96, dtype=torch.bfloat16, device="cuda")
    codes = torch.empty(128, 96, dtype=torch.int8, device="cuda")
    with pytest.raises(mod.I4Error):
        mod.hadamard_quant(X, 6, 0.1, codes)            # 96 % 64 != 0 -> I4_ERR_SHAPE
    with pytest.raises(mod.I4Error):
        mod.hadamard_quant(X[:, :64].contiguous(), 2, -1.0, codes)   # negative step -> I4_ERR_ARG


# ----------------------------------------------------------------------------- full size
@pytest.mark.parametrize("cfg", ["cfg3_bert_large_ffn_up", "cfg2_bert_base_ffn1"])
def test_full_size_sampled_parity(cfg):
    """BASELINE configs at full size in the bench's launch configuration: codes
    and sampler lists in full, outputs on sampled rows the oracle computes one
    by one from the GPU's intermediates."""
    c = synth.CONFIGS[cfg]
    N, D, C, k = c["N"], c["D"], c["C"], c["k"]
    x, w, s_x, s_w, layer, g, dX, dW = _bwd_case(N, D, C, k, dense=False)
    xq, wq = layer.xq.cpu().numpy(), layer.wq.cpu().numpy()
    rows = np.random.default_rng(1).choice(N, 64, replace=False)
    # codes: sampled rows exactly vs oracle
    oc, om, osq = o_hq.hadamard_quant(x[rows], k, s_x)
    nbad, maxdiff = code_mismatch(xq[rows], oc)
    assert maxdiff <= 1 and nbad <= CODE_FRAC_TOL * oc.size    # fraction of the codes compared
    # forward rows
    Y = torch.empty(N, C, dtype=torch.float32, device="cuda")
    layer.forward(to_bf16_cuda(x), to_bf16_cuda(w), s_x, s_w, Y, reuse_weight=True)
    acc = o_gemm.int_matmul_abt(xq[rows], wq)
    y_ref = acc * (np.float64(s_x) * np.float64(s_w))
    assert rel_frob(Y.cpu().numpy()[rows], y_ref) < FROB_TOL
    # backward: full sampler parity, outputs on sampled tokens / channels
    bs = o_bs.bit_split(g, synth.PHILOX_SEED, 3, 0)
    assert np.array_equal(layer.q8.cpu().numpy().astype(np.int64)[:N], bs["q"])
    x_sq = layer.x_sqnorm.cpu().numpy().astype(np.int64)
    mw = o_lss.sample_weight_mask(bs["a_sq"], x_sq, synth.PHILOX_SEED, 3, 0)
    mx = o_lss.sample_activation_mask(bs["a_sq"], synth.PHILOX_SEED, 3, 0)
    cw, cx = [int(v) for v in layer.counts().cpu().numpy()]
    assert (cw, cx) == (mw["count"], mx["count"])
    assert same_item_set(layer.items_w.cpu().numpy()[:cw], layer.wexp_w.cpu().numpy()[:cw], mw)
    assert same_item_set(layer.items_x.cpu().numpy()[:cx], layer.wexp_x.cpu().numpy()[:cx], mx)
    x_mask = unpack_bits(layer.x_mask, D)
    w_mask = unpack_bits(layer.w_mask, D)
    # grad_X rows of sampled tokens
    sel = np.isin(mx["items"] % N, rows)
    dx_ref, _ = o_lin.grad_x_from_items(bs, mx["items"][sel], mx["wexp"][sel], wq, x_mask, k, np.float32(s_w))
    assert rel_frob(dX[rows], dx_ref[rows]) < FROB_TOL
    # grad_W rows of sampled channels
    ch = np.random.default_rng(2).choice(C, 32, replace=False)
    bs_c = dict(bs, hi=bs["hi"][:, ch], lo=bs["lo"][:, ch])
    dw_ref, _ = o_lin.grad_w_from_items(bs_c, mw["items"], mw["wexp"], xq, w_mask[ch], k, np.float32(s_x))
    assert rel_frob(dW[ch], dw_ref) < FROB_TOL


# ----------------------------------------------------------------------------- bit split fast paths
@pytest.mark.parametrize("C", [256, 512, 768, 1024, 3072, 320])
@pytest.mark.parametrize("clamp", [False, True])
def test_bitsplit_unit_paths(C, clamp):
    """grad_split phase 2 for every unit size (C % 1024, 768, 512, 256 and the
    generic row loop), with and without an element landing above 119 after the
    fp32 scaling (reading Z-10 clamp), bit-exact planes and norms."""
    N = 37
    g = synth.grad_output(N, C, seed=C, dense=True)
    g = synth.bf16_bits(g).view(np.uint16).astype(np.uint32)
    g = (g << 16).view(np.float32)                          # exactly representable in bf16
    if clamp:
        a = np.float32(np.max(np.abs(g)) * 1.5)
        for m in range(1, 128):                            # bf16 values above the current max
            cand = (np.uint32((np.float32(a).view(np.uint32) >> 16) + m) << 16).view(np.float32)
            if np.float32(cand * (np.float32(119.0) / cand)) > np.float32(119.0):
                a = cand
                break
        else:
            pytest.skip("no rounding-up bf16 amax near this scale")
        g[5, 7] = -a
        g[11, C - 1] = a
    bs = o_bs.bit_split(g, synth.PHILOX_SEED, 9, 123)
    if clamp:
        assert np.float32(bs["amax"] * (np.float32(119.0) / bs["amax"])) > np.float32(119.0)
    mod = p()
    plan = mod._PlanBuffers(N, C, "cuda")
    xsq = torch.ones(N, dtype=torch.int32, device="cuda")
    mod.bitsplit_lss(to_bf16_cuda(g), xsq, synth.PHILOX_SEED, 9, 123, o_lss.MODE_BERNOULLI, plan.plan)
    torch.cuda.synchronize()
    q8 = plan.q8.cpu().numpy().astype(np.int64)
    assert np.array_equal(q8[:N], bs["q"]) and not q8[N].any()
    assert np.array_equal(plan.a_sq.cpu().numpy().reshape(2, N), bs["a_sq"])


def test_bitsplit_repeated_calls_reuse_counters():
    """grad_split's amax / arrival / pool counters live in plan->scratch (zero on
    first use) and every launch returns them to zero: back-to-back calls on the
    same plan with different grad_Y give the oracle's planes every time."""
    N, C = 300, 1024
    mod = p()
    plan = mod._PlanBuffers(N, C, "cuda")
    xsq = torch.ones(N, dtype=torch.int32, device="cuda")
    for it, scale in enumerate((1.0, 1e-3, 40.0)):
        g = synth.grad_output(N, C, seed=it, dense=True) * scale
        g = (synth.bf16_bits(g).view(np.uint16).astype(np.uint32) << 16).view(np.float32)
        bs = o_bs.bit_split(g, synth.PHILOX_SEED, it, 0)
        mod.bitsplit_lss(to_bf16_cuda(g), xsq, synth.PHILOX_SEED, it, 0, o_lss.MODE_BERNOULLI, plan.plan)
        torch.cuda.synchronize()
        assert np.array_equal(plan.q8.cpu().numpy().astype(np.int64)[:N], bs["q"]), it
        assert not plan.scratch.cpu().numpy()[-8:].any(), "counters not returned to zero"


@pytest.mark.parametrize("mode,dense_g,expect", [(o_lss.MODE_KEEP_POSITIVE, True, (1, 1)), (o_lss.MODE_NONE, True, (1, 1)),
                                                 (o_lss.MODE_BERNOULLI, True, (0, 0))])
def test_dense_path_selection_and_parity(mode, dense_g, expect):
    """Reading Z-32: a deterministic mask (every positive item kept with weight 1)
    makes its GEMM run on the code plane Q (and X_hat); a sampled (binding) mask
    keeps the compacted path.  The device-side choice is visible in the flags and
    both paths give the oracle's gradients."""
    N, D, C, k = 640, 256, 384, 5                          # dense grad_Y: 2N positive items > budget N
    x, w, s_x, s_w, layer, g, dX, dW = _bwd_case(N, D, C, k, dense=dense_g, mode=mode)
    assert tuple(int(v) for v in layer.dense_flags().cpu().numpy()) == expect
    _check_backward(layer, g, s_x, s_w, k, dX, dW, mode)


@pytest.mark.parametrize("N,D,C,k", [(333, 256, 192, 5), (1000, 512, 768, 4)])
def test_dense_path_ragged_tokens(N, D, C, k):
    """The dense form (Z-32) with N not a multiple of the 128-row tile: the tail
    rows of Q / X_hat beyond N read as zeros (TMA bounds), and every token row of
    grad_X is written by the GEMM."""
    x, w, s_x, s_w, layer, g, dX, dW = _bwd_case(N, D, C, k, dense=True, mode=o_lss.MODE_KEEP_POSITIVE)
    assert tuple(int(v) for v in layer.dense_flags().cpu().numpy()) == (1, 1)
    _check_backward(layer, g, s_x, s_w, k, dX, dW, o_lss.MODE_KEEP_POSITIVE)


@pytest.mark.parametrize("dense_g", [True, False])
def test_sampler_16cta_cluster_parity(dense_g):
    """N > 32768 tokens (> 8 K items per CTA) runs the sampler as 16-CTA clusters:
    kept item lists, weight exponents and counts bit-exact against the oracle
    (binding budget with dense grad_Y, non-binding with sparse)."""
    N, C = 40000, 256
    g = synth.grad_output(N, C, seed=7, dense=dense_g)
    g = (synth.bf16_bits(g).view(np.uint16).astype(np.uint32) << 16).view(np.float32)
    xsq_np = np.random.default_rng(3).integers(1, 49 * 64, size=N).astype(np.int32)
    mod = p()
    plan = mod._PlanBuffers(N, C, "cuda")
    xsq = torch.from_numpy(xsq_np).cuda()
    mod.bitsplit_lss(to_bf16_cuda(g), xsq, synth.PHILOX_SEED, 5, 0, o_lss.MODE_BERNOULLI, plan.plan)
    torch.cuda.synchronize()
    bs = o_bs.bit_split(g, synth.PHILOX_SEED, 5, 0)
    assert np.array_equal(plan.a_sq.cpu().numpy().reshape(2, N), bs["a_sq"])
    mw = o_lss.sample_weight_mask(bs["a_sq"], xsq_np.astype(np.int64), synth.PHILOX_SEED, 5, 0)
    mx = o_lss.sample_activation_mask(bs["a_sq"], synth.PHILOX_SEED, 5, 0)
    cw, cx = int(plan.scalars[2].item()), int(plan.scalars[3].item())
    assert cw == mw["count"] and cx == mx["count"]
    assert same_item_set(plan.items_w.cpu().numpy()[:cw], plan.wexp_w.cpu().numpy()[:cw], mw)
    assert same_item_set(plan.items_x.cpu().numpy()[:cx], plan.wexp_x.cpu().numpy()[:cx], mx)
    # the 16-CTA variant is the one that ran, whenever the device can schedule it
    assert mod.lib.int4_sampler_cluster_ctas(N) in (8, 16)
    if mod.lib.int4_sampler_cluster_ctas(N) != 16:
        pytest.skip("16-CTA clusters not schedulable on this device: the 8-CTA sampler ran (checked above)")
