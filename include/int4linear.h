/*
 * int4linear.h -- C ABI of the B200-native INT4 quantized linear operator of
 * arXiv 2306.11987 ("Training Transformers with 4-bit Integers": HQ + LSS).
 *
 * Problem (Eq. 1): Y = X W^T with X in R^{N x D} (N = S T
 * tokens), W in R^{C x D}.  Forward = Procedure HQ-MM;
 * backward = the STE gradients of Eq. 4 with the "type 3"
 * MMs computed by Procedure LSS-MM.
 *
 * Conventions common to every entry point
 *   - All tensors are row-major and contiguous.  Every pointer is a DEVICE
 *     pointer unless stated otherwise; every pointer must be 16-byte aligned.
 *   - X, W and grad_Y are bf16 (PAPER.md:56 uses 16-bit floats; bf16 matches the
 *     cuBLAS BF16 baseline).  Step sizes are fp32 host scalars.
 *   - Ownership: the caller allocates EVERY buffer (outputs, caches, plans,
 *     workspace); the library never allocates device memory and keeps no
 *     per-call state.  Buffer sizes are stated per field below.  Library-owned
 *     global state: per-device caches of launch parameters (SM count, occupancy,
 *     the sampler's cluster size) and the PDL switch (int4_set_pdl).  The
 *     library creates no streams: every launch goes to `stream`.
 *   - No environment variables are read by the library.
 *   - Execution: stream-ordered and asynchronous on `stream` (a cudaStream_t
 *     passed as void*; NULL = legacy default stream).  No entry point
 *     synchronises the device or reads device memory from the host, so the
 *     sequence is CUDA-graph capturable.  Sampled counts stay on the device.
 *   - Errors: return codes, never abort.  On a non-OK status nothing has been
 *     launched, except I4_ERR_CUDA (a launch failed; see int4_last_error()).
 *   - Integer codes are int8 holding INT4 values: X_hat, W_hat in [-7, 7]
 *     (Q_N = Q_P = 7); grad_up in [-7, 7]; grad_down in [-8, 7].
 *   - Clamp masks are bit-packed uint32 words [rows, cols / 32]; bit j of word
 *     w is column 32 w + j (1 = inside [-Q_N, Q_P]).
 *   - Shape limits: cols % 64 == 0 for D and C; D % 2^k == 0;
 *     0 <= k <= 7; backward N <= 65536 (INT32 accumulator bound of the grad_W
 *     GEMM, reading Z-21).
 *   - Determinism: identical inputs and identical (seed, call_id, token_offset)
 *     give byte-identical outputs.  Philox4x32-10 streams use GLOBAL token
 *     indices (token_offset + t), so a token-sharded run draws the same numbers
 *     as an unsharded one (reading Z-20).
 */
#ifndef INT4LINEAR_H
#define INT4LINEAR_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define I4_API __attribute__((visibility("default")))
#else
#define I4_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    I4_OK = 0,
    I4_ERR_SHAPE = 1,        /* shape / k out of the supported set            */
    I4_ERR_ALIGN = 2,        /* pointer not 16-byte aligned                   */
    I4_ERR_ARG = 3,          /* step size <= 0 or non-finite, bad enum, NULL  */
    I4_ERR_UNSUPPORTED = 4,  /* device is not sm_100 (tcgen05 kind::i8)       */
    I4_ERR_WORKSPACE = 5,    /* ws_bytes smaller than the *_workspace_size    */
    I4_ERR_CUDA = 6          /* a CUDA API call or kernel launch failed       */
} i4_status;

typedef enum { I4_OUT_F32 = 0, I4_OUT_BF16 = 1 } i4_out_dtype;

typedef enum {
    I4_LSS_BERNOULLI = 0,      /* §4.2 + A.2 probabilities, dyadic weights (Z-17) */
    I4_LSS_KEEP_POSITIVE = 1,  /* A.6: keep every item with score > 0 */
    I4_LSS_NONE = 2            /* no sampling: all 2N items, the exact BS product  */
} i4_lss_mode;

/* Forward cache ("X_hat and W_hat have been already calculated
 * in forward propagation").  Written by int4_linear_fwd, read by
 * int4_linear_bwd.  Device buffers, caller-allocated:
 *   xq       int8  [N, D]      X_hat = <XH>_{s_X}
 *   wq       int8  [C, D]      W_hat = <WH>_{s_W} (read K-major by the forward GEMM and
 *                              MN-major by the grad_X GEMM: never transposed in memory)
 *   x_mask   uint32 [N, D/32]  I_X (on XH / s_X, reading Z-8)
 *   w_mask   uint32 [C, D/32]  I_W
 *   x_sqnorm int32 [N]         sum_d X_hat[t, d]^2 (leverage scores)
 *   x_delta  float [N, D]      nullable: delta_X = <v> - I_X o v of the quantizer input
 *                              v = XH / s_X (A.3, reading Z-27), exact
 *                              in fp32; needed only for the step-size gradients
 *   w_delta  float [C, D]      nullable: delta_W, the same for W
 *   dev_status int32 [1]      nullable: device status word.  The forward ORs in
 *                              I4_STATUS_NONFINITE when an element of X (or of W,
 *                              when it is quantized) is Inf / NaN or its block
 *                              transform overflows fp32 ("input error",
 *                              which a stream-ordered call cannot return
 *                              synchronously).  The codes of such a block are not
 *                              meaningful.  The library only ORs bits in; the caller
 *                              zeroes the word and reads it when it wants to (like
 *                              a GradScaler's found-inf flag).
 * Host scalars: N, D, C, k, s_x, s_w are filled by int4_linear_fwd.  Set
 * w_valid = 1 to reuse wq / w_mask (/ w_delta) from a previous call with the
 * same W and s_w (one weight quantization per weight version); the library
 * never changes w_valid. */
typedef struct {
    int8_t* xq;
    int8_t* wq;
    uint32_t* x_mask;
    uint32_t* w_mask;
    int32_t* x_sqnorm;
    int64_t N, D, C;
    int32_t k;
    float s_x, s_w;
    int32_t w_valid;
    float* x_delta;
    float* w_delta;
    int32_t* dev_status;
} i4_fwd_cache;

/* Bits of the device status words (i4_fwd_cache::dev_status, i4_lss_plan::dev_status). */
#define I4_STATUS_NONFINITE 1   /* an input element was Inf / NaN                  */
#define I4_STATUS_ZERO_GRAD 2   /* grad_Y was all zero ("degenerate"): s_down = 0    */

/* Bit-split + sampling plan (Procedure LSS-MM steps 1-4).  Device buffers,
 * caller-allocated, written by bitsplit_lss:
 *   q8       int8  [N+1, C]    the 8-bit stochastically rounded codes q = 16 hi + lo of
 *                              grad_Y / s_down (|q| <= 119, reading Z-9); the bit split
 *                              (Eq. 5) is q's high half hi = floor((q + 8) / 16) and low
 *                              half lo = q - 16 hi (Z-11), split on the fly where a
 *                              half-row is needed; row N = zeros
 *   a_sq     int32 [2N]        sum_c code^2 per half-row (unscaled codes hi, lo)
 *   amax_bits uint32 [1]       out: bf16 bit pattern of max |grad_Y|
 *   s_down   float [1]         out: s_down = amax / 119 (s_up = 16 s_down), reading Z-9
 *   scratch  uint32 [2048]     scratch of the fused amax pass: ZERO-INITIALISE before the
 *                              first call; every call leaves it zero again (its last words
 *                              hold the amax word and the CTA arrival / departure counters)
 *   items_w  int32 [2N + 128]  kept items of the grad_W mask (ids h*N + t) in token-major
 *                              order (slot 2t + h, like items_x), padded with the
 *                              sentinel 2N up to a multiple of 128
 *   wexp_w   int8  [2N + 128]  log2 of each kept item's weight (~ m_i / p_i)
 *   count_w  int32 [1]         number of kept items (device)
 *   items_x, wexp_x, count_x   the same for the grad_X mask (a token's two items are
 *                              adjacent rows of the grad_X GEMM)
 *   x_touched uint8 [N]        1 if token t has a kept grad_X item
 *   grad_s   float [2]         nullable out (int4_linear_bwd): the LSQ step-size gradients
 *                              {grad s_X, grad s_W} (A.3; readings
 *                              Z-27..Z-29), computed when the cache holds x_delta and w_delta
 *   n_elem_x, n_elem_w         host: N_X, N_W of g(s) = 1/sqrt(Q_P N) (0 = this call's
 *                              N*D and C*D; a token-sharded caller passes the global counts)
 *   dw_multicast float [C, D]  nullable (int4_linear_bwd): multicast (NVLS) address of a
 *                              symmetric grad_W buffer spanning the data-parallel ranks (e.g.
 *                              torch symmetric memory's multicast_ptr).  When set, the grad_W
 *                              epilogue reduces each finished tile into EVERY rank's copy with
 *                              multimem.red.add.f32 instead of storing to dW: the all-reduce of
 *                              grad_W happens inside the GEMM, tile by tile (
 *                              PAPER.md:978).  The caller zeroes the buffer on every rank before
 *                              the backward and synchronises the ranks after it before reading.
 *                              fp32 sums of G addends onto zero: bit-identical to a serial sum
 *                              for G <= 2, addition order of the switch otherwise; subnormal
 *                              sums flush to zero.  dW is not written in this mode.
 *   dev_status int32 [1]       nullable: device status word, bits ORed in by the backward:
 *                              I4_STATUS_NONFINITE when grad_Y holds an Inf / NaN (the
 *                              tensor is then treated as all-zero: codes 0, s_down = 0, no
 *                              item kept, grad_X = grad_W = 0 -- the caller must check the
 *                              word, like a GradScaler's found-inf flag, and skip the step);
 *                              I4_STATUS_ZERO_GRAD when grad_Y is all zero (a valid,
 *                              degenerate call: zero gradients). */
typedef struct {
    int8_t* q8;
    int32_t* a_sq;
    uint32_t* amax_bits;
    float* s_down;
    uint32_t* scratch;
    int32_t* items_w;
    int8_t* wexp_w;
    int32_t* count_w;
    int32_t* items_x;
    int8_t* wexp_x;
    int32_t* count_x;
    uint8_t* x_touched;
    float* grad_s;
    int64_t n_elem_x, n_elem_w;
    int32_t* dev_status;
    float* dw_multicast;
} i4_lss_plan;

/* F1+F2 / F3: block-Hadamard transform + LSQ quantize of a bf16 matrix
 * (Procedure HQ-MM steps 1-2; Eq. 2).
 *   x_bf16      [rows, cols] input
 *   k           Hadamard block exponent, block 2^k
 *   step        LSQ step size s > 0
 *   codes       int8 [rows, cols] out: clamp(round_half_even(v), -7, 7) with
 *               v = fl32(fl32(x H_pm1) * fl32(2^{-k/2} / s))   (readings Z-1, Z-4, Z-7)
 *   clamp_bits  uint32 [rows, cols/32] out, nullable: 1(-7 <= v <= 7)
 *   row_sqnorm  int32 [rows] out, nullable: sum of code^2 per row */
I4_API i4_status hadamard_quant(const void* x_bf16, int64_t rows, int64_t cols, int32_t k, float step,
                         int8_t* codes, uint32_t* clamp_bits, int32_t* row_sqnorm, void* stream);

/* Forward HQ-MM: quantizes X (and W unless cache->w_valid)
 * into `cache`, then Y = s_X s_W (X_hat W_hat^T) with an INT32 tcgen05 GEMM
 * and a dequantizing epilogue fl32(acc) * fl32(s_x s_w) (reading Z-22).
 *   X [N, D] bf16, W [C, D] bf16, Y [N, C] fp32 or bf16 (y_dtype). */
I4_API i4_status int4_linear_fwd(const void* X, const void* W, int64_t N, int64_t D, int64_t C, int32_t k,
                          float s_x, float s_w, void* Y, i4_out_dtype y_dtype, i4_fwd_cache* cache,
                          void* stream);

/* LSS-MM steps 1-4: per-tensor amax, stochastic
 * 8-bit code, bit split (Eq. 5), integer leverage scores of both masks
 * (PAPER.md:296 with b = x_sqnorm, :365), A.2 probabilities (PAPER.md:606-610,
 * budget N per mask), Philox Bernoulli masks with dyadic weights, compaction.
 * The 8-bit code is floor-form stochastic rounding (reading Z-10):
 *   q = floor((ceil(v 2^32) + u) / 2^32), v = clamp(fl32(dY r8), -119, 119),
 * u = (16-bit half L mod 8 of Philox block L/8, purpose 1) << 16 | (the same half
 * of purpose 4), L = (token_offset + t) C + c (Z-20).
 *   dY [N, C] bf16; x_sqnorm int32 [N] (from the forward cache; may be NULL
 *   only for mode I4_LSS_NONE).  seed/call_id/token_offset select the Philox
 *   streams (Z-20).  Outputs in *plan (see i4_lss_plan). */
I4_API i4_status bitsplit_lss(const void* dY, int64_t N, int64_t C, const int32_t* x_sqnorm, uint64_t seed,
                       uint32_t call_id, int64_t token_offset, i4_lss_mode mode, const i4_lss_plan* plan,
                       void* stream);

/* Full LSS-MM backward (Eq. 4):
 *   grad_X = [I_X o (s_W sum_kept w_i s_h code_i W_hat)] H^T   -> dX [N, D]
 *   grad_W = s_X [(sum_kept w_i s_h code_i (x) X_hat_t) o I_W] H^T -> dW [C, D] fp32
 * Runs bitsplit_lss into *plan, then the compaction and the two INT32 GEMMs
 * whose epilogues apply scale, mask and the inverse transform (reading Z-23).
 * dX is fp32 (dx_dtype = I4_OUT_F32, parity mode) or bf16 (I4_OUT_BF16, perf
 * mode as the cuBLAS BF16 baseline; reading Z-24); dW stays fp32 (the data-
 * parallel all-reduce operand).  ws: device scratch of
 * int4_bwd_workspace_size(N, D, C) bytes.
 * Step-size gradients (A.3): if plan->grad_s is non-NULL and the cache holds
 * x_delta and w_delta, the two GEMM epilogues also reduce sum(acc o delta) over
 * their tiles (fp32 per 32-column chunk, fp64 across chunks, per-CTA partials)
 * and a final one-CTA launch writes
 *   grad_s[0] = g(N_X) s_W s_down sum_{kept i} w_i sum_d acc_i[d] delta_X[t_i, d]
 *   grad_s[1] = g(N_W) s_X s_down sum_{c,d} acc_W[c, d] delta_W[c, d]
 * (reading Z-28: the partner step size is included, the sum runs over all
 * elements).  Deterministic: fixed tile-to-CTA assignment and fixed-order sums. */
I4_API i4_status int4_linear_bwd(const void* dY, const i4_fwd_cache* cache, uint64_t seed, uint32_t call_id,
                                 int64_t token_offset, i4_lss_mode mode, const i4_lss_plan* plan, void* dX,
                                 i4_out_dtype dx_dtype, float* dW, void* ws, size_t ws_bytes, void* stream);

/* Cold-start step size (A.4; reading Z-25): step = fl32(2 mean|x| /
 * sqrt(Q_P)) over the n bf16 values of x_bf16 (one fixed-order fp64 reduction,
 * deterministic).  step: device float out.  ws: zero-initialised device scratch of
 * lsq_cold_start_workspace_size() bytes, left zeroed on return. */
I4_API i4_status lsq_cold_start_step(const void* x_bf16, int64_t n, float* step, void* ws, size_t ws_bytes,
                                     void* stream);
I4_API size_t lsq_cold_start_workspace_size(void);

/* Adaptive Hadamard block size (A.5; reading Z-30): for every
 * k in [k_min, k_max] the reconstructions X_bar_k = s_X <XH>_{s_X} H^T and W_bar_k
 * (the forward path's quantizer) are compared with X and W;
 *   mse[2k] = MSE(X_bar_k, X), mse[2k+1] = MSE(W_bar_k, W)   (device double [16]),
 *   *k_best = argmin_k mse[2k] mse[2k+1], ties to the smaller k (device int32).
 * X [N, D], W [C, D] bf16; D % 64 == 0, D % 2^k_max == 0, 0 <= k_min <= k_max <= 7.
 * ws: zero-initialised scratch of hq_select_k_workspace_size() bytes, left zeroed.
 * One launch per candidate k plus one selection launch; deterministic. */
I4_API i4_status hq_select_k(const void* X, int64_t N, const void* W, int64_t C, int64_t D, float s_x, float s_w,
                             int32_t k_min, int32_t k_max, int32_t* k_best, double* mse, void* ws,
                             size_t ws_bytes, void* stream);
I4_API size_t hq_select_k_workspace_size(void);

/* BMM in attention (A.1; reading Z-31): T = BMM(Q, K^T) with
 * Q [B, N, M], K [B, P, M] bf16 and per-batch step sizes s_q[B], s_k[B] (HOST
 * float arrays).  Batch b is the linear operator above with
 * X = Q_b, W = K_b (D = M, C = P): T_b = s_q[b] s_k[b] Q_hat_b K_hat_b^T, and
 * H_hat = Repeat_B(BlockDiag(H_k, ...)) is the per-row block
 * transform of the linear operator.  The batch dimension is inside the kernels:
 * the forward is 3 launches for all B batches (step table, hadamard_quant over
 * the B N + B P rows, one batched GEMM over 3-D tensor maps), the backward 4
 * (grad_split with per-batch amax, one sampler cluster per (mask, batch), compact,
 * one GEMM launch over every batch's grad_Q and grad_K tiles).
 * The cache holds all batches (device buffers, caller-allocated):
 *   qq int8 [B, N, M], kq int8 [B, P, M], q_mask uint32 [B, N, M/32],
 *   k_mask uint32 [B, P, M/32], q_sqnorm int32 [B, N],
 *   steps float [B, 8] (library-written per-batch step table: 1/s_q and 1/s_k
 *   scaled by 2^{-k/2}, fl32(s_q s_k), fl32(s_k 2^{-k/2}), fl32(s_q 2^{-k/2}), s_q, s_k),
 *   dev_status int32 (optional, NULL = off; status bits as i4_fwd_cache);
 * B, N, P, M, k are filled by int4_bmm_fwd.  Shape rules: M, P positive multiples
 * of 64 (M <= 8192, M % 2^k == 0); N > 0; the backward needs N <= 65536. */
typedef struct {
    int8_t* qq;
    int8_t* kq;
    uint32_t* q_mask;
    uint32_t* k_mask;
    int32_t* q_sqnorm;
    float* steps;
    int32_t* dev_status;
    int64_t B, N, P, M;
    int32_t k;
} i4_bmm_cache;

/* T [B, N, P] fp32 or bf16. */
I4_API i4_status int4_bmm_fwd(const void* Q, const void* K, int64_t B, int64_t N, int64_t P, int64_t M, int32_t k,
                              const float* s_q, const float* s_k, void* T, i4_out_dtype t_dtype, i4_bmm_cache* cache,
                              void* stream);

/* Per-batch LSS-MM backward, batched inside the kernels: dQ [B, N, M] (fp32 or
 * bf16), dK [B, P, M] fp32.  Batch b is int4_linear_bwd of its forward with
 * token_offset = b N (distinct Philox streams, reading Z-31), its own amax and
 * budget N, the step sizes of the forward (cache->steps), operand form 0 (the
 * compacted kept items) for both masks.  ws: int4_bmm_bwd_workspace_size(B, N, P, M)
 * bytes, ZERO-INITIALISED BEFORE ITS FIRST USE (it holds grad_split's per-batch
 * amax words; every call leaves them zero again).  B is processed in
 * chunks of at most 2048 batches (one launch sequence per chunk). */
I4_API size_t int4_bmm_bwd_workspace_size(int64_t B, int64_t N, int64_t P, int64_t M);
I4_API i4_status int4_bmm_bwd(const void* dT, const i4_bmm_cache* cache, uint64_t seed, uint32_t call_id,
                              i4_lss_mode mode, void* dQ, i4_out_dtype dq_dtype, float* dK, void* ws,
                              size_t ws_bytes, void* stream);
/* Introspection (tests): byte offset inside the BMM backward workspace of
 *   what = 0  s_down float [B]           1  amax bits uint32 [B]
 *          2  kept counts int32 [2][B] ([0][b] grad_K mask, [1][b] grad_Q mask)
 *          3  grad_K item list int32 [B][2N + 128]   4  its weight exponents int8 [B][2N + 128]
 *          5  grad_Q item list int32 [B][2N + 128]   6  its weight exponents int8 [B][2N + 128]
 *          7  8-bit SR codes q int8 [B N + 1, P]
 * of the last call's first chunk; (size_t)-1 for an unknown `what`. */
I4_API size_t int4_bmm_bwd_ws_offset(int64_t B, int64_t N, int64_t P, int64_t M, int32_t what);

/* Bytes of device scratch int4_linear_bwd needs for these shapes. */
I4_API size_t int4_bwd_workspace_size(int64_t N, int64_t D, int64_t C);

/* Introspection: byte offset, inside int4_linear_bwd's workspace, of two int32
 * flags the last backward left there: [0] the grad_W mask, [1] the grad_X mask was
 * deterministic (every item with a positive score kept with weight 1; DESIGN.md
 * reading Z-32), so that GEMM ran on the 8-bit code plane q8 (and X_hat) with no
 * compaction; 0: the GEMM ran on the compacted kept items; 2: a binding budget left
 * few items sampled, so the GEMM ran on q8 / X_hat plus correction rows (reading
 * Z-33).  Informational only: results do not depend on which form ran. */
I4_API size_t int4_bwd_ws_det_offset(int64_t N, int64_t D, int64_t C);

/* Introspection: byte offset, inside the backward workspace, of two int32 counts of the
 * last backward's operand form 2 (dense + correction, reading Z-33; flag
 * value 2 above): [0] grad_W correction rows, [1] grad_X rows of the sampled tokens. */
I4_API size_t int4_bwd_ws_form2_offset(int64_t N, int64_t D, int64_t C);

/* Exact INT8 x INT8 -> INT32 product acc[m, n] = sum_k A(m, k) B(n, k) on the
 * tcgen05 path used by every GEMM of the operator ("Multiply the
 * two INT4 matrices").  A is [M, K] (a_mn_major = 0) or [K, M] (a_mn_major = 1);
 * B is [Nn, K] or [K, Nn]; acc [M, Nn] int32.  K % 16 == 0, Nn % 64 == 0.
 * Exposed for the bit-exact accumulator parity check. */
I4_API i4_status int4_gemm_s8s8s32(const int8_t* A, int32_t a_mn_major, const int8_t* B, int32_t b_mn_major, int64_t M,
                                   int64_t Nn, int64_t K, int32_t* acc, void* stream);

/* Measurement hook (used by bench.py).  int4_trace_begin arms tracing on the
 * calling thread with `capacity` caller-created cudaEvent_t handles (passed as
 * void*) for a window of launches starting at the library's `first_launch`-th
 * launch (0-based, counted from this call): events[0] is recorded on the launch
 * stream just before that launch and events[i+1] right after the window's i-th
 * launch, so consecutive events bracket each launch of the window (under
 * stream capture the records become graph event nodes).  int4_trace_end
 * disarms tracing, writes the static names of all launches seen into
 * names[0..n) and returns n.  The events stay caller-owned. */
I4_API i4_status int4_trace_begin(void* const* events, int32_t capacity, int32_t first_launch);
I4_API int32_t int4_trace_end(const char** names, int32_t capacity);

/* Programmatic dependent launch: every kernel of the library is launched so that
 * the next kernel in the stream may start launching while it drains (each kernel
 * waits for its predecessor's completion before touching its data).  On by
 * default; int4_set_pdl(0/1) switches it process-wide and returns the previous
 * setting.  Timing per kernel (bench.py's
 * breakdown) is taken with it off, since an early-launched kernel's duration
 * includes its wait. */
I4_API int32_t int4_set_pdl(int32_t enable);

/* Introspection (tests): CTAs per mask in the thread-block cluster the LSS sampler
 * launches for N tokens on the current device -- 1, 8, or 16 (non-portable, chosen
 * only when the occupancy API reports that a 16-CTA cluster fits). */
I4_API int32_t int4_sampler_cluster_ctas(int64_t N);

/* Thread-local message describing the last non-OK status of this thread. */
I4_API const char* int4_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* INT4LINEAR_H */
