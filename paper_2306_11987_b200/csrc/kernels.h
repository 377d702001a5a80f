// Internal host-side launchers of the sm_100a kernels (not part of the C ABI;
// the ABI is include/int4linear.h, implemented in api.cu).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace i4 {

// Programmatic dependent launch attribute for every launch of the library
// (int4_set_pdl(0) turns it off, for per-kernel timing).
bool pdl_enabled();
inline int add_pdl_attr(cudaLaunchAttribute* attrs, int n) {
    if (pdl_enabled()) {
        attrs[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attrs[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    return n;
}

constexpr int kMaxDevices = 64;          // per-device caches of launch parameters
// device status word bits (i4_fwd_cache::dev_status, i4_lss_plan::dev_status)
constexpr int32_t kStatusNonFinite = 1;  // an input element is Inf / NaN ("input error")
constexpr int32_t kStatusZeroGrad = 2;   // grad_Y is all zero ("degenerate")

// quant.cu --------------------------------------------------------------------
constexpr int kStepTabChunk = 128;       // batches per step-table launch (8 floats each, kernel parameters)
struct HqArgs {                          // two independent hadamard_quant jobs in one launch
    const uint16_t* x0; int64_t rows0; float r0; int8_t* codes0; uint32_t* bits0; int32_t* sqnorm0;
    const uint16_t* x1; int64_t rows1; float r1; int8_t* codes1; uint32_t* bits1; int32_t* sqnorm1;
    int64_t cols; int k;
    float* delta0; float* delta1;        // optional A.3 delta = <v> - I o v (fp32, exact)
    int32_t* status;                     // optional device status word (bit 0: non-finite input)
    // batched (BMM): row i of job j uses r = r_tabj[8 (i / rpbj)] (device table) instead of rj
    const float* r_tab0; int64_t rpb0; const float* r_tab1; int64_t rpb1;
    // batched, <= kStepTabChunk batches: the host step table [tab_n][8] travels as a kernel
    // parameter (r of job j = entry j of the row's batch) and is written to tab_dst
    const float* tab_host; int tab_n; float* tab_dst;
};
cudaError_t launch_hadamard_quant2(const HqArgs& a, cudaStream_t s);
cudaError_t launch_hadamard_quant(const uint16_t* x, int64_t rows, int64_t cols, int k, float r,
                                  int8_t* codes, uint32_t* bits, int32_t* sqnorm, int32_t* status, cudaStream_t s);
constexpr int kGradSplitMaxBlocks = 2048;   // block-max scratch words the plan provides
int grad_split_stamps(unsigned long long* host, int n);
int sampler_stamps(unsigned long long* host, int enable);   // timing experiment (-DI4_STAMPS=1 builds)
cudaError_t launch_grad_split(const uint16_t* g, int64_t N, int64_t C, uint32_t* block_max, uint64_t seed,
                              uint32_t call_id, int64_t token_offset, int8_t* q8, int32_t* a_sq, float* s_down,
                              uint32_t* amax_out, int32_t* status, cudaStream_t s);
// batched (attention BMM): rows = B nb, batch b = rows [b nb, (b+1) nb) with its own amax word
// bamax[b] (zero on entry; the caller zeroes it again after use), s_down[b], amax_out[b] and
// norm block a_sq[b][2 nb]; two launches (amax, split)
cudaError_t launch_grad_split_batched(const uint16_t* g, int64_t rows, int64_t C, int64_t nb, uint64_t seed,
                                      uint32_t call_id, int64_t token_offset, int8_t* q8, int32_t* a_sq,
                                      float* s_down, uint32_t* amax_out, int32_t* status, uint32_t* bamax,
                                      cudaStream_t s);

// sampler.cu ------------------------------------------------------------------
struct SamplerArgs {
    const int32_t* a_sq;      // [2N]
    const int32_t* x_sqnorm;  // [N]  (weight-gradient scores)
    int32_t N;
    int32_t mode;             // i4_lss_mode
    uint32_t seed_lo, seed_hi, call_id;
    int64_t token_offset;
    int32_t* items[2];        // [0] grad_W mask, [1] grad_X mask
    int8_t* wexp[2];
    int32_t* count[2];
    uint8_t* x_touched;       // [N]: 1 if the token has a kept grad_X item (optional)
    uint32_t* zero_words;     // optional: words zeroed by the launch (the GEMMs' A.3 partial slots)
    int32_t n_zero_words;
    int32_t* det_flags;       // optional [2]: operand form of mask m's GEMM: 1 deterministic (every
                              // positive item kept with weight 1: dense Q / X_hat), 0 sampled
                              // (compacted kept items), 2 dense + correction (a binding budget
                              // that left few items sampled: see corr_* / sub_*)
    // optional, form 2 (all null: form 2 never chosen):
    int32_t* corr_items; int8_t* corr_wexp; int32_t* corr_count;   // grad_W: per sampled item a
                              // -1 row (removes its dense term) and, if kept, a +2^wexp row
    int32_t* sub_items; int8_t* sub_wexp; int32_t* sub_count;      // grad_X: the kept items of the
                              // tokens with a sampled item (token-major)
    uint8_t* tok_flag;        // [N] 1: token's grad_X row comes from sub-list rows, not Q
    // batched (attention BMM): `batch` > 1 independent masks pairs, one cluster per (mask,
    // batch); batch b reads a_sq + 2 N b, x_sqnorm + N b, writes items / wexp + b bs_list,
    // count + b, x_touched + N b, Philox token index token_offset + N b + t (no form 2)
    int32_t batch;
    int64_t bs_list;
};
int sampler_max_tokens();
int sampler_cluster_ctas(int64_t N);      // CTAs per mask the sampler launches for N tokens (introspection)
cudaError_t launch_lss_sampler(const SamplerArgs& a, cudaStream_t s);

// compact.cu ------------------------------------------------------------------
struct CompactArgs {
    const int8_t* q8;         // [N+1, C] 8-bit SR codes q = 16 hi + lo (row N: zeros)
    const int8_t* xq;         // [N, D] X_hat
    int32_t N, C, D;
    const int32_t* items_x; const int32_t* count_x;
    const int32_t* items_w; const int8_t* wexp_w; const int32_t* count_w;
    const uint8_t* x_touched; // [N]
    void* dx;                 // [N, D] fp32 or bf16: rows of untouched tokens / straddling pairs zeroed here
    int32_t dx_bf16;
    int8_t* a_x;              // [2N+128, C]
    int8_t* a_w;              // [kcap, C]
    int8_t* b_w;              // [kcap, D]
    const int32_t* det_flags; // optional [2] (sampler) operand forms: [1] grad_X, [0] grad_W:
                              // 1 dense (nothing to move), 0 sampled, 2 dense + correction
    const int32_t* corr_items; const int8_t* corr_wexp; const int32_t* corr_count;   // form 2
    const int32_t* sub_items; const int32_t* sub_count; const uint8_t* tok_flag;
    // batched (attention BMM, form 0 only): blockIdx.y = batch b; q8 / xq / x_touched / dx rows
    // offset by N b, lists by bs_list b, counts by b, a_x / a_w / b_w by their per-batch extents
    // (2N + 128, kcap, kcap rows)
    int32_t batch;
    int64_t bs_list;
};
cudaError_t launch_compact(const CompactArgs& a, cudaStream_t s);

// gemm.cu ---------------------------------------------------------------------
enum EpiKind : int { EPI_INT32 = 0, EPI_FWD = 1, EPI_DGRAD = 2, EPI_WGRAD = 3,
                     EPI_BWD = 4 };           // grad_X (args g) + grad_W (args g1) GEMMs in one launch

struct GemmArgs {
    // problem: acc[M, Nn] = A(M, K) . B(Nn, K)^T; M or K may come from device memory
    int32_t M, Nn, K;
    int32_t a_mn, b_mn;       // operand stored MN-major ([K, M] / [K, Nn] rows) instead of K-major
    const int32_t* m_dev;     // if non-null: M = roundup(*m_dev) rows are valid (dgrad)
    const int32_t* k_dev;     // if non-null: K = *m_dev-style count of K rows (wgrad)
    int32_t epi;
    // outputs
    void* out;                // int32 / fp32 / bf16 [M, Nn]
    int32_t out_bf16;
    float scale;              // fwd: fl32(s_x s_w); dgrad: s_w 2^{-k/2}; wgrad: s_x 2^{-k/2}
    const float* s_down;      // dgrad / wgrad: device s_down
    int32_t k_had;            // Hadamard exponent for the epilogue inverse transform
    const uint32_t* mask;     // dgrad: I_X [N, Nn/32]; wgrad: I_W [M, Nn/32]
    const int32_t* items;     // dgrad: item id of each A row
    const int8_t* wexp;       // dgrad: weight exponent of each A row
    int32_t n_tokens;         // dgrad: N (item id = h*N + t)
    // LSQ step-size gradient (A.3), optional: sum(acc o delta) per CTA epilogue warp
    const float* delta;       // dgrad: delta_X [N, Nn] (row = token); wgrad: delta_W [M, Nn]
    double* lsq_part;         // [gridDim.x * 8] fp64 partials (entries of absent CTAs pre-zeroed)
    // dgrad / wgrad: if *dense_flag != 0 the mask is deterministic (every nonzero item kept
    // with weight 1): dgrad reads A = Q (map a2, M = n_tokens rows = tokens), wgrad reads
    // A = Q and B = X_hat (maps a3, b2, K = n_tokens)
    const int32_t* dense_flag;
    // operand form 2 (dense + correction): grad_X sub list (rows after the token rows of Q,
    // which start at row round_up(N, 256)) and the per-token flags; grad_W correction-row
    // count (k-blocks after the round_up(N, 128) token rows)
    const int32_t* items2; const int8_t* wexp2; const int32_t* m_dev2; const uint8_t* tok_flag;
    const int32_t* k_dev2;
    // grad_W only, optional: multicast (NVLS) address of a symmetric [M, Nn] fp32 buffer that
    // spans the data-parallel ranks; the epilogue reduces its tile into every rank's copy with
    // multimem.red.add instead of storing to `out`
    float* out_mc;
    // batched launches only (attention BMM; batch > 0): `batch` independent
    // problems of these sizes in one launch.  Every tensor map is 3-D (coordinate 2 = batch);
    // m_dev / k_dev / s_down point at per-batch entries; grad_X item lists of batch b start at
    // items + b * bs_items; output and mask rows of batch b are b * rows + r (rows = n_tokens
    // for grad_X, M for grad_W); scale = tab[8 b + tab_idx].  Operand form 0 only.
    int32_t batch;
    int64_t bs_items;
    const float* tab;
    int32_t tab_idx;
};
constexpr int kMaxGemmBatch = 2048;       // batches per batched backward GEMM launch (shared-memory tile table)
constexpr int kGemmCG = 2;                // CTAs per MMA tile (tcgen05 cta_group::2)
// CUtensorMap* (host): A, B, C (output), A2 (grad_X dense A = Q), A3 / B2 (grad_W dense A = Q,
// B = X_hat), AW / BW (grad_W sampled A_W, B_W in an EPI_BWD launch); null = unused
struct GemmMaps { const void* a; const void* b; const void* c; const void* a2; const void* a3; const void* b2;
                  const void* aw; const void* bw; const void* dx; };   // dx: grad_X output (EPI_BWD)
cudaError_t launch_gemm(const GemmMaps& m, const GemmArgs& g, int num_sms, cudaStream_t s,
                        const GemmArgs* g1 = nullptr);
int gemm_block_n(int Nn, bool b_mn);
int gemm_stamps(unsigned long long* host);     // timing experiment (-DI4_STAMPS=1 builds): [16] u64, resets

// lsq.cu ----------------------------------------------------------------------
constexpr int kLsqPartials = 2048;        // fp64 partial slots per GEMM (>= max grid x 8 warps)
cudaError_t launch_lsq_finalize(const double* part_x, const double* part_w, const float* s_down, float s_x,
                                float s_w, double g_x, double g_w, float* grad_s, cudaStream_t s);
size_t lsq_cold_start_ws_bytes();
cudaError_t launch_lsq_cold_start(const uint16_t* x, int64_t n, float* step, void* ws, cudaStream_t s);

cudaError_t launch_step_table(const float* host, int64_t n, float* dst, cudaStream_t s);   // host [n][8] -> dst

// adaptive_k.cu -----------------------------------------------------------------
size_t select_k_ws_bytes();
cudaError_t launch_select_k(const uint16_t* x, int64_t n, const uint16_t* w, int64_t c, int64_t d, float r_x[8],
                            float r_w[8], double c_x[8], double c_w[8], int k_min, int k_max, int32_t* k_best,
                            double* mse, void* ws, cudaStream_t s);

}  // namespace i4
