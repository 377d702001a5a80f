// Quantizer kernels (HBM roofline; instruction issue is the co-limiter):
//   hadamard_quant : F1+F2 / F3 -- block FWHT + LSQ (Eq. 2);
//                    X and W are quantized by ONE launch (two row jobs); one
//                    thread per 32-column block, Hadamard order k compile-time,
//                    butterflies and scaling on fp32 pairs (FADD2 / FMUL2)
//   grad_split     : B1 + B2 -- per-tensor max |grad_Y| (reading
//                    Z-9), then Philox SR to the 8-bit code q (stored), its high /
//                    low 4-bit halves' per-row integer norms (PAPER.md:234-239,
//                    :680); one cooperative launch with one grid barrier
#include <algorithm>
#include <atomic>
#include <cstdlib>

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace i4 {


__device__ __forceinline__ void unpack_bf16x8(const uint4& u, float (&v)[8]) {
    v[0] = bf16_lo(u.x); v[1] = bf16_hi(u.x);
    v[2] = bf16_lo(u.y); v[3] = bf16_hi(u.y);
    v[4] = bf16_lo(u.z); v[5] = bf16_hi(u.z);
    v[6] = bf16_lo(u.w); v[7] = bf16_hi(u.w);
}

__device__ __forceinline__ uint32_t pack4_i8(int a, int b, int c, int d) {
    return (uint32_t(a) & 0xFF) | ((uint32_t(b) & 0xFF) << 8) | ((uint32_t(c) & 0xFF) << 16) |
           ((uint32_t(d) & 0xFF) << 24);
}

// ---------------------------------------------------------------------------
// hadamard_quant: one thread per 32-column block of a row (32 bf16 loaded as
// 4 x 16 B, 32 int8 codes stored as 2 x 16 B, one mask word), so Hadamard
// blocks of up to 2^5 columns are transformed entirely in registers; k = 6, 7
// add one / two xor-shuffle stages between neighbouring threads of the row.
// A CTA holds R whole rows (R * cols/32 threads); row norms are reduced in
// shared memory.  X and W are two row jobs of one launch.
// ---------------------------------------------------------------------------
struct HqJob {
    const uint16_t* x;
    int64_t rows;
    float r;
    int8_t* codes;
    uint32_t* bits;
    int32_t* sqnorm;
    float* delta;                        // optional: A.3 delta = code - I o v (fp32, exact)
    int blocks;                          // CTAs assigned to this job
    int32_t* status;                     // optional: device status word (bit 0 <- non-finite input)
    const float* r_tab;                  // batched (BMM): r of row i = r_tab[8 (i / rpb)] (else r)
    int64_t rpb;
};

constexpr int kHqMaxThreads = 256;

// One 32-column block of one row: FWHT (registers, + xor-shuffle stages for
// k = 6, 7), LSQ, code / mask / delta stores; returns the block's sum of squared codes.
template <int K, bool DELTA>
__device__ __forceinline__ int hq_block(const HqJob& J, float r, int64_t row, int blk, int tpr, int cols,
                                        bool active, const uint4 (&raw)[4]) {
    // column pairs (j, j + 16) in fp32x2 registers: the in-register FWHT stages
    // (strides 1 .. 8) and the LSQ scaling run as packed FADD2 / FMUL2
    uint64_t p[16];
    {
        float v[32];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float t[8];
            unpack_bf16x8(raw[q], t);
#pragma unroll
            for (int i = 0; i < 8; ++i) v[8 * q + i] = t[i];
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) p[j] = f2_pack(v[j], v[j + 16]);
    }
    fwht_pairs<32, (K < 5 ? K : 5)>(p);              // strides 1 .. 16: registers only
    if constexpr (K > 5) {                           // strides 32, 64 columns: partner thread blk ^ 1, ^ 2
#pragma unroll
        for (int s = 5; s < K; ++s) {
            const int lm = 1 << (s - 5);
            const float sgn = (blk & lm) ? -1.0f : 1.0f;   // upper block: o - v, lower: v + o
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                float a, b;
                f2_unpack(p[j], a, b);
                const float oa = __shfl_xor_sync(0xFFFFFFFFu, a, lm);
                const float ob = __shfl_xor_sync(0xFFFFFFFFu, b, lm);
                p[j] = f2_pack(__fmaf_rn(sgn, a, oa), __fmaf_rn(sgn, b, ob));   // one rounding = the add / sub
            }
        }
    }
    if (!active) return 0;
    if (J.status != nullptr) {
        // Inf / NaN anywhere in the block (or a transform that overflows fp32) makes
        // t * 0 NaN: flag the device status word ("input error")
        uint64_t z = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) z = f2_fma(p[j], 0, z);
        float z0, z1;
        f2_unpack(z, z0, z1);
        if (z0 != 0.0f || z1 != 0.0f) atomicOr(J.status, kStatusNonFinite);
    }
    // LSQ: v = fl32(t r); code = clamp(rint(v), -7, 7); mask = |v| <= 7.
    // rint on the clamped value by the magic-number add: fl32(c + 1.5 2^23) is
    // exact round-half-even for |c| <= 7 (ulp 1 there), and the low byte of its
    // bits is the int8 code (0x4B400000 + q) -- one FADD instead of an F2I.
    const uint64_t r2 = f2_pack(r, r);
    uint32_t qb[32];                                // code in byte 0
    uint32_t mask = 0;
    int sq = 0;
    float dl[DELTA ? 32 : 1];                       // A.3 delta, if requested
    // clamp mask from sign bits: o = 7 - |v| is exact near |v| = 7 (Sterbenz) and
    // never rounds across 0, so its sign bit is [|v| > 7]; a funnel shift moves it
    // into the mask word (one ALU op per element; elements taken 15 .. 0 so that
    // element j lands in bit j, the high 16 in a second word)
    uint32_t out_lo = 0, out_hi = 0;
#pragma unroll
    for (int j = 15; j >= 0; --j) {
        float s0, s1;
        f2_unpack(f2_mul(p[j], r2), s0, s1);
        const float c0 = fminf(fmaxf(s0, -7.0f), 7.0f), c1 = fminf(fmaxf(s1, -7.0f), 7.0f);
        const float m0 = __fadd_rn(c0, 12582912.0f), m1 = __fadd_rn(c1, 12582912.0f);
        qb[j] = __float_as_uint(m0);
        qb[j + 16] = __float_as_uint(m1);
        const float o0 = __fsub_rn(7.0f, fabsf(s0)), o1 = __fsub_rn(7.0f, fabsf(s1));
        out_lo = __funnelshift_l(__float_as_uint(o0), out_lo, 1);   // (out_lo << 1) | sign(o0)
        out_hi = __funnelshift_l(__float_as_uint(o1), out_hi, 1);
        const bool in0 = !(__float_as_uint(o0) >> 31), in1 = !(__float_as_uint(o1) >> 31);
        if constexpr (DELTA) {
            const float q0 = __fsub_rn(m0, 12582912.0f), q1 = __fsub_rn(m1, 12582912.0f);   // exact
            dl[j] = in0 ? __fsub_rn(q0, s0) : q0;                                    // exact (|.| <= 1/2)
            dl[j + 16] = in1 ? __fsub_rn(q1, s1) : q1;
        } else {
            (void)in0; (void)in1;
        }
    }
    mask = ~(out_lo | (out_hi << 16));
    if (DELTA && J.delta != nullptr) {
        float4* dd = reinterpret_cast<float4*>(J.delta + row * cols + blk * 32);
#pragma unroll
        for (int i = 0; i < 8; ++i) dd[i] = make_float4(dl[4 * i], dl[4 * i + 1], dl[4 * i + 2], dl[4 * i + 3]);
    }
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        w[i] = __byte_perm(__byte_perm(qb[4 * i], qb[4 * i + 1], 0x0040),
                           __byte_perm(qb[4 * i + 2], qb[4 * i + 3], 0x0040), 0x5410);
        sq = __dp4a(int(w[i]), int(w[i]), sq);     // sum of squared codes, 4 per instruction
    }
    int8_t* dst = J.codes + row * cols + blk * 32;
    *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
    *reinterpret_cast<uint4*>(dst + 16) = make_uint4(w[4], w[5], w[6], w[7]);
    if (J.bits != nullptr) J.bits[row * tpr + blk] = mask;
    return sq;
}

#ifndef I4_HQ_TMA
#define I4_HQ_TMA 0
#endif
static int hq_rows_per_cta(int64_t cols) {
    const int tpr = int(cols / 32);
    return tpr >= kHqMaxThreads ? 1 : kHqMaxThreads / tpr;
}

#if I4_HQ_TMA
// TMA-staged persistent variant (compile with -DI4_HQ_TMA=1).  Measured 4-15 %
// slower than the register-staged kernel above on every BASELINE shape (B200:
// BERT-large FFN-up 13.2 vs 11.5 us, ViT FFN-down 106 vs 103 us): the kernel is
// instruction-issue bound, not latency bound, and the per-stage CTA barriers
// cost more than the deeper prefetch gains.  A stage is RS whole rows (RS x cols bf16, one
// contiguous cp.async.bulk copy of ~16 KB); each CTA streams its stages through
// a kHqStages-deep shared-memory ring (mbarrier completion), so ~64 KB per CTA
// (~128 KB per SM) of X / W is in flight while the threads transform earlier
// stages: thread (row slot, 32-column block) pulls its 64 bytes from shared
// memory into registers for the FWHT + LSQ of hq_block, and stores its codes and
// mask word straight to global memory (a warp's stores cover contiguous bytes of
// one row).  Stages never cross the X / W job boundary.  Row norms: shared-memory
// integer atomics per stage (exact, order-independent).
constexpr int kHqStages = 4;
constexpr int kHqStageBytes = 16384;          // target bytes per stage (RS rows)

struct HqSched {
    int rs;                                    // rows per stage
    int64_t st0, st1;                          // stages of job 0 (X) and job 1 (W)
};

template <int K, bool DELTA>
__global__ void __launch_bounds__(kHqMaxThreads)
hadamard_quant_tma_kernel(HqJob j0, HqJob j1, int cols, HqSched hs) {
    extern __shared__ __align__(128) uint8_t hq_smem[];
    __shared__ uint64_t full[kHqStages];
    __shared__ int sq_row[kHqMaxThreads];
    const int tpr = cols >> 5;                       // threads (32-column blocks) per row
    const int r_local = int(threadIdx.x) / tpr;
    const int blk = int(threadIdx.x) - r_local * tpr;
    const int64_t n_stages = hs.st0 + hs.st1;
    const int64_t row_bytes = int64_t(cols) * 2;
    const int stage_bytes = hs.rs * int(row_bytes);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kHqStages; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    pdl_trigger();
    pdl_wait();                                        // X / W may be written by the previous kernel
    // stage i of this CTA = global stage blockIdx.x + i * gridDim.x
    auto issue = [&](int64_t gs, int slot) {
        const bool second = gs >= hs.st0;
        const HqJob& J = second ? j1 : j0;
        const int64_t row0 = (second ? gs - hs.st0 : gs) * hs.rs;
        const int64_t nrow = min(int64_t(hs.rs), J.rows - row0);
        const uint32_t bytes = uint32_t(nrow * row_bytes);
        mbar_arrive_expect_tx(&full[slot], bytes);
        bulk_copy_g2s(hq_smem + slot * stage_bytes, J.x + row0 * cols, bytes, &full[slot]);
    };
    if (threadIdx.x == 0)
        for (int s = 0; s < kHqStages; ++s) {
            const int64_t gs = int64_t(blockIdx.x) + int64_t(s) * gridDim.x;
            if (gs < n_stages) issue(gs, s);
        }
    int it = 0;
    for (int64_t gs = blockIdx.x; gs < n_stages; gs += gridDim.x, ++it) {
        const int slot = it % kHqStages;
        const uint32_t ph = uint32_t(it / kHqStages) & 1u;
        const bool second = gs >= hs.st0;
        const HqJob& J = second ? j1 : j0;
        const int64_t row0 = (second ? gs - hs.st0 : gs) * hs.rs;
        const int64_t row = row0 + r_local;
        const bool active = r_local < hs.rs && row < J.rows;
        if (threadIdx.x < hs.rs) sq_row[threadIdx.x] = 0;
        mbar_wait(&full[slot], ph);
        uint4 raw[4];
        const uint8_t* src = hq_smem + slot * stage_bytes + (active ? r_local * row_bytes + blk * 64 : 0);
#pragma unroll
        for (int q = 0; q < 4; ++q) raw[q] = active ? ld_shared_v4(src + 16 * q) : make_uint4(0, 0, 0, 0);
        __syncthreads();                               // slot drained (and sq_row zeroed): refill it
        if (threadIdx.x == 0) {
            const int64_t nx = gs + int64_t(kHqStages) * gridDim.x;
            fence_proxy_async_smem();                  // the generic reads above before the async refill
            if (nx < n_stages) issue(nx, slot);
        }
        const int sq = hq_block<K, DELTA>(J, J.r, row, blk, tpr, cols, active, raw);
        if (active && J.sqnorm != nullptr) atomicAdd(&sq_row[r_local], sq);
        if (J.sqnorm != nullptr) {
            __syncthreads();
            if (active && blk == 0) J.sqnorm[row] = sq_row[r_local];
        }
        __syncthreads();                               // sq_row reused by the next stage
    }
}

static cudaError_t launch_hadamard_quant_tma(const HqArgs& a, cudaStream_t s) {
    if (a.cols / 32 > kHqMaxThreads) return cudaErrorInvalidValue;   // cols > 8192: not supported
    // rows per stage: whole rows, one per thread-row slot of the CTA, at most ~16 KB
    const int R = hq_rows_per_cta(a.cols);
    int rs = int(kHqStageBytes / (a.cols * 2));
    if (rs > R) rs = R;
    if (rs < 1) rs = 1;
    HqJob j0{a.x0, a.rows0, a.r0, a.codes0, a.bits0, a.sqnorm0, a.delta0, 0, a.status};
    HqJob j1{a.x1, a.rows1, a.r1, a.codes1, a.bits1, a.sqnorm1, a.delta1, 0, a.status};
    HqSched hs{rs, (a.rows0 + rs - 1) / rs, (a.rows1 + rs - 1) / rs};
    const int64_t n_stages = hs.st0 + hs.st1;
    if (n_stages == 0) return cudaSuccess;
    static std::atomic<int> sms_cache[kMaxDevices];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDevices) dev = 0;
    int sms = sms_cache[dev].load(std::memory_order_relaxed);
    if (sms == 0) {
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        sms_cache[dev].store(sms, std::memory_order_relaxed);
    }
    // persistent: 3 CTAs per SM (3 x 64 KB ring), never more CTAs than stages
    int64_t grid = int64_t(sms) * 3;
    if (grid > n_stages) grid = n_stages;
    const int threads = (R * int(a.cols / 32) + 31) / 32 * 32;   // whole warps (xor-shuffle stages)
    const int smem = kHqStages * rs * int(a.cols) * 2;
    void (*kern)(HqJob, HqJob, int, HqSched) = nullptr;
    const bool delta = a.delta0 != nullptr || a.delta1 != nullptr;
#define I4_HQ_K(KK) kern = delta ? hadamard_quant_tma_kernel<KK, true> : hadamard_quant_tma_kernel<KK, false>; break;
    switch (a.k) {
        case 0: I4_HQ_K(0)
        case 1: I4_HQ_K(1)
        case 2: I4_HQ_K(2)
        case 3: I4_HQ_K(3)
        case 4: I4_HQ_K(4)
        case 5: I4_HQ_K(5)
        case 6: I4_HQ_K(6)
        case 7: I4_HQ_K(7)
        default: return cudaErrorInvalidValue;
    }
#undef I4_HQ_K
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(unsigned(threads));
    cfg.dynamicSmemBytes = size_t(smem);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    cfg.attrs = attr;
    cfg.numAttrs = add_pdl_attr(attr, 0);
    return cudaLaunchKernelEx(&cfg, kern, j0, j1, int(a.cols), hs);
}

#endif  // I4_HQ_TMA

// A CTA covers PASSES x R rows: the thread of (row slot, block) handles row
// slot + pass R for every pass, with the loads of all passes issued before the
// first block is transformed (measured on B200: 2 and 4 passes are 20-45 %
// slower than 1 -- the kernel is instruction-issue bound, not latency bound).
#ifndef I4_HQ_PASSES
#define I4_HQ_PASSES 1
#endif
constexpr int kHqPasses = I4_HQ_PASSES;

// TAB: batched BMM forward with at most kStepTabChunk batches: the per-batch step table
// travels as a kernel parameter (row i of job j uses r = v[8 (i / rpb) + j]) and CTA 0
// writes it to device memory for the GEMM and the backward (no separate launch)
template <bool TAB> struct HqTab { int n; float* dst; float v[kStepTabChunk * 8]; };
template <> struct HqTab<false> {};

template <int K, bool DELTA, bool TAB>
__global__ void __launch_bounds__(kHqMaxThreads)
hadamard_quant_kernel(HqJob j0, HqJob j1, int cols, int rows_per_cta, const HqTab<TAB> tab) {
    const bool second = int(blockIdx.x) >= j0.blocks;
    const HqJob& J = second ? j1 : j0;
    const int bid = second ? int(blockIdx.x) - j0.blocks : int(blockIdx.x);
    const int tpr = cols >> 5;                       // threads (32-column blocks) per row
    const int r_local = int(threadIdx.x) / tpr;
    const int blk = int(threadIdx.x) - r_local * tpr;
    const int64_t row0 = int64_t(bid) * rows_per_cta * kHqPasses + r_local;
    pdl_trigger();
    pdl_wait();                                        // X / W may be written by the previous kernel
    if constexpr (TAB) {
        if (blockIdx.x == 0)
            for (int i = threadIdx.x; i < tab.n * 8; i += blockDim.x) tab.dst[i] = tab.v[i];
    }
    __shared__ int sq_row[kHqPasses][kHqMaxThreads];
    if (threadIdx.x < rows_per_cta)
#pragma unroll
        for (int ps = 0; ps < kHqPasses; ++ps) sq_row[ps][threadIdx.x] = 0;
    uint4 raw[kHqPasses][4];
#pragma unroll
    for (int ps = 0; ps < kHqPasses; ++ps) {
        const int64_t row = row0 + int64_t(ps) * rows_per_cta;
        const bool active = r_local < rows_per_cta && row < J.rows;
        const uint16_t* src = J.x + (active ? row * cols + blk * 32 : 0);
#pragma unroll
        for (int q = 0; q < 4; ++q) raw[ps][q] = active ? ld_nc_v4(src + 8 * q) : make_uint4(0, 0, 0, 0);
    }
    __syncthreads();                                   // sq_row initialised
#pragma unroll
    for (int ps = 0; ps < kHqPasses; ++ps) {
        const int64_t row = row0 + int64_t(ps) * rows_per_cta;
        const bool active = r_local < rows_per_cta && row < J.rows;
        float r = J.r;
        if constexpr (TAB) {
            if (active) r = tab.v[8 * int(row / J.rpb) + (second ? 1 : 0)];
        } else {
            if (J.r_tab != nullptr && active) r = __ldg(J.r_tab + 8 * (row / J.rpb));
        }
        const int sq = hq_block<K, DELTA>(J, r, row, blk, tpr, cols, active, raw[ps]);
        if (active && J.sqnorm != nullptr) atomicAdd(&sq_row[ps][r_local], sq);
    }
    if (J.sqnorm != nullptr) {
        __syncthreads();
        if (r_local < rows_per_cta && blk == 0)
#pragma unroll
            for (int ps = 0; ps < kHqPasses; ++ps) {
                const int64_t row = row0 + int64_t(ps) * rows_per_cta;
                if (row < J.rows) J.sqnorm[row] = sq_row[ps][r_local];
            }
    }
}

static cudaError_t launch_hq_tab(const HqArgs& a, const HqJob& j0, const HqJob& j1, int R, int grid, int threads,
                                 cudaStream_t s) {
    if (a.tab_n < 1 || a.tab_n > kStepTabChunk || a.delta0 != nullptr || a.delta1 != nullptr) return cudaErrorInvalidValue;
    HqTab<true> t{};
    t.n = a.tab_n;
    t.dst = a.tab_dst;
    for (int i = 0; i < a.tab_n * 8; ++i) t.v[i] = a.tab_host[i];
    void (*kern)(HqJob, HqJob, int, int, HqTab<true>) = nullptr;
    switch (a.k) {
        case 0: kern = hadamard_quant_kernel<0, false, true>; break;
        case 1: kern = hadamard_quant_kernel<1, false, true>; break;
        case 2: kern = hadamard_quant_kernel<2, false, true>; break;
        case 3: kern = hadamard_quant_kernel<3, false, true>; break;
        case 4: kern = hadamard_quant_kernel<4, false, true>; break;
        case 5: kern = hadamard_quant_kernel<5, false, true>; break;
        case 6: kern = hadamard_quant_kernel<6, false, true>; break;
        case 7: kern = hadamard_quant_kernel<7, false, true>; break;
        default: return cudaErrorInvalidValue;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(unsigned(threads));
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    cfg.attrs = attr;
    cfg.numAttrs = add_pdl_attr(attr, 0);
    return cudaLaunchKernelEx(&cfg, kern, j0, j1, int(a.cols), R, t);
}

cudaError_t launch_hadamard_quant2(const HqArgs& a, cudaStream_t s) {
    if (a.cols / 32 > kHqMaxThreads) return cudaErrorInvalidValue;   // cols > 8192: not supported
#if I4_HQ_TMA
    return launch_hadamard_quant_tma(a, s);
#endif
    const int R = hq_rows_per_cta(a.cols);
    HqJob j0{a.x0, a.rows0, a.r0, a.codes0, a.bits0, a.sqnorm0, a.delta0, 0, a.status, a.r_tab0, a.rpb0};
    HqJob j1{a.x1, a.rows1, a.r1, a.codes1, a.bits1, a.sqnorm1, a.delta1, 0, a.status, a.r_tab1, a.rpb1};
    j0.blocks = int((a.rows0 + int64_t(R) * kHqPasses - 1) / (int64_t(R) * kHqPasses));
    j1.blocks = int((a.rows1 + int64_t(R) * kHqPasses - 1) / (int64_t(R) * kHqPasses));
    const int grid = j0.blocks + j1.blocks;
    if (grid == 0) return cudaSuccess;
    const int threads = (R * int(a.cols / 32) + 31) / 32 * 32;   // whole warps (xor-shuffle stages)
    if (a.tab_host != nullptr) return launch_hq_tab(a, j0, j1, R, grid, threads, s);
    void (*kern)(HqJob, HqJob, int, int, HqTab<false>) = nullptr;
    const bool delta = a.delta0 != nullptr || a.delta1 != nullptr;
#define I4_HQ_K(KK) kern = delta ? hadamard_quant_kernel<KK, true, false> : hadamard_quant_kernel<KK, false, false>; break;
    switch (a.k) {
        case 0: I4_HQ_K(0)
        case 1: I4_HQ_K(1)
        case 2: I4_HQ_K(2)
        case 3: I4_HQ_K(3)
        case 4: I4_HQ_K(4)
        case 5: I4_HQ_K(5)
        case 6: I4_HQ_K(6)
        case 7: I4_HQ_K(7)
        default: return cudaErrorInvalidValue;
    }
#undef I4_HQ_K
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(unsigned(threads));
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    cfg.attrs = attr;
    cfg.numAttrs = add_pdl_attr(attr, 0);
    return cudaLaunchKernelEx(&cfg, kern, j0, j1, int(a.cols), R, HqTab<false>{});
}

cudaError_t launch_hadamard_quant(const uint16_t* x, int64_t rows, int64_t cols, int k, float r,
                                  int8_t* codes, uint32_t* bits, int32_t* sqnorm, int32_t* status, cudaStream_t s) {
    HqArgs a{};
    a.status = status;
    a.x0 = x; a.rows0 = rows; a.r0 = r; a.codes0 = codes; a.bits0 = bits; a.sqnorm0 = sqnorm;
    a.cols = cols; a.k = k;
    return launch_hadamard_quant2(a, s);
}

// ---------------------------------------------------------------------------
// B1 + B2 fused: grad_split_kernel (cooperative launch: all CTAs co-resident).
//   phase 1  amax of grad_Y: max over |g| as bf16 bit patterns (non-negative bf16
//            values order like their 15-bit integers), exact and
//            order-independent; each CTA folds its maximum into one scratch
//            word (atomicMax) and counts itself in (fence + atomicAdd)
//   --- every CTA spins until all arrived (one acquire load per poll) ---
//   phase 2  s_down = fl32(amax / 119), r8 = fl32(119 / amax); v = fl32(g r8)
//            clamped to [-119, 119]; A = ceil(v 2^32) (v 2^32 is exact in fp32, the
//            conversion rounds up); q = floor((A + u) / 2^32) with u the element's
//            32-bit uniform: the floor form of SR, P(q = floor(v) + 1) =
//            ceil(frac(v) 2^32) / 2^32 (reading Z-10); u's high 16 bits come from
//            the purpose-1 Philox stream, its low 16 bits from purpose 4, drawn only
//            when the high half leaves the decision open (Z-20).  The code plane
//            stores q itself; hi = floor((q+8)/16), lo = q - 16 hi (Z-11) are formed
//            in registers for the per-row sum hi^2, sum lo^2 (the leverage scores'
//            INT data) and split again on the fly where a half-row is
//            an operand (compact).
//            grad_Y is re-read right after phase 1, mostly from L2.
// ---------------------------------------------------------------------------
constexpr int kSplitThreads = 256;
#ifndef I4_BS_GROUP
#define I4_BS_GROUP 4
#endif
#ifndef I4_BS_MINB
#define I4_BS_MINB 3
#endif
constexpr int kBsGroup = I4_BS_GROUP;
#ifndef I4_BS_GMAX
#define I4_BS_GMAX 3                      // largest unit size (chunks of 256 columns) phase 2 uses
#endif
constexpr int kBsGMax = I4_BS_GMAX;
#ifndef I4_BS_AMAX_UNROLL
#define I4_BS_AMAX_UNROLL 4
#endif
constexpr int kAmaxUnroll = I4_BS_AMAX_UNROLL;

__device__ __forceinline__ uint32_t bf16x2_absmax(uint32_t w) {
    return max(w & 0x7FFFu, (w >> 16) & 0x7FFFu);
}

// Philox4x32-10 of the SR stream (purpose word c2 = 1) for counters whose high
// word c1 is 0 (block index L/8 < 2^32, checked on the host): round 0's
// multiply of c2 is the constant M1, and round 1 multiplies c0 = k0[0], a
// kernel constant the compiler hoists -- 18 IMAD.WIDE per call instead of 20.
// Same function as philox4x32_10(c0, 0, 1, call_id, K), restated.
__device__ __forceinline__ Philox4 philox_sr_c1z(uint32_t c0, uint32_t call_id, const PhiloxKeys& K) {
    const uint64_t p0 = uint64_t(0xD2511F53u) * c0;
    uint32_t x0 = K.k0[0], x1 = 0xCD9E8D57u;                 // hi(M1 * 1) ^ c1 ^ k0 ; lo(M1 * 1)
    uint32_t x2 = uint32_t(p0 >> 32) ^ call_id ^ K.k1[0], x3 = uint32_t(p0);
#pragma unroll
    for (int r = 1; r < 10; ++r) {
        const uint64_t q0 = uint64_t(0xD2511F53u) * x0;
        const uint64_t q1 = uint64_t(0xCD9E8D57u) * x2;
        const uint32_t n0 = uint32_t(q1 >> 32) ^ x1 ^ K.k0[r], n2 = uint32_t(q0 >> 32) ^ x3 ^ K.k1[r];
        x0 = n0; x1 = uint32_t(q1); x2 = n2; x3 = uint32_t(q0);
    }
    return {x0, x1, x2, x3};
}

// Fast phase 2 for one 8-element chunk (readings Z-10, Z-11, Z-20):
//   v = fl32(g r8) on fp32 pairs (FMUL2), y = v 2^32 (exact power-of-two scaling, also
//       for a subnormal fl32(g r8)); CLAMP: y in [-119 2^32, 119 2^32]
//   A = ceil(y) as s64 (F2I.S64.CEIL); q = hi32(A + u): the floor form of SR
//   u = (h1 << 16) | h4, h_p = 16-bit half (L mod 8) of Philox block L / 8 of purpose p.
//   The high half decides unless the low word of A + (h1 << 16) is above 0xFFFF0000
//   (probability < 2^-16 per element); only then is the purpose-4 block drawn and
//   q += [h4 > ~lo32(A + (h1 << 16))] (a divergent branch the warp rarely takes).
// then, on 4 packed codes: t = (q ^ 0x80) + 8 per byte = q + 136 (no cross-byte carry),
//   16 hi = (t ^ 0x80) & 0xF0 (signed byte), x = t & 0x0F = lo + 8, x | 0xF0 = lo - 8:
//   dp4a(16 hi, 16 hi) = 256 sum hi^2 and dp4a(x, x | 0xF0) = sum lo^2 - 64 per element
//   (the 64 s are added back per chunk).
constexpr uint32_t kPurposeSRLow = 4;
#ifndef I4_GS_UNPACK
#define I4_GS_UNPACK 1
#endif
#ifndef I4_GS_PACK
#define I4_GS_PACK 1
#endif
template <bool CLAMP, bool C1Z>
__device__ __forceinline__ void split_chunk8(const uint4 raw, uint64_t blk, uint32_t call_id, const PhiloxKeys& keys,
                                             const float r8, uint2& pq, int& shi, int& slo) {
    const Philox4 p = C1Z ? philox_sr_c1z(uint32_t(blk), call_id, keys)
                          : philox4x32_10(uint32_t(blk), uint32_t(blk >> 32), kPurposeSR, call_id, keys);
    const uint32_t pw[4] = {p.x, p.y, p.z, p.w};
    const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
    const uint64_t r2 = f2_pack(r8, r8);
    int qv[8];
    uint32_t L[8];
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
        // elements i (low bf16) and i + 1 (high bf16) as one fp32 pair
        const uint32_t wv = w[i >> 1];
#if I4_GS_UNPACK
        uint32_t lo16;                                                 // low bf16 as fp32 by a shift (fma pipe)
        asm("mul.lo.u32 %0, %1, 65536;" : "=r"(lo16) : "r"(wv));
#else
        const uint32_t lo16 = __byte_perm(wv, 0u, 0x1044u);
#endif
        const uint64_t g2 = f2_pack(__uint_as_float(lo16), __uint_as_float(wv & 0xFFFF0000u));
        float y0, y1;
        f2_unpack(f2_mul(f2_mul(g2, r2), f2_pack(4294967296.0f, 4294967296.0f)), y0, y1);
        if (CLAMP) {                                                   // 119 2^32
            y0 = fmaxf(fminf(y0, 511101108224.0f), -511101108224.0f);
            y1 = fmaxf(fminf(y1, 511101108224.0f), -511101108224.0f);
        }
        const uint64_t s0 = uint64_t(__float2ll_ru(y0)) + uint64_t(pw[i >> 1] << 16);
        const uint64_t s1 = uint64_t(__float2ll_ru(y1)) + uint64_t(pw[i >> 1] & 0xFFFF0000u);
        qv[i] = int(uint32_t(s0 >> 32));
        qv[i + 1] = int(uint32_t(s1 >> 32));
        L[i] = uint32_t(s0);
        L[i + 1] = uint32_t(s1);
    }
    const uint32_t lmax = max(max(max(L[0], L[1]), max(L[2], L[3])), max(max(L[4], L[5]), max(L[6], L[7])));
    if (__builtin_expect(lmax > 0xFFFF0000u, 0)) {                     // the low halves decide
        const Philox4 pl = philox4x32_10(uint32_t(blk), uint32_t(blk >> 32), kPurposeSRLow, call_id, keys);
        const uint32_t lw[4] = {pl.x, pl.y, pl.z, pl.w};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t h4 = (i & 1) ? (lw[i >> 1] >> 16) : (lw[i >> 1] & 0xFFFFu);
            if (L[i] > 0xFFFF0000u && h4 > ~L[i]) qv[i] += 1;
        }
    }
    const uint32_t c80 = 0x80808080u;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#if I4_GS_PACK
        uint32_t q, q23;                                               // saturating packs (exact: |q| <= 119)
        asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, 0;" : "=r"(q23) : "r"(qv[4 * h + 3]), "r"(qv[4 * h + 2]));
        asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(q) : "r"(qv[4 * h + 1]), "r"(qv[4 * h]), "r"(q23));
#else
        const uint32_t q = __byte_perm(__byte_perm(uint32_t(qv[4 * h]), uint32_t(qv[4 * h + 1]), 0x0040),
                                       __byte_perm(uint32_t(qv[4 * h + 2]), uint32_t(qv[4 * h + 3]), 0x0040), 0x5410);
#endif
        const uint32_t t = (q ^ c80) + 0x08080808u;
        uint32_t hi16;                                                  // (t ^ 0x80) & 0xF0 per byte
        asm("lop3.b32 %0, %1, %2, %3, 0x28;" : "=r"(hi16) : "r"(t), "r"(c80), "r"(0xF0F0F0F0u));
        shi = __dp4a(int(hi16), int(hi16), shi);
        slo = __dp4a(int(t & 0x0F0F0F0Fu), int(t | 0xF0F0F0F0u), slo);
        if (h == 0) pq.x = q; else pq.y = q;
    }
    slo += 8 * 64;
}

// Work unit = G chunks of 256 columns of one row (one 16-byte load of 8 bf16 per
// lane per chunk).  With C % (256 G) == 0 unit u starts at flat element 256 G u,
// so addresses and Philox counters need no division.
//
// Each warp takes a contiguous unit range (keeps the next unit's loads in flight,
// the first ones issued before the phase-1 -> phase-2 wait), accumulates the row
// norms in registers and flushes them (exact int32 atomics onto the zeroed a_sq)
// when the row changes.  (Measured and dropped: a dynamic pool of units claimed
// from a counter -- the per-CTA finish spread is not load imbalance; Philox words
// precomputed into shared memory during phase 1 -- no gain; a software pipeline that
// generates unit u+1's Philox words beside unit u's split, at 2 or 3 CTAs / SM --
// 1-4 % slower; a threshold / floor without the F2I conversion (FADD2.RM magic
// numbers) -- more ALU work, 15 % slower.  Phase 2 is ALU-pipe bound: ~12 LOP3 /
// PRMT / IADD3 per element, 5 of them Philox's XORs.)

// scratch words (uint32 [kGradSplitMaxBlocks], zero before the first call; every
// launch returns them to zero): amax word, arrival / departure counters
constexpr int kAmaxWord = kGradSplitMaxBlocks - 8, kArriveWord = kAmaxWord + 1, kDepartWord = kAmaxWord + 2;

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// last CTA out returns the counters to zero for the next launch (every CTA read
// the amax word and the arrival count before it departed)
__device__ __forceinline__ void depart(uint32_t* scratch) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(scratch + kDepartWord, 1u) == gridDim.x - 1) {
            scratch[kAmaxWord] = 0u;
            scratch[kArriveWord] = 0u;
            scratch[kDepartWord] = 0u;
        }
    }
}

template <int G>
__device__ __forceinline__ void load_unit(const uint4* src, int64_t un, uint4 (&dst)[G]) {
#pragma unroll
    for (int gi = 0; gi < G; ++gi) dst[gi] = ld_nc_v4(src + (un * G + gi) * 32);
}

// One unit: SR words (Philox), codes stored to the Q plane, half-row norms into shi / slo.
template <int G, bool CLAMP, bool C1Z>
__device__ __forceinline__ void split_unit(const uint4 (&cur)[G], int64_t un, const float r8, const PhiloxKeys& keys,
                                           uint32_t call_id, uint64_t tbase, int8_t* __restrict__ q8,
                                           int& shi, int& slo) {
    const int lane = lane_id();
#pragma unroll
    for (int gi = 0; gi < G; ++gi) {
        const int64_t flat = (un * G + gi) * 256 + lane * 8;
        uint2 pq;
        split_chunk8<CLAMP, C1Z>(cur[gi], (tbase + uint64_t(flat)) >> 3, call_id, keys, r8, pq, shi, slo);
        *reinterpret_cast<uint2*>(q8 + flat) = pq;
    }
}

__device__ __forceinline__ void flush_norms(int& shi, int& slo, int32_t* __restrict__ a_sq, int64_t N, int64_t row) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        shi += __shfl_xor_sync(0xFFFFFFFFu, shi, o);
        slo += __shfl_xor_sync(0xFFFFFFFFu, slo, o);
    }
    if (lane_id() == 0) {
        atomicAdd(a_sq + row, shi >> 8);                              // exact: every term is 256 hi^2
        atomicAdd(a_sq + N + row, slo);
    }
    shi = 0; slo = 0;
}

template <int G, bool CLAMP, bool C1Z>
__device__ __forceinline__ void split_units(const uint16_t* __restrict__ g, int64_t N, int C, const float r8,
                                            const PhiloxKeys& keys, uint32_t call_id, int64_t token_offset,
                                            int8_t* __restrict__ q8, int32_t* __restrict__ a_sq, int64_t u0,
                                            int64_t u1, uint4 (&buf)[G]) {
    const int upr = C / (256 * G);                                    // units per row
    const uint4* src = reinterpret_cast<const uint4*>(g) + lane_id();
    const uint64_t tbase = uint64_t(token_offset) * uint64_t(C);       // Z-20: L = (t0 + t) C + c
    int shi = 0, slo = 0;
    // range [u0, u1): its first unit's loads were issued before the phase-1 wait
    if (u0 < u1) {
        int64_t row = u0 / upr;
        int seg = int(u0 - row * upr);
        for (int64_t un = u0; un < u1; ++un) {
            uint4 cur[G];
#pragma unroll
            for (int gi = 0; gi < G; ++gi) cur[gi] = buf[gi];
            if (un + 1 < u1) load_unit<G>(src, un + 1, buf);        // next unit's loads in flight
            split_unit<G, CLAMP, C1Z>(cur, un, r8, keys, call_id, tbase, q8, shi, slo);
            if (++seg == upr || un + 1 == u1) {                       // row done (or range end): flush
                flush_norms(shi, slo, a_sq, N, row);
                seg = 0; ++row;
            }
        }
    }
}

// timing experiment, compiled in only by -DI4_STAMPS=1 (tools/build_variants.sh,
// tools/gs_stamps.py): per-CTA globaltimer stamps -- start, phase 1 done,
// barrier passed, amax known, phase 2 done (max over warps)
#ifndef I4_STAMPS
#define I4_STAMPS 0
#endif
constexpr bool kStamps = I4_STAMPS != 0;
__device__ unsigned long long g_gs_stamp[kStamps ? 5 : 1][kStamps ? kGradSplitMaxBlocks : 1];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

template <int G, bool C1Z>
__global__ void __launch_bounds__(kSplitThreads, I4_BS_MINB)
grad_split_kernel(const uint16_t* __restrict__ g, int64_t N, int C, uint32_t* __restrict__ scratch,
                  const PhiloxKeys keys, uint32_t call_id, int64_t token_offset, int8_t* __restrict__ q8,
                  int32_t* __restrict__ a_sq, float* __restrict__ s_down_out, uint32_t* __restrict__ amax_out,
                  int32_t* __restrict__ status) {
    const int lane = lane_id();
    const int warp = threadIdx.x >> 5;
    pdl_trigger();
    pdl_wait();
    constexpr bool stamp = kStamps;
    if (stamp && threadIdx.x == 0) g_gs_stamp[0][blockIdx.x] = gtimer();

    // ---- phase 1: amax ----------------------------------------------------
    {
        const uint4* g4 = reinterpret_cast<const uint4*>(g);
        const int64_t n8 = N * int64_t(C) / 8;
        const int64_t stride = int64_t(gridDim.x) * blockDim.x;
        uint32_t m = 0;
        for (int64_t i0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i0 < n8; i0 += stride * kAmaxUnroll) {
            uint4 u[kAmaxUnroll];
#pragma unroll
            for (int j = 0; j < kAmaxUnroll; ++j) {
                const int64_t i = i0 + j * stride;
                // streamed past L1: the phase-2 re-reads come from L2 on other SMs
                // (measured equal or faster on every config with a flushed L2)
                u[j] = i < n8 ? ld_nc_v4(g4 + i) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int j = 0; j < kAmaxUnroll; ++j)
                m = max(m, max(max(bf16x2_absmax(u[j].x), bf16x2_absmax(u[j].y)),
                               max(bf16x2_absmax(u[j].z), bf16x2_absmax(u[j].w))));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
        if (G > 0)                                        // the fast phase 2 accumulates norms atomically
            for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < 2 * N; i += stride) a_sq[i] = 0;
        __shared__ uint32_t red[kSplitThreads / 32];
        if (lane == 0) red[warp] = m;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < kSplitThreads / 32; ++w) m = max(m, red[w]);
            // arrive: fold the CTA maximum into the amax word, then count this CTA
            // (the fence orders this CTA's a_sq zeroing and the max before the count)
            atomicMax(scratch + kAmaxWord, m);
            __threadfence();
            atomicAdd(scratch + kArriveWord, 1u);
            if (stamp) g_gs_stamp[1][blockIdx.x] = gtimer();
        }
    }
    // unit range of this warp; its first loads go in flight across the wait
    int64_t pu0 = 0, pu1 = 0;
    uint4 pbuf[G > 0 ? G : 1];
    if constexpr (G > 0) {
        const int64_t units = N * int64_t(C / (256 * G));
        const int64_t nwarps = int64_t(gridDim.x) * (kSplitThreads / 32);
        const int64_t wid = int64_t(blockIdx.x) * (kSplitThreads / 32) + warp;
        pu0 = units * wid / nwarps;
        pu1 = units * (wid + 1) / nwarps;
        if (pu0 < pu1) load_unit<G>(reinterpret_cast<const uint4*>(g) + lane, pu0, pbuf);
    }
    // wait until every CTA arrived (co-resident: cooperative launch), read amax
    __shared__ uint32_t amax_sh;
    if (threadIdx.x == 0) {
        while (ld_acquire_gpu(scratch + kArriveWord) < gridDim.x) __nanosleep(32);
        amax_sh = ld_acquire_gpu(scratch + kAmaxWord);
        if (stamp) g_gs_stamp[2][blockIdx.x] = gtimer();
    }
    __syncthreads();
    const uint32_t amax_b = amax_sh;
    const float amax = __uint_as_float(amax_b << 16);
    // |g| bit patterns >= 0x7F80 are Inf / NaN ("input error"): the
    // device status word gets bit 0 and the tensor is treated as all-zero (codes 0,
    // s_down = 0, no items kept, zero gradients); an all-zero grad_Y sets bit 1
    // ("degenerate")
    const bool nonfinite = amax_b >= 0x7F80u;
    const bool zero = nonfinite || !(amax > 0.0f);
    const float r8 = zero ? 0.0f : __fdiv_rn(119.0f, amax);
    if (stamp && threadIdx.x == 0) { g_gs_stamp[3][blockIdx.x] = gtimer(); g_gs_stamp[4][blockIdx.x] = 0; }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *s_down_out = zero ? 0.0f : __fdiv_rn(amax, 119.0f);
        *amax_out = amax_b;
        if (status != nullptr && zero) atomicOr(status, nonfinite ? kStatusNonFinite : kStatusZeroGrad);
    }

    // ---- phase 2: SR + bit split ------------------------------------------
    if (blockIdx.x == gridDim.x - 1)                      // code row N: the all-zero pad row
        for (int c = threadIdx.x * 16; c < C; c += kSplitThreads * 16)
            *reinterpret_cast<uint4*>(q8 + N * C + c) = make_uint4(0, 0, 0, 0);
    if constexpr (G > 0) {
        if (zero) {                                       // all-zero / non-finite grad_Y: codes 0, norms 0
            for (int64_t un = pu0; un < pu1; ++un)        // (zeroed in phase 1)
#pragma unroll
                for (int gi = 0; gi < G; ++gi)
                    *reinterpret_cast<uint2*>(q8 + (un * G + gi) * 256 + lane * 8) = make_uint2(0u, 0u);
        } else {
            // only elements with |g| = amax can land above 119 (fl32(amax r8) may round up by an ulp)
            if (__fmul_rn(amax, r8) > 119.0f)
                split_units<G, true, C1Z>(g, N, C, r8, keys, call_id, token_offset, q8, a_sq, pu0, pu1, pbuf);
            else
                split_units<G, false, C1Z>(g, N, C, r8, keys, call_id, token_offset, q8, a_sq, pu0, pu1, pbuf);
        }
        if (stamp && lane == 0) atomicMax(&g_gs_stamp[4][blockIdx.x], gtimer());
        depart(scratch);
        return;
    }
    // generic path (C not a multiple of 256): one warp per row
    const int64_t warp0 = int64_t(blockIdx.x) * (kSplitThreads / 32) + warp;
    const int64_t wstride = int64_t(gridDim.x) * (kSplitThreads / 32);
    const int nch = (C + 255) >> 8;
    for (int64_t row = warp0; row < N; row += wstride) {
        const uint16_t* gr = g + row * C;
        int8_t* qr = q8 + row * C;
        const uint64_t tglob = uint64_t(token_offset + row);
        int shi = 0, slo = 0;
        for (int g0 = 0; g0 < nch; g0 += kBsGroup) {
            uint4 raw[kBsGroup];
#pragma unroll
            for (int gi = 0; gi < kBsGroup; ++gi) {
                const int col = (g0 + gi) * 256 + lane * 8;
                raw[gi] = (g0 + gi < nch && col < C) ? ld_nc_v4(gr + col) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int gi = 0; gi < kBsGroup; ++gi) {
                const int col = (g0 + gi) * 256 + lane * 8;
                if (g0 + gi >= nch || col >= C) continue;
                uint2 qp = make_uint2(0u, 0u);
                if (!zero)                                             // L = tglob C + col (Z-20)
                    split_chunk8<true, C1Z>(raw[gi], (tglob * uint64_t(C) + uint64_t(col)) >> 3, call_id, keys, r8,
                                            qp, shi, slo);
                *reinterpret_cast<uint2*>(qr + col) = qp;              // the 8-bit code plane Q
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            shi += __shfl_xor_sync(0xFFFFFFFFu, shi, o);
            slo += __shfl_xor_sync(0xFFFFFFFFu, slo, o);
        }
        if (lane == 0) {
            a_sq[row] = shi >> 8;                             // exact: every term is 256 hi^2
            a_sq[N + row] = slo;
        }
    }
    depart(scratch);
}

template <int G, bool C1Z>
static int grad_split_max_blocks() {
    static std::atomic<int> cached[kMaxDevices];        // per device ordinal (0 = not yet queried)
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDevices) dev = 0;
    int v = cached[dev].load(std::memory_order_relaxed);
    if (v == 0) {
        int per_sm = 0, sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, grad_split_kernel<G, C1Z>, kSplitThreads, 0);
        v = per_sm * sms;
        cached[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

int grad_split_max_blocks() { return grad_split_max_blocks<0, false>(); }

template <int G, bool C1Z>
static cudaError_t launch_grad_split_g(const uint16_t* g, int64_t N, int C, uint32_t* block_max, const PhiloxKeys& keys,
                                       uint32_t call_id, int64_t token_offset, int8_t* q8, int32_t* a_sq,
                                       float* s_down, uint32_t* amax_out, int32_t* status, cudaStream_t s) {
    int blocks = grad_split_max_blocks<G, C1Z>();
    const int64_t want = G > 0 ? (N * (C / (256 * G)) + 7) / 8 : (N + 7) / 8;   // one warp per unit at most
    if (want < blocks) blocks = int(want);
    if (blocks > kAmaxWord) blocks = kAmaxWord;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(blocks));
    cfg.blockDim = dim3(kSplitThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = add_pdl_attr(attr, 1);
    cudaError_t e = cudaLaunchKernelEx(&cfg, grad_split_kernel<G, C1Z>, g, N, C, block_max, keys, call_id,
                                       token_offset, q8, a_sq, s_down, amax_out, status);
    if (e != cudaSuccess && cfg.numAttrs == 2) {       // cooperative + PDL refused: plain cooperative
        (void)cudaGetLastError();
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, grad_split_kernel<G, C1Z>, g, N, C, block_max, keys, call_id, token_offset,
                               q8, a_sq, s_down, amax_out, status);
    }
    return e;
}

template <int G>
static cudaError_t launch_grad_split_c(const uint16_t* g, int64_t N, int C, uint32_t* block_max,
                                       const PhiloxKeys& keys, uint32_t call_id, int64_t token_offset, int8_t* q8,
                                       int32_t* a_sq, float* s_down, uint32_t* amax_out, int32_t* status,
                                       cudaStream_t s) {
    // every SR block index L / 8 below 2^32 (L < (token_offset + N) C): Philox counter word c1 = 0
    const bool c1z = (uint64_t(token_offset) + uint64_t(N)) * uint64_t(C) <= (uint64_t(1) << 35);
    if (c1z)
        return launch_grad_split_g<G, true>(g, N, C, block_max, keys, call_id, token_offset, q8, a_sq, s_down,
                                            amax_out, status, s);
    return launch_grad_split_g<G, false>(g, N, C, block_max, keys, call_id, token_offset, q8, a_sq, s_down,
                                         amax_out, status, s);
}

cudaError_t launch_grad_split(const uint16_t* g, int64_t N, int64_t C, uint32_t* block_max, uint64_t seed,
                              uint32_t call_id, int64_t token_offset, int8_t* q8, int32_t* a_sq, float* s_down,
                              uint32_t* amax_out, int32_t* status, cudaStream_t s) {
    if (N == 0) return cudaSuccess;
    const PhiloxKeys keys = philox_keys(uint32_t(seed), uint32_t(seed >> 32));
    const int Ci = int(C);
#define I4_GS(GG) launch_grad_split_c<GG>(g, N, Ci, block_max, keys, call_id, token_offset, q8, a_sq, s_down, amax_out, status, s)
    // unit size: 2 chunks when C allows (no register spills at 3 CTAs / SM; 4 and 3
    // measured equal or slower), else 3, 1; the one-warp-per-row loop otherwise
    if (kBsGMax >= 2 && C % 512 == 0) return I4_GS(2);
    if (kBsGMax >= 3 && C % 768 == 0) return I4_GS(3);
    if (C % 256 == 0) return I4_GS(1);
#undef I4_GS
    return launch_grad_split_c<0>(g, N, Ci, block_max, keys, call_id, token_offset, q8, a_sq, s_down, amax_out,
                                  status, s);
}

// ---------------------------------------------------------------------------
// Batched grad_split (attention BMM, reading Z-31): rows [b nb, (b+1) nb) are batch b,
// with its own amax, s_down and [2 nb] norm block.  Two launches and no grid-wide
// barrier (a cooperative barrier and one cluster per batch both measured slower on the
// BMM shapes: the SR pass needs every SM and many warps, the batches are small):
//   batch_amax_kernel   warp w takes R consecutive rows; its running max goes to the
//                       batch's word by atomicMax when the batch changes (the words are
//                       zero on entry: the sampler launch of the previous call zeroes them)
//   batch_split_kernel  warp per row: r8 of the row's batch, Philox SR codes, half-row
//                       norms stored directly; CTA 0 writes s_down[b] / amax[b] / status
constexpr int kBatchSplitKB = 4;                 // 256-column chunks per lane in flight

__global__ void __launch_bounds__(256)
batch_amax_kernel(const uint16_t* __restrict__ g, int64_t rows, int C, int64_t nb, int R,
                  uint32_t* __restrict__ bamax) {
    pdl_trigger();
    pdl_wait();
    const int lane = lane_id();
    const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t r0 = w * R, r1 = min(rows, r0 + R);
    if (r0 >= rows) return;
    const int c8 = C / 8;
    uint32_t m = 0;
    int64_t cb = r0 / nb;
    auto flush = [&](int64_t b) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
        if (lane == 0) atomicMax(bamax + b, m);
        m = 0;
    };
    for (int64_t row = r0; row < r1; ++row) {
        if (row / nb != cb) { flush(cb); cb = row / nb; }
        const uint4* g4 = reinterpret_cast<const uint4*>(g + row * C);
        for (int i0 = lane; i0 < c8; i0 += 32 * kBatchSplitKB) {
            uint4 u[kBatchSplitKB];
#pragma unroll
            for (int q = 0; q < kBatchSplitKB; ++q)
                u[q] = i0 + 32 * q < c8 ? ld_nc_v4(g4 + i0 + 32 * q) : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int q = 0; q < kBatchSplitKB; ++q)
                m = max(m, max(max(bf16x2_absmax(u[q].x), bf16x2_absmax(u[q].y)),
                               max(bf16x2_absmax(u[q].z), bf16x2_absmax(u[q].w))));
        }
    }
    flush(cb);
}

template <bool C1Z>
__global__ void __launch_bounds__(256)
batch_split_kernel(const uint16_t* __restrict__ g, int64_t rows, int C, int64_t nb, const PhiloxKeys keys,
                   uint32_t call_id, int64_t token_offset, int8_t* __restrict__ q8, int32_t* __restrict__ a_sq,
                   float* __restrict__ s_down_out, uint32_t* __restrict__ amax_out, int32_t* __restrict__ status,
                   const uint32_t* __restrict__ bamax) {
    pdl_trigger();
    pdl_wait();                                   // the batch amax words
    const int lane = lane_id();
    if (blockIdx.x == 0)
        for (int64_t b = threadIdx.x; b < rows / nb; b += blockDim.x) {
            const uint32_t ab = bamax[b];
            const float am = __uint_as_float(ab << 16);
            const bool nf = ab >= 0x7F80u, zr = nf || !(am > 0.0f);
            s_down_out[b] = zr ? 0.0f : __fdiv_rn(am, 119.0f);
            amax_out[b] = ab;
            if (status != nullptr && zr) atomicOr(status, nf ? kStatusNonFinite : kStatusZeroGrad);
        }
    if (blockIdx.x == gridDim.x - 1)               // code row B nb: the all-zero pad row
        for (int c = threadIdx.x * 16; c < C; c += blockDim.x * 16)
            *reinterpret_cast<uint4*>(q8 + rows * C + c) = make_uint4(0, 0, 0, 0);
    const uint64_t tbase = uint64_t(token_offset) * uint64_t(C);
    const int64_t nwarps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; row < rows; row += nwarps) {
        const int64_t b = row / nb;
        const uint32_t ab = bamax[b];
        const float amax = __uint_as_float(ab << 16);
        const bool zero = ab >= 0x7F80u || !(amax > 0.0f);
        const float r8 = zero ? 0.0f : __fdiv_rn(119.0f, amax);
        int shi = 0, slo = 0;
        for (int c0 = 0; c0 < C; c0 += 256 * kBatchSplitKB) {
            uint4 u[kBatchSplitKB];
#pragma unroll
            for (int q = 0; q < kBatchSplitKB; ++q) {
                const int col = c0 + 256 * q + lane * 8;
                u[q] = col < C ? ld_nc_v4(g + row * C + col) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int q = 0; q < kBatchSplitKB; ++q) {
                const int col = c0 + 256 * q + lane * 8;
                if (col >= C) break;
                const int64_t flat = row * C + col;
                uint2 pq = make_uint2(0u, 0u);
                if (!zero) {
                    split_chunk8<true, C1Z>(u[q], (tbase + uint64_t(flat)) >> 3, call_id, keys, r8, pq, shi, slo);
                }
                *reinterpret_cast<uint2*>(q8 + flat) = pq;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            shi += __shfl_xor_sync(0xFFFFFFFFu, shi, o);
            slo += __shfl_xor_sync(0xFFFFFFFFu, slo, o);
        }
        if (lane == 0) {
            const int64_t lr = row - b * nb;
            a_sq[b * 2 * nb + lr] = shi >> 8;                          // exact: every term is 256 hi^2
            a_sq[b * 2 * nb + nb + lr] = slo;
        }
    }
}

cudaError_t launch_grad_split_batched(const uint16_t* g, int64_t rows, int64_t C, int64_t nb, uint64_t seed,
                                      uint32_t call_id, int64_t token_offset, int8_t* q8, int32_t* a_sq,
                                      float* s_down, uint32_t* amax_out, int32_t* status, uint32_t* bamax,
                                      cudaStream_t s) {
    if (rows == 0) return cudaSuccess;
    static std::atomic<int> sms_cache[kMaxDevices];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDevices) dev = 0;
    int sms = sms_cache[dev].load(std::memory_order_relaxed);
    if (sms == 0) {
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        sms_cache[dev].store(sms, std::memory_order_relaxed);
    }
    // amax: R consecutive rows per warp, about 32 warps per SM
    const int64_t target_warps = int64_t(sms) * 32;
    const int R = int(std::max<int64_t>(1, (rows + target_warps - 1) / target_warps));
    const int64_t warps_a = (rows + R - 1) / R;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned((warps_a + 7) / 8));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    cfg.attrs = attr;
    cfg.numAttrs = add_pdl_attr(attr, 0);
    cudaError_t e = cudaLaunchKernelEx(&cfg, batch_amax_kernel, g, rows, int(C), nb, R, bamax);
    if (e != cudaSuccess) return e;
    // split: one warp per row (grid-stride beyond 16 warps per SM)
    const int64_t blocks = std::min<int64_t>((rows + 7) / 8, int64_t(sms) * 8);
    cfg.gridDim = dim3(unsigned(blocks));
    const PhiloxKeys keys = philox_keys(uint32_t(seed), uint32_t(seed >> 32));
    const bool c1z = (uint64_t(token_offset) + uint64_t(rows)) * uint64_t(C) <= (uint64_t(1) << 35);
    if (c1z)
        return cudaLaunchKernelEx(&cfg, batch_split_kernel<true>, g, rows, int(C), nb, keys, call_id, token_offset,
                                  q8, a_sq, s_down, amax_out, status, static_cast<const uint32_t*>(bamax));
    return cudaLaunchKernelEx(&cfg, batch_split_kernel<false>, g, rows, int(C), nb, keys, call_id, token_offset, q8,
                              a_sq, s_down, amax_out, status, static_cast<const uint32_t*>(bamax));
}

// debug export for the timing experiment: copies the stamps of the last launch
// ([5][n] u64, n <= kGradSplitMaxBlocks) to host memory (-DI4_STAMPS=1 builds only)
int grad_split_stamps(unsigned long long* host, int n) {
    if (!kStamps) return -1;
    if (n > kGradSplitMaxBlocks) n = kGradSplitMaxBlocks;
    for (int r = 0; r < 5; ++r)
        if (cudaMemcpyFromSymbol(host + size_t(r) * n, g_gs_stamp, sizeof(unsigned long long) * n,
                                 sizeof(unsigned long long) * kGradSplitMaxBlocks * r) != cudaSuccess)
            return -1;
    return n;
}

}  // namespace i4
