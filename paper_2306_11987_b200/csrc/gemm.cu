// INT8 x INT8 -> INT32 GEMM on the 5th-generation tensor cores, used for every
// "INT4 MM" of the operator.  INT4
// codes are stored sign-extended in int8 (sm_100a has no s4 tcgen05 kind), so
// tcgen05.mma.kind::i8 is exact for them; accumulation is int32 in TMEM.
//
//   acc[m, n] = sum_k A[m, k] B[n, k]      (A, B K-major: rows of K bytes)
//
// Structure (one CTA per SM, persistent over output tiles, warp-specialised):
//   warp 0   TMA producer: 128-byte-swizzled A (128 x 128 B) and B (BN x 128 B)
//            tiles into a STAGES-deep shared-memory ring (mbarrier full/empty).
//   warp 1   allocates 2 x BN TMEM columns; one lane issues tcgen05.mma
//            (M = 128, N = BN, K = 32 per instruction, 4 per 128-byte k-block)
//            and tcgen05.commit to release smem stages / publish accumulators.
//   warps 2-5  epilogue: tcgen05.ld 32 lanes x 32 columns -> registers, then
//            EPI_INT32  raw accumulators (bit-exact parity checks)
//            EPI_FWD    Y = fl32(acc) * fl32(s_x s_w)   (HQ-MM step 4)
//            EPI_DGRAD  row = kept item (h, t): v = acc * s_w s_h 2^wexp 2^{-k/2};
//                       v = I_X[t] o v; v = v H (in-register FWHT); red.add into
//                       dX[t] (<= 2 addends per element onto 0: order-independent)
//            EPI_WGRAD  v = acc * s_x s_down 2^{-k/2}; v = I_W o v; v = v H; store dW
//   Two TMEM accumulator stages let the epilogue of tile i overlap the MMAs of
//   tile i+1.  M (grad_X: kept items) or K (grad_W: kept items) may be read
//   from device memory, so the sampled sizes never travel to the host.
#include <cuda.h>

#include "common.cuh"
#include "kernels.h"

namespace i4 {

constexpr int kBM = 128;
constexpr int kBK = 128;                     // bytes = int8 elements along K per stage
constexpr int kGemmThreads = 192;
constexpr int kRingBytes = 192 * 1024;

template <int BN>
struct GemmCfg {
    static constexpr int A_BYTES = kBM * kBK;
    static constexpr int B_BYTES = BN * kBK;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int STAGES = kRingBytes / STAGE_BYTES;
    static constexpr int TMEM_COLS = 2 * BN;
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

template <int BN, int EPI, int CH>
__global__ void __launch_bounds__(kGemmThreads, 1)
gemm_i8_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const GemmArgs g) {
    using Cfg = GemmCfg<BN>;
    constexpr int STAGES = Cfg::STAGES;
    extern __shared__ uint8_t smem_dyn[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = base;
    uint8_t* sB = base + STAGES * Cfg::A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(base + STAGES * Cfg::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // problem size (possibly data-dependent)
    const int M = g.m_dev ? __ldg(g.m_dev) : g.M;
    const int K = g.k_dev ? ((__ldg(g.k_dev) + kBK - 1) / kBK) * kBK : g.K;
    const int m_tiles = (M + kBM - 1) / kBM;
    const int n_tiles = g.Nn / BN;
    const int total = m_tiles * n_tiles;
    const int nk = (K + kBK - 1) / kBK;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 4 * 32); }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------- producer
        if (lane == 0) {
            int stage = 0; uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
                const int m0 = (tile / n_tiles) * kBM, n0 = (tile % n_tiles) * BN;
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
                    tma_load_2d(sA + stage * Cfg::A_BYTES, &tmA, &full[stage], kb * kBK, m0);
                    tma_load_2d(sB + stage * Cfg::B_BYTES, &tmB, &full[stage], kb * kBK, n0);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------- MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_i8(kBM, BN);
            int stage = 0; uint32_t phase = 0; int it = 0;
            for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
                const int as = it & 1;
                const uint32_t ap = (it >> 1) & 1;
                mbar_wait(&tempty[as], ap ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + uint32_t(as * BN);
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint64_t adesc = sdesc_kmajor_sw128(smem_u32(sA + stage * Cfg::A_BYTES));
                    const uint64_t bdesc = sdesc_kmajor_sw128(smem_u32(sB + stage * Cfg::B_BYTES));
#pragma unroll
                    for (int kk = 0; kk < kBK / 32; ++kk)
                        umma_i8(d_tmem, adesc + uint64_t(kk * 2), bdesc + uint64_t(kk * 2), idesc,
                                (kb | kk) != 0 ? 1u : 0u);
                    umma_commit(&empty[stage]);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                umma_commit(&tfull[as]);
            }
        }
    } else {
        // ------------------------------------------------------------- epilogue
        const int lg = warp & 3;                       // TMEM lane group of this warp
        const int r_in_tile = lg * 32 + lane;
        const int words = g.Nn >> 5;
        float sd = 1.0f;
        if (EPI == EPI_DGRAD || EPI == EPI_WGRAD) sd = __ldg(g.s_down);
        int it = 0;
        for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
            const int as = it & 1;
            const uint32_t ap = (it >> 1) & 1;
            const int m0 = (tile / n_tiles) * kBM, n0 = (tile % n_tiles) * BN;
            const int row = m0 + r_in_tile;
            mbar_wait(&tfull[as], ap);
            tc_fence_after();
            const uint32_t t_row = tmem_base + (uint32_t(lg * 32) << 16) + uint32_t(as * BN);

            // per-row setup
            bool valid = row < M;
            int64_t out_row = row;
            float rscale = g.scale;
            if (EPI == EPI_DGRAD) {
                const int item = valid ? __ldg(g.items + row) : 2 * g.n_tokens;
                valid = valid && item < 2 * g.n_tokens;
                const int h = item >= g.n_tokens ? 1 : 0;
                out_row = item - h * g.n_tokens;
                const int e = valid ? int(__ldg(g.wexp + row)) : 0;
                rscale = ldexpf(__fmul_rn(g.scale, sd), e + (h == 0 ? 4 : 0));
            } else if (EPI == EPI_WGRAD) {
                rscale = __fmul_rn(g.scale, sd);
            }

#pragma unroll 1
            for (int c = 0; c < BN; c += CH) {
                uint32_t r[CH / 32][32];
#pragma unroll
                for (int q = 0; q < CH / 32; ++q) tmem_ld_32x32b_x32(t_row + uint32_t(c + 32 * q), r[q]);
                tmem_ld_wait();
                if (nk == 0) {
#pragma unroll
                    for (int q = 0; q < CH / 32; ++q)
#pragma unroll
                        for (int i = 0; i < 32; ++i) r[q][i] = 0;
                }
                const int col0 = n0 + c;
                if (EPI == EPI_INT32) {
                    if (valid) {
                        int32_t* dst = reinterpret_cast<int32_t*>(g.out) + out_row * g.Nn + col0;
#pragma unroll
                        for (int i = 0; i < 32; i += 4)
                            *reinterpret_cast<int4*>(dst + i) = make_int4(r[0][i], r[0][i + 1], r[0][i + 2], r[0][i + 3]);
                    }
                } else if (EPI == EPI_FWD) {
                    if (valid) {
                        float v[32];
#pragma unroll
                        for (int i = 0; i < 32; ++i) v[i] = __fmul_rn(float(int32_t(r[0][i])), rscale);
                        if (g.out_bf16) {
                            __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(g.out) + out_row * g.Nn + col0;
#pragma unroll
                            for (int i = 0; i < 32; i += 8) {
                                uint4 u;
                                __nv_bfloat162 p0 = __floats2bfloat162_rn(v[i], v[i + 1]);
                                __nv_bfloat162 p1 = __floats2bfloat162_rn(v[i + 2], v[i + 3]);
                                __nv_bfloat162 p2 = __floats2bfloat162_rn(v[i + 4], v[i + 5]);
                                __nv_bfloat162 p3 = __floats2bfloat162_rn(v[i + 6], v[i + 7]);
                                u.x = *reinterpret_cast<uint32_t*>(&p0); u.y = *reinterpret_cast<uint32_t*>(&p1);
                                u.z = *reinterpret_cast<uint32_t*>(&p2); u.w = *reinterpret_cast<uint32_t*>(&p3);
                                *reinterpret_cast<uint4*>(dst + i) = u;
                            }
                        } else {
                            float* dst = reinterpret_cast<float*>(g.out) + out_row * g.Nn + col0;
#pragma unroll
                            for (int i = 0; i < 32; i += 4)
                                *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                        }
                    }
                } else {
                    // DGRAD / WGRAD: scale, clamp mask, inverse block Hadamard, write
                    if (valid) {
                        float v[CH];
#pragma unroll
                        for (int q = 0; q < CH / 32; ++q) {
                            const uint32_t mw = __ldg(g.mask + out_row * words + (col0 >> 5) + q);
#pragma unroll
                            for (int i = 0; i < 32; ++i)
                                v[32 * q + i] = ((mw >> i) & 1u) ? __fmul_rn(float(int32_t(r[q][i])), rscale) : 0.0f;
                        }
                        fwht_inplace<CH>(v, g.k_had);
                        float* dst = reinterpret_cast<float*>(g.out) + out_row * g.Nn + col0;
                        if (EPI == EPI_DGRAD) {
#pragma unroll
                            for (int i = 0; i < CH; i += 4)
                                atomicAdd(reinterpret_cast<float4*>(dst + i), make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]));
                        } else {
#pragma unroll
                            for (int i = 0; i < CH; i += 4)
                                *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                        }
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[as]);
        }
    }

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
}

int gemm_block_n(int Nn) {
    if (Nn % 256 == 0) return 256;
    if (Nn % 128 == 0) return 128;
    return 64;
}

template <int BN, int EPI, int CH>
static cudaError_t launch_one(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& g, int grid, cudaStream_t s) {
    auto kern = gemm_i8_kernel<BN, EPI, CH>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<BN>::SMEM);
    if (e != cudaSuccess) return e;
    kern<<<grid, kGemmThreads, GemmCfg<BN>::SMEM, s>>>(a, b, g);
    return cudaGetLastError();
}

template <int BN>
static cudaError_t dispatch_epi(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& g, int grid, cudaStream_t s) {
    const int ch = g.k_had >= 7 ? 128 : (g.k_had == 6 ? 64 : 32);
    switch (g.epi) {
        case EPI_INT32: return launch_one<BN, EPI_INT32, 32>(a, b, g, grid, s);
        case EPI_FWD: return launch_one<BN, EPI_FWD, 32>(a, b, g, grid, s);
        case EPI_DGRAD:
            if (ch == 32) return launch_one<BN, EPI_DGRAD, 32>(a, b, g, grid, s);
            if (ch == 64) return launch_one<BN, EPI_DGRAD, 64>(a, b, g, grid, s);
            if constexpr (BN >= 128) return launch_one<BN, EPI_DGRAD, 128>(a, b, g, grid, s);
            return cudaErrorInvalidValue;
        case EPI_WGRAD:
            if (ch == 32) return launch_one<BN, EPI_WGRAD, 32>(a, b, g, grid, s);
            if (ch == 64) return launch_one<BN, EPI_WGRAD, 64>(a, b, g, grid, s);
            if constexpr (BN >= 128) return launch_one<BN, EPI_WGRAD, 128>(a, b, g, grid, s);
            return cudaErrorInvalidValue;
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_gemm(const void* tmap_a, const void* tmap_b, const GemmArgs& g, int num_sms, cudaStream_t s) {
    const CUtensorMap& a = *reinterpret_cast<const CUtensorMap*>(tmap_a);
    const CUtensorMap& b = *reinterpret_cast<const CUtensorMap*>(tmap_b);
    const int bn = gemm_block_n(g.Nn);
    const int64_t tiles = int64_t((g.M + kBM - 1) / kBM) * (g.Nn / bn);   // g.M = upper bound when m_dev
    int grid = int(tiles < num_sms ? tiles : num_sms);
    if (grid < 1) grid = 1;
    switch (bn) {
        case 256: return dispatch_epi<256>(a, b, g, grid, s);
        case 128: return dispatch_epi<128>(a, b, g, grid, s);
        default: return dispatch_epi<64>(a, b, g, grid, s);
    }
}

}  // namespace i4
