// Memory-bound quantizer kernels (HBM roofline):
//   hadamard_quant : F1+F2 / F3 -- block FWHT + LSQ (Eq. 2);
//                    X and W are quantized by ONE launch (two row jobs)
//   amax_bf16      : B1 -- per-tensor max |grad_Y| (reading Z-9)
//   bitsplit       : B2 -- Philox SR to the 8-bit code, split into high / low
//                    4-bit planes, per-row integer norms
//
// Thread layout shared by the row kernels: one warp per row; the row is walked
// in 256-column chunks, lane l owning columns [c0 + 8 l, c0 + 8 l + 8) so each
// warp-wide 16-byte load covers 512 contiguous bytes.  All loads of a group of
// chunks are issued before any is consumed (memory-level parallelism: one DRAM
// latency per group instead of one per chunk).  Hadamard blocks of 2^k <= 8
// columns are transformed in registers; larger blocks (k = 4..7) add
// xor-shuffle butterfly stages across lanes 1, 2, 4, 8 apart.
#include "common.cuh"
#include "kernels.h"

namespace i4 {

constexpr int kRowWarps = 8;            // warps per CTA in the row kernels

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

static int row_grid(int64_t rows) {
    int64_t blocks = (rows + kRowWarps - 1) / kRowWarps;
    const int64_t cap = 148 * 8;        // 8 resident CTAs of 256 threads per SM
    return int(blocks < cap ? blocks : cap);
}

// ---------------------------------------------------------------------------
// hadamard_quant
// ---------------------------------------------------------------------------
struct HqJob {
    const uint16_t* x;
    int64_t rows;
    float r;
    int8_t* codes;
    uint32_t* bits;
    int32_t* sqnorm;
    int blocks;                          // CTAs assigned to this job
};

constexpr int kHqGroup = 4;              // chunks (of 256 columns) loaded per group

__global__ void __launch_bounds__(kRowWarps * 32, 4)
hadamard_quant_kernel(HqJob j0, HqJob j1, int cols, int k) {
    const bool second = int(blockIdx.x) >= j0.blocks;
    const HqJob& J = second ? j1 : j0;
    const int bid = second ? int(blockIdx.x) - j0.blocks : int(blockIdx.x);
    const int lane = lane_id();
    const int64_t warp0 = int64_t(bid) * kRowWarps + (threadIdx.x >> 5);
    const int64_t wstride = int64_t(J.blocks) * kRowWarps;
    const int words_per_row = cols >> 5;
    const int nch = (cols + 255) >> 8;
    for (int64_t row = warp0; row < J.rows; row += wstride) {
        const uint16_t* xr = J.x + row * cols;
        int sq = 0;
        for (int g0 = 0; g0 < nch; g0 += kHqGroup) {
            uint4 raw[kHqGroup];
#pragma unroll
            for (int g = 0; g < kHqGroup; ++g) {
                const int col = (g0 + g) * 256 + lane * 8;
                raw[g] = (g0 + g < nch && col < cols) ? ld_nc_v4(xr + col) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int g = 0; g < kHqGroup; ++g) {
                if (g0 + g >= nch) break;
                const int col = (g0 + g) * 256 + lane * 8;
                const bool active = col < cols;
                float v[8];
                unpack_bf16x8(raw[g], v);
                // in-register butterflies: strides 1, 2, 4
#pragma unroll
                for (int s = 0; s < 3; ++s) {
                    if (s < k) {
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            if (((i >> s) & 1) == 0) {
                                const float a = v[i], b = v[i + (1 << s)];
                                v[i] = __fadd_rn(a, b);
                                v[i + (1 << s)] = __fsub_rn(a, b);
                            }
                        }
                    }
                }
                // cross-lane butterflies: strides 8, 16, 32, 64 columns = lanes 1, 2, 4, 8 apart
#pragma unroll
                for (int s = 3; s < 7; ++s) {
                    if (s < k) {
                        const int lm = 1 << (s - 3);
                        const float sgn = (lane & lm) ? -1.0f : 1.0f;   // upper lane: o - v, lower: v + o
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const float o = __shfl_xor_sync(0xFFFFFFFFu, v[i], lm);
                            v[i] = __fmaf_rn(sgn, v[i], o);              // one rounding, = the add/sub
                        }
                    }
                }
                // LSQ: v = fl32(t * r); code = clamp(rint(v), -7, 7); mask = -7 <= v <= 7
                int q[8];
                uint32_t m8 = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float sv = __fmul_rn(v[i], J.r);
                    const int c = __float2int_rn(fminf(fmaxf(sv, -7.0f), 7.0f));
                    q[i] = c;
                    m8 |= uint32_t(fabsf(sv) <= 7.0f) << i;
                    sq += c * c;
                }
                // 32-column mask word = 4 lanes x 8 bits
                uint32_t word = m8 << (8 * (lane & 3));
                word |= __shfl_xor_sync(0xFFFFFFFFu, word, 1);
                word |= __shfl_xor_sync(0xFFFFFFFFu, word, 2);
                if (active) {
                    *reinterpret_cast<uint2*>(J.codes + row * cols + col) =
                        make_uint2(pack4_i8(q[0], q[1], q[2], q[3]), pack4_i8(q[4], q[5], q[6], q[7]));
                    if (J.bits != nullptr && (lane & 3) == 0) J.bits[row * words_per_row + (col >> 5)] = word;
                }
            }
        }
        if (J.sqnorm != nullptr) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xFFFFFFFFu, sq, o);
            if (lane == 0) J.sqnorm[row] = sq;
        }
    }
}

cudaError_t launch_hadamard_quant2(const HqArgs& a, cudaStream_t s) {
    HqJob j0{a.x0, a.rows0, a.r0, a.codes0, a.bits0, a.sqnorm0, 0};
    HqJob j1{a.x1, a.rows1, a.r1, a.codes1, a.bits1, a.sqnorm1, 0};
    j0.blocks = a.rows0 > 0 ? row_grid(a.rows0) : 0;
    j1.blocks = a.rows1 > 0 ? row_grid(a.rows1) : 0;
    const int grid = j0.blocks + j1.blocks;
    if (grid == 0) return cudaSuccess;
    hadamard_quant_kernel<<<grid, kRowWarps * 32, 0, s>>>(j0, j1, int(a.cols), a.k);
    return cudaGetLastError();
}

cudaError_t launch_hadamard_quant(const uint16_t* x, int64_t rows, int64_t cols, int k, float r,
                                  int8_t* codes, uint32_t* bits, int32_t* sqnorm, cudaStream_t s) {
    HqArgs a{};
    a.x0 = x; a.rows0 = rows; a.r0 = r; a.codes0 = codes; a.bits0 = bits; a.sqnorm0 = sqnorm;
    a.cols = cols; a.k = k;
    return launch_hadamard_quant2(a, s);
}

// ---------------------------------------------------------------------------
// amax of a bf16 tensor: max over |g| as bf16 bit patterns (non-negative bf16
// values order like their 15-bit integers), exact and order-independent.
// ---------------------------------------------------------------------------
constexpr int kAmaxUnroll = 4;

__global__ void __launch_bounds__(256) amax_bf16_kernel(const uint4* __restrict__ g, int64_t n8,
                                                        uint32_t* __restrict__ amax_bits) {
    uint32_t m = 0;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i0 < n8; i0 += stride * kAmaxUnroll) {
        uint4 u[kAmaxUnroll];
#pragma unroll
        for (int j = 0; j < kAmaxUnroll; ++j) {
            const int64_t i = i0 + j * stride;
            u[j] = i < n8 ? ld_nc_v4(g + i) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int j = 0; j < kAmaxUnroll; ++j) {
            const uint32_t w[4] = {u[j].x, u[j].y, u[j].z, u[j].w};
#pragma unroll
            for (int q = 0; q < 4; ++q) m = max(m, max(w[q] & 0x7FFFu, (w[q] >> 16) & 0x7FFFu));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
    __shared__ uint32_t red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < int(blockDim.x >> 5); ++w) m = max(m, red[w]);
        atomicMax(amax_bits, m);
    }
}

cudaError_t launch_amax_bf16(const uint16_t* g, int64_t n, uint32_t* amax_bits, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(amax_bits, 0, sizeof(uint32_t), s);
    if (e != cudaSuccess) return e;
    const int64_t n8 = n / 8;           // n is a multiple of 64 (C % 64 == 0)
    if (n8 == 0) return cudaSuccess;
    int64_t blocks = (n8 + 256 * kAmaxUnroll - 1) / (256 * kAmaxUnroll);
    if (blocks > 148 * 8) blocks = 148 * 8;
    amax_bf16_kernel<<<int(blocks), 256, 0, s>>>(reinterpret_cast<const uint4*>(g), n8, amax_bits);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// bitsplit: v = clamp(fl32(g r8), -119, 119); sign-magnitude stochastic
// rounding with Philox word u: q = sign(v) (floor|v| + [u < ceil(frac|v| 2^32)]);
// hi = floor((q + 8) / 16), lo = q - 16 hi  (readings Z-9, Z-10, Z-11).
// ---------------------------------------------------------------------------
constexpr int kBsGroup = 4;

__global__ void __launch_bounds__(kRowWarps * 32, 4)
bitsplit_kernel(const uint16_t* __restrict__ g, int64_t N, int C, const uint32_t* __restrict__ amax_bits,
                uint32_t k0, uint32_t k1, uint32_t call_id, int64_t token_offset,
                int8_t* __restrict__ hilo, int32_t* __restrict__ a_sq, float* __restrict__ s_down_out) {
    const int lane = lane_id();
    const float amax = __uint_as_float(__ldg(amax_bits) << 16);
    const bool zero = !(amax > 0.0f);
    const float r8 = zero ? 0.0f : __fdiv_rn(119.0f, amax);
    if (blockIdx.x == 0 && threadIdx.x == 0) *s_down_out = zero ? 0.0f : __fdiv_rn(amax, 119.0f);
    const int64_t warp0 = int64_t(blockIdx.x) * kRowWarps + (threadIdx.x >> 5);
    const int64_t wstride = int64_t(gridDim.x) * kRowWarps;
    const int nch = (C + 255) >> 8;
    const PhiloxKeys keys = philox_keys(k0, k1);
    for (int64_t row = warp0; row < N; row += wstride) {
        const uint16_t* gr = g + row * C;
        int8_t* hr = hilo + row * C;
        int8_t* lr = hilo + (N + row) * C;
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
                float v[8];
                unpack_bf16x8(raw[gi], v);
                // Philox words for the 8 elements: L = tglob * C + col + i, block L / 4
                const uint64_t b0 = (tglob * uint64_t(C) + uint64_t(col)) >> 2;
                const Philox4 p0 = philox4x32_10(uint32_t(b0), uint32_t(b0 >> 32), kPurposeSR, call_id, keys);
                const Philox4 p1 = philox4x32_10(uint32_t(b0 + 1), uint32_t((b0 + 1) >> 32), kPurposeSR, call_id, keys);
                const uint32_t u[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
                int hi[8], lo[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    int q = 0;
                    if (!zero) {
                        // A = ceil(|v| 2^32) (|v| 2^32 is exact in fp32): high word = floor|v|
                        // (+1 when the fraction's threshold wraps to 2^32), low word =
                        // T = ceil(frac|v| 2^32) mod 2^32; P(round up) = T / 2^32 exactly.
                        // a = min(|g r8|, 119); floor / fraction exact in fp32; T = ceil(f 2^32) < 2^32
                        const float sv = __fmul_rn(v[i], r8);
                        const float a = fminf(fabsf(sv), 119.0f);
                        const float fl = floorf(a);
                        const uint32_t T = __float2uint_ru(__fmul_rn(__fsub_rn(a, fl), 4294967296.0f));
                        const int mag = int(fl) + int(u[i] < T);
                        q = sv < 0.0f ? -mag : mag;
                    }
                    hi[i] = (q + 8) >> 4;                                     // floor division
                    lo[i] = q - 16 * hi[i];
                    shi += hi[i] * hi[i];
                    slo += lo[i] * lo[i];
                }
                *reinterpret_cast<uint2*>(hr + col) =
                    make_uint2(pack4_i8(hi[0], hi[1], hi[2], hi[3]), pack4_i8(hi[4], hi[5], hi[6], hi[7]));
                *reinterpret_cast<uint2*>(lr + col) =
                    make_uint2(pack4_i8(lo[0], lo[1], lo[2], lo[3]), pack4_i8(lo[4], lo[5], lo[6], lo[7]));
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            shi += __shfl_xor_sync(0xFFFFFFFFu, shi, o);
            slo += __shfl_xor_sync(0xFFFFFFFFu, slo, o);
        }
        if (lane == 0) {
            a_sq[row] = shi;
            a_sq[N + row] = slo;
        }
    }
}

cudaError_t launch_bitsplit(const uint16_t* g, int64_t N, int64_t C, const uint32_t* amax_bits,
                            uint64_t seed, uint32_t call_id, int64_t token_offset, int8_t* hilo,
                            int32_t* a_sq, float* s_down, cudaStream_t s) {
    if (N == 0) return cudaSuccess;
    bitsplit_kernel<<<row_grid(N), kRowWarps * 32, 0, s>>>(g, N, int(C), amax_bits, uint32_t(seed),
                                                            uint32_t(seed >> 32), call_id, token_offset,
                                                            hilo, a_sq, s_down);
    return cudaGetLastError();
}

}  // namespace i4
