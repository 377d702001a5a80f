// Operand compaction of the sampled items (LSS-MM step 4, "Sample rows of
// grad_Y and X_hat given the masks"; zero padding of the
// sampled K / M to the MMA tile).  HBM-bound gathers.
//
//   The grad_X and grad_W GEMMs gather the kept items' bit-split plane rows
//   themselves (TMA tile::gather4); the only copy left is the grad_W B operand,
//   which carries the item weights.
#include "common.cuh"
#include "kernels.h"

namespace i4 {

constexpr int kGroup = 8;                 // 16-byte loads in flight per lane

// One warp per kept item j of the grad_W mask (row gather + shift):
//   B_W[j, :] = 2^wexp_j X_hat[t_j, :]      (D bytes, |.| <= 16 * 7 = 112)
// The A operand (the item's plane row, which holds 16 hi or lo) is gathered by
// the GEMM itself, so acc[c, d] = sum_j plane[item_j, c] B_W[j, d] is the
// weighted bit-split product with s_up = 16 s_down folded in (reading Z-17).
__device__ __forceinline__ uint4 scale_i8x16(uint4 u, int mul) {
    int8_t* b = reinterpret_cast<int8_t*>(&u);
#pragma unroll
    for (int q = 0; q < 16; ++q) b[q] = int8_t(int(b[q]) * mul);
    return u;
}

__global__ void __launch_bounds__(256) compact_wgrad_kernel(const int8_t* __restrict__ xq, int N, int D,
                                                            const int32_t* __restrict__ items,
                                                            const int8_t* __restrict__ wexp,
                                                            const int32_t* __restrict__ count,
                                                            int8_t* __restrict__ b_w) {
    const int64_t padded = (int64_t(__ldg(count)) + 127) & ~int64_t(127);
    const int lane = threadIdx.x & 31;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t j = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); j < padded; j += warps) {
        const int32_t item = __ldg(items + j);
        int8_t* db = b_w + j * D;
        const bool pad = item >= 2 * N;
        const int t = pad ? 0 : (item >= N ? item - N : item);
        const int mul = pad ? 0 : (1 << __ldg(wexp + j));
        const int8_t* sb = xq + int64_t(t) * D;
        for (int c0 = 0; c0 < D; c0 += 512 * kGroup) {
            uint4 u[kGroup];
#pragma unroll
            for (int gq = 0; gq < kGroup; ++gq) {          // all loads of the group first
                const int c = c0 + 512 * gq + lane * 16;
                u[gq] = (c < D && !pad) ? ld_nc_v4(sb + c) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int gq = 0; gq < kGroup; ++gq) {
                const int c = c0 + 512 * gq + lane * 16;
                if (c < D) *reinterpret_cast<uint4*>(db + c) = scale_i8x16(u[gq], mul);
            }
        }
    }
}

cudaError_t launch_compact_wgrad(const int8_t* xq, int64_t N, int64_t D, const int32_t* items, const int8_t* wexp,
                                 const int32_t* count, int64_t kcap, int8_t* b_w, cudaStream_t s) {
    int64_t blocks = (kcap + 7) / 8;
    if (blocks > 148 * 8) blocks = 148 * 8;
    compact_wgrad_kernel<<<int(blocks), 256, 0, s>>>(xq, int(N), int(D), items, wexp, count, b_w);
    return cudaGetLastError();
}

}  // namespace i4
