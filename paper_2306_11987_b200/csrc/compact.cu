// Operand compaction of the sampled items (LSS-MM step 4, "Sample rows of
// grad_Y and X_hat given the masks"; zero padding of the
// sampled K / M to the MMA tile).  HBM-bound gathers.
//
//   compact_rows   grad_X GEMM A operand: A_X[j, :] = hilo[items_x[j], :]
//                  (K-major rows of C bytes), zero rows up to the 128 multiple.
//   compact_wgrad  grad_W GEMM operands (read MN-major by the GEMM):
//                  A_W[j, c] = 2^wexp_j code_j[c]      (|.| <= 128, reading Z-17)
//                  B_W[j, d] = 16^[h_j = up] X_hat[t_j, d]   (|.| <= 112)
//                  so that acc[c, d] = sum_j A_W[j, c] B_W[j, d] is the
//                  weighted bit-split product with s_up = 16 s_down folded in.
#include "common.cuh"
#include "kernels.h"

namespace i4 {

constexpr int kGroup = 8;                 // 16-byte loads in flight per lane

__global__ void __launch_bounds__(256) compact_rows_kernel(const int8_t* __restrict__ hilo, int C,
                                                           const int32_t* __restrict__ items,
                                                           const int32_t* __restrict__ count,
                                                           int64_t max_rows, int8_t* __restrict__ out,
                                                           int32_t sentinel) {
    const int64_t padded = (int64_t(__ldg(count)) + 127) & ~int64_t(127);
    const int lane = threadIdx.x & 31;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t j = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); j < padded && j < max_rows;
         j += warps) {
        const int32_t item = __ldg(items + j);
        int8_t* dst = out + j * C;
        const int8_t* src = hilo + int64_t(item < sentinel ? item : 0) * C;
        for (int c0 = 0; c0 < C; c0 += 512 * kGroup) {
            uint4 u[kGroup];
#pragma unroll
            for (int g = 0; g < kGroup; ++g) {          // all loads of the group first
                const int c = c0 + 512 * g + lane * 16;
                u[g] = (c < C && item < sentinel) ? ld_nc_v4(src + c) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int g = 0; g < kGroup; ++g) {
                const int c = c0 + 512 * g + lane * 16;
                if (c < C) *reinterpret_cast<uint4*>(dst + c) = u[g];
            }
        }
    }
}

cudaError_t launch_compact_rows(const int8_t* hilo, int64_t C, const int32_t* items, const int32_t* count,
                                int64_t n_items, int8_t* out, cudaStream_t s) {
    const int64_t max_rows = n_items + 128;     // count <= n_items, padded to a multiple of 128
    int64_t blocks = (max_rows + 7) / 8;
    if (blocks > 148 * 8) blocks = 148 * 8;
    compact_rows_kernel<<<int(blocks), 256, 0, s>>>(hilo, int(C), items, count, max_rows, out, int32_t(n_items));
    return cudaGetLastError();
}

// One warp per kept item j (row gathers; the grad_W GEMM reads both operands
// MN-major, so no transpose is needed):
//   A_W[j, :] = 2^wexp_j hilo[item_j, :]       (C bytes, |.| <= 128)
//   B_W[j, :] = 16^[h_j = up] X_hat[t_j, :]    (D bytes, |.| <= 112)
__device__ __forceinline__ uint4 scale_i8x16(uint4 u, int mul) {
    int8_t* b = reinterpret_cast<int8_t*>(&u);
#pragma unroll
    for (int q = 0; q < 16; ++q) b[q] = int8_t(int(b[q]) * mul);
    return u;
}

__global__ void __launch_bounds__(256) compact_wgrad_kernel(const int8_t* __restrict__ hilo,
                                                            const int8_t* __restrict__ xq, int N, int C, int D,
                                                            const int32_t* __restrict__ items,
                                                            const int8_t* __restrict__ wexp,
                                                            const int32_t* __restrict__ count,
                                                            int8_t* __restrict__ a_w, int8_t* __restrict__ b_w) {
    const int64_t padded = (int64_t(__ldg(count)) + 127) & ~int64_t(127);
    const int lane = threadIdx.x & 31;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t j = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); j < padded; j += warps) {
        const int32_t item = __ldg(items + j);
        int8_t* da = a_w + j * C;
        int8_t* db = b_w + j * D;
        if (item >= 2 * N) {
            for (int c = lane * 16; c < C; c += 512) *reinterpret_cast<uint4*>(da + c) = make_uint4(0, 0, 0, 0);
            for (int c = lane * 16; c < D; c += 512) *reinterpret_cast<uint4*>(db + c) = make_uint4(0, 0, 0, 0);
            continue;
        }
        const int h = item >= N ? 1 : 0;
        const int t = item - h * N;
        const int mul_a = 1 << __ldg(wexp + j);
        const int mul_b = h == 0 ? 16 : 1;
        const int8_t* sa = hilo + int64_t(item) * C;
        const int8_t* sb = xq + int64_t(t) * D;
        const int ca = (C + 511) / 512, cb = (D + 511) / 512;   // 16-byte pieces per lane
        for (int p0 = 0; p0 < ca + cb; p0 += kGroup) {
            uint4 u[kGroup];
#pragma unroll
            for (int g = 0; g < kGroup; ++g) {
                const int p = p0 + g;
                const int c = (p < ca ? p : p - ca) * 512 + lane * 16;
                u[g] = make_uint4(0, 0, 0, 0);
                if (p < ca) { if (c < C) u[g] = ld_nc_v4(sa + c); }
                else if (p < ca + cb && c < D) u[g] = ld_nc_v4(sb + c);
            }
#pragma unroll
            for (int g = 0; g < kGroup; ++g) {
                const int p = p0 + g;
                const int c = (p < ca ? p : p - ca) * 512 + lane * 16;
                if (p < ca) { if (c < C) *reinterpret_cast<uint4*>(da + c) = scale_i8x16(u[g], mul_a); }
                else if (p < ca + cb && c < D) *reinterpret_cast<uint4*>(db + c) = scale_i8x16(u[g], mul_b);
            }
        }
    }
}

cudaError_t launch_compact_wgrad(const int8_t* hilo, const int8_t* xq, int64_t N, int64_t C, int64_t D,
                                 const int32_t* items, const int8_t* wexp, const int32_t* count,
                                 int64_t kcap, int8_t* a_w, int8_t* b_w, cudaStream_t s) {
    int64_t blocks = (kcap + 7) / 8;
    if (blocks > 148 * 8) blocks = 148 * 8;
    compact_wgrad_kernel<<<int(blocks), 256, 0, s>>>(hilo, xq, int(N), int(C), int(D), items, wexp, count, a_w, b_w);
    return cudaGetLastError();
}

}  // namespace i4
