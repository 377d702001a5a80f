// Operand compaction of the sampled items (LSS-MM step 4, "Sample rows of
// grad_Y and X_hat given the masks"; zero padding of the
// sampled K / M to the MMA tile).  HBM-bound gathers.
//
//   compact_rows   grad_X GEMM A operand: A_X[j, :] = hilo[items_x[j], :]
//                  (K-major rows of C bytes), zero rows up to the 128 multiple.
//   compact_wgrad  grad_W GEMM operands, written K-major (items contiguous):
//                  A_W^T[c, j] = 2^wexp_j code_j[c]      (|.| <= 128, reading Z-17)
//                  B_W^T[d, j] = 16^[h_j = up] X_hat[t_j, d]   (|.| <= 112)
//                  so that acc[c, d] = sum_j A_W^T[c, j] B_W^T[d, j] is the
//                  weighted bit-split product with s_up = 16 s_down folded in.
#include "common.cuh"
#include "kernels.h"

namespace i4 {

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
        if (item >= sentinel) {
            for (int c = lane * 16; c < C; c += 512) *reinterpret_cast<uint4*>(dst + c) = make_uint4(0, 0, 0, 0);
        } else {
            const int8_t* src = hilo + int64_t(item) * C;
            for (int c = lane * 16; c < C; c += 512)
                *reinterpret_cast<uint4*>(dst + c) = ld_nc_v4(src + c);
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

// 64 items x 64 columns per CTA.  blockIdx.z = 0: A_W^T from hilo (C columns);
// blockIdx.z = 1: B_W^T from X_hat (D columns).
__global__ void __launch_bounds__(256) compact_wgrad_kernel(const int8_t* __restrict__ hilo,
                                                            const int8_t* __restrict__ xq, int N, int C, int D,
                                                            const int32_t* __restrict__ items,
                                                            const int8_t* __restrict__ wexp,
                                                            const int32_t* __restrict__ count, int64_t kcap,
                                                            int8_t* __restrict__ a_t, int8_t* __restrict__ b_t) {
    __shared__ int8_t tile[64][64 + 4];
    const int64_t padded = (int64_t(__ldg(count)) + 127) & ~int64_t(127);
    const int64_t j0 = int64_t(blockIdx.x) * 64;
    if (j0 >= padded) return;
    const bool is_b = blockIdx.z == 1;
    const int cols = is_b ? D : C;
    const int64_t c0 = int64_t(blockIdx.y) * 64;
    if (c0 >= cols) return;
    {
        const int r = threadIdx.x >> 2, seg = (threadIdx.x & 3) * 16;
        const int64_t j = j0 + r;
        uint4 u = make_uint4(0, 0, 0, 0);
        const int32_t item = __ldg(items + j);
        if (item < 2 * N && c0 + seg < cols) {
            const int h = item >= N ? 1 : 0;
            const int t = item - h * N;
            if (!is_b) {
                u = ld_nc_v4(hilo + int64_t(item) * C + c0 + seg);
                const int sh = __ldg(wexp + j);
                int8_t* b = reinterpret_cast<int8_t*>(&u);
#pragma unroll
                for (int q = 0; q < 16; ++q) b[q] = int8_t(int(b[q]) * (1 << sh));
            } else {
                u = ld_nc_v4(xq + int64_t(t) * D + c0 + seg);
                if (h == 0) {
                    int8_t* b = reinterpret_cast<int8_t*>(&u);
#pragma unroll
                    for (int q = 0; q < 16; ++q) b[q] = int8_t(int(b[q]) * 16);
                }
            }
        }
        const int8_t* b = reinterpret_cast<const int8_t*>(&u);
#pragma unroll
        for (int q = 0; q < 16; ++q) tile[r][seg + q] = b[q];
    }
    __syncthreads();
    {
        const int c = threadIdx.x >> 2, seg = (threadIdx.x & 3) * 16;
        if (c0 + c < cols) {
            alignas(16) int8_t b[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) b[q] = tile[seg + q][c];
            int8_t* dst = (is_b ? b_t : a_t) + (c0 + c) * kcap + j0 + seg;
            *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(b);
        }
    }
}

cudaError_t launch_compact_wgrad(const int8_t* hilo, const int8_t* xq, int64_t N, int64_t C, int64_t D,
                                 const int32_t* items, const int8_t* wexp, const int32_t* count,
                                 int64_t kcap, int8_t* a_t, int8_t* b_t, cudaStream_t s) {
    const int64_t cmax = C > D ? C : D;
    dim3 grid(unsigned(kcap / 64), unsigned((cmax + 63) / 64), 2);
    compact_wgrad_kernel<<<grid, 256, 0, s>>>(hilo, xq, int(N), int(C), int(D), items, wexp, count, kcap, a_t, b_t);
    return cudaGetLastError();
}

}  // namespace i4
