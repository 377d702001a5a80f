// Adaptive Hadamard block size (Appendix A.5): for each
// candidate k the reconstruction X_bar_k = s <XH>_s H^T is formed on the fly and
// its squared error against X accumulated; a final launch picks
// k* = argmin MSE(X_bar_k, X) x MSE(W_bar_k, W) (first on ties, reading Z-30).
//
// hq_error_kernel<k>: one thread per 32-column block of a row (as hadamard_quant):
// the forward transform and the LSQ code are the forward path's (fp32 pairs,
// v = fl32(t r), RNE, clamp), the inverse transform of the integer codes is exact
// integer arithmetic (|.| <= 7 2^k), and x_bar = (s 2^{-k/2}) ic, the error and its
// square are fp64.  X and W are two row jobs of one launch; per-CTA fp64 partials
// are reduced in a fixed order by the last CTA (ticket), so the result is
// deterministic.  Runs rarely (once per fine-tuning run / re-initialisation).
#include "common.cuh"
#include "kernels.h"

namespace i4 {

constexpr int kErrThreads = 256;
constexpr int kErrBlocks = 592;

struct ErrJob { const uint16_t* x; int64_t rows; float r; double c; };

struct SelectKWs {
    double partial[2][kErrBlocks];
    uint32_t ticket;
    uint32_t pad[3];
};

size_t select_k_ws_bytes() { return sizeof(SelectKWs); }

__device__ double block_sum_err(double v, double* sh) {
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = kErrThreads / 2; o > 0; o >>= 1) {
        if (int(threadIdx.x) < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    const double r = sh[0];
    __syncthreads();
    return r;
}

// integer butterflies over the 32 codes of one thread (strides 1 .. 2^(K-1) <= 16)
template <int K>
__device__ __forceinline__ void iwht32(int (&v)[32]) {
#pragma unroll
    for (int s = 0; s < K; ++s) {
        const int h = 1 << s;
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (((i >> s) & 1) == 0) {
                const int a = v[i], b = v[i + h];
                v[i] = a + b;
                v[i + h] = a - b;
            }
    }
}

template <int K>
__global__ void __launch_bounds__(kErrThreads) hq_error_kernel(ErrJob j0, ErrJob j1, int cols, SelectKWs* ws,
                                                               double* mse_out) {
    pdl_trigger();
    pdl_wait();
    __shared__ double sh[kErrThreads];
    __shared__ bool last;
    const int tpr = cols >> 5;
    const int64_t items0 = j0.rows * tpr, items = items0 + j1.rows * tpr;
    const int64_t stride = int64_t(gridDim.x) * kErrThreads;
    const int64_t span = (items + stride - 1) / stride * stride;      // warp-uniform trip count
    double e0 = 0.0, e1 = 0.0;
    for (int64_t i = int64_t(blockIdx.x) * kErrThreads + threadIdx.x; i < span; i += stride) {
        const bool active = i < items;
        const bool second = i >= items0;
        const ErrJob& J = second ? j1 : j0;
        const int64_t li = active ? (second ? i - items0 : i) : 0;
        const int64_t row = li / tpr;
        const int blk = int(li - row * tpr);
        float xv[32];
        {
            const uint16_t* src = J.x + row * cols + blk * 32;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 u = active ? ld_nc_v4(src + 8 * q) : make_uint4(0, 0, 0, 0);
                xv[8 * q + 0] = bf16_lo(u.x); xv[8 * q + 1] = bf16_hi(u.x);
                xv[8 * q + 2] = bf16_lo(u.y); xv[8 * q + 3] = bf16_hi(u.y);
                xv[8 * q + 4] = bf16_lo(u.z); xv[8 * q + 5] = bf16_hi(u.z);
                xv[8 * q + 6] = bf16_lo(u.w); xv[8 * q + 7] = bf16_hi(u.w);
            }
        }
        // forward transform + LSQ code: the forward path's arithmetic
        uint64_t p[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) p[j] = f2_pack(xv[j], xv[j + 16]);
        fwht_pairs<32, (K < 5 ? K : 5)>(p);
        if constexpr (K > 5) {
#pragma unroll
            for (int s = 5; s < K; ++s) {
                const int lm = 1 << (s - 5);
                const float sgn = (blk & lm) ? -1.0f : 1.0f;
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    float a, b;
                    f2_unpack(p[j], a, b);
                    const float oa = __shfl_xor_sync(0xFFFFFFFFu, a, lm);
                    const float ob = __shfl_xor_sync(0xFFFFFFFFu, b, lm);
                    p[j] = f2_pack(__fmaf_rn(sgn, a, oa), __fmaf_rn(sgn, b, ob));
                }
            }
        }
        int code[32];
        const uint64_t r2 = f2_pack(J.r, J.r);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            float s0, s1;
            f2_unpack(f2_mul(p[j], r2), s0, s1);
            code[j] = __float2int_rn(fminf(fmaxf(s0, -7.0f), 7.0f));
            code[j + 16] = __float2int_rn(fminf(fmaxf(s1, -7.0f), 7.0f));
        }
        // inverse transform of the integer codes (H symmetric): exact
        iwht32<(K < 5 ? K : 5)>(code);
        if constexpr (K > 5) {
#pragma unroll
            for (int s = 5; s < K; ++s) {
                const int lm = 1 << (s - 5);
                const bool upper = (blk & lm) != 0;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const int o = __shfl_xor_sync(0xFFFFFFFFu, code[j], lm);
                    code[j] = upper ? o - code[j] : code[j] + o;
                }
            }
        }
        double e = 0.0;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const double d = double(code[j]) * J.c - double(xv[j]);
            e += d * d;
        }
        if (active) { if (second) e1 += e; else e0 += e; }
    }
    e0 = block_sum_err(e0, sh);
    e1 = block_sum_err(e1, sh);
    if (threadIdx.x == 0) {
        ws->partial[0][blockIdx.x] = e0;
        ws->partial[1][blockIdx.x] = e1;
        __threadfence();
        last = atomicAdd(&ws->ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double t0 = 0.0, t1 = 0.0;
    for (int i = threadIdx.x; i < int(gridDim.x); i += kErrThreads) {
        t0 += __ldcg(&ws->partial[0][i]);
        t1 += __ldcg(&ws->partial[1][i]);
        ws->partial[0][i] = 0.0;
        ws->partial[1][i] = 0.0;
    }
    t0 = block_sum_err(t0, sh);
    t1 = block_sum_err(t1, sh);
    if (threadIdx.x == 0) {
        mse_out[2 * K] = j0.rows > 0 ? t0 / double(j0.rows * cols) : 0.0;
        mse_out[2 * K + 1] = j1.rows > 0 ? t1 / double(j1.rows * cols) : 0.0;
        ws->ticket = 0u;
    }
}

__global__ void select_k_kernel(const double* mse, int k_min, int k_max, int32_t* k_best) {
    pdl_trigger();
    pdl_wait();
    if (threadIdx.x != 0) return;
    int best = k_min;
    double bv = mse[2 * k_min] * mse[2 * k_min + 1];
    for (int k = k_min + 1; k <= k_max; ++k) {
        const double v = mse[2 * k] * mse[2 * k + 1];
        if (v < bv) { bv = v; best = k; }                 // strict: ties keep the smaller k
    }
    *k_best = best;
}

template <int K>
static cudaError_t launch_err(const ErrJob& a, const ErrJob& b, int cols, SelectKWs* ws, double* mse, cudaStream_t s) {
    const int64_t items = (a.rows + b.rows) * (cols / 32);
    int64_t blocks = (items + kErrThreads - 1) / kErrThreads;
    if (blocks > kErrBlocks) blocks = kErrBlocks;
    if (blocks < 1) blocks = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(blocks));
    cfg.blockDim = dim3(kErrThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    cfg.attrs = attr;
    cfg.numAttrs = add_pdl_attr(attr, 0);
    return cudaLaunchKernelEx(&cfg, hq_error_kernel<K>, a, b, cols, ws, mse);
}

cudaError_t launch_select_k(const uint16_t* x, int64_t n, const uint16_t* w, int64_t c, int64_t d, float r_x[8],
                            float r_w[8], double c_x[8], double c_w[8], int k_min, int k_max, int32_t* k_best,
                            double* mse, void* ws, cudaStream_t s) {
    SelectKWs* W = static_cast<SelectKWs*>(ws);
    for (int k = k_min; k <= k_max; ++k) {
        const ErrJob a{x, n, r_x[k], c_x[k]}, b{w, c, r_w[k], c_w[k]};
        cudaError_t e = cudaSuccess;
        switch (k) {
            case 0: e = launch_err<0>(a, b, int(d), W, mse, s); break;
            case 1: e = launch_err<1>(a, b, int(d), W, mse, s); break;
            case 2: e = launch_err<2>(a, b, int(d), W, mse, s); break;
            case 3: e = launch_err<3>(a, b, int(d), W, mse, s); break;
            case 4: e = launch_err<4>(a, b, int(d), W, mse, s); break;
            case 5: e = launch_err<5>(a, b, int(d), W, mse, s); break;
            case 6: e = launch_err<6>(a, b, int(d), W, mse, s); break;
            case 7: e = launch_err<7>(a, b, int(d), W, mse, s); break;
            default: return cudaErrorInvalidValue;
        }
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(32);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    cfg.attrs = attr;
    cfg.numAttrs = add_pdl_attr(attr, 0);
    return cudaLaunchKernelEx(&cfg, select_k_kernel, static_cast<const double*>(mse), k_min, k_max, k_best);
}

}  // namespace i4
