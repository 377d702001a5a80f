// LSQ step-size learning support (Appendix A.3 / A.4 of the paper):
//   lsq_finalize   : grad s_X, grad s_W from the per-CTA fp64 partials the two grad
//                    GEMM epilogues leave (sum acc o delta), times g(s) = 1/sqrt(Q_P N)
//                     and the partner step / s_down scales (reading Z-28)
//   lsq_cold_start : the A.4 rule step = 2 mean|X| / sqrt(Q_P) (reading Z-25)
// Both are tiny reductions; every sum runs in a fixed order (deterministic).
#include "common.cuh"
#include "kernels.h"

namespace i4 {

constexpr int kLsqThreads = 256;

// fixed-shape block sum of one double per thread (tree over shared memory)
__device__ double block_sum_fixed(double v, double* sh) {
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = kLsqThreads / 2; o > 0; o >>= 1) {
        if (int(threadIdx.x) < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    const double r = sh[0];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kLsqThreads) lsq_finalize_kernel(const double* part_x, const double* part_w,
                                                                   const float* s_down, float s_x, float s_w,
                                                                   double g_x, double g_w, float* grad_s) {
    pdl_trigger();
    pdl_wait();                                             // partials of the two grad GEMMs
    __shared__ double sh[kLsqThreads];
    double ax = 0.0, aw = 0.0;
    for (int i = threadIdx.x; i < kLsqPartials; i += kLsqThreads) {   // fixed order per thread
        ax += part_x[i];
        aw += part_w[i];
    }
    ax = block_sum_fixed(ax, sh);
    aw = block_sum_fixed(aw, sh);
    if (threadIdx.x == 0) {
        const double sd = double(*s_down);
        grad_s[0] = float(g_x * double(s_w) * sd * ax);    // g(s_X) s_W s_down sum_i w_i acc_i . delta_X
        grad_s[1] = float(g_w * double(s_x) * sd * aw);    // g(s_W) s_X s_down sum acc_W . delta_W
    }
}

cudaError_t launch_lsq_finalize(const double* part_x, const double* part_w, const float* s_down, float s_x,
                                float s_w, double g_x, double g_w, float* grad_s, cudaStream_t s) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(kLsqThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    cfg.attrs = attr;
    cfg.numAttrs = add_pdl_attr(attr, 0);
    return cudaLaunchKernelEx(&cfg, lsq_finalize_kernel, part_x, part_w, s_down, s_x, s_w, g_x, g_w, grad_s);
}

// ---------------------------------------------------------------------------
// cold start: grid of kColdBlocks CTAs, each sums |x| over a fixed strided set
// of 8-element groups in fp64, block tree sum -> partial[b]; the last CTA to
// finish (ticket) adds the partials in index order and writes the step.
// ---------------------------------------------------------------------------
constexpr int kColdBlocks = 592;

struct ColdWs { double partial[1024]; uint32_t ticket; uint32_t pad[3]; };

size_t lsq_cold_start_ws_bytes() { return sizeof(ColdWs); }

__global__ void __launch_bounds__(kLsqThreads) lsq_cold_start_kernel(const uint16_t* __restrict__ x, int64_t n,
                                                                     float* step, ColdWs* ws) {
    pdl_trigger();
    pdl_wait();
    __shared__ double sh[kLsqThreads];
    __shared__ bool last;
    const int64_t n8 = n / 8;
    const int64_t stride = int64_t(gridDim.x) * kLsqThreads;
    double acc = 0.0;
    for (int64_t i = int64_t(blockIdx.x) * kLsqThreads + threadIdx.x; i < n8; i += stride) {
        const uint4 u = ld_nc_v4(x + 8 * i);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
        double p8 = 0.0;                                    // fp64 for every add, fixed order
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            p8 += double(fabsf(bf16_lo(w[j])));
            p8 += double(fabsf(bf16_hi(w[j])));
        }
        acc += p8;
    }
    if (blockIdx.x == 0)                                    // tail elements (n % 8)
        for (int64_t i = 8 * n8 + threadIdx.x; i < n; i += kLsqThreads)
            acc += double(fabsf(__uint_as_float(uint32_t(x[i]) << 16)));
    acc = block_sum_fixed(acc, sh);
    if (threadIdx.x == 0) {
        ws->partial[blockIdx.x] = acc;
        __threadfence();
        last = atomicAdd(&ws->ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double t = 0.0;
    for (int i = threadIdx.x; i < int(gridDim.x); i += kLsqThreads) {
        t += __ldcg(ws->partial + i);
        ws->partial[i] = 0.0;                               // scratch left zeroed
    }
    t = block_sum_fixed(t, sh);
    if (threadIdx.x == 0) {
        *step = float(2.0 * (t / double(n)) / sqrt(7.0));  // 2 mean|X| / sqrt(Q_P), one rounding
        ws->ticket = 0u;                                    // left zeroed for the next call
    }
}

cudaError_t launch_lsq_cold_start(const uint16_t* x, int64_t n, float* step, void* ws, cudaStream_t s) {
    int64_t blocks = (n / 8 + kLsqThreads - 1) / kLsqThreads;
    if (blocks > kColdBlocks) blocks = kColdBlocks;
    if (blocks < 1) blocks = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(blocks));
    cfg.blockDim = dim3(kLsqThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    cfg.attrs = attr;
    cfg.numAttrs = add_pdl_attr(attr, 0);
    return cudaLaunchKernelEx(&cfg, lsq_cold_start_kernel, x, n, step, static_cast<ColdWs*>(ws));
}

// ---------------------------------------------------------------------------
// Step table of a batched BMM (host values -> device): the values travel as kernel
// parameters, so the copy is stream-ordered and graph-capturable without pinned
// host memory.  One launch per kStepTabChunk batches.
struct StepTab { float v[kStepTabChunk * 8]; };

__global__ void __launch_bounds__(256) step_table_kernel(const StepTab t, int n, float* __restrict__ dst) {
    pdl_trigger();
    pdl_wait();                                   // earlier kernels may still read the previous table
    for (int i = threadIdx.x; i < n * 8; i += blockDim.x) dst[i] = t.v[i];
}

cudaError_t launch_step_table(const float* host, int64_t n, float* dst, cudaStream_t s) {
    for (int64_t b0 = 0; b0 < n; b0 += kStepTabChunk) {
        const int m = int(n - b0 < kStepTabChunk ? n - b0 : kStepTabChunk);
        StepTab t{};
        for (int i = 0; i < m * 8; ++i) t.v[i] = host[b0 * 8 + i];
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(1);
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        cfg.attrs = attr;
        cfg.numAttrs = add_pdl_attr(attr, 0);
        const cudaError_t e = cudaLaunchKernelEx(&cfg, step_table_kernel, t, m, dst + b0 * 8);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace i4
