// Microbenchmark: Philox4x32-10 throughput on one B200 (words / s), by ILP and occupancy.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o philox_tput philox_tput.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct Keys { uint32_t k0[10], k1[10]; };

__device__ __forceinline__ void philox(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, const Keys& K) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = uint64_t(0xD2511F53u) * c0;
        const uint64_t p1 = uint64_t(0xCD9E8D57u) * c2;
        const uint32_t n0 = uint32_t(p1 >> 32) ^ c1 ^ K.k0[r], n2 = uint32_t(p0 >> 32) ^ c3 ^ K.k1[r];
        c0 = n0; c1 = uint32_t(p1); c2 = n2; c3 = uint32_t(p0);
    }
}

// same rounds with the 32x32 -> 64 products as mul.hi + mul.lo (IMAD.HI + IMAD)
__device__ __forceinline__ void philox_hilo(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, const Keys& K) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t h0 = __umulhi(0xD2511F53u, c0), l0 = 0xD2511F53u * c0;
        const uint32_t h1 = __umulhi(0xCD9E8D57u, c2), l1 = 0xCD9E8D57u * c2;
        const uint32_t n0 = h1 ^ c1 ^ K.k0[r], n2 = h0 ^ c3 ^ K.k1[r];
        c0 = n0; c1 = l1; c2 = n2; c3 = l0;
    }
}

template <int ILP, bool HILO = false>
__global__ void __launch_bounds__(256) kern(uint32_t* out, int iters, Keys K, uint32_t call) {
    uint32_t acc = 0;
    const uint32_t base = (blockIdx.x * blockDim.x + threadIdx.x) * ILP;
    for (int it = 0; it < iters; ++it) {
        uint32_t c0[ILP], c1[ILP], c2[ILP], c3[ILP];
#pragma unroll
        for (int j = 0; j < ILP; ++j) { c0[j] = base + j + it * 0x10000000u; c1[j] = 0; c2[j] = 1; c3[j] = call; }
#pragma unroll
        for (int j = 0; j < ILP; ++j) {
            if (HILO) philox_hilo(c0[j], c1[j], c2[j], c3[j], K);
            else philox(c0[j], c1[j], c2[j], c3[j], K);
        }
#pragma unroll
        for (int j = 0; j < ILP; ++j) acc += c0[j] ^ c1[j] ^ c2[j] ^ c3[j];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// integer-op throughput probes: IMAD.WIDE chain vs LOP3 chain
__global__ void __launch_bounds__(256) wide_only(uint32_t* out, int iters) {
    uint32_t a[8];
    for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int j = 0; j < 8; ++j) { uint64_t p = uint64_t(0xD2511F53u) * a[j]; a[j] = uint32_t(p >> 32) + uint32_t(p); }
    }
    uint32_t s = 0; for (int j = 0; j < 8; ++j) s += a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ILP, bool HILO = false>
float run(int blocks_per_sm, int iters, uint32_t* out) {
    Keys K; uint32_t k0 = 1, k1 = 2;
    for (int r = 0; r < 10; ++r) { K.k0[r] = k0; K.k1[r] = k1; k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    int blocks = 148 * blocks_per_sm;
    kern<ILP, HILO><<<blocks, 256>>>(out, iters, K, 3);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<ILP, HILO><<<blocks, 256>>>(out, iters, K, 3);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double words = double(blocks) * 256 * ILP * iters * 4;
    printf("%s ILP %d  blocks/SM %d: %.3f ms  %.1f Gwords/s  (33.5M words -> %.1f us)\n", HILO ? "hi/lo" : "wide ", ILP, blocks_per_sm, ms,
           words / ms / 1e6, 33.5e6 / (words / ms / 1e3) * 1e6);
    return ms;
}

int main() {
    uint32_t* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
    for (int bps : {4, 8}) {
        run<2>(bps, 32, out); run<4>(bps, 16, out);
        run<2, true>(bps, 32, out); run<4, true>(bps, 16, out);
    }
    {
        int blocks = 148 * 8; int iters = 64;
        wide_only<<<blocks, 256>>>(out, iters);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a); wide_only<<<blocks, 256>>>(out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double ops = double(blocks) * 256 * iters * 16 * 8;   // IMAD.WIDE (+ 1 IADD each)
        int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        printf("IMAD.WIDE+IADD pairs: %.3f ms, %.2f per SM per clk (clock %d MHz)\n", ms, ops / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1000);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
