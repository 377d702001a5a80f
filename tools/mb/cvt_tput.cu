// Microbenchmark: per-SM throughput of the float -> integer conversions the SR
// step can use (F2I.U64.CEIL, F2I.U32.CEIL on the XU pipe) against FFMA / LOP3 /
// IMAD.WIDE, in warp-instructions per cycle per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cvt_tput tools/mb/cvt_tput.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int OP>
__global__ void __launch_bounds__(256) kern(uint32_t* out, int iters, float seed) {
    float f[8];
    uint32_t a[8];
    uint64_t acc = 0;
    for (int j = 0; j < 8; ++j) { f[j] = seed * (threadIdx.x + j) * 1.37f; a[j] = threadIdx.x * 7 + j; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (OP == 0) { acc += __float2ull_ru(f[j]); f[j] = f[j] * 1.0001f; }        // F2I.U64 + FMUL
                if (OP == 1) { acc += __float2uint_ru(f[j]); f[j] = f[j] * 1.0001f; }       // F2I.U32 + FMUL
                if (OP == 2) { f[j] = f[j] * 1.0001f + 0.5f; }                               // FFMA only
                if (OP == 3) { a[j] = (a[j] ^ 0x9E3779B9u) ^ (a[j] >> 3); }                 // ALU
                if (OP == 4) { uint64_t p = uint64_t(0xD2511F53u) * a[j]; a[j] = uint32_t(p >> 32) ^ uint32_t(p); }   // IMAD.WIDE
                if (OP == 5) { acc += __float2uint_rz(f[j]); f[j] = f[j] * 1.0001f; }       // F2I.U32.TRUNC
                if (OP == 6) { f[j] = __uint_as_float(__float_as_uint(f[j]) + 1u); acc += __float_as_uint(f[j] * 3.0f); } // magic tricks
            }
    }
    uint32_t s = uint32_t(acc);
    for (int j = 0; j < 8; ++j) s += __float_as_uint(f[j]) + a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    uint32_t* out;
    cudaMalloc(&out, 148 * 8 * 256 * 4 * 4);
    const char* names[] = {"F2I.U64.CEIL+FMUL", "F2I.U32.CEIL+FMUL", "FFMA", "LOP3/SHF", "IMAD.WIDE+LOP", "F2I.U32.TRUNC+FMUL", "IADD+FMUL"};
    for (int op = 0; op < 7; ++op) {
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        const int iters = 2000, blocks = sms * 8;
        void (*k)(uint32_t*, int, float) = nullptr;
        switch (op) { case 0: k = kern<0>; break; case 1: k = kern<1>; break; case 2: k = kern<2>; break;
                      case 3: k = kern<3>; break; case 4: k = kern<4>; break; case 5: k = kern<5>; break; default: k = kern<6>; }
        k<<<blocks, 256>>>(out, 10, 1.0f);
        cudaEventRecord(a);
        k<<<blocks, 256>>>(out, iters, 1.0f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double ops = double(blocks) * 256 * iters * 64;              // thread-ops of the main statement
        const double per_clk_sm = ops / (ms * 1e-3) / (sms * clk * 1e3);     // lanes per cycle per SM
        printf("%-22s %8.3f ms  %7.1f lane-ops/clk/SM  (%.2f warp-instr/clk/SM)\n", names[op], ms, per_clk_sm, per_clk_sm / 32);
    }
    return 0;
}
