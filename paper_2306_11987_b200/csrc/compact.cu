// Operand compaction of the sampled items (LSS-MM step 4, "Sample rows of
// grad_Y and X_hat given the masks"; zero padding of the
// sampled K / M to the MMA tile).  HBM-bound gathers.
//
//   compact_kernel builds the grad_X GEMM's A and the grad_W GEMM's A and B in
//   one launch (row copies; TMA tile::gather4 inside the GEMM producers measured
//   ~3x slower than these copies on B200).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace i4 {

constexpr int kGroup = 8;                 // 16-byte loads in flight per lane

// One launch builds all three compacted operands; one warp per output row:
//   A_X[j, :] = half h of Q[t, :] for item (h, t)  (C bytes; grad_X GEMM A, K-major):
//               16 hi (h = 0) or lo (h = 1), split from the 8-bit codes on the fly
//   A_W[j, :] = the same for items_w[j]           (C bytes; grad_W GEMM A, MN-major)
//   B_W[j, :] = 2^wexp_w[j] X_hat[t(items_w[j]), :]   (D bytes, |.| <= 112; grad_W GEMM B)
// The A rows hold 16 hi or lo, so acc[c, d] = sum_j A_W[j, c] B_W[j, d] is the
// weighted bit-split product with s_up = 16 s_down folded in (reading Z-17).
// Rows past a list's count, up to its multiple of 128, are zero (the MMA pad).
__device__ __forceinline__ uint4 scale_i8x16(uint4 u, int mul) {
    int8_t* b = reinterpret_cast<int8_t*>(&u);
#pragma unroll
    for (int q = 0; q < 16; ++q) b[q] = int8_t(int(b[q]) * mul);
    return u;
}

// bit split of 4 packed 8-bit codes q (reading Z-11): t = (q + 128) + 8 per byte
// (no carries: q + 136 <= 255); 16 hi = (t & 0xF0) ^ 0x80, lo = ((t & 0x0F) + 0x78) ^ 0x80
__device__ __forceinline__ uint32_t split_word(uint32_t q, int half) {
    const uint32_t t = (q ^ 0x80808080u) + 0x08080808u;
    return half == 0 ? ((t & 0xF0F0F0F0u) ^ 0x80808080u) : (((t & 0x0F0F0F0Fu) + 0x78787878u) ^ 0x80808080u);
}

// half: -1 copy (optionally scaled by mul), 0 / 1: the high (16 hi) / low half of the codes
__device__ __forceinline__ void copy_row(const int8_t* __restrict__ src, int8_t* __restrict__ dst, int n, int lane,
                                         bool zero, int mul, int half = -1) {
    if (n <= 512) {                                   // short row (attention head dims): one chunk per lane
        const int c = lane * 16;
        if (c < n) {
            uint4 v = zero ? make_uint4(0, 0, 0, 0) : ld_nc_v4(src + c);
            if (half >= 0)
                v = make_uint4(split_word(v.x, half), split_word(v.y, half), split_word(v.z, half), split_word(v.w, half));
            else if (mul != 1)
                v = scale_i8x16(v, mul);
            *reinterpret_cast<uint4*>(dst + c) = v;
        }
        return;
    }
    for (int c0 = 0; c0 < n; c0 += 512 * kGroup) {
        uint4 u[kGroup];
#pragma unroll
        for (int gq = 0; gq < kGroup; ++gq) {          // all loads of the group first
            const int c = c0 + 512 * gq + lane * 16;
            u[gq] = (c < n && !zero) ? ld_nc_v4(src + c) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int gq = 0; gq < kGroup; ++gq) {
            const int c = c0 + 512 * gq + lane * 16;
            if (c >= n) continue;
            uint4 v = u[gq];
            if (half >= 0)
                v = make_uint4(split_word(v.x, half), split_word(v.y, half), split_word(v.z, half), split_word(v.w, half));
            else if (mul != 1)
                v = scale_i8x16(v, mul);
            *reinterpret_cast<uint4*>(dst + c) = v;
        }
    }
}

__device__ __forceinline__ void zero_row(void* base, int64_t row, int n, bool bf16, int lane) {
    uint8_t* dst = static_cast<uint8_t*>(base) + row * n * (bf16 ? 2 : 4);
    const int bytes = n * (bf16 ? 2 : 4);
    for (int c = lane * 16; c < bytes; c += 512) *reinterpret_cast<uint4*>(dst + c) = make_uint4(0, 0, 0, 0);
}

__global__ void __launch_bounds__(256) compact_kernel(CompactArgs a) {
    pdl_wait();                                               // counts / lists of the sampler
    pdl_trigger();                                            // after the wait: the backward GEMM reads the
                                                              // sampler's sizes before its own PDL wait
    if (a.batch > 1) {                                        // this CTA's batch: its slices
        const int64_t b = blockIdx.y, N = a.N, kcap = (2 * N + 127) / 128 * 128;
        a.q8 += b * N * a.C; a.xq += b * N * a.D;
        a.items_x += b * a.bs_list; a.items_w += b * a.bs_list; a.wexp_w += b * a.bs_list;
        a.count_x += b; a.count_w += b;
        a.x_touched += b * N;
        a.dx = static_cast<uint8_t*>(a.dx) + b * N * a.D * (a.dx_bf16 ? 2 : 4);
        a.a_x += b * (2 * N + 128) * a.C; a.a_w += b * kcap * a.C; a.b_w += b * kcap * a.D;
    }
    const int lane = threadIdx.x & 31;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    // operand forms (the sampler's flags; the GEMMs pick their operands by the same
    // values): 1 dense -> nothing to move (the GEMM reads Q / X_hat and writes every
    // grad_X token row); 0 sampled -> every kept item; 2 dense + correction -> the
    // grad_W correction rows and the grad_X sub list of the tokens with sampled items
    const int fx = a.det_flags != nullptr ? __ldg(a.det_flags + 1) : 0;
    const int fw = a.det_flags != nullptr ? __ldg(a.det_flags) : 0;
    const int32_t* lx = fx == 2 ? a.sub_items : a.items_x;   // grad_X rows to gather
    const int64_t cnt_x = fx == 1 ? 0 : __ldg(fx == 2 ? a.sub_count : a.count_x);
    const int32_t* lw = fw == 2 ? a.corr_items : a.items_w;  // grad_W rows to gather
    const int8_t* ew = fw == 2 ? a.corr_wexp : a.wexp_w;
    const int64_t cnt_w = fw == 1 ? 0 : __ldg(fw == 2 ? a.corr_count : a.count_w);
    const int64_t pad_x = (cnt_x + 127) & ~int64_t(127);
    const int64_t pad_w = (cnt_w + 127) & ~int64_t(127);
    const int64_t n_straddle = (cnt_x + 31) / 32;            // candidate positions 31, 63, ...
    const int64_t seg_bw = pad_x + pad_w;                    // first B_W row job
    // short rows (D < 512 bytes, e.g. attention head dims) share a warp: rpj rows per job,
    // D / 16 lanes per row, so every lane moves 16 bytes
    const int rpj_b = a.D < 512 ? 512 / a.D : 1;
    const int64_t n_bw = (pad_w + rpj_b - 1) / rpj_b;
    const int zb = a.D * (a.dx_bf16 ? 2 : 4);                // bytes of a grad_X row
    const int rpj_z = zb < 512 ? 512 / zb : 1;
    const int64_t n_zero = fx == 1 ? 0 : (a.N + rpj_z - 1) / rpj_z;
    const int64_t seg_z = seg_bw + n_bw, seg_s = seg_z + n_zero;
    const int64_t total = seg_s + n_straddle;
    const int two_n = 2 * a.N;
    for (int64_t j = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); j < total; j += warps) {
        if (j >= seg_s) {
            // tokens whose two items straddle a 32-row group (both red.add onto a zero row)
            const int64_t p = 32 * (j - seg_s) + 31;
            if (p + 1 < cnt_x) {
                const int32_t i0 = __ldg(lx + p), i1 = __ldg(lx + p + 1);
                const int t0 = i0 >= a.N ? i0 - a.N : i0, t1 = i1 >= a.N ? i1 - a.N : i1;
                if (t0 == t1) zero_row(a.dx, t0, a.D, a.dx_bf16, lane);
            }
        } else if (j >= seg_z) {
            // grad_X rows the GEMM epilogue does not store: tokens without a kept item
            // (form 2: only among the flagged tokens -- the others are Q rows)
            if (rpj_z == 1) {
                const int64_t r = j - seg_z;
                if (__ldg(a.x_touched + r) == 0 && (fx != 2 || __ldg(a.tok_flag + r) != 0))
                    zero_row(a.dx, r, a.D, a.dx_bf16, lane);
            } else {
                const int lpr = zb / 16;
                const int64_t r = (j - seg_z) * rpj_z + lane / lpr;
                if (r < a.N && __ldg(a.x_touched + r) == 0 && (fx != 2 || __ldg(a.tok_flag + r) != 0))
                    *reinterpret_cast<uint4*>(static_cast<uint8_t*>(a.dx) + r * zb + (lane % lpr) * 16) =
                        make_uint4(0, 0, 0, 0);
            }
        } else if (j < pad_x) {
            const int32_t item = __ldg(lx + j);
            const bool pad = item >= two_n;
            const int h = item >= a.N ? 1 : 0;
            copy_row(a.q8 + int64_t(pad ? 0 : item - h * a.N) * a.C, a.a_x + j * a.C, a.C, lane, pad, 1, h);
        } else if (j < seg_bw) {
            const int64_t r = j - pad_x;
            const int32_t item = __ldg(lw + r);
            const bool pad = item >= two_n;
            const int h = item >= a.N ? 1 : 0;
            copy_row(a.q8 + int64_t(pad ? 0 : item - h * a.N) * a.C, a.a_w + r * a.C, a.C, lane, pad, 1, h);
        } else {
            // B_W row = weight x X_hat[t]: 2^wexp for kept items, -1 for a form-2
            // correction row that removes the item's dense term (|.| <= 112)
            if (rpj_b == 1) {
                const int64_t r = j - seg_bw;
                const int32_t item = __ldg(lw + r);
                const bool pad = item >= two_n;
                const int t = pad ? 0 : (item >= a.N ? item - a.N : item);
                const int e = pad ? 0 : int(__ldg(ew + r));
                copy_row(a.xq + int64_t(t) * a.D, a.b_w + r * a.D, a.D, lane, pad, e < 0 ? -1 : (1 << e));
            } else {
                const int lpr = a.D / 16;
                const int64_t r = (j - seg_bw) * rpj_b + lane / lpr;
                if (r < pad_w) {
                    const int32_t item = __ldg(lw + r);
                    const bool pad = item >= two_n;
                    const int t = pad ? 0 : (item >= a.N ? item - a.N : item);
                    const int e = pad ? 0 : int(__ldg(ew + r));
                    const int c = (lane % lpr) * 16;
                    uint4 v = pad ? make_uint4(0, 0, 0, 0) : ld_nc_v4(a.xq + int64_t(t) * a.D + c);
                    if (!pad) v = scale_i8x16(v, e < 0 ? -1 : (1 << e));
                    *reinterpret_cast<uint4*>(a.b_w + r * a.D + c) = v;
                }
            }
        }
    }
}

cudaError_t launch_compact(const CompactArgs& a, cudaStream_t s) {
    const int64_t rows = (2 * int64_t(a.N) + 128) * 3 + a.N;  // upper bound of the row count
    int64_t blocks = (rows + 7) / 8;
    if (blocks > 148 * 4) blocks = 148 * 4;        // grid-stride rows; a smaller grid launches faster when little is to move
    cudaLaunchConfig_t cfg{};
    const int64_t nbat = a.batch > 1 ? a.batch : 1;
    // batched: one warp per row job where the device holds them (8 CTAs of 8 warps per SM)
    if (nbat > 1) blocks = std::max<int64_t>(1, std::min<int64_t>((rows + 7) / 8, (148 * 8 + nbat - 1) / nbat));
    cfg.gridDim = dim3(unsigned(blocks), unsigned(nbat));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    cfg.attrs = attr;
    cfg.numAttrs = add_pdl_attr(attr, 0);
    return cudaLaunchKernelEx(&cfg, compact_kernel, a);
}

}  // namespace i4
