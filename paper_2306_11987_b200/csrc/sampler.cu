// Leverage-score sampler: LSS-MM steps 2-4 for
// the grad_W mask and the grad_X mask: one CTA per mask (N <= 8192), or one
// 8-CTA thread-block cluster per mask with distributed-shared-memory reductions.
//
//   scores   integer-exact (reading Z-13): w = floor(sqrt(a b) 2^(16 + 4[h = up]))
//            for grad_W (a = sum code^2 of the half-row, b = sum X_hat^2 of the
//            token), w = floor(sqrt(a) 2^(16 + 4[h = up])) for
//            grad_X.  One IEEE double sqrt per item.
//   A.2      PAPER.md:606-610 run to its fixed point in exact integers: an item
//            is clamped (p = 1) when R w >= W with R = budget - |S| and W the sum
//            of the unclamped positive scores; each round is one cluster-wide
//            reduction through distributed shared memory.  Budget = N (:269).
//   Bernoulli  dyadic two-threshold rule (reading Z-17): e = floor(log2(W/(R w))),
//            T2 = floor(R w 2^32 / W), T1 = 2 T2 - 2^(32-e); Philox word u of item
//            (h, t): keep iff u < T2, weight 2^e if u < T1 else 2^(e+1); floor
//            weight 2^E_MAX (4 for grad_W whose weights fold into int8, 24 for grad_X).
//   compaction  token-major item ids (slot 2t + h) via block scan + cluster prefix, list
//            padded to a multiple of 128 with the sentinel 2N; count stays on device.
//
// The item scores live in shared memory (16384 items per CTA -> N <= 65536,
// the same bound the grad_W INT32 accumulator imposes).  The kernel is
// latency-bound (it moves < 2 MB); it is not an HBM-roofline kernel.
#include <atomic>
#include <cstdlib>

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace i4 {

constexpr int kClusterCTAs = 8;
// threads per CTA: 512 when a CTA holds at most 4096 items (the A.2 rounds and
// the scan are barrier-bound, fewer warps sync faster: cfg2 sampler 8.5 -> 6.9 us,
// BERT-large FFN-up 24.6 -> 21.4 us), 1024 above (ViT: 12.6 K items per CTA)
constexpr int kSamplerThreads = 1024;                 // the maximum
constexpr int kSmallItemsPerCTA = 4096;
constexpr int kItemsPerCTA = 16384;
constexpr int kEMaxW = 4;
constexpr int kEMaxX = 24;

// fixed part of the shared memory; the per-item arrays follow it, sized for the
// CTA's share of the items (launch-time: a small N gets a small footprint):
//   uint64_t w[per] (scores), uint8_t clamped[per] (A.2 set S), int8_t wexp[per]
struct SamplerSmem {
    // group sums: one 16-byte {w lo, w hi, c, 0} partial per (CTA, warp) and parity, written
    // by st.async into every CTA of the cluster; mbar[p] counts their bytes
    uint4 wpart[2][kSamplerThreads / 32];     // this CTA's warp partials
    uint4 part[2][16];                        // CTA partials of the cluster (clusters of up to 16)
    uint64_t mbar[2];
    uint32_t scan[32];
    uint32_t cta_tot[16];
    uint32_t scan2[32];
    uint32_t cta_tot2[16];
};


__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}
__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}

#ifndef I4_STAMPS
#define I4_STAMPS 0
#endif
constexpr bool kSmpStamps = I4_STAMPS != 0;
__device__ int g_smp_stamp_on = 0;
__device__ unsigned long long g_smp_stamp[32];
// fixed-slot stamp (slots 24..30: the phases inside one A.2 round)
__device__ __forceinline__ void smp_mark(int slot, bool on) {
    if (kSmpStamps && on) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        g_smp_stamp[slot] = t;
    }
}

// CTA group of one mask: a single CTA (2N <= 16384 items) or an 8-CTA cluster
// sharing partial sums through distributed shared memory.
template <int CL> struct Group {                  // CL > 1: a thread-block cluster
    cg::cluster_group g = cg::this_cluster();
    __device__ unsigned rank() const { return g.block_rank(); }
    __device__ void sync() const { g.sync(); }
    template <class T> __device__ T* map(T* p, int r) const { return g.map_shared_rank(p, r); }
};
template <> struct Group<1> {
    __device__ unsigned rank() const { return 0; }
    __device__ void sync() const { __syncthreads(); }
    template <class T> __device__ T* map(T* p, int) const { return p; }
};

// items per CTA of a CL-CTA group: even, so a token's two items (slots 2t, 2t+1)
// never straddle two CTAs
__host__ __device__ inline int sampler_per(int N, int CL) { return ((2 * N + CL - 1) / CL + 1) & ~1; }

// Exclusive prefix of v over all threads of the CTA group (thread order within a CTA,
// CTA rank order across the cluster) and the group total.  Collective: every thread of
// every CTA of the group calls it; scan / tot are shared arrays of the caller.
template <int CL, int NT>
__device__ uint32_t group_scan(const Group<CL>& cl, uint32_t v, uint32_t* scan, uint32_t* tot, uint32_t& total) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = int(cl.rank());
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t n = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += n;
    }
    if (lane == 31) scan[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < NT / 32 ? scan[lane] : 0u;
        uint32_t x = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t n = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= o) x += n;
        }
        if (lane < NT / 32) scan[lane] = x - w;            // exclusive warp offsets
        if (lane == 31)
            for (int r = 0; r < CL; ++r) *cl.map(&tot[rank], r) = x;
    }
    cl.sync();
    uint32_t cta_off = 0;
    total = 0;
    for (int r = 0; r < CL; ++r) {
        if (r < rank) cta_off += tot[r];
        total += tot[r];
    }
    return cta_off + scan[warp] + (incl - v);
}

// Exact floor(num 2^32 / W) for 0 < num < W < 2^64 without a 128-bit division:
// a double-precision estimate (relative error < 2^-52, so off by at most a few
// units) corrected by exact 128-bit products.
// est: num 2^32 / W in double precision -- here num * fl(2^32 / W) with the reciprocal
// computed once per CTA (relative error a few 2^-53: the start is off by at most a few
// units, which the exact loops below remove).
__device__ __forceinline__ uint64_t floor_mul2_32_div(uint64_t num, uint64_t W, double est) {
    const unsigned __int128 lhs = (unsigned __int128)num << 32;
    uint64_t q = uint64_t(est);
    if (q > 0) q -= 1;                                  // start at or below the true quotient
    while ((unsigned __int128)(q + 1) * W <= lhs) ++q;  // at most a few steps
    while ((unsigned __int128)q * W > lhs) --q;
    return q;
}

// Group-wide (sum w, sum c); every thread of every CTA receives the totals.  Warp sums go
// to shared memory; after one block barrier every warp forms the CTA total itself (a
// single CTA is done); in a cluster, warp 0's lanes r < CL send it to CTA r with st.async
// into part[parity][rank], completion counted in bytes on CTA r's mbar[parity], and every
// warp sums the CL partials after its CTA's barrier phase completes -- no cluster barrier.
// Integer sums: exact in any order.  Buffers of parity p are reused two rounds later, when
// every CTA has read them (a CTA sends round k + 2 only after receiving everyone's round
// k + 1, which each sent after reading round k).
template <int CL>
__device__ void cluster_sum(const Group<CL>& cl, SamplerSmem& sm, int& parity, uint32_t& mph, uint64_t w,
                            uint32_t c, uint64_t& W, uint32_t& Cn, bool mark = false) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int NW = int(blockDim.x) >> 5;
    w = warp_sum_u64(w);
    c = warp_sum_u32(c);
    smp_mark(26, mark && (w + c) != 1234567);
    if (lane == 0) sm.wpart[parity][warp] = make_uint4(uint32_t(w), uint32_t(w >> 32), c, 0u);
    __syncthreads();
    if (CL == 1 || warp == 0) {
        const uint4 v = lane < NW ? sm.wpart[parity][lane] : make_uint4(0u, 0u, 0u, 0u);
        W = warp_sum_u64(uint64_t(v.x) | (uint64_t(v.y) << 32));
        Cn = warp_sum_u32(v.z);
    }
    if constexpr (CL > 1) {
        if (threadIdx.x == 0) mbar_arrive_expect_tx(&sm.mbar[parity], uint32_t(CL * 16));
        if (warp == 0 && lane < CL)
            st_async_v4(mapa_shared(smem_u32(&sm.part[parity][cl.rank()]), uint32_t(lane)), uint32_t(W),
                        uint32_t(W >> 32), Cn, 0u, mapa_shared(smem_u32(&sm.mbar[parity]), uint32_t(lane)));
        smp_mark(27, mark);
        mbar_wait(&sm.mbar[parity], (mph >> parity) & 1u);
        mph ^= 1u << parity;
        smp_mark(28, mark);
        const uint4 v = lane < CL ? sm.part[parity][lane] : make_uint4(0u, 0u, 0u, 0u);
        W = warp_sum_u64(uint64_t(v.x) | (uint64_t(v.y) << 32));
        Cn = warp_sum_u32(v.z);
    }
    smp_mark(29, mark && (W + Cn) != 1234567);
    parity ^= 1;
}

// timing experiment, compiled in only by -DI4_STAMPS=1 (tools/smp_stamps.py):
// globaltimer stamps of CTA (rank 0, mask 0), thread 0: [0] start [1] scores
// summed [2..] after each A.2 round, then Bernoulli done, compaction done, end;
// slot 31 = number of stamps
__device__ __forceinline__ void smp_stamp(int& n, bool on) {
    if (on) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        if (n < 31) g_smp_stamp[n] = t;
        ++n;
        g_smp_stamp[31] = (unsigned long long)n;
    }
}

int sampler_stamps(unsigned long long* host, int enable) {
    if (!kSmpStamps) return -1;
    if (cudaMemcpyToSymbol(g_smp_stamp_on, &enable, sizeof(int)) != cudaSuccess) return -1;
    if (host && cudaMemcpyFromSymbol(host, g_smp_stamp, sizeof(unsigned long long) * 32) != cudaSuccess) return -1;
    return 0;
}

template <int CL, int NT>
__global__ void __launch_bounds__(NT, 1)
lss_sampler_kernel(SamplerArgs a) {
    pdl_trigger();
    pdl_wait();                                   // a_sq / s_down of grad_split
    const bool st_on = kSmpStamps && g_smp_stamp_on && threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 &&
                       blockIdx.z == 0;
    int st_n = 0;
    smp_stamp(st_n, st_on);
    extern __shared__ __align__(16) uint8_t smem_raw[];
    SamplerSmem& sm = *reinterpret_cast<SamplerSmem*>(smem_raw);
    const Group<CL> cl;
    const int rank = int(cl.rank());
    const int mask_id = blockIdx.y;                      // 0: grad_W, 1: grad_X
    const int N = a.N;
    // batch of this cluster (batched launches: blockIdx.z) and its slices
    const int64_t bz = blockIdx.z;
    const int32_t* const a_sq = a.a_sq + bz * 2 * N;
    const int32_t* const x_sqnorm = a.x_sqnorm != nullptr ? a.x_sqnorm + bz * N : nullptr;
    uint8_t* const x_touched = a.x_touched != nullptr ? a.x_touched + bz * N : nullptr;
    const int64_t tok_off = a.token_offset + bz * N;
    const int n_items = 2 * N;
    const int per = sampler_per(N, CL);
    const int per16 = (per + 15) & ~15;
    uint64_t* sw = reinterpret_cast<uint64_t*>(smem_raw + sizeof(SamplerSmem));
    int8_t* swe = reinterpret_cast<int8_t*>(sw + per16);
    // sw[j]: score (< 2^47: floor(sqrt(a b) 2^20) with a b < 2^53) | kClamped once A.2 clamped
    // the item to p = 1 (the set S) -- one 8-byte word per item, read and written by the rounds
    constexpr uint64_t kClamped = 1ull << 63;
    const int base = rank * per;
    const int nloc = max(0, min(per, n_items - base));
    const int ipt = (per + NT - 1) / NT;                 // items per thread
    const int t_lo = min(nloc, int(threadIdx.x) * ipt);
    const int t_hi = min(nloc, t_lo + ipt);
    const int e_max = mask_id == 0 ? kEMaxW : kEMaxX;
    const uint32_t purpose = mask_id == 0 ? kPurposeMaskW : kPurposeMaskX;
    // slot -> item id: both lists are token-major (slot 2t + h): a token's two items
    // are adjacent rows of the grad_X GEMM (they combine in its epilogue without
    // atomics), and when both masks keep the same set (deterministic masks with
    // equal counts) the two lists are identical, so the grad_W GEMM reads the
    // grad_X GEMM's compacted A and compact skips its own copy
    auto item_of = [&](int slot) { return (slot & 1) * N + (slot >> 1); };
    int parity = 0;
    uint32_t mph = 0;                                    // phase bit of mbar[0] / mbar[1]
    if constexpr (CL > 1) {
        if (threadIdx.x == 0) {
            mbar_init(&sm.mbar[0], 1);
            mbar_init(&sm.mbar[1], 1);
            fence_mbar_init();
        }
        cl.sync();                                       // barriers initialised before any st.async
    }
    if (blockIdx.y == 0 && blockIdx.z == 0 && rank == 0)
        for (int i = threadIdx.x; i < a.n_zero_words; i += NT) a.zero_words[i] = 0u;

    // ---- scores -------------------------------------------------------------
    // the inputs of 8 items are loaded before any is used (one round of load
    // latency per 8 items, not per item: 12 items per thread at ViT sizes)
    uint64_t sum_pos = 0; uint32_t cnt_pos = 0;
    for (int j0 = t_lo; j0 < t_hi; j0 += 8) {
        int32_t av[8], bv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            av[q] = 0; bv[q] = 1;
            const int j = j0 + q;
            if (j < t_hi && a.mode != 2) {
                const int i = item_of(base + j);
                const int t = i >= N ? i - N : i;
                av[q] = __ldg(a_sq + i);
                if (mask_id == 0) bv[q] = __ldg(x_sqnorm + t);
            }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int j = j0 + q;
            if (j >= t_hi) break;
            const int i = item_of(base + j);
            const int h = i >= N ? 1 : 0;
            const int t = i - h * N;
            if (mask_id == 1 && h == 0 && x_touched) x_touched[t] = 0;   // set below for kept items
            uint64_t w = 0;
            if (a.mode != 2) {                                       // I4_LSS_NONE needs no scores
                const double prod = double(av[q]) * double(bv[q]);   // exact: < 2^53
                const double root = __dsqrt_rn(prod);
                w = uint64_t(root * (h == 0 ? 1048576.0 : 65536.0));   // floor(root 2^(16+4[up]))
            }
            sw[j] = w;
            sum_pos += w;
            cnt_pos += (w > 0);
        }
    }
    uint64_t Wall; uint32_t Z;
    cluster_sum(cl, sm, parity, mph, sum_pos, cnt_pos, Wall, Z);
    smp_stamp(st_n, st_on);

    // ---- A.2 water-filling ----------------------------------------------------
    const uint64_t B = uint64_t(N);
    const bool bernoulli = a.mode == 0;
    const bool binding = bernoulli && uint64_t(Z) > B;
    // deterministic set (every positive item with weight 1, or all items): the
    // grad_W set is then a subset of the grad_X set (w_W > 0 implies w_X > 0), so
    // equal counts mean equal lists

    uint64_t R = B, W = Wall;
    uint32_t s_cnt = 0;                                   // |S|: items clamped to p = 1 by A.2
    if (binding) {
        for (int round = 0; round <= n_items + 1; ++round) {
            uint64_t wun = 0; uint32_t sc = 0;
            const bool mk = st_on && round == 2;
            smp_mark(24, mk);
            for (int j0 = t_lo; j0 < t_hi; j0 += 4) {      // 4 items' loads in flight
                uint64_t v[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) v[q] = j0 + q < t_hi ? sw[j0 + q] : 0ull;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint64_t w = v[q] & ~kClamped;
                    bool c = (v[q] & kClamped) != 0;
                    if (w != 0 && !c && R * w >= W) {
                        c = true;
                        sw[j0 + q] = v[q] | kClamped;
                    }
                    sc += (w != 0 && c) ? 1u : 0u;
                    wun += (w != 0 && !c) ? w : 0ull;
                }
            }
            smp_mark(25, mk && (wun + sc) != 1234567);
            uint64_t Wn; uint32_t Sc;
            cluster_sum(cl, sm, parity, mph, wun, sc, Wn, Sc, mk);
            smp_stamp(st_n, st_on);
            if (Sc == s_cnt) break;
            s_cnt = Sc;
            R = B - Sc;
            W = Wn;
        }
    }

    // operand form of this mask's GEMM (reading Z-33): a binding budget that
    // leaves only a few items sampled (0 < p < 1) runs the dense Q / X_hat GEMM plus
    // correction rows for those items instead of compacting every kept item
    const uint32_t n_samp = binding ? Z - s_cnt : 0u;
    const bool corr = binding && a.corr_items != nullptr && uint64_t(n_samp) * 16 <= B;
    if (a.det_flags && rank == 0 && threadIdx.x == 0) a.det_flags[mask_id] = binding ? (corr ? 2 : 0) : 1;

    // ---- Bernoulli with dyadic weights ---------------------------------------
    uint32_t my_keep = 0;
    auto emit = [&](int j, int8_t out) {
        swe[j] = out;
        my_keep += (out >= 0);
        if (mask_id == 1 && out >= 0 && x_touched) {
            const int i = item_of(base + j);
            x_touched[i >= N ? i - N : i] = 1;
        }
    };
    if (a.mode == 2 || !binding) {
        // deterministic: every item (I4_LSS_NONE) or every positive item, weight 1
        // (Z-16: a non-binding budget gives every positive item p = 1)
        for (int j = t_lo; j < t_hi; ++j) emit(j, (a.mode == 2 || (sw[j] & ~kClamped) != 0) ? int8_t(0) : int8_t(-1));
    } else {
        // 4 items per step: their Philox words (computed for every item, straight-line code)
        // and threshold divisions are independent chains whose latencies overlap
        const double rW = 4294967296.0 / double(W);
        for (int j0 = t_lo; j0 < t_hi; j0 += 4) {
            uint64_t v[4];
            uint32_t u[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int j = j0 + q < t_hi ? j0 + q : t_lo;
                v[q] = sw[j];
                const int i = item_of(base + j);
                const int h = i >= N ? 1 : 0;
                const uint64_t idx = 2ull * uint64_t(tok_off + (i - h * N)) + uint64_t(h);
                u[q] = philox4x32_10(uint32_t(idx), uint32_t(idx >> 32), purpose, a.call_id, a.seed_lo, a.seed_hi).x;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (j0 + q >= t_hi) break;
                const uint64_t w = v[q] & ~kClamped;
                int8_t out = -1;
                if (w > 0) {
                    if ((v[q] & kClamped) != 0) {
                        out = 0;               // p = 1 (clamped by A.2)
                    } else {
                        const uint64_t num = R * w;                       // R w < W
                        int e = (63 - __clzll((long long)W)) - (63 - __clzll((long long)num));
                        if ((num << e) > W) --e;
                        uint64_t T1, T2;
                        if (e >= e_max) {
                            e = e_max;
                            T1 = T2 = 1ull << (32 - e_max);
                        } else {
                            T2 = floor_mul2_32_div(num, W, double(num) * rW);
                            T1 = 2 * T2 - (1ull << (32 - e));
                        }
                        if (u[q] < T2) out = int8_t(u[q] < T1 ? e : e + 1);
                    }
                }
                emit(j0 + q, out);
            }
        }
    }

    smp_stamp(st_n, st_on);
    // ---- compaction: block exclusive scan + cluster prefix --------------------
    uint32_t total = 0;
    uint32_t pos = group_scan<CL, NT>(cl, my_keep, sm.scan, sm.cta_tot, total);
    int32_t* items = a.items[mask_id] + bz * a.bs_list;
    int8_t* wexp = a.wexp[mask_id] + bz * a.bs_list;
    for (int j = t_lo; j < t_hi; ++j) {
        const int8_t e = swe[j];
        if (e >= 0) {
            items[pos] = item_of(base + j);
            wexp[pos] = e;
            ++pos;
        }
    }
    if (rank == 0) {
        const uint32_t padded = (total + 127u) & ~127u;
        for (uint32_t p = total + threadIdx.x; p < padded; p += NT) {
            items[p] = n_items;                // sentinel: an all-zero row
            wexp[p] = 0;
        }
        if (threadIdx.x == 0) a.count[mask_id][bz] = int32_t(total);
    }
    if (corr) {
        // form 2 lists.  An item is sampled when its score is positive and A.2 did not
        // clamp it.  grad_W: per sampled item a -1 row and, when kept, a +2^e row (the
        // dense Q^T X_hat already holds weight 1 for every item).  grad_X: every kept
        // item of a token that has a sampled item (its Q row is not used; tok_flag).
        __syncthreads();                       // swe of the whole CTA written
        auto sampled = [&](int j) { return sw[j] != 0 && (sw[j] & kClamped) == 0; };
        uint32_t my_n = 0;
        for (int j = t_lo; j < t_hi; ++j) {
            if (mask_id == 0) my_n += sampled(j) ? 1u + (swe[j] >= 0 ? 1u : 0u) : 0u;
            else my_n += ((sampled(j) || sampled(j ^ 1)) && swe[j] >= 0) ? 1u : 0u;
        }
        uint32_t tot2 = 0;
        uint32_t p2 = group_scan<CL, NT>(cl, my_n, sm.scan2, sm.cta_tot2, tot2);
        int32_t* li = mask_id == 0 ? a.corr_items : a.sub_items;
        int8_t* le = mask_id == 0 ? a.corr_wexp : a.sub_wexp;
        for (int j = t_lo; j < t_hi; ++j) {
            const int it = item_of(base + j);
            if (mask_id == 0) {
                if (!sampled(j)) continue;
                li[p2] = it; le[p2] = -1; ++p2;
                if (swe[j] >= 0) { li[p2] = it; le[p2] = swe[j]; ++p2; }
            } else {
                const bool ts = sampled(j) || sampled(j ^ 1);
                if ((j & 1) == 0) a.tok_flag[it] = ts ? 1 : 0;            // slot 2t: item t (h = 0)
                if (ts && swe[j] >= 0) { li[p2] = it; le[p2] = swe[j]; ++p2; }
            }
        }
        if (rank == 0) {
            const uint32_t padded = (tot2 + 127u) & ~127u;
            for (uint32_t p = tot2 + threadIdx.x; p < padded; p += NT) { li[p] = n_items; le[p] = 0; }
            if (threadIdx.x == 0) *(mask_id == 0 ? a.corr_count : a.sub_count) = int32_t(tot2);
        }
    }
    smp_stamp(st_n, st_on);
    cl.sync();
    smp_stamp(st_n, st_on);                                 // keep DSMEM alive until all remote writes landed
}

template <int CL, int NT>
static void sampler_config(const SamplerArgs& a, cudaStream_t s, cudaLaunchConfig_t& cfg, cudaLaunchAttribute (&attr)[2]) {
    const int per = sampler_per(a.N, CL);
    const int per16 = (per + 15) & ~15;
    cfg = cudaLaunchConfig_t{};
    cfg.gridDim = dim3(CL, 2, unsigned(a.batch > 1 ? a.batch : 1));   // y: 0 = grad_W mask, 1 = grad_X mask; z: batch
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = sizeof(SamplerSmem) + size_t(per16) * (8 + 1);
    cfg.stream = s;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = CL > 1 ? 1 : 0;
}

// function attributes (largest footprint; non-portable cluster size) once per
// (instantiation, device) -- they are per-device state of the CUDA context
template <int CL, int NT>
static cudaError_t set_attrs() {
    static std::atomic<int> done[kMaxDevices];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    if (done[dev].load(std::memory_order_relaxed)) return cudaSuccess;
    auto kern = lss_sampler_kernel<CL, NT>;
    const size_t smem_max = sizeof(SamplerSmem) + size_t(kItemsPerCTA) * (8 + 1);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_max));
    if (e == cudaSuccess && CL > 8) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e == cudaSuccess) done[dev].store(1, std::memory_order_relaxed);
    return e;
}

template <int CL, int NT>
static cudaError_t launch_cl(const SamplerArgs& a, cudaStream_t s) {
    const cudaError_t e = set_attrs<CL, NT>();
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute attr[2];
    sampler_config<CL, NT>(a, s, cfg, attr);
    if (CL == 1) attr[0] = attr[1];
    cfg.attrs = attr;
    cfg.numAttrs = add_pdl_attr(attr, CL > 1 ? 1 : 0);
    return cudaLaunchKernelEx(&cfg, lss_sampler_kernel<CL, NT>, a);
}

// Whether a 16-CTA cluster of the 1024-thread sampler at its largest shared-memory
// footprint can be scheduled on this device (it cannot under MIG / MPS SM limits or
// with GPCs of fewer than 16 usable SMs).  Queried once per device with the
// occupancy API, outside any stream capture, so a captured launch never fails.
static bool cluster16_ok() {
    static std::atomic<int> ok[kMaxDevices];        // 0 unknown, 1 yes, 2 no
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return false;
    int v = ok[dev].load(std::memory_order_relaxed);
    if (v == 0) {
        v = 2;
        if (set_attrs<16, 1024>() == cudaSuccess) {
            SamplerArgs probe{};
            probe.N = kItemsPerCTA * 16 / 2;            // the largest footprint a 16-CTA launch uses
            cudaLaunchConfig_t cfg;
            cudaLaunchAttribute attr[2];
            sampler_config<16, 1024>(probe, nullptr, cfg, attr);
            int n = 0;
            if (cudaOccupancyMaxActiveClusters(&n, lss_sampler_kernel<16, 1024>, &cfg) == cudaSuccess && n >= 1) v = 1;
        }
        (void)cudaGetLastError();
        ok[dev].store(v, std::memory_order_relaxed);
    }
    return v == 1;
}

int sampler_max_tokens() { return kClusterCTAs * kItemsPerCTA / 2; }

cudaError_t launch_lss_sampler(const SamplerArgs& a, cudaStream_t s) {
    // an 8-CTA cluster per mask: the A.2 rounds are dominated by the per-item
    // work, which the cluster spreads over 8 SMs (a single CTA measured 6x slower
    // on binding budgets); tiny problems use one CTA
    // tiny problems (attention BMM batches): one CTA, fewer threads the fewer the items
    // (a barrier of 8 warps is cheaper than one of 32; 4 items per thread at most)
    if (2 * int64_t(a.N) <= 1024) return launch_cl<1, 256>(a, s);
    if (2 * int64_t(a.N) <= 2048) return launch_cl<1, 512>(a, s);
    if (2 * int64_t(a.N) <= int64_t(kClusterCTAs) * kSmallItemsPerCTA) return launch_cl<kClusterCTAs, 512>(a, s);
    // > 8 K items per CTA: a 16-CTA (non-portable) cluster halves each CTA's share
    // (ViT sizes 22.6 -> 15.5 us), when two of them (one per mask) fit on the device
    if (2 * int64_t(a.N) > int64_t(kClusterCTAs) * 2 * kSmallItemsPerCTA && cluster16_ok())
        return launch_cl<16, 1024>(a, s);
    return launch_cl<kClusterCTAs, 1024>(a, s);
}

int sampler_cluster_ctas(int64_t N) {
    if (2 * N <= 2048) return 1;
    if (2 * N > int64_t(kClusterCTAs) * 2 * kSmallItemsPerCTA && cluster16_ok()) return 16;
    return kClusterCTAs;
}

}  // namespace i4
