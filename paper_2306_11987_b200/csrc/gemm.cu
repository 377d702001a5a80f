// INT8 x INT8 -> INT32 GEMM on the 5th-generation tensor cores, used for every
// "INT4 MM" of the operator.  INT4
// codes are stored sign-extended in int8 (sm_100a has no s4 tcgen05 kind), so
// tcgen05.mma.kind::i8 is exact for them; accumulation is int32 in TMEM.
//
//   acc[m, n] = sum_k A(m, k) B(n, k)
//   A is K-major ([M, K] rows) or MN-major ([K, M] rows); the same for B.  The
//   UMMA descriptors read MN-major int8 directly, so no operand is ever
//   transposed in memory (the paper's CUTLASS path needed explicit
//   transpose+contiguous copies).
//
// Structure (one CTA per SM, persistent over output tiles, warp-specialised).
// CG = 2 (default): a CTA pair (thread-block cluster of 2 on one TPC) computes a
// 256 x BN tile with tcgen05.mma.cta_group::2: each CTA stages its 128 rows of
// A and BN/2 rows of B, so per-SM operand traffic is half that of a 1-SM
// 128 x BN tile; the leader CTA issues the MMAs for both.
//   warp 0   TMA producer: 128-byte-swizzled A (128 x 128 B) and B (BN/CG x 128 B)
//            tiles into a STAGES-deep shared-memory ring; completion counted on
//            the leader's mbarrier (2-SM TMA), slots released by a multicast commit.
//   warp 1   allocates 2 x BN TMEM columns (cta_group::CG); the leader's lane 0
//            issues tcgen05.mma (M = 128 CG, N = BN, K = 32 per instruction, 4 per
//            128-deep k-block) and tcgen05.commit to release stages / publish
//            accumulators to both CTAs.
//   warps 2-5 (2-9)  epilogue, one (two) per TMEM lane group -- with 8 warps each
//            takes half of the tile's columns: tcgen05.ld (32 lanes x 32 columns) -> registers, then
//            EPI_INT32  raw accumulators (bit-exact parity checks)
//            EPI_FWD    Y = fl32(acc) * fl32(s_x s_w)   (HQ-MM step 4)
//            EPI_WGRAD  v = acc * s_x s_down 2^{-k/2}; v = I_W o v; v = v H; dW
//            -> swizzled shared-memory staging -> TMA bulk tensor store
//            EPI_DGRAD  row = kept item (h, t): v = acc * s_w s_down 2^wexp 2^{-k/2} (the
//                       A row holds 16 hi or lo -- or q = 16 hi + lo in the dense form --
//                       so s_up = 16 s_down is folded in);
//                       v = I_X[t] o v; v = v H; rows are token-major, so a token's
//                       two items are adjacent lanes: summed by a shuffle and stored
//                       once (pairs straddling a 32-row group: red.add.v4 of 2
//                       addends onto a zeroed row -- order-independent)
//   Two TMEM accumulator stages let the epilogue of tile i overlap the MMAs of
//   tile i+1.  M (grad_X: kept items) or K (grad_W: kept items) may be read
//   from device memory, so the sampled sizes never travel to the host.
#include <cuda.h>

#include "common.cuh"
#include "kernels.h"

namespace i4 {

constexpr int kBM = 128;
constexpr int kBK = 128;                     // bytes = int8 elements along K per stage
constexpr int kStageOutBytes = 4096;         // per epilogue warp per buffer: 32 rows x 128 B
constexpr int kMaxEpiWarps = 8;

// Epilogue warps: 4 (one per TMEM lane group) or 8 (two per lane group, each
// taking one half of the tile's columns) -- the epilogue (tcgen05.ld, scaling,
// masking, the k-level FWHT, stores) is the bottleneck for short-K tiles, so
// it gets twice the warps whenever the register budget of a chunk allows.
// columns per epilogue chunk for Hadamard order 2^KH (one row's block must be
// in one thread's registers)
constexpr int kh_ch(int KH) { return KH <= 5 ? 32 : (1 << KH); }

template <int BN, int EPI, int CH>
struct EpiShape {
    static constexpr int CW = (EPI == EPI_FWD) ? 64 : CH;          // columns per chunk
    static constexpr int WARPS = (CH <= 64 && BN / 2 >= CW) ? 8 : 4;
    static constexpr int COLS = BN / (WARPS / 4);                    // columns per warp
    static constexpr int THREADS = 64 + 32 * WARPS;
};

template <int BN, int CG, int EPW, int EPI, int COLS>
struct GemmCfg {
    static constexpr int A_BYTES = kBM * kBK;
    static constexpr int B_BYTES = (BN / CG) * kBK;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int OUT_BYTES = EPI == EPI_DGRAD ? 0 : EPW * 2 * kStageOutBytes;   // grad_X: direct stores
    static constexpr int MAX_SMEM = 232448 - 1024 - 256;
    static constexpr int STAGES_FIT = (MAX_SMEM - OUT_BYTES) / STAGE_BYTES;
    static constexpr int STAGES = STAGES_FIT < 6 ? STAGES_FIT : 6;
    static constexpr int TMEM_COLS = 2 * BN;
    static constexpr int SMEM = STAGES * STAGE_BYTES + OUT_BYTES + 1024 + 256;
    static_assert(STAGES >= 3, "shared memory ring too shallow");
};

// 16-byte chunk c of staging row r (128-byte rows, SWIZZLE_128B pattern)
__device__ __forceinline__ uint8_t* stage_chunk(uint8_t* buf, int r, int c) {
    return buf + r * 128 + ((c ^ (r & 7)) << 4);
}

// Deterministic split-K (used when there are fewer output tiles than CTA pairs,
// e.g. the grad_W GEMM whose K is the sampled-item count): S splits of the K
// range are separate work units; the unit of the highest K split writes its raw
// INT32 accumulators to a workspace tile, each lower split waits for it, adds
// its own accumulators (integer adds: exact and order-independent) and passes
// it on, and split 0 runs the real epilogue.  Units are numbered so that a unit
// only ever waits on a lower-numbered one, so a persistent grid of co-resident
// CTAs cannot deadlock.
// The partial-sum hand-over costs about kSplitHandoverKb k-blocks of MMA time
// (measured: a 2-way split of a 32-k-block grad_W took longer than none).
#ifndef I4_SPLIT_HANDOVER_KB
#define I4_SPLIT_HANDOVER_KB 24
#endif
constexpr int kSplitHandoverKb = I4_SPLIT_HANDOVER_KB;
__device__ __forceinline__ int choose_splits(int tiles, int pairs, int nk, int max_splits) {
    int best = 1, best_cost = ((tiles + pairs - 1) / pairs) * nk;
    for (int s = 2; s <= max_splits; ++s) {
        if (nk < 2 * s) break;
        const int cost = ((s * tiles + pairs - 1) / pairs) * ((nk + s - 1) / s) + kSplitHandoverKb;
        if (cost < best_cost) { best = s; best_cost = cost; }
    }
    return best;
}

// mask word j of a warp's preloaded column range (j is a compile-time index
// after unrolling the chunk loop only when the range is one chunk; otherwise a
// small select chain keeps the array in registers)
template <int NW>
__device__ __forceinline__ uint32_t mask_word(const uint32_t (&mw)[NW], int j) {
    uint32_t v = mw[0];
#pragma unroll
    for (int q = 1; q < NW; ++q) v = j == q ? mw[q] : v;
    return v;
}

// v = H_k (I o (acc * rscale)) for one CW-column chunk of a row: the mask is
// applied to the integer accumulators, the scale and the butterflies run on
// fp32 pairs (element j with element j + CW/2); same roundings as the scalar
// formula fl(fl(acc) * rscale) followed by the FWHT stages in order.
template <int CW, int KH, int NW>
__device__ __forceinline__ void masked_scaled_fwht(const uint32_t (&r)[CW / 32][32], const uint32_t (&mw)[NW],
                                                   int w0, float rscale, float (&v)[CW]) {
    constexpr int HALF = CW / 2;
    uint32_t m[CW / 32];
#pragma unroll
    for (int q = 0; q < CW / 32; ++q) m[q] = mask_word(mw, w0 + q);
    const uint64_t rs2 = f2_pack(rscale, rscale);
    uint64_t p[HALF];
#pragma unroll
    for (int j = 0; j < HALF; ++j) {
        const int e0 = j, e1 = j + HALF;
        const int32_t a = ((m[e0 >> 5] >> (e0 & 31)) & 1u) ? int32_t(r[e0 >> 5][e0 & 31]) : 0;
        const int32_t b = ((m[e1 >> 5] >> (e1 & 31)) & 1u) ? int32_t(r[e1 >> 5][e1 & 31]) : 0;
        p[j] = f2_mul(f2_pack(float(a), float(b)), rs2);
    }
    fwht_pairs<CW, KH>(p);
#pragma unroll
    for (int j = 0; j < HALF; ++j) f2_unpack(p[j], v[j], v[j + HALF]);
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// KH: Hadamard order k of the grad epilogues (compile-time, 0 for FWD / INT32)
template <int BN, int EPI, int KH, bool A_MN, bool B_MN, int CG>
__global__ void __launch_bounds__(EpiShape<BN, EPI, kh_ch(KH)>::THREADS, 1)
gemm_i8_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmA2,
               const __grid_constant__ CUtensorMap tmA3, const __grid_constant__ CUtensorMap tmB2, const GemmArgs g) {
    constexpr int CH = kh_ch(KH);
    using Epi = EpiShape<BN, EPI, CH>;
    constexpr int kEpiWarps = Epi::WARPS;
    using Cfg = GemmCfg<BN, CG, kEpiWarps, EPI, Epi::COLS>;
    constexpr int BMP = kBM * CG;                // rows per (pair) tile
    constexpr int BNC = BN / CG;                 // B rows / columns staged by this CTA
    constexpr int STAGES = Cfg::STAGES;
    extern __shared__ uint8_t smem_dyn[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = base;
    uint8_t* sB = base + STAGES * Cfg::A_BYTES;
    uint8_t* sOut = base + STAGES * Cfg::STAGE_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sOut + Cfg::OUT_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
    const bool leader = rank == 0;
    const int pair0 = int(blockIdx.x) / CG, n_pairs = int(gridDim.x) / CG;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        if (EPI == EPI_DGRAD) tma_prefetch_desc(&tmA2);
        if (EPI == EPI_WGRAD) { tma_prefetch_desc(&tmA3); tma_prefetch_desc(&tmB2); }
        tma_prefetch_desc(&tmB);
        if (EPI != EPI_DGRAD) tma_prefetch_desc(&tmC);
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], CG * kEpiWarps); }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc<CG>(tmem_slot, Cfg::TMEM_COLS);
    tc_fence_before();
    if (CG == 2) cluster_sync_all(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_trigger();
    pdl_wait();                                  // operands / metadata of the previous kernels

    // problem size (possibly data-dependent, so read after the PDL wait) and work units
    // dense mode (the mask kept every nonzero item with weight 1, reading Z-12): the
    // operands are the 8-bit code plane Q and X_hat themselves, one row per token
    const bool dense = (EPI == EPI_DGRAD || EPI == EPI_WGRAD) && g.dense_flag != nullptr && __ldg(g.dense_flag) != 0;
    const int M = (EPI == EPI_DGRAD && dense) ? g.n_tokens : (g.m_dev ? __ldg(g.m_dev) : g.M);
    const int K = (EPI == EPI_WGRAD && dense) ? ((g.n_tokens + kBK - 1) / kBK) * kBK
                                                : (g.k_dev ? ((__ldg(g.k_dev) + kBK - 1) / kBK) * kBK : g.K);
    const int m_tiles = (M + BMP - 1) / BMP;
    const int n_tiles = (g.Nn + BN - 1) / BN;
    const int T = m_tiles * n_tiles;
    const int nk = (K + kBK - 1) / kBK;
    const int S = (g.partial != nullptr && T <= g.max_tiles_split) ? choose_splits(T, n_pairs, nk, g.max_splits) : 1;
    const int units = S * T;
    // unit u: tile = u % T; split s = S - 1 - u / T (s = 0 is the final one), k-blocks [kb0, kb1)
#define UNIT_DECODE(u)                                          \
    const int tile = (u) % T;                                   \
    const int split = S - 1 - (u) / T;                          \
    const int kb0 = split * nk / S, kb1 = (split + 1) * nk / S;


    if (warp == 0) {
        // ------------------------------------------------------------- producer (warp 0)
        // lane 0 issues the TMA; with a gathered A the 32 lanes first fetch the
        // 128 row indices of the stage (4 per lane) and hand them out by shuffles.
        const bool gather = g.a_gather != nullptr;
        const CUtensorMap* pA = &tmA;
        const CUtensorMap* pB = &tmB;
        if (EPI == EPI_DGRAD && dense) pA = &tmA2;                     // Q, K-major
        if (EPI == EPI_WGRAD) {
            if (dense) { pA = &tmA3; pB = &tmB2; }                    // Q and X_hat, MN-major
        }
        const int gcount = gather ? __ldg(g.gather_count) : 0;
        auto load_idx4 = [&](int r) {
            int4 v;
            v.x = r + 0 < gcount ? __ldg(g.a_gather + r + 0) : g.gather_zero_row;
            v.y = r + 1 < gcount ? __ldg(g.a_gather + r + 1) : g.gather_zero_row;
            v.z = r + 2 < gcount ? __ldg(g.a_gather + r + 2) : g.gather_zero_row;
            v.w = r + 3 < gcount ? __ldg(g.a_gather + r + 3) : g.gather_zero_row;
            return v;
        };
        int stage = 0; uint32_t phase = 0;
        for (int u = pair0; u < units; u += n_pairs) {
            UNIT_DECODE(u)
            const int m0 = (tile / n_tiles) * BMP + kBM * int(rank);   // this CTA's A rows
            const int nb = (tile % n_tiles) * BN + BNC * int(rank);    // this CTA's B rows
            int4 gidx = make_int4(0, 0, 0, 0), gnext = make_int4(0, 0, 0, 0);
            if (gather && !A_MN) gidx = load_idx4(m0 + 4 * lane);       // rows of the tile (grad_X)
            if (gather && A_MN && kb0 < kb1) gnext = load_idx4(kb0 * kBK + 4 * lane);   // K rows (grad_W)
            for (int kb = kb0; kb < kb1; ++kb) {
                if (gather && A_MN) {                 // indices of this stage; prefetch the next stage's
                    gidx = gnext;
                    if (kb + 1 < kb1) gnext = load_idx4((kb + 1) * kBK + 4 * lane);
                }
                if (lane == 0) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (leader) mbar_arrive_expect_tx(&full[stage], CG * Cfg::STAGE_BYTES);
                }
                __syncwarp();
                uint8_t* a_dst = sA + stage * Cfg::A_BYTES;
                uint8_t* b_dst = sB + stage * Cfg::B_BYTES;
                const uint32_t fb = CG == 2 ? mapa_shared(smem_u32(&full[stage]), 0) : smem_u32(&full[stage]);
                if (gather)                            // every lane issues the gather of its own 4 rows
                    tma_gather4<CG>(a_dst + lane * 4 * 128, pA, fb, A_MN ? m0 : kb * kBK,
                                    gidx.x, gidx.y, gidx.z, gidx.w);
                if (lane == 0) {
                    if constexpr (CG == 2) {
                        if (!gather) {
                            if (A_MN) tma_load_2d_2sm(a_dst, pA, fb, m0, kb * kBK);
                            else      tma_load_2d_2sm(a_dst, pA, fb, kb * kBK, m0);
                        }
                        if (B_MN) {
#pragma unroll
                            for (int j = 0; j < BNC / 128; ++j)
                                tma_load_2d_2sm(b_dst + j * 128 * kBK, pB, fb, nb + 128 * j, kb * kBK);
                        } else {
                            tma_load_2d_2sm(b_dst, pB, fb, kb * kBK, nb);
                        }
                    } else {
                        if (!gather) {
                            if (A_MN) tma_load_2d(a_dst, pA, &full[stage], m0, kb * kBK);
                            else      tma_load_2d(a_dst, pA, &full[stage], kb * kBK, m0);
                        }
                        if (B_MN) {
#pragma unroll
                            for (int j = 0; j < BNC / 128; ++j)
                                tma_load_2d(b_dst + j * 128 * kBK, pB, &full[stage], nb + 128 * j, kb * kBK);
                        } else {
                            tma_load_2d(b_dst, pB, &full[stage], kb * kBK, nb);
                        }
                    }
                }
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------- MMA issuer (leader CTA)
        if (lane == 0 && leader) {
            constexpr uint32_t idesc = idesc_i8(BMP, BN, A_MN, B_MN);
            // descriptor advance per K = 32 MMA: K-major +32 B; MN-major +32 rows x 128 B
            constexpr uint64_t a_step = A_MN ? (32 * 128) >> 4 : 32 >> 4;
            constexpr uint64_t b_step = B_MN ? (32 * 128) >> 4 : 32 >> 4;
            int stage = 0; uint32_t phase = 0; int it = 0;
            for (int u = pair0; u < units; u += n_pairs, ++it) {
                UNIT_DECODE(u)
                (void)tile;
                const int as = it & 1;
                const uint32_t ap = (it >> 1) & 1;
                mbar_wait(&tempty[as], ap ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + uint32_t(as * BN);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a_addr = smem_u32(sA + stage * Cfg::A_BYTES);
                    const uint32_t b_addr = smem_u32(sB + stage * Cfg::B_BYTES);
                    const uint64_t adesc = A_MN ? sdesc_mnmajor_sw128(a_addr, 128 * kBK) : sdesc_kmajor_sw128(a_addr);
                    const uint64_t bdesc = B_MN ? sdesc_mnmajor_sw128(b_addr, 128 * kBK) : sdesc_kmajor_sw128(b_addr);
#pragma unroll
                    for (int kk = 0; kk < kBK / 32; ++kk) {
                        const uint32_t acc = (kb > kb0 || kk > 0) ? 1u : 0u;
                        if constexpr (CG == 2) umma_i8_2sm(d_tmem, adesc + a_step * kk, bdesc + b_step * kk, idesc, acc);
                        else umma_i8(d_tmem, adesc + a_step * kk, bdesc + b_step * kk, idesc, acc);
                    }
                    if constexpr (CG == 2) umma_commit_2sm(&empty[stage]); else umma_commit(&empty[stage]);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                if constexpr (CG == 2) umma_commit_2sm(&tfull[as]); else umma_commit(&tfull[as]);
            }
        }
    } else {
        // ------------------------------------------------------------- epilogue
        const int lg = warp & 3;                       // TMEM lane group of this warp
        const int ew = warp - 2;                       // epilogue warp index
        const int cbeg = (ew >> 2) * Epi::COLS;        // this warp's column range [cbeg, cbeg + COLS)
        const int r_in_tile = lg * 32 + lane;
        const int words = g.Nn >> 5;
        uint8_t* stg = sOut + (warp - 2) * (Cfg::OUT_BYTES / kEpiWarps);
        int sbuf = 0;
        float sd = 1.0f;
        if (EPI == EPI_DGRAD || EPI == EPI_WGRAD) sd = __ldg(g.s_down);
        // Row metadata (kept item, its neighbours, its weight exponent) and the mask
        // words of this warp's columns are loaded two / one tile(s) ahead: the mask
        // row of a grad_X item depends on the item index, and both loads would
        // otherwise sit as two dependent global-memory latencies on every tile.
        constexpr bool kMask = EPI == EPI_DGRAD || EPI == EPI_WGRAD;
        constexpr int NW = kMask ? Epi::COLS / 32 : 1;
        const int two_n = 2 * g.n_tokens;
        // Loaded two tiles ahead and left raw until the tile is processed (a consumer
        // right after the load -- e.g. the int8 sign extension of the weight
        // exponent -- made every tile wait for the load, ncu: long-scoreboard on
        // the epilogue warps): the item of this lane's row, the items of the rows
        // just outside the warp's 32 (lanes 31 / 0 only; inner neighbours come by
        // shuffle at use time) and the 32-bit word holding the weight exponent.
        struct RowInfo { int item, edge, eword, rw; };
        auto load_ri = [&](int u) {
            RowInfo x{two_n, two_n, 0, 0};
            if (EPI == EPI_DGRAD && u < units) {
                const int tl = u % T;
                const int rw = (tl / n_tiles) * BMP + kBM * int(rank) + r_in_tile;
                x.rw = rw;
                if (rw < M && dense) {
                    x.item = rw;                       // token rw, weight 1, never paired
                } else if (rw < M) {
                    x.item = __ldg(g.items + rw);
                    x.eword = int(__ldg(reinterpret_cast<const uint32_t*>(g.wexp + (rw & ~3))));
                    if (lane == 31 && rw + 1 < M) x.edge = __ldg(g.items + rw + 1);
                    if (lane == 0 && rw > 0) x.edge = __ldg(g.items + rw - 1);
                }
            }
            return x;
        };
        auto load_mask = [&](int u, const RowInfo& x, uint32_t (&mw)[NW]) {
#pragma unroll
            for (int q = 0; q < NW; ++q) mw[q] = 0u;
            if (!kMask || u >= units) return;
            const int tl = u % T;
            const int rw = (tl / n_tiles) * BMP + kBM * int(rank) + r_in_tile;
            int64_t mrow = rw;
            if (EPI == EPI_DGRAD) {
                if (x.item >= two_n) return;
                mrow = x.item >= g.n_tokens ? x.item - g.n_tokens : x.item;
            } else if (rw >= M) {
                return;
            }
            const int cw0 = ((tl % n_tiles) * BN + cbeg) >> 5;
#pragma unroll
            for (int q = 0; q < NW; ++q)
                if (cw0 + q < words) mw[q] = __ldg(g.mask + mrow * words + cw0 + q);
        };
        RowInfo ri_cur = load_ri(pair0), ri_next = load_ri(pair0 + n_pairs);
        uint32_t mw_cur[NW];
        load_mask(pair0, ri_cur, mw_cur);
        double lsq_acc = 0.0;                          // A.3 partial of this lane
        int it = 0;
        for (int u = pair0; u < units; u += n_pairs, ++it) {
            UNIT_DECODE(u)
            uint32_t mw_next[NW];
            load_mask(u + n_pairs, ri_next, mw_next);  // ri_next arrived during the previous tile
            const RowInfo ri_next2 = load_ri(u + 2 * n_pairs);
            const int as = it & 1;
            const uint32_t ap = (it >> 1) & 1;
            const int m0 = (tile / n_tiles) * BMP + kBM * int(rank), n0 = (tile % n_tiles) * BN;
            const int row = m0 + r_in_tile;
            const bool no_acc = kb1 == kb0;            // empty K range: accumulator is zero
            // split-K bookkeeping for this warp's 32 rows of the tile
            int32_t* part = nullptr;
            uint32_t* flag = nullptr;
            if (S > 1) {
                part = g.partial + (int64_t(tile) * BMP + kBM * int(rank) + r_in_tile) * BN;
                flag = g.flags + (tile * CG + int(rank)) * kMaxEpiWarps + ew;
                if (split < S - 1) {                   // wait until the higher splits are in `part`
                    if (lane == 0) while (ld_acquire_u32(flag) < uint32_t(S - 1 - split)) { }
                    __syncwarp();
                }
            }

            // per-row setup
            bool valid = row < M;
            int64_t out_row = row;
            float rscale = g.scale;
            // grad_X rows are token-major kept items: a token's two items are adjacent
            // rows; the first adds its neighbour's values (shuffle) and stores plainly;
            // pairs straddling a 32-row group use red.add onto rows zeroed beforehand
            int dmode = 0;                             // 0 store, 1 store pair sum, 2 skip, 3 red.add
            int row_e = 0;                             // dgrad: log2 of the item's weight
            if (EPI == EPI_DGRAD) {
                const int item = ri_cur.item;
                valid = valid && item < two_n;
                const int h = item >= g.n_tokens ? 1 : 0;
                out_row = item - h * g.n_tokens;
                const int e = valid ? int(int8_t(uint32_t(ri_cur.eword) >> (8 * (ri_cur.rw & 3)))) : 0;
                // neighbours: rows rw + 1 / rw - 1 (lanes 31 / 0 loaded them; others shuffle);
                // rows at or past M read as the sentinel
                int nx = __shfl_down_sync(0xFFFFFFFFu, ri_cur.item, 1);
                int pv = __shfl_up_sync(0xFFFFFFFFu, ri_cur.item, 1);
                if (lane == 31) nx = ri_cur.edge;
                if (lane == 0) pv = ri_cur.edge;
                if (row + 1 >= M || dense) nx = two_n;
                if (row == 0 || dense) pv = two_n;
                row_e = e;
                rscale = ldexpf(__fmul_rn(g.scale, sd), e);   // s_up = 16 s_down is inside the A codes
                const int inext = valid ? nx : two_n;
                const int iprev = valid ? pv : two_n;
                const bool first = inext < two_n && (inext >= g.n_tokens ? inext - g.n_tokens : inext) == out_row;
                const bool second = iprev < two_n && (iprev >= g.n_tokens ? iprev - g.n_tokens : iprev) == out_row;
                if ((first && lane == 31) || (second && lane == 0)) dmode = 3;
                else if (second) dmode = 2;
                else if (first) dmode = 1;
            } else if (EPI == EPI_WGRAD) {
                rscale = __fmul_rn(g.scale, sd);
            }
            mbar_wait(&tfull[as], ap);
            tc_fence_after();
            const uint32_t t_row = tmem_base + (uint32_t(lg * 32) << 16) + uint32_t(as * BN);

            constexpr int CW = Epi::CW;
#pragma unroll 1
            for (int c = cbeg; c < cbeg + Epi::COLS; c += CW) {
                uint32_t r[CW / 32][32];
#pragma unroll
                for (int q = 0; q < CW / 32; ++q) tmem_ld_32x32b_x32(t_row + uint32_t(c + 32 * q), r[q]);
                tmem_ld_wait();
                if (c + CW >= cbeg + Epi::COLS) {     // this warp's part drained -> MMA may reuse it
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if constexpr (CG == 2) mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(&tempty[as]), 0));
                        else mbar_arrive(&tempty[as]);
                    }
                }
                if (nk == 0 || no_acc) {
#pragma unroll
                    for (int q = 0; q < CW / 32; ++q)
#pragma unroll
                        for (int i = 0; i < 32; ++i) r[q][i] = 0;
                }
                if (S > 1) {
                    int32_t* pc = part + c;
                    if (split < S - 1) {               // add the higher splits' partial sums (exact)
#pragma unroll
                        for (int q = 0; q < CW / 32; ++q)
#pragma unroll
                            for (int i = 0; i < 32; i += 4) {
                                const int4 v = __ldcg(reinterpret_cast<const int4*>(pc + 32 * q + i));
                                r[q][i] += uint32_t(v.x); r[q][i + 1] += uint32_t(v.y);
                                r[q][i + 2] += uint32_t(v.z); r[q][i + 3] += uint32_t(v.w);
                            }
                    }
                    if (split > 0) {                   // pass the running sum on; no output yet
#pragma unroll
                        for (int q = 0; q < CW / 32; ++q)
#pragma unroll
                            for (int i = 0; i < 32; i += 4)
                                __stcg(reinterpret_cast<int4*>(pc + 32 * q + i),
                                       make_int4(int(r[q][i]), int(r[q][i + 1]), int(r[q][i + 2]), int(r[q][i + 3])));
                        continue;
                    }
                }
                const int col0 = n0 + c;
                if (col0 >= g.Nn) continue;           // ragged N (MN-major B): nothing to write
                if (kMask && g.lsq_part != nullptr && valid) {
                    // A.3 step-size gradient: sum_d acc[d] delta[row, d] (fp32 in column order,
                    // then fp64 across chunks; the dgrad item weight 2^e applied exactly)
                    const float* dp = g.delta + (EPI == EPI_DGRAD ? out_row : int64_t(row)) * g.Nn + col0;
                    float cs = 0.0f;
#pragma unroll
                    for (int q = 0; q < CW / 32; ++q)
#pragma unroll
                        for (int i = 0; i < 32; i += 4) {
                            const float4 d4 = __ldg(reinterpret_cast<const float4*>(dp + 32 * q + i));
                            cs = __fmaf_rn(float(int32_t(r[q][i])), d4.x, cs);
                            cs = __fmaf_rn(float(int32_t(r[q][i + 1])), d4.y, cs);
                            cs = __fmaf_rn(float(int32_t(r[q][i + 2])), d4.z, cs);
                            cs = __fmaf_rn(float(int32_t(r[q][i + 3])), d4.w, cs);
                        }
                    lsq_acc += EPI == EPI_DGRAD ? ldexp(double(cs), row_e) : double(cs);
                }

                if (EPI == EPI_DGRAD) {
                    float v[CW];
                    masked_scaled_fwht<CW, KH>(r, mw_cur, (c - cbeg) / 32, rscale, v);
                    if (!dense) {                           // token rows (dense) have no partner item
#pragma unroll
                        for (int i = 0; i < CW; ++i) {     // warp-wide: every lane takes part
                            const float o = __shfl_down_sync(0xFFFFFFFFu, v[i], 1);
                            if (dmode == 1) v[i] = __fadd_rn(v[i], o);
                        }
                    }
                    if (g.out_bf16) {                       // perf mode: bf16 grad_X (reading Z-24)
                        uint32_t pk[CW / 2];
#pragma unroll
                        for (int i = 0; i < CW / 2; ++i) {
                            __nv_bfloat162 p2 = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
                            pk[i] = *reinterpret_cast<uint32_t*>(&p2);
                        }
                        __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(g.out) + (valid ? out_row : 0) * g.Nn + col0;
                        if (valid && dmode == 3) {          // 2 bf16 addends onto 0: order-independent
#pragma unroll
                            for (int i = 0; i < CW / 2; ++i) red_add_bf16x2(dst + 2 * i, pk[i]);
                        } else if (valid && dmode != 2) {
#pragma unroll
                            for (int i = 0; i < CW / 2; i += 4)
                                *reinterpret_cast<uint4*>(dst + 2 * i) = make_uint4(pk[i], pk[i + 1], pk[i + 2], pk[i + 3]);
                        }
                        continue;
                    }
                    const int64_t mrow = valid ? out_row : 0;
                    float* dst = reinterpret_cast<float*>(g.out) + mrow * g.Nn + col0;
                    if (valid && dmode == 3) {
#pragma unroll
                        for (int i = 0; i < CW; i += 4) red_add_v4(dst + i, v[i], v[i + 1], v[i + 2], v[i + 3]);
                    } else if (valid && dmode != 2) {
#pragma unroll
                        for (int i = 0; i < CW; i += 4)
                            *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                    }
                    continue;
                }

                // value transform into 32-bit words, then stage 32 x 128 B sub-tiles
                if (EPI == EPI_FWD && g.out_bf16) {
                    // 64 bf16 columns = one 128-byte staging row
                    uint32_t packed[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const float a = __fmul_rn(float(int32_t(r[i >> 4][(2 * i) & 31])), rscale);
                        const float b = __fmul_rn(float(int32_t(r[i >> 4][(2 * i + 1) & 31])), rscale);
                        __nv_bfloat162 p2 = __floats2bfloat162_rn(a, b);
                        packed[i] = *reinterpret_cast<uint32_t*>(&p2);
                    }
                    if (lane == 0) bulk_wait_read<1>();
                    __syncwarp();
                    uint8_t* buf = stg + sbuf * kStageOutBytes;
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        *reinterpret_cast<uint4*>(stage_chunk(buf, lane, q)) =
                            make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) { tma_store_2d(&tmC, buf, col0, m0 + lg * 32); bulk_commit(); }
                    sbuf ^= 1;
                    continue;
                }

                uint32_t wv[CW];                      // 32-bit output words (int32 or fp32 bits)
                if (EPI == EPI_INT32) {
#pragma unroll
                    for (int i = 0; i < CW; ++i) wv[i] = r[i >> 5][i & 31];
                } else if (EPI == EPI_FWD) {
#pragma unroll
                    for (int i = 0; i < CW; ++i)
                        wv[i] = __float_as_uint(__fmul_rn(float(int32_t(r[i >> 5][i & 31])), rscale));
                } else {                              // EPI_WGRAD
                    float v[CW];
                    masked_scaled_fwht<CW, KH>(r, mw_cur, (c - cbeg) / 32, rscale, v);
#pragma unroll
                    for (int i = 0; i < CW; ++i) wv[i] = __float_as_uint(v[i]);
                }
#pragma unroll
                for (int q = 0; q < CW / 32; ++q) {
                    if (col0 + 32 * q >= g.Nn) break;
                    if (lane == 0) bulk_wait_read<1>();
                    __syncwarp();
                    uint8_t* buf = stg + sbuf * kStageOutBytes;
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        *reinterpret_cast<uint4*>(stage_chunk(buf, lane, j)) =
                            make_uint4(wv[32 * q + 4 * j], wv[32 * q + 4 * j + 1], wv[32 * q + 4 * j + 2], wv[32 * q + 4 * j + 3]);
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) { tma_store_2d(&tmC, buf, col0 + 32 * q, m0 + lg * 32); bulk_commit(); }
                    sbuf ^= 1;
                }
            }
            ri_cur = ri_next; ri_next = ri_next2;
#pragma unroll
            for (int q = 0; q < NW; ++q) mw_cur[q] = mw_next[q];
            if (S > 1) {
                __syncwarp();
                if (split > 0) {                       // publish: this warp's rows now hold S - split splits
                    __threadfence();
                    if (lane == 0) st_release_u32(flag, uint32_t(S - split));
                } else if (lane == 0) {
                    *flag = 0u;                        // consumed: reset for the next launch
                }
            }
        }
#undef UNIT_DECODE
        if (kMask && g.lsq_part != nullptr) {          // fixed-order warp sum -> this warp's slot
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) lsq_acc += __shfl_xor_sync(0xFFFFFFFFu, lsq_acc, o);
            if (lane == 0) g.lsq_part[int(blockIdx.x) * kMaxEpiWarps + ew] = lsq_acc;
        }
        bulk_wait<0>();                                // every lane: its own copies are done
        __syncwarp();
    }

    tc_fence_before();
    if (CG == 2) cluster_sync_all(); else __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc<CG>(tmem_base, Cfg::TMEM_COLS);
}

size_t gemm_split_partial_bytes() { return size_t(kSplitMaxTiles) * (kBM * kGemmCG) * 256 * sizeof(int32_t); }
size_t gemm_split_flag_words() { return size_t(kSplitMaxTiles) * kGemmCG * kMaxEpiWarps; }

int gemm_block_n(int Nn, bool b_mn) {
    if (Nn % 256 == 0 || b_mn) return 256;      // MN-major B halves are whole 128-byte atoms
    if (Nn % 128 == 0) return 128;
    return 64;
}

constexpr int kCG = kGemmCG;                    // CTA pairs (cta_group::2) for every GEMM

template <int BN, int EPI, int KH, bool A_MN, bool B_MN>
static cudaError_t launch_one(const GemmMaps& m, const GemmArgs& g, int grid, cudaStream_t s) {
    auto kern = gemm_i8_kernel<BN, EPI, KH, A_MN, B_MN, kCG>;
    using Epi = EpiShape<BN, EPI, kh_ch(KH)>;
    constexpr int smem = GemmCfg<BN, kCG, Epi::WARPS, EPI, Epi::COLS>::SMEM;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(Epi::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kCG; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = add_pdl_attr(attr, 1);
    return cudaLaunchKernelEx(&cfg, kern, *reinterpret_cast<const CUtensorMap*>(m.a),
                              *reinterpret_cast<const CUtensorMap*>(m.b), *reinterpret_cast<const CUtensorMap*>(m.c),
                              *reinterpret_cast<const CUtensorMap*>(m.a2 ? m.a2 : m.a),
                              *reinterpret_cast<const CUtensorMap*>(m.a3 ? m.a3 : m.a),
                              *reinterpret_cast<const CUtensorMap*>(m.b2 ? m.b2 : m.b), g);
}

template <int EPI, int KH, bool A_MN, bool B_MN>
static cudaError_t dispatch_bn(int bn, const GemmMaps& m, const GemmArgs& g, int grid, cudaStream_t s) {
    if (bn == 256) return launch_one<256, EPI, KH, A_MN, B_MN>(m, g, grid, s);
    if constexpr (!B_MN) {
        if (bn == 128) return launch_one<128, EPI, KH, A_MN, B_MN>(m, g, grid, s);
        if constexpr (kh_ch(KH) <= 64) return launch_one<64, EPI, KH, A_MN, B_MN>(m, g, grid, s);
    }
    return cudaErrorInvalidValue;
}

template <int EPI, bool A_MN, bool B_MN>
static cudaError_t dispatch_ch(int bn, const GemmMaps& m, const GemmArgs& g, int grid, cudaStream_t s) {
    if constexpr (EPI == EPI_DGRAD || EPI == EPI_WGRAD) {
        switch (g.k_had) {
            case 0: return dispatch_bn<EPI, 0, A_MN, B_MN>(bn, m, g, grid, s);
            case 1: return dispatch_bn<EPI, 1, A_MN, B_MN>(bn, m, g, grid, s);
            case 2: return dispatch_bn<EPI, 2, A_MN, B_MN>(bn, m, g, grid, s);
            case 3: return dispatch_bn<EPI, 3, A_MN, B_MN>(bn, m, g, grid, s);
            case 4: return dispatch_bn<EPI, 4, A_MN, B_MN>(bn, m, g, grid, s);
            case 5: return dispatch_bn<EPI, 5, A_MN, B_MN>(bn, m, g, grid, s);
            case 6: return dispatch_bn<EPI, 6, A_MN, B_MN>(bn, m, g, grid, s);
            case 7: return dispatch_bn<EPI, 7, A_MN, B_MN>(bn, m, g, grid, s);
            default: return cudaErrorInvalidValue;
        }
    } else {
        return dispatch_bn<EPI, 0, A_MN, B_MN>(bn, m, g, grid, s);
    }
}

cudaError_t launch_gemm(const GemmMaps& m, const GemmArgs& g, int num_sms, cudaStream_t s) {
    const int bn = gemm_block_n(g.Nn, g.b_mn);
    const int64_t tiles = int64_t((g.M + kBM * kCG - 1) / (kBM * kCG)) * ((g.Nn + bn - 1) / bn);   // g.M = bound
    const int64_t pairs = num_sms / kCG;
    // split-K turns each of few tiles into several work units: size the grid for those
    const int64_t units = (g.partial != nullptr && tiles <= g.max_tiles_split) ? tiles * g.max_splits : tiles;
    int grid = kCG * int(units < pairs ? units : pairs);
    if (grid < kCG) grid = kCG;
    switch (g.epi) {
        case EPI_FWD: return dispatch_ch<EPI_FWD, false, false>(bn, m, g, grid, s);
        case EPI_DGRAD: return dispatch_ch<EPI_DGRAD, false, true>(bn, m, g, grid, s);
        case EPI_WGRAD: return dispatch_ch<EPI_WGRAD, true, true>(bn, m, g, grid, s);
        case EPI_INT32:
            if (!g.a_mn && !g.b_mn) return dispatch_ch<EPI_INT32, false, false>(bn, m, g, grid, s);
            if (!g.a_mn && g.b_mn) return dispatch_ch<EPI_INT32, false, true>(bn, m, g, grid, s);
            if (g.a_mn && g.b_mn) return dispatch_ch<EPI_INT32, true, true>(bn, m, g, grid, s);
            return dispatch_ch<EPI_INT32, true, false>(bn, m, g, grid, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace i4
