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
// Structure (one CTA per SM, persistent, warp-specialised).  A CTA pair
// (thread-block cluster of 2 on one TPC) computes a 256 x BN tile with
// tcgen05.mma.cta_group::2: each CTA stages its 128 rows of A and BN/2 rows of
// B, so per-SM operand traffic is half that of a 1-SM 128 x BN tile; the leader
// CTA issues the MMAs for both.
//   warp 0   TMA producer: 128-byte-swizzled A (128 x 128 B) and B (BN/CG x 128 B)
//            tiles into a STAGES-deep shared-memory ring; completion counted on
//            the leader's mbarrier (2-SM TMA), slots released by a multicast commit.
//   warp 1   allocates 2 x BN TMEM columns (cta_group::CG); the leader's lane 0
//            issues tcgen05.mma (M = 256, N = BN, K = 32 per instruction, 4 per
//            128-deep k-block) and tcgen05.commit to release stages / publish
//            accumulators to both CTAs.
//   warps 2-9 (2-5)  epilogue, two (one) per TMEM lane group: tcgen05.ld (32 lanes x
//            32 columns) -> registers, then
//            EPI_INT32  raw accumulators (bit-exact parity checks)
//            EPI_FWD    Y = fl32(acc) * fl32(s_x s_w)   (HQ-MM step 4)
//            EPI_WGRAD  v = acc * s_x s_down 2^{-k/2}; v = I_W o v; v = v H; dW
//            -> swizzled shared-memory staging -> TMA bulk tensor store
//            EPI_DGRAD  row = kept item (h, t): v = acc * s_w s_down 2^wexp 2^{-k/2} (the
//                       A row holds 16 hi or lo -- or q = 16 hi + lo in the dense form --
//                       so s_up = 16 s_down is folded in);
//                       v = I_X[t] o v; v = v H; rows are token-major, so a token's
//                       two items are adjacent lanes: summed by a shuffle and stored
//                       once (pairs straddling a 32-row group: red.add of 2
//                       addends onto a zeroed row -- order-independent)
//            EPI_BWD    the grad_X (problem 0, EPI_DGRAD) and grad_W (problem 1,
//                       EPI_WGRAD) GEMMs of one backward in ONE persistent launch:
//                       their tiles share one schedule, so neither under-fills the GPU
//   Two TMEM accumulator stages let the epilogue of tile i overlap the MMAs of
//   tile i+1.  M (grad_X: kept items) or K (grad_W: kept items) may be read
//   from device memory, so the sampled sizes never travel to the host.
//
// Schedule (static, deterministic).  The output tiles of the launch are dealt
// to the CTA pairs before any work starts; every CTA derives the same
// assignment from the (device-resident) problem sizes.  One problem: tile
// p + j P goes to pair p.  EPI_BWD (two problems whose tiles have different
// lengths in k-blocks, e.g. 64 k-block grad_W tiles next to 24 k-block grad_X
// tiles for BERT-large QKV): the long tiles are dealt round-robin, then every
// pair gets a contiguous run of short tiles sized so that its k-block total
// comes as close as the tile granularity allows to the average W / P (extra
// tiles first to the pairs with the most room) -- a closed-form longest-first
// balance (QKV: 96 k-blocks on the busiest pair instead of 112 round-robin).
// (A stream-K split of tiles across pairs, with exact INT32 partial sums, was
// built and measured slower on every shape here: each piece costs a full
// accumulator hand-over through L2.)
#include <cuda.h>

#include "common.cuh"
#include "kernels.h"

namespace i4 {

constexpr int kBM = 128;
constexpr int kBK = 128;                     // bytes = int8 elements along K per stage
constexpr int kStageOutBytes = 4096;         // per epilogue warp per buffer: 32 rows x 128 B
constexpr int kMaxEpiWarps = 8;
#ifndef I4_GEMM_SCHED
#define I4_GEMM_SCHED 2                      // 0 round-robin, 1 balanced long-first, 2 balanced short-first
#endif
constexpr bool kBalance = I4_GEMM_SCHED != 0;
constexpr bool kShortFirst = I4_GEMM_SCHED == 2;
#ifndef I4_EPI_KB_DGRAD
#define I4_EPI_KB_DGRAD 14                   // measured: a 256 x 256 grad_X tile's epilogue ~ 14 k-blocks of MMA
#endif
#ifndef I4_EPI_KB_WGRAD
#define I4_EPI_KB_WGRAD 8
#endif

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

template <int BN, int CG, int EPW, int EPI, int COLS, int EXTRA = 0>
struct GemmCfg {
    static constexpr int A_BYTES = kBM * kBK;
    static constexpr int B_BYTES = (BN / CG) * kBK;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int OUT_BYTES = EPI == EPI_DGRAD ? 0 : EPW * 2 * kStageOutBytes;   // grad_X: direct stores
    static constexpr int MAX_SMEM = 232448 - 1024 - 256;
    static constexpr int STAGES_FIT = (MAX_SMEM - OUT_BYTES - EXTRA) / STAGE_BYTES;
    static constexpr int STAGES = STAGES_FIT < 6 ? STAGES_FIT : 6;
    static constexpr int TMEM_COLS = 2 * BN;
    static constexpr int SMEM = STAGES * STAGE_BYTES + OUT_BYTES + 1024 + 256 + EXTRA;
    static_assert(STAGES >= 3, "shared memory ring too shallow");
};

// 16-byte chunk c of staging row r (128-byte rows, SWIZZLE_128B pattern)
__device__ __forceinline__ uint8_t* stage_chunk(uint8_t* buf, int r, int c) {
    return buf + r * 128 + ((c ^ (r & 7)) << 4);
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

// ---------------------------------------------------------------------------- schedule
// Device-resolved size of one problem of the launch.
// form: the operand form the sampler chose for this mask -- 0 the compacted kept items,
// 1 dense (reading Z-32: Q and X_hat, one row per token), 2 dense + correction (reading
// Z-33): grad_X = Q token rows (m-tiles 0 .. mtd-1) then sub-list item rows; grad_W = Q /
// X_hat token k-blocks (0 .. nkd-1) then correction k-blocks
struct ProbSize { int M, K, m_tiles, n_tiles, T, nk; int form, mtd, nkd; };

template <int EPI, int BMP, int BN>
__device__ __forceinline__ ProbSize prob_size(const GemmArgs& g) {
    ProbSize s{};
    // every word the size may depend on is loaded up front (independent loads: one
    // L2 round trip after the PDL wait instead of a dependent chain)
    const int f = (EPI == EPI_DGRAD || EPI == EPI_WGRAD) && g.dense_flag != nullptr ? __ldg(g.dense_flag) : 0;
    const int md = g.m_dev != nullptr ? __ldg(g.m_dev) : g.M;
    const int md2 = EPI == EPI_DGRAD && g.m_dev2 != nullptr ? __ldg(g.m_dev2) : 0;
    const int kd = g.k_dev != nullptr ? __ldg(g.k_dev) : 0;
    const int kd2 = EPI == EPI_WGRAD && g.k_dev2 != nullptr ? __ldg(g.k_dev2) : 0;
    s.form = f;
    const int tok_kb = (g.n_tokens + kBK - 1) / kBK;
    if (EPI == EPI_DGRAD && s.form == 1) s.M = g.n_tokens;
    else if (EPI == EPI_DGRAD && s.form == 2) { s.mtd = (g.n_tokens + BMP - 1) / BMP; s.M = s.mtd * BMP + md2; }
    else s.M = md;
    if (EPI == EPI_WGRAD && s.form == 1) s.K = tok_kb * kBK;
    else if (EPI == EPI_WGRAD && s.form == 2) { s.nkd = tok_kb; s.K = (tok_kb + (kd2 + kBK - 1) / kBK) * kBK; }
    else s.K = g.k_dev != nullptr ? ((kd + kBK - 1) / kBK) * kBK : g.K;
    s.m_tiles = (s.M + BMP - 1) / BMP;
    s.n_tiles = (g.Nn + BN - 1) / BN;
    s.T = s.m_tiles * s.n_tiles;
    s.nk = (s.K + kBK - 1) / kBK;
    return s;
}

// Tile assignment.  Tiles are numbered problem 0 first (T0 tiles of L0 k-blocks)
// then problem 1 (T1 of L1).  The "long" class (larger k-blocks per tile) is dealt
// round-robin; the "short" class is cut into contiguous runs, run p of length
// quota(p) starting at start(p), so that pair p's total approaches W / P.
struct Sched {
    int P;                         // CTA pairs
    int T0, L0, T1, L1;            // tiles and k-blocks per tile of problem 0 and problem 1
    bool two;                      // two-class balance (else round-robin over all tiles)
    int long_prob;                 // problem of the long class
    int TL, LL, TS, LS;            // long / short class: tiles, k-blocks per tile
    int r1;                        // pairs 0 .. r1-1 hold one long tile more than the others
    int qx, qy;                    // base short quota of those pairs / of the others
    int R;                         // short tiles left after the base quotas (>= 0 here)
    bool y_first;                  // the extra short tiles go to pairs r1.. first
    int my_nl, my_ns, my_start;    // this pair's long tiles, short quota, first short tile
    // E0, E1: a tile's cost floor in k-blocks (its epilogue time: a short-K grad_X tile
    // is epilogue-bound), so tile p's weight is max(k-blocks, E).  32-bit arithmetic (every
    // quantity is below 2^31): this runs between the PDL wait and the first TMA load.
    __device__ void init(int P_, int T0_, int L0_, int T1_, int L1_, int E0, int E1, int p) {
        P = P_; T0 = T0_; L0 = L0_; T1 = T1_; L1 = L1_;
        two = kBalance && T1 > 0 && T0 > 0 && L0 > 0 && L1 > 0;
        if (!two) return;
        const int w0 = L0 > E0 ? L0 : E0, w1 = L1 > E1 ? L1 : E1;
        long_prob = w1 >= w0 ? 1 : 0;
        TL = long_prob ? T1 : T0; LL = long_prob ? w1 : w0;
        TS = long_prob ? T0 : T1; LS = long_prob ? w0 : w1;
        const int W = TL * LL + TS * LS;
        const int tau = (W + P - 1) / P;
        const int tlp = TL / P;
        r1 = TL - tlp * P;
        const int lx = (tlp + 1) * LL, ly = tlp * LL;
        qx = tau > lx ? (tau - lx) / LS : 0;
        qy = tau > ly ? (tau - ly) / LS : 0;
        int base = r1 * qx + (P - r1) * qy;
        // never more short tiles than there are: trim the base quotas (pairs with long
        // tiles first) -- only possible through the rounding of tau
        while (base > TS) {
            if (qx > 0 && r1 > 0 && lx + qx * LS >= ly + qy * LS) { --qx; base -= r1; }
            else if (qy > 0) { --qy; base -= P - r1; }
            else { --qx; base -= r1; }
        }
        R = TS - base;
        const int slack_x = tau - lx - qx * LS, slack_y = tau - ly - qy * LS;
        y_first = r1 == 0 || slack_y >= slack_x;
        my_nl = tlp + (p < r1 ? 1 : 0);
        const int rp = R / P, rm = R - rp * P;
        my_ns = (p < r1 ? qx : qy) + rp + (extra(p, rm) ? 1 : 0);
        my_start = min(p, r1) * qx + max(0, p - r1) * qy + p * rp + n_extra_before(p, rm);
    }
    // number of pairs r < p whose priority rank is below m (the first m of the order
    // get one extra short tile)
    __device__ int n_extra_before(int p, int m) const {
        if (m <= 0) return 0;
        if (!y_first) return p < m ? p : m;                                   // order 0, 1, ..., P-1
        const int xs = min(p, r1), ys = max(0, p - r1);                       // order r1.., then 0..r1-1
        const int cy = min(ys, m);
        const int cx = max(0, min(xs, m - (P - r1)));
        return cy + cx;
    }
    __device__ bool extra(int p, int m) const {
        const int rank = y_first ? (p >= r1 ? p - r1 : (P - r1) + p) : p;
        return rank < m;
    }
};

// j-th tile of pair p (b: its batch in a batched launch)
struct Seg { int prob, tile, nk, b; bool valid; };

// batched backward launches: per-batch tile table in shared memory after the barriers
// ([B + 1] prefix of tiles per batch, [B] grad_X tiles per batch)
constexpr int kBatSmem = ((2 * kMaxGemmBatch + 1) * 4 + 15) / 16 * 16;

__device__ __forceinline__ Seg seg_at(const Sched& s, int p, int j) {
    Seg r{};
    if (!s.two) {
        const int t = p + j * s.P;
        if (t >= s.T0 + s.T1) return r;
        r.prob = t < s.T0 ? 0 : 1;
        r.tile = t < s.T0 ? t : t - s.T0;
    } else {
        const int nl = s.my_nl, ns = s.my_ns;             // p is the pair Sched::init was given
        if (kShortFirst ? j >= ns : j < nl) {          // a long tile
            const int jl = kShortFirst ? j - ns : j;
            if (jl >= nl) return r;
            r.prob = s.long_prob;
            r.tile = p + jl * s.P;
        } else {
            const int js = kShortFirst ? j : j - nl;
            if (js >= ns) return r;
            r.prob = 1 - s.long_prob;
            r.tile = s.my_start + js;
        }
    }
    r.nk = r.prob == 0 ? s.L0 : s.L1;
    r.valid = true;
    return r;
}

// timing experiment, compiled in only by -DI4_STAMPS=1 (tools/gemm_stamps.py): globaltimer
// stamps of CTA 0 -- [0] entry [1] setup done [2] PDL wait done [3] first TMA issued [4] first
// stage full (MMA) [5] last MMA committed [6] first accumulator ready (epilogue warp 2)
// [7] epilogue done [8] exit; [9] earliest CTA entry, [10] latest CTA exit (all CTAs)
#ifndef I4_STAMPS
#define I4_STAMPS 0
#endif
constexpr bool kGemmStamps = I4_STAMPS != 0;
__device__ unsigned long long g_gemm_stamp[16];
__device__ __forceinline__ void gstamp(int i, bool on) {
    if (kGemmStamps && on) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        if (i == 9) atomicMin(&g_gemm_stamp[9], t);
        else if (i == 10) atomicMax(&g_gemm_stamp[10], t);
        else g_gemm_stamp[i] = t;
    }
}

int gemm_stamps(unsigned long long* host) {
    if (!kGemmStamps) return -1;
    if (cudaMemcpyFromSymbol(host, g_gemm_stamp, sizeof(unsigned long long) * 16) != cudaSuccess) return -1;
    unsigned long long init[16] = {};
    init[9] = ~0ull;
    return cudaMemcpyToSymbol(g_gemm_stamp, init, sizeof(init)) == cudaSuccess ? 0 : -1;
}

// ---------------------------------------------------------------------------- kernel
struct GemmMapSet { CUtensorMap m[9]; };
enum { MAP_A = 0, MAP_B = 1, MAP_C = 2, MAP_A2 = 3, MAP_A3 = 4, MAP_B2 = 5, MAP_AW = 6, MAP_BW = 7, MAP_DX = 8 };

// KH: Hadamard order k of the grad epilogues (compile-time, 0 for FWD / INT32).
// EPI_BWD: problem 0 = grad_X (A K-major, B MN-major, args g), problem 1 = grad_W
// (A and B MN-major, args g1); A_MN / B_MN describe the single-problem kinds.
// BAT: batched launch (EPI_FWD / EPI_BWD of the attention BMM): 3-D maps, tiles of
// every batch dealt round-robin to the pairs (GemmArgs::batch).
template <int BN, int EPI, int KH, bool A_MN, bool B_MN, int CG, bool BAT>
__global__ void __launch_bounds__(EpiShape<BN, (EPI == EPI_BWD ? EPI_WGRAD : EPI), kh_ch(KH)>::THREADS, 1)
gemm_i8_kernel(const __grid_constant__ GemmMapSet maps, const GemmArgs g, const GemmArgs g1) {
    constexpr bool kBwd = EPI == EPI_BWD;
    constexpr int EPI0 = kBwd ? EPI_DGRAD : EPI;                 // kind of problem 0
    constexpr int CH = kh_ch(KH);
    using Epi = EpiShape<BN, (kBwd ? EPI_WGRAD : EPI), CH>;
    constexpr int kEpiWarps = Epi::WARPS;
    using Cfg = GemmCfg<BN, CG, kEpiWarps, (kBwd ? EPI_WGRAD : EPI), Epi::COLS, (BAT && kBwd) ? kBatSmem : 0>;
    static_assert(!BAT || (CG == 2 && (EPI == EPI_FWD || EPI == EPI_BWD)), "batched: FWD / BWD pairs only");
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
    int* bpref = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(full) + 256);   // BAT bwd: [B + 1]
    int* btd = bpref + kMaxGemmBatch + 1;                                         // BAT bwd: [B]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
    const bool leader = rank == 0;
    const int pair0 = int(blockIdx.x) / CG, n_pairs = int(gridDim.x) / CG;
    const bool st0 = blockIdx.x == 0;
    gstamp(0, st0 && threadIdx.x == 0);
    gstamp(9, threadIdx.x == 0);

    if (warp == 0 && lane == 0) {
#pragma unroll
        for (int i = 0; i < 9; ++i) tma_prefetch_desc(&maps.m[i]);
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], CG * kEpiWarps); }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc<CG>(tmem_slot, Cfg::TMEM_COLS);
    tc_fence_before();
    if (CG == 2) cluster_sync_all(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    gstamp(1, st0 && threadIdx.x == 0);
    pdl_trigger();

    // Problem sizes and the schedule, BEFORE the PDL wait: the only device-resident sizes
    // (kept counts, operand forms) are the sampler's, two launches back, and the backward
    // GEMM's predecessor (compact_kernel) signals its dependents only after its own PDL
    // wait, i.e. after the sampler grid completed -- so they are final when this grid
    // starts, and their L2 round trip overlaps compact instead of delaying the first TMA.
    // Everything compact writes (the gathered operands, zeroed rows) is read after the wait.
    const ProbSize s0 = prob_size<EPI0, BMP, BN>(g);
    ProbSize s1{};
    if constexpr (kBwd) s1 = prob_size<EPI_WGRAD, BMP, BN>(g1);
    gstamp(11, st0 && threadIdx.x == 0 && (s0.M + s1.M) >= 0);
    Sched sc;
    if constexpr (!BAT)
        sc.init(n_pairs, s0.T, s0.nk, kBwd ? s1.T : 0, kBwd ? s1.nk : 0, I4_EPI_KB_DGRAD, I4_EPI_KB_WGRAD, pair0);
    if constexpr (BAT && kBwd) {
        // tile table: batch b has ceil(M_b / 256) grad_X m-tiles (M_b = its kept items, from
        // the sampler) and a fixed number of grad_W tiles; prefix over the batches by warp 0
        // (lane l scans a contiguous chunk).  Identical in both CTAs of a pair.
        const int B = g.batch;
        for (int b = threadIdx.x; b < B; b += blockDim.x) {
            const int td = ((__ldg(g.m_dev + b) + BMP - 1) / BMP) * s0.n_tiles;
            btd[b] = td;
            bpref[b + 1] = td + s1.T;
        }
        __syncthreads();
        if (warp == 0) {
            const int ch = (B + 31) / 32, lo = min(B, lane * ch), hi = min(B, lo + ch);
            int run = 0;
            for (int b = lo; b < hi; ++b) { run += bpref[b + 1]; bpref[b + 1] = run; }
            int incl = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int n = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= o) incl += n;
            }
            const int off = incl - run;
            for (int b = lo; b < hi; ++b) bpref[b + 1] += off;
            if (lane == 0) bpref[0] = 0;
        }
        __syncthreads();
    }
    // j-th tile of this pair.  Batched: global tile t = pair + j P over all batches (forward:
    // uniform tiles per batch; backward: the tile table above, binary-searched)
    auto seg = [&](int j) -> Seg {
        if constexpr (!BAT) {
            return seg_at(sc, pair0, j);
        } else {
            Seg r{};
            const int t = pair0 + j * n_pairs;
            if constexpr (!kBwd) {
                if (t >= g.batch * s0.T) return r;
                r.b = t / s0.T; r.tile = t - r.b * s0.T; r.prob = 0; r.nk = s0.nk;
            } else {
                if (t >= bpref[g.batch]) return r;
                int lo = 0, hi = g.batch - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (bpref[mid] <= t) lo = mid; else hi = mid - 1;
                }
                r.b = lo;
                const int l = t - bpref[lo];
                if (l < btd[lo]) { r.prob = 0; r.tile = l; r.nk = s0.nk; }
                else { r.prob = 1; r.tile = l - btd[lo]; r.nk = (__ldg(g1.k_dev + lo) + kBK - 1) / kBK; }
            }
            r.valid = true;
            return r;
        }
    };
    // size of a tile's problem (batched backward: the batch's kept-item counts)
    auto psz = [&](const Seg& sg) -> ProbSize {
        const bool p1 = kBwd && sg.prob == 1;
        ProbSize ps = p1 ? s1 : s0;
        if constexpr (BAT && kBwd) {
            if (!p1) { ps.M = __ldg(g.m_dev + sg.b); ps.m_tiles = (ps.M + BMP - 1) / BMP; ps.T = ps.m_tiles * ps.n_tiles; }
            else { ps.nk = sg.nk; ps.K = sg.nk * kBK; }
        }
        return ps;
    };
#define SEG(j) seg(j)
    gstamp(12, st0 && threadIdx.x == 0);
    pdl_wait();                                  // operands of the previous kernels
    gstamp(2, st0 && threadIdx.x == 0);

    if (warp == 0) {
        // ------------------------------------------------------------- producer (warp 0)
        int stage = 0; uint32_t phase = 0;
        for (int j = 0;; ++j) {
            const Seg sg = SEG(j);
            if (!sg.valid) break;
            gstamp(13, st0 && lane == 0 && j == 0);
            const bool p1 = kBwd && sg.prob == 1;
            const ProbSize ps = psz(sg);
            const bool a_mn = kBwd ? p1 : A_MN;
            const int m0 = (sg.tile / ps.n_tiles) * BMP + kBM * int(rank);     // this CTA's output rows
            const int nb = (sg.tile % ps.n_tiles) * BN + BNC * int(rank);      // this CTA's B rows
            const bool is_w = EPI == EPI_WGRAD || p1;
            const CUtensorMap* pA = &maps.m[MAP_A];
            const CUtensorMap* pB = &maps.m[MAP_B];
            int a_row = m0;                                                    // this CTA's A rows
            if (EPI == EPI_DGRAD || (kBwd && !p1)) {
                const int mb = sg.tile / ps.n_tiles;
                if (ps.form == 1 || (ps.form == 2 && mb < ps.mtd)) pA = &maps.m[MAP_A2];   // Q token rows, K-major
                else if (ps.form == 2) a_row -= ps.mtd * BMP;                                // sub-list rows of A_X
            }
            const CUtensorMap* pAs = kBwd ? &maps.m[MAP_AW] : &maps.m[MAP_A];  // grad_W gathered rows
            const CUtensorMap* pBs = kBwd ? &maps.m[MAP_BW] : &maps.m[MAP_B];
            for (int kb = 0; kb < sg.nk; ++kb) {
                int kr = kb;                                                   // k-block of the map
                if (is_w) {
                    if (ps.form == 1 || (ps.form == 2 && kb < ps.nkd)) { pA = &maps.m[MAP_A3]; pB = &maps.m[MAP_B2]; }
                    else { pA = pAs; pB = pBs; if (ps.form == 2) kr = kb - ps.nkd; }   // Q / X_hat, then A_W / B_W
                }
                if (lane == 0) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (leader) mbar_arrive_expect_tx(&full[stage], CG * Cfg::STAGE_BYTES);
                    uint8_t* a_dst = sA + stage * Cfg::A_BYTES;
                    uint8_t* b_dst = sB + stage * Cfg::B_BYTES;
                    if constexpr (BAT) {                   // 3-D maps: coordinate 2 = batch
                        const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
                        if (a_mn) tma_load_3d_2sm(a_dst, pA, fb, a_row, kr * kBK, sg.b);
                        else      tma_load_3d_2sm(a_dst, pA, fb, kr * kBK, a_row, sg.b);
                        if (B_MN || kBwd) {
#pragma unroll
                            for (int q = 0; q < BNC / 128; ++q)
                                tma_load_3d_2sm(b_dst + q * 128 * kBK, pB, fb, nb + 128 * q, kr * kBK, sg.b);
                        } else {
                            tma_load_3d_2sm(b_dst, pB, fb, kr * kBK, nb, sg.b);
                        }
                    } else if constexpr (CG == 2) {
                        const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
                        if (a_mn) tma_load_2d_2sm(a_dst, pA, fb, a_row, kr * kBK);
                        else      tma_load_2d_2sm(a_dst, pA, fb, kr * kBK, a_row);
                        if (B_MN || kBwd) {
#pragma unroll
                            for (int q = 0; q < BNC / 128; ++q)
                                tma_load_2d_2sm(b_dst + q * 128 * kBK, pB, fb, nb + 128 * q, kr * kBK);
                        } else {
                            tma_load_2d_2sm(b_dst, pB, fb, kr * kBK, nb);
                        }
                    } else {
                        if (a_mn) tma_load_2d(a_dst, pA, &full[stage], a_row, kr * kBK);
                        else      tma_load_2d(a_dst, pA, &full[stage], kr * kBK, a_row);
                        if (B_MN || kBwd) {
#pragma unroll
                            for (int q = 0; q < BNC / 128; ++q)
                                tma_load_2d(b_dst + q * 128 * kBK, pB, &full[stage], nb + 128 * q, kr * kBK);
                        } else {
                            tma_load_2d(b_dst, pB, &full[stage], kr * kBK, nb);
                        }
                    }
                }
                __syncwarp();
                gstamp(3, st0 && lane == 0 && j == 0 && kb == 0);
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------- MMA issuer (leader CTA)
        if (lane == 0 && leader) {
            int stage = 0; uint32_t phase = 0;
            for (int j = 0;; ++j) {
                const Seg sg = SEG(j);
                if (!sg.valid) break;
                const bool a_mn = kBwd ? sg.prob == 1 : A_MN;
                constexpr bool b_mn = B_MN || kBwd;
                const uint32_t idesc = idesc_i8(BMP, BN, a_mn, b_mn);
                // descriptor advance per K = 32 MMA: K-major +32 B; MN-major +32 rows x 128 B
                const uint64_t a_step = a_mn ? (32 * 128) >> 4 : 32 >> 4;
                constexpr uint64_t b_step = b_mn ? (32 * 128) >> 4 : 32 >> 4;
                const int as = j & 1;
                const uint32_t ap = (j >> 1) & 1;
                mbar_wait(&tempty[as], ap ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + uint32_t(as * BN);
                for (int kb = 0; kb < sg.nk; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    gstamp(4, st0 && j == 0 && kb == 0);
                    const uint32_t a_addr = smem_u32(sA + stage * Cfg::A_BYTES);
                    const uint32_t b_addr = smem_u32(sB + stage * Cfg::B_BYTES);
                    const uint64_t adesc = a_mn ? sdesc_mnmajor_sw128(a_addr, 128 * kBK) : sdesc_kmajor_sw128(a_addr);
                    const uint64_t bdesc = b_mn ? sdesc_mnmajor_sw128(b_addr, 128 * kBK) : sdesc_kmajor_sw128(b_addr);
#pragma unroll
                    for (int kk = 0; kk < kBK / 32; ++kk) {
                        const uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
                        if constexpr (CG == 2) umma_i8_2sm(d_tmem, adesc + a_step * kk, bdesc + b_step * kk, idesc, acc);
                        else umma_i8(d_tmem, adesc + a_step * kk, bdesc + b_step * kk, idesc, acc);
                    }
                    if constexpr (CG == 2) umma_commit_2sm(&empty[stage]); else umma_commit(&empty[stage]);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                if constexpr (CG == 2) umma_commit_2sm(&tfull[as]); else umma_commit(&tfull[as]);
                gstamp(5, st0);
            }
        }
    } else {
        // ------------------------------------------------------------- epilogue
        const int lg = warp & 3;                       // TMEM lane group of this warp
        const int ew = warp - 2;                       // epilogue warp index
        const int cbeg = (ew >> 2) * Epi::COLS;        // this warp's column range [cbeg, cbeg + COLS)
        const int r_in_tile = lg * 32 + lane;
        uint8_t* stg = sOut + (warp - 2) * (Cfg::OUT_BYTES > 0 ? Cfg::OUT_BYTES / kEpiWarps : 0);
        int sbuf = 0;
        float sd = 1.0f;
        if (EPI0 == EPI_DGRAD || EPI0 == EPI_WGRAD) sd = __ldg(g.s_down);
        constexpr bool kMask = EPI0 == EPI_DGRAD || EPI0 == EPI_WGRAD;
        constexpr int NW = kMask ? Epi::COLS / 32 : 1;
        const int two_n = 2 * g.n_tokens;
        // Row metadata (kept item, its neighbours, its weight exponent) and the mask
        // words of this warp's columns are loaded two / one segment(s) ahead: the mask
        // row of a grad_X item depends on the item index, and both loads would
        // otherwise sit as two dependent global-memory latencies on every tile.  Left
        // raw until the tile is processed (a consumer right after the load made every
        // tile wait for it, ncu: long-scoreboard on the epilogue warps).
        // dense: a Q token row (weight 1, never paired); skip: its token's grad_X row comes
        // from sub-list item rows (form 2), so this row is not stored; li: list index
        struct RowInfo { int item, edge, eword, li; bool dense, skip; };
        auto is_dg = [&](const Seg& sg) { return EPI0 == EPI_DGRAD && (!kBwd || sg.prob == 0); };
        auto load_ri = [&](const Seg& sg) {
            RowInfo x{two_n, two_n, 0, 0, false, false};
            if (sg.valid && is_dg(sg)) {
                const ProbSize q0 = psz(sg);
                const int rw = (sg.tile / q0.n_tiles) * BMP + kBM * int(rank) + r_in_tile;
                if (q0.form == 1 || (q0.form == 2 && rw < q0.mtd * BMP)) {
                    x.dense = true;
                    if (rw < g.n_tokens) {
                        x.item = rw;                   // token rw, weight 1, never paired
                        x.skip = q0.form == 2 && __ldg(g.tok_flag + rw) != 0;
                    }
                } else {
                    const int li = q0.form == 2 ? rw - q0.mtd * BMP : rw;        // index into the item list
                    const int cnt = q0.form == 2 ? q0.M - q0.mtd * BMP : q0.M;
                    const int64_t lo = BAT ? int64_t(sg.b) * g.bs_items : 0;   // this batch's list
                    const int32_t* items = (q0.form == 2 ? g.items2 : g.items) + lo;
                    const int8_t* wexp = (q0.form == 2 ? g.wexp2 : g.wexp) + lo;
                    x.li = li;
                    if (li < cnt) {
                        x.item = __ldg(items + li);
                        x.eword = int(__ldg(reinterpret_cast<const uint32_t*>(wexp + (li & ~3))));
                        if (lane == 31 && li + 1 < cnt) x.edge = __ldg(items + li + 1);
                        if (lane == 0 && li > 0) x.edge = __ldg(items + li - 1);
                    }
                }
            }
            return x;
        };
        auto load_mask = [&](const Seg& sg, const RowInfo& x, uint32_t (&mw)[NW]) {
#pragma unroll
            for (int q = 0; q < NW; ++q) mw[q] = 0u;
            if (!kMask || !sg.valid) return;
            const bool dg = is_dg(sg);
            const ProbSize ps = psz(sg);
            const GemmArgs& G = (kBwd && sg.prob == 1) ? g1 : g;
            const int rw = (sg.tile / ps.n_tiles) * BMP + kBM * int(rank) + r_in_tile;
            int64_t mrow = rw;
            if (dg) {
                if (x.item >= two_n) return;
                mrow = x.item >= g.n_tokens ? x.item - g.n_tokens : x.item;
                if (BAT) mrow += int64_t(sg.b) * g.n_tokens;
            } else if (rw >= ps.M) {
                return;
            } else if (BAT) {
                mrow += int64_t(sg.b) * ps.M;
            }
            const int words = G.Nn >> 5;
            const int cw0 = ((sg.tile % ps.n_tiles) * BN + cbeg) >> 5;
#pragma unroll
            for (int q = 0; q < NW; ++q)
                if (cw0 + q < words) mw[q] = __ldg(G.mask + mrow * words + cw0 + q);
        };
        Seg sg_cur = SEG(0), sg_next = SEG(1);
        RowInfo ri_cur = load_ri(sg_cur), ri_next = load_ri(sg_next);
        uint32_t mw_cur[NW];
        load_mask(sg_cur, ri_cur, mw_cur);
        double lsq_acc[2] = {0.0, 0.0};                // A.3 partials of this lane (per problem)
        for (int j = 0; sg_cur.valid; ++j) {
            const Seg sg = sg_cur;
            const Seg sg_next2 = SEG(j + 2);
            uint32_t mw_next[NW];
            load_mask(sg_next, ri_next, mw_next);      // ri_next arrived during the previous segment
            const RowInfo ri_next2 = load_ri(sg_next2);
            const bool p1 = kBwd && sg.prob == 1;
            const bool dg = is_dg(sg);
            const GemmArgs& G = p1 ? g1 : g;
            const ProbSize ps = psz(sg);
            const int as = j & 1;
            const uint32_t ap = (j >> 1) & 1;
            const int m0 = (sg.tile / ps.n_tiles) * BMP + kBM * int(rank), n0 = (sg.tile % ps.n_tiles) * BN;
            const int row = m0 + r_in_tile;
            const bool no_acc = sg.nk == 0;            // empty K range: accumulator is zero

            // per-row setup
            bool valid = row < ps.M;
            int64_t out_row = row;
            float rscale = BAT ? __ldg(G.tab + 8 * sg.b + G.tab_idx) : G.scale;
            if (BAT && kMask) sd = __ldg(g.s_down + sg.b);
            int dmode = 0;                             // 0 store, 1 store pair sum, 2 skip, 3 red.add
            int row_e = 0;                             // dgrad: log2 of the item's weight
            if (dg) {
                const int item = ri_cur.item;
                valid = item < two_n && !ri_cur.skip;
                const int h = item >= g.n_tokens ? 1 : 0;
                out_row = item - h * g.n_tokens;
                const int e = valid && !ri_cur.dense ? int(int8_t(uint32_t(ri_cur.eword) >> (8 * (ri_cur.li & 3)))) : 0;
                // neighbours: list rows li + 1 / li - 1 (lanes 31 / 0 loaded them; others shuffle);
                // rows past the list read as the sentinel; token rows have none
                int nx = __shfl_down_sync(0xFFFFFFFFu, ri_cur.item, 1);
                int pv = __shfl_up_sync(0xFFFFFFFFu, ri_cur.item, 1);
                if (lane == 31) nx = ri_cur.edge;
                if (lane == 0) pv = ri_cur.edge;
                if (ri_cur.dense) { nx = two_n; pv = two_n; }
                row_e = e;
                rscale = ldexpf(__fmul_rn(rscale, sd), e);    // s_up = 16 s_down is inside the A codes
                const int inext = valid ? nx : two_n;
                const int iprev = valid ? pv : two_n;
                const bool first = inext < two_n && (inext >= g.n_tokens ? inext - g.n_tokens : inext) == out_row;
                const bool second = iprev < two_n && (iprev >= g.n_tokens ? iprev - g.n_tokens : iprev) == out_row;
                if ((first && lane == 31) || (second && lane == 0)) dmode = 3;
                else if (second) dmode = 2;
                else if (first) dmode = 1;
            } else if (EPI0 == EPI_WGRAD || p1) {
                rscale = __fmul_rn(rscale, sd);
            }
            if (BAT && dg) out_row += int64_t(sg.b) * g.n_tokens;      // global grad_X row of the batch
            mbar_wait(&tfull[as], ap);
            tc_fence_after();
            gstamp(6, st0 && warp == 2 && lane == 0 && j == 0);
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
                if (no_acc) {
#pragma unroll
                    for (int q = 0; q < CW / 32; ++q)
#pragma unroll
                        for (int i = 0; i < 32; ++i) r[q][i] = 0;
                }
                const int col0 = n0 + c;
                if (col0 >= G.Nn) continue;           // ragged N (MN-major B): nothing to write
                if (kMask && G.lsq_part != nullptr && valid) {
                    // A.3 step-size gradient: sum_d acc[d] delta[row, d] (fp32 in column order,
                    // then fp64 across chunks; the dgrad item weight 2^e applied exactly)
                    const float* dp = G.delta + (dg ? out_row : int64_t(row)) * G.Nn + col0;
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
                    lsq_acc[p1 ? 1 : 0] += dg ? ldexp(double(cs), row_e) : double(cs);
                }

                if (dg) {
                    float v[CW];
                    masked_scaled_fwht<CW, KH>(r, mw_cur, (c - cbeg) / 32, rscale, v);
                    if constexpr (kBwd && CW == 32 && !BAT) {
                        if (ps.form == 1) {
                            // token rows of Q (form 1): the tile's rows are contiguous grad_X rows, so
                            // they go out through swizzled shared-memory staging and TMA tensor
                            // stores (full-line writes) instead of one row per lane
                            const int part = ((c - cbeg) / 32) & 1;        // bf16: two chunks per 128 B row
                            if (!g.out_bf16 || part == 0) {
                                if (lane == 0) bulk_wait_read<1>();
                                __syncwarp();
                            }
                            uint8_t* buf = stg + sbuf * kStageOutBytes;
                            if (g.out_bf16) {
                                uint32_t pk[16];
#pragma unroll
                                for (int i = 0; i < 16; ++i) {
                                    __nv_bfloat162 p2 = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
                                    pk[i] = *reinterpret_cast<uint32_t*>(&p2);
                                }
#pragma unroll
                                for (int q = 0; q < 4; ++q)
                                    *reinterpret_cast<uint4*>(stage_chunk(buf, lane, 4 * part + q)) =
                                        make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
                                if (part == 1 || c + CW >= cbeg + Epi::COLS) {
                                    fence_proxy_async_smem();
                                    __syncwarp();
                                    if (lane == 0) {
                                        tma_store_2d(&maps.m[MAP_DX], buf, col0 - 32 * part, m0 + lg * 32);
                                        bulk_commit();
                                    }
                                    sbuf ^= 1;
                                }
                            } else {
#pragma unroll
                                for (int q = 0; q < 8; ++q)
                                    *reinterpret_cast<uint4*>(stage_chunk(buf, lane, q)) =
                                        make_uint4(__float_as_uint(v[4 * q]), __float_as_uint(v[4 * q + 1]),
                                                   __float_as_uint(v[4 * q + 2]), __float_as_uint(v[4 * q + 3]));
                                fence_proxy_async_smem();
                                __syncwarp();
                                if (lane == 0) {
                                    tma_store_2d(&maps.m[MAP_DX], buf, col0, m0 + lg * 32);
                                    bulk_commit();
                                }
                                sbuf ^= 1;
                            }
                            continue;
                        }
                    }
                    if (!ri_cur.dense) {                    // token rows have no partner item (warp-uniform:
                                                            // the form-2 segment border is 256-row aligned)
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
                if constexpr (EPI == EPI_FWD) {
                    if (g.out_bf16) {
                        // 64 bf16 columns = one 128-byte staging row
                        uint32_t packed[CW / 2];
#pragma unroll
                        for (int i = 0; i < CW / 2; ++i) {
                            const float a = __fmul_rn(float(int32_t(r[(2 * i) >> 5][(2 * i) & 31])), rscale);
                            const float b = __fmul_rn(float(int32_t(r[(2 * i + 1) >> 5][(2 * i + 1) & 31])), rscale);
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
                        if (lane == 0) {
                            if constexpr (BAT) tma_store_3d(&maps.m[MAP_C], buf, col0, m0 + lg * 32, sg.b);
                            else tma_store_2d(&maps.m[MAP_C], buf, col0, m0 + lg * 32);
                            bulk_commit();
                        }
                        sbuf ^= 1;
                        continue;
                    }
                }

                uint32_t wv[CW];                      // 32-bit output words (int32 or fp32 bits)
                if constexpr (EPI == EPI_INT32) {
#pragma unroll
                    for (int i = 0; i < CW; ++i) wv[i] = r[i >> 5][i & 31];
                } else if constexpr (EPI == EPI_FWD) {
#pragma unroll
                    for (int i = 0; i < CW; ++i)
                        wv[i] = __float_as_uint(__fmul_rn(float(int32_t(r[i >> 5][i & 31])), rscale));
                } else {                              // EPI_WGRAD (or problem 1 of EPI_BWD)
                    float v[CW];
                    masked_scaled_fwht<CW, KH>(r, mw_cur, (c - cbeg) / 32, rscale, v);
                    if (G.out_mc != nullptr) {        // f4: the data-parallel all-reduce inside the GEMM
                        if (row < ps.M) {
                            float* dst = G.out_mc + int64_t(row) * G.Nn + col0;
#pragma unroll
                            for (int i = 0; i < CW; i += 4)
                                if (col0 + i < G.Nn) multimem_red_add_v4(dst + i, v[i], v[i + 1], v[i + 2], v[i + 3]);
                        }
                        continue;
                    }
#pragma unroll
                    for (int i = 0; i < CW; ++i) wv[i] = __float_as_uint(v[i]);
                }
#pragma unroll
                for (int q = 0; q < CW / 32; ++q) {
                    if (col0 + 32 * q >= G.Nn) break;
                    if (lane == 0) bulk_wait_read<1>();
                    __syncwarp();
                    uint8_t* buf = stg + sbuf * kStageOutBytes;
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj)
                        *reinterpret_cast<uint4*>(stage_chunk(buf, lane, jj)) =
                            make_uint4(wv[32 * q + 4 * jj], wv[32 * q + 4 * jj + 1], wv[32 * q + 4 * jj + 2], wv[32 * q + 4 * jj + 3]);
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        if constexpr (BAT) tma_store_3d(&maps.m[MAP_C], buf, col0 + 32 * q, m0 + lg * 32, sg.b);
                        else tma_store_2d(&maps.m[MAP_C], buf, col0 + 32 * q, m0 + lg * 32);
                        bulk_commit();
                    }
                    sbuf ^= 1;
                }
            }
            ri_cur = ri_next; ri_next = ri_next2;
#pragma unroll
            for (int q = 0; q < NW; ++q) mw_cur[q] = mw_next[q];
            sg_cur = sg_next; sg_next = sg_next2;
        }
#undef SEG
        if (kMask && g.lsq_part != nullptr) {          // fixed-order warp sum -> this warp's slot
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) lsq_acc[0] += __shfl_xor_sync(0xFFFFFFFFu, lsq_acc[0], o);
            if (lane == 0) g.lsq_part[int(blockIdx.x) * kMaxEpiWarps + ew] = lsq_acc[0];
        }
        if (kBwd && g1.lsq_part != nullptr) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) lsq_acc[1] += __shfl_xor_sync(0xFFFFFFFFu, lsq_acc[1], o);
            if (lane == 0) g1.lsq_part[int(blockIdx.x) * kMaxEpiWarps + ew] = lsq_acc[1];
        }
        bulk_wait_read<0>();                           // every lane: its staging buffers were read (the
                                                       // global writes complete with the grid)
        gstamp(7, st0 && warp == 2 && lane == 0);
        if ((EPI0 == EPI_WGRAD && g.out_mc != nullptr) || (kBwd && g1.out_mc != nullptr))
            __threadfence_system();                    // multimem reductions performed before the kernel ends
        __syncwarp();
    }

    tc_fence_before();
    if (CG == 2) cluster_sync_all(); else __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc<CG>(tmem_base, Cfg::TMEM_COLS);
    gstamp(8, st0 && threadIdx.x == 0);
    gstamp(10, threadIdx.x == 0);
}

int gemm_block_n(int Nn, bool b_mn) {
    if (Nn % 256 == 0 || b_mn) return 256;      // MN-major B halves are whole 128-byte atoms
    if (Nn % 128 == 0) return 128;
    return 64;
}

constexpr int kCG = kGemmCG;                    // CTA pairs (cta_group::2) for every GEMM

template <int BN, int EPI, int KH, bool A_MN, bool B_MN, bool BAT>
static cudaError_t launch_one(const GemmMaps& m, const GemmArgs& g, const GemmArgs& g1, int grid, cudaStream_t s) {
    auto kern = gemm_i8_kernel<BN, EPI, KH, A_MN, B_MN, kCG, BAT>;
    constexpr int EPIC = EPI == EPI_BWD ? EPI_WGRAD : EPI;
    using Epi = EpiShape<BN, EPIC, kh_ch(KH)>;
    constexpr int smem = GemmCfg<BN, kCG, Epi::WARPS, EPIC, Epi::COLS, (BAT && EPI == EPI_BWD) ? kBatSmem : 0>::SMEM;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    GemmMapSet ms;
    const void* src[9] = {m.a, m.b, m.c, m.a2, m.a3, m.b2, m.aw, m.bw, m.dx};
    for (int i = 0; i < 9; ++i) ms.m[i] = *reinterpret_cast<const CUtensorMap*>(src[i] ? src[i] : m.a);
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
    return cudaLaunchKernelEx(&cfg, kern, ms, g, g1);
}

template <int EPI, int KH, bool A_MN, bool B_MN, bool BAT>
static cudaError_t dispatch_bn(int bn, const GemmMaps& m, const GemmArgs& g, const GemmArgs& g1, int grid,
                               cudaStream_t s) {
    if (bn == 256) return launch_one<256, EPI, KH, A_MN, B_MN, BAT>(m, g, g1, grid, s);
    if constexpr (!B_MN && EPI != EPI_BWD) {
        if (bn == 128) return launch_one<128, EPI, KH, A_MN, B_MN, BAT>(m, g, g1, grid, s);
        if constexpr (kh_ch(KH) <= 64) return launch_one<64, EPI, KH, A_MN, B_MN, BAT>(m, g, g1, grid, s);
    }
    return cudaErrorInvalidValue;
}

template <int EPI, bool A_MN, bool B_MN, bool BAT = false>
static cudaError_t dispatch_ch(int bn, const GemmMaps& m, const GemmArgs& g, const GemmArgs& g1, int grid,
                               cudaStream_t s) {
    if constexpr (EPI == EPI_DGRAD || EPI == EPI_WGRAD || EPI == EPI_BWD) {
        switch (g.k_had) {
            case 0: return dispatch_bn<EPI, 0, A_MN, B_MN, BAT>(bn, m, g, g1, grid, s);
            case 1: return dispatch_bn<EPI, 1, A_MN, B_MN, BAT>(bn, m, g, g1, grid, s);
            case 2: return dispatch_bn<EPI, 2, A_MN, B_MN, BAT>(bn, m, g, g1, grid, s);
            case 3: return dispatch_bn<EPI, 3, A_MN, B_MN, BAT>(bn, m, g, g1, grid, s);
            case 4: return dispatch_bn<EPI, 4, A_MN, B_MN, BAT>(bn, m, g, g1, grid, s);
            case 5: return dispatch_bn<EPI, 5, A_MN, B_MN, BAT>(bn, m, g, g1, grid, s);
            case 6: return dispatch_bn<EPI, 6, A_MN, B_MN, BAT>(bn, m, g, g1, grid, s);
            case 7: return dispatch_bn<EPI, 7, A_MN, B_MN, BAT>(bn, m, g, g1, grid, s);
            default: return cudaErrorInvalidValue;
        }
    } else {
        return dispatch_bn<EPI, 0, A_MN, B_MN, BAT>(bn, m, g, g1, grid, s);
    }
}

cudaError_t launch_gemm(const GemmMaps& m, const GemmArgs& g, int num_sms, cudaStream_t s, const GemmArgs* g1) {
    const int bn = g.epi == EPI_BWD ? 256 : gemm_block_n(g.Nn, g.b_mn);
    const int64_t pairs = num_sms / kCG;
    // persistent grid: at most one pair per tile (every pair when two problems share
    // the launch: their tile counts may come from device memory)
    int64_t grid_pairs = pairs;
    const int64_t nb = g.batch > 0 ? g.batch : 1;
    if (g.epi != EPI_BWD) {
        const int64_t tiles = nb * ((g.M + kBM * kCG - 1) / (kBM * kCG)) * ((g.Nn + bn - 1) / bn);   // g.M = bound
        grid_pairs = tiles < pairs ? tiles : pairs;
    } else if (g.batch > 0 && g1) {             // batched backward: capacity tiles (g.M = list capacity)
        const int64_t tiles = nb * (((g.M + kBM * kCG - 1) / (kBM * kCG)) * ((g.Nn + bn - 1) / bn) +
                                    ((g1->M + kBM * kCG - 1) / (kBM * kCG)) * ((g1->Nn + bn - 1) / bn));
        grid_pairs = tiles < pairs ? tiles : pairs;
    }
    if (grid_pairs < 1) grid_pairs = 1;
    const int grid = kCG * int(grid_pairs);
    const GemmArgs none{};
    const GemmArgs& gg1 = g1 ? *g1 : none;
    if (g.batch > 0) {
        if (g.epi == EPI_FWD) return dispatch_ch<EPI_FWD, false, false, true>(bn, m, g, gg1, grid, s);
        if (g.epi == EPI_BWD && g.batch <= kMaxGemmBatch) return dispatch_ch<EPI_BWD, false, true, true>(bn, m, g, gg1, grid, s);
        return cudaErrorInvalidValue;
    }
    switch (g.epi) {
        case EPI_FWD: return dispatch_ch<EPI_FWD, false, false>(bn, m, g, gg1, grid, s);
        case EPI_DGRAD: return dispatch_ch<EPI_DGRAD, false, true>(bn, m, g, gg1, grid, s);
        case EPI_WGRAD: return dispatch_ch<EPI_WGRAD, true, true>(bn, m, g, gg1, grid, s);
        case EPI_BWD: return dispatch_ch<EPI_BWD, false, true>(bn, m, g, gg1, grid, s);
        case EPI_INT32:
            if (!g.a_mn && !g.b_mn) return dispatch_ch<EPI_INT32, false, false>(bn, m, g, gg1, grid, s);
            if (!g.a_mn && g.b_mn) return dispatch_ch<EPI_INT32, false, true>(bn, m, g, gg1, grid, s);
            if (g.a_mn && g.b_mn) return dispatch_ch<EPI_INT32, true, true>(bn, m, g, gg1, grid, s);
            return dispatch_ch<EPI_INT32, true, false>(bn, m, g, gg1, grid, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace i4
