// C ABI of libint4linear (declared in include/int4linear.h): argument
// validation, TMA tensor-map construction and the stream-ordered launch
// sequence of HQ-MM and LSS-MM.
// No host<->device synchronisation and no device allocation happen here.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdarg>
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/int4linear.h"
#include "kernels.h"

#include <atomic>
#include <cstdlib>

namespace i4 {
// process-wide PDL switch: on by default; int4_set_pdl() changes it
static std::atomic<int> g_pdl{1};
bool pdl_enabled() { return g_pdl.load(std::memory_order_relaxed) != 0; }
}  // namespace i4

namespace {

thread_local std::string g_last_error;

i4_status fail(i4_status st, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
i4_status fail(i4_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

i4_status cuda_fail(cudaError_t e, const char* where) {
    return fail(I4_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define I4_CHECK_CUDA(expr, where)                      \
    do {                                                \
        cudaError_t e_ = (expr);                        \
        if (e_ != cudaSuccess) return cuda_fail(e_, where); \
    } while (0)

// Launch tracing (int4_trace_begin / int4_trace_end): caller-owned events are
// recorded on the launch stream around a window of the library's launches.
constexpr int kMaxTrace = 64;
struct TraceState {
    bool active = false;
    cudaEvent_t ev[kMaxTrace + 1];
    int cap = 0;                 // events available
    int first = 0;               // index of the first launch inside the window
    int n = 0;                   // launches seen since int4_trace_begin
    const char* names[kMaxTrace];
};
thread_local TraceState g_trace;

void trace_record(cudaEvent_t e, cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &st);
    if (st == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);  // graph node
    else cudaEventRecord(e, s);
}
void trace_pre(cudaStream_t s) {
    if (g_trace.active && g_trace.n == g_trace.first && g_trace.cap > 0) trace_record(g_trace.ev[0], s);
}
void trace_post(const char* name, cudaStream_t s) {
    if (!g_trace.active) return;
    const int w = g_trace.n - g_trace.first;                 // position inside the window
    if (w >= 0 && w + 1 < g_trace.cap) trace_record(g_trace.ev[w + 1], s);
    if (g_trace.n < kMaxTrace) g_trace.names[g_trace.n] = name;
    ++g_trace.n;
}

// Every kernel launch of the library goes through this macro.
#define I4_LAUNCH(expr, name, stream)                       \
    do {                                                    \
        trace_pre(stream);                                  \
        cudaError_t e_ = (expr);                            \
        if (e_ != cudaSuccess) return cuda_fail(e_, name);  \
        trace_post(name, stream);                           \
    } while (0)

struct DeviceInfo {
    bool ok = false;
    int sms = 0;
    std::string why;
};

DeviceInfo query_device() {
    DeviceInfo d;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { d.why = "no CUDA device"; return d; }
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) { d.why = "cudaGetDeviceProperties failed"; return d; }
    if (!(p.major == 10 && p.minor == 0)) {
        char b[128];
        snprintf(b, sizeof b, "device is sm_%d%d; this library is built for sm_100a (tcgen05 kind::i8)", p.major, p.minor);
        d.why = b;
        return d;
    }
    d.ok = true;
    d.sms = p.multiProcessorCount;
    return d;
}

// cached per device ordinal (a process may drive several GPUs)
const DeviceInfo& device_info() {
    static DeviceInfo info[i4::kMaxDevices];
    static std::once_flag once[i4::kMaxDevices];
    static DeviceInfo none;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= i4::kMaxDevices) {
        none.why = "no CUDA device (or device ordinal >= 64)";
        return none;
    }
    std::call_once(once[dev], [dev] { info[dev] = query_device(); });
    return info[dev];
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// 2-D int8 tensor [rows, inner] with row pitch `pitch` bytes; box = 128 B x box_rows,
// 128-byte swizzle (matches the UMMA SWIZZLE_128B descriptors, K- or MN-major).
bool make_tmap_i8(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t rows, uint64_t pitch, uint32_t box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {inner, rows};
    cuuint64_t strides[1] = {pitch};
    cuuint32_t box[2] = {128, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// Output tensor [rows, cols] of 4-byte (int32 / fp32) or 2-byte (bf16) elements;
// box = 128 bytes x 32 rows (one epilogue warp's staging tile), 128-byte swizzle.
bool make_tmap_out(CUtensorMap* m, void* ptr, bool bf16, bool is_int, uint64_t cols, uint64_t rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    const uint32_t esz = bf16 ? 2 : 4;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * esz};
    cuuint32_t box[2] = {128 / esz, 32};
    cuuint32_t estr[2] = {1, 1};
    const CUtensorMapDataType dt = bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                        : (is_int ? CU_TENSOR_MAP_DATA_TYPE_INT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
    CUresult r = fn(m, dt, 2, ptr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

i4_status check_device() {
    const DeviceInfo& d = device_info();
    if (!d.ok) return fail(I4_ERR_UNSUPPORTED, "%s", d.why.c_str());
    return I4_OK;
}

i4_status check_step(float s, const char* name) {
    if (!(s > 0.0f) || !std::isfinite(s)) return fail(I4_ERR_ARG, "%s must be positive and finite (got %g)", name, double(s));
    return I4_OK;
}

i4_status check_k(int32_t k, int64_t cols) {
    if (k < 0 || k > 7) return fail(I4_ERR_SHAPE, "k = %d outside [0, 7]", k);
    if (cols % (int64_t(1) << k) != 0) return fail(I4_ERR_SHAPE, "cols = %lld not a multiple of 2^k (PAPER.md:132)", (long long)cols);
    return I4_OK;
}

float step_recip(int32_t k, float s) { return float(std::pow(2.0, -double(k) / 2.0) / double(s)); }
float inv_sqrt_block(int32_t k) { return float(std::pow(2.0, -double(k) / 2.0)); }

int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

constexpr int64_t kMaxBwdTokens = 65536;

#define I4_RETURN_IF(st) do { i4_status s_ = (st); if (s_ != I4_OK) return s_; } while (0)

// One operand of a GEMM: `rows` x `inner` int8 with row pitch `pitch` bytes.
// K-major: rows = M (or Nn), inner = K.  MN-major: rows = K, inner = M (or Nn).
struct Operand { const int8_t* p; int64_t rows, inner, pitch; };

// A_alt (optional): a second A the kernel may read instead, chosen on the device
// (the grad_X GEMM reads the code plane Q when its mask is deterministic, Z-32);
// A_dense / B_dense: the grad_W GEMM's operands Q and X_hat for that case
i4_status gemm(const Operand& A, const Operand& B, const i4::GemmArgs& args, cudaStream_t s, int sms = 0,
               const Operand* A_alt = nullptr, const Operand* A_dense = nullptr, const Operand* B_dense = nullptr) {
    CUtensorMap ta, tb, tc, ta2, ta3, tb2;
    const int bn = i4::gemm_block_n(args.Nn, args.b_mn != 0);
    bool ok = make_tmap_i8(&ta, A.p, uint64_t(A.inner), uint64_t(A.rows), uint64_t(A.pitch), 128u) &&
              make_tmap_i8(&tb, B.p, uint64_t(B.inner), uint64_t(B.rows), uint64_t(B.pitch),
                           args.b_mn ? 128u : uint32_t(bn / i4::kGemmCG));
    if (A_alt) ok = ok && make_tmap_i8(&ta2, A_alt->p, uint64_t(A_alt->inner), uint64_t(A_alt->rows),
                                       uint64_t(A_alt->pitch), 128u);
    else ta2 = ta;
    // dense-mode operands (device-selected): A_dense MN-major like A, B_dense MN-major like B
    if (A_dense) ok = ok && make_tmap_i8(&ta3, A_dense->p, uint64_t(A_dense->inner), uint64_t(A_dense->rows),
                                         uint64_t(A_dense->pitch), 128u);
    else ta3 = ta;
    if (B_dense) ok = ok && make_tmap_i8(&tb2, B_dense->p, uint64_t(B_dense->inner), uint64_t(B_dense->rows),
                                         uint64_t(B_dense->pitch), 128u);
    else tb2 = tb;
    if (args.epi == i4::EPI_DGRAD) tc = ta;                 // grad_X is written with red.add, no map
    else ok = ok && make_tmap_out(&tc, args.out, args.out_bf16 != 0, args.epi == i4::EPI_INT32,
                                  uint64_t(args.Nn), uint64_t(args.M));
    if (!ok) return fail(I4_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    static const char* kNames[] = {"gemm_i8_int32", "gemm_i8_fwd", "gemm_i8_dgrad", "gemm_i8_wgrad"};
    const i4::GemmMaps maps{&ta, &tb, &tc, &ta2, &ta3, &tb2, nullptr, nullptr, nullptr};
    I4_LAUNCH(i4::launch_gemm(maps, args, sms > 0 ? sms : device_info().sms, s), kNames[args.epi], s);
    return I4_OK;
}

// The grad_X and grad_W GEMMs of one backward as ONE persistent launch
// (EPI_BWD): problem 0 = grad_X (A = compacted items A_X or the code plane Q, K-major;
// B = W_hat read MN-major), problem 1 = grad_W (A = A_W or Q, B = B_W or X_hat, both
// MN-major; output dW by TMA store).  Which operands each problem reads (compacted or
// dense, reading Z-32) is decided on the device from the sampler's flags.
i4_status gemm_bwd(const Operand& a_x, const Operand& q_rows, const Operand& w_mn, const Operand& a_w,
                   const Operand& b_w, const Operand& q_mn, const Operand& xq_mn, const i4::GemmArgs& gx,
                   const i4::GemmArgs& gw, cudaStream_t s) {
    CUtensorMap ta, tb, tc, ta2, ta3, tb2, taw, tbw, tdx;
    bool ok = make_tmap_i8(&ta, a_x.p, uint64_t(a_x.inner), uint64_t(a_x.rows), uint64_t(a_x.pitch), 128u) &&
              make_tmap_i8(&ta2, q_rows.p, uint64_t(q_rows.inner), uint64_t(q_rows.rows), uint64_t(q_rows.pitch), 128u) &&
              make_tmap_i8(&tb, w_mn.p, uint64_t(w_mn.inner), uint64_t(w_mn.rows), uint64_t(w_mn.pitch), 128u) &&
              make_tmap_i8(&taw, a_w.p, uint64_t(a_w.inner), uint64_t(a_w.rows), uint64_t(a_w.pitch), 128u) &&
              make_tmap_i8(&tbw, b_w.p, uint64_t(b_w.inner), uint64_t(b_w.rows), uint64_t(b_w.pitch), 128u) &&
              make_tmap_i8(&ta3, q_mn.p, uint64_t(q_mn.inner), uint64_t(q_mn.rows), uint64_t(q_mn.pitch), 128u) &&
              make_tmap_i8(&tb2, xq_mn.p, uint64_t(xq_mn.inner), uint64_t(xq_mn.rows), uint64_t(xq_mn.pitch), 128u) &&
              make_tmap_out(&tc, gw.out, false, false, uint64_t(gw.Nn), uint64_t(gw.M)) &&
              make_tmap_out(&tdx, gx.out, gx.out_bf16 != 0, false, uint64_t(gx.Nn), uint64_t(gx.n_tokens));
    if (!ok) return fail(I4_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    const i4::GemmMaps maps{&ta, &tb, &tc, &ta2, &ta3, &tb2, &taw, &tbw, &tdx};
    I4_LAUNCH(i4::launch_gemm(maps, gx, device_info().sms, s, &gw), "gemm_i8_bwd", s);
    return I4_OK;
}

// 3-D variants for the batched BMM launches: [batches, rows, inner] with batch pitch
// `bpitch` bytes; coordinate 2 = batch, so a box never crosses into another batch.
bool make_tmap_i8_3d(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t rows, uint64_t pitch,
                     uint64_t batches, uint64_t bpitch, uint32_t box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {inner, rows, batches};
    cuuint64_t strides[2] = {pitch, bpitch};
    cuuint32_t box[3] = {128, box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool make_tmap_out_3d(CUtensorMap* m, void* ptr, bool bf16, uint64_t cols, uint64_t rows, uint64_t batches) {
    auto fn = encode_fn();
    if (!fn) return false;
    const uint32_t esz = bf16 ? 2 : 4;
    cuuint64_t dims[3] = {cols, rows, batches};
    cuuint64_t strides[2] = {cols * esz, cols * rows * esz};
    cuuint32_t box[3] = {128 / esz, 32, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    const CUtensorMapDataType dt = bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    CUresult r = fn(m, dt, 3, ptr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace

extern "C" {

const char* int4_last_error(void) { return g_last_error.c_str(); }

// timing-experiment hook (tools/gs_stamps.py), not part of the documented ABI
__attribute__((visibility("default"))) int32_t int4_debug_grad_split_stamps(unsigned long long* host, int32_t n) {
    return i4::grad_split_stamps(host, n);
}
__attribute__((visibility("default"))) int32_t int4_debug_sampler_stamps(unsigned long long* host, int32_t enable) {
    return i4::sampler_stamps(host, enable);
}

__attribute__((visibility("default"))) int32_t int4_debug_gemm_stamps(unsigned long long* host) {
    return i4::gemm_stamps(host);
}

int32_t int4_sampler_cluster_ctas(int64_t N) { return i4::sampler_cluster_ctas(N); }

int32_t int4_set_pdl(int32_t enable) {
    const int32_t prev = i4::pdl_enabled() ? 1 : 0;
    i4::g_pdl.store(enable ? 1 : 0, std::memory_order_relaxed);
    return prev;
}

i4_status int4_trace_begin(void* const* events, int32_t capacity, int32_t first_launch) {
    if (!events || capacity < 2 || capacity > kMaxTrace + 1 || first_launch < 0)
        return fail(I4_ERR_ARG, "int4_trace_begin: 2 <= capacity <= %d, first_launch >= 0", kMaxTrace + 1);
    for (int i = 0; i < capacity; ++i) g_trace.ev[i] = static_cast<cudaEvent_t>(events[i]);
    g_trace.cap = capacity;
    g_trace.first = first_launch;
    g_trace.n = 0;
    g_trace.active = true;
    return I4_OK;
}

int32_t int4_trace_end(const char** names, int32_t capacity) {
    const int n = g_trace.n < kMaxTrace ? g_trace.n : kMaxTrace;
    for (int i = 0; i < n && i < capacity; ++i) names[i] = g_trace.names[i];
    g_trace.active = false;
    g_trace.cap = 0;
    return n;
}

i4_status hadamard_quant(const void* x_bf16, int64_t rows, int64_t cols, int32_t k, float step, int8_t* codes,
                         uint32_t* clamp_bits, int32_t* row_sqnorm, void* stream) {
    I4_RETURN_IF(check_device());
    if (!x_bf16 || !codes) return fail(I4_ERR_ARG, "hadamard_quant: NULL input/output");
    if (rows < 0 || cols <= 0 || cols % 32 != 0 || cols > 8192)
        return fail(I4_ERR_SHAPE, "hadamard_quant: cols = %lld must be a multiple of 32 in [32, 8192]", (long long)cols);
    I4_RETURN_IF(check_k(k, cols));
    I4_RETURN_IF(check_step(step, "step"));
    if (!aligned16(x_bf16) || !aligned16(codes)) return fail(I4_ERR_ALIGN, "hadamard_quant: pointers must be 16-byte aligned");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    I4_LAUNCH(i4::launch_hadamard_quant(static_cast<const uint16_t*>(x_bf16), rows, cols, k, step_recip(k, step),
                                        codes, clamp_bits, row_sqnorm, nullptr, s),
              "hadamard_quant", s);
    return I4_OK;
}

i4_status int4_linear_fwd(const void* X, const void* W, int64_t N, int64_t D, int64_t C, int32_t k, float s_x,
                          float s_w, void* Y, i4_out_dtype y_dtype, i4_fwd_cache* cache, void* stream) {
    I4_RETURN_IF(check_device());
    if (!X || !W || !Y || !cache || !cache->xq || !cache->wq || !cache->x_mask || !cache->w_mask ||
        !cache->x_sqnorm)
        return fail(I4_ERR_ARG, "int4_linear_fwd: NULL pointer");
    if (N <= 0 || D <= 0 || C <= 0 || D % 64 || C % 64 || D > 8192)
        return fail(I4_ERR_SHAPE, "int4_linear_fwd: need N > 0 and D, C positive multiples of 64 (N=%lld D=%lld C=%lld)",
                    (long long)N, (long long)D, (long long)C);
    if (N > (int64_t(1) << 31) / 2) return fail(I4_ERR_SHAPE, "int4_linear_fwd: N too large");
    I4_RETURN_IF(check_k(k, D));
    I4_RETURN_IF(check_step(s_x, "s_x"));
    I4_RETURN_IF(check_step(s_w, "s_w"));
    if (y_dtype != I4_OUT_F32 && y_dtype != I4_OUT_BF16) return fail(I4_ERR_ARG, "bad y_dtype");
    if (!aligned16(X) || !aligned16(W) || !aligned16(Y) || !aligned16(cache->x_delta) || !aligned16(cache->w_delta))
        return fail(I4_ERR_ALIGN, "int4_linear_fwd: unaligned pointer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);

    {
        // F1-F3: X and (unless cached) W quantized by one launch
        i4::HqArgs h{};
        h.x0 = static_cast<const uint16_t*>(X); h.rows0 = N; h.r0 = step_recip(k, s_x);
        h.codes0 = cache->xq; h.bits0 = cache->x_mask; h.sqnorm0 = cache->x_sqnorm;
        h.delta0 = cache->x_delta;              // A.3 deltas only when the caller asks for them
        if (!cache->w_valid) {
            h.x1 = static_cast<const uint16_t*>(W); h.rows1 = C; h.r1 = step_recip(k, s_w);
            h.codes1 = cache->wq; h.bits1 = cache->w_mask; h.sqnorm1 = nullptr;
            h.delta1 = cache->w_delta;
        }
        h.cols = D; h.k = k;
        h.status = cache->dev_status;
        I4_LAUNCH(i4::launch_hadamard_quant2(h, s), "hadamard_quant", s);
    }
    i4::GemmArgs g{};
    g.M = int32_t(N); g.Nn = int32_t(C); g.K = int32_t(D);
    g.epi = i4::EPI_FWD;
    g.out = Y;
    g.out_bf16 = y_dtype == I4_OUT_BF16;
    g.scale = s_x * s_w;                      // fl32(s_x s_w), reading Z-22

    I4_RETURN_IF(gemm(Operand{cache->xq, N, D, D}, Operand{cache->wq, C, D, D}, g, s));
    cache->N = N; cache->D = D; cache->C = C; cache->k = k; cache->s_x = s_x; cache->s_w = s_w;
    return I4_OK;
}

// Operand form 2 buffers of the backward workspace (reading Z-33), handed to the sampler.
struct Form2 { int32_t* corr_items; int8_t* corr_wexp; int32_t* counts2; int32_t* sub_items; int8_t* sub_wexp;
               uint8_t* tok_flag; };

static i4_status bitsplit_lss_impl(const void* dY, int64_t N, int64_t C, const int32_t* x_sqnorm, uint64_t seed,
                            uint32_t call_id, int64_t token_offset, i4_lss_mode mode, const i4_lss_plan* plan,
                            cudaStream_t s, uint32_t* zero_words, int32_t n_zero_words,
                            int32_t* det_flags = nullptr, const Form2* f2 = nullptr) {
    I4_RETURN_IF(check_device());
    if (!dY || !plan || !plan->q8 || !plan->a_sq || !plan->amax_bits || !plan->s_down || !plan->scratch || !plan->items_w ||
        !plan->wexp_w || !plan->count_w || !plan->items_x || !plan->wexp_x || !plan->count_x || !plan->x_touched)
        return fail(I4_ERR_ARG, "bitsplit_lss: NULL pointer");
    if (mode != I4_LSS_BERNOULLI && mode != I4_LSS_KEEP_POSITIVE && mode != I4_LSS_NONE)
        return fail(I4_ERR_ARG, "bitsplit_lss: bad mode");
    if (mode != I4_LSS_NONE && !x_sqnorm) return fail(I4_ERR_ARG, "bitsplit_lss: x_sqnorm required");
    if (N <= 0 || C <= 0 || C % 64) return fail(I4_ERR_SHAPE, "bitsplit_lss: need N > 0, C a multiple of 64");
    if (N > kMaxBwdTokens || N > i4::sampler_max_tokens())
        return fail(I4_ERR_SHAPE, "bitsplit_lss: N = %lld exceeds %lld tokens per call (reading Z-21)", (long long)N,
                    (long long)kMaxBwdTokens);
    if (token_offset < 0) return fail(I4_ERR_ARG, "bitsplit_lss: token_offset < 0");
    if (!aligned16(dY) || !aligned16(plan->q8)) return fail(I4_ERR_ALIGN, "bitsplit_lss: unaligned pointer");
    I4_LAUNCH(i4::launch_grad_split(static_cast<const uint16_t*>(dY), N, C, plan->scratch, seed, call_id, token_offset,
                                    plan->q8, plan->a_sq, plan->s_down, plan->amax_bits, plan->dev_status, s),
              "grad_split", s);
    i4::SamplerArgs a{};
    a.a_sq = plan->a_sq;
    a.x_sqnorm = x_sqnorm;
    a.N = int32_t(N);
    a.mode = int32_t(mode);
    a.seed_lo = uint32_t(seed);
    a.seed_hi = uint32_t(seed >> 32);
    a.call_id = call_id;
    a.token_offset = token_offset;
    a.items[0] = plan->items_w; a.wexp[0] = plan->wexp_w; a.count[0] = plan->count_w;
    a.items[1] = plan->items_x; a.wexp[1] = plan->wexp_x; a.count[1] = plan->count_x;
    a.zero_words = zero_words; a.n_zero_words = n_zero_words;
    a.det_flags = det_flags;
    a.x_touched = plan->x_touched;
    if (f2 != nullptr) {                         // int4_linear_bwd: operand form 2 available
        a.corr_items = f2->corr_items; a.corr_wexp = f2->corr_wexp; a.corr_count = f2->counts2;
        a.sub_items = f2->sub_items; a.sub_wexp = f2->sub_wexp; a.sub_count = f2->counts2 + 1;
        a.tok_flag = f2->tok_flag;
    }
    I4_LAUNCH(i4::launch_lss_sampler(a, s), "lss_sampler", s);
    return I4_OK;
}

i4_status bitsplit_lss(const void* dY, int64_t N, int64_t C, const int32_t* x_sqnorm, uint64_t seed, uint32_t call_id,
                       int64_t token_offset, i4_lss_mode mode, const i4_lss_plan* plan, void* stream) {
    return bitsplit_lss_impl(dY, N, C, x_sqnorm, seed, call_id, token_offset, mode, plan,
                             static_cast<cudaStream_t>(stream), nullptr, 0);
}

}  // extern "C"

namespace {

// Backward workspace layout (bytes, each region 256-aligned):
//   A_X [2N+128, C] | A_W [kcap, C] | B_W [kcap, D] | A.3 partials (grad_X, grad_W) | det flags
struct BwdWs {
    int8_t* a_x; int8_t* a_w; int8_t* b_w;
    double* lsq_x; double* lsq_w;        // A.3 fp64 partials (zeroed by the sampler launch)
    int32_t* det;                        // [2] operand forms of the two masks (written by the sampler)
    // operand form 2 (dense + correction, reading Z-33): grad_W correction rows, grad_X
    // sub-list of the tokens with sampled items, their counts and per-token flags
    int32_t* corr_items; int8_t* corr_wexp; int32_t* sub_items; int8_t* sub_wexp;
    int32_t* counts2;                    // [0] correction rows, [1] sub-list items
    uint8_t* tok_flag;                   // [N]
    size_t total;
};

BwdWs carve_bwd_ws(void* ws, int64_t N, int64_t D, int64_t C) {
    const int64_t kcap = round_up(2 * N, 128);
    BwdWs w{};
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += size_t(round_up(int64_t(bytes), 256)); return o; };
    const size_t o_ax = take(size_t((2 * N + 128) * C));
    const size_t o_aw = take(size_t(C * kcap));
    const size_t o_bw = take(size_t(D * kcap));
    const size_t o_f = take(2 * i4::kLsqPartials * sizeof(double));   // the sampler zeroes it
    const size_t o_det = take(2 * sizeof(int32_t));
    const size_t o_ci = take(size_t(2 * N + 128) * sizeof(int32_t));
    const size_t o_ce = take(size_t(2 * N + 128));
    const size_t o_si = take(size_t(2 * N + 128) * sizeof(int32_t));
    const size_t o_se = take(size_t(2 * N + 128));
    const size_t o_c2 = take(2 * sizeof(int32_t));
    const size_t o_tf = take(size_t(N));
    w.total = off;
    if (ws) {
        uint8_t* b = static_cast<uint8_t*>(ws);
        w.a_x = reinterpret_cast<int8_t*>(b + o_ax);
        w.a_w = reinterpret_cast<int8_t*>(b + o_aw);
        w.b_w = reinterpret_cast<int8_t*>(b + o_bw);
        w.lsq_x = reinterpret_cast<double*>(b + o_f);
        w.lsq_w = w.lsq_x + i4::kLsqPartials;
        w.det = reinterpret_cast<int32_t*>(b + o_det);
        w.corr_items = reinterpret_cast<int32_t*>(b + o_ci);
        w.corr_wexp = reinterpret_cast<int8_t*>(b + o_ce);
        w.sub_items = reinterpret_cast<int32_t*>(b + o_si);
        w.sub_wexp = reinterpret_cast<int8_t*>(b + o_se);
        w.counts2 = reinterpret_cast<int32_t*>(b + o_c2);
        w.tok_flag = b + o_tf;
    }
    return w;
}

}  // namespace

extern "C" {

size_t int4_bwd_workspace_size(int64_t N, int64_t D, int64_t C) { return carve_bwd_ws(nullptr, N, D, C).total; }

// introspection (bench / tests): byte offset in the backward workspace of the two
// int32 flags the sampler writes -- [0] grad_W mask deterministic, [1] grad_X mask
// deterministic (reading Z-32: the GEMMs then read Q / X_hat and compact moves nothing)
size_t int4_bwd_ws_det_offset(int64_t N, int64_t D, int64_t C) {
    uint8_t* const base = reinterpret_cast<uint8_t*>(uintptr_t(1) << 20);
    const BwdWs w = carve_bwd_ws(base, N, D, C);
    return size_t(reinterpret_cast<uint8_t*>(w.det) - base);
}

size_t int4_bwd_ws_form2_offset(int64_t N, int64_t D, int64_t C) {
    uint8_t* const base = reinterpret_cast<uint8_t*>(uintptr_t(1) << 20);
    const BwdWs w = carve_bwd_ws(base, N, D, C);
    return size_t(reinterpret_cast<uint8_t*>(w.counts2) - base);
}

static i4_status linear_bwd_impl(const void* dY, const i4_fwd_cache* cache, uint64_t seed, uint32_t call_id,
                                 int64_t token_offset, i4_lss_mode mode, const i4_lss_plan* plan, void* dX,
                                 i4_out_dtype dx_dtype, float* dW, void* ws, size_t ws_bytes, void* stream);

i4_status int4_linear_bwd(const void* dY, const i4_fwd_cache* cache, uint64_t seed, uint32_t call_id,
                          int64_t token_offset, i4_lss_mode mode, const i4_lss_plan* plan, void* dX,
                          i4_out_dtype dx_dtype, float* dW, void* ws, size_t ws_bytes, void* stream) {
    return linear_bwd_impl(dY, cache, seed, call_id, token_offset, mode, plan, dX, dx_dtype, dW, ws, ws_bytes, stream);
}

}  // extern "C"

static i4_status linear_bwd_impl(const void* dY, const i4_fwd_cache* cache, uint64_t seed, uint32_t call_id,
                                 int64_t token_offset, i4_lss_mode mode, const i4_lss_plan* plan, void* dX,
                                 i4_out_dtype dx_dtype, float* dW, void* ws, size_t ws_bytes, void* stream) {
    I4_RETURN_IF(check_device());
    if (!cache || !dX || !dW || !ws) return fail(I4_ERR_ARG, "int4_linear_bwd: NULL pointer");
    if (dx_dtype != I4_OUT_F32 && dx_dtype != I4_OUT_BF16) return fail(I4_ERR_ARG, "int4_linear_bwd: bad dx_dtype");
    const int64_t N = cache->N, D = cache->D, C = cache->C;
    const int32_t k = cache->k;
    if (N <= 0 || D <= 0 || C <= 0) return fail(I4_ERR_ARG, "int4_linear_bwd: cache not filled by int4_linear_fwd");
    if (ws_bytes < int4_bwd_workspace_size(N, D, C))
        return fail(I4_ERR_WORKSPACE, "int4_linear_bwd: ws_bytes %zu < %zu", ws_bytes, int4_bwd_workspace_size(N, D, C));
    if (!aligned16(dX) || !aligned16(dW) || !aligned16(ws)) return fail(I4_ERR_ALIGN, "int4_linear_bwd: unaligned pointer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool want_lsq = plan && plan->grad_s != nullptr;
    if (want_lsq && (!cache->x_delta || !cache->w_delta))
        return fail(I4_ERR_ARG, "int4_linear_bwd: plan->grad_s needs cache->x_delta and cache->w_delta");
    {
        const BwdWs w0 = carve_bwd_ws(ws, N, D, C);
        const Form2 f2{w0.corr_items, w0.corr_wexp, w0.counts2, w0.sub_items, w0.sub_wexp, w0.tok_flag};
        // the sampler launch also zeroes the A.3 partial slots of the GEMM launch below
        const int32_t words = int32_t(want_lsq ? 2 * i4::kLsqPartials * sizeof(double) / sizeof(uint32_t) : 0);
        I4_RETURN_IF(bitsplit_lss_impl(dY, N, C, cache->x_sqnorm, seed, call_id, token_offset, mode, plan, s,
                                       reinterpret_cast<uint32_t*>(w0.lsq_x), words, w0.det, &f2));
    }

    const int64_t kcap = round_up(2 * N, 128);
    const BwdWs w = carve_bwd_ws(ws, N, D, C);
    {
        i4::CompactArgs ca{};
        ca.q8 = plan->q8; ca.xq = cache->xq;
        ca.N = int32_t(N); ca.C = int32_t(C); ca.D = int32_t(D);
        ca.items_x = plan->items_x; ca.count_x = plan->count_x;
        ca.items_w = plan->items_w; ca.wexp_w = plan->wexp_w; ca.count_w = plan->count_w;
        ca.a_x = w.a_x; ca.a_w = w.a_w; ca.b_w = w.b_w;
        ca.x_touched = plan->x_touched; ca.dx = dX; ca.dx_bf16 = dx_dtype == I4_OUT_BF16;
        ca.det_flags = w.det;
        ca.corr_items = w.corr_items; ca.corr_wexp = w.corr_wexp; ca.corr_count = w.counts2;
        ca.sub_items = w.sub_items; ca.sub_count = w.counts2 + 1; ca.tok_flag = w.tok_flag;
        I4_LAUNCH(i4::launch_compact(ca, s), "compact", s);
    }
    // grad_X and grad_W: one persistent launch over both GEMMs' tiles
    i4::GemmArgs gx{};                           // grad_X: rows = kept items (count on device), K = C, N = D
    gx.M = int32_t(2 * N + 128); gx.m_dev = plan->count_x;
    gx.Nn = int32_t(D); gx.K = int32_t(C);
    gx.epi = i4::EPI_BWD;
    gx.out = dX;
    gx.out_bf16 = dx_dtype == I4_OUT_BF16;
    gx.scale = cache->s_w * inv_sqrt_block(k);
    gx.s_down = plan->s_down;
    gx.k_had = k;
    gx.mask = cache->x_mask;
    gx.items = plan->items_x;
    gx.wexp = plan->wexp_x;
    gx.n_tokens = int32_t(N);
    gx.b_mn = 1;                                 // B = W_hat [C, D] read MN-major (K = C, N = D)
    if (want_lsq) { gx.delta = cache->x_delta; gx.lsq_part = w.lsq_x; }
    gx.dense_flag = w.det + 1;                   // grad_X operand form (sampler): 1 rows = tokens of Q,
                                                 // 2 Q rows + sub-list rows of the sampled tokens
    gx.items2 = w.sub_items; gx.wexp2 = w.sub_wexp; gx.m_dev2 = w.counts2 + 1; gx.tok_flag = w.tok_flag;
    i4::GemmArgs gw{};                           // grad_W: M = C, N = D, K = kept items (count on device)
    gw.M = int32_t(C); gw.Nn = int32_t(D); gw.K = int32_t(kcap); gw.k_dev = plan->count_w;
    gw.epi = i4::EPI_WGRAD;
    gw.out = dW;
    gw.scale = cache->s_x * inv_sqrt_block(k);
    gw.s_down = plan->s_down;
    gw.k_had = k;
    gw.mask = cache->w_mask;
    gw.a_mn = 1; gw.b_mn = 1;                    // A_W [K items, C], B_W [K, D]: both MN-major
    if (want_lsq) { gw.delta = cache->w_delta; gw.lsq_part = w.lsq_w; }
    gw.dense_flag = w.det;                       // grad_W operand form: 1 K = tokens (A = Q, B = X_hat),
    gw.k_dev2 = w.counts2;                       // 2 the same plus the correction rows (A_W, B_W)
    if (plan) gw.out_mc = plan->dw_multicast;    // f4: grad_W all-reduced inside the GEMM (NVLS)
    gw.n_tokens = int32_t(N);
    I4_RETURN_IF(gemm_bwd(Operand{w.a_x, 2 * N + 128, C, C}, Operand{plan->q8, N + 1, C, C},
                          Operand{cache->wq, C, D, D}, Operand{w.a_w, kcap, C, C}, Operand{w.b_w, kcap, D, D},
                          Operand{plan->q8, N + 1, C, C}, Operand{cache->xq, N, D, D}, gx, gw, s));
    if (want_lsq) {
        // A.3: g(s) = 1 / sqrt(Q_P N_elem), Q_P = 7 (reading Z-29 for N_elem)
        const double nx = double(plan->n_elem_x > 0 ? plan->n_elem_x : N * D);
        const double nw = double(plan->n_elem_w > 0 ? plan->n_elem_w : C * D);
        I4_LAUNCH(i4::launch_lsq_finalize(w.lsq_x, w.lsq_w, plan->s_down, cache->s_x, cache->s_w,
                                          1.0 / std::sqrt(7.0 * nx), 1.0 / std::sqrt(7.0 * nw), plan->grad_s, s),
                  "lsq_finalize", s);
    }
    return I4_OK;
}

extern "C" {

namespace {

// Backward workspace of the batched BMM (int4_bmm_bwd), for a chunk of Bc <= 2048
// batches; each region 256-aligned.  The first region (grad_split's per-batch amax
// words) must be zero before the first call; every call leaves it zero.
struct BmmWs {
    uint32_t* bamax; uint32_t* amax; float* s_down; int32_t* counts;
    int32_t* items_w; int8_t* wexp_w; int32_t* items_x; int8_t* wexp_x;
    uint8_t* x_touched; int32_t* a_sq; int8_t* q8; int8_t* a_x; int8_t* a_w; int8_t* b_w;
    size_t off[8];
    size_t total;
};

BmmWs carve_bmm_ws(void* ws, int64_t B, int64_t N, int64_t P, int64_t M) {
    const int64_t Bc = std::min<int64_t>(B, i4::kMaxGemmBatch);
    const int64_t L = 2 * N + 128, kcap = round_up(2 * N, 128);
    BmmWs w{};
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += size_t(round_up(int64_t(bytes), 256)); return o; };
    const size_t o_bam = take(size_t(Bc) * 4);
    const size_t o_am = take(size_t(Bc) * 4);
    const size_t o_sd = take(size_t(Bc) * 4);
    const size_t o_cn = take(size_t(2 * Bc) * 4);
    const size_t o_iw = take(size_t(Bc * L) * 4);
    const size_t o_ew = take(size_t(Bc * L));
    const size_t o_ix = take(size_t(Bc * L) * 4);
    const size_t o_ex = take(size_t(Bc * L));
    const size_t o_xt = take(size_t(Bc * N));
    const size_t o_sq = take(size_t(Bc * 2 * N) * 4);
    const size_t o_q8 = take(size_t(Bc * N + 1) * size_t(P));
    const size_t o_ax = take(size_t(Bc * L) * size_t(P));
    const size_t o_aw = take(size_t(Bc * kcap) * size_t(P));
    const size_t o_bw = take(size_t(Bc * kcap) * size_t(M));
    w.total = off;
    const size_t offs[8] = {o_sd, o_am, o_cn, o_iw, o_ew, o_ix, o_ex, o_q8};
    for (int i = 0; i < 8; ++i) w.off[i] = offs[i];
    if (ws) {
        uint8_t* b = static_cast<uint8_t*>(ws);
        w.bamax = reinterpret_cast<uint32_t*>(b + o_bam);
        w.amax = reinterpret_cast<uint32_t*>(b + o_am);
        w.s_down = reinterpret_cast<float*>(b + o_sd);
        w.counts = reinterpret_cast<int32_t*>(b + o_cn);
        w.items_w = reinterpret_cast<int32_t*>(b + o_iw);
        w.wexp_w = reinterpret_cast<int8_t*>(b + o_ew);
        w.items_x = reinterpret_cast<int32_t*>(b + o_ix);
        w.wexp_x = reinterpret_cast<int8_t*>(b + o_ex);
        w.x_touched = b + o_xt;
        w.a_sq = reinterpret_cast<int32_t*>(b + o_sq);
        w.q8 = reinterpret_cast<int8_t*>(b + o_q8);
        w.a_x = reinterpret_cast<int8_t*>(b + o_ax);
        w.a_w = reinterpret_cast<int8_t*>(b + o_aw);
        w.b_w = reinterpret_cast<int8_t*>(b + o_bw);
    }
    return w;
}

}  // namespace

i4_status int4_bmm_fwd(const void* Q, const void* K, int64_t B, int64_t N, int64_t P, int64_t M, int32_t k,
                       const float* s_q, const float* s_k, void* T, i4_out_dtype t_dtype, i4_bmm_cache* cache,
                       void* stream) {
    I4_RETURN_IF(check_device());
    if (!Q || !K || !T || !cache || !s_q || !s_k || !cache->qq || !cache->kq || !cache->q_mask || !cache->k_mask ||
        !cache->q_sqnorm || !cache->steps)
        return fail(I4_ERR_ARG, "int4_bmm_fwd: NULL pointer");
    if (B <= 0) return fail(I4_ERR_SHAPE, "int4_bmm_fwd: B must be positive");
    if (N <= 0 || P <= 0 || M <= 0 || M % 64 || P % 64 || M > 8192)
        return fail(I4_ERR_SHAPE, "int4_bmm_fwd: need N > 0 and M, P positive multiples of 64 (M <= 8192)");
    if (B * N > (int64_t(1) << 31) || B * P > (int64_t(1) << 31))
        return fail(I4_ERR_SHAPE, "int4_bmm_fwd: B N and B P must stay below 2^31 rows");
    I4_RETURN_IF(check_k(k, M));
    for (int64_t b = 0; b < B; ++b) {
        I4_RETURN_IF(check_step(s_q[b], "s_q[b]"));
        I4_RETURN_IF(check_step(s_k[b], "s_k[b]"));
    }
    if (t_dtype != I4_OUT_F32 && t_dtype != I4_OUT_BF16) return fail(I4_ERR_ARG, "int4_bmm_fwd: bad t_dtype");
    if (!aligned16(Q) || !aligned16(K) || !aligned16(T) || !aligned16(cache->qq) || !aligned16(cache->kq))
        return fail(I4_ERR_ALIGN, "int4_bmm_fwd: unaligned pointer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // per-batch step table (the same host arithmetic as int4_linear_fwd / _bwd per batch)
    std::vector<float> tab(size_t(B) * 8, 0.0f);
    const float isb = inv_sqrt_block(k);
    for (int64_t b = 0; b < B; ++b) {
        float* t = tab.data() + 8 * b;
        t[0] = step_recip(k, s_q[b]);
        t[1] = step_recip(k, s_k[b]);
        t[2] = s_q[b] * s_k[b];                  // fwd scale fl32(s_q s_k), reading Z-22
        t[3] = s_k[b] * isb;                     // grad_Q GEMM scale (as gx.scale of the linear backward)
        t[4] = s_q[b] * isb;                     // grad_K GEMM scale
        t[5] = s_q[b];
        t[6] = s_k[b];
    }
    const bool tab_in_hq = B <= i4::kStepTabChunk;     // the table rides on the quantizer launch
    if (!tab_in_hq) I4_LAUNCH(i4::launch_step_table(tab.data(), B, cache->steps, s), "step_table", s);
    {
        // F1-F3 for every row of Q and K (one launch; per-row r from the batch's table entry)
        i4::HqArgs h{};
        h.x0 = static_cast<const uint16_t*>(Q); h.rows0 = B * N; h.r0 = 1.0f;
        h.codes0 = cache->qq; h.bits0 = cache->q_mask; h.sqnorm0 = cache->q_sqnorm;
        h.r_tab0 = cache->steps; h.rpb0 = N;
        h.x1 = static_cast<const uint16_t*>(K); h.rows1 = B * P; h.r1 = 1.0f;
        h.codes1 = cache->kq; h.bits1 = cache->k_mask; h.sqnorm1 = nullptr;
        h.r_tab1 = cache->steps + 1; h.rpb1 = P;
        h.cols = M; h.k = k;
        h.status = cache->dev_status;
        if (tab_in_hq) { h.tab_host = tab.data(); h.tab_n = int(B); h.tab_dst = cache->steps; }
        I4_LAUNCH(i4::launch_hadamard_quant2(h, s), "hadamard_quant", s);
    }
    {
        // T_b = fl32(s_q s_k) (Q_hat_b K_hat_b^T): one GEMM launch over every batch's tiles
        i4::GemmArgs g{};
        g.M = int32_t(N); g.Nn = int32_t(P); g.K = int32_t(M);
        g.epi = i4::EPI_FWD;
        g.out = T;
        g.out_bf16 = t_dtype == I4_OUT_BF16;
        g.batch = int32_t(B);
        g.tab = cache->steps; g.tab_idx = 2;
        const int bn = i4::gemm_block_n(int(P), false);
        CUtensorMap ta, tb, tc;
        const bool ok =
            make_tmap_i8_3d(&ta, cache->qq, uint64_t(M), uint64_t(N), uint64_t(M), uint64_t(B), uint64_t(N * M), 128u) &&
            make_tmap_i8_3d(&tb, cache->kq, uint64_t(M), uint64_t(P), uint64_t(M), uint64_t(B), uint64_t(P * M),
                            uint32_t(bn / i4::kGemmCG)) &&
            make_tmap_out_3d(&tc, T, g.out_bf16 != 0, uint64_t(P), uint64_t(N), uint64_t(B));
        if (!ok) return fail(I4_ERR_CUDA, "cuTensorMapEncodeTiled failed");
        const i4::GemmMaps maps{&ta, &tb, &tc, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
        I4_LAUNCH(i4::launch_gemm(maps, g, device_info().sms, s), "gemm_i8_fwd", s);
    }
    cache->B = B; cache->N = N; cache->P = P; cache->M = M; cache->k = k;
    return I4_OK;
}

size_t int4_bmm_bwd_workspace_size(int64_t B, int64_t N, int64_t P, int64_t M) {
    if (B <= 0 || N <= 0 || P <= 0 || M <= 0) return 0;
    return carve_bmm_ws(nullptr, B, N, P, M).total;
}

size_t int4_bmm_bwd_ws_offset(int64_t B, int64_t N, int64_t P, int64_t M, int32_t what) {
    if (what < 0 || what > 7 || B <= 0 || N <= 0 || P <= 0 || M <= 0) return size_t(-1);
    return carve_bmm_ws(nullptr, B, N, P, M).off[what];
}

i4_status int4_bmm_bwd(const void* dT, const i4_bmm_cache* cache, uint64_t seed, uint32_t call_id, i4_lss_mode mode,
                       void* dQ, i4_out_dtype dq_dtype, float* dK, void* ws, size_t ws_bytes, void* stream) {
    I4_RETURN_IF(check_device());
    if (!dT || !cache || !dQ || !dK || !ws) return fail(I4_ERR_ARG, "int4_bmm_bwd: NULL pointer");
    if (cache->B <= 0 || !cache->steps) return fail(I4_ERR_ARG, "int4_bmm_bwd: cache not filled by int4_bmm_fwd");
    if (mode != I4_LSS_BERNOULLI && mode != I4_LSS_KEEP_POSITIVE && mode != I4_LSS_NONE)
        return fail(I4_ERR_ARG, "int4_bmm_bwd: bad mode");
    if (dq_dtype != I4_OUT_F32 && dq_dtype != I4_OUT_BF16) return fail(I4_ERR_ARG, "int4_bmm_bwd: bad dq_dtype");
    const int64_t B = cache->B, N = cache->N, P = cache->P, M = cache->M;
    const int32_t k = cache->k;
    if (N > kMaxBwdTokens || N > i4::sampler_max_tokens())
        return fail(I4_ERR_SHAPE, "int4_bmm_bwd: N = %lld exceeds %lld tokens per batch (reading Z-21)", (long long)N,
                    (long long)kMaxBwdTokens);
    if (ws_bytes < int4_bmm_bwd_workspace_size(B, N, P, M))
        return fail(I4_ERR_WORKSPACE, "int4_bmm_bwd: ws_bytes %zu < %zu", ws_bytes, int4_bmm_bwd_workspace_size(B, N, P, M));
    if (!aligned16(dT) || !aligned16(dQ) || !aligned16(dK) || !aligned16(ws))
        return fail(I4_ERR_ALIGN, "int4_bmm_bwd: unaligned pointer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const BmmWs w = carve_bmm_ws(ws, B, N, P, M);
    const int64_t Bc = std::min<int64_t>(B, i4::kMaxGemmBatch);
    const int64_t L = 2 * N + 128, kcap = round_up(2 * N, 128);
    const size_t oq = dq_dtype == I4_OUT_BF16 ? 2 : 4;
    for (int64_t b0 = 0; b0 < B; b0 += Bc) {
        const int64_t nb = std::min<int64_t>(Bc, B - b0);
        const int64_t toff = b0 * N;                  // Philox token index of the chunk's first row (Z-31)
        // B1 + B2: per-batch amax, SR codes, half-row norms
        I4_LAUNCH(i4::launch_grad_split_batched(static_cast<const uint16_t*>(dT) + b0 * N * P, nb * N, P, N, seed,
                                                call_id, toff, w.q8, w.a_sq, w.s_down, w.amax, cache->dev_status,
                                                w.bamax, s),
                  "grad_split", s);
        // LSS steps 2-4: one cluster per (mask, batch)
        i4::SamplerArgs a{};
        a.a_sq = w.a_sq;
        a.x_sqnorm = cache->q_sqnorm + b0 * N;
        a.N = int32_t(N);
        a.mode = int32_t(mode);
        a.seed_lo = uint32_t(seed);
        a.seed_hi = uint32_t(seed >> 32);
        a.call_id = call_id;
        a.token_offset = toff;
        a.items[0] = w.items_w; a.wexp[0] = w.wexp_w; a.count[0] = w.counts;
        a.items[1] = w.items_x; a.wexp[1] = w.wexp_x; a.count[1] = w.counts + Bc;
        a.x_touched = w.x_touched;
        a.zero_words = w.bamax; a.n_zero_words = int32_t(nb);   // grad_split's amax words, for the next call
        a.batch = int32_t(nb);
        a.bs_list = L;
        I4_LAUNCH(i4::launch_lss_sampler(a, s), "lss_sampler", s);
        void* dq_chunk = static_cast<uint8_t*>(dQ) + size_t(b0 * N * M) * oq;
        float* dk_chunk = dK + b0 * P * M;
        i4::CompactArgs ca{};
        ca.q8 = w.q8; ca.xq = cache->qq + b0 * N * M;
        ca.N = int32_t(N); ca.C = int32_t(P); ca.D = int32_t(M);
        ca.items_x = w.items_x; ca.count_x = w.counts + Bc;
        ca.items_w = w.items_w; ca.wexp_w = w.wexp_w; ca.count_w = w.counts;
        ca.a_x = w.a_x; ca.a_w = w.a_w; ca.b_w = w.b_w;
        ca.x_touched = w.x_touched; ca.dx = dq_chunk; ca.dx_bf16 = dq_dtype == I4_OUT_BF16;
        ca.batch = int32_t(nb); ca.bs_list = L;
        I4_LAUNCH(i4::launch_compact(ca, s), "compact", s);
        // grad_Q and grad_K of every batch: one persistent launch
        i4::GemmArgs gx{};
        gx.M = int32_t(L); gx.m_dev = w.counts + Bc;
        gx.Nn = int32_t(M); gx.K = int32_t(P);
        gx.epi = i4::EPI_BWD;
        gx.out = dq_chunk;
        gx.out_bf16 = dq_dtype == I4_OUT_BF16;
        gx.s_down = w.s_down;
        gx.k_had = k;
        gx.mask = cache->q_mask + b0 * N * (M / 32);
        gx.items = w.items_x; gx.wexp = w.wexp_x;
        gx.n_tokens = int32_t(N);
        gx.b_mn = 1;
        gx.batch = int32_t(nb); gx.bs_items = L;
        gx.tab = cache->steps + 8 * b0; gx.tab_idx = 3;
        i4::GemmArgs gw{};
        gw.M = int32_t(P); gw.Nn = int32_t(M); gw.K = int32_t(kcap); gw.k_dev = w.counts;
        gw.epi = i4::EPI_WGRAD;
        gw.out = dk_chunk;
        gw.s_down = w.s_down;
        gw.k_had = k;
        gw.mask = cache->k_mask + b0 * P * (M / 32);
        gw.a_mn = 1; gw.b_mn = 1;
        gw.n_tokens = int32_t(N);
        gw.batch = int32_t(nb);
        gw.tab = cache->steps + 8 * b0; gw.tab_idx = 4;
        CUtensorMap ta, tb, tc, taw, tbw;
        const bool ok =
            make_tmap_i8_3d(&ta, w.a_x, uint64_t(P), uint64_t(L), uint64_t(P), uint64_t(nb), uint64_t(L * P), 128u) &&
            make_tmap_i8_3d(&tb, cache->kq + b0 * P * M, uint64_t(M), uint64_t(P), uint64_t(M), uint64_t(nb),
                            uint64_t(P * M), 128u) &&
            make_tmap_i8_3d(&taw, w.a_w, uint64_t(P), uint64_t(kcap), uint64_t(P), uint64_t(nb), uint64_t(kcap * P), 128u) &&
            make_tmap_i8_3d(&tbw, w.b_w, uint64_t(M), uint64_t(kcap), uint64_t(M), uint64_t(nb), uint64_t(kcap * M), 128u) &&
            make_tmap_out_3d(&tc, dk_chunk, false, uint64_t(M), uint64_t(P), uint64_t(nb));
        if (!ok) return fail(I4_ERR_CUDA, "cuTensorMapEncodeTiled failed");
        const i4::GemmMaps maps{&ta, &tb, &tc, nullptr, nullptr, nullptr, &taw, &tbw, nullptr};
        I4_LAUNCH(i4::launch_gemm(maps, gx, device_info().sms, s, &gw), "gemm_i8_bwd", s);
    }
    return I4_OK;
}

size_t hq_select_k_workspace_size(void) { return i4::select_k_ws_bytes(); }

i4_status hq_select_k(const void* X, int64_t N, const void* W, int64_t C, int64_t D, float s_x, float s_w,
                      int32_t k_min, int32_t k_max, int32_t* k_best, double* mse, void* ws, size_t ws_bytes,
                      void* stream) {
    I4_RETURN_IF(check_device());
    if (!X || !W || !k_best || !mse || !ws) return fail(I4_ERR_ARG, "hq_select_k: NULL pointer");
    if (N <= 0 || C <= 0 || D <= 0 || D % 64 || D > 8192)
        return fail(I4_ERR_SHAPE, "hq_select_k: need N, C > 0 and D a positive multiple of 64 (<= 8192)");
    if (k_min < 0 || k_max > 7 || k_min > k_max) return fail(I4_ERR_SHAPE, "hq_select_k: need 0 <= k_min <= k_max <= 7");
    I4_RETURN_IF(check_k(k_max, D));
    I4_RETURN_IF(check_step(s_x, "s_x"));
    I4_RETURN_IF(check_step(s_w, "s_w"));
    if (ws_bytes < i4::select_k_ws_bytes()) return fail(I4_ERR_WORKSPACE, "hq_select_k: ws too small");
    if (!aligned16(X) || !aligned16(W) || !aligned16(ws) || (reinterpret_cast<uintptr_t>(mse) & 7u))
        return fail(I4_ERR_ALIGN, "hq_select_k: unaligned pointer");
    float r_x[8], r_w[8];
    double c_x[8], c_w[8];
    for (int k = 0; k < 8; ++k) {
        r_x[k] = step_recip(k, s_x);                    // the forward path's quantizer (Z-4)
        r_w[k] = step_recip(k, s_w);
        c_x[k] = double(s_x) * std::pow(2.0, -double(k) / 2.0);   // x_bar = s 2^{-k/2} (codes H_pm1)
        c_w[k] = double(s_w) * std::pow(2.0, -double(k) / 2.0);
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    I4_LAUNCH(i4::launch_select_k(static_cast<const uint16_t*>(X), N, static_cast<const uint16_t*>(W), C, D, r_x, r_w,
                                  c_x, c_w, k_min, k_max, k_best, mse, ws, s),
              "hq_select_k", s);
    return I4_OK;
}

size_t lsq_cold_start_workspace_size(void) { return i4::lsq_cold_start_ws_bytes(); }

i4_status lsq_cold_start_step(const void* x_bf16, int64_t n, float* step, void* ws, size_t ws_bytes, void* stream) {
    I4_RETURN_IF(check_device());
    if (!x_bf16 || !step || !ws) return fail(I4_ERR_ARG, "lsq_cold_start_step: NULL pointer");
    if (n <= 0) return fail(I4_ERR_SHAPE, "lsq_cold_start_step: n must be positive");
    if (ws_bytes < i4::lsq_cold_start_ws_bytes()) return fail(I4_ERR_WORKSPACE, "lsq_cold_start_step: ws too small");
    if (!aligned16(x_bf16) || !aligned16(ws)) return fail(I4_ERR_ALIGN, "lsq_cold_start_step: unaligned pointer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    I4_LAUNCH(i4::launch_lsq_cold_start(static_cast<const uint16_t*>(x_bf16), n, step, ws, s), "lsq_cold_start", s);
    return I4_OK;
}

i4_status int4_gemm_s8s8s32(const int8_t* A, int32_t a_mn_major, const int8_t* B, int32_t b_mn_major, int64_t M,
                            int64_t Nn, int64_t K, int32_t* acc, void* stream) {
    I4_RETURN_IF(check_device());
    if (!A || !B || !acc) return fail(I4_ERR_ARG, "int4_gemm_s8s8s32: NULL pointer");
    if (M <= 0 || Nn <= 0 || K <= 0 || Nn % 64 || K % 16 || (a_mn_major && M % 16))
        return fail(I4_ERR_SHAPE, "int4_gemm_s8s8s32: unsupported shape M=%lld Nn=%lld K=%lld", (long long)M,
                    (long long)Nn, (long long)K);
    if (!aligned16(A) || !aligned16(B) || !aligned16(acc)) return fail(I4_ERR_ALIGN, "int4_gemm_s8s8s32: unaligned pointer");
    i4::GemmArgs g{};
    g.M = int32_t(M); g.Nn = int32_t(Nn); g.K = int32_t(K);
    g.a_mn = a_mn_major != 0; g.b_mn = b_mn_major != 0;
    g.epi = i4::EPI_INT32;
    g.out = acc;
    const Operand a = g.a_mn ? Operand{A, K, M, M} : Operand{A, M, K, K};
    const Operand b = g.b_mn ? Operand{B, K, Nn, Nn} : Operand{B, Nn, K, K};
    return gemm(a, b, g, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
