"""B200-native INT4 quantized linear operator of arXiv 2306.11987 (HQ + LSS).

Thin Python binding over the C ABI in include/int4linear.h: argument
marshalling only (torch tensors -> device pointers + sizes + the current
stream).  Every step of the operator runs in the sm_100a kernels of
libint4linear.so; there is no CPU or PyTorch fallback -- importing this
package without the built library raises.

Functions carry the ABI names: hadamard_quant, int4_linear_fwd,
bitsplit_lss, int4_linear_bwd, int4_gemm_s8s8s32.  `Int4Linear` owns the
caller-side buffers (forward cache, sampling plan, workspace) for one layer
shape.
"""
import ctypes
import os

__all__ = [
    "LIB_PATH", "lib", "I4Error", "I4FwdCache", "I4LssPlan",
    "LSS_BERNOULLI", "LSS_KEEP_POSITIVE", "LSS_NONE", "OUT_F32", "OUT_BF16",
    "hadamard_quant", "int4_linear_fwd", "bitsplit_lss", "int4_linear_bwd",
    "int4_bwd_workspace_size", "int4_gemm_s8s8s32", "int4_set_pdl", "lsq_cold_start_step", "hq_select_k", "hq_select_k_workspace_size",
    "int4_bmm_fwd", "int4_bmm_bwd", "int4_bmm_bwd_workspace_size", "Int4BMM", "I4BmmCache",
    "lsq_cold_start_workspace_size", "cold_start_step", "Int4Linear", "BwdScratch", "LaunchTrace",
    "STATUS_NONFINITE", "STATUS_ZERO_GRAD",
]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libint4linear.so")
# development knob of the timing tools (tools/exp_bwd.py, tools/hq_time.py): load a
# compile variant of the same sources (tools/build_variants.sh -D knobs) instead
LIB_PATH = os.environ.get("I4_LIB_OVERRIDE", LIB_PATH)

LSS_BERNOULLI, LSS_KEEP_POSITIVE, LSS_NONE = 0, 1, 2
STATUS_NONFINITE, STATUS_ZERO_GRAD = 1, 2
OUT_F32, OUT_BF16 = 0, 1
_STATUS = {0: "I4_OK", 1: "I4_ERR_SHAPE", 2: "I4_ERR_ALIGN", 3: "I4_ERR_ARG",
           4: "I4_ERR_UNSUPPORTED", 5: "I4_ERR_WORKSPACE", 6: "I4_ERR_CUDA"}


class I4Error(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class I4FwdCache(ctypes.Structure):
    _fields_ = [("xq", ctypes.c_void_p), ("wq", ctypes.c_void_p),
                ("x_mask", ctypes.c_void_p), ("w_mask", ctypes.c_void_p), ("x_sqnorm", ctypes.c_void_p),
                ("N", ctypes.c_int64), ("D", ctypes.c_int64), ("C", ctypes.c_int64),
                ("k", ctypes.c_int32), ("s_x", ctypes.c_float), ("s_w", ctypes.c_float),
                ("w_valid", ctypes.c_int32), ("x_delta", ctypes.c_void_p), ("w_delta", ctypes.c_void_p),
                ("dev_status", ctypes.c_void_p)]


class I4LssPlan(ctypes.Structure):
    _fields_ = [("q8", ctypes.c_void_p), ("a_sq", ctypes.c_void_p), ("amax_bits", ctypes.c_void_p),
                ("s_down", ctypes.c_void_p), ("scratch", ctypes.c_void_p), ("items_w", ctypes.c_void_p),
                ("wexp_w", ctypes.c_void_p),
                ("count_w", ctypes.c_void_p), ("items_x", ctypes.c_void_p), ("wexp_x", ctypes.c_void_p),
                ("count_x", ctypes.c_void_p), ("x_touched", ctypes.c_void_p), ("grad_s", ctypes.c_void_p),
                ("n_elem_x", ctypes.c_int64), ("n_elem_w", ctypes.c_int64), ("dev_status", ctypes.c_void_p),
                ("dw_multicast", ctypes.c_void_p)]


class I4BmmCache(ctypes.Structure):
    _fields_ = [("qq", ctypes.c_void_p), ("kq", ctypes.c_void_p), ("q_mask", ctypes.c_void_p),
                ("k_mask", ctypes.c_void_p), ("q_sqnorm", ctypes.c_void_p), ("steps", ctypes.c_void_p),
                ("dev_status", ctypes.c_void_p),
                ("B", ctypes.c_int64), ("N", ctypes.c_int64), ("P", ctypes.c_int64), ("M", ctypes.c_int64),
                ("k", ctypes.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, i32, u32, u64, f32 = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32,
                                   ctypes.c_uint64, ctypes.c_float)
    sigs = {
        "hadamard_quant": [vp, i64, i64, i32, f32, vp, vp, vp, vp],
        "int4_linear_fwd": [vp, vp, i64, i64, i64, i32, f32, f32, vp, i32, ctypes.POINTER(I4FwdCache), vp],
        "bitsplit_lss": [vp, i64, i64, vp, u64, u32, i64, i32, ctypes.POINTER(I4LssPlan), vp],
        "int4_linear_bwd": [vp, ctypes.POINTER(I4FwdCache), u64, u32, i64, i32, ctypes.POINTER(I4LssPlan), vp, i32,
                            vp, vp, ctypes.c_size_t, vp],
        "int4_gemm_s8s8s32": [vp, i32, vp, i32, i64, i64, i64, vp, vp],
        "lsq_cold_start_step": [vp, i64, vp, vp, ctypes.c_size_t, vp],
        "hq_select_k": [vp, i64, vp, i64, i64, f32, f32, i32, i32, vp, vp, vp, ctypes.c_size_t, vp],
        "int4_bmm_fwd": [vp, vp, i64, i64, i64, i64, i32, vp, vp, vp, i32, ctypes.POINTER(I4BmmCache), vp],
        "int4_bmm_bwd": [vp, ctypes.POINTER(I4BmmCache), u64, u32, i32, vp, i32, vp, vp, ctypes.c_size_t, vp],
    }
    for name, args in sigs.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    L.lsq_cold_start_workspace_size.argtypes = []
    L.lsq_cold_start_workspace_size.restype = ctypes.c_size_t
    L.hq_select_k_workspace_size.argtypes = []
    L.hq_select_k_workspace_size.restype = ctypes.c_size_t
    L.int4_bwd_ws_form2_offset.argtypes = [i64, i64, i64]
    L.int4_bwd_ws_form2_offset.restype = ctypes.c_size_t
    L.int4_bmm_bwd_workspace_size.argtypes = [i64, i64, i64, i64]
    L.int4_bmm_bwd_workspace_size.restype = ctypes.c_size_t
    L.int4_bmm_bwd_ws_offset.argtypes = [i64, i64, i64, i64, i32]
    L.int4_bmm_bwd_ws_offset.restype = ctypes.c_size_t
    L.int4_bwd_ws_det_offset.argtypes = [i64, i64, i64]
    L.int4_bwd_ws_det_offset.restype = ctypes.c_size_t
    L.int4_bwd_workspace_size.argtypes = [i64, i64, i64]
    L.int4_bwd_workspace_size.restype = ctypes.c_size_t
    L.int4_sampler_cluster_ctas.argtypes = [i64]
    L.int4_sampler_cluster_ctas.restype = i32
    L.int4_set_pdl.argtypes = [i32]
    L.int4_set_pdl.restype = i32
    L.int4_last_error.argtypes = []
    L.int4_last_error.restype = ctypes.c_char_p
    L.int4_trace_begin.argtypes = [ctypes.POINTER(ctypes.c_void_p), i32, i32]
    L.int4_trace_begin.restype = ctypes.c_int
    L.int4_trace_end.argtypes = [ctypes.POINTER(ctypes.c_char_p), i32]
    L.int4_trace_end.restype = i32
    return L


lib = _load()


def _check(status):
    if status != 0:
        raise I4Error(status, lib.int4_last_error().decode())


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def hadamard_quant(x, k, step, codes, clamp_bits=None, row_sqnorm=None, stream=None):
    """F1+F2: block-Hadamard + LSQ of a bf16 [rows, cols] tensor."""
    rows, cols = x.shape
    _check(lib.hadamard_quant(_ptr(x), rows, cols, k, float(step), _ptr(codes), _ptr(clamp_bits),
                              _ptr(row_sqnorm), _stream(stream)))


def int4_linear_fwd(X, W, k, s_x, s_w, Y, cache, stream=None):
    """HQ-MM forward; cache is an I4FwdCache with device buffers."""
    import torch
    N, D = X.shape
    C = W.shape[0]
    y_dtype = OUT_BF16 if Y.dtype == torch.bfloat16 else OUT_F32
    _check(lib.int4_linear_fwd(_ptr(X), _ptr(W), N, D, C, k, float(s_x), float(s_w), _ptr(Y), y_dtype,
                               ctypes.byref(cache), _stream(stream)))


def bitsplit_lss(dY, x_sqnorm, seed, call_id, token_offset, mode, plan, stream=None):
    """LSS-MM steps 1-4 into an I4LssPlan."""
    N, C = dY.shape
    _check(lib.bitsplit_lss(_ptr(dY), N, C, _ptr(x_sqnorm), int(seed), int(call_id), int(token_offset), int(mode),
                            ctypes.byref(plan), _stream(stream)))


def int4_linear_bwd(dY, cache, seed, call_id, token_offset, mode, plan, dX, dW, ws, stream=None):
    """LSS-MM backward; dX fp32 or bf16, dW fp32."""
    import torch
    dx_dtype = OUT_BF16 if dX.dtype == torch.bfloat16 else OUT_F32
    _check(lib.int4_linear_bwd(_ptr(dY), ctypes.byref(cache), int(seed), int(call_id), int(token_offset), int(mode),
                               ctypes.byref(plan), _ptr(dX), dx_dtype, _ptr(dW), _ptr(ws),
                               ws.numel() * ws.element_size(), _stream(stream)))


def int4_bwd_workspace_size(N, D, C):
    return int(lib.int4_bwd_workspace_size(N, D, C))


def int4_gemm_s8s8s32(A, B, acc, a_mn_major=False, b_mn_major=False, stream=None):
    """acc[m, n] = sum_k A(m, k) B(n, k), int8 x int8 -> int32 on tcgen05.
    A is [M, K] or, if a_mn_major, [K, M]; B is [Nn, K] or, if b_mn_major, [K, Nn]."""
    M, Nn = acc.shape
    K = A.shape[0] if a_mn_major else A.shape[1]
    _check(lib.int4_gemm_s8s8s32(_ptr(A), int(a_mn_major), _ptr(B), int(b_mn_major), M, Nn, K, _ptr(acc),
                                 _stream(stream)))


def hq_select_k_workspace_size():
    return int(lib.hq_select_k_workspace_size())


def hq_select_k(X, W, s_x, s_w, k_min, k_max, k_best, mse, ws, stream=None):
    """A.5: per-k reconstruction MSEs of X and W into mse (float64
    device [16]) and the argmin of their product into k_best (int32 device [1])."""
    N, D = X.shape
    C = W.shape[0]
    _check(lib.hq_select_k(_ptr(X), N, _ptr(W), C, D, float(s_x), float(s_w), int(k_min), int(k_max),
                           _ptr(k_best), _ptr(mse), _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)))


def lsq_cold_start_workspace_size():
    return int(lib.lsq_cold_start_workspace_size())


def lsq_cold_start_step(x, step, ws, stream=None):
    """A.4 cold start: step[0] = fl32(2 mean|x| / sqrt(7)) on the device.
    x: bf16 tensor; step: float32 device tensor; ws: zeroed uint8 tensor of
    lsq_cold_start_workspace_size() bytes (left zeroed)."""
    _check(lib.lsq_cold_start_step(_ptr(x), x.numel(), _ptr(step), _ptr(ws), ws.numel() * ws.element_size(),
                                   _stream(stream)))


def cold_start_step(x, stream=None):
    """A.4 cold-start step size of a bf16 device tensor, computed by the library's
    lsq_cold_start_step kernel and returned as a host float (synchronises `stream`;
    a setup-time convenience, not for the hot path)."""
    import torch
    step = torch.empty(1, dtype=torch.float32, device=x.device)
    ws = torch.zeros(lsq_cold_start_workspace_size(), dtype=torch.uint8, device=x.device)
    lsq_cold_start_step(x, step, ws, stream)
    return float(step.cpu()[0])


def int4_set_pdl(enable):
    """Switch programmatic dependent launch for all library launches; returns the previous setting."""
    return bool(lib.int4_set_pdl(1 if enable else 0))


class LaunchTrace:
    """Context manager around the library's launch-tracing hook: the events
    (torch.cuda.Event, enable_timing) bracket the library launches
    first_launch, first_launch + 1, ... made on its stream while the context is
    open (inside a CUDA graph capture the records become graph nodes; create
    the events with external=True then).  `names` lists every launch seen."""

    def __init__(self, events, first_launch=0):
        import torch
        self.events = events
        self.first = first_launch
        for e in events:                           # force lazy creation of the handles
            e.record(torch.cuda.current_stream())
        torch.cuda.current_stream().synchronize()
        self.handles = (ctypes.c_void_p * len(events))(*[e.cuda_event for e in events])
        self.names = []

    def __enter__(self):
        _check(lib.int4_trace_begin(self.handles, len(self.events), self.first))
        return self

    def __exit__(self, *exc):
        buf = (ctypes.c_char_p * 64)()
        n = lib.int4_trace_end(buf, 64)
        self.names = [buf[i].decode() for i in range(n)]
        return False

    def durations_ms(self):
        """[(name, ms)] of the launches inside the window (events must have completed)."""
        win = self.names[self.first:self.first + len(self.events) - 1]
        return [(nm, self.events[i].elapsed_time(self.events[i + 1])) for i, nm in enumerate(win)]


class _PlanBuffers:
    """Device buffers of one i4_lss_plan (N tokens, C output features)."""

    def __init__(self, N, C, dev):
        import torch
        i8, i32 = torch.int8, torch.int32
        n2 = 2 * N + 128
        self.q8 = torch.empty(N + 1, C, dtype=i8, device=dev)   # 8-bit SR codes q = 16 hi + lo; row N: zeros
        self.a_sq = torch.empty(2 * N, dtype=i32, device=dev)
        self.scalars = torch.zeros(8, dtype=i32, device=dev)      # amax_bits, s_down, count_w, count_x
        self.scratch = torch.zeros(2048, dtype=i32, device=dev)  # fused-amax block maxima
        self.items_w = torch.empty(n2, dtype=i32, device=dev)
        self.wexp_w = torch.empty(n2, dtype=i8, device=dev)
        self.items_x = torch.empty(n2, dtype=i32, device=dev)
        self.wexp_x = torch.empty(n2, dtype=i8, device=dev)
        self.x_touched = torch.empty(N, dtype=torch.uint8, device=dev)
        sp = self.scalars.data_ptr()
        self.plan = I4LssPlan(q8=self.q8.data_ptr(), a_sq=self.a_sq.data_ptr(), amax_bits=sp, s_down=sp + 4,
                              scratch=self.scratch.data_ptr(),
                              items_w=self.items_w.data_ptr(), wexp_w=self.wexp_w.data_ptr(), count_w=sp + 8,
                              items_x=self.items_x.data_ptr(), wexp_x=self.wexp_x.data_ptr(), count_x=sp + 12,
                              x_touched=self.x_touched.data_ptr())

    def views(self):
        return {k: getattr(self, k) for k in ("q8", "a_sq", "scalars", "scratch", "items_w", "wexp_w",
                                              "items_x", "wexp_x", "x_touched")}


class BwdScratch:
    """Transient backward buffers (sampling plan, workspace, status word) for
    token count N and shapes up to D_max x C_max.  They are only live during one
    int4_linear_bwd, so the linears of a network that run their backwards one
    after another on one stream share one BwdScratch (the forward caches stay
    per layer)."""

    def __init__(self, N, D_max, C_max, device="cuda"):
        import torch
        dev = torch.device(device)
        self.N, self.D_max, self.C_max = N, D_max, C_max
        self.plan_bufs = _PlanBuffers(N, C_max, dev)
        self.ws = torch.empty(int4_bwd_workspace_size(N, D_max, C_max), dtype=torch.uint8, device=dev)
        self.status_buf = torch.zeros(1, dtype=torch.int32, device=dev)
        self.plan_bufs.plan.dev_status = self.status_buf.data_ptr()

    def fits(self, N, D, C):
        return N == self.N and D <= self.D_max and C <= self.C_max


class Int4Linear:
    """Caller-side buffers of one INT4 linear layer shape [N, D] x [C, D].

    Allocates (torch, on `device`) the forward cache once, and the sampling plan
    and backward workspace unless a shared BwdScratch is passed; forward /
    backward then only launch kernels.
    """

    def __init__(self, N, D, C, k, device="cuda", step_grads=False, scratch=None):
        """step_grads: also keep the A.3 deltas in the forward cache and return the
        step-size gradients {grad s_X, grad s_W} from backward (see grad_s()).
        scratch: a BwdScratch shared with other layers (None: a private one)."""
        import torch
        self.N, self.D, self.C, self.k = N, D, C, k
        dev = torch.device(device)
        i8, i32, f32 = torch.int8, torch.int32, torch.float32
        self.xq = torch.empty(N, D, dtype=i8, device=dev)
        self.wq = torch.empty(C, D, dtype=i8, device=dev)
        self.x_mask = torch.empty(N, D // 32, dtype=i32, device=dev)
        self.w_mask = torch.empty(C, D // 32, dtype=i32, device=dev)
        self.x_sqnorm = torch.empty(N, dtype=i32, device=dev)
        self.cache = I4FwdCache(xq=self.xq.data_ptr(), wq=self.wq.data_ptr(),
                                x_mask=self.x_mask.data_ptr(), w_mask=self.w_mask.data_ptr(),
                                x_sqnorm=self.x_sqnorm.data_ptr(), w_valid=0)
        if scratch is None:
            scratch = BwdScratch(N, D, C, dev)
        elif not scratch.fits(N, D, C):
            raise ValueError(f"BwdScratch(N={scratch.N}, D<={scratch.D_max}, C<={scratch.C_max}) too small")
        self.scratch = scratch
        self._plan_bufs = scratch.plan_bufs
        self.__dict__.update(self._plan_bufs.views())
        self.plan = self._plan_bufs.plan
        self.ws = scratch.ws
        # device status word shared by the forward cache and the plan (I4_STATUS_* bits)
        self.status_buf = scratch.status_buf
        self.cache.dev_status = self.status_buf.data_ptr()
        self.step_grads = bool(step_grads)
        if self.step_grads:
            self.x_delta = torch.empty(N, D, dtype=f32, device=dev)
            self.w_delta = torch.empty(C, D, dtype=f32, device=dev)
            self.grad_s_buf = torch.zeros(2, dtype=f32, device=dev)
            self.cache.x_delta = self.x_delta.data_ptr()
            self.cache.w_delta = self.w_delta.data_ptr()

    def forward(self, X, W, s_x, s_w, Y, reuse_weight=False, stream=None):
        self.cache.w_valid = 1 if reuse_weight else 0
        int4_linear_fwd(X, W, self.k, s_x, s_w, Y, self.cache, stream)

    def backward(self, dY, dX, dW, seed, call_id=0, token_offset=0, mode=LSS_BERNOULLI, stream=None,
                 dw_multicast=None):
        """dw_multicast: optional multicast address (int) of a symmetric grad_W buffer; the
        grad_W GEMM then all-reduces into it in its epilogue (NVLS, see the header)."""
        # the plan may be shared with other layers: point it at this layer's outputs
        self.plan.grad_s = self.grad_s_buf.data_ptr() if self.step_grads else None
        self.plan.dw_multicast = dw_multicast
        int4_linear_bwd(dY, self.cache, seed, call_id, token_offset, mode, self.plan, dX, dW, self.ws, stream)

    def status(self):
        """Device status word (int32 tensor [1]): bit 0 = I4_STATUS_NONFINITE (an Inf / NaN
        input), bit 1 = I4_STATUS_ZERO_GRAD (all-zero grad_Y).  Bits accumulate until
        clear_status()."""
        return self.status_buf

    def clear_status(self):
        self.status_buf.zero_()

    # views of the device-side sampling state (for tests and reports)
    def s_down(self):
        return self.scalars[1:2].view(__import__("torch").float32)

    def counts(self):
        return self.scalars[2:4]

    def dense_flags(self):
        """[grad_W mask deterministic, grad_X mask deterministic] of the last backward
        (reading Z-32: the GEMMs then ran on Q / X_hat), an int32 device tensor."""
        import torch
        off = lib.int4_bwd_ws_det_offset(self.N, self.D, self.C)
        return self.ws[off:off + 8].view(torch.int32)

    def form2_counts(self):
        """[grad_W correction rows, grad_X sampled-token rows] of the last backward when a
        mask ran in operand form 2 (reading Z-33), an int32 device tensor."""
        import torch
        off = lib.int4_bwd_ws_form2_offset(self.N, self.D, self.C)
        return self.ws[off:off + 8].view(torch.int32)

    def q8_codes(self):
        """The code plane of the last backward as an [N + 1, C] int8 view."""
        return self.q8.view(-1)[:(self.N + 1) * self.C].view(self.N + 1, self.C)

    def grad_s(self):
        """{grad s_X, grad s_W} of the last backward (A.3), a float32 device tensor."""
        if not self.step_grads:
            raise RuntimeError("Int4Linear(step_grads=True) is required for step-size gradients")
        return self.grad_s_buf


def int4_bmm_fwd(Q, K, k, s_q, s_k, T, cache, stream=None):
    """A.1 BMM forward: per-batch HQ-MM; s_q, s_k host float32 arrays."""
    import numpy as np
    import torch
    B, N, M = Q.shape
    P = K.shape[1]
    sq = np.ascontiguousarray(s_q, dtype=np.float32)
    sk = np.ascontiguousarray(s_k, dtype=np.float32)
    t_dtype = OUT_BF16 if T.dtype == torch.bfloat16 else OUT_F32
    _check(lib.int4_bmm_fwd(_ptr(Q), _ptr(K), B, N, P, M, k, sq.ctypes.data, sk.ctypes.data, _ptr(T), t_dtype,
                            ctypes.byref(cache), _stream(stream)))


def int4_bmm_bwd(dT, cache, seed, call_id, mode, dQ, dK, ws, stream=None):
    """A.1 BMM backward, batched inside the kernels: per-batch LSS-MM with token offsets
    b N (reading Z-31).  ws: uint8 device tensor of int4_bmm_bwd_workspace_size bytes,
    zeroed before its first use."""
    import torch
    dq_dtype = OUT_BF16 if dQ.dtype == torch.bfloat16 else OUT_F32
    _check(lib.int4_bmm_bwd(_ptr(dT), ctypes.byref(cache), int(seed), int(call_id), int(mode), _ptr(dQ), dq_dtype,
                            _ptr(dK), _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)))


def int4_bmm_bwd_workspace_size(B, N, P, M):
    return int(lib.int4_bmm_bwd_workspace_size(B, N, P, M))


class Int4BMM:
    """Caller-side buffers of one attention BMM shape T = BMM(Q [B,N,M], K [B,P,M]^T)."""

    def __init__(self, B, N, P, M, k, device="cuda"):
        import torch
        self.B, self.N, self.P, self.M, self.k = B, N, P, M, k
        dev = torch.device(device)
        i8, i32 = torch.int8, torch.int32
        self.qq = torch.empty(B, N, M, dtype=i8, device=dev)
        self.kq = torch.empty(B, P, M, dtype=i8, device=dev)
        self.q_mask = torch.empty(B, N, M // 32, dtype=i32, device=dev)
        self.k_mask = torch.empty(B, P, M // 32, dtype=i32, device=dev)
        self.q_sqnorm = torch.empty(B, N, dtype=i32, device=dev)
        self.steps = torch.zeros(B, 8, dtype=torch.float32, device=dev)
        self.status_buf = torch.zeros(1, dtype=i32, device=dev)
        self.cache = I4BmmCache(qq=self.qq.data_ptr(), kq=self.kq.data_ptr(), q_mask=self.q_mask.data_ptr(),
                                k_mask=self.k_mask.data_ptr(), q_sqnorm=self.q_sqnorm.data_ptr(),
                                steps=self.steps.data_ptr(), dev_status=self.status_buf.data_ptr())
        self.ws = torch.zeros(int4_bmm_bwd_workspace_size(B, N, P, M), dtype=torch.uint8, device=dev)

    def forward(self, Q, K, s_q, s_k, T, stream=None):
        int4_bmm_fwd(Q, K, self.k, s_q, s_k, T, self.cache, stream)

    def backward(self, dT, dQ, dK, seed, call_id=0, mode=LSS_BERNOULLI, stream=None):
        int4_bmm_bwd(dT, self.cache, seed, call_id, mode, dQ, dK, self.ws, stream)

    def status(self):
        return int(self.status_buf.item())

    def ws_view(self, what):
        """A region of the last backward's workspace (its first chunk of <= 2048 batches) as a
        device tensor: 0 s_down [B] f32, 1 amax bits [B] i32, 2 kept counts [2, B] i32
        ([0] grad_K mask, [1] grad_Q mask), 3 / 5 grad_K / grad_Q item lists [B, 2N+128] i32,
        4 / 6 their weight exponents [B, 2N+128] i8, 7 SR codes q [B N + 1, P] i8."""
        import torch
        B, N, P, M = min(self.B, 2048), self.N, self.P, self.M
        off = int(lib.int4_bmm_bwd_ws_offset(self.B, N, P, M, what))
        L = 2 * N + 128
        dt, shape = {0: (torch.float32, (B,)), 1: (torch.int32, (B,)), 2: (torch.int32, (2, B)),
                     3: (torch.int32, (B, L)), 4: (torch.int8, (B, L)), 5: (torch.int32, (B, L)),
                     6: (torch.int8, (B, L)), 7: (torch.int8, (B * N + 1, P))}[what]
        n = 1
        for d in shape:
            n *= d
        esz = torch.tensor([], dtype=dt).element_size()
        return self.ws[off:off + n * esz].view(dt).view(*shape)
