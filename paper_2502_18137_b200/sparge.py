"""Thin Python binding of libsparge.so (include/sparge.h).

Argument marshalling only: every step of the SpargeAttn path runs in the
library's CUDA kernels.  torch supplies device memory and the stream.  There
is no CPU fallback -- importing this module without the built library raises.
"""

import ctypes
import math
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# SPARGE_LIB selects an instrumented build of the same sources (debug only)
LIB_PATH = os.path.join(_HERE, os.environ.get("SPARGE_LIB", "libsparge.so"))

SPARGE_OK, SPARGE_EINVAL, SPARGE_EINTERNAL, SPARGE_ECUDA, SPARGE_ENOTIMPL = 0, 2, 3, 4, 5
SPARGE_BF16, SPARGE_FP16 = 0, 1
SPARGE_SIM_COSINE, SPARGE_SIM_LITERAL = 0, 1
# QK^T operand: INT8 (SageAttention, the default) or the input dtype ("SpargeAttn+FA2", row f1)
SPARGE_QK_INT8, SPARGE_QK_INPUT = 0, 1
# P~V operand: the input dtype (default) or FP8 E4M3 (SageAttention2-style, row f4)
SPARGE_PV_SAME_AS_INPUT, SPARGE_PV_FP8_E4M3 = 0, 1

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2502_18137_b200.build` "
                      "(there is no CPU fallback)")
_lib = ctypes.CDLL(LIB_PATH)


class SpargeError(RuntimeError):
    def __init__(self, fn, code):
        msg = _lib.sparge_strerror(code).decode()
        super().__init__(f"{fn} failed: {msg} ({code})")
        self.code = code


class Strides(ctypes.Structure):
    _fields_ = [("b", ctypes.c_int64), ("h", ctypes.c_int64), ("n", ctypes.c_int64)]


class Shape(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int) for f in
                ("B", "Hq", "Hkv", "N", "d", "bq", "bk", "cw", "causal", "in_dtype",
                 "pv_dtype", "sim_mode", "smooth_k", "qk_dtype")]


_vp, _i32p, _f32p, _f64p, _u8p, _u64p, _i8p = (ctypes.c_void_p,) * 7
_lib.sparge_strerror.restype = ctypes.c_char_p
_lib.sparge_strerror.argtypes = [ctypes.c_int]
_lib.hilbert_permute.restype = ctypes.c_int
_lib.hilbert_permute.argtypes = [ctypes.c_int] * 4 + [_vp, _vp]
_lib.sparge_quantize.restype = ctypes.c_int
_lib.sparge_quantize.argtypes = [ctypes.POINTER(Shape), _vp, Strides, ctypes.c_int, _vp,
                                 _vp, _vp, _vp, _vp, _vp]
_lib.sparge_predict_mask.restype = ctypes.c_int
_lib.sparge_predict_mask.argtypes = [ctypes.POINTER(Shape), _vp, _vp, _vp, _vp,
                                     ctypes.c_float, ctypes.c_float, _vp, _vp, _vp, _vp,
                                     ctypes.c_size_t, _vp]
_lib.sparge_predict_workspace.restype = ctypes.c_size_t
_lib.sparge_predict_workspace.argtypes = [ctypes.POINTER(Shape)]
_lib.sparge_attn_workspace.restype = ctypes.c_size_t
_lib.sparge_attn_workspace.argtypes = [ctypes.POINTER(Shape)]
_lib.sparge_attn_fwd.restype = ctypes.c_int
_lib.sparge_attn_fwd.argtypes = [ctypes.POINTER(Shape), _vp, _vp, _vp, _vp, _vp, Strides,
                                 _vp, _vp, ctypes.c_float, _vp, _vp, Strides, _vp, _vp,
                                 ctypes.c_size_t, _vp]
_lib.sparge_attn_fwd_ex.restype = ctypes.c_int
_lib.sparge_attn_fwd_ex.argtypes = _lib.sparge_attn_fwd.argtypes + [ctypes.c_uint]
_lib.sparge_attn_fwd_mpv.restype = ctypes.c_int
_lib.sparge_attn_fwd_mpv.argtypes = _lib.sparge_attn_fwd.argtypes + [_vp]
_lib.sparge_l1_sums.restype = ctypes.c_int
_lib.sparge_l1_sums.argtypes = [_vp, _vp, ctypes.c_int, ctypes.c_int64, _vp, _vp]
SPARGE_L1_OUT_DOUBLES = 1186
_lib.sparge_attn_status.restype = ctypes.c_int
_lib.sparge_attn_status.argtypes = [_vp, _vp]
_lib.sparge_smooth_k_workspace.restype = ctypes.c_size_t
_lib.sparge_smooth_k_workspace.argtypes = [ctypes.POINTER(Shape)]
_lib.sparge_smooth_k_mean.restype = ctypes.c_int
_lib.sparge_smooth_k_mean.argtypes = [ctypes.POINTER(Shape), _vp, Strides, _vp, ctypes.c_size_t,
                                      _vp, _vp]
_lib.sparge_quantize_smooth_k.restype = ctypes.c_int
_lib.sparge_quantize_smooth_k.argtypes = [ctypes.POINTER(Shape), _vp, Strides, _vp, _vp, _vp,
                                          _vp, _vp, _vp, _vp]

EXPORTED = ("sparge_strerror", "hilbert_permute", "sparge_quantize", "sparge_predict_mask",
            "sparge_predict_workspace",
            "sparge_attn_workspace", "sparge_attn_fwd", "sparge_attn_fwd_ex", "sparge_attn_fwd_mpv",
            "sparge_attn_status", "sparge_l1_sums", "sparge_smooth_k_workspace",
            "sparge_smooth_k_mean", "sparge_quantize_smooth_k")
SPARGE_ATTN_VPREP_ONLY, SPARGE_ATTN_SKIP_VPREP = 1, 2


def _check(fn, code):
    if code != SPARGE_OK:
        raise SpargeError(fn, code)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _strides(t):
    """Element strides of the b, h, n axes of a [B, H, N, d] tensor."""
    if t.stride(3) != 1:
        raise ValueError("the last (d) axis must be contiguous")
    return Strides(t.stride(0), t.stride(1), t.stride(2))


def make_shape(B, Hq, Hkv, N, d, causal=False, dtype=torch.bfloat16, sim_mode=SPARGE_SIM_COSINE,
               qk_dtype=SPARGE_QK_INT8, pv_dtype=SPARGE_PV_SAME_AS_INPUT, smooth_k=False):
    return Shape(B, Hq, Hkv, N, d, 128, 64, 4, int(bool(causal)),
                 SPARGE_FP16 if dtype == torch.float16 else SPARGE_BF16, int(pv_dtype), sim_mode,
                 int(bool(smooth_k)), int(qk_dtype))


# ------------------------------------------------------------------ C-ABI calls
def hilbert_permute(T, H, W, text_prefix=0):
    """Host call -> (perm, inv) int32 numpy arrays (§3.7)."""
    L = text_prefix + T * H * W
    perm = np.empty(L, np.int32)
    inv = np.empty(L, np.int32)
    _check("hilbert_permute", _lib.hilbert_permute(T, H, W, text_prefix,
                                                   perm.ctypes.data_as(ctypes.c_void_p),
                                                   inv.ctypes.data_as(ctypes.c_void_p)))
    return perm, inv


def sparge_quantize(shape, x, is_key, perm, xq, delta, pooled, sim, stream=None):
    _check("sparge_quantize", _lib.sparge_quantize(
        ctypes.byref(shape), _ptr(x), _strides(x), int(is_key), _ptr(perm), _ptr(xq),
        _ptr(delta), _ptr(pooled), _ptr(sim), _stream(stream)))


def sparge_smooth_k_workspace(shape):
    return int(_lib.sparge_smooth_k_workspace(ctypes.byref(shape)))


def sparge_smooth_k_mean(shape, k, workspace, mean, stream=None):
    """K smoothing mean (row f4, R28) -> mean fp32 [B, Hkv, d]."""
    _check("sparge_smooth_k_mean", _lib.sparge_smooth_k_mean(
        ctypes.byref(shape), _ptr(k), _strides(k), _ptr(workspace),
        workspace.numel() * workspace.element_size(), _ptr(mean), _stream(stream)))


def sparge_quantize_smooth_k(shape, k, perm, mean, kq, delta, pooled, sim, stream=None):
    _check("sparge_quantize_smooth_k", _lib.sparge_quantize_smooth_k(
        ctypes.byref(shape), _ptr(k), _strides(k), _ptr(perm), _ptr(mean), _ptr(kq),
        _ptr(delta), _ptr(pooled), _ptr(sim), _stream(stream)))


def sparge_predict_workspace(shape):
    return int(_lib.sparge_predict_workspace(ctypes.byref(shape)))


def sparge_predict_mask(shape, q_pooled, q_sim, k_pooled, k_sim, tau, theta, mask, lut, cnt,
                        workspace, stream=None):
    _check("sparge_predict_mask", _lib.sparge_predict_mask(
        ctypes.byref(shape), _ptr(q_pooled), _ptr(q_sim), _ptr(k_pooled), _ptr(k_sim),
        float(tau), float(theta), _ptr(mask), _ptr(lut), _ptr(cnt), _ptr(workspace),
        workspace.numel() * workspace.element_size(), _stream(stream)))


def sparge_attn_workspace(shape):
    return int(_lib.sparge_attn_workspace(ctypes.byref(shape)))


def sparge_attn_fwd(shape, qq, dq, kq, dk, v, lut, cnt, lam, perm, o, counters, workspace,
                    stream=None):
    _check("sparge_attn_fwd", _lib.sparge_attn_fwd(
        ctypes.byref(shape), _ptr(qq), _ptr(dq), _ptr(kq), _ptr(dk), _ptr(v), _strides(v),
        _ptr(lut), _ptr(cnt), float(lam), _ptr(perm), _ptr(o), _strides(o), _ptr(counters),
        _ptr(workspace), workspace.numel() * workspace.element_size(), _stream(stream)))


def sparge_attn_fwd_ex(shape, qq, dq, kq, dk, v, lut, cnt, lam, perm, o, counters, workspace,
                       flags, stream=None):
    _check("sparge_attn_fwd_ex", _lib.sparge_attn_fwd_ex(
        ctypes.byref(shape), _ptr(qq), _ptr(dq), _ptr(kq), _ptr(dk), _ptr(v), _strides(v),
        _ptr(lut), _ptr(cnt), float(lam), _ptr(perm), _ptr(o), _strides(o), _ptr(counters),
        _ptr(workspace), workspace.numel() * workspace.element_size(), _stream(stream),
        int(flags)))


def sparge_attn_fwd_mpv(shape, qq, dq, kq, dk, v, lut, cnt, lam, perm, o, counters, workspace,
                        mpv, stream=None):
    """sparge_attn_fwd plus the lambda-gate decision dump mpv uint8
    [B, Hq, T_m, T_n, 4] (caller-zeroed; 2 computed, 1 skipped, 0 not kept)."""
    _check("sparge_attn_fwd_mpv", _lib.sparge_attn_fwd_mpv(
        ctypes.byref(shape), _ptr(qq), _ptr(dq), _ptr(kq), _ptr(dk), _ptr(v), _strides(v),
        _ptr(lut), _ptr(cnt), float(lam), _ptr(perm), _ptr(o), _strides(o), _ptr(counters),
        _ptr(workspace), workspace.numel() * workspace.element_size(), _stream(stream),
        _ptr(mpv)))


def sparge_l1_sums(o, o_ref, out=None, stream=None):
    """Device relative-L1 sums of two same-shape contiguous bf16/fp16 tensors
    (§3.6).  Returns the device fp64 buffer; out[0] = sum|o - o_ref|,
    out[1] = sum|o_ref|."""
    if o.shape != o_ref.shape or o.dtype != o_ref.dtype:
        raise ValueError("o and o_ref must have the same shape and dtype")
    if not (o.is_contiguous() and o_ref.is_contiguous()):
        raise ValueError("o and o_ref must be contiguous")
    if out is None:
        out = torch.empty(SPARGE_L1_OUT_DOUBLES, dtype=torch.float64, device=o.device)
    _check("sparge_l1_sums", _lib.sparge_l1_sums(
        _ptr(o), _ptr(o_ref), SPARGE_FP16 if o.dtype == torch.float16 else SPARGE_BF16,
        o.numel(), _ptr(out), _stream(stream)))
    return out


def relative_l1(o, o_ref, stream=None):
    """sum|o - o_ref| / sum|o_ref| computed by the library kernel (host float)."""
    s = sparge_l1_sums(o, o_ref, stream=stream)[:2].cpu()
    return float(s[0] / s[1])


def sparge_attn_status(workspace, stream=None):
    """Synchronises the stream; raises SpargeError(SPARGE_EINTERNAL) if a valid
    row ended with l = 0."""
    _check("sparge_attn_status", _lib.sparge_attn_status(_ptr(workspace), _stream(stream)))


# ------------------------------------------------------------------ plumbing
class Buffers:
    """Device buffers of one forward pass, allocated once with torch."""

    def __init__(self, shape, device="cuda", with_mask=True):
        B, Hq, Hkv, N, d = shape.B, shape.Hq, shape.Hkv, shape.N, shape.d
        tm, tn = math.ceil(N / 128), math.ceil(N / 64)
        kw = dict(device=device)
        self.shape = shape
        if shape.qk_dtype == SPARGE_QK_INPUT:
            qk_t = torch.float16 if shape.in_dtype == SPARGE_FP16 else torch.bfloat16
        else:
            qk_t = torch.int8
        self.qq = torch.empty(B, Hq, N, d, dtype=qk_t, **kw)
        self.kq = torch.empty(B, Hkv, N, d, dtype=qk_t, **kw)
        self.dq = torch.empty(B, Hq, tm, dtype=torch.float32, **kw)
        self.dk = torch.empty(B, Hkv, tn, dtype=torch.float32, **kw)
        self.q_pooled = torch.empty(B, Hq, tm, d, dtype=torch.float64, **kw)
        self.k_pooled = torch.empty(B, Hkv, tn, d, dtype=torch.float64, **kw)
        self.q_sim = torch.empty(B, Hq, tm, dtype=torch.float64, **kw)
        self.k_sim = torch.empty(B, Hkv, tn, dtype=torch.float64, **kw)
        self.mask = torch.empty(B, Hq, tm, tn, dtype=torch.uint8, **kw) if with_mask else None
        self.lut = torch.empty(B, Hq, tm, tn, dtype=torch.int32, **kw)
        self.cnt = torch.empty(B, Hq, tm, dtype=torch.int32, **kw)
        self.counters = torch.zeros(B, Hq, 3, dtype=torch.int64, **kw)
        ws = sparge_attn_workspace(shape)
        self.workspace = torch.zeros((ws + 255) // 256 * 256, dtype=torch.uint8, **kw)
        pws = sparge_predict_workspace(shape)
        self.pred_workspace = torch.empty((pws + 255) // 256 * 256, dtype=torch.uint8, **kw)
        if shape.smooth_k:
            sws = sparge_smooth_k_workspace(shape)
            self.smooth_workspace = torch.empty((sws + 255) // 256 * 256, dtype=torch.uint8, **kw)
            self.k_mean = torch.empty(B, Hkv, d, dtype=torch.float32, **kw)


def _same_shape(a, b):
    return all(getattr(a, f) == getattr(b, f) for f, _ in Shape._fields_)


def _validate(q, k, v, out, perm, causal):
    """Reject what the C ABI cannot see: dtypes, devices and shape agreement
    (the library gets raw pointers and would read e.g. fp32 bytes as bf16)."""
    ts = [("q", q), ("k", k), ("v", v)] + ([("out", out)] if out is not None else [])
    for name, t in ts:
        if not isinstance(t, torch.Tensor) or t.dim() != 4:
            raise ValueError(f"{name} must be a 4-D torch tensor [B, H, N, d]")
        if t.dtype not in (torch.bfloat16, torch.float16):
            raise ValueError(f"{name} must be bf16 or fp16, got {t.dtype}")
        if t.dtype != q.dtype or t.device != q.device:
            raise ValueError(f"{name} must have q's dtype and device")
    B, Hq, N, d = q.shape
    if k.shape != v.shape or k.shape[0] != B or k.shape[2] != N or k.shape[3] != d:
        raise ValueError(f"k/v must be [B, Hkv, N, d] = [{B}, Hkv, {N}, {d}]; got "
                         f"{tuple(k.shape)} / {tuple(v.shape)}")
    if Hq % k.shape[1]:
        raise ValueError("Hq must be a multiple of Hkv (GQA)")
    if out is not None and out.shape != q.shape:
        raise ValueError("out must have q's shape")
    if q.device.type != "cuda":
        raise ValueError("q, k, v must be CUDA tensors (there is no CPU path)")
    if perm is not None:
        if perm.dtype != torch.int32 or perm.device != q.device or perm.numel() != N:
            raise ValueError("perm must be an int32 tensor of N elements on q's device")
        if causal:
            raise ValueError("causal attention with a token permutation is undefined (R8)")


def sparge_forward(q, k, v, tau, theta, lam, causal=False, perm=None, buffers=None, out=None,
                   sim_mode=SPARGE_SIM_COSINE, stream=None, qk_dtype=SPARGE_QK_INT8,
                   pv_dtype=SPARGE_PV_SAME_AS_INPUT, smooth_k=False, counters=None, mpv=None):
    """The whole hot path (a1 quantise Q, K -> a2 predict -> a3 attention) on
    device tensors q [B,Hq,N,d], k/v [B,Hkv,N,d] (bf16 or fp16).  perm: optional
    int32 device tensor [N] (Hilbert order); O is returned in original order.
    qk_dtype=SPARGE_QK_INPUT selects the unquantised "SpargeAttn+FA2" kernel;
    pv_dtype=SPARGE_PV_FP8_E4M3 the FP8 P~V product and smooth_k=True the K
    smoothing (row f4, R28).
    counters: None -> buffers.counters, zeroed first (the C ABI accumulates);
    False -> not counted.  mpv: optional caller-zeroed uint8 [B,Hq,T_m,T_n,4]
    device tensor that receives the lambda-gate decisions (debug mode).
    Returns (O, buffers)."""
    _validate(q, k, v, out, perm, causal)
    B, Hq, N, d = q.shape
    Hkv = k.shape[1]
    shape = make_shape(B, Hq, Hkv, N, d, causal, q.dtype, sim_mode, qk_dtype, pv_dtype, smooth_k)
    if buffers is None:
        buffers = Buffers(shape, device=q.device)
    elif not _same_shape(buffers.shape, shape):
        raise ValueError("buffers were allocated for a different shape / mode")
    bf = buffers
    if counters is None:
        counters = bf.counters
        counters.zero_()
    elif counters is False:
        counters = None
    o = torch.empty_like(q) if out is None else out
    sparge_quantize(shape, q, 0, perm, bf.qq, bf.dq, bf.q_pooled, bf.q_sim, stream)
    if smooth_k:
        sparge_smooth_k_mean(shape, k, bf.smooth_workspace, bf.k_mean, stream)
        sparge_quantize_smooth_k(shape, k, perm, bf.k_mean, bf.kq, bf.dk, bf.k_pooled, bf.k_sim,
                                 stream)
    else:
        sparge_quantize(shape, k, 1, perm, bf.kq, bf.dk, bf.k_pooled, bf.k_sim, stream)
    sparge_predict_mask(shape, bf.q_pooled, bf.q_sim, bf.k_pooled, bf.k_sim, tau, theta,
                        bf.mask, bf.lut, bf.cnt, bf.pred_workspace, stream)
    if mpv is not None:
        sparge_attn_fwd_mpv(shape, bf.qq, bf.dq, bf.kq, bf.dk, v, bf.lut, bf.cnt, lam, perm, o,
                            counters, bf.workspace, mpv, stream)
    else:
        sparge_attn_fwd(shape, bf.qq, bf.dq, bf.kq, bf.dk, v, bf.lut, bf.cnt, lam, perm, o,
                        counters, bf.workspace, stream)
    return o, bf


def pipeline_plan(Hq, Hkv, chunks, tail_split=True):
    """Chunks of q-heads for HostPipeline: [(q0, q1, k0, k1, copy_kv)], q-heads
    [q0, q1) against kv-heads [k0, k1); copy_kv = this chunk brings K/V of
    [k0, k1) to the device (the first chunk that reads them).  `chunks` equal
    runs of whole kv-groups; with tail_split the last run is split so the
    step's tail -- the last chunk's compute and its O copy, which nothing
    overlaps -- is one q-head (or one MHA head): its kv-groups but the last
    become one chunk, the last group's q-heads pieces of halving size
    (group 4 -> 2, 1, 1).  Every chunk is whole kv-groups or lies inside one,
    so each is an independent (B, q-heads, kv-heads) problem."""
    group = Hq // Hkv
    if Hkv % chunks:
        chunks = 1
    kv_per = Hkv // chunks
    plan = [(c * kv_per * group, (c + 1) * kv_per * group, c * kv_per, (c + 1) * kv_per, True)
            for c in range(chunks)]
    if not tail_split:
        return plan
    q0, _, k0, k1, _ = plan.pop()
    if k1 - k0 > 1:                                   # whole groups but the last
        plan.append((q0, q0 + (k1 - 1 - k0) * group, k0, k1 - 1, True))
    g0 = (k1 - 1) * group                             # the last group's q-heads
    left, first = group, True
    while left > 0:
        n = max(1, left // 2) if left > 1 else 1
        if left == 2:
            n = 1
        plan.append((g0, g0 + n, k1 - 1, k1, first))
        g0, left, first = g0 + n, left - n, False
    return plan


class HostPipeline:
    """End-to-end SpargeAttn from pinned HOST buffers with copy/compute overlap.

    The (batch, kv-head group) problems are independent, so
    the work is split into chunks of heads (pipeline_plan): chunk c's
    host->device copy runs on one stream, its kernels (quantise Q, K; predict;
    k_order + V stage; attention) on a second, and its O device->host copy on
    a third, overlapping with the neighbouring chunks; the last chunk is small
    (tail_split) because its compute and O copy follow the last input byte.
    Device buffers are allocated once.  All compute is the C-ABI kernels; this
    class only orchestrates copies and streams (torch)."""

    def __init__(self, B, Hq, Hkv, N, d, causal=False, dtype=torch.bfloat16, chunks=4,
                 device="cuda", sim_mode=SPARGE_SIM_COSINE, qk_dtype=SPARGE_QK_INT8,
                 tail_split=None):
        self.B, self.Hq, self.Hkv, self.N, self.d = B, Hq, Hkv, N, d
        if tail_split is None:
            # split the tail when a chunk's Q is large enough that its compute
            # and O copy outweigh the extra chunks' fixed costs (measured,
            # profiles/r02/r02_s14_e2e_tail_split.txt: Llama 32K -1.2 %,
            # Mochi -4.6 %, CogVideoX -1.8 %, Flux 4.6K +5 %)
            per = Hq // max(1, chunks if Hkv % max(1, chunks) == 0 else 1)
            tail_split = B * per * N * d * 2 >= (8 << 20)
        self.plan = pipeline_plan(Hq, Hkv, chunks, tail_split)
        self.chunks = len(self.plan)
        self.shapes, self.bufs = [], {}
        for q0, q1, k0, k1, _ in self.plan:
            sh = make_shape(B, q1 - q0, k1 - k0, N, d, causal, dtype, sim_mode, qk_dtype)
            key = (q1 - q0, k1 - k0)
            if key not in self.bufs:
                self.bufs[key] = Buffers(sh, device=device, with_mask=False)
            self.shapes.append(sh)
        self.causal, self.qk_dtype = causal, qk_dtype
        kw = dict(device=device, dtype=dtype)
        self.q = torch.empty(B, Hq, N, d, **kw)
        self.k = torch.empty(B, Hkv, N, d, **kw)
        self.v = torch.empty(B, Hkv, N, d, **kw)
        self.o = torch.empty(B, Hq, N, d, **kw)
        self.s_h2d = torch.cuda.Stream(device)
        self.s_comp = torch.cuda.Stream(device)
        self.s_d2h = torch.cuda.Stream(device)

    def __call__(self, qh, kh, vh, oh, tau, theta, lam, perm=None):
        """qh/kh/vh: pinned host [B,H,N,d]; oh: pinned host output.  Enqueues
        everything after the current stream's pending work and makes the
        current stream wait for the final copy."""
        cur = torch.cuda.current_stream()
        for s in (self.s_h2d, self.s_comp, self.s_d2h):
            s.wait_stream(cur)
        for (q0, q1, k0, k1, copy_kv), sh in zip(self.plan, self.shapes):
            qs, ks = slice(q0, q1), slice(k0, k1)
            with torch.cuda.stream(self.s_h2d):
                if copy_kv:
                    self.k[:, ks].copy_(kh[:, ks], non_blocking=True)
                    self.v[:, ks].copy_(vh[:, ks], non_blocking=True)
                self.q[:, qs].copy_(qh[:, qs], non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(self.s_h2d)
            bf = self.bufs[(q1 - q0, k1 - k0)]
            with torch.cuda.stream(self.s_comp):
                self.s_comp.wait_event(ev_in)
                sparge_forward(self.q[:, qs], self.k[:, ks], self.v[:, ks], tau, theta, lam,
                               causal=bool(self.causal), perm=perm, buffers=bf,
                               out=self.o[:, qs], stream=self.s_comp,
                               qk_dtype=self.qk_dtype, counters=False)
                ev_out = torch.cuda.Event()
                ev_out.record(self.s_comp)
            with torch.cuda.stream(self.s_d2h):
                self.s_d2h.wait_event(ev_out)
                oh[:, qs].copy_(self.o[:, qs], non_blocking=True)
        cur.wait_stream(self.s_d2h)
        return oh
