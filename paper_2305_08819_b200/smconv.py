"""Thin Python binding of libsmconv (include/smconv.h): argument marshalling only.

Every arithmetic step of the three operators runs in the library's sm_100a kernels;
torch provides device memory and the current CUDA stream (north_star: "PyTorch is
used only for device memory, streams and process groups").  There is no CPU
fallback: if the CUDA library is missing this module raises on import-time use.
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsmconv.so")

CONV_OK, CONV_EARG, CONV_EALIGN, CONV_EALIAS, CONV_EWORKSPACE, CONV_EUNSUPPORTED, CONV_ECUDA = range(7)
CONV_MATH_FP32_3XTF32, CONV_MATH_TF32 = 0, 1
CONV_OP_FWD, CONV_OP_BWD_DATA, CONV_OP_BWD_FILTER = 0, 1, 2
CONV_VARIANT_AUTO, CONV_VARIANT_GENERIC, CONV_VARIANT_TMA, CONV_VARIANT_STRIP, CONV_VARIANT_DIRECT = 0, 1, 2, 3, 4
CONV_VARIANT_DWS = 5
CONV_VARIANT_STEM = 6
MATH = {"3xtf32": CONV_MATH_FP32_3XTF32, "fp32": CONV_MATH_FP32_3XTF32, "tf32": CONV_MATH_TF32}

EXPORTS = ("conv2d_out_hw", "conv2d_workspace_bytes", "conv2d_fwd", "conv2d_bwd_data", "conv2d_bwd_filter",
           "conv2d_strerror", "conv2d_last_error_detail")
MCAST_EXPORTS = ("conv2d_bwd_filter_mcast_workspace_bytes", "conv2d_bwd_filter_mcast",
                 "conv2d_bwd_filter_mcast_plan_describe")
EPI_EXPORTS = ("conv2d_epi_workspace_bytes", "conv2d_fwd_epi", "conv2d_bwd_data_epi", "conv2d_epi_plan_describe")
GEMM_EXPORTS = ("gemm_workspace_bytes", "gemm_matmul", "gemm_matmul_t1", "gemm_matmul_t2", "gemm_plan_describe")
EXT_EXPORTS = ("conv2d_force_variant", "conv2d_plan_describe", "conv2d_plan_kernels", "smconv_selftest_host",
               "smconv_probe_tf32", "smconv_set_trace", "smconv_set_hybrid_min_gflop")


class ConvError(RuntimeError):
    def __init__(self, code, detail):
        self.code = code
        self.detail = detail
        super().__init__("%s: %s" % (_strerror(code), detail))


_lib = None
_lock = threading.Lock()


def lib():
    """Load libsmconv.so (built by paper_2305_08819_b200.build / __graft_entry__.build)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                # SMCONV_LIB: an alternative in-tree build of the same library (A/B timing experiments)
                path = os.environ.get("SMCONV_LIB") or LIB_PATH
                if not os.path.exists(path):
                    raise ImportError("libsmconv.so not built (%s); run `python -c \"import __graft_entry__ as g; "
                                      "g.build()\"`" % path)
                L = ctypes.CDLL(path)
                I, P, Z = ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t
                L.conv2d_out_hw.argtypes = [I] * 8 + [ctypes.POINTER(I)] * 2
                L.conv2d_out_hw.restype = I
                L.conv2d_workspace_bytes.argtypes = [I] * 13
                L.conv2d_workspace_bytes.restype = Z
                for f in ("conv2d_fwd", "conv2d_bwd_data", "conv2d_bwd_filter"):
                    fn = getattr(L, f)
                    fn.argtypes = [P, P, P] + [I] * 11 + [I, P, Z, P]
                    fn.restype = I
                L.conv2d_strerror.argtypes = [I]
                L.conv2d_strerror.restype = ctypes.c_char_p
                L.conv2d_last_error_detail.argtypes = []
                L.conv2d_last_error_detail.restype = ctypes.c_char_p
                L.conv2d_force_variant.argtypes = [I, I]
                L.conv2d_force_variant.restype = I
                L.conv2d_plan_describe.argtypes = [I] * 13 + [ctypes.c_char_p, Z]
                L.conv2d_plan_describe.restype = I
                L.conv2d_plan_kernels.argtypes = [I] * 13
                L.conv2d_plan_kernels.restype = I
                L.smconv_selftest_host.argtypes = []
                L.smconv_selftest_host.restype = I
                L.gemm_workspace_bytes.argtypes = [I] * 5
                L.gemm_workspace_bytes.restype = Z
                for f in ("gemm_matmul", "gemm_matmul_t1", "gemm_matmul_t2"):
                    fn = getattr(L, f)
                    fn.argtypes = [P, P, P, I, I, I, I, P, Z, P]
                    fn.restype = I
                L.gemm_plan_describe.argtypes = [I] * 5 + [ctypes.c_char_p, Z]
                L.gemm_plan_describe.restype = I
                F = ctypes.c_float
                L.conv2d_epi_workspace_bytes.argtypes = [I] * 14
                L.conv2d_epi_workspace_bytes.restype = Z
                L.conv2d_fwd_epi.argtypes = [P, P, P, P] + [I] * 11 + [I, I, F, P, Z, P]
                L.conv2d_fwd_epi.restype = I
                L.conv2d_bwd_data_epi.argtypes = [P, P, P, P, P] + [I] * 11 + [I, I, F, P, Z, P]
                L.conv2d_bwd_data_epi.restype = I
                L.conv2d_epi_plan_describe.argtypes = [I] * 14 + [ctypes.c_char_p, Z]
                L.conv2d_epi_plan_describe.restype = I
                L.conv2d_bwd_filter_mcast_workspace_bytes.argtypes = [I] * 12
                L.conv2d_bwd_filter_mcast_workspace_bytes.restype = Z
                L.conv2d_bwd_filter_mcast.argtypes = [P, P, P] + [I] * 11 + [I, P, Z, P]
                L.conv2d_bwd_filter_mcast.restype = I
                L.conv2d_bwd_filter_mcast_plan_describe.argtypes = [I] * 12 + [ctypes.c_char_p, Z]
                L.conv2d_bwd_filter_mcast_plan_describe.restype = I
                L.smconv_set_trace.argtypes = [P]
                L.smconv_set_trace.restype = I
                L.smconv_probe_tf32.argtypes = [P]
                L.smconv_probe_tf32.restype = I
                L.smconv_set_hybrid_min_gflop.argtypes = [ctypes.c_double]
                L.smconv_set_hybrid_min_gflop.restype = ctypes.c_double
                _lib = L
    return _lib


def _strerror(code):
    try:
        return lib().conv2d_strerror(code).decode()
    except Exception:  # pragma: no cover
        return "CONV_%d" % code


def _check(rc):
    if rc != CONV_OK:
        raise ConvError(rc, lib().conv2d_last_error_detail().decode())


def out_hw(IH, IW, FH, FW, stride=(1, 1), padding=(1, 1)):
    oh, ow = ctypes.c_int(), ctypes.c_int()
    _check(lib().conv2d_out_hw(IH, IW, FH, FW, stride[0], stride[1], padding[0], padding[1],
                               ctypes.byref(oh), ctypes.byref(ow)))
    return oh.value, ow.value


def workspace_bytes(op, dims, math=CONV_MATH_FP32_3XTF32):
    n = lib().conv2d_workspace_bytes(op, *dims, math)
    if n == ctypes.c_size_t(-1).value:
        buf = ctypes.create_string_buffer(8)
        rc = lib().conv2d_plan_describe(op, *dims, math, buf, 8)  # recovers the precise status code
        raise ConvError(rc if rc != CONV_OK else CONV_EARG, lib().conv2d_last_error_detail().decode())
    return n


def plan_describe(op, dims, math=CONV_MATH_FP32_3XTF32):
    buf = ctypes.create_string_buffer(256)
    _check(lib().conv2d_plan_describe(op, *dims, math, buf, 256))
    return buf.value.decode()


def plan_kernels(op, dims, math=CONV_MATH_FP32_3XTF32):
    return int(lib().conv2d_plan_kernels(op, *dims, math))


def force_variant(op, variant):
    _check(lib().conv2d_force_variant(op, variant))


def set_hybrid_min_gflop(gflop):
    """TMA fwd / dX calls below `gflop` GFLOP run three TF32 MMAs instead of the hybrid W' form; returns
    the previous threshold (smconv_ext.h)."""
    return float(lib().smconv_set_hybrid_min_gflop(float(gflop)))


def set_pair(on):
    """CTA-pair (cta_group::2) tiles for TMA fwd/dX in 3xTF32 (on by default); returns the old value."""
    return int(lib().smconv_set_pair(1 if on else 0))


def _math(m):
    return MATH[m] if isinstance(m, str) else int(m)


# ------------------------------------------------------------------ torch-facing API
_ws_cache = {}


def _workspace(nbytes, device):
    import torch
    if nbytes == 0:
        return None
    key = (device.index, torch.cuda.current_stream(device).cuda_stream)
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        _ws_cache[key] = buf
    return buf


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def _need(t, name):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise ValueError("%s must be a contiguous float32 CUDA tensor" % name)


def _same_device(*ts):
    d = ts[0].device
    for t in ts[1:]:
        if t.device != d:
            raise ValueError("all tensors must be on the same device (%s vs %s)" % (d, t.device))


def _out(out, shape, like):
    """Allocate the output, or check a caller-supplied one: the C ABI only sees dims derived from the
    inputs, so a mis-shaped `out` would be written out of bounds."""
    import torch
    if out is None:
        return torch.empty(shape, dtype=torch.float32, device=like.device)
    _need(out, "out")
    if tuple(out.shape) != tuple(shape):
        raise ValueError("out has shape %s, expected %s" % (tuple(out.shape), tuple(shape)))
    if out.device != like.device:
        raise ValueError("out is on %s, inputs on %s" % (out.device, like.device))
    return out


def _rank4(t, name):
    if t.dim() != 4:
        raise ValueError("%s must be 4-D (got shape %s)" % (name, tuple(t.shape)))


def raw_call(op, a_ptr, b_ptr, out_ptr, dims, math, ws_ptr, ws_bytes, stream_handle):
    """Direct C-ABI call with raw device pointers (ints) — used by bench.py's step."""
    f = (lib().conv2d_fwd, lib().conv2d_bwd_data, lib().conv2d_bwd_filter)[op]
    _check(f(ctypes.c_void_p(a_ptr), ctypes.c_void_p(b_ptr), ctypes.c_void_p(out_ptr), *dims, math,
             ctypes.c_void_p(ws_ptr or 0), ws_bytes, ctypes.c_void_p(stream_handle)))


def raw_call_epi(op, a_ptr, b_ptr, act_ptr, out_ptr, stats_ptr, dims, math, epi, k, ws_ptr, ws_bytes, stream_handle):
    """Direct C-ABI call of conv2d_fwd_epi (op 0) / conv2d_bwd_data_epi (op 1) with raw device pointers."""
    P = ctypes.c_void_p
    if op == CONV_OP_FWD:
        rc = lib().conv2d_fwd_epi(P(a_ptr), P(b_ptr), P(out_ptr), P(stats_ptr or 0), *dims, math, epi, float(k),
                                  P(ws_ptr or 0), ws_bytes, P(stream_handle))
    else:
        rc = lib().conv2d_bwd_data_epi(P(a_ptr), P(b_ptr), P(act_ptr), P(out_ptr), P(stats_ptr or 0), *dims, math, epi,
                                       float(k), P(ws_ptr or 0), ws_bytes, P(stream_handle))
    _check(rc)


def conv2d_fwd(x, w, stride=(1, 1), padding=(1, 1), math="3xtf32", out=None):
    """Y[N,OH,OW,OC] = X[N,IH,IW,IC] (*) W[OC,FH,FW,IC] (include/smconv.h conv2d_fwd)."""
    import torch
    _need(x, "x")
    _need(w, "w")
    _rank4(x, "x")
    _rank4(w, "w")
    _same_device(x, w)
    N, IH, IW, IC = x.shape
    OC, FH, FW, wic = w.shape
    if wic != IC:
        raise ValueError("w has %d input channels, x has %d" % (wic, IC))
    OH, OW = out_hw(IH, IW, FH, FW, stride, padding)
    out = _out(out, (N, OH, OW, OC), x)
    dims = (N, IH, IW, IC, OC, FH, FW, stride[0], stride[1], padding[0], padding[1])
    m = _math(math)
    nb = workspace_bytes(CONV_OP_FWD, dims, m)
    ws = _workspace(nb, x.device)
    st = torch.cuda.current_stream(x.device).cuda_stream
    _check(lib().conv2d_fwd(_ptr(x), _ptr(w), _ptr(out), *dims, m, _ptr(ws) if ws is not None else None, nb,
                            ctypes.c_void_p(st)))
    return out


def conv2d_bwd_data(dy, w, input_hw, stride=(1, 1), padding=(1, 1), math="3xtf32", out=None):
    """dX[N,IH,IW,IC] = dY (*)^T W  — deconvolution (include/smconv.h conv2d_bwd_data)."""
    import torch
    _need(dy, "dy")
    _need(w, "w")
    _rank4(dy, "dy")
    _rank4(w, "w")
    _same_device(dy, w)
    N, OH, OW, OC = dy.shape
    woc, FH, FW, IC = w.shape
    if woc != OC:
        raise ValueError("w has %d output channels, dy has %d" % (woc, OC))
    IH, IW = input_hw
    out = _out(out, (N, IH, IW, IC), dy)
    dims = (N, IH, IW, IC, OC, FH, FW, stride[0], stride[1], padding[0], padding[1])
    if out_hw(IH, IW, FH, FW, stride, padding) != (OH, OW):
        raise ValueError("dy extent %s does not match input_hw %s" % ((OH, OW), (IH, IW)))
    m = _math(math)
    nb = workspace_bytes(CONV_OP_BWD_DATA, dims, m)
    ws = _workspace(nb, dy.device)
    st = torch.cuda.current_stream(dy.device).cuda_stream
    _check(lib().conv2d_bwd_data(_ptr(dy), _ptr(w), _ptr(out), *dims, m, _ptr(ws) if ws is not None else None, nb,
                                 ctypes.c_void_p(st)))
    return out


def conv2d_bwd_filter(x, dy, kernel_hw, stride=(1, 1), padding=(1, 1), math="3xtf32", out=None):
    """dW[OC,FH,FW,IC] = sum_{n,oh,ow} dY x X-patch (include/smconv.h conv2d_bwd_filter)."""
    import torch
    _need(x, "x")
    _need(dy, "dy")
    _rank4(x, "x")
    _rank4(dy, "dy")
    _same_device(x, dy)
    N, IH, IW, IC = x.shape
    dn, OH, OW, OC = dy.shape
    if dn != N:
        raise ValueError("dy has batch %d, x has %d" % (dn, N))
    FH, FW = kernel_hw
    out = _out(out, (OC, FH, FW, IC), x)
    dims = (N, IH, IW, IC, OC, FH, FW, stride[0], stride[1], padding[0], padding[1])
    if out_hw(IH, IW, FH, FW, stride, padding) != (OH, OW):
        raise ValueError("dy extent does not match the forward output")
    m = _math(math)
    nb = workspace_bytes(CONV_OP_BWD_FILTER, dims, m)
    ws = _workspace(nb, x.device)
    st = torch.cuda.current_stream(x.device).cuda_stream
    _check(lib().conv2d_bwd_filter(_ptr(x), _ptr(dy), _ptr(out), *dims, m, _ptr(ws) if ws is not None else None, nb,
                                   ctypes.c_void_p(st)))
    return out


# ------------------------------------------------------------------ fused epilogues (include/smconv_epi.h)
EPI = {"none": 0, "bn_stats": 1, "leaky": 2, "leaky_bwd": 3, "leaky_bwd_stats": 4}


def _epi(e):
    return EPI[e] if isinstance(e, str) else int(e)


def epi_workspace_bytes(op, dims, math, epi):
    n = lib().conv2d_epi_workspace_bytes(op, *dims, _math(math), _epi(epi))
    if n == ctypes.c_size_t(-1).value:
        raise ConvError(CONV_EARG, lib().conv2d_last_error_detail().decode())
    return n


def epi_plan_describe(op, dims, math, epi):
    buf = ctypes.create_string_buffer(384)
    _check(lib().conv2d_epi_plan_describe(op, *dims, _math(math), _epi(epi), buf, 384))
    return buf.value.decode()


def epi_plan_kernels(op, dims, math, epi):
    """Kernels one fused-epilogue call enqueues (main + split-K / zero fill / W' + epilogue pass + stats)."""
    return int(epi_plan_describe(op, dims, math, epi).rsplit("kernels_epi=", 1)[1])


def conv2d_fwd_epi(x, w, stride=(1, 1), padding=(1, 1), math="3xtf32", epi="bn_stats", k=0.01, out=None):
    """Y = conv(X, W) with a fused epilogue (include/smconv_epi.h conv2d_fwd_epi):
    epi="bn_stats" -> (Y, stats[2, OC] float64: per-channel sum y, sum y^2);  epi="leaky" -> (leaky_k(Y), None)."""
    import torch
    _need(x, "x")
    _need(w, "w")
    _rank4(x, "x")
    _rank4(w, "w")
    _same_device(x, w)
    N, IH, IW, IC = x.shape
    OC, FH, FW, wic = w.shape
    if wic != IC:
        raise ValueError("w has %d input channels, x has %d" % (wic, IC))
    OH, OW = out_hw(IH, IW, FH, FW, stride, padding)
    out = _out(out, (N, OH, OW, OC), x)
    e = _epi(epi)
    stats = torch.empty((2, OC), dtype=torch.float64, device=x.device) if e == EPI["bn_stats"] else None
    dims = (N, IH, IW, IC, OC, FH, FW, stride[0], stride[1], padding[0], padding[1])
    m = _math(math)
    nb = epi_workspace_bytes(CONV_OP_FWD, dims, m, e)
    ws = _workspace(nb, x.device)
    st = torch.cuda.current_stream(x.device).cuda_stream
    _check(lib().conv2d_fwd_epi(_ptr(x), _ptr(w), _ptr(out), _ptr(stats) if stats is not None else None, *dims, m, e,
                                float(k), _ptr(ws) if ws is not None else None, nb, ctypes.c_void_p(st)))
    return out, stats


def conv2d_bwd_data_epi(dy, w, a, input_hw, stride=(1, 1), padding=(1, 1), math="3xtf32", epi="leaky_bwd_stats",
                        k=0.01, out=None):
    """G = deconv(dY, W) * slope_k(A) with a fused epilogue (include/smconv_epi.h conv2d_bwd_data_epi);
    epi="leaky_bwd_stats" also returns stats[2, IC] float64 (sum G, sum G*z).  `out` may be `a` (in place)."""
    import torch
    _need(dy, "dy")
    _need(w, "w")
    _need(a, "a")
    _rank4(dy, "dy")
    _rank4(w, "w")
    _same_device(dy, w, a)
    N, OH, OW, OC = dy.shape
    woc, FH, FW, IC = w.shape
    if woc != OC:
        raise ValueError("w has %d output channels, dy has %d" % (woc, OC))
    IH, IW = input_hw
    if tuple(a.shape) != (N, IH, IW, IC):
        raise ValueError("a has shape %s, expected %s" % (tuple(a.shape), (N, IH, IW, IC)))
    out = _out(out, (N, IH, IW, IC), dy)
    dims = (N, IH, IW, IC, OC, FH, FW, stride[0], stride[1], padding[0], padding[1])
    if out_hw(IH, IW, FH, FW, stride, padding) != (OH, OW):
        raise ValueError("dy extent %s does not match input_hw %s" % ((OH, OW), (IH, IW)))
    e = _epi(epi)
    stats = torch.empty((2, IC), dtype=torch.float64, device=dy.device) if e == EPI["leaky_bwd_stats"] else None
    m = _math(math)
    nb = epi_workspace_bytes(CONV_OP_BWD_DATA, dims, m, e)
    ws = _workspace(nb, dy.device)
    st = torch.cuda.current_stream(dy.device).cuda_stream
    _check(lib().conv2d_bwd_data_epi(_ptr(dy), _ptr(w), _ptr(a), _ptr(out), _ptr(stats) if stats is not None else None,
                                     *dims, m, e, float(k), _ptr(ws) if ws is not None else None, nb,
                                     ctypes.c_void_p(st)))
    return out, stats


# ------------------------------------------------------------------ fused dW all-reduce (include/smconv_mcast.h)
def mcast_workspace_bytes(dims, math=CONV_MATH_FP32_3XTF32):
    n = lib().conv2d_bwd_filter_mcast_workspace_bytes(*dims, _math(math))
    if n == ctypes.c_size_t(-1).value:
        raise ConvError(CONV_EARG, lib().conv2d_last_error_detail().decode())
    return n


def mcast_plan_describe(dims, math=CONV_MATH_FP32_3XTF32):
    buf = ctypes.create_string_buffer(256)
    _check(lib().conv2d_bwd_filter_mcast_plan_describe(*dims, _math(math), buf, 256))
    return buf.value.decode()


def raw_call_mcast(x_ptr, dy_ptr, dw_mc_ptr, dims, math, ws_ptr, ws_bytes, stream_handle):
    """conv2d_bwd_filter_mcast with raw device pointers; dw_mc_ptr is a MULTICAST address (smconv_mcast.h)."""
    P = ctypes.c_void_p
    _check(lib().conv2d_bwd_filter_mcast(P(x_ptr), P(dy_ptr), P(dw_mc_ptr), *dims, _math(math), P(ws_ptr or 0),
                                         ws_bytes, P(stream_handle)))


# ------------------------------------------------------------------ GEMM (include/smgemm.h)
GEMM_MATMUL, GEMM_MATMUL_T1, GEMM_MATMUL_T2 = 0, 1, 2


def gemm_workspace_bytes(g, M, N, K, math=CONV_MATH_FP32_3XTF32):
    n = lib().gemm_workspace_bytes(g, M, N, K, _math(math))
    if n == ctypes.c_size_t(-1).value:
        raise ConvError(CONV_EARG, "gemm_workspace_bytes: invalid arguments (M=%d N=%d K=%d)" % (M, N, K))
    return n


def gemm_plan_describe(g, M, N, K, math=CONV_MATH_FP32_3XTF32):
    buf = ctypes.create_string_buffer(256)
    _check(lib().gemm_plan_describe(g, M, N, K, _math(math), buf, 256))
    return buf.value.decode()


def _gemm(g, a, b, M, N, K, math, out):
    import torch
    _same_device(a, b)
    out = _out(out, (M, N), a)
    m = _math(math)
    nb = gemm_workspace_bytes(g, M, N, K, m)
    ws = _workspace(nb, a.device)
    st = torch.cuda.current_stream(a.device).cuda_stream
    f = (lib().gemm_matmul, lib().gemm_matmul_t1, lib().gemm_matmul_t2)[g]
    _check(f(_ptr(a), _ptr(b), _ptr(out), M, N, K, m, _ptr(ws) if ws is not None else None, nb, ctypes.c_void_p(st)))
    return out


def _mat(t, name):
    _need(t, name)
    if t.dim() != 2:
        raise ValueError("%s must be 2-D (got shape %s)" % (name, tuple(t.shape)))


def matmul(a, b, math="3xtf32", out=None):
    """C[M,N] = A[M,K] . B[K,N]  (matMul, include/smgemm.h)."""
    _mat(a, "a")
    _mat(b, "b")
    (M, K), (K2, N) = a.shape, b.shape
    if K != K2:
        raise ValueError("inner dimensions differ: a %s, b %s" % (tuple(a.shape), tuple(b.shape)))
    return _gemm(GEMM_MATMUL, a, b, M, N, K, math, out)


def matmul_t1(a, b, math="3xtf32", out=None):
    """C[M,N] = A[K,M]^T . B[K,N]  (matMulT1, Fig. 3)."""
    _mat(a, "a")
    _mat(b, "b")
    (K, M), (K2, N) = a.shape, b.shape
    if K != K2:
        raise ValueError("inner dimensions differ: a %s, b %s" % (tuple(a.shape), tuple(b.shape)))
    return _gemm(GEMM_MATMUL_T1, a, b, M, N, K, math, out)


def matmul_t2(a, b, math="3xtf32", out=None):
    """C[M,N] = A[M,K] . B[N,K]^T  (matMulT2)."""
    _mat(a, "a")
    _mat(b, "b")
    (M, K), (N, K2) = a.shape, b.shape
    if K != K2:
        raise ValueError("inner dimensions differ: a %s, b %s" % (tuple(a.shape), tuple(b.shape)))
    return _gemm(GEMM_MATMUL_T2, a, b, M, N, K, math, out)


def probe_tf32():
    """TEST-ONLY: run the tcgen05 TF32 precision probe (csrc/probe.cu); returns 64 floats."""
    import torch
    out = torch.full((64,), float("nan"), dtype=torch.float32, device="cuda")
    _check(lib().smconv_probe_tf32(_ptr(out)))
    return out.cpu().numpy()
