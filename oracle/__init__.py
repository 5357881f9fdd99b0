"""CPU oracle for the conv hot path of arXiv 2305.08819 — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference``) may import this package.  The product path
(``paper_2305_08819_b200``) never imports it, and the two share no code: this
wrapper marshals numpy arrays into ``liboracle.so`` (built from
``conv_oracle.c``), which computes the plain definitions O1-O3 with double
accumulation (see the C file for the paper/SPEC passages each follows).

Inputs are float32 arrays (the same host arrays the GPU path receives); outputs
are float64.

Pins: every function here is pinned by ``tests/test_oracle_pins.py`` against
things other than itself — closed forms, the trilinear adjoint identity, 1x1 conv
= BLAS matmul, delta kernels = shifts, exact finite differences of a bilinear
form, SPEC's worked values (tests/golden/), and torch's CPU float64 conv as an
independent library routine.  No function is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "conv_oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "net_oracle.c")]
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc -O2 -fopenmp (plain C, no vectorisation tricks needed)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(os.path.getmtime(f) for f in _SRCS):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c99"] + _SRCS + ["-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        fp = ctypes.POINTER(ctypes.c_float)
        dp = ctypes.POINTER(ctypes.c_double)
        ints = [ctypes.c_int] * 11
        for name, a, b in (("oracle_conv2d_fwd", fp, fp), ("oracle_conv2d_bwd_data", fp, fp),
                           ("oracle_conv2d_bwd_filter", fp, fp)):
            f = getattr(lib, name)
            f.argtypes = [a, b, dp] + ints
            f.restype = ctypes.c_int
        lib.oracle_conv2d_bwd_filter_at.argtypes = [fp, fp, ctypes.POINTER(ctypes.c_longlong), ctypes.c_int,
                                                    dp] + ints
        lib.oracle_conv2d_bwd_filter_at.restype = ctypes.c_int
        lib.oracle_out_hw.argtypes = [ctypes.c_int] * 8 + [ctypes.POINTER(ctypes.c_int)] * 2
        lib.oracle_out_hw.restype = ctypes.c_int
        lib.oracle_num_threads.restype = ctypes.c_int
        I, LL, D = ctypes.c_int, ctypes.c_longlong, ctypes.c_double
        lib.oracle_matmul.argtypes = [fp, fp, dp, I, I, I, I, I]
        lib.oracle_matmul.restype = I
        lib.oracle_channel_stats.argtypes = [dp, LL, I, dp, dp]
        lib.oracle_channel_stats.restype = I
        lib.oracle_leaky_relu.argtypes = [dp, dp, LL, D]
        lib.oracle_leaky_relu.restype = I
        lib.oracle_leaky_bwd_stats.argtypes = [dp, fp, LL, I, D, dp, dp, dp]
        lib.oracle_leaky_bwd_stats.restype = I
        lib.oracle_set_num_threads.argtypes = [ctypes.c_int]
        _lib = lib
    return _lib


def _f32(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def out_hw(IH, IW, FH, FW, sh, sw, ph, pw):
    lib = _load()
    oh, ow = ctypes.c_int(), ctypes.c_int()
    if lib.oracle_out_hw(IH, IW, FH, FW, sh, sw, ph, pw, ctypes.byref(oh), ctypes.byref(ow)):
        raise ValueError("invalid conv geometry")
    return oh.value, ow.value


def conv2d_fwd(X, W, stride=(1, 1), padding=(1, 1)):
    """Y[N,OH,OW,OC] (float64) = X[N,IH,IW,IC] (*) W[OC,FH,FW,IC]  (O1)."""
    X, xp = _f32(X)
    W, wp = _f32(W)
    N, IH, IW, IC = X.shape
    OC, FH, FW, IC2 = W.shape
    assert IC == IC2
    OH, OW = out_hw(IH, IW, FH, FW, stride[0], stride[1], padding[0], padding[1])
    Y = np.empty((N, OH, OW, OC), np.float64)
    rc = _load().oracle_conv2d_fwd(xp, wp, Y.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                   N, IH, IW, IC, OC, FH, FW, stride[0], stride[1],
                                   padding[0], padding[1])
    if rc:
        raise ValueError("oracle_conv2d_fwd: bad arguments")
    return Y


def conv2d_bwd_data(dY, W, input_hw, stride=(1, 1), padding=(1, 1)):
    """dX[N,IH,IW,IC] (float64) = dY (*)^T W  (O2), IH,IW given explicitly (reading L5)."""
    dY, dyp = _f32(dY)
    W, wp = _f32(W)
    N, OH, OW, OC = dY.shape
    OC2, FH, FW, IC = W.shape
    assert OC == OC2
    IH, IW = input_hw
    if out_hw(IH, IW, FH, FW, stride[0], stride[1], padding[0], padding[1]) != (OH, OW):
        raise ValueError("dY extent does not match the forward output of input_hw")
    dX = np.empty((N, IH, IW, IC), np.float64)
    rc = _load().oracle_conv2d_bwd_data(dyp, wp, dX.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                        N, IH, IW, IC, OC, FH, FW, stride[0], stride[1],
                                        padding[0], padding[1])
    if rc:
        raise ValueError("oracle_conv2d_bwd_data: bad arguments")
    return dX


def conv2d_bwd_filter(X, dY, kernel_hw, stride=(1, 1), padding=(1, 1)):
    """dW[OC,FH,FW,IC] (float64) = sum_{n,oh,ow} dY x X-patch  (O3)."""
    X, xp = _f32(X)
    dY, dyp = _f32(dY)
    N, IH, IW, IC = X.shape
    N2, OH, OW, OC = dY.shape
    assert N == N2
    FH, FW = kernel_hw
    if out_hw(IH, IW, FH, FW, stride[0], stride[1], padding[0], padding[1]) != (OH, OW):
        raise ValueError("dY extent does not match the forward output")
    dW = np.empty((OC, FH, FW, IC), np.float64)
    rc = _load().oracle_conv2d_bwd_filter(xp, dyp, dW.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                          N, IH, IW, IC, OC, FH, FW, stride[0], stride[1],
                                          padding[0], padding[1])
    if rc:
        raise ValueError("oracle_conv2d_bwd_filter: bad arguments")
    return dW


def conv2d_bwd_filter_at(X, dY, kernel_hw, flat_idx, stride=(1, 1), padding=(1, 1)):
    """O3 at selected flat indices of dW[OC,FH,FW,IC] (float64), full reduction over the batch —
    for full-size parity on sampled outputs; equals conv2d_bwd_filter(...).ravel()[flat_idx]."""
    X, xp = _f32(X)
    dY, dyp = _f32(dY)
    N, IH, IW, IC = X.shape
    N2, OH, OW, OC = dY.shape
    assert N == N2
    FH, FW = kernel_hw
    if out_hw(IH, IW, FH, FW, stride[0], stride[1], padding[0], padding[1]) != (OH, OW):
        raise ValueError("dY extent does not match the forward output")
    idx = np.ascontiguousarray(flat_idx, dtype=np.int64)
    out = np.empty(idx.shape[0], np.float64)
    rc = _load().oracle_conv2d_bwd_filter_at(xp, dyp, idx.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)),
                                             int(idx.shape[0]), out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                             N, IH, IW, IC, OC, FH, FW, stride[0], stride[1],
                                             padding[0], padding[1])
    if rc:
        raise ValueError("oracle_conv2d_bwd_filter_at: bad arguments")
    return out


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def set_num_threads(n: int) -> None:
    _load().oracle_set_num_threads(int(n))


# ---------------------------------------------------------------- net_oracle.c
def _f64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def matmul(A, B, ta=False, tb=False):
    """C = op(A) . op(B) in float64 (net_oracle.c oracle_matmul).  A is [M,K] ([K,M] if ta: matMulT1),
    B is [K,N] ([N,K] if tb: matMulT2)."""
    A, ap = _f32(A)
    B, bp = _f32(B)
    M, K = (A.shape[1], A.shape[0]) if ta else A.shape
    N, K2 = (B.shape[0], B.shape[1]) if tb else (B.shape[1], B.shape[0])
    if K != K2:
        raise ValueError("inner dimensions differ: %d vs %d" % (K, K2))
    C = np.empty((M, N), np.float64)
    if _load().oracle_matmul(ap, bp, C.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), M, N, K, int(ta), int(tb)):
        raise ValueError("oracle_matmul: bad arguments")
    return C


def channel_stats(Y):
    """(sum, sum of squares) per channel (last axis) over all other axes, float64."""
    Y, yp = _f64(Y)
    C = Y.shape[-1]
    rows = Y.size // C
    s1, s2 = np.empty(C), np.empty(C)
    if _load().oracle_channel_stats(yp, rows, C, s1.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                    s2.ctypes.data_as(ctypes.POINTER(ctypes.c_double))):
        raise ValueError("oracle_channel_stats: bad arguments")
    return s1, s2


def leaky_relu(X, k=0.01):
    X, xp = _f64(X)
    Y = np.empty_like(X)
    if _load().oracle_leaky_relu(xp, Y.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), X.size, float(k)):
        raise ValueError("oracle_leaky_relu: bad arguments")
    return Y


def leaky_bwd_stats(dA, A, k=0.01):
    """(G, S1, S2): G = dA * leaky'(A) (from the output A), S1 = sum G, S2 = sum G * leaky^-1(A) per channel."""
    dA, dap = _f64(dA)
    A, ap = _f32(A)
    assert dA.shape == A.shape
    C = A.shape[-1]
    rows = A.size // C
    G = np.empty_like(dA)
    s1, s2 = np.empty(C), np.empty(C)
    dp = ctypes.POINTER(ctypes.c_double)
    if _load().oracle_leaky_bwd_stats(dap, ap, rows, C, float(k), G.ctypes.data_as(dp), s1.ctypes.data_as(dp),
                                      s2.ctypes.data_as(dp)):
        raise ValueError("oracle_leaky_bwd_stats: bad arguments")
    return G, s1, s2
