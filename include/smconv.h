/*
 * smconv.h — C ABI of the B200-native (sm_100a) small-feature-map fp32 convolution
 * library built for the hot path of arXiv 2305.08819 (Dragon-Alpha & cu32).
 *
 * The paper's native library cu32 "takes the most effort to optimize the
 * conv\deconv operators, especially for 'big channel and small feature maps'"
 * (§III Layer-1) and reaches them through a primitive layer that
 * takes "numerous" parameters and "64bit-addresses".  This
 * header is that primitive layer for the three operators of the path:
 *
 *   conv2d_fwd         Y  = X (*) W            (Fig. 2 nn.conv3D at P:42;
 *                                               SPEC.md:104-112)
 *   conv2d_bwd_data    dX = dY (*)^T W  ("deconv")
 *   conv2d_bwd_filter  dW = X^T (*) dY         ("find gradients")
 *
 * Every entry point takes the conv tuple (N,IH,IW,IC,OC,FH,FW,sh,sw,ph,pw)
 * exactly as BASELINE.json's north_star states the operators.
 *
 * Layouts ("[N, H, W, C]"; SPEC.md:104 filter [out_c,kh,kw,in_c]):
 *   X, dX : dense NHWC float32  [N][IH][IW][IC]
 *   Y, dY : dense NHWC float32  [N][OH][OW][OC],  OH = floor((IH+2ph-FH)/sh)+1 (reading L1)
 *   W, dW : dense OHWI float32  [OC][FH][FW][IC]
 *   IC % 4 == 0 and OC % 4 == 0 ("the last dimension of tensors is transparently
 *   padded to 4x ... using 128bit as the minimum unit of memory-access");
 *   a logical channel count of 3 is zero-padded to 4 by the caller.  Pad lanes of
 *   inputs must be zero; pad lanes of dX / dW then come out zero.
 *
 * Semantics: cross-correlation (no kernel flip); symmetric zero
 * padding (one pad per axis); dX has the forward input's extent
 * (IH,IW) given explicitly, positions no tap reaches are written 0 (reading L5);
 * all three outputs are OVERWRITTEN (reading L6).
 *
 * Pointers: X, W, dY, Y, dX, dW and workspace are DEVICE pointers (cudaMalloc /
 * torch CUDA storage) on the current device, 16-byte aligned.  The caller owns
 * every buffer; the library never allocates on the call path.  Outputs must not
 * overlap inputs (CONV_EALIAS).
 *
 * Streams: each call validates synchronously, then enqueues its kernels on
 * `stream` and returns (the paper's async mode).  Validation
 * errors return before any launch; a failed launch returns CONV_ECUDA.  Device
 * faults surface at the caller's next synchronisation.  If the calling thread already has a
 * CUDA error pending (cudaPeekAtLastError() != cudaSuccess) the call returns CONV_ECUDA
 * without enqueuing anything and WITHOUT clearing that error (it is the caller's to handle).
 *
 * Math modes (north_star (b)):
 *   CONV_MATH_FP32_3XTF32  fp32-accurate (normwise error <= 1e-5 against the fp64 definition, the
 *                          north_star bar; measured margins in profiles/r02_parity_errors.json).
 *                          Each operand is split a = a_hi + a_lo: a_hi = trunc_tf32(a) (the tensor
 *                          core's own operand read) and a_lo = a - a_hi exactly in fp32 on the TMA /
 *                          STRIP / DWS variants; a_hi = rna_tf32(a), a_lo = rna_tf32(a - a_hi) on the
 *                          GENERIC variant.  The a_lo*b_lo term (~2^-22 relative) is dropped.
 *                          Products per k-step:
 *                          - dW on the STEM / GENERIC variants, the transposed-GEMM dW (OC <= 64)
 *                            and every op on the GENERIC variant: three TF32 MMAs,
 *                            a_lo*b_hi + a_hi*b_lo + a_hi*b_hi (strict 3xTF32);
 *                          - fwd / dX on the TMA and STRIP variants (the default for 32x-channel
 *                            layers) and dW on the TMA (OC > 64) and DWS variants (SMCONV_DW_HYB=0 /
 *                            SMCONV_DWS_HYB=0 restore three TF32 MMAs there; plan text "hybw"):
 *                            one TF32 MMA a_hi*b_hi plus ONE bf16 MMA of doubled K computing
 *                            [bf16(a_hi) | bf16(a_lo)] . [bf16(b_lo) | bf16(b)] = the two cross terms
 *                            (+ a_lo*b_lo) with each cross term rounded to bf16 (<= 2^-9 relative on a
 *                            term <= 2^-10 of |a||b|, i.e. ~2^-19 of |a||b| per product, random sign),
 *                            against ~2^-22 for strict 3xTF32.  "3xtf32+bf16x" in reports.
 *                          Accumulation: TMEM chunks of <= 8 k-blocks promoted into fp32 registers
 *                          with round-to-nearest; split-K partials summed in a fixed order.
 *   CONV_MATH_TF32         one TF32 product per term (operands truncated by the tensor core),
 *                          reported separately (normwise <= 5e-3).
 *
 * Determinism: for a fixed (shape, math, plan) results are bitwise reproducible —
 * no floating-point atomics; split-K partials are summed in a fixed order.
 *
 * Errors never print and never abort; conv2d_last_error_detail() returns a
 * thread-local message naming the operator, the argument and the violated
 * constraint.
 */
#ifndef SMCONV_H
#define SMCONV_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    CONV_OK = 0,
    CONV_EARG = 1,         /* non-positive dim/stride, negative pad, OH/OW < 1, bad math/op */
    CONV_EALIGN = 2,       /* IC or OC not a multiple of 4, pointer not 16-B aligned */
    CONV_EALIAS = 3,       /* an output buffer overlaps an input buffer */
    CONV_EWORKSPACE = 4,   /* workspace NULL or smaller than conv2d_workspace_bytes() */
    CONV_EUNSUPPORTED = 5, /* outside the library's limits (tensor >= 2^31 elements, sh*sw > 16,
                              FH*FW > 256) */
    CONV_ECUDA = 6         /* a CUDA runtime/driver call failed (launch error) */
};

enum { CONV_MATH_FP32_3XTF32 = 0, CONV_MATH_TF32 = 1 };
enum { CONV_OP_FWD = 0, CONV_OP_BWD_DATA = 1, CONV_OP_BWD_FILTER = 2 };

/* cudaStream_t without including CUDA headers: pass a cudaStream_t (0 = legacy default). */
typedef void* conv_stream_t;

/* Output extent, reading L1: OH = floor((IH+2ph-FH)/sh)+1.  Returns CONV_EARG if any
 * argument is out of range or OH/OW < 1; OH/OW untouched then.  Host only. */
int conv2d_out_hw(int IH, int IW, int FH, int FW, int sh, int sw, int ph, int pw,
                  int* OH, int* OW);

/* Bytes of device workspace the call with these arguments needs (split-K partials).
 * 0 means workspace may be NULL.  Returns (size_t)-1 for invalid arguments. */
size_t conv2d_workspace_bytes(int op, int N, int IH, int IW, int IC, int OC, int FH, int FW,
                              int sh, int sw, int ph, int pw, int math);

/* Y[N,OH,OW,OC] = sum_{fh,fw,ic} X[N, oh*sh-ph+fh, ow*sw-pw+fw, ic] * W[oc,fh,fw,ic]. */
int conv2d_fwd(const float* X, const float* W, float* Y,
               int N, int IH, int IW, int IC, int OC, int FH, int FW,
               int sh, int sw, int ph, int pw,
               int math, void* workspace, size_t workspace_bytes, conv_stream_t stream);

/* Deconvolution (input gradient):
 * dX[n,ih,iw,ic] = sum over (fh,fw,oc) with ih+ph-fh = oh*sh, iw+pw-fw = ow*sw,
 *                  0<=oh<OH, 0<=ow<OW of dY[n,oh,ow,oc] * W[oc,fh,fw,ic]. */
int conv2d_bwd_data(const float* dY, const float* W, float* dX,
                    int N, int IH, int IW, int IC, int OC, int FH, int FW,
                    int sh, int sw, int ph, int pw,
                    int math, void* workspace, size_t workspace_bytes, conv_stream_t stream);

/* Weight gradient: dW[oc,fh,fw,ic] = sum_{n,oh,ow} dY[n,oh,ow,oc] * X[n, oh*sh-ph+fh, ow*sw-pw+fw, ic]. */
int conv2d_bwd_filter(const float* X, const float* dY, float* dW,
                      int N, int IH, int IW, int IC, int OC, int FH, int FW,
                      int sh, int sw, int ph, int pw,
                      int math, void* workspace, size_t workspace_bytes, conv_stream_t stream);

/* Name of a status code ("CONV_OK", ...).  Never NULL. */
const char* conv2d_strerror(int code);

/* Thread-local detail of the last non-OK status returned on this thread ("" if none). */
const char* conv2d_last_error_detail(void);

#ifdef __cplusplus
}
#endif
#endif /* SMCONV_H */
