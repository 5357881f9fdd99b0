/*
 * smconv_epi.h — convolutions with fused epilogues from the paper's network vocabulary
 * (SURVEY.md §8(f) row 2), on the same sm_100a library (libsmconv.so).
 *
 * The paper's block is  X = F.leakyRelu(bn1.forward(conv1.forward(X))),
 * with in-place BatchNorm (eps = 1e-8) and LeakyReLU
 * y = x if x > 0 else k*x.  A conv kernel can take over, without changing the conv:
 *
 *   conv2d_fwd_epi(..., epi = CONV_EPI_BN_STATS, stats)  Y = conv(X, W) exactly as conv2d_fwd, and
 *       stats[c] = S1[c] = sum_{n,oh,ow} Y[n,oh,ow,c],  stats[OC + c] = S2[c] = sum Y[n,oh,ow,c]^2
 *       — the BatchNorm batch statistics (mean = S1/M, biased var = S2/M - mean^2 with M = N*OH*OW;
 *       SPEC.md:134-137), so BN needs no separate pass over Y.
 *   conv2d_fwd_epi(..., epi = CONV_EPI_LEAKY, k)          Y = leakyRelu_k(conv(X, W)).
 *   conv2d_bwd_data_epi(..., epi = CONV_EPI_LEAKY_BWD, A, k)
 *       G = dX * (1 if A > 0 else k), dX = conv2d_bwd_data(dY, W): the deconvolution's output is the
 *       gradient w.r.t. A = leakyRelu_k(Z), the forward input of this conv; G = dL/dZ (the slope is
 *       read from the output A: "invertible sign").
 *   conv2d_bwd_data_epi(..., epi = CONV_EPI_LEAKY_BWD_STATS, A, k, stats)
 *       G as above, plus stats[c] = S1[c] = sum G[...,c] and stats[IC + c] = S2[c] = sum G*z with
 *       z = A if A > 0 else A / k (the BN output): dbeta = S1, dgamma = (S2 - beta*S1) / gamma
 *       (SPEC.md:144-147 batchnorm_backward).
 *
 * Arguments: as conv2d_fwd / conv2d_bwd_data (smconv.h: DEVICE pointers, NHWC, [OC,FH,FW,IC],
 * 16-byte alignment, caller-owned buffers, stream semantics, CONV_* error codes), plus
 *   epi    CONV_EPI_* (fwd: NONE, BN_STATS, LEAKY; dX: NONE, LEAKY_BWD, LEAKY_BWD_STATS; else CONV_EARG)
 *   k      the LeakyReLU slope, finite and > 0 for the LEAKY modes (CONV_EARG otherwise); ignored else
 *   A      dX only, LEAKY_BWD modes: the activation [N,IH,IW,IC] (device, 16-B aligned).  It may be the
 *          SAME buffer as dX (in-place, "calculate gradients directly on the memory-space
 *          of the precursors": each element of A is read before the thread that owns it writes G
 *          there); any other overlap with dX, and any overlap with dY / W, is CONV_EALIAS
 *   stats  the stats modes: 2*C doubles (C = OC for fwd, IC for dX), device, 8-byte aligned,
 *          overwritten; NULL otherwise
 * The workspace is conv2d_epi_workspace_bytes(...) (>= conv2d_workspace_bytes of the same conv).
 *
 * Where the plan's main kernel writes final values (TMA / STRIP variants without split-K) the
 * transform and the statistics run in its epilogue warps (warp-shuffle column sums of 32 output
 * rows); otherwise one extra pass over the output applies them.  The per-32-row partial sums are
 * added in a FIXED order in double: the results are bitwise reproducible.  Accuracy: Y / G as the
 * plain ops (normwise 1e-5 in 3xTF32, 5e-3 in TF32); S1, S2 are the sums of the stored fp32 values
 * (32-row fp32 partials, then double).
 */
#ifndef SMCONV_EPI_H
#define SMCONV_EPI_H

#include <stddef.h>

#include "smconv.h"

#ifdef __cplusplus
extern "C" {
#endif

enum {
    CONV_EPI_NONE = 0,
    CONV_EPI_BN_STATS = 1,
    CONV_EPI_LEAKY = 2,
    CONV_EPI_LEAKY_BWD = 3,
    CONV_EPI_LEAKY_BWD_STATS = 4
};

/* Device workspace bytes of a fused-epilogue call; (size_t)-1 for invalid arguments. */
size_t conv2d_epi_workspace_bytes(int op, int N, int IH, int IW, int IC, int OC, int FH, int FW, int sh, int sw,
                                  int ph, int pw, int math, int epi);

int conv2d_fwd_epi(const float* X, const float* W, float* Y, double* stats, int N, int IH, int IW, int IC, int OC,
                   int FH, int FW, int sh, int sw, int ph, int pw, int math, int epi, float k, void* workspace,
                   size_t workspace_bytes, conv_stream_t stream);

int conv2d_bwd_data_epi(const float* dY, const float* W, const float* A, float* dX, double* stats, int N, int IH,
                        int IW, int IC, int OC, int FH, int FW, int sh, int sw, int ph, int pw, int math, int epi,
                        float k, void* workspace, size_t workspace_bytes, conv_stream_t stream);

/* Test hook: the plan as text, with "epi=fused" (in the conv kernel's epilogue) or "epi=pass". */
int conv2d_epi_plan_describe(int op, int N, int IH, int IW, int IC, int OC, int FH, int FW, int sh, int sw, int ph,
                             int pw, int math, int epi, char* buf, size_t len);

#ifdef __cplusplus
}
#endif

#endif
