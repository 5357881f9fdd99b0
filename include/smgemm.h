/*
 * smgemm.h — the paper's matrix-multiply operators on the same sm_100a library (libsmconv.so).
 *
 * "In Alpha, the matrix-multiply and convolution\deconvolution (conv\deconv) operators are highly
 * optimized.  The last dimension of tensors is transparently padded to 4x" (§II);
 * Fig. 3 submits "opt3_{matMulT1}" next to a conv3D; the fully connected layer
 * nn.fullconnect is a matMul.  SPEC.md:94-101 (gemm): c[i,j] = sum_k a'[i,k] b[k,j],
 * "transpose_a=true corresponds to matMulT1".
 *
 *   gemm_matmul     C[M][N] = A[M][K] . B[K][N]          (FC forward X.W;  T1 = A^T, T2 = B^T)
 *   gemm_matmul_t1  C[M][N] = A[K][M]^T . B[K][N]        (FC weight gradient X^T.dY)
 *   gemm_matmul_t2  C[M][N] = A[M][K] . B[N][K]^T        (FC input gradient dY.W^T)
 *
 * All matrices are dense row-major fp32 DEVICE buffers, 16-byte aligned, owned by the caller; C is
 * overwritten.  The row length of every operand must be a multiple of 4 (the paper's padding rule):
 * matMul needs K % 4 == N % 4 == 0, matMulT1 M % 4 == N % 4 == 0, matMulT2 K % 4 == N % 4 == 0
 * (else CONV_EALIGN).  Each call runs as a 1x1 convolution on a 1x1 map (rows = "pixels"):
 * matMul = conv2d_bwd_data, matMulT1 = conv2d_bwd_filter, matMulT2 = conv2d_fwd, so the math
 * modes, determinism, stream semantics, workspace rule and error codes are those of smconv.h
 * (CONV_* codes; conv2d_last_error_detail() names the gemm entry point).
 */
#ifndef SMGEMM_H
#define SMGEMM_H

#include <stddef.h>

#include "smconv.h"

#ifdef __cplusplus
extern "C" {
#endif

enum { GEMM_OP_MATMUL = 0, GEMM_OP_MATMUL_T1 = 1, GEMM_OP_MATMUL_T2 = 2 };

/* Device workspace bytes the call needs (split-K partials); (size_t)-1 for invalid arguments. */
size_t gemm_workspace_bytes(int gemm_op, int M, int N, int K, int math);

int gemm_matmul(const float* A, const float* B, float* C, int M, int N, int K, int math, void* workspace,
                size_t workspace_bytes, conv_stream_t stream);
int gemm_matmul_t1(const float* A, const float* B, float* C, int M, int N, int K, int math, void* workspace,
                   size_t workspace_bytes, conv_stream_t stream);
int gemm_matmul_t2(const float* A, const float* B, float* C, int M, int N, int K, int math, void* workspace,
                   size_t workspace_bytes, conv_stream_t stream);

/* Test hook: the plan the call would run (variant, tile width, splits), like conv2d_plan_describe. */
int gemm_plan_describe(int gemm_op, int M, int N, int K, int math, char* buf, size_t len);

#ifdef __cplusplus
}
#endif

#endif
