/*
 * net_oracle.c — TEST INFRASTRUCTURE ONLY (same rules as conv_oracle.c: only tests/,
 * __graft_entry__.smoke() and bench.py's oracle legs load it; it shares nothing with the CUDA path).
 *
 * Plain definitions of the operators next to the convolutions on the paper's network path
 * (SURVEY.md §8(f) rows 2 and 4), written out as loops with double accumulation:
 *
 *   oracle_matmul            C = op(A) . op(B)  — the paper's matrix-multiply operators
 *                            ("the matrix-multiply and convolution\deconvolution
 *                            (conv\deconv) operators are highly optimized"; Fig. 3
 *                            "opt3_{matMulT1}"; SPEC.md:94-101 gemm, "transpose_a=true corresponds
 *                            to matMulT1"; the FC layer nn.fullconnect).
 *   oracle_channel_stats     per-channel sum and sum of squares over the N*H*W rows of an NHWC
 *                            tensor — the batch statistics of the BatchNorm that follows every conv
 *                            in the paper's blocks ("F.leakyRelu(bn1.forward(conv1.
 *                            forward(X)))", PAPER.md:184 BatchNorm eps = 1e-8
 *                            "per-channel batch mean and biased variance over N*H*W elements").
 *   oracle_leaky_relu        y = x if x > 0 else k*x (PAPER.md:52,55,68 F.leakyRelu).
 *   oracle_leaky_bwd_stats   the backward of leakyRelu(BN(.)) as far as a conv's dX epilogue can
 *                            take it: g = dA * (1 if A > 0 else k) ("computed from the
 *                            output (invertible sign)"), z = A if A > 0 else A / k (the BN output
 *                            the activation was computed from), and per channel S1 = sum g,
 *                            S2 = sum g*z — from which the BN parameter gradients are
 *                            dbeta = S1 and dgamma = sum g*xhat = (S2 - beta*S1) / gamma
 *                            (SPEC.md:144-147 batchnorm_backward: dbeta = sum dy, dgamma = sum dy*xhat).
 *
 * Summation order is the row order n, h, w (rows = N*H*W, channel fastest in memory), fixed.
 */
#include <stddef.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_EARG 1

/*
 * C[i][j] = sum_{k<K} a(i,k) * b(k,j),  i < M, j < N, k in increasing order, double accumulation
 * (fp32 x fp32 products are exact in double).
 *   a(i,k) = A[i*K + k]  (A stored [M][K], ta = 0)   or A[k*M + i]  (A stored [K][M], ta = 1: matMulT1)
 *   b(k,j) = B[k*N + j]  (B stored [K][N], tb = 0)   or B[j*K + k]  (B stored [N][K], tb = 1: matMulT2)
 */
int oracle_matmul(const float* A, const float* B, double* C, int M, int N, int K, int ta, int tb) {
    if (M < 1 || N < 1 || K < 1) return ORACLE_EARG;
#pragma omp parallel for schedule(static)
    for (long long e = 0; e < (long long)M * N; ++e) {
        const long long i = e / N, j = e % N;
        double s = 0.0;
        for (long long k = 0; k < K; ++k) {
            const double a = ta ? A[k * M + i] : A[i * K + k];
            const double b = tb ? B[j * K + k] : B[k * N + j];
            s += a * b;
        }
        C[e] = s;
    }
    return ORACLE_OK;
}

/* S1[c] = sum_r Y[r*C + c],  S2[c] = sum_r Y[r*C + c]^2,  r < rows (= N*H*W), in row order. */
int oracle_channel_stats(const double* Y, long long rows, int C, double* S1, double* S2) {
    if (rows < 0 || C < 1) return ORACLE_EARG;
#pragma omp parallel for schedule(static)
    for (int c = 0; c < C; ++c) {
        double s = 0.0, q = 0.0;
        for (long long r = 0; r < rows; ++r) {
            const double y = Y[r * C + c];
            s += y;
            q += y * y;
        }
        S1[c] = s;
        S2[c] = q;
    }
    return ORACLE_OK;
}

/* Y[i] = X[i] if X[i] > 0 else k * X[i] */
int oracle_leaky_relu(const double* X, double* Y, long long n, double k) {
    if (n < 0) return ORACLE_EARG;
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < n; ++i) Y[i] = X[i] > 0.0 ? X[i] : k * X[i];
    return ORACLE_OK;
}

/*
 * G[r,c]  = dA[r,c] * (1 if A[r,c] > 0 else k)           (leakyRelu backward, from the output)
 * S1[c]   = sum_r G[r,c]
 * S2[c]   = sum_r G[r,c] * z[r,c],  z = A if A > 0 else A / k   (the activation's input)
 * k > 0 (an invertible slope).  Rows in order.
 */
int oracle_leaky_bwd_stats(const double* dA, const float* A, long long rows, int C, double k, double* G, double* S1,
                           double* S2) {
    if (rows < 0 || C < 1 || !(k > 0.0)) return ORACLE_EARG;
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < rows * C; ++i) {
        const double a = A[i];
        G[i] = a > 0.0 ? dA[i] : k * dA[i];
    }
#pragma omp parallel for schedule(static)
    for (int c = 0; c < C; ++c) {
        double s = 0.0, q = 0.0;
        for (long long r = 0; r < rows; ++r) {
            const double a = A[r * C + c];
            const double z = a > 0.0 ? a : a / k;
            s += G[r * C + c];
            q += G[r * C + c] * z;
        }
        S1[c] = s;
        S2[c] = q;
    }
    return ORACLE_OK;
}
