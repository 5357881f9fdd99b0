// epilogue.cuh — fused conv epilogues from the paper's network vocabulary.
//
// The paper's building block is `F.leakyRelu(bn1.forward(conv1.forward(X)))` (PAPER.md:52, :55,
// :67-68) with an in-place BatchNorm (eps = 1e-8).  What a conv kernel
// can take over from the layers around it, without changing what the conv computes:
//
//   CONV_EPI_BN_STATS        (fwd)  Y as usual, plus the per-channel batch statistics of Y that the
//                                   BatchNorm needs: S1[c] = sum y, S2[c] = sum y^2 over the N*OH*OW
//                                   rows ("per-channel batch mean and biased variance")
//   CONV_EPI_LEAKY           (fwd)  Y = leakyRelu(conv(X)) (y = x if x > 0 else k x)
//   CONV_EPI_LEAKY_BWD       (dX)   G = dX * (1 if A > 0 else k): the deconvolution's output is the
//                                   gradient of A = leakyRelu(Z) (the next conv's input); G = dL/dZ
//                                   ("computed from the output (invertible sign)")
//   CONV_EPI_LEAKY_BWD_STATS (dX)   G as above plus S1[c] = sum G, S2[c] = sum G*z with
//                                   z = A if A > 0 else A / k (the BN output), from which
//                                   dbeta = S1, dgamma = (S2 - beta S1) / gamma
//
// Where the conv kernel writes final values (TMA / STRIP variants, no split-K) the transform and the
// statistics run in its epilogue warps ("fused"): each warp holds 32 output rows (TMEM lanes) of 16
// consecutive columns at a time; the column sums over its 32 rows are a warp-shuffle reduce-scatter
// (north_star (d)), written as one fp32 partial row per 32-row group into the workspace.  Otherwise
// (split-K, in-cluster split-K, GENERIC, DIRECT) `epi_pass_kernel` applies the same transform to the
// finished output and writes the same partial rows ("pass").  Two small kernels then sum
// the partial rows in a FIXED order in double (deterministic, SURVEY.md §8(b) contract 6).
#pragma once
#include "common.cuh"

namespace smconv {

enum { EPI_NONE = 0, EPI_BN_STATS = 1, EPI_LEAKY = 2, EPI_LEAKY_BWD = 3, EPI_LEAKY_BWD_STATS = 4 };

SMCONV_HD bool epi_has_stats(int e) { return e == EPI_BN_STATS || e == EPI_LEAKY_BWD_STATS; }
SMCONV_HD bool epi_reads_a(int e) { return e == EPI_LEAKY_BWD || e == EPI_LEAKY_BWD_STATS; }

// Column sums over the 32 lanes (= 32 output rows) of a warp for 16 columns held by every lane:
// a butterfly reduce-scatter (16 shuffles for 16 columns).  On return lane l holds the sum over all
// 32 lanes of column (l & 15).  Fixed combination order: deterministic.  v is destroyed.
SMCONV_DEV float warp_colsum16(float (&v)[16], int lane) {
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const float send = up ? v[i] : v[i + o];
            const float keep = up ? v[i + o] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
}

struct EpiArgs {
    int mode;          // EPI_*
    float k;           // leaky slope (> 0)
    const float* A;    // LEAKY_BWD*: the activation A, same layout and addresses as the output
    float* part;       // stats: fp32 partial rows [2][ngroups][ncols]
    int ngroups;       // 32-row groups of the output rows
    int ncols;         // GEMM columns (= channels, or 4 * IC for the super-pixel dX)
};

// Warp-collective: 16 consecutive columns col0..col0+15 (col0 uniform across the warp) of this lane's
// output row.  `addr` = element offset of column col0 of this row in the output tensor, or -1 when the
// row is not an output row (ragged tile rows, dropped super-pixel rows): its values are ignored.
// Transforms v in place (LEAKY: y -> leaky(y); LEAKY_BWD*: dx -> dx * slope(A[addr])) and, in the
// stats modes, writes the 16 column sums of the warp's 32 rows to partial row `grp`.
// `ncols_valid` bounds the columns (a ragged last n-tile).
// Inlined (an out-of-line call passes v through local memory: 576 threads x ~300-B stack frames do not
// fit L1, and the fused ResNet step went 53.7 -> 78 ms, r02bf).  Code size: the kernels keep ONE
// unrolled column loop that calls it (the row-coalesced store path; conv_tma.cuh), since every inlined
// copy is ~1.3k SASS instructions and a cold instruction cache stalls the short small-map calls
// (ncu r02be, VGG conv11: stall_no_inst 39 % of the samples).
SMCONV_DEV void epi_apply16(const EpiArgs& e, float (&v)[16], long long addr, int col0, int ncols_valid, int grp,
                            int lane) {
    const bool row_ok = addr >= 0;
    float s2[16];
    if (e.mode == EPI_LEAKY) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = v[i] > 0.f ? v[i] : e.k * v[i];
        return;
    }
    if (e.mode == EPI_LEAKY_BWD || e.mode == EPI_LEAKY_BWD_STATS) {
        const float rk = 1.0f / e.k;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
            if (row_ok && col0 + 4 * q < ncols_valid) a = *reinterpret_cast<const float4*>(e.A + addr + 4 * q);
            const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int i = 4 * q + j;
                const bool pos = av[j] > 0.f;
                v[i] = pos ? v[i] : e.k * v[i];
                s2[i] = v[i] * (pos ? av[j] : av[j] * rk);  // g * z
            }
        }
    } else {  // BN_STATS
#pragma unroll
        for (int i = 0; i < 16; ++i) s2[i] = v[i] * v[i];
    }
    if (!epi_has_stats(e.mode)) return;
    float s1[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        s1[i] = row_ok ? v[i] : 0.f;
        s2[i] = row_ok ? s2[i] : 0.f;
    }
    const float t1 = warp_colsum16(s1, lane);
    const float t2 = warp_colsum16(s2, lane);
    const int col = col0 + (lane & 15);
    if (lane < 16 && col < ncols_valid && grp >= 0 && grp < e.ngroups) {
        e.part[(long long)grp * e.ncols + col] = t1;
        e.part[((long long)e.ngroups + grp) * e.ncols + col] = t2;
    }
}

// "pass" form: the conv output `src` [rows][C] is final; apply the transform and write it to `out`
// (src == out, in place, for the fwd modes; a workspace staging buffer for the LEAKY_BWD modes, so that
// A may alias `out`), and write the partial rows.  One warp per (32-row group, 16-column chunk) work
// item; lane = row, as in the fused epilogue (so both forms produce the same partial-row layout).
template <int UNUSED = 0>
__global__ void __launch_bounds__(256) epi_pass_kernel(const float* src, float* out, long long rows, int C,
                                                       EpiArgs e) {
    pdl_trigger();
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    const int chunks = (C + 15) / 16;
    const long long items = (long long)e.ngroups * chunks;
    for (long long it = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); it < items; it += warps) {
        const int grp = (int)(it / chunks), ch = (int)(it - (long long)grp * chunks);
        const long long r = (long long)grp * 32 + lane;
        const int col0 = ch * 16;
        const long long addr = r < rows ? r * C + col0 : -1;
        float v[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
            if (addr >= 0 && col0 + 4 * q < C) x = *reinterpret_cast<const float4*>(src + addr + 4 * q);
            v[4 * q] = x.x;
            v[4 * q + 1] = x.y;
            v[4 * q + 2] = x.z;
            v[4 * q + 3] = x.w;
        }
        epi_apply16(e, v, addr, col0, C, grp, lane);
        if ((e.mode != EPI_BN_STATS || src != out) && addr >= 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (col0 + 4 * q < C)
                    *reinterpret_cast<float4*>(out + addr + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
    }
}

// Statistics, stage 1: chunk c of the partial rows, column j: part2[c][s][j] = sum over the chunk's
// rows in increasing order (double).  Stage 2: out[s][ch] = sum over chunks c in order, then over the
// columns j == ch (mod C) in increasing j (the super-pixel dX's 4 phase column groups fold onto IC).
template <int UNUSED = 0>
__global__ void __launch_bounds__(256) epi_stats_stage1(const float* __restrict__ part, double* __restrict__ part2,
                                                        int ngroups, int ncols, int nchunks) {
    pdl_trigger();
    pdl_wait();
    const int per = (ngroups + nchunks - 1) / nchunks;
    const long long n = 2LL * nchunks * ncols;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int j = (int)(i % ncols);
        const long long q = i / ncols;
        const int s = (int)(q % 2), c = (int)(q / 2);
        const int g0 = c * per, g1 = min(ngroups, g0 + per);
        const float* p = part + ((long long)s * ngroups) * ncols + j;
        double acc = 0.0;
        int g = g0;
        for (; g + 4 <= g1; g += 4) {  // 4 independent loads in flight; added in order
            const float a0 = p[(long long)g * ncols], a1 = p[(long long)(g + 1) * ncols];
            const float a2 = p[(long long)(g + 2) * ncols], a3 = p[(long long)(g + 3) * ncols];
            acc += a0;
            acc += a1;
            acc += a2;
            acc += a3;
        }
        for (; g < g1; ++g) acc += p[(long long)g * ncols];
        part2[((long long)c * 2 + s) * ncols + j] = acc;
    }
}

template <int UNUSED = 0>
__global__ void __launch_bounds__(256) epi_stats_stage2(const double* __restrict__ part2, double* __restrict__ stats,
                                                        int ncols, int nchunks, int C) {
    pdl_trigger();
    pdl_wait();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * C; i += gridDim.x * blockDim.x) {
        const int s = i / C, ch = i - s * C;
        double acc = 0.0;
        for (int j = ch; j < ncols; j += C)
            for (int c = 0; c < nchunks; ++c) acc += part2[((long long)c * 2 + s) * ncols + j];
        stats[i] = acc;
    }
}

}  // namespace smconv
