// conv_direct.cu — DIRECT variant: CUDA-core fp32 direct convolution for few-channel inputs
// (the IC = 3 -> 4 padded RGB stems), fwd and dW.
//
// A stem has K = FH*FW*IC = 36 and arithmetic intensity ~16 FLOP/B: it is HBM-bound (Y resp. dY,
// 1 GB at batch 4096, dominates the traffic), so it is NOT reshaped into tensor-core GEMMs (their
// 128-row tiles would be 90% padding at K = 36).  Plain fp32 FMA with register tiles, inputs
// staged through shared memory, outputs / dY streamed with coalesced 16-B accesses; exact fp32
// products (more accurate than 3xTF32), deterministic (dW partials reduced in a fixed order by
// the split-K reduction kernel).
#include <cstdio>
#include <cstdlib>

#include "../../include/smconv.h"
#include "launch.cuh"
#include "conv_gen.cuh"

namespace smconv {

constexpr int kDirThreads = 256;
constexpr int kDirOWB = 8;        // fwd: output columns per thread
constexpr int kDirKMax = 128;     // FH*FW*IC limit (W^T in shared memory)
constexpr int kDirOWMax = 64;
constexpr int kDirDwFWIC = 24;    // dW: FW*IC accumulator columns per thread (x 4 oc)

struct DirectParams {
    const float* X;
    const float* W;
    const float* dY;
    float* out;  // fwd: Y; dw: per-block partial dW [blocks][OC][K]
    int N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw, OH, OW;
    int K, WIN;  // FH*FW*IC; input columns touched by one output row
    int rows_per_block;
};

constexpr int kDirNB = 4;  // dW: cp.async row ring depth (3 rows in flight per block; 8 measured slower, r01y)

SMCONV_DEV void cp_async16(uint32_t dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
                 : "memory");
}
SMCONV_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
SMCONV_DEV void cp_async_wait_nb2() { asm volatile("cp.async.wait_group %0;" ::"n"(kDirNB - 2) : "memory"); }
SMCONV_DEV void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// cp.async the FH input rows of output row (n, oh) into Xs[fh][WIN][IC] (padding -> zero fill)
SMCONV_DEV void direct_issue_rows(const DirectParams& p, float* Xs, int n, int oh, int t, int nthreads) {
    const int IC4 = p.IC >> 2;
    const uint32_t base = smem_u32(Xs);
    for (int i = t; i < p.FH * p.WIN * IC4; i += nthreads) {
        const int c4 = i % IC4, r = i / IC4;
        const int col = r % p.WIN, fh = r / p.WIN;
        const int ih = oh * p.sh - p.ph + fh, iw = col - p.pw;
        const bool ok = (unsigned)ih < (unsigned)p.IH && (unsigned)iw < (unsigned)p.IW;
        cp_async16(base + i * 16u, ok ? p.X + (((size_t)n * p.IH + ih) * p.IW + iw) * p.IC + 4 * c4 : p.X, ok);
    }
}

// stage the FH input rows of output row (n, oh) into Xs[fh][WIN][IC] (padding -> zeros)
SMCONV_DEV void direct_load_rows(const DirectParams& p, float* Xs, int n, int oh, int t, int nthreads) {
    const int IC4 = p.IC >> 2;
    for (int i = t; i < p.FH * p.WIN * IC4; i += nthreads) {
        const int c4 = i % IC4, r = i / IC4;
        const int col = r % p.WIN, fh = r / p.WIN;
        const int ih = oh * p.sh - p.ph + fh, iw = col - p.pw;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if ((unsigned)ih < (unsigned)p.IH && (unsigned)iw < (unsigned)p.IW)
            v = ldg_f4(p.X + (((size_t)n * p.IH + ih) * p.IW + iw) * p.IC + 4 * c4);
        reinterpret_cast<float4*>(Xs)[i] = v;
    }
}

// ---------------------------------------------------------------- forward
// thread tile: 8 output columns x 4 output channels; W^T [K][OC] resident in smem per block.
// TFH/TFW/TIC4/TSW: compile-time filter rows/cols, channel quads, column stride (0 = runtime):
// the RGB stem instance <3,3,1,1> is fully unrolled (the runtime-bound loops issued ~2.5 non-FMA
// instructions per FMA: FMA pipe 41 % busy); RAG = ragged last column block (OW % 8 != 0).
template <int TFH, int TFW, int TIC4, int TSW, bool RAG>
__global__ void __launch_bounds__(kDirThreads) conv_direct_fwd_kernel(const __grid_constant__ DirectParams p) {
    extern __shared__ float4 sm4[];
    pdl_trigger();
    pdl_wait();  // launch.cuh
    float* Ws = reinterpret_cast<float*>(sm4);  // [K][OC]
    const int FH = TFH ? TFH : p.FH, FW = TFW ? TFW : p.FW, SW = TSW ? TSW : p.sw;
    const int OC4 = p.OC >> 2, IC4 = TIC4 ? TIC4 : p.IC >> 2;
    const int owblocks = (p.OW + kDirOWB - 1) / kDirOWB;
    const int trow = OC4 * owblocks;                           // threads per output row
    const int rp = trow >= kDirThreads ? 1 : kDirThreads / trow;  // rows in flight per block
    float* Xs0 = Ws + p.K * p.OC;                               // rp x [FH][WIN][IC]
    const int xs_stride = p.FH * p.WIN * p.IC;
    const int t = threadIdx.x;
    for (int i = t; i < p.K * OC4; i += kDirThreads) {  // transpose W[oc][k] -> Ws[k][oc]
        const int oc4 = i % OC4, k = i / OC4;
        float4 w;
        w.x = __ldg(p.W + (size_t)(4 * oc4 + 0) * p.K + k);
        w.y = __ldg(p.W + (size_t)(4 * oc4 + 1) * p.K + k);
        w.z = __ldg(p.W + (size_t)(4 * oc4 + 2) * p.K + k);
        w.w = __ldg(p.W + (size_t)(4 * oc4 + 3) * p.K + k);
        reinterpret_cast<float4*>(Ws)[i] = w;
    }
    const int slot = t / trow, tl = t - slot * trow;
    const int q = tl % OC4, ob = tl / OC4;
    const int rows = p.N * p.OH;
    // double-buffered row groups: group g+1 is cp.async'ed while group g is computed
    auto issue_group = [&](int r0, int b) {
        for (int s = 0; s < rp; ++s)
            if (r0 + s < rows) {
                const int rr = r0 + s, n = rr / p.OH, oh = rr - n * p.OH;
                direct_issue_rows(p, Xs0 + (b * rp + s) * xs_stride, n, oh, t, kDirThreads);
            }
        cp_async_commit();
    };
    int buf = 0;
    if (blockIdx.x * rp < rows) issue_group(blockIdx.x * rp, 0);
    for (int r0 = blockIdx.x * rp; r0 < rows; r0 += gridDim.x * rp) {
        const int nx = r0 + gridDim.x * rp;
        if (nx < rows) issue_group(nx, buf ^ 1);
        else cp_async_commit();
        cp_async_wait_1();
        __syncthreads();
        const int row = r0 + slot;
        if (slot < rp && row < rows && tl < trow) {
            const float* Xs = Xs0 + (buf * rp + slot) * xs_stride;
            float acc[kDirOWB][4];
#pragma unroll
            for (int j = 0; j < kDirOWB; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
            const int ow0 = ob * kDirOWB;
#pragma unroll
            for (int fh = 0; fh < FH; ++fh)
#pragma unroll
                for (int fw = 0; fw < FW; ++fw)
#pragma unroll
                    for (int c4 = 0; c4 < IC4; ++c4) {
                        const int k0 = ((fh * FW + fw) * IC4 + c4) * 4;
                        const float4* wv = reinterpret_cast<const float4*>(Ws) + (size_t)k0 * OC4 + q;
                        const float4 w0 = wv[0], w1 = wv[OC4], w2 = wv[2 * OC4], w3 = wv[3 * OC4];
                        const float4* xv = reinterpret_cast<const float4*>(Xs) + (fh * p.WIN + fw) * IC4 + c4;
#pragma unroll
                        for (int j = 0; j < kDirOWB; ++j) {
                            if (RAG && ow0 + j >= p.OW) break;  // ragged last column block
                            const float4 x = xv[(ow0 + j) * SW * IC4];
                            acc[j][0] = fmaf(x.x, w0.x, fmaf(x.y, w1.x, fmaf(x.z, w2.x, fmaf(x.w, w3.x, acc[j][0]))));
                            acc[j][1] = fmaf(x.x, w0.y, fmaf(x.y, w1.y, fmaf(x.z, w2.y, fmaf(x.w, w3.y, acc[j][1]))));
                            acc[j][2] = fmaf(x.x, w0.z, fmaf(x.y, w1.z, fmaf(x.z, w2.z, fmaf(x.w, w3.z, acc[j][2]))));
                            acc[j][3] = fmaf(x.x, w0.w, fmaf(x.y, w1.w, fmaf(x.z, w2.w, fmaf(x.w, w3.w, acc[j][3]))));
                        }
                    }
            const int n = row / p.OH, oh = row - n * p.OH;
            float* y = p.out + (((size_t)n * p.OH + oh) * p.OW) * p.OC + 4 * q;
#pragma unroll
            for (int j = 0; j < kDirOWB; ++j)
                if (ow0 + j < p.OW)
                    *reinterpret_cast<float4*>(y + (size_t)(ow0 + j) * p.OC) =
                        make_float4(acc[j][0], acc[j][1], acc[j][2], acc[j][3]);
        }
        __syncthreads();  // everyone is done with `buf` before the next group is issued into it
        buf ^= 1;
    }
    cp_async_commit();
    asm volatile("cp.async.wait_all;" ::: "memory");
}

// ---------------------------------------------------------------- weight gradient
// thread = (4-oc quad, filter row fh, pixel partition); accumulates dW[4 oc][fh][FW][IC] over the
// block's (n, oh) rows, partitions summed in fixed order at the end -> per-block partial.
// Rows stream through a 4-deep cp.async ring in smem (3 rows in flight per block): the kernel is
// HBM-streaming (dY is 1 GB at batch 4096) and a one-row-at-a-time loop was latency bound.
template <int ACC4>  // accumulator float4 columns per thread = ceil(FW*IC / 4)
__global__ void __launch_bounds__(kDirThreads) conv_direct_dw_kernel(const __grid_constant__ DirectParams p) {
    extern __shared__ float4 sm4[];
    pdl_trigger();
    pdl_wait();  // launch.cuh
    const int OC4 = p.OC >> 2, IC4 = p.IC >> 2;
    const int nD4 = p.OW * OC4, nX4 = p.FH * p.WIN * IC4, nR4 = nD4 + nX4;  // float4 per row
    float* Red = reinterpret_cast<float*>(sm4 + kDirNB * nR4);
    const uint32_t ring = smem_u32(sm4);
    const int tpp = OC4 * p.FH;  // threads per partition
    const int P = kDirThreads / tpp;
    const int t = threadIdx.x;
    const int part = t / tpp, tl = t - part * tpp;
    const int q = tl % OC4, fh = tl / OC4;
    const int FWIC = p.FW * p.IC;
    float acc[ACC4 * 4][4];
#pragma unroll
    for (int i = 0; i < ACC4 * 4; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    const int r0 = blockIdx.x * p.rows_per_block;
    const int r1 = min(r0 + p.rows_per_block, p.N * p.OH);

    auto issue = [&](int rr, int b) {  // row rr (dY row, then the FH input rows) -> ring buffer b
        const int n = rr / p.OH, oh = rr - n * p.OH;
        const uint32_t base = ring + (uint32_t)(b * nR4) * 16u;
        for (int i = t; i < nR4; i += kDirThreads) {
            if (i < nD4) {
                cp_async16(base + i * 16u, p.dY + ((size_t)n * p.OH + oh) * p.OW * p.OC + 4 * i, true);
            } else {
                const int xi = i - nD4;
                const int c4 = xi % IC4, r = xi / IC4;
                const int col = r % p.WIN, f = r / p.WIN;
                const int ih = oh * p.sh - p.ph + f, iw = col - p.pw;
                const bool ok = (unsigned)ih < (unsigned)p.IH && (unsigned)iw < (unsigned)p.IW;
                cp_async16(base + i * 16u, ok ? p.X + (((size_t)n * p.IH + ih) * p.IW + iw) * p.IC + 4 * c4 : p.X, ok);
            }
        }
    };
#pragma unroll
    for (int d = 0; d < kDirNB - 1; ++d) {
        if (r0 + d < r1) issue(r0 + d, d);
        cp_async_commit();
    }
    for (int rr = r0; rr < r1; ++rr) {
        cp_async_wait_nb2();
        __syncthreads();
        const float4* Ds = sm4 + ((rr - r0) % kDirNB) * nR4;
        const float4* Xs = Ds + nD4;
        if (part < P) {
            for (int ow = part; ow < p.OW; ow += P) {
                const float4 dy = Ds[ow * OC4 + q];
                const float4* xv = Xs + (fh * p.WIN + ow * p.sw) * IC4;
#pragma unroll
                for (int i4 = 0; i4 < ACC4; ++i4) {
                    if (4 * i4 < FWIC) {
                        const float4 x = xv[i4];  // flattened (fw, c) = 4*i4 .. 4*i4+3
                        const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            acc[4 * i4 + e][0] = fmaf(xs[e], dy.x, acc[4 * i4 + e][0]);
                            acc[4 * i4 + e][1] = fmaf(xs[e], dy.y, acc[4 * i4 + e][1]);
                            acc[4 * i4 + e][2] = fmaf(xs[e], dy.z, acc[4 * i4 + e][2]);
                            acc[4 * i4 + e][3] = fmaf(xs[e], dy.w, acc[4 * i4 + e][3]);
                        }
                    }
                }
            }
        }
        __syncthreads();
        const int nxt = rr + kDirNB - 1;
        if (nxt < r1) issue(nxt, (nxt - r0) % kDirNB);
        cp_async_commit();
    }
    // fixed-order reduction over partitions: Red[tl][i][o] = part 0 + part 1 + ...
    float* part_out = p.out + (size_t)blockIdx.x * p.OC * p.K;
    for (int pp = 0; pp < P; ++pp) {
        __syncthreads();
        if (part == pp) {
#pragma unroll
            for (int i = 0; i < ACC4 * 4; ++i)
                if (i < FWIC)
#pragma unroll
                    for (int o = 0; o < 4; ++o) {
                        float* r = Red + ((size_t)tl * ACC4 * 4 + i) * 4 + o;
                        *r = (pp == 0 ? 0.f : *r) + acc[i][o];
                    }
        }
    }
    __syncthreads();
    if (part == 0) {
        for (int i = 0; i < FWIC; ++i)
#pragma unroll
            for (int o = 0; o < 4; ++o)
                part_out[(size_t)(4 * q + o) * p.K + fh * FWIC + i] = Red[((size_t)tl * ACC4 * 4 + i) * 4 + o];
    }
}

// ---------------------------------------------------------------- host side
// Dynamic shared memory of the direct kernels, shared by direct_supported() and direct_launch() so
// that the AUTO heuristic only picks DIRECT when the launch fits (0 = the shape does not fit).
constexpr size_t kDirSmemMax = 200 * 1024;
size_t direct_smem(int op, int IC, int OC, int FH, int FW, int OW, int sw) {
    const int WIN = (OW - 1) * sw + FW;
    const int xs = FH * WIN * IC;
    if (op == CONV_OP_FWD) {
        const int trow = (OC / 4) * ((OW + kDirOWB - 1) / kDirOWB);
        if (trow > kDirThreads) return 0;
        const int rp = trow >= kDirThreads ? 1 : kDirThreads / trow;
        const size_t s = (size_t)(FH * FW * IC * OC + 2 * rp * xs) * sizeof(float);  // W^T + 2 row-group buffers
        return s > kDirSmemMax ? 0 : s;
    }
    const int tpp = (OC / 4) * FH;
    if (tpp > kDirThreads) return 0;
    const int acc4 = (FW * IC + 3) / 4;
    const int nR4 = OW * OC / 4 + xs / 4;
    const size_t s = (size_t)(kDirNB * nR4 * 4 + (size_t)tpp * (acc4 <= 3 ? 3 : 6) * 16) * sizeof(float);
    return s > kDirSmemMax ? 0 : s;
}

bool direct_supported(int op, int IC, int OC, int FH, int FW, int OW, int sw) {
    if (op != CONV_OP_FWD && op != CONV_OP_BWD_FILTER) return false;
    if (IC > 8 || FH * FW * IC > kDirKMax || OW > kDirOWMax) return false;
    if (op == CONV_OP_BWD_FILTER) {
        if (FW * IC > kDirDwFWIC) return false;
        const int WIN = (OW - 1) * sw + FW;
        if ((OW * OC / 4 + FH * WIN * IC / 4) * 16 * kDirNB > 150 * 1024) return false;  // cp.async ring
    }
    return direct_smem(op, IC, OC, FH, FW, OW, sw) != 0;
}

// dW blocks (= split-K partials summed by splitk_reduce_kernel)
int direct_dw_blocks(int N, int OH) {
    // >= 32 rows per block: with fewer, the per-block ring fill and partition reduction and the
    // fixed-order sum of the per-block partials dominated (VGG stem dW at batch 128: 352 GB/s)
    static const int min_rows = getenv("SMCONV_DIRECT_DW_ROWS") ? atoi(getenv("SMCONV_DIRECT_DW_ROWS")) : 32;
    static const int max_blocks = getenv("SMCONV_DIRECT_DW_BLOCKS") ? atoi(getenv("SMCONV_DIRECT_DW_BLOCKS")) : 148 * 3;
    const int rows = N * OH;
    int b = max_blocks;
    if (b > rows / min_rows) b = rows / min_rows;
    return b < 1 ? 1 : b;
}

int direct_launch(int op, const GenParams& g, int blocks, cudaStream_t st, char* err, size_t errlen) {
    DirectParams p;
    p.N = g.N; p.IH = g.IH; p.IW = g.IW; p.IC = g.IC; p.OC = g.OC; p.FH = g.FH; p.FW = g.FW;
    p.sh = g.sh; p.sw = g.sw; p.ph = g.ph; p.pw = g.pw; p.OH = g.OH; p.OW = g.OW;
    p.K = g.FH * g.FW * g.IC;
    p.WIN = (p.OW - 1) * p.sw + p.FW;
    p.X = p.W = p.dY = nullptr;
    p.out = g.out;
    p.rows_per_block = 0;
    size_t smem;
    if (op == CONV_OP_FWD) {
        p.X = g.A;
        p.W = g.B;
        const int trow = (p.OC / 4) * ((p.OW + kDirOWB - 1) / kDirOWB);
        const int rp = trow >= kDirThreads ? 1 : kDirThreads / trow;
        smem = direct_smem(CONV_OP_FWD, p.IC, p.OC, p.FH, p.FW, p.OW, p.sw);
        if (smem == 0) {
            snprintf(err, errlen, "direct fwd: OC*OW too large (threads %d)", trow);
            return CONV_EUNSUPPORTED;
        }
        int grid = (p.N * p.OH + rp - 1) / rp;
        if (grid > 148 * 8) grid = 148 * 8;
        auto kern = conv_direct_fwd_kernel<0, 0, 0, 0, true>;
        if (p.FH == 3 && p.FW == 3 && p.IC == 4 && p.sw == 1 && p.OW % kDirOWB == 0)
            kern = conv_direct_fwd_kernel<3, 3, 1, 1, false>;  // the RGB stems
        if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        launch_k(kern, dim3(grid), dim3(kDirThreads), smem, st, 1, p);
    } else {
        p.dY = g.A;  // run(): dW gets A = dY, B = X
        p.X = g.B;
        p.rows_per_block = (p.N * p.OH + blocks - 1) / blocks;
        const int tpp = (p.OC / 4) * p.FH;
        const int acc4 = (p.FW * p.IC + 3) / 4;
        smem = direct_smem(CONV_OP_BWD_FILTER, p.IC, p.OC, p.FH, p.FW, p.OW, p.sw);
        if (smem == 0) {
            snprintf(err, errlen, "direct dw: OC*FH too large (threads %d)", tpp);
            return CONV_EUNSUPPORTED;
        }
        if (acc4 <= 3) {
            if (smem > 48 * 1024)
                cudaFuncSetAttribute(conv_direct_dw_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            launch_k(conv_direct_dw_kernel<3>, dim3(blocks), dim3(kDirThreads), smem, st, 1, p);
        } else {
            if (smem > 48 * 1024)
                cudaFuncSetAttribute(conv_direct_dw_kernel<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            launch_k(conv_direct_dw_kernel<6>, dim3(blocks), dim3(kDirThreads), smem, st, 1, p);
        }
    }
    return CONV_OK;
}

}  // namespace smconv
