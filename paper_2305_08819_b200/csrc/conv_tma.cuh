// conv_tma.cuh — TMA variant: TMA-staged implicit GEMM on tcgen05 (sm_100a), the fast path for
// channel extents that are multiples of 32 and batches that are multiples of 32.
//
// Same GEMM mapping as conv_gen.cuh (fwd / dX / dW; position-major "batch-folded" rows), but
// operand tiles are moved HBM/L2 -> shared memory by the Tensor Memory Accelerator
// (cp.async.bulk.tensor, north_star (a)) as plain tiled boxes of the NHWC / OHWI tensors:
//
//   fwd A : X  [N][IH][IW][IC]  box (32 ch, 1, 1, G imgs) at (c0, ow*sw-pw+fw, oh*sh-ph+fh, n0)
//   dX  A : dY [N][OH][OW][OC]  box (32 ch, 1, 1, G imgs) at (c0, j'+dw, i'+dh, n0)
//   fwd B : W  as (IC, T, OC)            box (32, 1, BN)           K-major
//   dX  B : W  as (32 ic, OC, IC/32, T)  box (32, 32, BN/32, 1)    MN-major
//   dW  A : dY as (32 oc, N, OC/32, OH*OW) box (32, 32, 4, 1)      MN-major
//   dW  B : X  as (32 ic, N, IC/32, IW, IH) box (32, 32, cols/32, 1, 1) per tap   MN-major
//
// Zero padding, ragged tiles and taps that fall off the map are TMA out-of-bounds zero fill
// (CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE): no predication in the data path at all.  K-major
// boxes use SWIZZLE_128B, MN-major boxes SWIZZLE_128B_ATOM_32B (= UMMA SWIZZLE_128B_BASE32B).
//
// Warp roles: warps 0-7 epilogue (+ accumulator promotion), warp 8 TMA producer (1 lane),
// warp 9 TMEM owner + MMA issuer (1 lane), warps 10-13 (3xTF32 only) split converters.
//
// 3xTF32 here exploits what the probe measured: tcgen05 kind::tf32 reads an
// fp32 operand by TRUNCATION to TF32, so the raw TMA tile IS a_hi = trunc_tf32(a); the
// converters only write a_lo = a - trunc_tf32(a) (exact in fp32).  Per k-step:
// a_lo*b_hi + a_hi*b_lo + a_hi*b_hi.  The accumulator adds by truncation too, so the K loop
// is cut into chunks of kChunkKb k-blocks accumulated in alternating TMEM buffers and
// promoted into fp32 registers (round-to-nearest) by the epilogue warps while the next
// chunk runs (SURVEY.md §7 hard part 1).
#pragma once
#include <cuda.h>

#include "conv_gen.cuh"

namespace smconv {

struct __align__(64) TmaParams {
    CUtensorMap mapA;
    CUtensorMap mapB;
    int G;           // images per A box (fwd/dx): 128 when N % 128 == 0, else 32
    int CB;          // fwd/dx: channel blocks of 32 per tap (IC/32 resp. OC/32)
    int NB32;        // dw: N / 32 (image blocks per position)
    int b_boxes;     // dw: B boxes (taps) per tile
    int b_box_cols;  // dw: GEMM columns per B box
    int chunk_kb;    // promotion interval in k-blocks (3xTF32)
};

template <int OP, int BN, int PLANES>
struct TmaCfg {
    static constexpr int BM = 128, BK = 32;
    static constexpr int NEPI = 8;                       // epilogue warps 0-7
    static constexpr int TMA_W = 8, MMA_W = 9, CONV_W0 = 10;
    static constexpr int NCONV = PLANES == 2 ? 4 : 0;
    static constexpr int NTHREADS = (10 + NCONV) * 32;
    static constexpr int A_BYTES = BM * BK * 4;
    static constexpr int B_BYTES = BN * BK * 4;
    static constexpr int STAGE_BYTES = PLANES * (A_BYTES + B_BYTES);
    static constexpr int STAGES_RAW = (200 * 1024) / STAGE_BYTES;
    static constexpr int STAGES = STAGES_RAW > 6 ? 6 : STAGES_RAW;
    static constexpr bool A_MN = (OP == OP_DW);
    static constexpr bool B_MN = (OP != OP_FWD);
    static constexpr int ACC_COLS = PLANES == 2 ? 2 * BN : BN;
    static constexpr int TMEM_COLS = ACC_COLS <= 32 ? 32 : ACC_COLS <= 64 ? 64 : ACC_COLS <= 128 ? 128 : ACC_COLS <= 256 ? 256 : 512;
    static constexpr int AUX_BYTES = 2048 + kMaxTaps * 16;
    static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + AUX_BYTES;
    static_assert(STAGES >= 2, "stage does not fit");
    static_assert(PLANES == 1 || BN <= 128, "3xTF32 promotion keeps BN/2 fp32 per epilogue thread");
};

struct TmaAux {
    uint64_t full[8], conv[8], empty[8];
    uint64_t tfull[2], tempty[2];
    uint32_t tmem_base;
    int ntaps;
    int4 grp[4];          // A-box groups: {h0, w0, n0, valid}
    int4 taps[kMaxTaps];  // {dh, dw, tapfull, 0}
};

SMCONV_DEV void tma_load_4d(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

SMCONV_DEV void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

SMCONV_DEV void tma_load_5d(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2, int c3,
                            int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
        : "memory");
}

SMCONV_DEV void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

template <int OP, int BN, int PLANES>
__global__ void __launch_bounds__(TmaCfg<OP, BN, PLANES>::NTHREADS, 1)
    conv_tma_kernel(const __grid_constant__ TmaParams tp, const __grid_constant__ GenParams p) {
    using C = TmaCfg<OP, BN, PLANES>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    const uint32_t tiles_addr = (raw_addr + 1023u) & ~1023u;
    uint8_t* tiles_ptr = smem_raw + (tiles_addr - raw_addr);
    TmaAux* aux = reinterpret_cast<TmaAux*>(tiles_ptr + C::STAGES * C::STAGE_BYTES);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    int phase = 0, mt = blockIdx.x;
    if (OP == OP_DX) {
        while (phase + 1 < p.nphase && mt >= p.phase_tile0[phase + 1]) ++phase;
        mt -= p.phase_tile0[phase];
    }
    const int m0 = mt * C::BM;
    const int n0 = blockIdx.y * BN;
    const int split = blockIdx.z;
    const int Mrows = OP == OP_DX ? p.phase_IHp[phase] * p.phase_IWp[phase] * p.N : p.M;

    if (tid == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&aux->full[s], 1);
            mbar_init(&aux->conv[s], C::NCONV * 32);
            mbar_init(&aux->empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&aux->tfull[b], 1);
            mbar_init(&aux->tempty[b], C::NEPI * 32);
        }
        fence_mbar_init();
    }
    if (OP != OP_DW && warp == 0) {
        // A-box groups (G images each) and the union of their valid taps
        const int ngrp = C::BM / tp.G;
        if (lane < ngrp) {
            const int m = m0 + lane * tp.G;
            int4 gi = make_int4(-(1 << 20), -(1 << 20), 0, 0);
            if (m < Mrows) {
                RowInfo ri = row_info<OP>(p, phase, m);
                gi = make_int4(ri.h0, ri.w0, ri.n, 1);
            }
            aux->grp[lane] = gi;
        }
        __syncwarp();
        const int srcH = OP == OP_FWD ? p.IH : p.OH;
        const int srcW = OP == OP_FWD ? p.IW : p.OW;
        int nt = 0;
        for (int fh = 0; fh < p.FH; ++fh)
            for (int fw = 0; fw < p.FW; ++fw) {
                int dh = fh, dw = fw;
                if (OP == OP_DX) {
                    const int th = p.phase_rh[phase] + p.ph - fh, tw = p.phase_rw[phase] + p.pw - fw;
                    if (((th % p.sh) + p.sh) % p.sh != 0 || ((tw % p.sw) + p.sw) % p.sw != 0) continue;
                    dh = th / p.sh;
                    dw = tw / p.sw;
                }
                bool any = false;
                if (lane < ngrp) {
                    const int4 gi = aux->grp[lane];
                    any = gi.w && (unsigned)(gi.x + dh) < (unsigned)srcH && (unsigned)(gi.y + dw) < (unsigned)srcW;
                }
                if (__any_sync(0xffffffffu, any)) {
                    if (lane == 0) aux->taps[nt] = make_int4(dh, dw, fh * p.FW + fw, 0);
                    ++nt;
                }
            }
        if (lane == 0) aux->ntaps = nt;
    }
    if (warp == C::TMA_W && lane == 0) {
        prefetch_tmap(&tp.mapA);
        prefetch_tmap(&tp.mapB);
    }
    if (warp == C::MMA_W) tmem_alloc(&aux->tmem_base, C::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = aux->tmem_base;

    int kb_begin, kb_end;
    {
        int nkb;
        if (OP == OP_DW) {
            nkb = p.OH * p.OW * tp.NB32;
            kb_begin = split * p.kb_per_split;
            kb_end = min(nkb, kb_begin + p.kb_per_split);
        } else {
            nkb = aux->ntaps * tp.CB;
            const int per = (nkb + p.splits - 1) / p.splits;
            kb_begin = split * per;
            kb_end = min(nkb, kb_begin + per);
        }
    }
    const int nkb_local = max(0, kb_end - kb_begin);
    const int CHK = PLANES == 2 ? tp.chunk_kb : (1 << 30);
    const int nchunks = nkb_local > 0 ? (nkb_local + CHK - 1) / CHK : 0;

    if (warp == C::TMA_W) {
        // ======================= TMA producer
        if (lane == 0) {
            for (int it = 0; it < nkb_local; ++it) {
                const int kb = kb_begin + it;
                const int s = it % C::STAGES, r = it / C::STAGES;
                if (r > 0) mbar_wait(&aux->empty[s], (r - 1) & 1);
                const uint32_t sA = tiles_addr + s * C::STAGE_BYTES;
                const uint32_t sB = sA + PLANES * C::A_BYTES;
                if (OP == OP_FWD || OP == OP_DX) {
                    const int j = kb / tp.CB, cb = kb - j * tp.CB;
                    const int4 t = aux->taps[j];
                    mbar_arrive_expect_tx(&aux->full[s], C::A_BYTES + C::B_BYTES);
                    const int ngrp = C::BM / tp.G;
                    for (int g = 0; g < ngrp; ++g) {
                        const int4 gi = aux->grp[g];
                        tma_load_4d(sA + g * tp.G * 128, &tp.mapA, &aux->full[s], cb * 32, gi.y + t.y, gi.x + t.x, gi.z);
                    }
                    if (OP == OP_FWD) tma_load_3d(sB, &tp.mapB, &aux->full[s], cb * 32, t.z, n0);
                    else tma_load_4d(sB, &tp.mapB, &aux->full[s], 0, cb * 32, n0 / 32, t.z);
                } else {
                    const int pos = kb / tp.NB32, nb = kb - pos * tp.NB32;
                    const int oh = pos / p.OW, ow = pos - oh * p.OW;
                    int nbox = 0;
                    for (int b = 0; b < tp.b_boxes; ++b) {
                        const int col0 = n0 + b * tp.b_box_cols;
                        if (col0 < p.Ngemm) ++nbox;
                    }
                    mbar_arrive_expect_tx(&aux->full[s], C::A_BYTES + nbox * tp.b_box_cols * 128);
                    tma_load_4d(sA, &tp.mapA, &aux->full[s], 0, nb * 32, m0 / 32, pos);
                    for (int b = 0; b < tp.b_boxes; ++b) {
                        const int col0 = n0 + b * tp.b_box_cols;
                        if (col0 >= p.Ngemm) break;
                        const int tap = col0 / p.IC, icb = (col0 - tap * p.IC) / 32;
                        const int fh = tap / p.FW, fw = tap - fh * p.FW;
                        tma_load_5d(sB + b * tp.b_box_cols * 128, &tp.mapB, &aux->full[s], 0, nb * 32, icb,
                                    ow * p.sw - p.pw + fw, oh * p.sh - p.ph + fh);
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == C::MMA_W) {
        // ======================= MMA issuer
        if (lane == 0) {
            constexpr uint32_t IDESC = idesc_tf32(128, BN, C::A_MN, C::B_MN);
            const uint32_t albo = C::A_MN ? 4096u : 16u, blbo = C::B_MN ? 4096u : 16u;
            const uint32_t asbo = C::A_MN ? 512u : 1024u, bsbo = C::B_MN ? 512u : 1024u;
            const uint32_t alay = C::A_MN ? kLayoutSW128Base32 : kLayoutSW128;
            const uint32_t blay = C::B_MN ? kLayoutSW128Base32 : kLayoutSW128;
            for (int it = 0; it < nkb_local; ++it) {
                const int s = it % C::STAGES, r = it / C::STAGES;
                const int c = it / CHK, first = (it - c * CHK) == 0;
                const int buf = c & 1;
                if (PLANES == 2 && first && c >= 2) {
                    mbar_wait(&aux->tempty[buf], ((c >> 1) - 1) & 1);
                }
                mbar_wait(PLANES == 2 ? &aux->conv[s] : &aux->full[s], r & 1);
                tc_fence_after();
                const uint32_t d = tmem + (PLANES == 2 ? (uint32_t)(buf * BN) : 0u);
                const uint32_t aH = tiles_addr + s * C::STAGE_BYTES, aL = aH + C::A_BYTES;
                const uint32_t bH = aH + PLANES * C::A_BYTES, bL = bH + C::B_BYTES;
#pragma unroll
                for (int g = 0; g < C::BK / 8; ++g) {
                    const uint32_t aoff = C::A_MN ? g * 1024u : g * 32u;
                    const uint32_t boff = C::B_MN ? g * 1024u : g * 32u;
                    const uint64_t adH = make_sdesc(aH + aoff, albo, asbo, alay);
                    const uint64_t bdH = make_sdesc(bH + boff, blbo, bsbo, blay);
                    const uint32_t acc0 = (PLANES == 2 ? (!first || g > 0) : (it > 0 || g > 0)) ? 1u : 0u;
                    if (PLANES == 2) {
                        const uint64_t adL = make_sdesc(aL + aoff, albo, asbo, alay);
                        const uint64_t bdL = make_sdesc(bL + boff, blbo, bsbo, blay);
                        mma_tf32_ss(d, adL, bdH, IDESC, acc0);
                        mma_tf32_ss(d, adH, bdL, IDESC, 1u);
                        mma_tf32_ss(d, adH, bdH, IDESC, 1u);
                    } else {
                        mma_tf32_ss(d, adH, bdH, IDESC, acc0);
                    }
                }
                mma_commit(&aux->empty[s]);
                if (PLANES == 2 && (it - c * CHK == CHK - 1 || it == nkb_local - 1)) mma_commit(&aux->tfull[buf]);
            }
            if (PLANES == 1) mma_commit(&aux->tfull[0]);
            if (nkb_local == 0 && PLANES == 2) mma_commit(&aux->tfull[0]);
        }
        __syncwarp();
    } else if (warp >= C::CONV_W0) {
        // ======================= 3xTF32 split converters: lo = a - trunc_tf32(a)
        const int ct = tid - C::CONV_W0 * 32;
        constexpr int NCT = C::NCONV * 32;
        for (int it = 0; it < nkb_local; ++it) {
            const int s = it % C::STAGES, r = it / C::STAGES;
            mbar_wait(&aux->full[s], r & 1);
            uint8_t* st = tiles_ptr + s * C::STAGE_BYTES;
            const float4* aH = reinterpret_cast<const float4*>(st);
            float4* aL = reinterpret_cast<float4*>(st + C::A_BYTES);
            const float4* bH = reinterpret_cast<const float4*>(st + PLANES * C::A_BYTES);
            float4* bL = reinterpret_cast<float4*>(st + PLANES * C::A_BYTES + C::B_BYTES);
#pragma unroll 4
            for (int i = ct; i < C::A_BYTES / 16; i += NCT) {
                const float4 v = aH[i];
                float4 o;
                o.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
                o.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
                o.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
                o.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
                aL[i] = o;
            }
#pragma unroll 4
            for (int i = ct; i < C::B_BYTES / 16; i += NCT) {
                const float4 v = bH[i];
                float4 o;
                o.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
                o.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
                o.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
                o.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
                bL[i] = o;
            }
            fence_proxy_async_smem();
            mbar_arrive(&aux->conv[s]);
        }
    } else {
        // ======================= epilogue warps 0-7 (+ promotion of TMEM chunks, 3xTF32)
        const int q = warp & 3, half = warp >> 2;
        const int row = q * 32 + lane;
        constexpr int HALF = BN / 2;
        const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
        float* outp = p.out + (long long)split * p.split_stride;
        long long obase = -1;
        if (OP == OP_DW) {
            const int oc = m0 + row;
            if (oc < p.OC) obase = (long long)oc * p.Ngemm;
        } else {
            RowInfo ri = row_info<OP>(p, phase, m0 + row);
            if (ri.ok) obase = (long long)ri.orow * p.Ngemm;
        }
        if (PLANES == 2) {
            float acc[HALF];
#pragma unroll
            for (int e = 0; e < HALF; ++e) acc[e] = 0.f;
            for (int c = 0; c < nchunks; ++c) {
                const int buf = c & 1;
                mbar_wait(&aux->tfull[buf], (c >> 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int c0 = 0; c0 < HALF; c0 += 16) {
                    uint32_t v[16];
                    tmem_ld_32x32b_x16(tmem + lane_addr + (uint32_t)(buf * BN + half * HALF + c0), v);
                    tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 16; ++e) acc[c0 + e] += __uint_as_float(v[e]);
                }
                tc_fence_before();
                mbar_arrive(&aux->tempty[buf]);
            }
            if (obase >= 0) {
#pragma unroll
                for (int e = 0; e < HALF; e += 4) {
                    const int col = n0 + half * HALF + e;
                    if (col < p.Ngemm)
                        *reinterpret_cast<float4*>(outp + obase + col) =
                            make_float4(acc[e], acc[e + 1], acc[e + 2], acc[e + 3]);
                }
            }
        } else {
            mbar_wait(&aux->tfull[0], 0);
            tc_fence_after();
#pragma unroll 1
            for (int c0 = 0; c0 < HALF; c0 += 16) {
                uint32_t v[16];
                if (nkb_local > 0) {
                    tmem_ld_32x32b_x16(tmem + lane_addr + (uint32_t)(half * HALF + c0), v);
                    tmem_ld_wait();
                } else {
#pragma unroll
                    for (int e = 0; e < 16; ++e) v[e] = 0u;
                }
                if (obase >= 0) {
#pragma unroll
                    for (int e = 0; e < 16; e += 4) {
                        const int col = n0 + half * HALF + c0 + e;
                        if (col < p.Ngemm)
                            *reinterpret_cast<float4*>(outp + obase + col) =
                                make_float4(__uint_as_float(v[e]), __uint_as_float(v[e + 1]),
                                            __uint_as_float(v[e + 2]), __uint_as_float(v[e + 3]));
                    }
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == C::MMA_W) {
        tc_fence_after();
        tmem_dealloc(tmem, C::TMEM_COLS);
    }
}

// ------------------------------------------------------------------ host side
bool tma_supported(int op, int N, int IC, int OC, int FH, int FW, int sh, int sw);
int tma_make_plan(int op, GenParams& g, int& BN, int planes, TmaParams& tp, dim3& grid, char* err, size_t errlen);
int tma_launch(int op, int BN, int planes, const GenParams& g, TmaParams& tp, dim3 grid, cudaStream_t st, char* err,
               size_t errlen);

}  // namespace smconv
