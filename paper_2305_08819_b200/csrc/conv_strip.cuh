// conv_strip.cuh — STRIP variant: stride-1 fwd / dX (3-wide filters) with input-slab reuse
// across the filter columns; the fast path for the 64/128-channel 32x32 and 16x16 layers.
//
// With a 128 x BN output tile of the plain implicit GEMM, every A (activation) byte brought in by
// TMA feeds only BN output channels, and for BN = 64 (ResNet l1 / VGG conv2: 64 channels) the
// kernel is bound by TMA traffic, not by the tensor core.  Here a tile is a strip of 4R output
// positions of one output row x 32 images x BN channels.  Per (filter row fh, 32-channel block)
// one TMA box brings the (4R + FW - 1) input "slabs" [32 images x 32 channels] of the source row
// into shared memory, contiguously; the 128-row A operand of accumulator j and filter column fw
// is then the 4-slab window starting at slab 4j + fw (fwd) / 4j + FW-1-fw (dX) -- a plain
// descriptor offset, no copy.  Each slab is loaded once and used FW times (3x fewer A bytes),
// and one stage feeds R * FW * 4 MMAs (6-12x fewer TMA instructions per MMA).
//
// Row of an accumulator: position p = row / 32 of its 4-group, image = row % 32, so epilogue
// warp quadrant q handles position 4j + q.  Zero padding / ragged strips = TMA OOB zero fill.
// Roles, 3xTF32 handling (TF32 a_hi*b_hi + bf16 cross terms on the precomputed W' plane) and
// TMEM double buffering are those of conv_tma.cuh.
//
// PAIR (3xTF32, BN = 64): a 2-CTA cluster runs two strips of the same output row and columns for
// consecutive 32-image groups as ONE M = 256 tile (tcgen05 cta_group::2): each CTA stages its own
// slabs (A windows in its own TMEM) and half of B (32 filter columns); CTA 0 issues the MMAs, the
// commits arrive in both CTAs.  N = 64 MMAs run at ~57 % of the pair rate on one CTA.
#pragma once
#include "conv_tma.cuh"

namespace smconv {

constexpr int kStripFW = 3;

struct __align__(64) StripParams {
    CUtensorMap mapA;  // activations viewed (32 ch, N, W, H, C/32)
    CUtensorMap mapB;  // fwd: W viewed (IC, OC, T); dX: W viewed (32 ic, OC, IC/32, T)
    CUtensorMap mapBx;  // 3xTF32: the precomputed bf16 W' plane (wx_prep_kernel), box (64, 1, BN, 1)
    int CB;            // 32-channel blocks of the reduction (fwd: IC/32, dX: OC/32)
    int NG;            // 32-image groups
    int OHo, OWo;      // output extent (fwd: OH x OW, dX: IH x IW)
    int SH, SW;        // source extent (fwd: IH x IW, dX: OH x OW)
    int strips;        // strips per output row
    int n_tiles, work, chunk_kb;
    int row_off;       // source row = out row + row_off + (fwd: fh | dX: -fh)   (fwd: -ph, dX: +ph)
    int col_off;       // first slab column = strip origin + col_off (fwd: -pw, dX: pw - (FW-1))
    int pair;          // work items are pair tiles (two 32-image groups), kernel template PAIR
    FastDiv fd_ntiles, fd_strips, fd_OHo;
    int coalesce;      // row-coalesced epilogue stores (StripCfg::EPW)
    int alt_conv;      // 3xTF32 converter warps in two groups on alternate stages
    int tstore;        // ... leaving by TMA tensor store (conv_tma.cuh warp_rows_tstore): mapY = output (C, pixels, N)
    CUtensorMap mapY;
};

template <int OP, int BN, int PLANES, int R, bool PAIR = false>
struct StripCfg {
    static constexpr int FW = kStripFW;
    static constexpr int SLABS = 4 * R + FW - 1;
    static constexpr int A_BYTES = SLABS * 4096;
    static constexpr int BNC = PAIR ? BN / 2 : BN;  // B columns staged by this CTA (a pair splits B)
    static constexpr int B_BYTES = FW * BNC * 128;
    // 3xTF32: the converters write the R*FW A windows (hi and lo) into TMEM, so the 3 MMAs per
    // k-step read A from TMEM and only b_lo is stored in shared memory (smem-bandwidth bound path)
    static constexpr bool A_TMEM = (PLANES == 2);
    static constexpr int B_OFF = A_TMEM ? A_BYTES : PLANES * A_BYTES;
    static constexpr int STAGE_BYTES = A_TMEM ? A_BYTES + 2 * B_BYTES : PLANES * (A_BYTES + B_BYTES);
    static constexpr int A_SLOT_COLS = R * FW * 64;  // TMEM columns per stage: (j, fw) windows x (hi 32 + lo 32)
    // smem stages (TMA ring) and TMEM A-window slots (converter -> MMA ring) are separate rings, as
    // in conv_tma.cuh: at BN = 64 in 3xTF32 TMEM holds only 2 slots but 3 smem stages fit in 216 KB
    static constexpr int STAGES_RAW = (214 * 1024) / STAGE_BYTES;
    static constexpr int STAGES = STAGES_RAW > 6 ? 6 : STAGES_RAW;
    static constexpr int NT_RAW = A_TMEM ? (512 - 2 * R * BN) / A_SLOT_COLS : 1;
    static constexpr int NT = NT_RAW > 6 ? 6 : NT_RAW;
    static constexpr int NEPI = 8, TMA_W = 8, MMA_W = 9, CONV_W0 = 10;
    static constexpr int NCONV = PLANES == 2 ? 8 : 0;
    static constexpr int NTHREADS = (10 + NCONV) * 32;
    static constexpr bool B_MN = (OP == OP_DX);
    static constexpr int A_TCOL0 = 2 * R * BN;
    static constexpr int ACC_COLS = 2 * R * BN + (A_TMEM ? NT * A_SLOT_COLS : 0);
    static constexpr int TMEM_COLS = ACC_COLS <= 32 ? 32 : ACC_COLS <= 64 ? 64 : ACC_COLS <= 128 ? 128 : ACC_COLS <= 256 ? 256 : 512;
    static constexpr int SMEM_BASE = 1024 + STAGES * STAGE_BYTES + 1024;
    // row-coalesced epilogue stores (conv_tma.cuh warp_rows_store): a lane is one image, so a warp's
    // direct st.global.v4 scatter over 32 rows OH*OW*C*4 bytes apart
    static constexpr int SMEM_FREE = 232448 - SMEM_BASE;
    static constexpr int EPW = (BN / 2 >= 32 && SMEM_FREE >= NEPI * 32 * 32 * 4) ? 32
                             : (BN / 2 >= 16 && SMEM_FREE >= NEPI * 32 * 16 * 4) ? 16 : 0;
    static constexpr int SMEM_BYTES = SMEM_BASE + NEPI * 32 * EPW * 4;
    static_assert(STAGES >= 2 && NT >= 1, "strip stage does not fit");
    static_assert(!A_TMEM || (R == 1 && NT * FW <= 8), "3xTF32 strips: one window per filter column, per-window barriers");
    static_assert(ACC_COLS <= 512, "TMEM");
    static_assert(PLANES == 1 || R * BN <= 128, "3xTF32 promotion keeps R*BN/2 fp32 per epilogue thread");
    static_assert(!PAIR || (A_TMEM && R == 1 && BN == 64), "strip pairs: 3xTF32, BN 64");
};

struct StripTile {
    int g, orow, s, nt;
    SMCONV_DEV void init(const StripParams& sp, int w, int rank = 0) {
        // fast divisors (host-built): generic divisions are ~150-cycle dependent chains
        int r = (int)fdiv((uint32_t)w, sp.fd_ntiles);
        nt = w - r * sp.n_tiles;
        const int r2 = (int)fdiv((uint32_t)r, sp.fd_strips);
        s = r - r2 * sp.strips;
        g = (int)fdiv((uint32_t)r2, sp.fd_OHo);
        orow = r2 - g * sp.OHo;
        if (sp.pair) g = 2 * g + rank;  // pair tile: image groups 2g' (CTA 0) and 2g'+1 (CTA 1)
    }
};

// 32-row group of an epilogue warp (32 images of one output position) for the fused-epilogue
// statistics partial rows: (image group, output row, output column); -1 past the ragged strip end
template <int R>
SMCONV_DEV int strip_grp(const StripParams& sp, const StripTile& t, int j, int qd) {
    const int ocol = t.s * 4 * R + 4 * j + qd;
    return ocol < sp.OWo ? (t.g * sp.OHo + t.orow) * sp.OWo + ocol : -1;
}

template <int OP>
SMCONV_DEV int strip_src_row(const StripParams& sp, int orow, int fh) {
    return OP == OP_FWD ? orow + sp.row_off + fh : orow + sp.row_off - fh;
}

// number of filter rows whose source row is inside the map (others are all-zero stages: skipped)
template <int OP>
SMCONV_DEV int strip_rows(const StripParams& sp, const GenParams& p, int orow) {
    int n = 0;
    for (int fh = 0; fh < p.FH; ++fh) n += (unsigned)strip_src_row<OP>(sp, orow, fh) < (unsigned)sp.SH;
    return n;
}

template <int OP, int BN, int PLANES, int R, bool PAIR = false>
__global__ void __launch_bounds__(StripCfg<OP, BN, PLANES, R, PAIR>::NTHREADS, 1)
    conv_strip_kernel(const __grid_constant__ StripParams sp, const __grid_constant__ GenParams p) {
    using C = StripCfg<OP, BN, PLANES, R, PAIR>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    const uint32_t tiles_addr = (raw_addr + 1023u) & ~1023u;
    uint8_t* tiles_ptr = smem_raw + (tiles_addr - raw_addr);
    TmaAux* aux = reinterpret_cast<TmaAux*>(tiles_ptr + C::STAGES * C::STAGE_BYTES);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int CHK = PLANES == 2 ? sp.chunk_kb : (1 << 30);
    // pairs: both CTAs of a cluster walk the same pair tiles; CTA 0 issues the MMAs and owns the
    // conv / tempty barriers (per-warp arrivals from both CTAs), commits arrive in both CTAs
    const int rank = PAIR ? (int)cluster_ctarank() : 0;
    const int wfirst = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
    const int wstep = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;

    if (tid == 0) {
        for (int t = 0; t < C::NT; ++t) mbar_init(&aux->tfree[t], 1);
        // 3xTF32: one conv barrier per (slot, filter column) so the MMAs of window 0 start while
        // windows 1 and 2 are still being split (the converters' per-stage latency bounded the strip)
        for (int t = 0; t < (C::A_TMEM ? C::NT * C::FW : C::NT); ++t)
            mbar_init(&aux->conv[t], PAIR ? 2 * (sp.alt_conv ? C::NCONV / 2 : C::NCONV)
                                          : (sp.alt_conv ? C::NCONV / 2 : C::NCONV) * 32);
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&aux->full[s], 1);
            mbar_init(&aux->empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&aux->tfull[b], 1);
            mbar_init(&aux->tempty[b], PAIR ? 2 * C::NEPI : C::NEPI * 32);
        }
        fence_mbar_init();
    }
    if (warp == C::TMA_W && lane == 0) {
        prefetch_tmap(&sp.mapA);
        prefetch_tmap(&sp.mapB);
        if (C::A_TMEM) prefetch_tmap(&sp.mapBx);
    }
    if (warp == C::MMA_W) {
        if (PAIR) tmem_alloc2(&aux->tmem_base, C::TMEM_COLS);
        else tmem_alloc(&aux->tmem_base, C::TMEM_COLS);
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync_all();  // the peer's barriers exist before any remote arrival
    tc_fence_after();
    const uint32_t tmem = aux->tmem_base;
    pdl_trigger();
    pdl_wait();  // launch.cuh

    if (warp == C::TMA_W) {
        // ======================= TMA producer: 2 boxes per stage (slab row, FW filter taps)
        int s = 0;
        uint32_t r = 0;
        for (int w = wfirst; w < sp.work; w += wstep) {
            StripTile t;
            t.init(sp, w, rank);
            const int col0 = t.s * 4 * R + sp.col_off;
            const int nb0 = t.nt * BN + rank * C::BNC;  // this CTA's half of B (pairs)
            for (int fh = 0; fh < p.FH; ++fh) {
                const int srow = strip_src_row<OP>(sp, t.orow, fh);
                if ((unsigned)srow >= (unsigned)sp.SH) continue;
                for (int cb = 0; cb < sp.CB; ++cb) {
                    if (r > 0) {
                        if (PAIR) mbar_wait_cluster(&aux->empty[s], (r - 1) & 1);
                        else mbar_wait(&aux->empty[s], (r - 1) & 1);
                    }
                    const uint32_t sA = tiles_addr + s * C::STAGE_BYTES;
                    const uint32_t sB = sA + C::B_OFF;
                    if (elect_one()) {
                        mbar_arrive_expect_tx(&aux->full[s], C::A_BYTES + (C::A_TMEM ? 2 : 1) * C::B_BYTES);
                        tma_load_5d(sA, &sp.mapA, &aux->full[s], 0, t.g * 32, col0, srow, cb);
                        if (OP == OP_FWD) tma_load_3d(sB, &sp.mapB, &aux->full[s], cb * 32, nb0, fh * C::FW);
                        else tma_load_4d(sB, &sp.mapB, &aux->full[s], 0, cb * 32, nb0 / 32, fh * C::FW);
                        if (C::A_TMEM)  // W' planes of the FW taps: [fw][BNC rows][128 B]
#pragma unroll
                            for (int fw = 0; fw < C::FW; ++fw)
                                tma_load_4d(sB + C::B_BYTES + fw * C::BNC * 128, &sp.mapBx, &aux->full[s], 0, cb, nb0,
                                            fh * C::FW + fw);
                    }
                    __syncwarp();
                    if (++s == C::STAGES) {
                        s = 0;
                        ++r;
                    }
                }
            }
        }
    } else if (warp == C::MMA_W) {
        // ======================= MMA issuer: R accumulators x FW taps x 4 k-steps per stage
        // (pairs: CTA 0 issues M = 256 MMAs for both CTAs; CTA 1's MMA warp only owns its TMEM)
        if (PAIR && rank != 0) goto strip_done;
        constexpr uint32_t IDESC = idesc_tf32(PAIR ? 256 : 128, BN, false, C::B_MN);
        const uint64_t adH0 = make_sdesc(tiles_addr, 16u, 1024u, kLayoutSW128);
        const uint64_t bdH0 = make_sdesc(tiles_addr + C::B_OFF, C::B_MN ? 4096u : 16u,
                                         C::B_MN ? 512u : 1024u, C::B_MN ? kLayoutSW128Base32 : kLayoutSW128);
        // 3xTF32 cross terms: bf16 B' planes [b_lo | b] (K-major, 128 B per row) after the b_hi taps
        constexpr uint32_t IDESC_X = idesc_bf16(PAIR ? 256 : 128, BN, false, false);
        const uint64_t bx0 = make_sdesc(tiles_addr + C::B_OFF + C::B_BYTES, 16u, 1024u, kLayoutSW128);
        constexpr uint64_t B_G = C::B_MN ? 64 : 2, B_TAP = (C::BNC * 128) >> 4;
        int s = 0, in_chunk = 0;
        uint32_t r = 0, c = 0, q = 0;
        for (int w = wfirst; w < sp.work; w += wstep) {
            StripTile t;
            t.init(sp, w, rank);
            const int nkb = strip_rows<OP>(sp, p, t.orow) * sp.CB;
            for (int it = 0; it < nkb; ++it, ++q) {
                const int buf = c & 1;
                const uint32_t ts = q % C::NT, rts = q / C::NT;  // TMEM A-window slot
                if (in_chunk == 0 && c >= 2) {
                    if (PAIR) mbar_wait_cluster(&aux->tempty[buf], ((c >> 1) - 1) & 1);
                    else mbar_wait(&aux->tempty[buf], ((c >> 1) - 1) & 1);
                    tc_fence_after();
                }
                if (!C::A_TMEM) {
                    if (PLANES == 2) mbar_wait(&aux->conv[ts], rts & 1);
                    else mbar_wait(&aux->full[s], r & 1);
                    tc_fence_after();
                }
                const uint64_t so = (uint64_t)(s * C::STAGE_BYTES) >> 4;
                const bool last = (in_chunk + 1 == CHK || it == nkb - 1);
                {
#pragma unroll
                    for (int j = 0; j < R; ++j) {
                        const uint32_t d = tmem + (uint32_t)((buf * R + j) * BN);
#pragma unroll
                        for (int fw = 0; fw < C::FW; ++fw) {
                            if (C::A_TMEM) {
                                if (PAIR) mbar_wait_cluster(&aux->conv[ts * C::FW + fw], rts & 1);
                                else mbar_wait(&aux->conv[ts * C::FW + fw], rts & 1);
                                tc_fence_after();
                            }
                            const int woff = OP == OP_FWD ? fw : C::FW - 1 - fw;
                            const uint64_t a0 = adH0 + so + (uint64_t)((4 * j + woff) * 4096 >> 4);
                            const uint64_t b0 = bdH0 + so + fw * B_TAP;
                            const bool issuer = elect_one();
#pragma unroll
                            for (int g = 0; g < 4; ++g) {
                                if (!issuer) break;
                                const uint64_t adH = a0 + g * 2, bdH = b0 + g * B_G;
                                const uint32_t acc0 = (in_chunk > 0 || fw > 0 || g > 0) ? 1u : 0u;
                                if (C::A_TMEM) {
                                    const uint32_t ahi =
                                        tmem + (uint32_t)(C::A_TCOL0 + ts * C::A_SLOT_COLS + (j * C::FW + fw) * 64 + g * 8);
                                    if (PAIR) mma2_tf32_ts(d, ahi, bdH, IDESC, acc0);  // a_hi * b_hi
                                    else mma_tf32_ts(d, ahi, bdH, IDESC, acc0);
                                } else {
                                    mma_tf32_ss(d, adH, bdH, IDESC, acc0);
                                }
                            }
                            if (C::A_TMEM && issuer) {  // cross terms, bf16, K = 64 in 4 MMAs
                                const uint32_t ax = tmem + (uint32_t)(C::A_TCOL0 + ts * C::A_SLOT_COLS + (j * C::FW + fw) * 64 + 32);
#pragma unroll
                                for (int jj = 0; jj < 4; ++jj) {
                                    if (PAIR) mma2_bf16_ts(d, ax + jj * 8, bx0 + so + fw * B_TAP + jj * 2, IDESC_X, 1u);
                                    else mma_bf16_ts(d, ax + jj * 8, bx0 + so + fw * B_TAP + jj * 2, IDESC_X, 1u);
                                }
                            }
                            __syncwarp();
                        }
                    }
                    if (elect_one()) {
                        if (PAIR) {
                            mma2_commit_both(&aux->empty[s]);
                            mma2_commit_both(&aux->tfree[ts]);
                            if (last) mma2_commit_both(&aux->tfull[buf]);
                        } else {
                            mma_commit(&aux->empty[s]);
                            if (C::A_TMEM) mma_commit(&aux->tfree[ts]);
                            if (last) mma_commit(&aux->tfull[buf]);
                        }
                    }
                }
                __syncwarp();
                if (last) {
                    ++c;
                    in_chunk = 0;
                } else {
                    ++in_chunk;
                }
                if (++s == C::STAGES) {
                    s = 0;
                    ++r;
                }
            }
        }
    } else if (warp >= C::CONV_W0 && C::A_TMEM && sp.alt_conv) {
        // ======================= 3xTF32 converters in two groups of 4 warps on alternate stages (conv_tma.cuh
        // TmaParams::alt_conv): a warp = one TMEM lane quadrant, both K halves of each window
        const int grp = (warp - C::CONV_W0) >> 2;
        const int qd = warp & 3;
        uint32_t q = 0;
        for (int w = wfirst; w < sp.work; w += wstep) {
            StripTile t;
            t.init(sp, w, rank);
            const int nkb = strip_rows<OP>(sp, p, t.orow) * sp.CB;
            for (int it = 0; it < nkb; ++it, ++q) {
                if ((int)(q & 1u) != grp) continue;
                const int s = q % C::STAGES;
                const uint32_t r = q / C::STAGES;
                const uint32_t ts = q % C::NT, rts = q / C::NT;  // TMEM A-window slot
                mbar_wait(&aux->full[s], r & 1);
                if (rts > 0) {  // the slot's previous windows have been multiplied
                    if (PAIR) mbar_wait_cluster(&aux->tfree[ts], (rts - 1) & 1);
                    else mbar_wait(&aux->tfree[ts], (rts - 1) & 1);
                    tc_fence_after();
                }
                const uint8_t* st = tiles_ptr + s * C::STAGE_BYTES;
#pragma unroll
                for (int fw = 0; fw < C::FW; ++fw) {
                    const int woff = OP == OP_FWD ? fw : C::FW - 1 - fw;
                    const uint8_t* slab = st + (woff + qd) * 4096;
                    const uint32_t ta = tmem + ((uint32_t)(qd * 32) << 16) +
                                        (uint32_t)(C::A_TCOL0 + ts * C::A_SLOT_COLS + fw * 64);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        float e[16];
#pragma unroll
                        for (int cq = 0; cq < 4; ++cq) {
                            const float4 v = *reinterpret_cast<const float4*>(
                                slab + kmaj_off((uint32_t)lane, (uint32_t)(4 * h + cq)));
                            e[4 * cq] = v.x, e[4 * cq + 1] = v.y, e[4 * cq + 2] = v.z, e[4 * cq + 3] = v.w;
                        }
                        uint32_t hi[16], xh[8], xl[8];
                        split_a16(e, hi, xh, xl);
                        tmem_st_32x32b_x16(ta + h * 16, hi);
                        tmem_st_32x32b_x8(ta + 32 + h * 8, xh);
                        tmem_st_32x32b_x8(ta + 48 + h * 8, xl);
                    }
                    tmem_st_wait();
                    tc_fence_before();
                    if (PAIR) {  // one arrival per warp, on CTA 0's barrier (it issues the MMAs)
                        __syncwarp();
                        if (lane == 0) mbar_arrive_remote(&aux->conv[ts * C::FW + fw], 0);
                    } else {
                        mbar_arrive(&aux->conv[ts * C::FW + fw]);
                    }
                }
            }
        }
    } else if (warp >= C::CONV_W0) {
        // ======================= 3xTF32 split converters (elementwise over the stage)
        const int ct = tid - C::CONV_W0 * 32;
        constexpr int NCT = C::NCONV > 0 ? C::NCONV * 32 : 32;
        int s = 0;
        uint32_t r = 0, q = 0;
        for (int w = wfirst; w < sp.work; w += wstep) {
            StripTile t;
            t.init(sp, w, rank);
            const int nkb = strip_rows<OP>(sp, p, t.orow) * sp.CB;
            for (int it = 0; it < nkb; ++it, ++q) {
                const uint32_t ts = q % C::NT, rts = q / C::NT;  // TMEM A-window slot
                mbar_wait(&aux->full[s], r & 1);
                if (C::A_TMEM && rts > 0) {  // the slot's previous windows have been multiplied
                    if (PAIR) mbar_wait_cluster(&aux->tfree[ts], (rts - 1) & 1);
                    else mbar_wait(&aux->tfree[ts], (rts - 1) & 1);
                    tc_fence_after();
                }
                uint8_t* st = tiles_ptr + s * C::STAGE_BYTES;
                auto lo4 = [](float4 v) {
                    float4 o;
                    o.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
                    o.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
                    o.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
                    o.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
                    return o;
                };
                if (C::A_TMEM) {
                    // window fw row 32*qd+lane = slab woff(fw)+qd, image lane; K half h.  Per filter
                    // column: split the window into TMEM and that tap's B block into b_lo, then
                    // release it to the MMA warp (conv[ts * FW + fw]) before starting the next one
                    const int qd = warp & 3, h = (warp - C::CONV_W0) >> 2;
                    // window fw's 16 values of this thread; the next window's loads are issued before
                    // this window's tcgen05.wait::st (the per-window chain LDS -> split -> STTM -> wait
                    // was serial; the converters bound the strip pipeline: 2 TMEM slots, ncu r02be)
                    auto ld16 = [&](int fw, float (&e)[16]) {
                        const int woff = OP == OP_FWD ? fw : C::FW - 1 - fw;
                        const uint8_t* slab = st + (woff + qd) * 4096;
#pragma unroll
                        for (int cq = 0; cq < 4; ++cq) {
                            const float4 v = *reinterpret_cast<const float4*>(
                                slab + kmaj_off((uint32_t)lane, (uint32_t)(4 * h + cq)));
                            e[4 * cq] = v.x, e[4 * cq + 1] = v.y, e[4 * cq + 2] = v.z, e[4 * cq + 3] = v.w;
                        }
                    };
                    float ebuf[2][16];
                    ld16(0, ebuf[0]);
#pragma unroll
                    for (int fw = 0; fw < C::FW; ++fw) {
                        // window columns: [0,32) a_hi, [32,48) bf16(a_hi) pairs, [48,64) bf16(a_lo) pairs
                        uint32_t hi[16], xh[8], xl[8];
                        split_a16(ebuf[fw & 1], hi, xh, xl);
                        const uint32_t ta = tmem + ((uint32_t)(qd * 32) << 16) +
                                            (uint32_t)(C::A_TCOL0 + ts * C::A_SLOT_COLS + fw * 64);
                        tmem_st_32x32b_x16(ta + h * 16, hi);
                        tmem_st_32x32b_x8(ta + 32 + h * 8, xh);
                        tmem_st_32x32b_x8(ta + 48 + h * 8, xl);
                        if (fw + 1 < C::FW) ld16(fw + 1, ebuf[(fw + 1) & 1]);
                        tmem_st_wait();  // (no generic-proxy shared-memory writes here: no proxy fence)
                        tc_fence_before();
                        if (PAIR) {  // one arrival per warp, on CTA 0's barrier (it issues the MMAs)
                            __syncwarp();
                            if (lane == 0) mbar_arrive_remote(&aux->conv[ts * C::FW + fw], 0);
                        } else {
                            mbar_arrive(&aux->conv[ts * C::FW + fw]);
                        }
                    }
                } else {
                    const float4* aH = reinterpret_cast<const float4*>(st);
                    float4* aL = reinterpret_cast<float4*>(st + C::A_BYTES);
                    constexpr int NA = (C::A_BYTES / 16 + NCT - 1) / NCT;
                    float4 v[NA];
#pragma unroll
                    for (int i = 0; i < NA; ++i)
                        if (ct + i * NCT < C::A_BYTES / 16) v[i] = aH[ct + i * NCT];
#pragma unroll
                    for (int i = 0; i < NA; ++i)
                        if (ct + i * NCT < C::A_BYTES / 16) aL[ct + i * NCT] = lo4(v[i]);
                    const float4* bH = reinterpret_cast<const float4*>(st + C::B_OFF);
                    float4* bL = reinterpret_cast<float4*>(st + C::B_OFF + C::B_BYTES);
                    constexpr int NB = (C::B_BYTES / 16 + NCT - 1) / NCT;
                    float4 vb[NB];
#pragma unroll
                    for (int i = 0; i < NB; ++i)
                        if (ct + i * NCT < C::B_BYTES / 16) vb[i] = bH[ct + i * NCT];
#pragma unroll
                    for (int i = 0; i < NB; ++i)
                        if (ct + i * NCT < C::B_BYTES / 16) bL[ct + i * NCT] = lo4(vb[i]);
                    fence_proxy_async_smem();
                    tc_fence_before();
                    mbar_arrive(&aux->conv[ts]);
                }
                if (++s == C::STAGES) {
                    s = 0;
                    ++r;
                }
            }
        }
    } else {
        // ======================= epilogue warps 0-7: quadrant q = position 4j+q, lane = image
        const int qd = warp & 3, half = warp >> 2;
        constexpr int HALF = BN / 2;
        const uint32_t lane_addr = (uint32_t)(qd * 32) << 16;
        uint8_t* const stg = tiles_ptr + C::STAGES * C::STAGE_BYTES + 1024 + warp * (32 * C::EPW * 4);
        const bool coal = C::EPW > 0 && (sp.coalesce || p.epi.mode != EPI_NONE);  // as conv_tma.cuh
        uint32_t c = 0;
        for (int w = wfirst; w < sp.work; w += wstep) {
            StripTile t;
            t.init(sp, w, rank);
            const int nkb = strip_rows<OP>(sp, p, t.orow) * sp.CB;
            const int nch = nkb > 0 ? (nkb + CHK - 1) / CHK : 0;
            const int n0 = t.nt * BN;
            const int img = t.g * 32 + lane;
            long long obase[R];
#pragma unroll
            for (int j = 0; j < R; ++j) {
                const int ocol = t.s * 4 * R + 4 * j + qd;
                obase[j] = (ocol < sp.OWo && img < p.N)
                               ? ((long long)(img * sp.OHo + t.orow) * sp.OWo + ocol) * p.Ngemm
                               : -1;
            }
            float* outp = p.out;
            if (PLANES == 2) {
                float acc[R][HALF];
#pragma unroll
                for (int j = 0; j < R; ++j)
#pragma unroll
                    for (int e = 0; e < HALF; ++e) acc[j][e] = 0.f;
                for (int k = 0; k < nch; ++k, ++c) {
                    const int buf = c & 1;
                    if (PAIR) mbar_wait_cluster(&aux->tfull[buf], (c >> 1) & 1);
                    else mbar_wait(&aux->tfull[buf], (c >> 1) & 1);
                    tc_fence_after();
#pragma unroll
                    for (int j = 0; j < R; ++j)
#pragma unroll
                        for (int c0 = 0; c0 < HALF; c0 += 16) {
                            uint32_t v[16];
                            tmem_ld_32x32b_x16(tmem + lane_addr + (uint32_t)((buf * R + j) * BN + half * HALF + c0), v);
                            tmem_ld_wait();
#pragma unroll
                            for (int e = 0; e < 16; ++e) acc[j][c0 + e] += __uint_as_float(v[e]);
                        }
                    tc_fence_before();
                    if (PAIR) {
                        __syncwarp();
                        if (lane == 0) mbar_arrive_remote(&aux->tempty[buf], 0);
                    } else {
                        mbar_arrive(&aux->tempty[buf]);
                    }
                }
                bool stored = false;
                if constexpr (C::EPW > 0) {
                    if (coal) {
#pragma unroll
                        for (int j = 0; j < R; ++j)
#pragma unroll
                            for (int c0 = 0; c0 < HALF; c0 += C::EPW) {
                                const int col0 = n0 + half * HALF + c0;
                                if (p.epi.mode != EPI_NONE) {  // in place on acc, 16 columns at a time
#pragma unroll
                                    for (int q = 0; q < C::EPW; q += 16)
                                        epi_apply16(p.epi, *reinterpret_cast<float(*)[16]>(&acc[j][c0 + q]),
                                                    obase[j] >= 0 && col0 + q < p.Ngemm ? obase[j] + col0 + q : -1,
                                                    col0 + q, p.Ngemm, strip_grp<R>(sp, t, j, qd), lane);
                                }
                                if (sp.tstore) {
                                    const int ocol = t.s * 4 * R + 4 * j + qd;
                                    warp_rows_tstore<C::EPW>(stg, *reinterpret_cast<const float(*)[C::EPW]>(&acc[j][c0]), &sp.mapY,
                                                             col0, t.orow * sp.OWo + ocol, t.g * 32, ocol < sp.OWo, lane);
                                } else {
                                    warp_rows_store<C::EPW>(stg, *reinterpret_cast<const float(*)[C::EPW]>(&acc[j][c0]), obase[j],
                                                            outp, col0, p.Ngemm, 0, lane);
                                }
                            }
                        stored = true;
                    }
                }
                if (stored) {
                } else if (C::EPW == 0 && p.epi.mode != EPI_NONE) {  // fused epilogue (epilogue.cuh)
#pragma unroll
                    for (int j = 0; j < R; ++j)
#pragma unroll
                        for (int c0 = 0; c0 < HALF; c0 += 16) {
                            const int col0 = n0 + half * HALF + c0;
                            float v[16];
#pragma unroll
                            for (int e = 0; e < 16; ++e) v[e] = acc[j][c0 + e];
                            epi_apply16(p.epi, v, obase[j] >= 0 && col0 < p.Ngemm ? obase[j] + col0 : -1, col0, p.Ngemm,
                                        strip_grp<R>(sp, t, j, qd), lane);
                            if (obase[j] >= 0)
#pragma unroll
                                for (int e = 0; e < 16; e += 4)
                                    if (col0 + e < p.Ngemm)
                                        *reinterpret_cast<float4*>(outp + obase[j] + col0 + e) =
                                            make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
                        }
                } else {
#pragma unroll
                for (int j = 0; j < R; ++j)
                    if (obase[j] >= 0)
#pragma unroll
                        for (int e = 0; e < HALF; e += 4) {
                            const int col = n0 + half * HALF + e;
                            if (col < p.Ngemm)
                                *reinterpret_cast<float4*>(outp + obase[j] + col) =
                                    make_float4(acc[j][e], acc[j][e + 1], acc[j][e + 2], acc[j][e + 3]);
                        }
                }
            } else {
                const int buf = c & 1;
                if (nch > 0) {
                    mbar_wait(&aux->tfull[buf], (c >> 1) & 1);
                    tc_fence_after();
                }
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    if constexpr (C::EPW > 0) {
                        if (coal) {
#pragma unroll 1
                            for (int c0 = 0; c0 < HALF; c0 += C::EPW) {
                                float f[C::EPW];
                                if (nch > 0) {
                                    uint32_t v[C::EPW];
#pragma unroll
                                    for (int q = 0; q < C::EPW / 16; ++q)
                                        tmem_ld_32x32b_x16(tmem + lane_addr + (uint32_t)((buf * R + j) * BN + half * HALF + c0 + 16 * q),
                                                           *reinterpret_cast<uint32_t(*)[16]>(&v[16 * q]));
                                    tmem_ld_wait();
#pragma unroll
                                    for (int e = 0; e < C::EPW; ++e) f[e] = __uint_as_float(v[e]);
                                } else {
#pragma unroll
                                    for (int e = 0; e < C::EPW; ++e) f[e] = 0.f;
                                }
                                const int col0 = n0 + half * HALF + c0;
                                if (p.epi.mode != EPI_NONE) {
#pragma unroll
                                    for (int q = 0; q < C::EPW; q += 16) {
                                        float v[16];
#pragma unroll
                                        for (int e = 0; e < 16; ++e) v[e] = f[q + e];
                                        epi_apply16(p.epi, v,
                                                    obase[j] >= 0 && col0 + q < p.Ngemm ? obase[j] + col0 + q : -1,
                                                    col0 + q, p.Ngemm, strip_grp<R>(sp, t, j, qd), lane);
#pragma unroll
                                        for (int e = 0; e < 16; ++e) f[q + e] = v[e];
                                    }
                                }
                                if (sp.tstore) {
                                    const int ocol = t.s * 4 * R + 4 * j + qd;
                                    warp_rows_tstore<C::EPW>(stg, f, &sp.mapY, col0, t.orow * sp.OWo + ocol, t.g * 32,
                                                             ocol < sp.OWo, lane);
                                } else {
                                    warp_rows_store<C::EPW>(stg, f, obase[j], outp, col0, p.Ngemm, 0, lane);
                                }
                            }
                            continue;
                        }
                    }
#pragma unroll 1
                    for (int c0 = 0; c0 < HALF; c0 += 16) {
                        uint32_t v[16];
                        if (nch > 0) {
                            tmem_ld_32x32b_x16(tmem + lane_addr + (uint32_t)((buf * R + j) * BN + half * HALF + c0), v);
                            tmem_ld_wait();
                        } else {
#pragma unroll
                            for (int e = 0; e < 16; ++e) v[e] = 0u;
                        }
                        if (C::EPW == 0 && p.epi.mode != EPI_NONE) {  // fused epilogue (epilogue.cuh)
                            const int col0 = n0 + half * HALF + c0;
                            float f[16];
#pragma unroll
                            for (int e = 0; e < 16; ++e) f[e] = __uint_as_float(v[e]);
                            epi_apply16(p.epi, f, obase[j] >= 0 && col0 < p.Ngemm ? obase[j] + col0 : -1, col0,
                                        p.Ngemm, strip_grp<R>(sp, t, j, qd), lane);
#pragma unroll
                            for (int e = 0; e < 16; ++e) v[e] = __float_as_uint(f[e]);
                        }
                        if (obase[j] >= 0)
#pragma unroll
                            for (int e = 0; e < 16; e += 4) {
                                const int col = n0 + half * HALF + c0 + e;
                                if (col < p.Ngemm)
                                    *reinterpret_cast<float4*>(outp + obase[j] + col) =
                                        make_float4(__uint_as_float(v[e]), __uint_as_float(v[e + 1]),
                                                    __uint_as_float(v[e + 2]), __uint_as_float(v[e + 3]));
                            }
                    }
                }
                if (nch > 0) {
                    tc_fence_before();
                    mbar_arrive(&aux->tempty[buf]);
                    ++c;
                }
            }
        }
    }

strip_done:
    if (warp < C::NEPI && lane == 0 && sp.tstore) bulk_wait_group0();  // the epilogue's TMA stores are done
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync_all();  // the peer's MMAs / arrivals are done before TMEM is released
    if (warp == C::MMA_W) {
        tc_fence_after();
        if (PAIR) tmem_dealloc2(tmem, C::TMEM_COLS);
        else tmem_dealloc(tmem, C::TMEM_COLS);
    }
}

bool strip_supported(int op, int N, int IC, int OC, int FW, int sh, int sw, int OWo, int BN, int planes);
int strip_launch(int op, int BN, int planes, const GenParams& g, cudaStream_t st, char* err, size_t errlen);
int strip_R(int BN, int planes);
bool strip_pair(int op, int N, int BN, int planes);

}  // namespace smconv
