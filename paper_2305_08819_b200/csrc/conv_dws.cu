// conv_dws.cu — DWS variant: weight gradient (O3; PAPER.md's deconvolution-side
// "dW = X^T (*) dY", north_star step (a)) of 3x3 stride-1 convolutions with 64 input and 64 output
// channels on 8/16/32-wide maps: ResNet-18 stage 1 and VGG conv2, the largest dW calls of the step.
//
// Why a separate kernel.  The transposed dW GEMM of the TMA variant ((tap, ic) rows x oc columns,
// K = pixels) gives every 128-row tile its own X operand: each X pixel crosses L2 -> SM nine times
// (once per tap) and every dY k-block five times (once per m-tile), 24 KB per 128x64x32 block.
// ncu on l1 dW: 15 GB L2->SM per call (7x the 2.1 GB compulsory), tensor pipe 51 % busy, the
// converters waiting on TMA data; prefetching made it slower (L2-throughput bound, not latency).
//
// Here a k-block is 32 CONSECUTIVE pixels of one image (RB = 32/OW output rows x OW columns) and
// a work item is a group of 4 taps (2 m-tiles of 2 taps x 64 ic) sharing ONE staged dY block and
// ONE activation slab: the RB+1 source rows x (OW+2) columns x 64 channels that all its taps read
// (4 consecutive taps of a 3x3 filter span at most 2 filter rows).  The A operand of tap (fh, fw)
// is the slab shifted by (fh - fh_lo) rows and fw columns; the 3xTF32 converter warps, which
// read A from shared memory anyway to split it into hi/lo planes in TMEM, apply the shift in
// their address arithmetic, so the shift costs nothing.  L2->SM bytes per 128x64x32 block drop
// from 24 KB to ~12.5 KB.  Groups: taps {0-3}, {4-7}, {8} (the last a half-empty m-tile).
//
// Pipelines: a shared-memory ring of SS stages (dY hi, dY lo, slab; freed by the MMA commit)
// is decoupled from a TMEM ring of ST A-slots (freed by the MMA commit, filled by the converters),
// so the TMA look-ahead is not capped by TMEM.  Accumulators (2 x 64 columns) are single
// buffered: the MMA warp waits for the epilogue to drain a promotion chunk (3xTF32: every
// chunk_kb k-blocks into fp32 registers, the truncating TMEM accumulation is bounded as in
// conv_tma.cuh).  Partials per split go to the workspace; splitk_reduce_kernel sums them in
// fixed order (deterministic).
//
// 3xTF32 (HYB, the default): per m-tile and k-block a_hi*b_hi as 4 TF32 MMAs and the cross terms
// a_hi*b_lo + a_lo*b as 4 bf16 MMAs (K' = 64) on A' = [bf16(a_hi) | bf16(a_lo)] (TMEM, written by
// the converters next to a_hi) and B' = [bf16(b_lo) | bf16(b)] (a bf16 MN-major plane the
// converters build from the dY tile in place of the old b_lo plane; common.cuh "3xTF32 operand
// split"): 8 MMAs of tensor-pipe time per m-tile and k-block instead of 12.  HYB = false keeps
// the three-TF32-MMA form (SMCONV_DWS_HYB=0, A/B and fallback).
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cudaTypedefs.h>

#include "../../include/smconv.h"
#include "conv_tma.cuh"
#include "launch.cuh"

namespace smconv {

bool tma_encode_f32(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                    const uint32_t* box, CUtensorMapSwizzle sw);  // conv_tma.cu

struct __align__(64) DwsParams {
    CUtensorMap mapXA;  // X (IC, IW, IH, N), no swizzle, box 1 source row: [XW][64 ch] (256-B rows)
    CUtensorMap mapXB;  // the same view, box RB rows: [RB][XW][64 ch]
    CUtensorMap mapY;  // dY viewed (32 oc, OW, OH, N, OC/32), 128B/32B-atom swizzle: MN-major B
    int OW, RB, XW, ohb;  // k-block = RB output rows x OW (RB * OW == 32); XW = OW + 2; ohb = OH / RB
    int cbs;              // wide maps (OW = 64, 128, 224, ...: kernel geometry of OW = 32): column blocks of 32
                          // per output row; k-block = (image, column block, output row), rows innermost
    int kb_total, kb_per_split, splits, work, chunk_kb;
    int ph, pw;
    int alt_conv;  // converter warps in two groups on alternate k-blocks (one-CTA kernel, not the hybrid form)
};

constexpr int kDwsGroups = 3;  // taps {0..3}, {4..7}, {8}
constexpr int kDwsTaps = 9;

template <int PLANES, int OW>
struct DwsCfg {
    // B' plane of the bf16 cross terms: [K' = 64][64 oc] bf16, MN-major SWIZZLE_128B (8-row x 128-B
    // atoms, SBO 1024), the same 8 KB as the fp32 b_lo plane it replaces
    static constexpr int YX_BYTES = 64 * 64 * 2;
    static constexpr int RB = 32 / OW, XW = OW + 2;  // k-block rows; slab columns
    static constexpr int BN = 64;                    // OC
    static constexpr int Y_BYTES = BN * 32 * 4;      // dY k-block [2 ocb][32 px][32 oc]
    static constexpr int Y_OFF_LO = Y_BYTES;         // b_lo plane (3xTF32)
    // activation slab rows [XW][64 ch]: 256-B TMA rows (a [32-ch block][XW][32] box issued 2x as many
    // 128-B requests, and the request count, not the bytes, bounded the skeleton pipeline)
    static constexpr int ROW_BYTES = XW * 256;       // one source row, all 64 channels
    static constexpr int XA_OFF = PLANES * Y_BYTES;  // slab row 0 (loaded only when fresh)
    static constexpr int XA_BYTES = ROW_BYTES;
    static constexpr int XB_OFF = XA_OFF + XA_BYTES;  // slab rows 1..RB
    static constexpr int XB_BYTES = RB * ROW_BYTES;
    static constexpr int STAGE_BYTES = ((XB_OFF + XB_BYTES + 1023) / 1024) * 1024;
    static constexpr int SS_RAW = (200 * 1024) / STAGE_BYTES;
    static constexpr int SS = SS_RAW > 8 ? 8 : SS_RAW;
    static constexpr int ACC_COLS = 128;             // 2 m-tiles x 64 fp32 columns, single buffer
    static constexpr int TILE_COLS = 32 * PLANES;    // one m-tile's A per k-block: hi 32 (| lo 32) columns
    static constexpr int SLOT_COLS = 2 * TILE_COLS;  // 2 m-tiles
    static constexpr int ST = (512 - ACC_COLS) / SLOT_COLS;  // 3 (3xTF32) / 6 (TF32)
    static constexpr int NEPI = 8, TMA_W = 8, MMA_W = 9, CONV_W0 = 10, NCONV = 8;
    static constexpr int NTHREADS = (10 + NCONV) * 32;
    static constexpr int SMEM_BYTES = 1024 + SS * STAGE_BYTES + 1024;
    static_assert(SS >= 2 && ST >= 2, "DWS pipeline does not fit");
};

struct DwsAux {
    uint64_t full[8], empty[8];
    uint64_t conv[16], tfree[8];
    uint64_t tfull, tempty;
    uint32_t tmem_base;
};

struct DwsItem {
    int split, g, ntile, fh_lo, kb0, kb1;
    SMCONV_DEV void init(const DwsParams& dp, int w) {
        split = w / kDwsGroups;  // split outermost: the 3 groups of one pixel range run together (L2 reuse)
        g = w - split * kDwsGroups;
        ntile = g < 2 ? 2 : 1;
        fh_lo = (4 * g) / 3;
        kb0 = split * dp.kb_per_split;
        kb1 = min(dp.kb_total, kb0 + dp.kb_per_split);
        if (kb1 < kb0) kb1 = kb0;
    }
};

// byte offset of bf16 elements (k, mn..mn+3), mn % 4 == 0, in a [K][64] MN-major SWIZZLE_128B tile
SMCONV_DEV uint32_t mnmaj16_off(uint32_t k, uint32_t mn) {
    return (k >> 3) * 1024u + (k & 7u) * 128u + ((((mn >> 3) & 7u) ^ (k & 7u)) << 4) + (mn & 7u) * 2u;
}

template <int PLANES, int OW, bool HYB>
__global__ void __launch_bounds__(DwsCfg<PLANES, OW>::NTHREADS, 1)
    conv_dws_kernel(const __grid_constant__ DwsParams dp, const __grid_constant__ GenParams p) {
    using C = DwsCfg<PLANES, OW>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    const uint32_t tiles_addr = (raw_addr + 1023u) & ~1023u;
    uint8_t* tiles_ptr = smem_raw + (tiles_addr - raw_addr);
    DwsAux* aux = reinterpret_cast<DwsAux*>(tiles_ptr + C::SS * C::STAGE_BYTES);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int CHK = PLANES == 2 ? dp.chunk_kb : (1 << 30);

    if (tid == 0) {
        for (int s = 0; s < C::SS; ++s) {
            mbar_init(&aux->full[s], 1);
            // MMA commit + next k-block's converter warps (DwsParams::alt_conv: one group of NCONV / 2)
            mbar_init(&aux->empty[s], 1 + (dp.alt_conv ? C::NCONV / 2 : C::NCONV));
        }
        for (int t = 0; t < C::ST; ++t) {
            // one barrier per (slot, m-tile): the MMAs of m-tile 0 start while m-tile 1 is being split;
            // one elected arrival per converter warp
            mbar_init(&aux->conv[2 * t], dp.alt_conv ? C::NCONV / 2 : C::NCONV);
            mbar_init(&aux->conv[2 * t + 1], dp.alt_conv ? C::NCONV / 2 : C::NCONV);
            mbar_init(&aux->tfree[t], 1);
        }
        mbar_init(&aux->tfull, 1);
        mbar_init(&aux->tempty, C::NEPI);
        fence_mbar_init();
    }
    if (warp == C::TMA_W && lane == 0) {
        prefetch_tmap(&dp.mapXA);
        prefetch_tmap(&dp.mapXB);
        prefetch_tmap(&dp.mapY);
    }
    if (warp == C::MMA_W) tmem_alloc(&aux->tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = aux->tmem_base;
    pdl_trigger();
    pdl_wait();  // launch.cuh

    if (warp == C::TMA_W) {
        // ======================= TMA producer: per k-block one dY box + one activation slab box
        int s = 0;
        uint32_t r = 0;
        for (int w = blockIdx.x; w < dp.work; w += gridDim.x) {
            DwsItem it;
            it.init(dp, w);
            for (int kb = it.kb0; kb < it.kb1; ++kb) {
                if (r > 0) mbar_wait(&aux->empty[s], (r - 1) & 1);
                const int ncb = kb / dp.ohb, oh0 = (kb - ncb * dp.ohb) * dp.RB;
                const int n = ncb / dp.cbs, cb = ncb - n * dp.cbs, ow0 = cb * 32;  // cbs == 1: ow0 = 0
                // slab rows: ih0 + 0 .. ih0 + RB.  Row 0 equals the previous k-block's last row when that
                // k-block is the previous output rows of the same image: then only rows 1..RB are loaded
                // and the converters read row 0 from the previous stage (1 of 2 rows saved at OW = 32).
                const int ih0 = oh0 + it.fh_lo - dp.ph;
                const bool fresh = (kb == it.kb0) || (oh0 == 0);
                const uint32_t sY = tiles_addr + s * C::STAGE_BYTES;
                if (elect_one()) {
                    mbar_arrive_expect_tx(&aux->full[s], C::Y_BYTES + C::XB_BYTES + (fresh ? C::XA_BYTES : 0));
                    tma_load_5d(sY, &dp.mapY, &aux->full[s], 0, ow0, oh0, n, 0);
                    tma_load_4d(sY + C::XB_OFF, &dp.mapXB, &aux->full[s], 0, ow0 - dp.pw, ih0 + 1, n);
                    if (fresh) tma_load_4d(sY + C::XA_OFF, &dp.mapXA, &aux->full[s], 0, ow0 - dp.pw, ih0, n);
                }
                __syncwarp();
                if (++s == C::SS) {
                    s = 0;
                    ++r;
                }
            }
        }
    } else if (warp == C::MMA_W) {
        // ======================= MMA issuer: ntile m-tiles x 4 k-steps (x3 for 3xTF32) per k-block
        constexpr uint32_t IDESC = idesc_tf32(128, C::BN, false, true);  // A from TMEM, B (dY) MN-major
        constexpr uint32_t IDESC_X = idesc_bf16(128, C::BN, false, true);
        const uint64_t bd0 = make_sdesc(tiles_addr, 4096u, 512u, kLayoutSW128Base32);
        const uint64_t bx0 = make_sdesc(tiles_addr + C::Y_OFF_LO, 8192u, 1024u, kLayoutSW128);  // B' plane
        constexpr uint64_t B_LO = C::Y_BYTES >> 4;
        uint32_t q = 0, c = 0;
        int in_chunk = 0;
        for (int w = blockIdx.x; w < dp.work; w += gridDim.x) {
            DwsItem it;
            it.init(dp, w);
            const int nkb = it.kb1 - it.kb0;
            for (int i = 0; i < nkb; ++i, ++q) {
                const uint32_t s = q % C::SS, t = q % C::ST, rt = q / C::ST;
                if (in_chunk == 0 && c >= 1) {
                    mbar_wait(&aux->tempty, (c - 1) & 1);  // epilogue drained the previous chunk
                    tc_fence_after();
                }
                const bool last = (in_chunk + 1 == CHK || i == nkb - 1);
                {
                    const uint64_t so = (uint64_t)(s * C::STAGE_BYTES) >> 4;
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        // both barriers complete once per k-block (also for 1-tile items), so their
                        // phase parity stays rt & 1
                        mbar_wait(&aux->conv[2 * t + j], rt & 1);
                        tc_fence_after();
                        if (j < it.ntile && elect_one()) {
                            const uint32_t d = tmem + (uint32_t)(j * C::BN);
#pragma unroll
                            for (int g4 = 0; g4 < 4; ++g4) {
                                const uint64_t bdH = bd0 + so + g4 * 64;  // 8 K-rows x 128 B
                                const uint32_t acc0 = (in_chunk > 0 || g4 > 0) ? 1u : 0u;
                                const uint32_t ahi = tmem + (uint32_t)(C::ACC_COLS + t * C::SLOT_COLS + j * C::TILE_COLS + g4 * 8);
                                if (PLANES == 2 && HYB) {
                                    mma_tf32_ts(d, ahi, bdH, IDESC, acc0);  // a_hi * b_hi
                                } else if (PLANES == 2) {
                                    mma_tf32_ts(d, ahi + 32, bdH, IDESC, acc0);  // a_lo * b_hi
                                    mma_tf32_ts(d, ahi, bdH + B_LO, IDESC, 1u);  // a_hi * b_lo
                                    mma_tf32_ts(d, ahi, bdH, IDESC, 1u);         // a_hi * b_hi
                                } else {
                                    mma_tf32_ts(d, ahi, bdH, IDESC, acc0);
                                }
                            }
                            if (PLANES == 2 && HYB) {
                                // cross terms: A' columns [32, 64) of the m-tile's slot, B' rows 16 j..16 j+15
#pragma unroll
                                for (int j4 = 0; j4 < 4; ++j4) {
                                    const uint32_t ax = tmem + (uint32_t)(C::ACC_COLS + t * C::SLOT_COLS + j * C::TILE_COLS + 32 + j4 * 8);
                                    mma_bf16_ts(d, ax, bx0 + so + j4 * (2048 >> 4), IDESC_X, 1u);
                                }
                            }
                        }
                        __syncwarp();
                    }
                    if (elect_one()) {
                        mma_commit(&aux->empty[s]);
                        mma_commit(&aux->tfree[t]);
                        if (last) mma_commit(&aux->tfull);
                    }
                }
                __syncwarp();
                if (last) {
                    ++c;
                    in_chunk = 0;
                } else {
                    ++in_chunk;
                }
            }
        }
    } else if (warp >= C::CONV_W0 && dp.alt_conv) {
        // ======================= converters, two groups of 4 warps on alternate k-blocks (DwsParams::alt_conv):
        // a warp = one TMEM lane quadrant, both K halves of both m-tiles of its k-block.  With all 8 warps on
        // every k-block the per-k-block chain LDS -> split -> tcgen05.st -> wait -> arrive ran one k-block at a
        // time (the pair kernel: 2.59 -> 2.02 ms with the groups, r02bx)
        const int grp = (warp - C::CONV_W0) >> 2;
        const int ct4 = tid - (C::CONV_W0 + 4 * grp) * 32;  // 0..127 within the group
        const int qd = warp & 3;
        const int ts = qd >> 1, icb = qd & 1;
        uint32_t q = 0;
        for (int w = blockIdx.x; w < dp.work; w += gridDim.x) {
            DwsItem it;
            it.init(dp, w);
            const int nkb = it.kb1 - it.kb0;
            for (int i = 0; i < nkb; ++i, ++q) {
                if ((int)(q & 1u) != grp) continue;
                const uint32_t s = q % C::SS, rs = q / C::SS, t = q % C::ST, rt = q / C::ST;
                const uint32_t sp = (s + C::SS - 1) % C::SS;
                const int kb = it.kb0 + i;
                const bool fresh = (i == 0) || (kb % dp.ohb == 0);
                mbar_wait(&aux->full[s], rs & 1);
                // slab row 0 of a non-fresh k-block is the previous stage's last row, loaded for the OTHER group
                if (!fresh) mbar_wait(&aux->full[sp], ((q - 1) / C::SS) & 1);
                uint8_t* st = tiles_ptr + s * C::STAGE_BYTES;
                if (PLANES == 2 && HYB) {  // B' = [bf16(b_lo) ; bf16(b)] MN-major plane from the dY k-block
#pragma unroll
                    for (int e2 = 0; e2 < 4; ++e2) {
                        const uint32_t i = (uint32_t)(ct4 + 128 * e2);
                        const uint32_t k = (i & 255u) >> 3, c32 = (i & 7u) >> 1;
                        const uint32_t mn = (i >> 8) * 32u + ((c32 ^ (k & 3u)) << 3) + ((i & 1u) << 2);
                        const float4 b = reinterpret_cast<const float4*>(st)[i];
                        const float l0 = b.x - __uint_as_float(__float_as_uint(b.x) & 0xFFFFE000u);
                        const float l1 = b.y - __uint_as_float(__float_as_uint(b.y) & 0xFFFFE000u);
                        const float l2 = b.z - __uint_as_float(__float_as_uint(b.z) & 0xFFFFE000u);
                        const float l3 = b.w - __uint_as_float(__float_as_uint(b.w) & 0xFFFFE000u);
                        *reinterpret_cast<uint2*>(st + C::Y_OFF_LO + mnmaj16_off(k, mn)) =
                            make_uint2(pack_bf16x2(l0, l1), pack_bf16x2(l2, l3));
                        *reinterpret_cast<uint2*>(st + C::Y_OFF_LO + mnmaj16_off(k + 32u, mn)) =
                            make_uint2(pack_bf16x2(b.x, b.y), pack_bf16x2(b.z, b.w));
                    }
                } else if (PLANES == 2) {  // b_lo of the dY k-block (8 KB: four float4 per thread of the group)
#pragma unroll
                    for (int e2 = 0; e2 < 4; ++e2) {
                        const float4 v = reinterpret_cast<const float4*>(st)[ct4 + 128 * e2];
                        float4 o;
                        o.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
                        o.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
                        o.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
                        o.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
                        reinterpret_cast<float4*>(st + C::Y_OFF_LO)[ct4 + 128 * e2] = o;
                    }
                }
                const uint8_t* row0 = fresh ? st + C::XA_OFF
                                            : tiles_ptr + sp * C::STAGE_BYTES + C::XB_OFF + (C::RB - 1) * C::ROW_BYTES;
                const uint8_t* row1 = st + C::XB_OFF;
                if (rt > 0) mbar_wait(&aux->tfree[t], (rt - 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    if (j < it.ntile) {
                        const int tap = 4 * it.g + 2 * j + ts;
                        const int fh = tap / 3, fw = tap - 3 * fh;
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            uint32_t hi[16], lo[16];
                            float ev[16];
                            const int bsr = tap < kDwsTaps ? fh - it.fh_lo + (16 * h) / OW : -1;
                            const int coff = (fw + (16 * h) % OW) * 256 + icb * 128 + lane * 4;
                            if (bsr >= 0) {
                                const uint8_t* p0 = (bsr == 0 ? row0 : row1 + (bsr - 1) * C::ROW_BYTES) + coff;
                                const uint8_t* p1 = row1 + bsr * C::ROW_BYTES + coff;
#pragma unroll
                                for (int k = 0; k < 16; ++k) {
                                    const float e = (k / OW == 0)
                                                        ? *reinterpret_cast<const float*>(p0 + (k % OW) * 256)
                                                        : *reinterpret_cast<const float*>(
                                                              p1 + (k / OW - 1) * C::ROW_BYTES + (k % OW) * 256);
                                    ev[k] = e;
                                    if (PLANES == 2) {
                                        const uint32_t hb = __float_as_uint(e) & 0xFFFFE000u;
                                        hi[k] = hb;
                                        lo[k] = __float_as_uint(e - __uint_as_float(hb));
                                    } else {
                                        hi[k] = __float_as_uint(e);
                                        lo[k] = 0u;
                                    }
                                }
                            } else {
#pragma unroll
                                for (int k = 0; k < 16; ++k) {  // half-empty last m-tile
                                    hi[k] = lo[k] = 0u;
                                    ev[k] = 0.f;
                                }
                            }
                            const uint32_t tb = tmem + ((uint32_t)(qd * 32) << 16) +
                                                (uint32_t)(C::ACC_COLS + t * C::SLOT_COLS + j * C::TILE_COLS);
                            if (PLANES == 2 && HYB) {
                                // slot columns [0,32) a_hi, [32,48) bf16(a_hi) pairs, [48,64) bf16(a_lo) pairs
                                uint32_t xh[8], xl[8];
                                split_a16(ev, hi, xh, xl);
                                tmem_st_32x32b_x16(tb + h * 16, hi);
                                tmem_st_32x32b_x8(tb + 32 + h * 8, xh);
                                tmem_st_32x32b_x8(tb + 48 + h * 8, xl);
                            } else {
                                tmem_st_32x32b_x16(tb + h * 16, hi);
                                if (PLANES == 2) tmem_st_32x32b_x16(tb + 32 + h * 16, lo);
                            }
                        }
                        tmem_st_wait();
                    }
                    if (j == 0) fence_proxy_async_smem();  // b_lo (written above) before the first release
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&aux->conv[2 * t + j]);  // per warp; also for empty m-tiles
                }
                __syncwarp();
                if (lane == 0 && q > 0) mbar_arrive(&aux->empty[sp]);  // previous stage: its row RB was read
            }
        }
    } else if (warp >= C::CONV_W0) {
        // ======================= converters: shifted slab rows -> A hi/lo in TMEM; dY -> b_lo in smem
        const int ct = tid - C::CONV_W0 * 32;
        const int qd = warp & 3, h = (warp - C::CONV_W0) >> 2;  // TMEM lane quadrant, K half
        const int ts = qd >> 1, icb = qd & 1;                      // row 32qd+lane = (tap slot ts, ic 32icb+lane)
        uint32_t q = 0;
        for (int w = blockIdx.x; w < dp.work; w += gridDim.x) {
            DwsItem it;
            it.init(dp, w);
            const int nkb = it.kb1 - it.kb0;
            // per item and m-tile: first slab row of this thread's K half (-1: no tap), column offset
            int bsr[2], coff[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int tap = 4 * it.g + 2 * j + ts;
                const int fh = tap / 3, fw = tap - 3 * fh;
                bsr[j] = (j < it.ntile && tap < kDwsTaps) ? fh - it.fh_lo + (16 * h) / OW : -1;
                coff[j] = (fw + (16 * h) % OW) * 256 + icb * 128 + lane * 4;
            }
            for (int i = 0; i < nkb; ++i, ++q) {
                const uint32_t s = q % C::SS, rs = q / C::SS, t = q % C::ST, rt = q / C::ST;
                const uint32_t sp = (s + C::SS - 1) % C::SS;  // previous k-block's stage
                const int kb = it.kb0 + i;
                const bool fresh = (i == 0) || (kb % dp.ohb == 0);
                mbar_wait(&aux->full[s], rs & 1);
                uint8_t* st = tiles_ptr + s * C::STAGE_BYTES;
                if (PLANES == 2) {  // b_lo needs only the stage: done before the TMEM-slot wait
                    const float4* bH = reinterpret_cast<const float4*>(st);
                    float4* bL = reinterpret_cast<float4*>(st + C::Y_OFF_LO);
                    constexpr int NB = C::Y_BYTES / 16 / (C::NCONV * 32);
                    float4 v[NB];
#pragma unroll
                    for (int e = 0; e < NB; ++e) v[e] = bH[ct + e * C::NCONV * 32];
#pragma unroll
                    for (int e = 0; e < NB && HYB; ++e) {
                        // float4 i of the fp32 MN-major tile: oc block i / 256, K-row (i % 256) / 8,
                        // 32-B chunk (i % 8) / 2 (swizzled with k % 4), 16-B half i % 2
                        const uint32_t i = (uint32_t)(ct + e * C::NCONV * 32);
                        const uint32_t k = (i & 255u) >> 3, c32 = (i & 7u) >> 1;
                        const uint32_t mn = (i >> 8) * 32u + ((c32 ^ (k & 3u)) << 3) + ((i & 1u) << 2);
                        const float4 b = v[e];
                        const float l0 = b.x - __uint_as_float(__float_as_uint(b.x) & 0xFFFFE000u);
                        const float l1 = b.y - __uint_as_float(__float_as_uint(b.y) & 0xFFFFE000u);
                        const float l2 = b.z - __uint_as_float(__float_as_uint(b.z) & 0xFFFFE000u);
                        const float l3 = b.w - __uint_as_float(__float_as_uint(b.w) & 0xFFFFE000u);
                        *reinterpret_cast<uint2*>(st + C::Y_OFF_LO + mnmaj16_off(k, mn)) =
                            make_uint2(pack_bf16x2(l0, l1), pack_bf16x2(l2, l3));
                        *reinterpret_cast<uint2*>(st + C::Y_OFF_LO + mnmaj16_off(k + 32u, mn)) =
                            make_uint2(pack_bf16x2(b.x, b.y), pack_bf16x2(b.z, b.w));
                    }
#pragma unroll
                    for (int e = 0; e < NB && !HYB; ++e) {
                        float4 o;
                        o.x = v[e].x - __uint_as_float(__float_as_uint(v[e].x) & 0xFFFFE000u);
                        o.y = v[e].y - __uint_as_float(__float_as_uint(v[e].y) & 0xFFFFE000u);
                        o.z = v[e].z - __uint_as_float(__float_as_uint(v[e].z) & 0xFFFFE000u);
                        o.w = v[e].w - __uint_as_float(__float_as_uint(v[e].w) & 0xFFFFE000u);
                        bL[ct + e * C::NCONV * 32] = o;
                    }
                }
                // slab row 0: this stage's row-0 buffer when fresh, else the previous stage's last row
                const uint8_t* row0 = fresh ? st + C::XA_OFF
                                            : tiles_ptr + sp * C::STAGE_BYTES + C::XB_OFF + (C::RB - 1) * C::ROW_BYTES;
                const uint8_t* row1 = st + C::XB_OFF;  // slab row 1
                if (rt > 0) mbar_wait(&aux->tfree[t], (rt - 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    if (j < it.ntile) {
                        uint32_t hi[16], lo[16];
                        float ev[16];
                        if (bsr[j] >= 0) {
                            const uint8_t* p0 = (bsr[j] == 0 ? row0 : row1 + (bsr[j] - 1) * C::ROW_BYTES) + coff[j];
                            const uint8_t* p1 = row1 + bsr[j] * C::ROW_BYTES + coff[j];  // rows after the first
#pragma unroll
                            for (int k = 0; k < 16; ++k) {  // pixel 16h + k: row k / OW (relative), column k % OW
                                const float e = (k / OW == 0)
                                                    ? *reinterpret_cast<const float*>(p0 + (k % OW) * 256)
                                                    : *reinterpret_cast<const float*>(
                                                          p1 + (k / OW - 1) * C::ROW_BYTES + (k % OW) * 256);
                                ev[k] = e;
                                if (PLANES == 2) {
                                    const uint32_t hb = __float_as_uint(e) & 0xFFFFE000u;
                                    hi[k] = hb;
                                    lo[k] = __float_as_uint(e - __uint_as_float(hb));
                                } else {
                                    hi[k] = __float_as_uint(e);  // the MMA truncates to TF32
                                    lo[k] = 0u;
                                }
                            }
                        } else {
#pragma unroll
                            for (int k = 0; k < 16; ++k) {  // half-empty last m-tile
                                hi[k] = lo[k] = 0u;
                                ev[k] = 0.f;
                            }
                        }
                        const uint32_t ta = tmem + ((uint32_t)(qd * 32) << 16) +
                                            (uint32_t)(C::ACC_COLS + t * C::SLOT_COLS + j * C::TILE_COLS + h * 16);
                        if (PLANES == 2 && HYB) {
                            // slot columns [0,32) a_hi, [32,48) bf16(a_hi) pairs, [48,64) bf16(a_lo) pairs
                            uint32_t xh[8], xl[8];
                            split_a16(ev, hi, xh, xl);
                            const uint32_t tb = ta - (uint32_t)(h * 16);
                            tmem_st_32x32b_x16(ta, hi);
                            tmem_st_32x32b_x8(tb + 32 + h * 8, xh);
                            tmem_st_32x32b_x8(tb + 48 + h * 8, xl);
                        } else {
                            tmem_st_32x32b_x16(ta, hi);
                            if (PLANES == 2) tmem_st_32x32b_x16(ta + 32, lo);
                        }
                        tmem_st_wait();
                    }
                    if (j == 0) fence_proxy_async_smem();  // b_lo (written above) before the first release
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&aux->conv[2 * t + j]);  // per warp; also for empty m-tiles
                }
                __syncwarp();
                // the previous stage (its last slab row was read above) may be refilled once its own
                // MMAs are done too; the CTA's first k-block has no predecessor
                if (lane == 0 && q > 0) mbar_arrive(&aux->empty[sp]);
            }
        }
    } else {
        // ======================= epilogue warps 0-7: promote chunks, write the split's partial dW
        const int qd = warp & 3, half = warp >> 2;
        const uint32_t lane_addr = (uint32_t)(qd * 32) << 16;
        const int M = kDwsTaps * 64;  // dW row stride per oc: [oc][tap][ic]
        uint32_t c = 0;
        for (int w = blockIdx.x; w < dp.work; w += gridDim.x) {
            DwsItem it;
            it.init(dp, w);
            const int nkb = it.kb1 - it.kb0;
            const int nch = nkb > 0 ? (nkb + CHK - 1) / CHK : 0;
            float acc[2][32];
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int e = 0; e < 32; ++e) acc[j][e] = 0.f;
            for (int k = 0; k < nch; ++k, ++c) {
                mbar_wait(&aux->tfull, c & 1);
                tc_fence_after();
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    if (j < it.ntile) {
#pragma unroll
                        for (int c0 = 0; c0 < 32; c0 += 16) {
                            uint32_t v[16];
                            tmem_ld_32x32b_x16(tmem + lane_addr + (uint32_t)(j * C::BN + half * 32 + c0), v);
                            tmem_ld_wait();
#pragma unroll
                            for (int e = 0; e < 16; ++e) acc[j][c0 + e] += __uint_as_float(v[e]);
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&aux->tempty);
            }
            float* outp = p.out + (long long)it.split * p.split_stride;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int tap = 4 * it.g + 2 * j + (qd >> 1);
                if (j < it.ntile && tap < kDwsTaps) {
                    float* o = outp + tap * 64 + (qd & 1) * 32 + lane + (long long)(half * 32) * M;
#pragma unroll
                    for (int e = 0; e < 32; ++e) o[(long long)e * M] = acc[j][e];  // 32 lanes: 128 contiguous B
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == C::MMA_W) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ------------------------------------------------------------------ CTA-pair form (cta_group::2)
// The 64-channel dW runs N = 64 MMAs, which a single CTA issues at ~60 % of the N = 128 rate, while a CTA
// pair (M = 256) runs them at full rate (tools/pair_bench.cu: 894 vs 507 TFLOP/s TF32 at the power cap).
// Here the two m-tiles of a group are the two CTAs of a cluster: CTA r converts m-tile r (taps 4g+2r,
// 4g+2r+1) into its own TMEM and stages its half of the dY k-block (32 of the 64 output channels); CTA 0
// issues ONE M = 256 MMA per k-step for both.  With one m-tile per CTA a TMEM A slot is 32 * PLANES
// columns, so the converter -> MMA ring is 7 (3xTF32) / 8 (TF32) slots deep instead of 3 / 6 -- the
// single-CTA pair attempt of round 1 (1.82 -> 2.53 ms) kept the shallow ring and stalled on the
// cross-CTA hand-offs.  Group 2 (tap 8) leaves CTA 1's rows empty (1/9 of the work at a quarter of
// the pair's rows).
template <int PLANES, int OW>
struct DwsPairCfg {
    static constexpr int RB = 32 / OW, XW = OW + 2;
    static constexpr int BN = 64;                   // OC (both CTAs)
    static constexpr int Y_BYTES = 32 * 32 * 4;     // this CTA's dY half: [32 px][32 oc]
    static constexpr int Y_OFF_LO = Y_BYTES;
    static constexpr int ROW_BYTES = XW * 256;
    static constexpr int XA_OFF = PLANES * Y_BYTES;
    static constexpr int XA_BYTES = ROW_BYTES;
    static constexpr int XB_OFF = XA_OFF + XA_BYTES;
    static constexpr int XB_BYTES = RB * ROW_BYTES;
    static constexpr int STAGE_BYTES = ((XB_OFF + XB_BYTES + 1023) / 1024) * 1024;
    static constexpr int SS_RAW = (200 * 1024) / STAGE_BYTES;
    static constexpr int SS = SS_RAW > 8 ? 8 : SS_RAW;
    static constexpr int ACC_COLS = 64;             // this CTA's 128 rows x 64 fp32 columns, single buffer
    static constexpr int SLOT_COLS = 32 * PLANES;   // one m-tile's A per k-block: hi 32 (| lo 32)
    static constexpr int ST_RAW = (512 - ACC_COLS) / SLOT_COLS;
    static constexpr int ST = ST_RAW > 8 ? 8 : ST_RAW;
    static constexpr int NEPI = 8, TMA_W = 8, MMA_W = 9, CONV_W0 = 10, NCONV = 8;
    static constexpr int NTHREADS = (10 + NCONV) * 32;
    static constexpr int SMEM_BYTES = 1024 + SS * STAGE_BYTES + 1024;
    static_assert(SS >= 2 && ST >= 2, "DWS pair pipeline does not fit");
};

template <int PLANES, int OW>
__global__ void __launch_bounds__(DwsPairCfg<PLANES, OW>::NTHREADS, 1)
    conv_dws_pair_kernel(const __grid_constant__ DwsParams dp, const __grid_constant__ GenParams p) {
    using C = DwsPairCfg<PLANES, OW>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    const uint32_t tiles_addr = (raw_addr + 1023u) & ~1023u;
    uint8_t* tiles_ptr = smem_raw + (tiles_addr - raw_addr);
    DwsAux* aux = reinterpret_cast<DwsAux*>(tiles_ptr + C::SS * C::STAGE_BYTES);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int CHK = PLANES == 2 ? dp.chunk_kb : (1 << 30);
    const int rank = (int)cluster_ctarank();
    const int wfirst = (int)(blockIdx.x >> 1), wstep = (int)(gridDim.x >> 1);

    if (tid == 0) {
        for (int s = 0; s < C::SS; ++s) {
            mbar_init(&aux->full[s], 1);
            mbar_init(&aux->empty[s], 1 + C::NCONV / 2);  // multicast MMA commit + the next k-block's 4 converter warps
        }
        for (int t = 0; t < C::ST; ++t) {
            mbar_init(&aux->conv[t], C::NCONV);  // CTA 0's: one arrival per converter warp of a k-block, both CTAs
            mbar_init(&aux->tfree[t], 1);
        }
        mbar_init(&aux->tfull, 1);
        mbar_init(&aux->tempty, 2 * C::NEPI);  // CTA 0's: one arrival per epilogue warp of both CTAs
        fence_mbar_init();
    }
    if (warp == C::TMA_W && lane == 0) {
        prefetch_tmap(&dp.mapXA);
        prefetch_tmap(&dp.mapXB);
        prefetch_tmap(&dp.mapY);
    }
    if (warp == C::MMA_W) tmem_alloc2(&aux->tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // the peer's barriers exist before any remote arrival
    tc_fence_after();
    const uint32_t tmem = aux->tmem_base;
    pdl_trigger();
    pdl_wait();

    if (warp == C::TMA_W) {
        // ======================= TMA producer: this CTA's dY half + the activation slab, per k-block
        int s = 0;
        uint32_t r = 0;
        for (int w = wfirst; w < dp.work; w += wstep) {
            DwsItem it;
            it.init(dp, w);
            for (int kb = it.kb0; kb < it.kb1; ++kb) {
                if (r > 0) mbar_wait(&aux->empty[s], (r - 1) & 1);
                const int ncb = kb / dp.ohb, oh0 = (kb - ncb * dp.ohb) * dp.RB;
                const int n = ncb / dp.cbs, cb = ncb - n * dp.cbs, ow0 = cb * 32;
                const int ih0 = oh0 + it.fh_lo - dp.ph;
                const bool fresh = (kb == it.kb0) || (oh0 == 0);
                const uint32_t sY = tiles_addr + s * C::STAGE_BYTES;
                if (elect_one()) {
                    mbar_arrive_expect_tx(&aux->full[s], C::Y_BYTES + C::XB_BYTES + (fresh ? C::XA_BYTES : 0));
                    tma_load_5d(sY, &dp.mapY, &aux->full[s], 0, ow0, oh0, n, rank);  // oc block `rank`
                    tma_load_4d(sY + C::XB_OFF, &dp.mapXB, &aux->full[s], 0, ow0 - dp.pw, ih0 + 1, n);
                    if (fresh) tma_load_4d(sY + C::XA_OFF, &dp.mapXA, &aux->full[s], 0, ow0 - dp.pw, ih0, n);
                }
                __syncwarp();
                if (++s == C::SS) {
                    s = 0;
                    ++r;
                }
            }
        }
    } else if (warp == C::MMA_W) {
        // ======================= MMA issuer (CTA 0): 4 k-steps x (3 | 1) M = 256 MMAs per k-block
        if (rank == 0) {
            constexpr uint32_t IDESC = idesc_tf32(256, C::BN, false, true);  // A from TMEM, B (dY) MN-major
            const uint64_t bd0 = make_sdesc(tiles_addr, 4096u, 512u, kLayoutSW128Base32);
            constexpr uint64_t B_LO = C::Y_BYTES >> 4;
            uint32_t q = 0, c = 0;
            int in_chunk = 0;
            for (int w = wfirst; w < dp.work; w += wstep) {
                DwsItem it;
                it.init(dp, w);
                const int nkb = it.kb1 - it.kb0;
                for (int i = 0; i < nkb; ++i, ++q) {
                    const uint32_t s = q % C::SS, t = q % C::ST, rt = q / C::ST;
                    if (in_chunk == 0 && c >= 1) {
                        mbar_wait(&aux->tempty, (c - 1) & 1);  // both CTAs' epilogues drained the previous chunk
                        tc_fence_after();
                    }
                    const bool last = (in_chunk + 1 == CHK || i == nkb - 1);
                    mbar_wait(&aux->conv[t], rt & 1);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint64_t so = (uint64_t)(s * C::STAGE_BYTES) >> 4;
#pragma unroll
                        for (int g4 = 0; g4 < 4; ++g4) {
                            const uint64_t bdH = bd0 + so + g4 * 64;  // 8 K-rows x 128 B
                            const uint32_t acc0 = (in_chunk > 0 || g4 > 0) ? 1u : 0u;
                            const uint32_t ahi = tmem + (uint32_t)(C::ACC_COLS + t * C::SLOT_COLS + g4 * 8);
                            if (PLANES == 2) {
                                mma2_tf32_ts(tmem, ahi + 32, bdH, IDESC, acc0);  // a_lo * b_hi
                                mma2_tf32_ts(tmem, ahi, bdH + B_LO, IDESC, 1u);  // a_hi * b_lo
                                mma2_tf32_ts(tmem, ahi, bdH, IDESC, 1u);         // a_hi * b_hi
                            } else {
                                mma2_tf32_ts(tmem, ahi, bdH, IDESC, acc0);
                            }
                        }
                        mma2_commit_both(&aux->empty[s]);
                        mma2_commit_both(&aux->tfree[t]);
                        if (last) mma2_commit_both(&aux->tfull);
                    }
                    __syncwarp();
                    if (last) {
                        ++c;
                        in_chunk = 0;
                    } else {
                        ++in_chunk;
                    }
                }
            }
        }
    } else if (warp >= C::CONV_W0) {
        // ======================= converters: this CTA's m-tile (taps 4g+2r, 4g+2r+1) -> TMEM; dY half -> b_lo.
        // Two groups of 4 warps take alternate k-blocks (warp = one TMEM lane quadrant, all 32 pixels of the
        // k-block): the per-k-block chain LDS -> split -> tcgen05.st -> wait -> arrive bounded the pair at one
        // k-block per chain latency with all 8 warps on the same k-block (r02bw: 0.49 us per k-block)
        const int grp = (warp - C::CONV_W0) >> 2;
        const int ct4 = tid - (C::CONV_W0 + 4 * grp) * 32;  // 0..127 within the group
        const int qd = warp & 3;
        const int ts = qd >> 1, icb = qd & 1;
        uint32_t q = 0;
        for (int w = wfirst; w < dp.work; w += wstep) {
            DwsItem it;
            it.init(dp, w);
            const int nkb = it.kb1 - it.kb0;
            const int tap = 4 * it.g + 2 * rank + ts;
            const int fh = tap / 3, fw = tap - 3 * fh;
            for (int i = 0; i < nkb; ++i, ++q) {
                if ((int)(q & 1u) != grp) continue;
                const uint32_t s = q % C::SS, rs = q / C::SS, t = q % C::ST, rt = q / C::ST;
                const uint32_t sp = (s + C::SS - 1) % C::SS;
                const int kb = it.kb0 + i;
                const bool fresh = (i == 0) || (kb % dp.ohb == 0);
                mbar_wait(&aux->full[s], rs & 1);
                // slab row 0 comes from the previous k-block's stage, whose TMA the OTHER group waited for: wait
                // for it here too (it cannot be refilled before this group's arrival on empty[sp] below)
                if (!fresh) mbar_wait(&aux->full[sp], ((q - 1) / C::SS) & 1);
                uint8_t* st = tiles_ptr + s * C::STAGE_BYTES;
                if (PLANES == 2) {  // b_lo of this CTA's dY half (4 KB: two float4 per thread of the group)
#pragma unroll
                    for (int e2 = 0; e2 < 2; ++e2) {
                        const float4 v = reinterpret_cast<const float4*>(st)[ct4 + 128 * e2];
                        float4 o;
                        o.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
                        o.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
                        o.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
                        o.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
                        reinterpret_cast<float4*>(st + C::Y_OFF_LO)[ct4 + 128 * e2] = o;
                    }
                }
                const uint8_t* row0 = fresh ? st + C::XA_OFF
                                            : tiles_ptr + sp * C::STAGE_BYTES + C::XB_OFF + (C::RB - 1) * C::ROW_BYTES;
                const uint8_t* row1 = st + C::XB_OFF;
                if (rt > 0) mbar_wait(&aux->tfree[t], (rt - 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int h = 0; h < 2; ++h) {  // pixels 16h .. 16h+15 of the k-block
                    uint32_t hi[16], lo[16];
                    const int bsr = tap < kDwsTaps ? fh - it.fh_lo + (16 * h) / OW : -1;
                    const int coff = (fw + (16 * h) % OW) * 256 + icb * 128 + lane * 4;
                    if (bsr >= 0) {
                        const uint8_t* p0 = (bsr == 0 ? row0 : row1 + (bsr - 1) * C::ROW_BYTES) + coff;
                        const uint8_t* p1 = row1 + bsr * C::ROW_BYTES + coff;
#pragma unroll
                        for (int k = 0; k < 16; ++k) {
                            const float e = (k / OW == 0) ? *reinterpret_cast<const float*>(p0 + (k % OW) * 256)
                                                          : *reinterpret_cast<const float*>(
                                                                p1 + (k / OW - 1) * C::ROW_BYTES + (k % OW) * 256);
                            if (PLANES == 2) {
                                const uint32_t hb = __float_as_uint(e) & 0xFFFFE000u;
                                hi[k] = hb;
                                lo[k] = __float_as_uint(e - __uint_as_float(hb));
                            } else {
                                hi[k] = __float_as_uint(e);
                                lo[k] = 0u;
                            }
                        }
                    } else {
#pragma unroll
                        for (int k = 0; k < 16; ++k) hi[k] = lo[k] = 0u;  // taps 9..11 of group 2: empty rows
                    }
                    const uint32_t ta = tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(C::ACC_COLS + t * C::SLOT_COLS + h * 16);
                    tmem_st_32x32b_x16(ta, hi);
                    if (PLANES == 2) tmem_st_32x32b_x16(ta + 32, lo);
                }
                tmem_st_wait();
                fence_proxy_async_smem();  // b_lo before the release
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_remote(&aux->conv[t], 0);  // on CTA 0's barrier (it issues the MMAs)
                if (lane == 0 && q > 0) mbar_arrive(&aux->empty[sp]);  // previous stage: its row RB was read
            }
        }
    } else {
        // ======================= epilogue warps 0-7: promote chunks, write this CTA's m-tile partial
        const int qd = warp & 3, half = warp >> 2;
        const uint32_t lane_addr = (uint32_t)(qd * 32) << 16;
        const int M = kDwsTaps * 64;
        uint32_t c = 0;
        for (int w = wfirst; w < dp.work; w += wstep) {
            DwsItem it;
            it.init(dp, w);
            const int nkb = it.kb1 - it.kb0;
            const int nch = nkb > 0 ? (nkb + CHK - 1) / CHK : 0;
            float acc[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) acc[e] = 0.f;
            for (int k = 0; k < nch; ++k, ++c) {
                mbar_wait(&aux->tfull, c & 1);
                tc_fence_after();
#pragma unroll
                for (int c0 = 0; c0 < 32; c0 += 16) {
                    uint32_t v[16];
                    tmem_ld_32x32b_x16(tmem + lane_addr + (uint32_t)(half * 32 + c0), v);
                    tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 16; ++e) acc[c0 + e] += __uint_as_float(v[e]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_remote(&aux->tempty, 0);
            }
            float* outp = p.out + (long long)it.split * p.split_stride;
            const int tap = 4 * it.g + 2 * rank + (qd >> 1);
            if (tap < kDwsTaps) {
                float* o = outp + tap * 64 + (qd & 1) * 32 + lane + (long long)(half * 32) * M;
#pragma unroll
                for (int e = 0; e < 32; ++e) o[(long long)e * M] = acc[e];
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // the peer's MMAs / arrivals are done before TMEM is released
    if (warp == C::MMA_W) {
        tc_fence_after();
        tmem_dealloc2(tmem, 512);
    }
}

namespace {

const int g_knob_chunk_d = getenv("SMCONV_TMA_CHUNK") ? atoi(getenv("SMCONV_TMA_CHUNK")) : 8;

// bf16 cross terms (the hybrid 3xTF32 form) for the DWS dW; SMCONV_DWS_HYB=0: three TF32 MMAs.  With the
// alternate-k-block converters it wins in the power-capped step (r02cb: l1.0a dW 1722 -> 1637 us isolated,
// 6.50 -> 6.11 pJ / flop, ResNet-18 b4096 step -0.2..1.3 ms in three same-box pairs); without them it lost
// (converter-bound, r02bj)
const int g_dws_hyb = getenv("SMCONV_DWS_HYB") ? atoi(getenv("SMCONV_DWS_HYB")) : 1;
// SMCONV_DWS_ALT=0: all 8 converter warps on every k-block (DwsParams::alt_conv)
const int g_dws_alt = getenv("SMCONV_DWS_ALT") ? atoi(getenv("SMCONV_DWS_ALT")) : 1;

template <int PLANES, int OW, bool HYB>
int launch_t(const DwsParams& dp, const GenParams& g, cudaStream_t st, char* err, size_t errlen) {
    using C = DwsCfg<PLANES, OW>;
    static std::atomic<unsigned long long> attr_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_done.load() & bit)) {
        if (cudaFuncSetAttribute(conv_dws_kernel<PLANES, OW, HYB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 C::SMEM_BYTES) != cudaSuccess) {
            snprintf(err, errlen, "cudaFuncSetAttribute(dws smem=%d): %s", C::SMEM_BYTES,
                     cudaGetErrorString(cudaGetLastError()));
            return CONV_ECUDA;
        }
        attr_done.fetch_or(bit);
    }
    const int grid = dp.work < 148 ? dp.work : 148;
    const cudaError_t e = launch_k(conv_dws_kernel<PLANES, OW, HYB>, dim3(grid), dim3(C::NTHREADS), C::SMEM_BYTES, st, 1,
                                   dp, g);
    if (e != cudaSuccess) {
        snprintf(err, errlen, "cudaLaunchKernelEx(dws): %s", cudaGetErrorString(e));
        return CONV_ECUDA;
    }
    return CONV_OK;
}

}  // namespace

template <int PLANES, int OW>
int launch_pair_t(const DwsParams& dp, const GenParams& g, cudaStream_t st, char* err, size_t errlen) {
    using C = DwsPairCfg<PLANES, OW>;
    static std::atomic<unsigned long long> attr_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_done.load() & bit)) {
        if (cudaFuncSetAttribute(conv_dws_pair_kernel<PLANES, OW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 C::SMEM_BYTES) != cudaSuccess) {
            snprintf(err, errlen, "cudaFuncSetAttribute(dws pair smem=%d): %s", C::SMEM_BYTES,
                     cudaGetErrorString(cudaGetLastError()));
            return CONV_ECUDA;
        }
        attr_done.fetch_or(bit);
    }
    const int pairs = dp.work < 74 ? dp.work : 74;
    const cudaError_t e = launch_k(conv_dws_pair_kernel<PLANES, OW>, dim3(2 * pairs), dim3(C::NTHREADS), C::SMEM_BYTES,
                                   st, 2, dp, g);
    if (e != cudaSuccess) {
        snprintf(err, errlen, "cudaLaunchKernelEx(dws pair): %s", cudaGetErrorString(e));
        return CONV_ECUDA;
    }
    return CONV_OK;
}

int dws_hyb_mode() { return g_dws_hyb; }

// SMCONV_DWS_PAIR=0: the single-CTA DWS kernel (A/B)
int dws_pair_mode() {
    static const int m = getenv("SMCONV_DWS_PAIR") ? atoi(getenv("SMCONV_DWS_PAIR")) : 0;
    return m;
}

bool dws_supported(int op, int IC, int OC, int FH, int FW, int sh, int sw, int OH, int OW) {
    if (op != CONV_OP_BWD_FILTER) return false;
    if (IC != 64 || OC != 64 || FH != 3 || FW != 3 || sh != 1 || sw != 1) return false;
    if (OW != 32 && OW != 16 && OW != 8 && (OW % 32 != 0 || OW > 4096)) return false;  // wide maps: OW % 32
    return OW >= 32 || OH % (32 / OW) == 0;
}

// Split choice: chains of <= 256 k-blocks (the precision bound shared with the TMA variant), and a
// number of work items (3 groups per split) that fills whole rounds of the 148-CTA persistent grid,
// at least 4 rounds: with 300 items (2.03 rounds) two thirds of the CTAs idled through the last one.
int dws_splits(int N, int OH, int OW, int* kb_per_split) {
    const long long ctas = dws_pair_mode() ? 74 : 148;  // work items are per CTA, or per CTA pair
    const int RB = OW >= 32 ? 1 : 32 / OW;
    const long long kb_total = (long long)N * (OH / RB) * (OW >= 32 ? OW / 32 : 1);
    const long long need = (kb_total + 255) / 256;
    // at least min_rounds waves of (3 x splits) CTAs; 4 cost the small batches a 196-split workspace
    // round trip: VGG b128 vgg2 dW 101 us at 4, 77 us at 2, 64.5 us at 1 (r02z); b4096 needs 11 anyway
    static const int min_rounds = getenv("SMCONV_DWS_MIN_ROUNDS") ? atoi(getenv("SMCONV_DWS_MIN_ROUNDS")) : 1;
    long long rounds = (3 * need + ctas - 1) / ctas;
    if (rounds < min_rounds) rounds = min_rounds;
    long long smax = rounds * ctas / 3;
    if (smax > kb_total) smax = kb_total;
    if (smax < 1) smax = 1;
    const long long kps = (kb_total + smax - 1) / smax;
    *kb_per_split = (int)kps;
    return (int)((kb_total + kps - 1) / kps);
}

int dws_launch(int planes, const GenParams& g, int splits, int kb_per_split, cudaStream_t st, char* err,
               size_t errlen) {
    DwsParams dp;
    memset(&dp, 0, sizeof dp);
    const int wow = g.OW >= 32 ? 32 : g.OW;  // geometry width (wide maps: 32-column blocks)
    dp.OW = wow;
    dp.cbs = g.OW >= 32 ? g.OW / 32 : 1;
    dp.RB = 32 / wow;
    dp.XW = wow + 2;
    dp.ohb = g.OH / dp.RB;
    dp.kb_total = g.N * dp.ohb * dp.cbs;
    dp.kb_per_split = kb_per_split;
    dp.splits = splits;
    dp.work = splits * kDwsGroups;
    dp.chunk_kb = g_knob_chunk_d > 0 ? g_knob_chunk_d : 8;
    dp.alt_conv = g_dws_alt;
    dp.ph = g.ph;
    dp.pw = g.pw;
    const uint64_t N = g.N, IH = g.IH, IW = g.IW, IC = g.IC, OC = g.OC, OH = g.OH, OW = g.OW;
    // dW convention of run(): g.A = dY, g.B = X
    uint64_t dx[4] = {IC, IW, IH, N}, sx[3] = {IC * 4, IW * IC * 4, IH * IW * IC * 4};
    uint32_t bxa[4] = {(uint32_t)IC, (uint32_t)dp.XW, 1, 1};
    uint32_t bxb[4] = {(uint32_t)IC, (uint32_t)dp.XW, (uint32_t)dp.RB, 1};
    bool ok = tma_encode_f32(&dp.mapXA, g.B, 4, dx, sx, bxa, CU_TENSOR_MAP_SWIZZLE_NONE);
    ok &= tma_encode_f32(&dp.mapXB, g.B, 4, dx, sx, bxb, CU_TENSOR_MAP_SWIZZLE_NONE);
    uint64_t dy[5] = {32, OW, OH, N, OC / 32}, sy[4] = {OC * 4, OW * OC * 4, OH * OW * OC * 4, 128};
    const bool pair = dws_pair_mode() != 0;
    uint32_t by[5] = {32, (uint32_t)wow, (uint32_t)dp.RB, 1, (uint32_t)(pair ? 1 : OC / 32)};  // pair: one oc block per CTA
    ok &= tma_encode_f32(&dp.mapY, g.A, 5, dy, sy, by, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    if (!ok) {
        snprintf(err, errlen, "dws: cuTensorMapEncodeTiled failed");
        return CONV_ECUDA;
    }
    if (pair) {
        if (planes == 2) {
            if (g.OW >= 32) return launch_pair_t<2, 32>(dp, g, st, err, errlen);
            if (g.OW == 16) return launch_pair_t<2, 16>(dp, g, st, err, errlen);
            return launch_pair_t<2, 8>(dp, g, st, err, errlen);
        }
        if (g.OW >= 32) return launch_pair_t<1, 32>(dp, g, st, err, errlen);
        if (g.OW == 16) return launch_pair_t<1, 16>(dp, g, st, err, errlen);
        return launch_pair_t<1, 8>(dp, g, st, err, errlen);
    }
    if (planes == 2 && g_dws_hyb) {
        if (g.OW >= 32) return launch_t<2, 32, true>(dp, g, st, err, errlen);
        if (g.OW == 16) return launch_t<2, 16, true>(dp, g, st, err, errlen);
        return launch_t<2, 8, true>(dp, g, st, err, errlen);
    }
    if (planes == 2) {
        if (g.OW >= 32) return launch_t<2, 32, false>(dp, g, st, err, errlen);
        if (g.OW == 16) return launch_t<2, 16, false>(dp, g, st, err, errlen);
        return launch_t<2, 8, false>(dp, g, st, err, errlen);
    }
    if (g.OW >= 32) return launch_t<1, 32, false>(dp, g, st, err, errlen);
    if (g.OW == 16) return launch_t<1, 16, false>(dp, g, st, err, errlen);
    return launch_t<1, 8, false>(dp, g, st, err, errlen);
}

}  // namespace smconv
