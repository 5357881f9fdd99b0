// conv_tma.cuh — TMA variant: persistent, warp-specialised, TMA-staged implicit GEMM on tcgen05
// (sm_100a); the fast path for channel extents and batches that are multiples of 32.
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
// (CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE): no predication in the data path.  K-major boxes use
// SWIZZLE_128B, MN-major boxes SWIZZLE_128B_ATOM_32B (= UMMA SWIZZLE_128B_BASE32B).
//
// Persistent CTAs (one per SM) walk the work list (m-tile, split, n-tile) round-robin.  The
// smem stage ring, the two TMEM accumulator buffers and all mbarrier phases run continuously
// across tiles, so the TMA of tile i+1 and its MMAs overlap the epilogue of tile i.
//
// Warp roles: warps 0-7 epilogue (+ accumulator promotion), warp 8 TMA producer (1 lane),
// warp 9 TMEM owner + MMA issuer (1 lane), warps 10-13 (3xTF32 only) split converters.
//
// 3xTF32 exploits what the probe measured: tcgen05 kind::tf32 reads an fp32
// operand by TRUNCATION to TF32, so the raw TMA tile IS b_hi = trunc_tf32(b).  fwd / dX: per
// k-block a_hi*b_hi as 4 TF32 MMAs, and the cross terms a_hi*b_lo + a_lo*b as 4 bf16 MMAs (K = 64)
// on A' = [bf16(a_hi) | bf16(a_lo)] (written to TMEM by the converters) and the precomputed W'
// plane B' = [bf16(b_lo) | bf16(b)] (wx_prep_kernel, TMA-loaded): 2 TF32-MMA-equivalents of
// tensor-pipe time and energy instead of 3 (the step runs at the power cap).  dW (B = an
// activation tile): a_lo*b_hi + a_hi*b_lo + a_hi*b_hi, b_lo split by the converters.
// The accumulator adds by truncation too, so K is cut into chunks of chunk_kb k-blocks that
// alternate between the two TMEM buffers and are promoted into fp32 registers (round to
// nearest) by the epilogue warps while the next chunk runs (SURVEY.md §7 hard part 1).
// TF32 mode: one chunk per tile; the buffers alternate per tile.
#pragma once
#include <cuda.h>

#include "conv_gen.cuh"

namespace smconv {

struct __align__(64) TmaParams {
    CUtensorMap mapA;
    CUtensorMap mapB;
    CUtensorMap mapBx;  // 3xTF32 fwd / dX: the precomputed bf16 W' plane (wx_prep_kernel), box (64, 1, BNC, 1)
    int G;           // images per A box (fwd/dx): 128 when N % 128 == 0, else 32
    int CB;          // fwd/dx: channel blocks of 32 per tap (IC/32 resp. OC/32)
    int NB32;        // dw: N / 32 (image blocks per position)
    int b_boxes;     // dw: B boxes per tile
    int b_box_cols;  // dw: GEMM columns per B box (never crosses a tap)
    int a_boxes;     // dwT: A boxes (X patches) per 128-row tile
    int a_box_cols;  // dwT: GEMM rows per A box (never crosses a tap)
    int chunk_kb;    // promotion interval in k-blocks (3xTF32)
    int pair;          // fwd/dx 3xTF32: CTA pairs (cta_group::2, M = 256); work items are pair tiles
    int dw_tap_tiles;  // dw: IC / BN when every n-tile lies inside one filter tap (else 0): the tile's
                       // k-blocks whose source pixels are all padding are skipped
    int m_tiles, n_tiles;  // work decomposition (dx: m_tiles over all phases)
    int work;        // m_tiles * splits * n_tiles
    int csk;         // fwd / dx: cluster split-K (GenParams::csk): one work item per CTA, the csk splits of a
                     // tile are the CTAs of one cluster, partials reduced through DSMEM (csk_reduce)
    // host-built fast divisors for TileInfo::init: a generic 32-bit division is a ~150-cycle dependent
    // I2F / MUFU.RCP / F2I chain, and the ~10 of them per work item kept every role ~3800 cycles in its
    // first TileInfo::init (smconv_set_trace, r02j) -- the TMA producer's first load waited on it
    FastDiv fd_ntiles, fd_csk, fd_splits, fd_mtiles, fd_CB, fd_dwtap;
    FastDiv fd_P[kMaxPhases];  // positions per (phase) map: fwd / dW OH*OW, dX phase IHp*IWp
    int dx_ragged;  // dX with IC % 32 != 0: B = W viewed (IC, OC, T), one (32 ic, 32 oc) box per 32-column
                    // block (the TMA zero-fills ic >= IC) instead of one 4-D box of BNC / 32 blocks
    int dw_a_ragged;  // dW with OC % 32 != 0: A = dY viewed (OC, N, P), 4 boxes (32 oc, 32 n, 1) per k-block
    int dw_b_ragged;  // dW with IC % 32 != 0: B = X viewed (IC, N, IW, IH), boxes (32 ic, 32 n, 1, 1)
    int coalesce;     // fwd / dX: row-coalesced epilogue stores through the per-warp staging (TmaCfg::EPW)
    // dX of a 1x1 stride-2 conv (only phase (0, 0) has a tap): the epilogue also writes the zeros of
    // pixels (2a, 2b+1), (2a+1, 2b), (2a+1, 2b+1) next to each row (2a, 2b) -- element offsets zf1
    // (one pixel) and zf2 (one dX row) -- instead of a separate zero_phases_kernel pass (0: off)
    long long zf1, zf2;
    // dX with the K-major transposed filter plane Wt[IC][T][OC] (written by wx_prep_kernel with the W'
    // plane, 3xTF32 hybrid only): B is staged like the fwd's W (box (32 oc, 1, BNC ic)), K-major
    // SWIZZLE_128B, instead of the MN-major 32-B-atom view of W
    int dx_bk;
    int dw_hyb;  // dW cross terms in bf16 (TmaCfg::HYBW)
    int alt_conv;  // 3xTF32 converter warps in two groups on alternate k-blocks
    // fwd / dX: the row-coalesced epilogue's pieces leave by TMA tensor store (cp.async.bulk.tensor) from
    // the warp's staging slice instead of LDS + SHFL + STG per thread: mapY views the output as
    // (C, pixels, N), box (EPW, 1, 32 images); the staging slice already holds the TMA's 64B / 128B
    // swizzle (warp_rows_store's XOR pattern).  0: per-thread stores (s2dx, zfill, csk, odd N)
    int tstore;
    CUtensorMap mapY;
};

SMCONV_DEV void tma_store_3d(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(src), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
SMCONV_DEV void bulk_commit_group() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
SMCONV_DEV void bulk_wait_group_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
SMCONV_DEV void bulk_wait_group0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// The same staging as warp_rows_store, then ONE TMA tensor store of the warp's 32 rows x PW columns
// (rows = 32 consecutive images at output pixel `pix`, starting at image n0).  Lane 0 owns the bulk
// group: it waits until the previous store has READ the slice before the lanes overwrite it.
template <int PW>
SMCONV_DEV void warp_rows_tstore(uint8_t* stg, const float (&f)[PW], const CUtensorMap* map, int col0, int pix, int n0,
                                 bool valid, int lane) {
    constexpr int F4 = PW / 4;
    static_assert(F4 == 4 || F4 == 8, "piece of 16 or 32 columns");
    auto swz = [](int r) { return F4 == 8 ? (r & 7) : ((r >> 1) & 3); };
    if (lane == 0) bulk_wait_group_read0();
    __syncwarp();
#pragma unroll
    for (int j = 0; j < F4; ++j)
        *reinterpret_cast<float4*>(stg + (lane * F4 + (j ^ swz(lane))) * 16) =
            make_float4(f[4 * j], f[4 * j + 1], f[4 * j + 2], f[4 * j + 3]);
    fence_proxy_async_smem();  // generic-proxy writes -> visible to the TMA (async proxy)
    __syncwarp();
    if (lane == 0 && valid) {
        tma_store_3d(map, smem_u32(stg), col0, pix, n0);
        bulk_commit_group();
    }
}

// byte offset of bf16 elements (k, mn..mn+3), mn % 4 == 0, in a [K][MN] MN-major SWIZZLE_128B bf16 tile:
// 64-element (128-B) MN atoms of K rows each (atom stride K * 128 B), 8-row x 128-B swizzle groups
SMCONV_DEV uint32_t mnmaj16_off(uint32_t k, uint32_t mn, uint32_t krows) {
    return (mn >> 6) * krows * 128u + (k >> 3) * 1024u + (k & 7u) * 128u + ((((mn >> 3) & 7u) ^ (k & 7u)) << 4) +
           (mn & 7u) * 2u;
}

template <int OP, int BN, int PLANES, bool PAIR = false>
struct TmaCfg {
    static constexpr int BM = 128, BK = 32;
    static constexpr int BNC = PAIR ? BN / 2 : BN;  // B columns staged by this CTA (a pair splits B)
    static constexpr int NEPI = 8;  // epilogue warps 0-7
    static constexpr int TMA_W = 8, MMA_W = 9, CONV_W0 = 10;
    static constexpr int NCONV = PLANES == 2 ? 8 : 0;  // converters: 8 warps keep up with N=64 MMAs
    static constexpr int NTHREADS = (10 + NCONV) * 32;
    static constexpr int A_BYTES = BM * BK * 4;
    static constexpr int B_BYTES = BNC * BK * 4;
    // 3xTF32 with a K-major A (fwd, dX): the converters write a_hi and a_lo straight into TMEM
    // (tcgen05.st) and the MMAs read A from TMEM, so A is read from shared memory once per k-block
    // instead of three times and no a_lo plane is stored there (the kernel is smem-bandwidth bound).
    static constexpr bool A_TMEM = (PLANES == 2);
    static constexpr int B_OFF = A_TMEM ? A_BYTES : PLANES * A_BYTES;  // B (hi) offset in a stage
    static constexpr int STAGE_BYTES = A_TMEM ? A_BYTES + 2 * B_BYTES : PLANES * (A_BYTES + B_BYTES);
    // shared-memory stages (TMA ring) and TMEM A slots (converter -> MMA ring) are separate rings:
    // an A slot is held only from its conversion to its MMAs' completion, a stage from the TMA issue
    // on, so tying both to one index capped the TMA look-ahead at the TMEM slot count (4 at BN 128)
    static constexpr int STAGES_RAW = (200 * 1024) / STAGE_BYTES;
    static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
    static constexpr int NT_RAW = A_TMEM ? (512 - 2 * BN) / 64 : 1;  // TMEM A slots (64 cols each)
    static constexpr int NT = NT_RAW > 8 ? 8 : NT_RAW;
    static constexpr bool IS_DW = (OP == OP_DW || OP == OP_DWT);
    // fwd / dX in 3xTF32: a_hi*b_hi as a TF32 MMA plus the cross terms as bf16 MMAs on the
    // precomputed W' plane (common.cuh "3xTF32 operand split"); dW keeps three TF32 MMAs with a
    // b_lo plane split by the converters (its B is an activation tile; the bf16 split of an
    // MN-major activation tile cost more converter time than the tensor pipe saved, r01l)
    static constexpr bool HYB = A_TMEM && !IS_DW;
    // dW (not transposed) with the same cross-term form (TmaParams::dw_hyb): A' = [bf16(a_hi) | bf16(a_lo)]
    // in TMEM next to a_hi, B' = [bf16(b_lo) ; bf16(b)] as a K' = 64 bf16 MN-major plane the converters
    // build from the X tile in place of the fp32 b_lo plane (same bytes): 2 MMA-equivalents per product
    static constexpr bool HYBW = A_TMEM && OP == OP_DW;
    static constexpr bool A_MN = IS_DW;
    static constexpr bool B_MN = (OP != OP_FWD);
    static constexpr int A_TCOL0 = 2 * BN;  // TMEM column of A slot 0 (A_TMEM)
    static constexpr int ACC_COLS = 2 * BN + (A_TMEM ? NT * 64 : 0);
    static constexpr int TMEM_COLS = ACC_COLS <= 32 ? 32 : ACC_COLS <= 64 ? 64 : ACC_COLS <= 128 ? 128 : ACC_COLS <= 256 ? 256 : 512;
    static constexpr int AUX_BYTES = 1024 + kMaxTaps * 16;
    static constexpr int SMEM_BASE = 1024 + STAGES * STAGE_BYTES + AUX_BYTES;
    // Row-coalesced epilogue (fwd / dX).  A TMEM lane is a GEMM row = one output pixel of one image, so a
    // warp's st.global.v4 of 32 lanes scatters 16 B to each of 32 rows (OH*OW*C*4 bytes apart under the
    // position-major walk): 32 L2 requests per instruction.  The 1x1 shortcut fwd (K = 2 k-blocks) was
    // bound by it (ncu r02bb: stall_long_sb on the registers of outstanding STGs, 2.5 TB/s).  Each
    // epilogue warp stages 32 rows x EPW columns in shared memory (XOR-swizzled 16-B units: both the
    // row-wise writes and the column-wise reads are bank-conflict free) and stores EPW*4-byte row runs.
    static constexpr int SMEM_FREE = 232448 - SMEM_BASE;  // 227 KB opt-in maximum per CTA
    static constexpr int EPW = IS_DW ? 0
                             : (BN / 2 >= 32 && SMEM_FREE >= NEPI * 32 * 32 * 4) ? 32
                             : (BN / 2 >= 16 && SMEM_FREE >= NEPI * 32 * 16 * 4) ? 16 : 0;
    static constexpr int STG_BYTES = NEPI * 32 * EPW * 4;
    static constexpr int SMEM_BYTES = SMEM_BASE + STG_BYTES;
    // cluster split-K partial [128 rows][BN + 4] fp32 in the (drained) stage ring; +4 floats per row
    // keep a quarter-warp's 16-B row stores on distinct banks
    static constexpr int PSTRIDE = BN + 4;
    static constexpr bool CSK_FITS = 128 * PSTRIDE * 4 <= STAGES * STAGE_BYTES;
    static_assert(STAGES >= 2, "stage does not fit");
    static_assert(PLANES == 1 || BN <= 128, "3xTF32 promotion keeps BN/2 fp32 per epilogue thread");
    static_assert(!PAIR || (PLANES == 2 && OP != OP_DWT && BN >= 64), "CTA pairs: fwd / dx / dW, 3xTF32");
};

struct TmaAux {
    uint64_t full[8], conv[8], empty[8], tfree[8];
    uint64_t tfull[2], tempty[2];
    uint32_t tmem_base;
    int4 ptaps[kMaxTaps];  // producer-private per-tile tap list / X-box geometry
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

// Everything a role needs to know about one work item; recomputed independently by every role
// (cheap: at most 4 A-box groups x FH*FW taps), so no smem hand-off between roles is needed.
template <int OP>
struct TileInfo {
    int phase, m0, n0, split;
    int ngrp;
    int4 grp[4];  // {h0, w0, n_img, valid}
    int kb_begin, kb_end;
    int nkb_eff;             // k-blocks that are issued (dw: positions where the tile's tap is in range)
    int vr_lo, vr_hi, vc_lo, vc_hi;  // dw single-tap tiles: output rows / cols whose source is in range

    SMCONV_DEV void init(const TmaParams& tp, const GenParams& p, int w, int rank = 0) {
        auto dv = [](int a, const FastDiv& f) { return (int)fdiv((uint32_t)a, f); };
        int rest = dv(w, tp.fd_ntiles);
        int nt = w - rest * tp.n_tiles;
        int mt;
        if (OP != OP_DWT && tp.csk) {
            // cluster split-K: the splits of one tile are consecutive CTAs (one cluster)
            const int tile = dv(w, tp.fd_csk);
            split = w - tile * tp.csk;
            mt = dv(tile, tp.fd_ntiles);
            nt = tile - mt * tp.n_tiles;
        } else if (OP == OP_DW || OP == OP_DWT) {
            // split (pixel range) outermost: all (m, n) tiles of one pixel range run together, so
            // that range's dY and X are read from HBM once and re-used from L2 by every tile
            // (m-tile-major order re-read them once per m-tile: 11.3 GB vs 2.1 GB compulsory, l1)
            split = dv(rest, tp.fd_mtiles);
            mt = rest - split * tp.m_tiles;
        } else {
            mt = dv(rest, tp.fd_splits);
            split = rest - mt * p.splits;
        }
        phase = 0;
        if (OP == OP_DX) {
            // phase-major walk.  (An image-block-major walk across the phases cut the l2.0a dX DRAM
            // reads 2.35 -> 0.93 GB but ran 1.44 -> 1.81 ms: measured r01g, reverted.)
            while (phase + 1 < p.nphase && mt >= p.phase_tile0[phase + 1]) ++phase;
            mt -= p.phase_tile0[phase];
        }
        constexpr bool DWK = (OP == OP_DW || OP == OP_DWT);  // reduction over pixels
        m0 = mt * 128;
        // dW pair tiles: the two CTAs take output-channel blocks 2*mt and 2*mt+1 (same n-tile, same
        // pixel range, so one shared k-loop)
        if (OP == OP_DW && tp.pair) m0 = (2 * mt + rank) * 128;
        if (!DWK && tp.G == 128) {
            // image-block-major walk over (128-image block, position): consecutive tiles are
            // neighbouring positions of the same images, so the 3x3 taps' source rows are reused
            // from L2 instead of re-read from HBM (a position-major walk thrashed L2: 3x X reads)
            const int P = OP == OP_DX ? p.phase_IHp[phase] * p.phase_IWp[phase] : p.OH * p.OW;
            const int ib = dv(mt, tp.fd_P[OP == OP_DX ? phase : 0]), pos = mt - ib * P;
            // pair tiles: the two CTAs take image blocks 2*ib and 2*ib+1 at the same position, so
            // both halves of the M = 256 tile have the same taps (one shared k-loop)
            m0 = tp.pair ? pos * p.N + (2 * ib + rank) * 128 : pos * p.N + ib * 128;
        }
        n0 = nt;  // caller multiplies by BN
        ngrp = 0;
        if (!DWK) {
            const int Mrows = OP == OP_DX ? p.phase_IHp[phase] * p.phase_IWp[phase] * p.N : p.M;
            ngrp = tp.G == 128 ? 1 : 4;  // G is 128 or 32
#pragma unroll
            for (int g = 0; g < 4; ++g) {  // static indexing keeps grp[] in registers
                if (g >= ngrp) break;
                const int m = m0 + g * tp.G;
                grp[g] = make_int4(-(1 << 20), -(1 << 20), 0, 0);
                if (m < Mrows) {
                    RowInfo ri = row_info<OP>(p, phase, m);
                    grp[g] = make_int4(ri.h0, ri.w0, ri.n, 1);
                }
            }
        }
        int nkb;
        if (DWK) {
            nkb = p.OH * p.OW * tp.NB32;
            kb_begin = split * p.kb_per_split;
            kb_end = min(nkb, kb_begin + p.kb_per_split);
        } else {
            nkb = ntaps(p) * tp.CB;
            const int per = dv(nkb + p.splits - 1, tp.fd_splits);
            kb_begin = split * per;
            kb_end = min(nkb, kb_begin + per);
        }
        if (kb_end < kb_begin) kb_end = kb_begin;
        nkb_eff = kb_end - kb_begin;
        vr_lo = 0, vr_hi = p.OH, vc_lo = 0, vc_hi = p.OW;
        if (OP == OP_DW && tp.dw_tap_tiles > 0 && nkb_eff > 0) {
            // a single-tap tile gets only zeros from the positions whose source pixel is padding
            // (4x4 maps: 7 of 16 positions for a corner tap): those k-blocks are not issued at all
            const int tap = dv(n0, tp.fd_dwtap), fh = dv(tap, p.fd_FW), fw = tap - fh * p.FW;
            auto fdiv = [](int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); };
            vr_lo = max(0, -fdiv(fh - p.ph, p.sh));  // ceil((ph - fh) / sh)
            vr_hi = min(p.OH, fdiv(p.IH - 1 + p.ph - fh, p.sh) + 1);
            vc_lo = max(0, -fdiv(fw - p.pw, p.sw));
            vc_hi = min(p.OW, fdiv(p.IW - 1 + p.pw - fw, p.sw) + 1);
            if (vr_hi < vr_lo) vr_hi = vr_lo;
            if (vc_hi < vc_lo) vc_hi = vc_lo;
            const int P = p.OH * p.OW, nvw = vc_hi - vc_lo, V = (vr_hi - vr_lo) * nvw;
            auto cnt = [&](int k) {  // valid k-blocks below k (k-block = image block x position)
                const int nb = dv(k, tp.fd_P[0]), pp = k - nb * P, r = dv(pp, p.fd_OW), c = pp - r * p.OW;
                const int rb = min(max(r, vr_lo), vr_hi) - vr_lo;
                const int cb = (r >= vr_lo && r < vr_hi) ? min(max(c, vc_lo), vc_hi) - vc_lo : 0;
                return nb * V + rb * nvw + cb;
            };
            nkb_eff = cnt(kb_end) - cnt(kb_begin);
        }
    }

    // Is candidate (kh, kw) of the tile's phase tap table used by this tile (some group has its
    // source pixel in bounds)?  If so and t != nullptr, writes {dh, dw, fh * FW + fw}.
    SMCONV_DEV bool tap_valid(const GenParams& p, int kh, int kw, int4* t) const {
        const int ph_ = OP == OP_DX ? phase : 0;
        // fwd: the tap table is the identity (offset = filter index); reading it anyway cost a dependent
        // dynamically indexed parameter load per candidate tap in every role's per-tile bookkeeping
        const int dh = OP == OP_FWD ? kh : p.tf_off[ph_][0][kh], dw = OP == OP_FWD ? kw : p.tf_off[ph_][1][kw];
        const int srcH = OP == OP_FWD ? p.IH : p.OH;
        const int srcW = OP == OP_FWD ? p.IW : p.OW;
        bool any = false;
#pragma unroll
        for (int g = 0; g < 4; ++g)
            if (g < ngrp) any |= grp[g].w && (unsigned)(grp[g].x + dh) < (unsigned)srcH && (unsigned)(grp[g].y + dw) < (unsigned)srcW;
        if (OP == OP_FWD && p.s2dx) any &= (p.s2_tapmask[n0 & 15] >> (kh * 2 + kw)) & 1;  // W2 block all zero
        if (any && t)
            *t = make_int4(dh, dw, OP == OP_FWD ? kh * p.FW + kw : p.tf_f[ph_][0][kh] * p.FW + p.tf_f[ph_][1][kw], 0);
        return any;
    }

    // Number of taps used by this tile: one position per tile (G = 128) -> rows x columns in range
    // (validity is separable); several positions -> the union over the groups, candidate by candidate.
    SMCONV_DEV int ntaps(const GenParams& p) const {
        const int ph_ = OP == OP_DX ? phase : 0;
        const int nh = OP == OP_FWD ? p.FH : p.tf_n[ph_][0], nw = OP == OP_FWD ? p.FW : p.tf_n[ph_][1];
        if (ngrp == 1) {
            if (!grp[0].w) return 0;
            const int srcH = OP == OP_FWD ? p.IH : p.OH;
            const int srcW = OP == OP_FWD ? p.IW : p.OW;
            if (OP == OP_FWD && !p.s2dx) {  // rows / columns of the filter whose source is in range: a clamp
                const int ch = min(nh, srcH - grp[0].x) - max(0, -grp[0].x);
                const int cw = min(nw, srcW - grp[0].y) - max(0, -grp[0].y);
                return ch > 0 && cw > 0 ? ch * cw : 0;
            }
            if (OP == OP_FWD) {  // s2dx: the zero W2 blocks of this n-tile are skipped
                int n = 0;
                for (int kh = 0; kh < nh; ++kh)
                    for (int kw = 0; kw < nw; ++kw) n += tap_valid(p, kh, kw, nullptr);
                return n;
            }
            int ch = 0, cw = 0;
            for (int k = 0; k < nh; ++k) ch += (unsigned)(grp[0].x + p.tf_off[ph_][0][k]) < (unsigned)srcH;
            for (int k = 0; k < nw; ++k) cw += (unsigned)(grp[0].y + p.tf_off[ph_][1][k]) < (unsigned)srcW;
            return ch * cw;
        }
        int n = 0;
        for (int kh = 0; kh < nh; ++kh)
            for (int kw = 0; kw < nw; ++kw) n += tap_valid(p, kh, kw, nullptr);
        return n;
    }
};

// In-cluster split-K reduction: CTA `crank` of the S-CTA cluster sums rows [crank*128/S, (crank+1)*128/S)
// of the tile over the S partials held in the cluster's shared memories ([128][PSTRIDE] fp32 each), in
// rank order (fixed: deterministic), and stores them.  Item = (row, 4 columns); consecutive threads take
// consecutive column quads of a row (coalesced 16-B stores).  16 / S items per thread are loaded before
// any is summed: 16 DSMEM loads in flight per thread (one item at a time left the reduce latency-bound,
// ~900 cycles per round trip: 11.6k of the 46k cycles of VGG conv6, trace r02i -> 6.5k, r02k).  Pushing
// the partial rows to their owners with remote stores from the epilogue instead was slower (15k cycles
// of remote stores per CTA, r02m/r02n: a lane holds a row, so a warp's stores scatter over 32 rows).
template <int OP, int BN, int PSTRIDE, int S>
SMCONV_DEV void csk_reduce(const TmaParams& tp, const GenParams& p, uint32_t tiles_addr, int crank, int tid,
                           int nthreads) {
    TileInfo<OP> ti;
    ti.init(tp, p, blockIdx.x, 0);
    constexpr int ROWS = 128 / S, C4 = BN / 4, ITEMS = ROWS * C4, UNR = 16 / S;
    const int n0 = ti.n0 * BN;
    for (int base = tid; base < ITEMS; base += nthreads * UNR) {
        float4 v[UNR][S];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int it = base + u * nthreads;
            if (it < ITEMS) {
                const int rr = crank * ROWS + it / C4, c4 = it % C4;
                const uint32_t la = tiles_addr + (uint32_t)((rr * PSTRIDE + 4 * c4) * 4);
#pragma unroll
                for (int q = 0; q < S; ++q) v[u][q] = ld_cluster_f4(la, (uint32_t)q);
            }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int it = base + u * nthreads;
            if (it >= ITEMS) break;
            const int rr = crank * ROWS + it / C4, c4 = it % C4;
            const int col = n0 + 4 * c4;
            if (col >= p.Ngemm) continue;
            long long o;
            if constexpr (OP == OP_DW) {  // row = output channel; padded (tap, ic) columns drop ic >= IC
                const int oc = ti.m0 + rr;
                if (oc >= p.OC) continue;
                if (p.dw_icp) {
                    const int tap = (int)fdiv((uint32_t)col, p.fd_icp), ic = col - tap * p.dw_icp;
                    if (ic >= p.IC) continue;
                    o = (long long)oc * p.FH * p.FW * p.IC + tap * p.IC + ic;
                } else {
                    o = (long long)oc * p.Ngemm + col;
                }
            } else {
                const RowInfo ri = row_info<OP>(p, ti.phase, ti.m0 + rr);
                if (!ri.ok) continue;
                o = (long long)ri.orow * p.Ngemm + col;
            }
            float4 a = v[u][0];
#pragma unroll
            for (int q = 1; q < S; ++q) {
                a.x += v[u][q].x;
                a.y += v[u][q].y;
                a.z += v[u][q].z;
                a.w += v[u][q].w;
            }
            *reinterpret_cast<float4*>(p.out + o) = a;
        }
    }
}

// Row-coalesced store of one epilogue warp's 32 rows x PW columns (TmaCfg::EPW): lane l holds columns
// [col0, col0 + PW) of row l in f; row r goes to out + ob(lane r) + shift + col (ob < 0: row dropped).
// Staged in the warp's slice of shared memory as 16-B units, unit j of row r at slot j ^ swz(r): the
// row-wise writes (8 lanes = 8 rows per phase) and the run-wise reads (8 lanes = 8 units of 1-2 rows)
// both hit 8 distinct 16-B bank groups.  One STG then covers 32 / (PW / 4) rows of PW * 4 bytes.
template <int PW>
SMCONV_DEV void warp_rows_store(uint8_t* stg, const float (&f)[PW], long long ob, float* out, int col0, int ncols,
                                long long shift, int lane, long long zf1 = 0, long long zf2 = 0) {
    constexpr int F4 = PW / 4, RPI = 32 / F4;
    static_assert(F4 == 4 || F4 == 8, "piece of 16 or 32 columns");
    auto swz = [](int r) { return F4 == 8 ? (r & 7) : ((r >> 1) & 3); };
    __syncwarp();  // the previous piece's reads are done
#pragma unroll
    for (int j = 0; j < F4; ++j)
        *reinterpret_cast<float4*>(stg + (lane * F4 + (j ^ swz(lane))) * 16) =
            make_float4(f[4 * j], f[4 * j + 1], f[4 * j + 2], f[4 * j + 3]);
    __syncwarp();
    const int j = lane % F4, col = col0 + 4 * j;
#pragma unroll
    for (int i = 0; i < F4; ++i) {
        const int r = lane / F4 + RPI * i;
        const long long o = __shfl_sync(0xffffffffu, ob, r);
        const float4 x = *reinterpret_cast<const float4*>(stg + (r * F4 + (j ^ swz(r))) * 16);
        if (o >= 0 && col < ncols) {
            float* const d = out + o + shift + col;
            *reinterpret_cast<float4*>(d) = x;
            if (zf1) {  // TmaParams::zf1 / zf2: the empty stride phases around this pixel
                const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
                *reinterpret_cast<float4*>(d + zf1) = z;
                *reinterpret_cast<float4*>(d + zf2) = z;
                *reinterpret_cast<float4*>(d + zf2 + zf1) = z;
            }
        }
    }
}

template <int OP, int BN, int PLANES, bool PAIR = false>
__global__ void __launch_bounds__(TmaCfg<OP, BN, PLANES, PAIR>::NTHREADS, 1)
    conv_tma_kernel(const __grid_constant__ TmaParams tp, const __grid_constant__ GenParams p) {
    using C = TmaCfg<OP, BN, PLANES, PAIR>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    const uint32_t tiles_addr = (raw_addr + 1023u) & ~1023u;
    uint8_t* tiles_ptr = smem_raw + (tiles_addr - raw_addr);
    TmaAux* aux = reinterpret_cast<TmaAux*>(tiles_ptr + C::STAGES * C::STAGE_BYTES);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int CHK = PLANES == 2 ? tp.chunk_kb : (1 << 30);
    // pairs: both CTAs of a cluster walk the same pair tiles; CTA 0 issues the MMAs and owns the
    // conv / tempty barriers (per-warp arrivals from both CTAs), commits arrive in both CTAs
    const int rank = PAIR ? (int)cluster_ctarank() : 0;
    const int wfirst = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
    const int wstep = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
    constexpr bool CSK_OK = OP != OP_DWT && !PAIR;  // cluster split-K: fwd / dX / dW (not transposed), 1-CTA tiles
    const uint32_t csk_rank = (CSK_OK && tp.csk) ? cluster_ctarank() : 0u;
    unsigned long long* const trc = p.trace;
    if (trc && tid == 0) {
        trace_mark(trc, 0);
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        trc[blockIdx.x * 16 + 15] = gt;
    }

    if (tid == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&aux->full[s], 1);
            mbar_init(&aux->empty[s], 1);
        }
        for (int t = 0; t < C::NT; ++t) {
            // per-warp arrivals of both CTAs (pairs) / per-thread arrivals; TmaParams::alt_conv: one group of
            // NCONV / 2 warps per k-block
            const int nconv = tp.alt_conv ? C::NCONV / 2 : C::NCONV;
            mbar_init(&aux->conv[t], PAIR ? 2 * nconv : nconv * 32);
            mbar_init(&aux->tfree[t], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&aux->tfull[b], 1);
            mbar_init(&aux->tempty[b], PAIR ? 2 * C::NEPI : C::NEPI * 32);
        }
        fence_mbar_init();
    }
    if (warp == C::TMA_W && lane == 0) {
        prefetch_tmap(&tp.mapA);
        prefetch_tmap(&tp.mapB);
        if (C::HYB && p.hyb) prefetch_tmap(&tp.mapBx);
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
    if (tid == 0) trace_mark(trc, 1);
    pdl_trigger();
    // launch.cuh: no global-memory access before the previous kernels completed.  The wait sits in
    // each role right before its first global access, so the producer's first-tile bookkeeping (work
    // item decode + tap list, ~1.5 us on a cold CTA, r02j trace) overlaps the previous kernel's tail
    // under programmatic dependent launch; the MMA and converter warps touch only smem / TMEM.

    if (warp == C::TMA_W) {
        // ======================= TMA producer
        // The single issuing thread is on the critical path when k-blocks are short (BN = 64: one
        // k-block is 128 tensor cycles in TF32), so per-tile bookkeeping is hoisted out of the
        // k-loop: the tap list / box geometry is built once per tile and the loop only adds.
        {
            int s = 0;
            uint32_t r = 0;  // stage index, ring round
            int4* taps = aux->ptaps;
            bool waited = false;  // pdl_wait before the first TMA load
            for (int w = wfirst; w < tp.work; w += wstep) {
                TileInfo<OP> ti;
                ti.init(tp, p, w, rank);
                if (trc && lane == 0 && w == wfirst) trace_mark(trc, 3);
                const int n0 = ti.n0 * BN;
                const int nkb = ti.kb_end - ti.kb_begin;
                if (ti.nkb_eff <= 0) continue;
                if (OP == OP_FWD || OP == OP_DX) {
                    int nt = 0;
                    const int ph_ = OP == OP_DX ? ti.phase : 0;
                    const int nth = OP == OP_FWD ? p.FH : p.tf_n[ph_][0], ntw = OP == OP_FWD ? p.FW : p.tf_n[ph_][1];
                    for (int kh = 0; kh < nth; ++kh)
                        for (int kw = 0; kw < ntw; ++kw)
                            if (ti.tap_valid(p, kh, kw, &taps[nt])) ++nt;  // same value from every lane
                    __syncwarp();
                    if (trc && lane == 0 && w == wfirst) trace_mark(trc, 12);
                    if (!waited) pdl_wait(), waited = true;
                    int j = (int)fdiv((uint32_t)ti.kb_begin, tp.fd_CB), cb = ti.kb_begin - j * tp.CB;
                    int4 tap = taps[j];
                    for (int it = 0; it < nkb; ++it) {
                        if (r > 0) {
                            if (PAIR) mbar_wait_cluster(&aux->empty[s], (r - 1) & 1);
                            else mbar_wait(&aux->empty[s], (r - 1) & 1);
                        }
                        const uint32_t sA = tiles_addr + s * C::STAGE_BYTES;
                        const uint32_t sB = sA + C::B_OFF;
                        if (trc && lane == 0 && r == 0 && s == 0) trace_mark(trc, 2);
                        if (elect_one()) {
                            mbar_arrive_expect_tx(&aux->full[s], C::A_BYTES + (C::HYB && p.hyb ? 2 : 1) * C::B_BYTES);
#pragma unroll
                            for (int g = 0; g < 4; ++g)
                                if (g < ti.ngrp) tma_load_4d(sA + g * tp.G * 128, &tp.mapA, &aux->full[s], cb * 32,
                                            ti.grp[g].y + tap.y, ti.grp[g].x + tap.x, ti.grp[g].z);
                            const int nb0 = n0 + rank * C::BNC;  // this CTA's half of B (pairs)
                            if (OP == OP_FWD || tp.dx_bk) {  // W (OC, T, IC) / Wt (IC, T, OC): K-major box
                                tma_load_3d(sB, &tp.mapB, &aux->full[s], cb * 32, tap.z, nb0);
                            } else if (tp.dx_ragged) {
#pragma unroll 1
                                for (int j = 0; j < C::BNC / 32; ++j)
                                    tma_load_3d(sB + j * 4096, &tp.mapB, &aux->full[s], nb0 + 32 * j, cb * 32, tap.z);
                            } else {
                                tma_load_4d(sB, &tp.mapB, &aux->full[s], 0, cb * 32, nb0 / 32, tap.z);
                            }
                            if (C::HYB && p.hyb) tma_load_4d(sB + C::B_BYTES, &tp.mapBx, &aux->full[s], 0, cb, nb0, tap.z);
                        }
                        __syncwarp();
                        if (++cb == tp.CB) {
                            cb = 0;
                            tap = taps[++j < nt ? j : 0];
                        }
                        if (++s == C::STAGES) {
                            s = 0;
                            ++r;
                        }
                    }
                } else {
                    // image-block-major reduction order (k-block = 32 images at one position)
                    const int P = p.OH * p.OW;
                    int nb = (int)fdiv((uint32_t)ti.kb_begin, tp.fd_P[0]), pos = ti.kb_begin - nb * P;
                    int oh = (int)fdiv((uint32_t)pos, p.fd_OW), ow = pos - oh * p.OW;
                    // X boxes of this tile (dw: B side; dwT: A side): tap offsets and channel block
                    const int nboxes = OP == OP_DWT ? tp.a_boxes : tp.b_boxes;
                    const int bcols = OP == OP_DWT ? tp.a_box_cols : tp.b_box_cols;
                    const int base = OP == OP_DWT ? ti.m0 : n0 + rank * C::BNC;  // this CTA's half of B (pairs)
                    const int lim = OP == OP_DWT ? p.M : p.Ngemm;
                    int nbox = 0;
                    for (int b = 0; b < nboxes; ++b) {
                        const int c0 = base + b * bcols;
                        if (c0 >= lim) break;
                        const int cpt = (OP == OP_DW && p.dw_icp) ? p.dw_icp : p.IC;  // GEMM columns per tap
                        const int tp_ = c0 / cpt, icb = (c0 - tp_ * cpt) / 32;
                        const int fh_ = tp_ / p.FW, fw_ = tp_ - fh_ * p.FW;
                        taps[b] = make_int4(fw_ - p.pw, fh_ - p.ph, icb, 0);  // same value from every lane
                        ++nbox;
                    }
                    __syncwarp();
                    if (!waited) pdl_wait(), waited = true;
                    const uint32_t xbytes = nbox * bcols * 128;
                    const uint32_t tx = OP == OP_DWT ? xbytes + C::B_BYTES : C::A_BYTES + xbytes;
                    for (int it = 0; it < nkb; ++it) {
                        if ((unsigned)(oh - ti.vr_lo) >= (unsigned)(ti.vr_hi - ti.vr_lo) ||
                            (unsigned)(ow - ti.vc_lo) >= (unsigned)(ti.vc_hi - ti.vc_lo)) {
                            // skipped k-block (all-padding source for this tile's tap): no stage
                            if (++ow == p.OW) {
                                ow = 0;
                                if (++oh == p.OH) oh = 0;
                            }
                            if (++pos == P) {
                                pos = 0;
                                ++nb;
                            }
                            continue;
                        }
                        if (r > 0) {
                            if (PAIR) mbar_wait_cluster(&aux->empty[s], (r - 1) & 1);
                            else mbar_wait(&aux->empty[s], (r - 1) & 1);
                        }
                        const uint32_t sA = tiles_addr + s * C::STAGE_BYTES;
                        const uint32_t sB = sA + C::B_OFF;
                        const uint32_t sX = OP == OP_DWT ? sA : sB;
                        const int iw0 = ow * p.sw, ih0 = oh * p.sh;
                        if (elect_one()) {
                            mbar_arrive_expect_tx(&aux->full[s], tx);
                            for (int b = 0; b < nbox; ++b) {
                                if (OP == OP_DW && tp.dw_b_ragged)  // (32 ic, 32 n, 1, 1); ic >= IC zero-filled
                                    tma_load_4d(sX + b * bcols * 128, &tp.mapB, &aux->full[s], taps[b].z * 32, nb * 32,
                                                iw0 + taps[b].x, ih0 + taps[b].y);
                                else
                                    tma_load_5d(sX + b * bcols * 128, OP == OP_DWT ? &tp.mapA : &tp.mapB, &aux->full[s],
                                                0, nb * 32, taps[b].z, iw0 + taps[b].x, ih0 + taps[b].y);
                            }
                            if (OP == OP_DWT) {
                                tma_load_4d(sB, &tp.mapB, &aux->full[s], 0, nb * 32, n0 / 32, pos);
                            } else if (tp.dw_a_ragged) {  // 4 x (32 oc, 32 n, 1); oc >= OC zero-filled
#pragma unroll 1
                                for (int j = 0; j < 4; ++j)
                                    tma_load_3d(sA + j * 4096, &tp.mapA, &aux->full[s], ti.m0 + 32 * j, nb * 32, pos);
                            } else {
                                tma_load_4d(sA, &tp.mapA, &aux->full[s], 0, nb * 32, ti.m0 / 32, pos);
                            }
                        }
                        __syncwarp();
                        if (++ow == p.OW) {
                            ow = 0;
                            if (++oh == p.OH) oh = 0;
                        }
                        if (++pos == P) {
                            pos = 0;
                            ++nb;
                        }
                        if (++s == C::STAGES) {
                            s = 0;
                            ++r;
                        }
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == C::MMA_W) {
        // ======================= MMA issuer (whole warp runs the loop, one elected lane issues)
        // pairs: CTA 0 issues M = 256 MMAs for both CTAs; CTA 1's MMA warp only owns its TMEM
        if (!PAIR || rank == 0) {
            // dX with the transposed plane (TmaParams::dx_bk): B K-major like the fwd
            const bool bmn = C::B_MN && !(OP == OP_DX && tp.dx_bk);
            constexpr uint32_t IDESC_MN = idesc_tf32(PAIR ? 256 : 128, BN, C::A_TMEM ? false : C::A_MN, C::B_MN);  // TMEM A: K along columns
            constexpr uint32_t IDESC_KM = idesc_tf32(PAIR ? 256 : 128, BN, C::A_TMEM ? false : C::A_MN, false);
            const uint32_t IDESC = bmn ? IDESC_MN : IDESC_KM;
            const uint32_t albo = C::A_MN ? 4096u : 16u, blbo = bmn ? 4096u : 16u;
            const uint32_t asbo = C::A_MN ? 512u : 1024u, bsbo = bmn ? 512u : 1024u;
            const uint32_t alay = C::A_MN ? kLayoutSW128Base32 : kLayoutSW128;
            const uint32_t blay = bmn ? kLayoutSW128Base32 : kLayoutSW128;
            // descriptors of stage 0; stage s / k-step g only add to the 14-bit start-address field
            const uint64_t adH0 = make_sdesc(tiles_addr, albo, asbo, alay);
            const uint64_t bdH0 = make_sdesc(tiles_addr + C::B_OFF, blbo, bsbo, blay);
            constexpr uint64_t A_G = C::A_MN ? 64 : 2;  // (1024 or 32 bytes) >> 4
            const uint64_t B_G = bmn ? 64 : 2;
            // 3xTF32 cross terms: bf16 B' plane [b_lo | b] (K-major, 128 B per row) after b_hi
            constexpr uint32_t IDESC_X = idesc_bf16(PAIR ? 256 : 128, BN, false, false);
            const uint64_t bx0 = make_sdesc(tiles_addr + C::B_OFF + C::B_BYTES, 16u, 1024u, kLayoutSW128);
            // dW hybrid: B' [64 k'][BNC] bf16 MN-major (LBO = one 64-column atom = 64 rows x 128 B)
            constexpr uint32_t IDESC_XW = idesc_bf16(PAIR ? 256 : 128, BN, false, true);
            const uint64_t bxw0 = make_sdesc(tiles_addr + C::B_OFF + C::B_BYTES, 8192u, 1024u, kLayoutSW128);
            const bool hybw = C::HYBW && tp.dw_hyb;
            int s = 0, in_chunk = 0;
            uint32_t r = 0, c = 0, q = 0;  // stage, ring round, chunk counter, k-block (global across tiles)
            for (int w = wfirst; w < tp.work; w += wstep) {
                TileInfo<OP> ti;
                ti.init(tp, p, w, rank);
                const int nkb = ti.nkb_eff;
                for (int it = 0; it < nkb; ++it) {
                    const int buf = c & 1;
                    if (in_chunk == 0 && c >= 2) {
                        if (PAIR) mbar_wait_cluster(&aux->tempty[buf], ((c >> 1) - 1) & 1);
                        else mbar_wait(&aux->tempty[buf], ((c >> 1) - 1) & 1);
                        tc_fence_after();
                    }
                    const uint32_t t = q % C::NT, rt = q / C::NT;  // TMEM A slot
                    if (PAIR) mbar_wait_cluster(&aux->conv[t], rt & 1);
                    else if (PLANES == 2) mbar_wait(&aux->conv[t], rt & 1);
                    else mbar_wait(&aux->full[s], r & 1);
                    tc_fence_after();
                    const uint32_t d = tmem + (uint32_t)(buf * BN);
                    const uint64_t so = (uint64_t)(s * C::STAGE_BYTES) >> 4;
                    const bool last = (in_chunk + 1 == CHK || it == nkb - 1);
                    if (trc && lane == 0 && q == 0) trace_mark(trc, 4);
                    if (elect_one()) {
#pragma unroll
                        for (int g = 0; g < C::BK / 8; ++g) {
                            const uint64_t adH = adH0 + so + g * A_G, bdH = bdH0 + so + g * B_G;
                            const uint32_t acc0 = (in_chunk > 0 || g > 0) ? 1u : 0u;
                            const uint32_t ahi = tmem + (uint32_t)(C::A_TCOL0 + t * 64 + g * 8);
                            if ((C::HYB && p.hyb) || hybw) {  // a_hi * b_hi (TF32); cross terms below
                                if (PAIR) mma2_tf32_ts(d, ahi, bdH, IDESC, acc0);
                                else mma_tf32_ts(d, ahi, bdH, IDESC, acc0);
                            } else if (C::A_TMEM && PAIR) {  // three TF32 MMAs, M = 256 (dW; fwd / dX !hyb)
                                mma2_tf32_ts(d, ahi + 32, bdH, IDESC, acc0);
                                mma2_tf32_ts(d, ahi, bdH + (C::B_BYTES >> 4), IDESC, 1u);
                                mma2_tf32_ts(d, ahi, bdH, IDESC, 1u);
                            } else if (C::A_TMEM) {  // three TF32 MMAs, b_lo plane after b_hi (dW; fwd / dX !hyb)
                                mma_tf32_ts(d, ahi + 32, bdH, IDESC, acc0);
                                mma_tf32_ts(d, ahi, bdH + (C::B_BYTES >> 4), IDESC, 1u);
                                mma_tf32_ts(d, ahi, bdH, IDESC, 1u);
                            } else {
                                mma_tf32_ss(d, adH, bdH, IDESC, acc0);
                            }
                        }
                        if (C::HYB && p.hyb) {
                            // cross terms a_hi*b_lo + a_lo*b in bf16: A' = [bf16(a_hi) | bf16(a_lo)]
                            // (TMEM, 32 columns), B' = [bf16(b_lo) | bf16(b)]: K = 64 in 4 MMAs
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                const uint32_t ax = tmem + (uint32_t)(C::A_TCOL0 + t * 64 + 32 + j * 8);
                                if (PAIR) mma2_bf16_ts(d, ax, bx0 + so + j * 2, IDESC_X, 1u);
                                else mma_bf16_ts(d, ax, bx0 + so + j * 2, IDESC_X, 1u);
                            }
                        }
                        if (hybw) {  // dW: the same cross terms, B' rows 16 j .. 16 j + 15 (2 KB apart)
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                const uint32_t ax = tmem + (uint32_t)(C::A_TCOL0 + t * 64 + 32 + j * 8);
                                if (PAIR) mma2_bf16_ts(d, ax, bxw0 + so + j * (2048 >> 4), IDESC_XW, 1u);
                                else mma_bf16_ts(d, ax, bxw0 + so + j * (2048 >> 4), IDESC_XW, 1u);
                            }
                        }
                        if (trc && last) trace_mark(trc, 5);
                        if (PAIR) {
                            mma2_commit_both(&aux->empty[s]);
                            mma2_commit_both(&aux->tfree[t]);
                            if (last) mma2_commit_both(&aux->tfull[buf]);
                        } else {
                            mma_commit(&aux->empty[s]);
                            if (C::A_TMEM) mma_commit(&aux->tfree[t]);
                            if (last) mma_commit(&aux->tfull[buf]);
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
                    ++q;
                }
            }
        }
        __syncwarp();
    } else if (warp >= C::CONV_W0 && tp.alt_conv) {
        // ======================= 3xTF32 converters in two groups of 4 warps on alternate k-blocks
        // (TmaParams::alt_conv): a warp = one TMEM lane quadrant, both K halves.  With all 8 warps on every
        // k-block the chain LDS -> split -> tcgen05.st -> wait -> arrive ran one k-block at a time (the same
        // split made the DWS dW converters 18 % faster in TF32, r02ca)
        const int grp = (warp - C::CONV_W0) >> 2;
        const int ct4 = tid - (C::CONV_W0 + 4 * grp) * 32;  // 0..127 within the group
        constexpr int NCT2 = C::NCONV > 0 ? C::NCONV * 16 : 32;
        const int qd = warp & 3;
        const int row = qd * 32 + lane;
        uint32_t q = 0;
        for (int w = wfirst; w < tp.work; w += wstep) {
            TileInfo<OP> ti;
            ti.init(tp, p, w, rank);
            const int nkb = ti.nkb_eff;
            for (int it = 0; it < nkb; ++it, ++q) {
                if ((int)(q & 1u) != grp) continue;
                const int s = q % C::STAGES;
                const uint32_t r = q / C::STAGES;
                const uint32_t t = q % C::NT, rt = q / C::NT;  // TMEM A slot
                mbar_wait(&aux->full[s], r & 1);
                if (rt > 0) {  // slot t's previous k-block has been multiplied
                    if (PAIR) mbar_wait_cluster(&aux->tfree[t], (rt - 1) & 1);
                    else mbar_wait(&aux->tfree[t], (rt - 1) & 1);
                    tc_fence_after();
                }
                uint8_t* st = tiles_ptr + s * C::STAGE_BYTES;
                constexpr int NB2 = C::B_BYTES / 16 / NCT2;
                static_assert(!C::A_TMEM || NB2 * NCT2 * 16 == C::B_BYTES, "converter split");
                const uint32_t ta = tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(C::A_TCOL0 + t * 64);
                const bool hyb_a = (C::HYB && p.hyb) || (C::HYBW && tp.dw_hyb);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    float e[16];
                    if (C::A_MN) {  // MN-major A tile [32 k][128 m]: one 4-byte element per k
#pragma unroll
                        for (int k = 0; k < 16; ++k)
                            e[k] = *reinterpret_cast<const float*>(st + mnmaj_off((uint32_t)(16 * h + k), (uint32_t)(row & ~3)) +
                                                                   (row & 3) * 4);
                    } else {  // K-major A tile [128 m][32 k]: four 16-B chunks of this row
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const float4 v =
                                *reinterpret_cast<const float4*>(st + kmaj_off((uint32_t)row, (uint32_t)(4 * h + c)));
                            e[4 * c] = v.x;
                            e[4 * c + 1] = v.y;
                            e[4 * c + 2] = v.z;
                            e[4 * c + 3] = v.w;
                        }
                    }
                    if (hyb_a) {
                        uint32_t hi[16], xh[8], xl[8];
                        split_a16(e, hi, xh, xl);
                        tmem_st_32x32b_x16(ta + h * 16, hi);
                        tmem_st_32x32b_x8(ta + 32 + h * 8, xh);
                        tmem_st_32x32b_x8(ta + 48 + h * 8, xl);
                    } else {
                        uint32_t hi[16], lo[16];
#pragma unroll
                        for (int k = 0; k < 16; ++k) {
                            const uint32_t hb = __float_as_uint(e[k]) & 0xFFFFE000u;
                            hi[k] = hb;
                            lo[k] = __float_as_uint(e[k] - __uint_as_float(hb));
                        }
                        tmem_st_32x32b_x16(ta + h * 16, hi);
                        tmem_st_32x32b_x16(ta + 32 + h * 16, lo);
                    }
                }
                if (C::HYBW && tp.dw_hyb) {  // dW: B' = [bf16(b_lo) ; bf16(b)] (as the 8-warp path below)
                    const float4* bH = reinterpret_cast<const float4*>(st + C::B_OFF);
                    uint8_t* bX = st + C::B_OFF + C::B_BYTES;
#pragma unroll
                    for (int e2 = 0; e2 < NB2; ++e2) {
                        const uint32_t i = (uint32_t)(ct4 + e2 * NCT2);
                        const uint32_t k = (i & 255u) >> 3, c32 = (i & 7u) >> 1;
                        const uint32_t mn = (i >> 8) * 32u + ((c32 ^ (k & 3u)) << 3) + ((i & 1u) << 2);
                        const float4 b = bH[i];
                        const float lx = b.x - __uint_as_float(__float_as_uint(b.x) & 0xFFFFE000u);
                        const float ly = b.y - __uint_as_float(__float_as_uint(b.y) & 0xFFFFE000u);
                        const float lz = b.z - __uint_as_float(__float_as_uint(b.z) & 0xFFFFE000u);
                        const float lw = b.w - __uint_as_float(__float_as_uint(b.w) & 0xFFFFE000u);
                        *reinterpret_cast<uint2*>(bX + mnmaj16_off(k, mn, 64u)) =
                            make_uint2(pack_bf16x2(lx, ly), pack_bf16x2(lz, lw));
                        *reinterpret_cast<uint2*>(bX + mnmaj16_off(k + 32u, mn, 64u)) =
                            make_uint2(pack_bf16x2(b.x, b.y), pack_bf16x2(b.z, b.w));
                    }
                } else if (!(C::HYB && p.hyb)) {  // b_lo plane (dW three-MMA form, fwd / dX without the W' plane)
                    const float4* bH = reinterpret_cast<const float4*>(st + C::B_OFF);
                    float4* bL = reinterpret_cast<float4*>(st + C::B_OFF + C::B_BYTES);
#pragma unroll
                    for (int e2 = 0; e2 < NB2; ++e2) {
                        const float4 v = bH[ct4 + e2 * NCT2];
                        float4 o;
                        o.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
                        o.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
                        o.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
                        o.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
                        bL[ct4 + e2 * NCT2] = o;
                    }
                }
                tmem_st_wait();
                if (!(C::HYB && p.hyb)) fence_proxy_async_smem();  // b_lo / B' planes -> the MMA's async proxy
                tc_fence_before();
                if (PAIR) {  // one arrival per warp, on CTA 0's barrier (it issues the MMAs)
                    __syncwarp();
                    if (lane == 0) mbar_arrive_remote(&aux->conv[t], 0);
                } else {
                    mbar_arrive(&aux->conv[t]);
                }
            }
        }
    } else if (warp >= C::CONV_W0) {
        // ======================= 3xTF32 split converters: lo = a - trunc_tf32(a)
        const int ct = tid - C::CONV_W0 * 32;
        constexpr int NCT = C::NCONV > 0 ? C::NCONV * 32 : 32;  // (dead code when PLANES == 1)
        uint32_t q = 0;
        for (int w = wfirst; w < tp.work; w += wstep) {
            TileInfo<OP> ti;
            ti.init(tp, p, w, rank);
            const int nkb = ti.nkb_eff;
            for (int it = 0; it < nkb; ++it, ++q) {
                const int s = q % C::STAGES;
                const uint32_t r = q / C::STAGES;
                const uint32_t t = q % C::NT, rt = q / C::NT;  // TMEM A slot
                mbar_wait(&aux->full[s], r & 1);
                if (C::A_TMEM && rt > 0) {  // slot t's previous k-block has been multiplied
                    if (PAIR) mbar_wait_cluster(&aux->tfree[t], (rt - 1) & 1);
                    else mbar_wait(&aux->tfree[t], (rt - 1) & 1);
                    tc_fence_after();
                }
                uint8_t* st = tiles_ptr + s * C::STAGE_BYTES;
                constexpr int NB = C::B_BYTES / 16 / NCT;
                static_assert(NB * NCT * 16 == C::B_BYTES, "converter split");
                auto lo4 = [](float4 v) {
                    float4 o;
                    o.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
                    o.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
                    o.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
                    o.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
                    return o;
                };
                if (C::A_TMEM) {
                    // this thread: A row 32*(warp%4)+lane, K half h: hi/lo -> TMEM slot s (tcgen05.st)
                    const int qd = warp & 3, h = (warp - C::CONV_W0) >> 2;
                    const int row = qd * 32 + lane;
                    float e[16];
                    if (C::A_MN) {  // MN-major A tile [32 k][128 m]: one 4-byte element per k
#pragma unroll
                        for (int k = 0; k < 16; ++k)
                            e[k] = *reinterpret_cast<const float*>(st + mnmaj_off((uint32_t)(16 * h + k), (uint32_t)(row & ~3)) +
                                                                   (row & 3) * 4);
                    } else {  // K-major A tile [128 m][32 k]: four 16-B chunks of this row
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const float4 v =
                                *reinterpret_cast<const float4*>(st + kmaj_off((uint32_t)row, (uint32_t)(4 * h + c)));
                            e[4 * c] = v.x;
                            e[4 * c + 1] = v.y;
                            e[4 * c + 2] = v.z;
                            e[4 * c + 3] = v.w;
                        }
                    }
                    // slot columns: [0,32) a_hi (TF32 operand), [32,48) bf16(a_hi) for k = 0..31 in
                    // pairs, [48,64) bf16(a_lo) likewise; this thread has k in [16h, 16h+16)
                    // (dW: [32,64) a_lo fp32 for the third TF32 MMA)
                    const uint32_t ta = tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(C::A_TCOL0 + t * 64);
                    if ((C::HYB && p.hyb) || (C::HYBW && tp.dw_hyb)) {
                        uint32_t hi[16], xh[8], xl[8];
                        split_a16(e, hi, xh, xl);
                        tmem_st_32x32b_x16(ta + h * 16, hi);
                        tmem_st_32x32b_x8(ta + 32 + h * 8, xh);
                        tmem_st_32x32b_x8(ta + 48 + h * 8, xl);
                    } else {
                        uint32_t hi[16], lo[16];
#pragma unroll
                        for (int k = 0; k < 16; ++k) {
                            const uint32_t hb = __float_as_uint(e[k]) & 0xFFFFE000u;
                            hi[k] = hb;
                            lo[k] = __float_as_uint(e[k] - __uint_as_float(hb));
                        }
                        tmem_st_32x32b_x16(ta + h * 16, hi);
                        tmem_st_32x32b_x16(ta + 32 + h * 16, lo);
                    }
                } else {
                    const float4* aH = reinterpret_cast<const float4*>(st);
                    float4* aL = reinterpret_cast<float4*>(st + C::A_BYTES);
                    constexpr int NA = C::A_BYTES / 16 / NCT;
                    static_assert(NA * NCT * 16 == C::A_BYTES, "converter split");
                    float4 va[NA];
#pragma unroll
                    for (int i = 0; i < NA; ++i) va[i] = aH[ct + i * NCT];
#pragma unroll
                    for (int i = 0; i < NA; ++i) aL[ct + i * NCT] = lo4(va[i]);
                }
                if (C::HYBW && tp.dw_hyb) {
                    // dW hybrid: B' = [bf16(b_lo) ; bf16(b)] from the fp32 MN-major X tile.  float4 i of the
                    // tile: 32-column block i / 256, K-row (i % 256) / 8, 32-B chunk (i % 8) / 2 stored
                    // swizzled with k % 4 (mnmaj_off), 16-B half i % 2
                    const float4* bH = reinterpret_cast<const float4*>(st + C::B_OFF);
                    uint8_t* bX = st + C::B_OFF + C::B_BYTES;
                    float4 vb[NB];
#pragma unroll
                    for (int i = 0; i < NB; ++i) vb[i] = bH[ct + i * NCT];
#pragma unroll
                    for (int e2 = 0; e2 < NB; ++e2) {
                        const uint32_t i = (uint32_t)(ct + e2 * NCT);
                        const uint32_t k = (i & 255u) >> 3, c32 = (i & 7u) >> 1;
                        const uint32_t mn = (i >> 8) * 32u + ((c32 ^ (k & 3u)) << 3) + ((i & 1u) << 2);
                        const float4 b = vb[e2];
                        const float4 l = lo4(b);
                        *reinterpret_cast<uint2*>(bX + mnmaj16_off(k, mn, 64u)) =
                            make_uint2(pack_bf16x2(l.x, l.y), pack_bf16x2(l.z, l.w));
                        *reinterpret_cast<uint2*>(bX + mnmaj16_off(k + 32u, mn, 64u)) =
                            make_uint2(pack_bf16x2(b.x, b.y), pack_bf16x2(b.z, b.w));
                    }
                } else if (!(C::HYB && p.hyb)) {  // b_lo plane (dW, fwd / dX without the W' plane, the SS fallback)
                    const float4* bH = reinterpret_cast<const float4*>(st + C::B_OFF);
                    float4* bL = reinterpret_cast<float4*>(st + C::B_OFF + C::B_BYTES);
                    float4 vb[NB];
#pragma unroll
                    for (int i = 0; i < NB; ++i) vb[i] = bH[ct + i * NCT];
#pragma unroll
                    for (int i = 0; i < NB; ++i) bL[ct + i * NCT] = lo4(vb[i]);
                }
                if (C::A_TMEM) tmem_st_wait();
                // generic-proxy shared-memory writes (a_lo / b_lo planes) must be visible to the MMA's
                // async proxy; the hybrid fwd / dX converters write TMEM only
                if (!C::A_TMEM || !(C::HYB && p.hyb)) fence_proxy_async_smem();
                tc_fence_before();
                if (PAIR) {  // one arrival per warp, on CTA 0's barrier (it issues the MMAs)
                    __syncwarp();
                    if (lane == 0) mbar_arrive_remote(&aux->conv[t], 0);
                } else {
                    mbar_arrive(&aux->conv[t]);
                }
            }
        }
    } else {
        // ======================= epilogue warps 0-7 (+ promotion of TMEM chunks, 3xTF32)
        pdl_wait();  // global stores (and the fused epilogue's reads of A) follow
        const int qd = warp & 3, half = warp >> 2;
        const int row = qd * 32 + lane;
        constexpr int HALF = BN / 2;
        const uint32_t lane_addr = (uint32_t)(qd * 32) << 16;
        uint8_t* const stg = tiles_ptr + C::STAGES * C::STAGE_BYTES + C::AUX_BYTES + warp * (32 * C::EPW * 4);
        // the fused epilogue (p.epi) always takes the coalesced path when the kernel has one, so its
        // inlined transform / statistics code exists once per column loop (code size: see epilogue.cuh)
        const bool coal = C::EPW > 0 && (tp.coalesce || p.epi.mode != EPI_NONE) && !(CSK_OK && tp.csk);
        uint32_t c = 0;
        for (int w = wfirst; w < tp.work; w += wstep) {
            TileInfo<OP> ti;
            ti.init(tp, p, w, rank);
            const int n0 = ti.n0 * BN;
            const int nkb = ti.nkb_eff;
            const int nch = nkb > 0 ? (nkb + CHK - 1) / CHK : 0;
            float* outp = p.out + (long long)ti.split * p.split_stride;
            long long obase = -1;
            int ts_n0 = 0, ts_pix = 0;
            bool ts_ok = false;
            if (OP == OP_DW) {
                const int oc = ti.m0 + row;
                if (oc < p.OC) obase = (long long)oc * (p.dw_icp ? p.FH * p.FW * p.IC : p.Ngemm);
            } else if (OP == OP_DWT) {
                const int m = ti.m0 + row;  // (tap, ic) index; dW[oc][m] at oc * M + m
                if (m < p.M) obase = m;
            } else {
                RowInfo ri = row_info<OP>(p, ti.phase, ti.m0 + row);
                // TMA-store coordinates of this warp's 32 rows (lane 0's row: 32 consecutive images at one pixel)
                const int P_ = OP == OP_FWD ? p.OH * p.OW : p.IH * p.IW;
                ts_n0 = __shfl_sync(0xffffffffu, ri.n, 0);
                ts_pix = __shfl_sync(0xffffffffu, ri.orow - ri.n * P_, 0);
                ts_ok = __shfl_sync(0xffffffffu, (int)ri.ok, 0) != 0;
                if (OP == OP_FWD && p.s2dx) {  // super-pixel (i', j') -> dX pixel (2i'-2, 2j'-2) of column block q = 0
                    const int i1 = ts_pix / p.OW, j1 = ts_pix - i1 * p.OW;
                    ts_ok = ts_ok && i1 >= 1 && j1 >= 1;
                    ts_pix = (2 * i1 - 2) * p.s2_IW + 2 * j1 - 2;
                }
                if (OP == OP_FWD && p.s2dx) {
                    if (ri.ok) {
                        const int pos = ri.orow - ri.n * p.OH * p.OW, oh = pos / p.OW, ow = pos - oh * p.OW;
                        if (oh >= 1 && ow >= 1)
                            obase = ((long long)(ri.n * p.s2_IH + 2 * oh - 2) * p.s2_IW + 2 * ow - 2) * p.s2_IC;
                    }
                } else if (ri.ok) {
                    obase = (long long)ri.orow * p.Ngemm;
                }
            }
            // element offset of GEMM column col of this thread's row in the output tensor (fwd / dX)
            auto out_off = [&](int col) -> long long {
                if (OP == OP_FWD && p.s2dx)  // column (pi, pj, ic): dX row 2i'-2+pi
                    return col >= 2 * p.s2_IC ? obase + col + (long long)(p.s2_IW - 2) * p.s2_IC : obase + col;
                return obase + col;
            };
            // fused epilogue (epilogue.cuh): 32-row group of this warp for the statistics partial rows
            // (dX: rows of phase k start at phase_tile0[k] tiles of 128 rows, or of 256 for pair tiles)
            const int egrp = (((OP == OP_DX ? p.phase_tile0[ti.phase] : 0) << (tp.pair ? 8 : 7)) + ti.m0 >> 5) + qd;
            // row-coalesced stores (TmaCfg::EPW): s2dx columns (pi = 1, pj, ic) land one dX row further
            auto s2shift = [&](int col0) -> long long {
                return (OP == OP_FWD && p.s2dx && col0 >= 2 * p.s2_IC) ? (long long)(p.s2_IW - 2) * p.s2_IC : 0;
            };
            // TMA-store coordinates of the piece starting at GEMM column col0: (channel, pixel); s2dx columns
            // (pi, pj, ic) land on dX pixel (2i'-2+pi, 2j'-2+pj) (IC % 64 == 0: a piece never straddles)
            auto ts_c = [&](int col0) -> int {
                return (OP == OP_FWD && p.s2dx) ? col0 - (col0 / p.s2_IC) * p.s2_IC : col0;
            };
            auto ts_p = [&](int col0) -> int {
                if (OP == OP_FWD && p.s2dx) {
                    const int q = col0 / p.s2_IC;
                    return ts_pix + (q >> 1) * p.s2_IW + (q & 1);
                }
                return ts_pix;
            };
            // 4 consecutive GEMM columns of this thread's row -> output
            auto st4 = [&](int col, float x, float y, float z, float w4) {
                if (CSK_OK && tp.csk) {  // cluster split-K: this CTA's partial -> own shared memory
                    *reinterpret_cast<float4*>(tiles_ptr + ((size_t)row * C::PSTRIDE + (col - n0)) * 4) =
                        make_float4(x, y, z, w4);
                } else if (C::IS_DW && p.mc_out) {  // fused dW all-reduce: add into every rank's copy
                    if (OP == OP_DWT) {
                        float* o = p.mc_out + obase + (long long)col * p.M;  // 4 output channels, one element each
                        asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(o), "f"(x) : "memory");
                        asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(o + p.M), "f"(y) : "memory");
                        asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(o + 2 * (long long)p.M),
                                     "f"(z) : "memory");
                        asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(o + 3 * (long long)p.M),
                                     "f"(w4) : "memory");
                    } else if (p.dw_icp) {
                        const int tap = (int)fdiv((uint32_t)col, p.fd_icp), ic = col - tap * p.dw_icp;
                        if (ic < p.IC) mc_red_add_f4(p.mc_out + obase + tap * p.IC + ic, make_float4(x, y, z, w4));
                    } else {
                        mc_red_add_f4(p.mc_out + obase + col, make_float4(x, y, z, w4));
                    }
                } else if (OP == OP_DWT) {  // column = oc: a warp's 32 rows are 128 contiguous bytes per column
                    float* o = outp + obase + (long long)col * p.M;
                    o[0] = x;
                    o[p.M] = y;
                    o[2 * (long long)p.M] = z;
                    o[3 * (long long)p.M] = w4;
                } else if (OP == OP_FWD && p.s2dx) {  // column (pi, pj, ic): dX row 2i'-2+pi
                    *reinterpret_cast<float4*>(outp + out_off(col)) = make_float4(x, y, z, w4);
                } else if (OP == OP_DW && p.dw_icp) {  // padded (tap, ic) column: drop ic >= IC
                    const int tap = (int)fdiv((uint32_t)col, p.fd_icp), ic = col - tap * p.dw_icp;
                    if (ic < p.IC)
                        *reinterpret_cast<float4*>(outp + obase + tap * p.IC + ic) = make_float4(x, y, z, w4);
                } else {
                    *reinterpret_cast<float4*>(outp + obase + col) = make_float4(x, y, z, w4);
                }
            };
            if (PLANES == 2) {
                float acc[HALF];
#pragma unroll
                for (int e = 0; e < HALF; ++e) acc[e] = 0.f;
                for (int k = 0; k < nch; ++k, ++c) {
                    const int buf = c & 1;
                    if (PAIR) mbar_wait_cluster(&aux->tfull[buf], (c >> 1) & 1);
                    else mbar_wait(&aux->tfull[buf], (c >> 1) & 1);
                    tc_fence_after();
                    if (trc && tid == 0) trace_mark(trc, 6);
#pragma unroll
                    for (int c0 = 0; c0 < HALF; c0 += 16) {
                        uint32_t v[16];
                        tmem_ld_32x32b_x16(tmem + lane_addr + (uint32_t)(buf * BN + half * HALF + c0), v);
                        tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 16; ++e) acc[c0 + e] += __uint_as_float(v[e]);
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
                        if (p.epi.mode != EPI_NONE) {  // in place on acc, 16 columns at a time
#pragma unroll
                            for (int c0 = 0; c0 < HALF; c0 += 16) {
                                const int col0 = n0 + half * HALF + c0;
                                epi_apply16(p.epi, *reinterpret_cast<float(*)[16]>(&acc[c0]),
                                            obase >= 0 && col0 < p.Ngemm ? out_off(col0) : -1, col0, p.Ngemm, egrp, lane);
                            }
                        }
#pragma unroll
                        for (int c0 = 0; c0 < HALF; c0 += C::EPW) {
                            const int col0 = n0 + half * HALF + c0;
                            if (tp.tstore)
                                warp_rows_tstore<C::EPW>(stg, *reinterpret_cast<const float(*)[C::EPW]>(&acc[c0]), &tp.mapY,
                                                         ts_c(col0), ts_p(col0), ts_n0, ts_ok, lane);
                            else
                                warp_rows_store<C::EPW>(stg, *reinterpret_cast<const float(*)[C::EPW]>(&acc[c0]), obase,
                                                        outp, col0, p.Ngemm, s2shift(col0), lane, tp.zf1, tp.zf2);
                        }
                        stored = true;
                    }
                }
                if (stored) {
                } else if (C::EPW == 0 && !C::IS_DW && p.epi.mode != EPI_NONE) {
#pragma unroll
                    for (int c0 = 0; c0 < HALF; c0 += 16) {
                        const int col0 = n0 + half * HALF + c0;
                        float v[16];
#pragma unroll
                        for (int e = 0; e < 16; ++e) v[e] = acc[c0 + e];
                        epi_apply16(p.epi, v, obase >= 0 && col0 < p.Ngemm ? out_off(col0) : -1, col0, p.Ngemm, egrp,
                                    lane);
                        if (obase >= 0)
#pragma unroll
                            for (int e = 0; e < 16; e += 4)
                                if (col0 + e < p.Ngemm) st4(col0 + e, v[e], v[e + 1], v[e + 2], v[e + 3]);
                    }
                } else if (obase >= 0) {
#pragma unroll
                    for (int e = 0; e < HALF; e += 4) {
                        const int col = n0 + half * HALF + e;
                        if (col < p.Ngemm) st4(col, acc[e], acc[e + 1], acc[e + 2], acc[e + 3]);
                    }
                }
            } else {
                const int buf = c & 1;
                if (nch > 0) {
                    if (PAIR) mbar_wait_cluster(&aux->tfull[buf], (c >> 1) & 1);
                    else mbar_wait(&aux->tfull[buf], (c >> 1) & 1);
                    tc_fence_after();
                }
                if (trc && tid == 0) trace_mark(trc, 6);
                // up to 64 columns per TMEM round trip: 4 tcgen05.ld in flight, one wait (one load + wait
                // per 16 columns made the epilogue of a 128 x 256 tile ~4k cycles of TMEM latency, r02k)
                constexpr int CH = HALF < 64 ? HALF : 64;
#pragma unroll 1
                for (int c0 = 0; c0 < HALF; c0 += CH) {
                    uint32_t v[CH];
                    if (nch > 0) {
#pragma unroll
                        for (int q = 0; q < CH / 16; ++q)
                            tmem_ld_32x32b_x16(tmem + lane_addr + (uint32_t)(buf * BN + half * HALF + c0 + 16 * q),
                                               *reinterpret_cast<uint32_t(*)[16]>(&v[16 * q]));
                        tmem_ld_wait();
                        if (c0 + CH >= HALF) {  // last TMEM read of this tile: release the buffer before the stores
                            tc_fence_before();
                            mbar_arrive(&aux->tempty[buf]);
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < CH; ++e) v[e] = 0u;
                    }
                    if constexpr (C::EPW > 0) {
                        if (coal) {
#pragma unroll
                            for (int q = 0; q < CH / 16; ++q) {
                                const int col0 = n0 + half * HALF + c0 + 16 * q;
                                if (p.epi.mode != EPI_NONE) {
                                    float f[16];
#pragma unroll
                                    for (int e = 0; e < 16; ++e) f[e] = __uint_as_float(v[16 * q + e]);
                                    epi_apply16(p.epi, f, obase >= 0 && col0 < p.Ngemm ? out_off(col0) : -1, col0,
                                                p.Ngemm, egrp, lane);
#pragma unroll
                                    for (int e = 0; e < 16; ++e) v[16 * q + e] = __float_as_uint(f[e]);
                                }
                            }
#pragma unroll
                            for (int p0 = 0; p0 < CH; p0 += C::EPW) {
                                float f[C::EPW];
#pragma unroll
                                for (int e = 0; e < C::EPW; ++e) f[e] = __uint_as_float(v[p0 + e]);
                                const int col0 = n0 + half * HALF + c0 + p0;
                                if (tp.tstore)
                                    warp_rows_tstore<C::EPW>(stg, f, &tp.mapY, ts_c(col0), ts_p(col0), ts_n0, ts_ok, lane);
                                else
                                    warp_rows_store<C::EPW>(stg, f, obase, outp, col0, p.Ngemm, s2shift(col0), lane, tp.zf1,
                                                            tp.zf2);
                            }
                            continue;
                        }
                    }
#pragma unroll
                    for (int q = 0; q < CH / 16; ++q) {
                        const int col0 = n0 + half * HALF + c0 + 16 * q;
                        if (C::EPW == 0 && !C::IS_DW && p.epi.mode != EPI_NONE) {
                            float f[16];
#pragma unroll
                            for (int e = 0; e < 16; ++e) f[e] = __uint_as_float(v[16 * q + e]);
                            epi_apply16(p.epi, f, obase >= 0 && col0 < p.Ngemm ? out_off(col0) : -1, col0, p.Ngemm,
                                        egrp, lane);
#pragma unroll
                            for (int e = 0; e < 16; ++e) v[16 * q + e] = __float_as_uint(f[e]);
                        }
                        if (obase >= 0) {
#pragma unroll
                            for (int e = 0; e < 16; e += 4) {
                                const int col = col0 + e;
                                if (col < p.Ngemm)
                                    st4(col, __uint_as_float(v[16 * q + e]), __uint_as_float(v[16 * q + e + 1]),
                                        __uint_as_float(v[16 * q + e + 2]), __uint_as_float(v[16 * q + e + 3]));
                            }
                        }
                    }
                }
                if (nch > 0) ++c;
            }
        }
    }

    if (warp < C::NEPI && lane == 0 && tp.tstore) bulk_wait_group0();  // the epilogue's TMA stores are done
    if (trc && tid == 0) trace_mark(trc, 7);
    tc_fence_before();
    __syncthreads();
    if (tid == 0) trace_mark(trc, 8);
    if (CSK_OK && tp.csk) {
        pdl_wait();  // every thread stores in the reduction (a no-op once satisfied)
        // cluster split-K: every CTA of the cluster holds its partial of the same tile in shared memory
        // [128 rows][PSTRIDE]; CTA r sums rows [r*128/S, (r+1)*128/S) over the S partials (csk_reduce)
        cluster_sync_all();  // release / acquire at cluster scope: all partials visible
        if (tid == 0) trace_mark(trc, 9);
        switch (tp.csk) {
            case 2: csk_reduce<OP, BN, C::PSTRIDE, 2>(tp, p, tiles_addr, (int)csk_rank, tid, C::NTHREADS); break;
            case 4: csk_reduce<OP, BN, C::PSTRIDE, 4>(tp, p, tiles_addr, (int)csk_rank, tid, C::NTHREADS); break;
            case 8: csk_reduce<OP, BN, C::PSTRIDE, 8>(tp, p, tiles_addr, (int)csk_rank, tid, C::NTHREADS); break;
            default: csk_reduce<OP, BN, C::PSTRIDE, 16>(tp, p, tiles_addr, (int)csk_rank, tid, C::NTHREADS); break;
        }
        if (tid == 0) trace_mark(trc, 10);
        cluster_sync_relaxed();  // no CTA exits while a peer still reads its shared memory
    }
    if (PAIR) cluster_sync_all();  // the peer's MMAs / arrivals are done before TMEM is released
    if (warp == C::MMA_W) {
        tc_fence_after();
        if (PAIR) tmem_dealloc2(tmem, C::TMEM_COLS);
        else tmem_dealloc(tmem, C::TMEM_COLS);
    }
    if (tid == 0) trace_mark(trc, 11);
}

// ------------------------------------------------------------------ host side
bool tma_supported(int op, int N, int IC, int OC, int FH, int FW, int sh, int sw);
int tma_epw(int op, int BN, int planes, int pair);  // TmaCfg::EPW of the kernel tma_launch would pick
int tma_make_plan(int op, GenParams& g, int& BN, int planes, TmaParams& tp, dim3& grid, char* err, size_t errlen);
int tma_launch(int op, int BN, int planes, const GenParams& g, TmaParams& tp, dim3 grid, cudaStream_t st, char* err,
               size_t errlen);

}  // namespace smconv
