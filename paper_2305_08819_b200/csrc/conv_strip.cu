// conv_strip.cu — host side of the STRIP variant (conv_strip.cuh): eligibility, maps, launch.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cudaTypedefs.h>

#include "../../include/smconv.h"
#include "conv_strip.cuh"
#include "launch.cuh"

namespace smconv {

bool tma_encode_f32(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                    const uint32_t* box, CUtensorMapSwizzle sw);  // conv_tma.cu
bool tma_encode_wx(CUtensorMap* m, const void* base, int Nn, int Kc, int T, int BNC);  // conv_tma.cu
int tma_get_pair();                                                                      // conv_tma.cu

namespace {

const int g_knob_chunk_s = getenv("SMCONV_TMA_CHUNK") ? atoi(getenv("SMCONV_TMA_CHUNK")) : 8;
const int g_knob_coalesce_s = getenv("SMCONV_COALESCE") ? atoi(getenv("SMCONV_COALESCE")) : 1;
// SMCONV_STRIP_ALT=1: 3xTF32 converter warps in two groups on alternate stages (StripParams::alt_conv)
const int g_knob_alt_s = getenv("SMCONV_STRIP_ALT") ? atoi(getenv("SMCONV_STRIP_ALT")) : 0;

const int g_knob_tstore_s = getenv("SMCONV_TSTORE") ? atoi(getenv("SMCONV_TSTORE")) : 1;

template <int OP, int BN, int PLANES, int R, bool PAIR = false>
int launch_t(const StripParams& sp0, const GenParams& g, cudaStream_t st, char* err, size_t errlen) {
    using C = StripCfg<OP, BN, PLANES, R, PAIR>;
    StripParams sp = sp0;
    sp.tstore = 0;
    if (C::EPW > 0 && sp.coalesce && g_knob_tstore_s && g.split_stride == 0) {  // TMA-store epilogue (DESIGN 6d)
        const uint64_t Cc = OP == OP_FWD ? g.OC : g.IC, P = OP == OP_FWD ? (uint64_t)g.OH * g.OW : (uint64_t)g.IH * g.IW;
        uint64_t dy[3] = {Cc, P, (uint64_t)g.N}, sy[2] = {Cc * 4, P * Cc * 4};
        uint32_t by[3] = {(uint32_t)(C::EPW > 0 ? C::EPW : 16), 1, 32};
        if (tma_encode_f32(&sp.mapY, g.out, 3, dy, sy, by,
                           C::EPW == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B))
            sp.tstore = 1;
    }
    static std::atomic<unsigned long long> attr_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_done.load() & bit)) {
        if (cudaFuncSetAttribute(conv_strip_kernel<OP, BN, PLANES, R, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 C::SMEM_BYTES) != cudaSuccess) {
            snprintf(err, errlen, "cudaFuncSetAttribute(strip smem=%d): %s", C::SMEM_BYTES,
                     cudaGetErrorString(cudaGetLastError()));
            return CONV_ECUDA;
        }
        attr_done.fetch_or(bit);
    }
    if (PAIR) {  // 2-CTA clusters: one M = 256 tile (two 32-image strips) per pair
        const int pairs = sp.work < 74 ? sp.work : 74;
        const cudaError_t e = launch_k(conv_strip_kernel<OP, BN, PLANES, R, PAIR>, dim3(2 * pairs), dim3(C::NTHREADS),
                                       C::SMEM_BYTES, st, 2, sp, g);
        if (e != cudaSuccess) {
            snprintf(err, errlen, "cudaLaunchKernelEx(strip pair): %s", cudaGetErrorString(e));
            return CONV_ECUDA;
        }
        return CONV_OK;
    }
    const int grid = sp.work < 148 ? sp.work : 148;
    const cudaError_t e = launch_k(conv_strip_kernel<OP, BN, PLANES, R, PAIR>, dim3(grid), dim3(C::NTHREADS),
                                   C::SMEM_BYTES, st, 1, sp, g);
    if (e != cudaSuccess) {
        snprintf(err, errlen, "cudaLaunchKernelEx(strip): %s", cudaGetErrorString(e));
        return CONV_ECUDA;
    }
    return CONV_OK;
}

template <int OP>
int launch_op(int BN, int planes, const StripParams& sp, const GenParams& g, cudaStream_t st, char* err, size_t n) {
    if (planes == 2) {
        if (sp.pair) return launch_t<OP, 64, 2, 1, true>(sp, g, st, err, n);
        if (BN == 32) return launch_t<OP, 32, 2, 1>(sp, g, st, err, n);
        return launch_t<OP, 64, 2, 1>(sp, g, st, err, n);
    }
    if (BN == 32) return launch_t<OP, 32, 1, 4>(sp, g, st, err, n);
    if (BN == 64) return launch_t<OP, 64, 1, 2>(sp, g, st, err, n);
    return launch_t<OP, 128, 1, 1>(sp, g, st, err, n);
}

}  // namespace

int strip_R(int BN, int planes) {
    if (planes == 2) return 1;
    return BN == 32 ? 4 : BN == 64 ? 2 : 1;
}

// CTA-pair strips (conv_strip.cuh PAIR): 3xTF32, BN 64, an even number of 32-image groups;
// follows the TMA variant's pair switch (smconv_set_pair / SMCONV_PAIR)
bool strip_pair(int op, int N, int BN, int planes) {
    (void)op;
    return planes == 2 && BN == 64 && N % 64 == 0 && tma_get_pair() != 0;
}

bool strip_supported(int op, int N, int IC, int OC, int FW, int sh, int sw, int OWo, int BN, int planes) {
    if (op != CONV_OP_FWD && op != CONV_OP_BWD_DATA) return false;
    if (sh != 1 || sw != 1 || FW != kStripFW) return false;
    if (N % 32 || IC % 32 || OC % 32) return false;
    if (OWo < 4) return false;
    if (planes == 2) return BN <= 64;
    return BN <= 128;
}

int strip_launch(int op, int BN, int planes, const GenParams& g, cudaStream_t st, char* err, size_t errlen) {
    StripParams sp;
    memset(&sp, 0, sizeof sp);
    const int R = strip_R(BN, planes);
    const bool fwd = op == CONV_OP_FWD;
    const uint64_t N = g.N, T = (uint64_t)g.FH * g.FW;
    const uint64_t C = fwd ? g.IC : g.OC;                 // channels of the activation operand
    const uint64_t H = fwd ? g.IH : g.OH, W = fwd ? g.IW : g.OW;
    sp.coalesce = g_knob_coalesce_s;
    sp.alt_conv = planes == 2 ? g_knob_alt_s : 0;
    sp.CB = (int)(C / 32);
    sp.NG = g.N / 32;
    sp.OHo = fwd ? g.OH : g.IH;
    sp.OWo = fwd ? g.OW : g.IW;
    sp.SH = (int)H;
    sp.SW = (int)W;
    sp.strips = (sp.OWo + 4 * R - 1) / (4 * R);
    sp.n_tiles = (g.Ngemm + BN - 1) / BN;
    sp.fd_ntiles = make_fastdiv(sp.n_tiles);
    sp.fd_strips = make_fastdiv(sp.strips);
    sp.fd_OHo = make_fastdiv(sp.OHo);
    sp.pair = strip_pair(op, g.N, BN, planes) ? 1 : 0;
    sp.work = (sp.pair ? sp.NG / 2 : sp.NG) * sp.OHo * sp.strips * sp.n_tiles;
    const int BNC = sp.pair ? BN / 2 : BN;  // B columns staged per CTA
    sp.chunk_kb = g_knob_chunk_s > 0 ? g_knob_chunk_s : 8;
    sp.row_off = fwd ? -g.ph : g.ph;
    sp.col_off = fwd ? -g.pw : g.pw - (kStripFW - 1);
    const uint32_t slabs = 4 * R + kStripFW - 1;
    // A: activations viewed (32 ch, N, W, H, C/32) -> smem [slab][32 images][32 ch]
    uint64_t da[5] = {32, N, W, H, C / 32}, sa[4] = {H * W * C * 4, C * 4, W * C * 4, 128};
    uint32_t ba[5] = {32, 32, slabs, 1, 1};
    bool ok = tma_encode_f32(&sp.mapA, g.A, 5, da, sa, ba, CU_TENSOR_MAP_SWIZZLE_128B);
    if (fwd) {
        uint64_t db[3] = {(uint64_t)g.IC, (uint64_t)g.OC, T}, sb[2] = {T * g.IC * 4, (uint64_t)g.IC * 4};
        uint32_t bb[3] = {32, (uint32_t)BNC, (uint32_t)kStripFW};
        ok &= tma_encode_f32(&sp.mapB, g.B, 3, db, sb, bb, CU_TENSOR_MAP_SWIZZLE_128B);
    } else {
        uint64_t db[4] = {32, (uint64_t)g.OC, (uint64_t)g.IC / 32, T}, sb[3] = {T * g.IC * 4, 128, (uint64_t)g.IC * 4};
        uint32_t bb[4] = {32, 32, (uint32_t)(BNC / 32), (uint32_t)kStripFW};
        ok &= tma_encode_f32(&sp.mapB, g.B, 4, db, sb, bb, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    }
    if (planes == 2)
        ok &= g.Bx && tma_encode_wx(&sp.mapBx, g.Bx, fwd ? g.OC : g.IC, fwd ? g.IC : g.OC, (int)T, BNC);
    if (!ok) {
        snprintf(err, errlen, "strip: cuTensorMapEncodeTiled failed (op %d)", op);
        return CONV_ECUDA;
    }
    return fwd ? launch_op<OP_FWD>(BN, planes, sp, g, st, err, errlen)
               : launch_op<OP_DX>(BN, planes, sp, g, st, err, errlen);
}

}  // namespace smconv
