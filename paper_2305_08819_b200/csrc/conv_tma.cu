// conv_tma.cu — host side of the TMA variant: eligibility, tensor-map encoding, launch.
#include <atomic>
#include <cstdlib>
#include <cstdio>
#include <cstring>

#include "../../include/smconv.h"
#include <cudaTypedefs.h>

#include "conv_tma.cuh"
#include "launch.cuh"

namespace smconv {

namespace {

// Tuning knobs (read once; for experiments only): SMCONV_TMA_G (32|128 images per A box),
// SMCONV_TMA_L2PROMO (0..3 = NONE/64B/128B/256B), SMCONV_TMA_CHUNK (promotion interval, k-blocks).
int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}
const int g_knob_G = env_int("SMCONV_TMA_G", 0);
const int g_knob_promo = env_int("SMCONV_TMA_L2PROMO", 3);
const int g_knob_chunk = env_int("SMCONV_TMA_CHUNK", 8);
// SMCONV_COALESCE=0: fwd / dX epilogue stores straight from the TMEM lanes (A/B experiments)
const int g_knob_coalesce = env_int("SMCONV_COALESCE", 1);
// 3xTF32 converter warps in two groups on alternate k-blocks (TmaParams::alt_conv; SMCONV_TMA_ALT=0: all 8 warps
// on every k-block).  r02cc: isolated l2-l4 dX -5..7 %, dW -2..7 %; ResNet-18 b4096 step -1.0 ms (three pairs)
const int g_knob_alt_conv = env_int("SMCONV_TMA_ALT", 1);
// SMCONV_TSTORE=0: the row-coalesced fwd / dX epilogue stores per thread instead of by TMA (A/B)
const int g_knob_tstore = env_int("SMCONV_TSTORE", 1);
const int g_knob_tstore_s2 = env_int("SMCONV_TSTORE_S2DX", 1);  // ... for the super-pixel dX too
// 3xTF32 TMA dW with bf16 cross terms (TmaCfg::HYBW; SMCONV_DW_HYB=0: three TF32 MMAs).  Measured
// r02bl: isolated l2-l4 dW -4..7 %, ResNet-18 b4096 step 54.5 -> 53.6 ms in three same-box A/B pairs
// (the step is power-capped: 2 instead of 3 MMA-equivalents per product is less energy per step)
const int g_knob_dw_hyb = env_int("SMCONV_DW_HYB", 1);
std::atomic<int> g_pair{env_int("SMCONV_PAIR", 1)};  // CTA pairs (smconv_set_pair); on by default since r01o
const int g_dw_pair = env_int("SMCONV_DW_PAIR", 1);  // dW pairs (A/B knob; follows g_pair when on)

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::atomic<int> g_encode_state{0};

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
    if (g_encode_state.load() == 0) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess && fn) {
            g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
            g_encode_state.store(1);
        } else {
            g_encode_state.store(2);
        }
    }
    return g_encode;
}

// Encode an fp32 tiled map. dims/strides/box in TMA order (dim 0 innermost, stride[0] = 4 implied).
bool encode(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
            const uint32_t* box, CUtensorMapSwizzle sw, CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32) {
    auto fn = encoder();
    if (!fn) return false;
    cuuint64_t gd[5], gs[4];
    cuuint32_t bd[5], es[5];
    for (int i = 0; i < rank; ++i) {
        gd[i] = dims[i];
        bd[i] = box[i];
        es[i] = 1;
    }
    for (int i = 0; i < rank - 1; ++i) gs[i] = strides_bytes[i];
    CUresult r = fn(m, dt, rank, const_cast<void*>(base), gd, gs, bd, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, sw, (CUtensorMapL2promotion)g_knob_promo,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int OP, int BN, int PLANES, bool PAIR>
int launch_t(const TmaParams& tp, const GenParams& g, dim3 grid, cudaStream_t st, char* err, size_t errlen) {
    using C = TmaCfg<OP, BN, PLANES, PAIR>;
    static std::atomic<unsigned long long> attr_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_done.load() & bit)) {
        if (cudaFuncSetAttribute(conv_tma_kernel<OP, BN, PLANES, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 C::SMEM_BYTES) != cudaSuccess) {
            snprintf(err, errlen, "cudaFuncSetAttribute(tma smem=%d): %s", C::SMEM_BYTES,
                     cudaGetErrorString(cudaGetLastError()));
            return CONV_ECUDA;
        }
        attr_done.fetch_or(bit);
    }
    if (PAIR || tp.csk) {  // 2-CTA clusters: one M = 256 tile per pair; csk-CTA clusters: split-K
        if (tp.csk && !C::CSK_FITS) {
            snprintf(err, errlen, "tma csk: partial tile does not fit the stage ring");
            return CONV_EUNSUPPORTED;
        }
        const cudaError_t e = launch_k(conv_tma_kernel<OP, BN, PLANES, PAIR>, grid, dim3(C::NTHREADS), C::SMEM_BYTES, st,
                                       PAIR ? 2 : tp.csk, tp, g);
        if (e != cudaSuccess) {
            snprintf(err, errlen, "cudaLaunchKernelEx(tma cluster %d): %s", PAIR ? 2 : tp.csk, cudaGetErrorString(e));
            return CONV_ECUDA;
        }
        return CONV_OK;
    }
    const cudaError_t e = launch_k(conv_tma_kernel<OP, BN, PLANES, PAIR>, grid, dim3(C::NTHREADS), C::SMEM_BYTES, st, 1,
                                   tp, g);
    if (e != cudaSuccess) {
        snprintf(err, errlen, "cudaLaunchKernelEx(tma): %s", cudaGetErrorString(e));
        return CONV_ECUDA;
    }
    return CONV_OK;
}

template <int OP, int PLANES>
int launch_bn(int BN, const TmaParams& tp, const GenParams& g, dim3 grid, cudaStream_t st, char* err, size_t n) {
    constexpr bool PAIRABLE = PLANES == 2 && (OP == OP_FWD || OP == OP_DX || OP == OP_DW);
    if (PAIRABLE && tp.pair) {
        if (BN == 64) return launch_t<OP, 64, PLANES, PAIRABLE>(tp, g, grid, st, err, n);
        return launch_t<OP, 128, PLANES, PAIRABLE>(tp, g, grid, st, err, n);
    }
    switch (BN) {
        case 32: return launch_t<OP, 32, PLANES, false>(tp, g, grid, st, err, n);
        case 64: return launch_t<OP, 64, PLANES, false>(tp, g, grid, st, err, n);
        case 128: return launch_t<OP, 128, PLANES, false>(tp, g, grid, st, err, n);
        default:
            if (PLANES == 2) return launch_t<OP, 128, PLANES, false>(tp, g, grid, st, err, n);  // unreachable (BN capped)
            return launch_t<OP, (PLANES == 2 ? 128 : 256), PLANES, false>(tp, g, grid, st, err, n);
    }
}

template <int OP, int PLANES>
int epw_bn(int BN, int pair) {
    constexpr bool PAIRABLE = PLANES == 2 && (OP == OP_FWD || OP == OP_DX || OP == OP_DW);
    if (PAIRABLE && pair) return BN == 64 ? TmaCfg<OP, 64, PLANES, PAIRABLE>::EPW : TmaCfg<OP, 128, PLANES, PAIRABLE>::EPW;
    switch (BN) {
        case 32: return TmaCfg<OP, 32, PLANES, false>::EPW;
        case 64: return TmaCfg<OP, 64, PLANES, false>::EPW;
        case 128: return TmaCfg<OP, 128, PLANES, false>::EPW;
        default: return TmaCfg<OP, (PLANES == 2 ? 128 : 256), PLANES, false>::EPW;
    }
}


template <int OP>
int launch_op(int BN, int planes, const TmaParams& tp, const GenParams& g, dim3 grid, cudaStream_t st, char* err,
              size_t n) {
    return planes == 2 ? launch_bn<OP, 2>(BN, tp, g, grid, st, err, n) : launch_bn<OP, 1>(BN, tp, g, grid, st, err, n);
}

}  // namespace

int tma_epw(int op, int BN, int planes, int pair) {
    if (op == CONV_OP_FWD) return planes == 2 ? epw_bn<OP_FWD, 2>(BN, pair) : epw_bn<OP_FWD, 1>(BN, pair);
    if (op == CONV_OP_BWD_DATA) return planes == 2 ? epw_bn<OP_DX, 2>(BN, pair) : epw_bn<OP_DX, 1>(BN, pair);
    return 0;
}

int tma_set_pair(int on) { return g_pair.exchange(on); }
int tma_get_pair() { return g_pair.load(); }

bool tma_encode_f32(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                    const uint32_t* box, CUtensorMapSwizzle sw) {
    return encode(m, base, rank, dims, strides, box, sw);
}

// the bf16 W' plane (wx_prep_kernel): rows (tap, n, cb) of 64 bf16, box (64, 1, BNC, 1) -> BNC
// K-major 128-B rows in shared memory, 128B swizzle (the UMMA SWIZZLE_128B K-major layout)
bool tma_encode_wx(CUtensorMap* m, const void* base, int Nn, int Kc, int T, int BNC) {
    const uint64_t CB = (Kc + 31) / 32;
    uint64_t d[4] = {64, CB, (uint64_t)Nn, (uint64_t)T}, s[3] = {128, CB * 128, (uint64_t)Nn * CB * 128};
    uint32_t b[4] = {64, 1, (uint32_t)BNC, 1};
    return encode(m, base, 4, d, s, b, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16);
}

bool tma_supported(int op, int N, int IC, int OC, int FH, int FW, int sh, int sw) {
    (void)sh; (void)sw;
    if (N % 32) return false;
    if (FH > kMaxTF || FW > kMaxTF) return false;  // per-phase tap tables (GenParams::tf_*)
    // the REDUCTION channels of fwd (IC) and dX (OC) need only the ABI's multiple of 4: their last
    // 32-channel block is completed by the TMA's out-of-bounds zero fill (A and B alike; the W' plane is
    // zero-padded by wx_prep_kernel).  The GEMM-column channels of dX (IC, an MN-major 32-channel view)
    // and both channel extents of dW still need multiples of 32.
    if (op == CONV_OP_FWD) return true;
    // ragged GEMM-column channels are padded to 32: below 16 channels (the RGB stems) that wastes >= 2x
    // of every MMA and B box, so those stay on the GENERIC / DIRECT variants
    if (op == CONV_OP_BWD_DATA) return IC % 32 == 0 || IC >= 16;  // IC % 32 != 0: TmaParams::dx_ragged
    return (IC % 32 == 0 || IC >= 16) && (OC % 32 == 0 || OC >= 16);  // dW: dw_a_ragged / dw_b_ragged, dw_icp
}

int tma_make_plan(int op, GenParams& g, int& BN, int planes, TmaParams& tp, dim3& grid, char* err, size_t errlen) {
    memset(&tp, 0, sizeof tp);
    // persistent: work items (m-tile, split, n-tile), one CTA per SM walks them round-robin
    tp.m_tiles = grid.x;
    tp.n_tiles = grid.y;
    tp.work = grid.x * grid.y * grid.z;
    grid = dim3(tp.work < 148 ? tp.work : 148, 1, 1);
    tp.G = (g.N % 128 == 0) ? 128 : 32;
    if (g_knob_G == 32) tp.G = 32;
    tp.chunk_kb = g_knob_chunk > 0 ? g_knob_chunk : 8;
    tp.coalesce = g_knob_coalesce;
    tp.alt_conv = planes == 2 ? g_knob_alt_conv : 0;
    tp.dw_hyb = (op == CONV_OP_BWD_FILTER && !g.dwt && planes == 2) ? g_knob_dw_hyb : 0;
    if (planes == 2 && BN > 128) {
        snprintf(err, errlen, "tma plan: BN %d > 128 in 3xTF32", BN);
        return CONV_EUNSUPPORTED;
    }
    if (op == CONV_OP_FWD) {
        tp.CB = (g.IC + 31) / 32;
    } else if (op == CONV_OP_BWD_DATA) {
        tp.CB = (g.OC + 31) / 32;
    }
    // CTA pairs (cta_group::2): fwd / dx in 3xTF32 when 256-row pair tiles (two 128-image blocks at
    // one position) tile every phase exactly; dW (not transposed) when OC is a multiple of 256
    const int pair_mode = g.csk ? 0 : g_pair.load();  // cluster split-K tiles are 1-CTA MMAs
    if (op == CONV_OP_BWD_FILTER && !g.dwt && planes == 2 && pair_mode && g_dw_pair && BN == 128 && g.OC % 256 == 0 &&
        tp.m_tiles % 2 == 0) {
        tp.pair = 1;
        tp.m_tiles /= 2;
        tp.work = tp.m_tiles * tp.n_tiles * g.splits;
        const int pairs = tp.work < 74 ? tp.work : 74;
        grid = dim3(2 * pairs, 1, 1);
    }
    if ((op == CONV_OP_FWD || op == CONV_OP_BWD_DATA) && planes == 2 && pair_mode && tp.G == 128 &&
        g.N % 256 == 0 && (BN == 64 || BN == 128) && tp.m_tiles % 2 == 0) {
        bool even = true;
        if (op == CONV_OP_BWD_DATA)
            for (int k = 0; k <= g.nphase; ++k) even &= g.phase_tile0[k] % 2 == 0;
        if (even) {
            tp.pair = 1;
            if (pair_mode == 2 && BN == 128) {  // experiment: N = 64 pair tiles (6 TMEM stages instead of 4)
                BN = 64;
                tp.n_tiles = (g.Ngemm + BN - 1) / BN;
            }
            if (op == CONV_OP_BWD_DATA)
                for (int k = 0; k <= g.nphase; ++k) g.phase_tile0[k] /= 2;
            tp.m_tiles /= 2;
            tp.work = tp.m_tiles * tp.n_tiles * g.splits;
            const int pairs = tp.work < 74 ? tp.work : 74;
            grid = dim3(2 * pairs, 1, 1);
        }
    }
    if (g.csk && !g.dwt) {
        // one work item per CTA; the csk splits of a tile form one cluster (TileInfo::init)
        tp.csk = g.csk;
        grid = dim3(tp.work, 1, 1);
    }
    // fast divisors for TileInfo::init (after every m_tiles / n_tiles / phase_tile0 adjustment above)
    tp.fd_ntiles = make_fastdiv(tp.n_tiles > 0 ? tp.n_tiles : 1);
    tp.fd_csk = make_fastdiv(tp.csk > 0 ? tp.csk : 1);
    tp.fd_splits = make_fastdiv(g.splits > 0 ? g.splits : 1);
    tp.fd_mtiles = make_fastdiv(tp.m_tiles > 0 ? tp.m_tiles : 1);
    tp.fd_CB = make_fastdiv(tp.CB > 0 ? tp.CB : 1);
    for (int k = 0; k < kMaxPhases; ++k) {
        int P = g.OH * g.OW;
        if (op == CONV_OP_BWD_DATA && k < g.nphase) P = g.phase_IHp[k] * g.phase_IWp[k];
        tp.fd_P[k] = make_fastdiv(P > 0 ? P : 1);
    }
    if (op == CONV_OP_FWD || op == CONV_OP_BWD_DATA) {
    } else {
        tp.NB32 = g.N / 32;
        // one X box per (tap, contiguous channel run): gcd(cols, IC) GEMM columns never cross a tap
        auto gcd = [](int a, int b) {
            while (b) {
                const int t = a % b;
                a = b;
                b = t;
            }
            return a;
        };
        if (g.dwt) {
            tp.a_box_cols = gcd(128, g.IC);
            tp.a_boxes = 128 / tp.a_box_cols;
        } else {
            const int bnc = tp.pair ? BN / 2 : BN;  // B columns staged per CTA
            const int cpt = g.dw_icp ? g.dw_icp : g.IC;  // GEMM columns per tap
            tp.b_box_cols = g.dw_icp ? 32 : gcd(bnc, g.IC);
            tp.b_boxes = bnc / tp.b_box_cols;
            if (cpt % BN == 0) tp.dw_tap_tiles = cpt / BN;  // n-tiles never straddle a tap
        }
    }
    tp.fd_dwtap = make_fastdiv(tp.dw_tap_tiles > 0 ? tp.dw_tap_tiles : 1);
    return CONV_OK;
}

int tma_launch(int op, int BN, int planes, const GenParams& g, TmaParams& tp, dim3 grid, cudaStream_t st, char* err,
               size_t errlen) {
    const uint64_t N = g.N, IH = g.IH, IW = g.IW, IC = g.IC, OC = g.OC, OH = g.OH, OW = g.OW;
    const uint64_t T = (uint64_t)g.FH * g.FW;
    bool ok = true;
    if (op == CONV_OP_FWD) {
        // A = X (IC, IW, IH, N); B = W (IC, T, OC)
        uint64_t da[4] = {IC, IW, IH, N}, sa[3] = {IC * 4, IW * IC * 4, IH * IW * IC * 4};
        uint32_t ba[4] = {32, 1, 1, (uint32_t)tp.G};
        ok &= encode(&tp.mapA, g.A, 4, da, sa, ba, CU_TENSOR_MAP_SWIZZLE_128B);
        uint64_t db[3] = {IC, T, OC}, sb[2] = {IC * 4, T * IC * 4};
        uint32_t bb[3] = {32, 1, (uint32_t)(tp.pair ? BN / 2 : BN)};  // a pair splits B by columns
        ok &= encode(&tp.mapB, g.B, 3, db, sb, bb, CU_TENSOR_MAP_SWIZZLE_128B);
        if (planes == 2 && g.hyb) ok &= g.Bx && tma_encode_wx(&tp.mapBx, g.Bx, (int)OC, (int)IC, (int)T, tp.pair ? BN / 2 : BN);
    } else if (op == CONV_OP_BWD_DATA) {
        // A = dY (OC, OW, OH, N); B = W viewed (32 ic, OC, IC/32, T), MN-major
        uint64_t da[4] = {OC, OW, OH, N}, sa[3] = {OC * 4, OW * OC * 4, OH * OW * OC * 4};
        uint32_t ba[4] = {32, 1, 1, (uint32_t)tp.G};
        ok &= encode(&tp.mapA, g.A, 4, da, sa, ba, CU_TENSOR_MAP_SWIZZLE_128B);
        if (tp.dx_bk) {  // Wt[IC][T][OC] (wx_prep_kernel, after the W' plane): like the fwd's W
            uint64_t db[3] = {OC, T, IC}, sb[2] = {OC * 4, T * OC * 4};
            uint32_t bb[3] = {32, 1, (uint32_t)(tp.pair ? BN / 2 : BN)};
            ok &= g.Bt && encode(&tp.mapB, g.Bt, 3, db, sb, bb, CU_TENSOR_MAP_SWIZZLE_128B);
        } else if (IC % 32 == 0) {
            uint64_t db[4] = {32, OC, IC / 32, T}, sb[3] = {T * IC * 4, 128, IC * 4};
            uint32_t bb[4] = {32, 32, (uint32_t)((tp.pair ? BN / 2 : BN) / 32), 1};
            ok &= encode(&tp.mapB, g.B, 4, db, sb, bb, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
        } else {  // ragged IC: W viewed (IC, OC, T), box (32 ic, 32 oc, 1) per 32-column block
            tp.dx_ragged = 1;
            uint64_t db[3] = {IC, OC, T}, sb[2] = {T * IC * 4, IC * 4};
            uint32_t bb[3] = {32, 32, 1};
            ok &= encode(&tp.mapB, g.B, 3, db, sb, bb, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
        }
        if (planes == 2 && g.hyb) ok &= g.Bx && tma_encode_wx(&tp.mapBx, g.Bx, (int)IC, (int)OC, (int)T, tp.pair ? BN / 2 : BN);
    } else if (g.dwt) {
        // transposed dW: A = X viewed (32 ic, N, IC/32, IW, IH), B = dY viewed (32 oc, N, OC/32, OH*OW)
        uint64_t da[5] = {32, N, IC / 32, IW, IH}, sa[4] = {IH * IW * IC * 4, 128, IC * 4, IW * IC * 4};
        uint32_t ba[5] = {32, 32, (uint32_t)(tp.a_box_cols / 32), 1, 1};
        ok &= encode(&tp.mapA, g.B, 5, da, sa, ba, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
        uint64_t db[4] = {32, N, OC / 32, OH * OW}, sb[3] = {OH * OW * OC * 4, 128, OC * 4};
        uint32_t bb[4] = {32, 32, (uint32_t)(BN / 32), 1};
        ok &= encode(&tp.mapB, g.A, 4, db, sb, bb, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    } else {
        // A = dY viewed (32 oc, N, OC/32, OH*OW), MN-major; B = X viewed (32 ic, N, IC/32, IW, IH), MN-major.
        // Ragged channel extents: views with the whole channel extent innermost, one 32-channel box at
        // a time (the TMA zero-fills channels past the extent)
        if (OC % 32 == 0) {
            uint64_t da[4] = {32, N, OC / 32, OH * OW}, sa[3] = {OH * OW * OC * 4, 128, OC * 4};
            uint32_t ba[4] = {32, 32, 4, 1};
            ok &= encode(&tp.mapA, g.A, 4, da, sa, ba, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
        } else {
            tp.dw_a_ragged = 1;
            uint64_t da[3] = {OC, N, OH * OW}, sa[2] = {OH * OW * OC * 4, OC * 4};
            uint32_t ba[3] = {32, 32, 1};
            ok &= encode(&tp.mapA, g.A, 3, da, sa, ba, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
        }
        if (IC % 32 == 0) {
            uint64_t db[5] = {32, N, IC / 32, IW, IH}, sb[4] = {IH * IW * IC * 4, 128, IC * 4, IW * IC * 4};
            uint32_t bb[5] = {32, 32, (uint32_t)(tp.b_box_cols / 32), 1, 1};
            ok &= encode(&tp.mapB, g.B, 5, db, sb, bb, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
        } else {
            tp.dw_b_ragged = 1;
            uint64_t db[4] = {IC, N, IW, IH}, sb[3] = {IH * IW * IC * 4, IC * 4, IW * IC * 4};
            uint32_t bb[4] = {32, 32, 1, 1};
            ok &= encode(&tp.mapB, g.B, 4, db, sb, bb, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
        }
    }
    // TMA-store epilogue (TmaParams::tstore): plain fwd / dX rows that go straight to the output tensor
    tp.tstore = 0;
    if ((op == CONV_OP_FWD || op == CONV_OP_BWD_DATA) && g_knob_tstore && tp.coalesce && !tp.csk &&
        (!g.s2dx || g_knob_tstore_s2) && !tp.zf1 && g.split_stride == 0 && !g.mc_out && g.N % 32 == 0) {
        const int epw = tma_epw(op, BN, planes, tp.pair);
        if (epw == 16 || epw == 32) {
            // s2dx: the super-pixel fwd conv's output is dX itself (IC, IH x IW pixels, N)
            const uint64_t C = g.s2dx ? (uint64_t)g.s2_IC : op == CONV_OP_FWD ? OC : IC;
            const uint64_t P = g.s2dx ? (uint64_t)g.s2_IH * g.s2_IW : op == CONV_OP_FWD ? OH * OW : IH * IW;
            uint64_t dy[3] = {C, P, N}, sy[2] = {C * 4, P * C * 4};
            uint32_t by[3] = {(uint32_t)epw, 1, 32};
            if (encode(&tp.mapY, g.out, 3, dy, sy, by,
                       epw == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B))
                tp.tstore = 1;
        }
    }
    if (!ok) {
        snprintf(err, errlen, "cuTensorMapEncodeTiled failed (op %d)", op);
        return CONV_ECUDA;
    }
    if (op == CONV_OP_FWD) return launch_op<OP_FWD>(BN, planes, tp, g, grid, st, err, errlen);
    if (op == CONV_OP_BWD_DATA) return launch_op<OP_DX>(BN, planes, tp, g, grid, st, err, errlen);
    if (g.dwt) return launch_op<OP_DWT>(BN, planes, tp, g, grid, st, err, errlen);
    return launch_op<OP_DW>(BN, planes, tp, g, grid, st, err, errlen);
}

}  // namespace smconv
