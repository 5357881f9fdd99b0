// conv_gen.cuh — GENERIC variant: register-staged implicit GEMM on tcgen05 (sm_100a).
//
// One kernel template serves the three operators of the path:
//
//   op   GEMM rows (M)              GEMM cols (N)        reduction (K)              A major / B major
//   fwd  output pixels, position-   OC                    (valid tap, IC)            K / K
//        major (pos, n)  [A2]
//   dX   input pixels of one stride (IC)                  (valid tap of the phase,   K / MN
//        phase, position-major                            OC)
//   dW   OC                          (tap, IC)            pixels (pos, n)            MN / MN
//
// "Position-major" rows (m = pos * N + n) make a 128-row tile hold ONE output position
// across 128 images whenever N % 128 == 0 (the batch-folded tiles of north_star (c)):
// then every row of the tile has the same set of in-bounds taps and the K loop visits
// only those (the small-map "complexity reduction", reading L12).  For
// other N the tile takes the union of its rows' valid taps and zero-fills per row.
//
// Warp roles (288 threads): warps 0-7 load operands (16-B ld.global -> TF32 split ->
// st.shared into the 128-B-swizzled canonical UMMA layouts) through a STAGES-deep
// mbarrier ring and afterwards run the epilogue (tcgen05.ld -> st.global.v4); warp 8
// allocates TMEM and one of its lanes issues tcgen05.mma.kind::tf32 (M=128, N=BN, K=8).
//
// 3xTF32 (PLANES == 2): a = a_hi + a_lo with a_hi = rna_tf32(a), a_lo = rna_tf32(a - a_hi);
// per k-step the MMA thread issues a_lo*b_hi, a_hi*b_lo, a_hi*b_hi (smallest terms first)
// into one FP32 TMEM accumulator.  TF32 (PLANES == 1): one product of rna_tf32 operands.
#pragma once
#include "common.cuh"
#include "epilogue.cuh"

namespace smconv {

enum { OP_FWD = 0, OP_DX = 1, OP_DW = 2, OP_DWT = 3 };  // OP_DWT: dW with (tap,IC) rows, OC cols (TMA variant, OC <= 64)

constexpr int kMaxTaps = 256;
constexpr int kMaxTF = 16;  // TMA variant: filter rows / columns covered by the per-phase tap tables
constexpr int kMaxPhases = 16;

struct GenParams {
    const float* A;  // fwd: X   dx: dY   dw: dY
    const float* B;  // fwd: W   dx: W    dw: X
    float* out;      // output tensor, or split-K workspace (slice s at out + s * split_stride)
    const void* Bx;  // 3xTF32 fwd / dX on TMA / STRIP: bf16 W' plane in the workspace (wx_prep_kernel)
    const float* Bt;  // 3xTF32 dX on TMA (TmaParams::dx_bk): fp32 Wt[IC][T][OC] in the workspace (wx_prep_kernel)
    long long split_stride;
    int N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw, OH, OW;
    int M;       // fwd: N*OH*OW; dw: OC (dx: per phase, see phase table)
    int Ngemm;   // fwd: OC; dx: IC; dw: FH*FW*IC
    int P;       // dw: N*OH*OW (reduction length)
    int splits;
    int kb_per_split;  // dw only
    int dwt;           // dw on the TMA variant with (tap,IC) rows x OC cols (OC <= 64): M = T*IC, Ngemm = OC
    FastDiv fd_N, fd_OW, fd_IC, fd_OC, fd_FW;
    // dx stride phases (rh, rw): rows ih = rh + sh*i', i' < IHp
    int nphase;
    int phase_tile0[kMaxPhases + 1];
    int phase_rh[kMaxPhases], phase_rw[kMaxPhases], phase_IHp[kMaxPhases], phase_IWp[kMaxPhases];
    FastDiv phase_fd_IWp[kMaxPhases];
    // TMA variant (fwd: phase 0; dx: per stride phase): the filter rows (d = 0) / columns (d = 1)
    // that can reach the phase, in increasing order, and their source offsets (source row =
    // tile row origin + tf_off).  Host-built, so a tile's tap list and k-block count need no
    // modulo / division per tap (that per-tile bookkeeping, run by every warp role, cost more
    // issue slots than the 3xTF32 split itself on the short-K stride-2 dX tiles).
    int8_t tf_n[kMaxPhases][2];
    int8_t tf_f[kMaxPhases][2][kMaxTF];
    int16_t tf_off[kMaxPhases][2][kMaxTF];
    // super-pixel stride-2 dX run as a fwd conv (smconv.cu "s2dx"): output row (n, i', j') and
    // column (pi, pj, ic) go to dX[n, 2i'-2+pi, 2j'-2+pj, ic] (rows / columns i' = 0 / j' = 0 dropped)
    int s2dx, s2_IH, s2_IW, s2_IC;
    // TMA fwd / dX in 3xTF32: 1 = hybrid (a_hi*b_hi TF32 + the cross terms as one K-doubled bf16 MMA on
    // the precomputed W' plane), 0 = three TF32 MMAs with b_lo split by the converter warps (no W' plane,
    // no wx_prep kernel: the small-map calls, where that launch cost more than the third MMA)
    int hyb;
    // s2dx: taps (a, b) of the 2x2 filter W2 (bit 2a+b) with a non-zero block in n-tile t's columns;
    // the others are skipped (phase (0,0) has 1 of the 4 taps, (0,1) / (1,0) 2, (1,1) 4)
    uint8_t s2_tapmask[16];
    // TMA fwd / dX: split-K inside a thread-block cluster of csk CTAs (0 = off): the partial tiles are
    // summed through distributed shared memory instead of an HBM workspace + reduce kernel
    int csk;
    // fused epilogue (epilogue.cuh): mode EPI_NONE unless the TMA / STRIP kernel
    // itself applies the transform and writes the statistics partial rows
    EpiArgs epi;
    // TMA dW with IC % 32 != 0: the GEMM columns are (tap, ic) with ic padded to dw_icp = roundup(IC, 32)
    // (a 32-column block never straddles a tap); the epilogue drops ic >= IC and stores at tap * IC + ic
    int dw_icp;
    FastDiv fd_icp;
    // fused dW all-reduce (smconv_mcast.h): the TMA dW epilogue adds its tile into this multicast address
    // (multimem.red) instead of storing it; NULL otherwise
    float* mc_out;
    // TEST/EXPERIMENT hook (smconv_set_trace): per-CTA phase timestamps, NULL in normal operation
    unsigned long long* trace;
};

// trace slot e of this CTA: clock64 (SM cycles; slot 15 = globaltimer at entry, ns)
SMCONV_DEV void trace_mark(unsigned long long* t, int e) {
    if (t) {
        unsigned long long c;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
        t[blockIdx.x * 16 + e] = c;
    }
}

template <int OP, int BN, int PLANES>
struct GenCfg {
    static constexpr int BM = 128, BK = 32;
    static constexpr int NLW = 8, NLT = NLW * 32, NTHREADS = NLT + 32;
    static constexpr int A_BYTES = BM * BK * 4;
    static constexpr int B_BYTES = BN * BK * 4;
    static constexpr int STAGE_BYTES = PLANES * (A_BYTES + B_BYTES);
    static constexpr int STAGES_RAW = (200 * 1024) / STAGE_BYTES;
    static constexpr int STAGES = STAGES_RAW > 4 ? 4 : STAGES_RAW;
    static constexpr int A_CH = BM * 8 / NLT;  // 16-B chunks per loader thread per k-block
    static constexpr int B_CH = BN * 8 / NLT;
    static constexpr bool A_MN = (OP == OP_DW);
    static constexpr bool B_MN = (OP != OP_FWD);
    static constexpr int AUX_BYTES = 2048 + kMaxTaps * 16;
    static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + AUX_BYTES;
    static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
    static_assert(STAGES >= 2, "stage does not fit");
    static_assert(BN % 32 == 0 && BN <= 256, "BN");
};

struct GenAux {
    uint64_t full[8];
    uint64_t empty[8];
    uint64_t done;
    uint32_t tmem_base;
    int ntaps;
    int4 taps[kMaxTaps];  // {dh, dw, tapfull, 0}
};

// Row geometry shared by loaders and epilogue: the source pixel of A for tap (dh,dw) is
// (h0 + dh, w0 + dw) of image n; the output row index is orow.
struct RowInfo {
    int h0, w0, n, orow;
    bool ok;
};

template <int OP>
SMCONV_DEV RowInfo row_info(const GenParams& p, int phase, int m) {
    RowInfo r;
    if (OP == OP_FWD) {
        r.ok = m < p.M;
        const int pos = (int)fdiv((uint32_t)m, p.fd_N);
        r.n = m - pos * p.N;
        const int oh = (int)fdiv((uint32_t)pos, p.fd_OW);
        const int ow = pos - oh * p.OW;
        r.h0 = oh * p.sh - p.ph;
        r.w0 = ow * p.sw - p.pw;
        r.orow = r.n * p.OH * p.OW + pos;
    } else {  // OP_DX
        const int IHp = p.phase_IHp[phase], IWp = p.phase_IWp[phase];
        r.ok = m < IHp * IWp * p.N;
        const int pos = (int)fdiv((uint32_t)m, p.fd_N);
        r.n = m - pos * p.N;
        const int i1 = (int)fdiv((uint32_t)pos, p.phase_fd_IWp[phase]);
        const int j1 = pos - i1 * IWp;
        r.h0 = i1;
        r.w0 = j1;
        const int ih = p.phase_rh[phase] + p.sh * i1, iw = p.phase_rw[phase] + p.sw * j1;
        r.orow = (r.n * p.IH + ih) * p.IW + iw;
    }
    return r;
}

// Union over the tile's rows of the taps with an in-bounds source pixel (warp 0).
template <int OP>
SMCONV_DEV void build_tap_list(const GenParams& p, int phase, int m0, int mrows, GenAux* aux) {
    const int lane = threadIdx.x & 31;
    const int srcH = OP == OP_FWD ? p.IH : p.OH;
    const int srcW = OP == OP_FWD ? p.IW : p.OW;
    const int pos_lo = (int)fdiv((uint32_t)m0, p.fd_N);
    const int pos_hi = (int)fdiv((uint32_t)(m0 + mrows - 1), p.fd_N);
    int nt = 0;
    for (int fh = 0; fh < p.FH; ++fh) {
        for (int fw = 0; fw < p.FW; ++fw) {
            int dh, dw;
            if (OP == OP_FWD) {
                dh = fh;
                dw = fw;
            } else {
                const int th = p.phase_rh[phase] + p.ph - fh, tw = p.phase_rw[phase] + p.pw - fw;
                // tap belongs to the phase iff th, tw are multiples of the stride
                if (((th % p.sh) + p.sh) % p.sh != 0 || ((tw % p.sw) + p.sw) % p.sw != 0) continue;
                dh = th >= 0 ? th / p.sh : -((-th) / p.sh);
                dw = tw >= 0 ? tw / p.sw : -((-tw) / p.sw);
            }
            bool any = false;
            for (int pos = pos_lo + lane; pos <= pos_hi; pos += 32) {
                int h0, w0;
                if (OP == OP_FWD) {
                    const int oh = (int)fdiv((uint32_t)pos, p.fd_OW);
                    h0 = oh * p.sh - p.ph;
                    w0 = (pos - oh * p.OW) * p.sw - p.pw;
                } else {
                    const int i1 = (int)fdiv((uint32_t)pos, p.phase_fd_IWp[phase]);
                    h0 = i1;
                    w0 = pos - i1 * p.phase_IWp[phase];
                }
                any |= ((unsigned)(h0 + dh) < (unsigned)srcH) && ((unsigned)(w0 + dw) < (unsigned)srcW);
            }
            if (__any_sync(0xffffffffu, any)) {
                if (lane == 0) aux->taps[nt] = make_int4(dh, dw, fh * p.FW + fw, 0);
                ++nt;
            }
        }
    }
    if (lane == 0) aux->ntaps = nt;
}

template <int PLANES>
SMCONV_DEV void store_chunk(uint32_t hi_addr, uint32_t lo_addr, float4 v) {
    if (PLANES == 2) {
        const float h0 = tf32_rna(v.x), h1 = tf32_rna(v.y), h2 = tf32_rna(v.z), h3 = tf32_rna(v.w);
        st_shared_v4(hi_addr, h0, h1, h2, h3);
        st_shared_v4(lo_addr, tf32_rna(v.x - h0), tf32_rna(v.y - h1), tf32_rna(v.z - h2), tf32_rna(v.w - h3));
    } else {
        st_shared_v4(hi_addr, tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
    }
}

template <int OP, int BN, int PLANES>
__global__ void __launch_bounds__(GenCfg<OP, BN, PLANES>::NTHREADS, 1)
    conv_gen_kernel(const __grid_constant__ GenParams p) {
    using C = GenCfg<OP, BN, PLANES>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    const uint32_t tiles_addr = (raw_addr + 1023u) & ~1023u;
    uint8_t* tiles_ptr = smem_raw + (tiles_addr - raw_addr);
    GenAux* aux = reinterpret_cast<GenAux*>(tiles_ptr + C::STAGES * C::STAGE_BYTES);

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;

    // ---------------- tile coordinates
    int phase = 0, mt = blockIdx.x;
    if (OP == OP_DX) {
        while (phase + 1 < p.nphase && mt >= p.phase_tile0[phase + 1]) ++phase;
        mt -= p.phase_tile0[phase];
    }
    const int m0 = mt * C::BM;
    const int n0 = blockIdx.y * BN;
    const int split = blockIdx.z;
    int Mrows;
    if (OP == OP_DX) Mrows = p.phase_IHp[phase] * p.phase_IWp[phase] * p.N;
    else Mrows = p.M;
    const int mrows = min(C::BM, Mrows - m0);

    // ---------------- setup
    if (tid == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&aux->full[s], C::NLT);
            mbar_init(&aux->empty[s], 1);
        }
        mbar_init(&aux->done, 1);
        fence_mbar_init();
    }
    if (OP != OP_DW && warp == 0) build_tap_list<OP>(p, phase, m0, mrows, aux);
    if (warp == C::NLW) tmem_alloc(&aux->tmem_base, C::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = aux->tmem_base;
    pdl_trigger();
    pdl_wait();  // launch.cuh

    // K extent of this tile / split
    int kb_begin, kb_end, Ktot;
    if (OP == OP_DW) {
        Ktot = p.P;
        const int nkb = (p.P + C::BK - 1) / C::BK;
        kb_begin = split * p.kb_per_split;
        kb_end = min(nkb, kb_begin + p.kb_per_split);
    } else {
        const int srcC = OP == OP_FWD ? p.IC : p.OC;
        Ktot = aux->ntaps * srcC;
        const int nkb = (Ktot + C::BK - 1) / C::BK;
        const int per = (nkb + p.splits - 1) / p.splits;
        kb_begin = split * per;
        kb_end = min(nkb, kb_begin + per);
    }
    const int nkb_local = max(0, kb_end - kb_begin);

    if (warp < C::NLW) {
        // ======================= loaders
        const int srcH = OP == OP_FWD ? p.IH : p.OH;
        const int srcW = OP == OP_FWD ? p.IW : p.OW;
        const int srcC = OP == OP_FWD ? p.IC : p.OC;
        const int T = p.FH * p.FW;
        // A rows (K-major ops): rows r_i = i*32 + tid/8, chunk c = tid % 8
        int a_h0[C::A_CH], a_w0[C::A_CH], a_nb[C::A_CH];
        const int cA = tid & 7;
        if (OP != OP_DW) {
#pragma unroll
            for (int i = 0; i < C::A_CH; ++i) {
                const int r = i * 32 + (tid >> 3);
                RowInfo ri = row_info<OP>(p, phase, m0 + r);
                a_h0[i] = ri.ok ? ri.h0 : -(1 << 20);
                a_w0[i] = ri.w0;
                a_nb[i] = ri.n * srcH * srcW * srcC;
            }
        }
        // dW per-thread fixed columns
        int dwB_fh = 0, dwB_fw = 0, dwB_ic = 0;
        bool dwB_ok = false;
        const int dwA_oc = n0 * 0 + m0 + 4 * (tid & 31);
        if (OP == OP_DW) {
            const int n = n0 + 4 * (tid % (BN / 4));
            dwB_ok = n < p.Ngemm;
            const int tap = (int)fdiv((uint32_t)n, p.fd_IC);
            dwB_ic = n - tap * p.IC;
            dwB_fh = (int)fdiv((uint32_t)tap, p.fd_FW);
            dwB_fw = tap - dwB_fh * p.FW;
        }

        for (int it = 0; it < nkb_local; ++it) {
            const int kb = kb_begin + it;
            const int s = it % C::STAGES;
            const int round = it / C::STAGES;
            float4 va[C::A_CH], vb[C::B_CH];
            const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
            if (OP != OP_DW) {
                // k -> (tap j, channel) for this thread's chunk (same c for A and, in fwd, B)
                const int k = kb * C::BK + cA * 4;
                const bool kok = k < Ktot;
                const int j = (int)fdiv((uint32_t)(kok ? k : 0), OP == OP_FWD ? p.fd_IC : p.fd_OC);
                const int ch = (kok ? k : 0) - j * srcC;
                const int4 tp = aux->taps[kok ? j : 0];
#pragma unroll
                for (int i = 0; i < C::A_CH; ++i) {
                    const int h = a_h0[i] + tp.x, w = a_w0[i] + tp.y;
                    const bool ok = kok && (unsigned)h < (unsigned)srcH && (unsigned)w < (unsigned)srcW;
                    va[i] = ok ? ldg_f4(p.A + a_nb[i] + (h * srcW + w) * srcC + ch) : z4;
                }
                if (OP == OP_FWD) {
#pragma unroll
                    for (int i = 0; i < C::B_CH; ++i) {
                        const int oc = n0 + i * 32 + (tid >> 3);
                        const bool ok = kok && oc < p.OC;
                        vb[i] = ok ? ldg_f4(p.B + (oc * T + tp.z) * p.IC + ch) : z4;
                    }
                } else {  // dx: B[n=ic][k=(j,oc)] MN-major
#pragma unroll
                    for (int i = 0; i < C::B_CH; ++i) {
                        const int q = i * C::NLT + tid;
                        const int mnc = q % (BN / 4), kr = q / (BN / 4);
                        const int kk = kb * C::BK + kr;
                        const bool kk_ok = kk < Ktot;
                        const int jj = (int)fdiv((uint32_t)(kk_ok ? kk : 0), p.fd_OC);
                        const int oc = (kk_ok ? kk : 0) - jj * p.OC;
                        const int ic = n0 + 4 * mnc;
                        const bool ok = kk_ok && ic < p.IC;
                        vb[i] = ok ? ldg_f4(p.B + (oc * T + aux->taps[jj].z) * p.IC + ic) : z4;
                    }
                }
            } else {
                // dW: A[m=oc][k=pixel] (MN-major), B[n=(tap,ic)][k=pixel] (MN-major)
#pragma unroll
                for (int i = 0; i < C::A_CH; ++i) {
                    const int kr = i * 8 + warp;
                    const int px = kb * C::BK + kr;
                    const bool ok = px < p.P && dwA_oc < p.OC;
                    const int pos = (int)fdiv((uint32_t)(ok ? px : 0), p.fd_N);
                    const int n = (ok ? px : 0) - pos * p.N;
                    va[i] = ok ? ldg_f4(p.A + (n * p.OH * p.OW + pos) * p.OC + dwA_oc) : z4;
                }
#pragma unroll
                for (int i = 0; i < C::B_CH; ++i) {
                    const int q = i * C::NLT + tid;
                    const int kr = q / (BN / 4);
                    const int px = kb * C::BK + kr;
                    bool ok = dwB_ok && px < p.P;
                    const int pos = (int)fdiv((uint32_t)(ok ? px : 0), p.fd_N);
                    const int n = (ok ? px : 0) - pos * p.N;
                    const int oh = (int)fdiv((uint32_t)pos, p.fd_OW);
                    const int ow = pos - oh * p.OW;
                    const int ih = oh * p.sh - p.ph + dwB_fh, iw = ow * p.sw - p.pw + dwB_fw;
                    ok = ok && (unsigned)ih < (unsigned)p.IH && (unsigned)iw < (unsigned)p.IW;
                    vb[i] = ok ? ldg_f4(p.B + ((n * p.IH + ih) * p.IW + iw) * p.IC + dwB_ic) : z4;
                }
            }

            if (round > 0) mbar_wait(&aux->empty[s], (round - 1) & 1);
            const uint32_t st = tiles_addr + s * C::STAGE_BYTES;
            const uint32_t aH = st, aL = st + C::A_BYTES;
            const uint32_t bH = st + PLANES * C::A_BYTES, bL = bH + C::B_BYTES;
#pragma unroll
            for (int i = 0; i < C::A_CH; ++i) {
                uint32_t off;
                if (C::A_MN) off = mnmaj_off(i * 8 + warp, 4 * (tid & 31));
                else off = kmaj_off(i * 32 + (tid >> 3), cA);
                store_chunk<PLANES>(aH + off, aL + off, va[i]);
            }
#pragma unroll
            for (int i = 0; i < C::B_CH; ++i) {
                uint32_t off;
                if (C::B_MN) {
                    const int q = i * C::NLT + tid;
                    off = mnmaj_off(q / (BN / 4), 4 * (q % (BN / 4)));
                } else {
                    off = kmaj_off(i * 32 + (tid >> 3), cA);
                }
                store_chunk<PLANES>(bH + off, bL + off, vb[i]);
            }
            fence_proxy_async_smem();
            mbar_arrive(&aux->full[s]);
        }

        // ======================= epilogue (warps 0-7)
        mbar_wait(&aux->done, 0);
        tc_fence_after();
        const int q = warp & 3, half = warp >> 2;
        const int row = q * 32 + lane;
        float* outp = p.out + (long long)split * p.split_stride;
        long long obase = -1;
        if (OP == OP_DW) {
            const int oc = m0 + row;
            if (oc < p.OC) obase = (long long)oc * p.Ngemm;
        } else {
            RowInfo ri = row_info<OP>(p, phase, m0 + row);
            if (ri.ok) obase = (long long)ri.orow * p.Ngemm;
        }
        constexpr int HALF = BN / 2;
#pragma unroll 1
        for (int c0 = half * HALF; c0 < half * HALF + HALF; c0 += 16) {
            uint32_t v[16];
            if (nkb_local > 0) {
                tmem_ld_32x32b_x16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, v);
                tmem_ld_wait();
            } else {
#pragma unroll
                for (int e = 0; e < 16; ++e) v[e] = 0u;
            }
            if (obase >= 0) {
#pragma unroll
                for (int e = 0; e < 16; e += 4) {
                    const int col = n0 + c0 + e;
                    if (col < p.Ngemm) {
                        float4 o = make_float4(__uint_as_float(v[e]), __uint_as_float(v[e + 1]),
                                               __uint_as_float(v[e + 2]), __uint_as_float(v[e + 3]));
                        *reinterpret_cast<float4*>(outp + obase + col) = o;
                    }
                }
            }
        }
    } else if (warp == C::NLW) {
        // ======================= MMA issuer (whole warp runs the loop, one elected lane issues)
        constexpr uint32_t IDESC = idesc_tf32(128, BN, C::A_MN, C::B_MN);
        // K-major: SWIZZLE_128B, SBO 1024;  MN-major: SWIZZLE_128B_BASE32B, LBO 4096, SBO 512
        const uint64_t adH0 = make_sdesc(tiles_addr, C::A_MN ? 4096u : 16u, C::A_MN ? 512u : 1024u,
                                         C::A_MN ? kLayoutSW128Base32 : kLayoutSW128);
        const uint64_t bdH0 = make_sdesc(tiles_addr + PLANES * C::A_BYTES, C::B_MN ? 4096u : 16u,
                                         C::B_MN ? 512u : 1024u, C::B_MN ? kLayoutSW128Base32 : kLayoutSW128);
        constexpr uint64_t A_LO = C::A_BYTES >> 4, B_LO = C::B_BYTES >> 4;
        constexpr uint64_t A_G = C::A_MN ? 64 : 2, B_G = C::B_MN ? 64 : 2;
        for (int it = 0; it < nkb_local; ++it) {
            const int s = it % C::STAGES;
            const int round = it / C::STAGES;
            mbar_wait(&aux->full[s], round & 1);
            tc_fence_after();
            const uint64_t so = (uint64_t)(s * C::STAGE_BYTES) >> 4;
            if (elect_one()) {
#pragma unroll
                for (int g = 0; g < C::BK / 8; ++g) {
                    const uint64_t adH = adH0 + so + g * A_G, bdH = bdH0 + so + g * B_G;
                    const uint32_t acc0 = (it > 0 || g > 0) ? 1u : 0u;
                    if (PLANES == 2) {
                        mma_tf32_ss(tmem, adH + A_LO, bdH, IDESC, acc0);
                        mma_tf32_ss(tmem, adH, bdH + B_LO, IDESC, 1u);
                        mma_tf32_ss(tmem, adH, bdH, IDESC, 1u);
                    } else {
                        mma_tf32_ss(tmem, adH, bdH, IDESC, acc0);
                    }
                }
                mma_commit(&aux->empty[s]);
            }
            __syncwarp();
        }
        if (elect_one()) mma_commit(&aux->done);
        __syncwarp();
    }

    tc_fence_before();
    __syncthreads();
    if (warp == C::NLW) {
        tc_fence_after();
        tmem_dealloc(tmem, C::TMEM_COLS);
    }
}

// dX positions of stride phases that no filter tap reaches (reading L5: written as 0), e.g. three
// of the four phases of a 1x1 stride-2 shortcut: a streaming zero fill instead of MMA tiles.
template <int UNUSED = 0>
__global__ void __launch_bounds__(256) zero_phases_kernel(float4* __restrict__ dx, long long rows, int IC4, int IH, int IW,
                                                          int sh, int sw, uint32_t empty_mask) {
    pdl_trigger();
    pdl_wait();
    // one (n, ih) row per block iteration, 32-bit index math (a 64-bit division per element made
    // this kernel 3x slower than the HBM write it does); rows whose phases are all empty are a
    // contiguous memset
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    const int per_row = IW * IC4;
    const uint32_t all = (1u << sw) - 1u;
    for (long long row = blockIdx.x; row < rows; row += gridDim.x) {
        const int ih = (int)(row % IH);
        const uint32_t rmask = (empty_mask >> ((ih % sh) * sw)) & all;
        if (!rmask) continue;
        float4* base = dx + row * per_row;
        if (rmask == all) {
            for (int i = threadIdx.x; i < per_row; i += blockDim.x) base[i] = z;
        } else {
            for (int i = threadIdx.x; i < per_row; i += blockDim.x)
                if ((rmask >> ((i / IC4) % sw)) & 1u) base[i] = z;
        }
    }
}

// Deterministic split-K reduction: out[i] = sum_{s=0..S-1} ws[s*stride + i] in fixed order.
// mc != NULL (smconv_mcast.h): the fixed-order sum is added into the multicast address (multimem.red:
// every rank's copy receives it) instead of being stored to out.
template <int UNUSED = 0>
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float4* __restrict__ ws, float4* __restrict__ out,
                                                            long long n4, int splits, long long stride4,
                                                            float* mc = nullptr) {
    pdl_trigger();
    pdl_wait();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
        // fixed summation order s = 0, 1, ..., splits-1 (deterministic); loads are batched 8 deep so
        // a thread keeps 8 independent requests in flight (one at a time: 137 us for l1 dW's 512 splits)
        float4 a = ws[i];
        int s = 1;
        for (; s + 8 <= splits; s += 8) {
            float4 b[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) b[u] = ws[(long long)(s + u) * stride4 + i];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                a.x += b[u].x;
                a.y += b[u].y;
                a.z += b[u].z;
                a.w += b[u].w;
            }
        }
        for (; s < splits; ++s) {
            const float4 b = ws[(long long)s * stride4 + i];
            a.x += b.x;
            a.y += b.y;
            a.z += b.z;
            a.w += b.w;
        }
        if (mc) mc_red_add_f4(mc + 4 * i, a);
        else out[i] = a;
    }
}

// The same fixed-order sum for MANY partials of a SMALL output (stem / 1x1 dW: 74..148 splits of a few
// KB): one warp per float4 of the output, lane l sums the splits l, l+32, l+64, ... in that order, then
// a fixed xor-shuffle tree combines the 32 lane sums -- the same order on every run (deterministic).
// With one thread per float4 the 147 partials of the stem dW were 147 dependent-latency loads for only
// 576 threads: 24.5 us for 1.35 MB (ncu launch list, r02aa); this form keeps ~5 loads per lane.
template <int DUMMY>
__global__ void __launch_bounds__(256) splitk_reduce_wide_kernel(const float4* __restrict__ ws,
                                                                 float4* __restrict__ out, long long n4,
                                                                 int splits, long long stride4, float* mc = nullptr) {
    pdl_trigger();
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long i = w0; i < n4; i += nw) {
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        int s = lane;
        for (; s + 96 < splits; s += 128) {  // 4 loads in flight per lane
            float4 b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) b[u] = ws[(long long)(s + 32 * u) * stride4 + i];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                a.x += b[u].x;
                a.y += b[u].y;
                a.z += b[u].z;
                a.w += b[u].w;
            }
        }
        for (; s < splits; s += 32) {
            const float4 b = ws[(long long)s * stride4 + i];
            a.x += b.x;
            a.y += b.y;
            a.z += b.z;
            a.w += b.w;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a.x += __shfl_xor_sync(0xffffffffu, a.x, o);
            a.y += __shfl_xor_sync(0xffffffffu, a.y, o);
            a.z += __shfl_xor_sync(0xffffffffu, a.z, o);
            a.w += __shfl_xor_sync(0xffffffffu, a.w, o);
        }
        if (lane == 0) {
            if (mc) mc_red_add_f4(mc + 4 * i, a);
            else out[i] = a;
        }
    }
}

}  // namespace smconv
