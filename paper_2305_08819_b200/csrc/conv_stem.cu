// conv_stem.cu — STEM variant: the few-channel input layers (RGB padded to IC = 4) on
// the tensor cores (tcgen05, TMEM accumulators), forward and weight gradient.
//
// The stem is HBM-bound (fwd: 16 B of X in, OC * 4 B of Y out per output pixel; K = 36), and its
// CUDA-core direct kernels (conv_direct.cu) ran at 0.15-0.22 of HBM (ResNet-18 b4096: fwd 0.80 ms,
// dW 1.16 ms for ~1.1 GB of compulsory traffic each, SURVEY §7 hard part 3).
// On CUDA cores the K = 36 products per output are FMA-bound at ~0.27 ms; as an MMA they are free.
//
// fwd, Y[m][oc] = sum_k Xcol[m][k] * W[oc][k], m = (n, oh, ow), k = (fh, fw, ic) (O1):
//  * tile = 128 consecutive output pixels (GEMM rows); the IM2COL row of pixel m (9 taps x one 16-B
//    pixel of X, zero outside the map) is gathered by the thread owning TMEM lane m % 128 and written
//    straight into TMEM (tcgen05.st): A = Xcol in TMEM (TS-form MMA), no shared-memory staging, no
//    swizzle; 3xTF32 also writes a_lo = a - trunc_tf32(a) next to it;
//  * B = W [OC][K] resident in shared memory for the whole kernel (K-major SWIZZLE_128B, K padded to
//    40 with zeros), w_lo likewise;
//  * 3xTF32: a*b ~ a_hi*b_hi + a_hi*b_lo + a_lo*b_hi, three TF32 MMAs per k-step (tcgen05 reads an
//    fp32 word by truncation, so the raw word IS the hi part); K = 36 needs no chunked
//    promotion (a 15-MMA chain);
//  * epilogue: TMEM -> registers -> a SWIZZLE_128B staging box per warp (conflict-free) -> TMA tensor
//    store (cp.async.bulk.tensor, 2-D view [M][OC] of Y, OOB rows of the last tile clipped): each
//    warp's 32 rows are 32 x OC x 4 contiguous bytes of Y.
// Persistent CTAs, warp-specialised: warps 0-3 epilogue, 4-11 two groups of IM2COL builders (even /
// odd tiles), 12 TMEM owner + MMA issuer; TMEM A slots and two accumulators are rings across tiles.
//
// dW, dW[oc][k] = sum_m dY[m][oc] * Xcol[m][k] (O3): GEMM rows = output channels (128 per m-tile),
// columns = k (36 -> 48), reduction over pixels in k-blocks of 32:
//  * A = dY^T: TMA boxes of dY viewed [M][OC] (32 oc x 32 px) land as the MN-major SWIZZLE_128B_BASE32B
//    tile the tensor core reads (SS-form MMA); 3xTF32 converter warps write the a_lo plane elementwise;
//  * B = Xcol^T [48][32 px] built in shared memory per k-block (thread = pixel, K-major SW128);
//  * each CTA walks a contiguous pixel range; the accumulator is promoted into fp32 registers every
//    8 k-blocks (the truncating TMEM adds) and the CTA's partial [OC][K] goes to the
//    workspace; splitk_reduce_kernel sums the partials in fixed order (deterministic).
#include <cuda.h>

#include <cstdio>
#include <cstring>

#include "../../include/smconv.h"
#include "common.cuh"
#include "conv_gen.cuh"
#include "launch.cuh"

namespace smconv {

bool tma_encode_f32(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                    const uint32_t* box, CUtensorMapSwizzle sw);

namespace {

constexpr int kTaps = 9;            // 3x3 filters
constexpr int kK = 4 * kTaps;       // 36 reduction elements (IC = 4)
constexpr int kKP = 40;             // padded to the TF32 MMA K-step of 8
constexpr int kSMs = 148;

struct __align__(64) StemParams {
    CUtensorMap mapY;  // fwd: Y viewed [M][OC], box (32 ch, 32 rows), SWIZZLE_128B
    const float* X;
    const float* W;
    const float* dY;
    float* out;        // dW: partials [gridDim.x][OC][kK]
    int N, IH, IW, OC, OH, OW, sh, sw, ph, pw;
    long long M;       // N * OH * OW
    int tiles;         // fwd: ceil(M / 128); dW: k-blocks of 32 pixels
    int kb_per_cta;    // dW
    int ts;            // dW 3xTF32: A (dY^T) in TMEM, TS-form MMAs (StemDwCfg::TS; SMCONV_STEM_TS=0: SS form)
    FastDiv fd_OW, fd_OHOW;
};

SMCONV_DEV void tma_store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(src), "r"(c0), "r"(c1)
                 : "memory");
}
SMCONV_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
SMCONV_DEV void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
SMCONV_DEV void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

SMCONV_DEV uint32_t lo_bits(float v) {
    return __float_as_uint(v - __uint_as_float(__float_as_uint(v) & 0xFFFFE000u));
}

SMCONV_DEV void tmem_st_x8(uint32_t taddr, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

// pixel m -> (n, oh, ow)
SMCONV_DEV void pix(const StemParams& p, long long m, int& n, int& oh, int& ow) {
    const uint32_t mm = (uint32_t)m;  // M < 2^31 (checked on the host)
    n = (int)fdiv(mm, p.fd_OHOW);
    const int r = (int)(mm - (uint32_t)n * (uint32_t)(p.OH * p.OW));
    oh = (int)fdiv((uint32_t)r, p.fd_OW);
    ow = r - oh * p.OW;
}

// the 9 taps x 4 channels of output pixel m (zeros outside the map / past M)
SMCONV_DEV void gather_row(const StemParams& p, long long m, float (&e)[kKP]) {
#pragma unroll
    for (int k = kK; k < kKP; ++k) e[k] = 0.f;
    if (m >= p.M) {
#pragma unroll
        for (int k = 0; k < kK; ++k) e[k] = 0.f;
        return;
    }
    int n, oh, ow;
    pix(p, m, n, oh, ow);
    const float4* X4 = reinterpret_cast<const float4*>(p.X);
    float4 v[kTaps];
#pragma unroll
    for (int t = 0; t < kTaps; ++t) {
        const int ih = oh * p.sh - p.ph + t / 3, iw = ow * p.sw - p.pw + t % 3;
        v[t] = ((unsigned)ih < (unsigned)p.IH && (unsigned)iw < (unsigned)p.IW)
                   ? __ldg(X4 + ((long long)(n * p.IH + ih) * p.IW + iw))
                   : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int t = 0; t < kTaps; ++t) {
        e[4 * t] = v[t].x;
        e[4 * t + 1] = v[t].y;
        e[4 * t + 2] = v[t].z;
        e[4 * t + 3] = v[t].w;
    }
}

template <int OCT, int PLANES>
struct StemFwdCfg {
    static constexpr int NEPI = 4, MMA_W = 12, NTHREADS = 13 * 32;  // builders: warps 4-11
    static constexpr int SLOT = PLANES * kKP;                          // TMEM columns per A slot
    // two accumulators when two A slots still fit beside them (OC 192 in 3xTF32: one accumulator)
    static constexpr int NACC = (512 - 2 * OCT) / SLOT >= 2 ? 2 : 1;
    static constexpr int NS_RAW = (512 - NACC * OCT) / SLOT;
    // A slots; >= 2 because the two builder groups alternate tiles: with one slot, the group of tile
    // i + 2 would wait on the slot barrier's phase of tile i + 1 while tile i's is still pending,
    // which a parity wait cannot tell apart (it hung, GoogLeNet stem r02y)
    static constexpr int NS = NS_RAW > 4 ? 4 : NS_RAW;
    static constexpr int NA = (kKP + 31) / 32;                        // SW128 atoms of 32 k
    static constexpr int B_PLANE = NA * OCT * 128;                    // bytes of one W plane
    static constexpr int NSTG = OCT <= 128 ? 2 : 1;                   // staging buffers per epilogue warp
    static constexpr int STG = OCT * 128;                             // 32 rows x OCT fp32 per warp
    // >= 120 KB: one CTA per SM (a second one would block in tcgen05.alloc of the 512 columns)
    static constexpr int SMEM_RAW = 1024 + PLANES * B_PLANE + NEPI * NSTG * STG + 256;
    static constexpr int SMEM = SMEM_RAW < 120 * 1024 ? 120 * 1024 : SMEM_RAW;
    static_assert(NS >= 2, "TMEM");
    static_assert(OCT % 32 == 0 && OCT <= 256, "OC tile");
};

struct StemAux {
    uint64_t afull[4], afree[4], accfull[2], accfree[2];
    uint32_t tmem_base;
};

template <int OCT, int PLANES>
__global__ void __launch_bounds__(StemFwdCfg<OCT, PLANES>::NTHREADS, 1)
    stem_fwd_kernel(const __grid_constant__ StemParams p) {
    using C = StemFwdCfg<OCT, PLANES>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* bptr = smem_raw + (base - raw);
    const uint32_t sB = base;                                   // W planes
    const uint32_t sStg = base + PLANES * C::B_PLANE;           // epilogue staging
    StemAux* aux = reinterpret_cast<StemAux*>(bptr + PLANES * C::B_PLANE + C::NEPI * C::NSTG * C::STG);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    if (tid == 0) {
        for (int s = 0; s < C::NS; ++s) {
            mbar_init(&aux->afull[s], 4);
            mbar_init(&aux->afree[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&aux->accfull[b], 1);
            mbar_init(&aux->accfree[b], C::NEPI);
        }
        fence_mbar_init();
    }
    if (warp == C::MMA_W) tmem_alloc(&aux->tmem_base, 512);
    if (warp == 0 && lane == 0)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.mapY)) : "memory");
    pdl_trigger();
    pdl_wait();
    // W -> shared memory (K-major SW128 atoms of 32 k; k >= 36 zero): raw words (= b_hi for the MMA)
    // and b_lo = b - trunc_tf32(b)
    for (int i = tid; i < OCT * C::NA * 8; i += C::NTHREADS) {
        const int oc = i / (C::NA * 8), ch = i % (C::NA * 8), a = ch >> 3, c = ch & 7;
        float w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int k = 32 * a + 4 * c + j;
            w[j] = (oc < p.OC && k < kK) ? __ldg(p.W + (long long)oc * kK + k) : 0.f;
        }
        const uint32_t off = (uint32_t)(a * OCT * 128) + kmaj_off((uint32_t)oc, (uint32_t)c);
        st_shared_v4(sB + off, w[0], w[1], w[2], w[3]);
        if (PLANES == 2)
            st_shared_v4(sB + C::B_PLANE + off, __uint_as_float(lo_bits(w[0])), __uint_as_float(lo_bits(w[1])),
                         __uint_as_float(lo_bits(w[2])), __uint_as_float(lo_bits(w[3])));
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = aux->tmem_base;
    const uint32_t A0 = C::NACC * OCT;  // TMEM column of A slot 0 (accumulators at [0, NACC * OCT))
    const int ntile = p.tiles > (int)blockIdx.x ? (p.tiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;

    if (warp == C::MMA_W) {
        constexpr uint32_t IDESC = idesc_tf32(128, OCT, false, false);
        const uint64_t bd0 = make_sdesc(sB, 16u, 1024u, kLayoutSW128);
        for (int i = 0; i < ntile; ++i) {
            const int s = i % C::NS, b = i % C::NACC;
            if (i >= C::NACC) {
                mbar_wait(&aux->accfree[b], ((i / C::NACC) - 1) & 1);
                tc_fence_after();
            }
            mbar_wait(&aux->afull[s], (i / C::NS) & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t d = tmem + (uint32_t)(b * OCT);
                const uint32_t a = tmem + A0 + (uint32_t)(s * C::SLOT);
#pragma unroll
                for (int j = 0; j < kKP / 8; ++j) {
                    const uint64_t bh = bd0 + (uint64_t)(((j >> 2) * OCT * 128 + (j & 3) * 32) >> 4);
                    mma_tf32_ts(d, a + 8 * j, bh, IDESC, j > 0 ? 1u : 0u);
                    if (PLANES == 2) {
                        mma_tf32_ts(d, a + 8 * j, bh + (uint64_t)(C::B_PLANE >> 4), IDESC, 1u);
                        mma_tf32_ts(d, a + kKP + 8 * j, bh, IDESC, 1u);
                    }
                }
                mma_commit(&aux->afree[s]);
                mma_commit(&aux->accfull[b]);
            }
            __syncwarp();
        }
    } else if (warp >= C::NEPI) {
        // IM2COL builders: group g takes this CTA's tiles i with i % 2 == g; warp quadrant q = warp % 4
        const int g = (warp - C::NEPI) >> 2, q = warp & 3;
        const uint32_t lanebase = (uint32_t)(q * 32) << 16;
        for (int i = g; i < ntile; i += 2) {
            const int s = i % C::NS;
            const long long m = ((long long)blockIdx.x + (long long)i * gridDim.x) * 128 + q * 32 + lane;
            float e[kKP];
            gather_row(p, m, e);  // loads issued before the slot wait: they overlap it
            if (i >= C::NS) {
                mbar_wait(&aux->afree[s], ((i / C::NS) - 1) & 1);
                tc_fence_after();
            }
            const uint32_t ta = tmem + lanebase + A0 + (uint32_t)(s * C::SLOT);
            uint32_t u[kKP];
#pragma unroll
            for (int k = 0; k < kKP; ++k) u[k] = __float_as_uint(e[k]);
#pragma unroll
            for (int j = 0; j < kKP / 8; ++j) tmem_st_x8(ta + 8 * j, u + 8 * j);
            if (PLANES == 2) {
#pragma unroll
                for (int k = 0; k < kKP; ++k) u[k] = lo_bits(e[k]);
#pragma unroll
                for (int j = 0; j < kKP / 8; ++j) tmem_st_x8(ta + kKP + 8 * j, u + 8 * j);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&aux->afull[s]);
        }
    } else {
        // epilogue warp q: rows 32q..32q+31 of each tile = 32 * OC * 4 contiguous bytes of Y
        const int q = warp;
        const uint32_t lanebase = (uint32_t)(q * 32) << 16;
        for (int i = 0; i < ntile; ++i) {
            const int b = i % C::NACC;
            const uint32_t stg = sStg + (uint32_t)((q * C::NSTG + (C::NSTG == 2 ? (i & 1) : 0)) * C::STG);
            if (lane == 0) bulk_wait_read<C::NSTG - 1>();  // the staging buffer's previous store has read it
            __syncwarp();
            mbar_wait(&aux->accfull[b], (i / C::NACC) & 1);
            tc_fence_after();
#pragma unroll 1
            for (int bx = 0; bx < OCT / 32; ++bx) {
                uint32_t v[32];
                tmem_ld_32x32b_x16(tmem + lanebase + (uint32_t)(b * OCT + 32 * bx), *reinterpret_cast<uint32_t(*)[16]>(v));
                tmem_ld_32x32b_x16(tmem + lanebase + (uint32_t)(b * OCT + 32 * bx + 16),
                                   *reinterpret_cast<uint32_t(*)[16]>(v + 16));
                tmem_ld_wait();
                // SWIZZLE_128B box [32 rows][32 ch]: chunk c of row r at r*128 + ((c ^ (r & 7)) << 4)
                const uint32_t rowa = stg + (uint32_t)(bx * 4096 + lane * 128);
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    st_shared_v4(rowa + (uint32_t)((c ^ (lane & 7)) << 4), __uint_as_float(v[4 * c]),
                                 __uint_as_float(v[4 * c + 1]), __uint_as_float(v[4 * c + 2]),
                                 __uint_as_float(v[4 * c + 3]));
            }
            tc_fence_before();
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&aux->accfree[b]);
                const long long row0 = ((long long)blockIdx.x + (long long)i * gridDim.x) * 128 + q * 32;
                for (int bx = 0; bx < OCT / 32; ++bx)
                    if (32 * bx < p.OC) tma_store_2d(&p.mapY, stg + (uint32_t)(bx * 4096), 32 * bx, (int)row0);
                bulk_commit();
            }
            __syncwarp();
        }
        if (lane == 0) bulk_wait_all();
        __syncwarp();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == C::MMA_W) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ------------------------------------------------------------------ dW
constexpr int kDwN = 48;  // GEMM columns (k = 36 padded to a multiple of 16)

SMCONV_DEV void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

template <int PLANES, int OCB>
struct StemDwCfg {
    static constexpr int TMA_W = 0, BLD_W0 = 1, NBLD = 4, CONV_W0 = 5, PRO_W0 = 9, MMA_W = 13;
    static constexpr int NTHREADS = 14 * 32;
    // A = [32 px][OCB x 32 oc] MN-major (OCB = 2 for OC <= 64: the M = 128 MMA's rows 64..127 then read
    // whatever follows in the stage -- rows nobody stores); the dY stream is latency-bound, so the
    // narrower stage buys ring depth (4 stages of 44 KB held ~3.6k cycles of look-ahead for ~1-2 us of
    // HBM latency: conv1 dW 2.7 TB/s, ncu r02aa)
    static constexpr int A_BYTES = OCB * 4096;
    static constexpr int B_BYTES = kDwN * 128;         // [48 k][32 px] K-major SW128
    static constexpr int STAGE = PLANES * (A_BYTES + B_BYTES);
    static constexpr int STAGES_RAW = (200 * 1024) / STAGE;
    static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
    static constexpr int CHUNK = 8;                    // promotion interval (k-blocks)
    static constexpr int PAD = (4 - OCB) * 4096;       // the last stage's junk-row reads stay inside the allocation
    static constexpr int SMEM = 1024 + STAGES * STAGE + PAD + 512;
    static_assert(STAGES >= NBLD, "builders own k-blocks mod 4: the ring must be at least that deep");
    // 3xTF32 (TS form): the converter warps write dY^T as a_hi | a_lo (32 + 32 columns per k-block) into
    // a TMEM slot ring, so the MMAs read only B from shared memory.  The SS form read the 128-row A tile
    // (half of it the junk rows of OC = 64) from shared memory for every one of the 12 MMAs per k-block:
    // ~100 KB of shared-memory traffic per k-block, the kernel's bound (r02bb ncu: l1tex 63 %, 0.33 of HBM)
    static constexpr bool TS = PLANES == 2;
    static constexpr int NTS = 6;                      // TMEM A slots (64 columns each) after 2 x 64 accumulators
    static constexpr int TCOLS = TS ? 512 : 128;
};

struct StemDwAux {
    uint64_t afull[8], cfull[8], bfull[8], sfree[8], accfull[2], accfree[2], tfree[8];
    uint32_t tmem_base;
};

// grid (pixel ranges, m-tiles of 128 output channels).  dY arrives by TMA as MN-major [32 px][32 oc]
// boxes (the layout the tensor core reads A from, SWIZZLE_128B_BASE32B), so the MMAs are SS-form:
// A = dY^T (M = oc), B = Xcol^T (N = k) built by CUDA-core threads, K = 32 pixels per k-block.
template <int PLANES, int OCB>
__global__ void __launch_bounds__(StemDwCfg<PLANES, OCB>::NTHREADS, 1)
    stem_dw_kernel(const __grid_constant__ StemParams p, const __grid_constant__ CUtensorMap mapA) {
    using C = StemDwCfg<PLANES, OCB>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* bptr = smem_raw + (base - raw);
    StemDwAux* aux = reinterpret_cast<StemDwAux*>(bptr + C::STAGES * C::STAGE + C::PAD);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int oc0 = blockIdx.y * 128;
    const int nblk = min(OCB, (p.OC - oc0 + 31) / 32);  // 32-channel dY boxes of this m-tile

    if (tid == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&aux->afull[s], 1);
            mbar_init(&aux->cfull[s], 4);
            mbar_init(&aux->bfull[s], 1);
            mbar_init(&aux->sfree[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&aux->accfull[b], 1);
            mbar_init(&aux->accfree[b], 4);
        }
        for (int t = 0; t < C::NTS; ++t) {
            mbar_init(&aux->tfree[t], 1);
        }
        fence_mbar_init();
    }
    if (warp == C::MMA_W) tmem_alloc(&aux->tmem_base, C::TCOLS);
    if (warp == C::TMA_W && lane == 0)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = aux->tmem_base;
    pdl_trigger();
    pdl_wait();
    const int kb0 = blockIdx.x * p.kb_per_cta;
    const int nkb = max(0, min(p.tiles, kb0 + p.kb_per_cta) - kb0);
    auto sA = [&](int s) { return base + (uint32_t)(s * C::STAGE); };
    auto sBb = [&](int s) { return base + (uint32_t)(s * C::STAGE + PLANES * C::A_BYTES); };

    if (warp == C::TMA_W) {
        for (int it = 0; it < nkb; ++it) {
            const int s = it % C::STAGES;
            if (it >= C::STAGES) mbar_wait(&aux->sfree[s], ((it / C::STAGES) - 1) & 1);
            if (elect_one()) {
                mbar_arrive_expect_tx(&aux->afull[s], (uint32_t)(nblk * 4096));
                for (int j = 0; j < nblk; ++j)
                    tma_load_2d(sA(s) + (uint32_t)(j * 4096), &mapA, &aux->afull[s], oc0 + 32 * j, (kb0 + it) * 32);
            }
            __syncwarp();
        }
    } else if (warp == C::MMA_W) {
        constexpr uint32_t IDESC = idesc_tf32(128, kDwN, true, false);  // A MN-major, B K-major
        constexpr uint32_t IDESC_TS = idesc_tf32(128, kDwN, false, false);  // A in TMEM (K along columns)
        const uint64_t ad0 = make_sdesc(base, 4096u, 512u, kLayoutSW128Base32);
        const uint64_t bd0 = make_sdesc(base + PLANES * C::A_BYTES, 16u, 1024u, kLayoutSW128);
        int c = 0;
        for (int it = 0; it < nkb; ++it) {
            const int s = it % C::STAGES, ic = it % C::CHUNK, b = c & 1;
            const int ts = it % C::NTS;
            if (ic == 0 && c >= 2) {
                mbar_wait(&aux->accfree[b], ((c >> 1) - 1) & 1);
                tc_fence_after();
            }
            if (PLANES == 2) mbar_wait(&aux->cfull[s], (it / C::STAGES) & 1);
            else mbar_wait(&aux->afull[s], (it / C::STAGES) & 1);
            mbar_wait(&aux->bfull[s], (it / C::STAGES) & 1);
            tc_fence_after();
            const bool last = ic == C::CHUNK - 1 || it == nkb - 1;
            if (elect_one()) {
                const uint32_t d = tmem + (uint32_t)(b * 64);
                const uint64_t so = (uint64_t)((s * C::STAGE) >> 4);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint64_t ah = ad0 + so + (uint64_t)j * 64;  // 8 px = 1024 B of the MN-major tile
                    const uint64_t bh = bd0 + so + (uint64_t)j * 2;   // 8 k = 32 B of the K-major tile
                    if (C::TS && p.ts) {  // a_hi | a_lo of this k-block in TMEM slot ts (columns 128 + 64 ts ..)
                        const uint32_t ahi = tmem + (uint32_t)(128 + ts * 64 + j * 8);
                        mma_tf32_ts(d, ahi, bh, IDESC_TS, (ic > 0 || j > 0) ? 1u : 0u);
                        mma_tf32_ts(d, ahi, bh + (uint64_t)(C::B_BYTES >> 4), IDESC_TS, 1u);
                        mma_tf32_ts(d, ahi + 32, bh, IDESC_TS, 1u);
                    } else {
                        mma_tf32_ss(d, ah, bh, IDESC, (ic > 0 || j > 0) ? 1u : 0u);
                        if (PLANES == 2) {
                            mma_tf32_ss(d, ah, bh + (uint64_t)(C::B_BYTES >> 4), IDESC, 1u);
                            mma_tf32_ss(d, ah + (uint64_t)(C::A_BYTES >> 4), bh, IDESC, 1u);
                        }
                    }
                }
                if (C::TS && p.ts) mma_commit(&aux->tfree[ts]);
                mma_commit(&aux->sfree[s]);
                if (last) mma_commit(&aux->accfull[b]);
            }
            __syncwarp();
            if (last) ++c;
        }
    } else if (warp >= C::BLD_W0 && warp < C::BLD_W0 + C::NBLD) {
        // IM2COL^T builders: warp w builds the k-blocks it % 4 == w; lane = pixel of the k-block
        // (the gather of the warp's NEXT k-block is issued before this one is stored: with one gather
        // in flight per warp the builders were latency-bound at small batch, VGG b128 stem dW 39 us, r02y)
        const int w = warp - C::BLD_W0;
        float e[kKP], en[kKP];
        if (w < nkb) gather_row(p, (long long)(kb0 + w) * 32 + lane, e);
        for (int it = w; it < nkb; it += C::NBLD) {
            const int s = it % C::STAGES;
            if (it + C::NBLD < nkb) gather_row(p, (long long)(kb0 + it + C::NBLD) * 32 + lane, en);
            if (it >= C::STAGES) mbar_wait(&aux->sfree[s], ((it / C::STAGES) - 1) & 1);
            const uint32_t sb = sBb(s);
            // element (k, px) of the K-major [48][32 px] tile: row k, 16-B chunk px / 4, word px % 4
            const uint32_t cw = (uint32_t)(lane & 3) * 4;
#pragma unroll
            for (int k = 0; k < kDwN; ++k) {
                const float x = k < kK ? e[k] : 0.f;
                const uint32_t off = kmaj_off((uint32_t)k, (uint32_t)(lane >> 2)) + cw;
                asm volatile("st.shared.f32 [%0], %1;" ::"r"(sb + off), "f"(x) : "memory");
                if (PLANES == 2)
                    asm volatile("st.shared.f32 [%0], %1;" ::"r"(sb + C::B_BYTES + off), "f"(__uint_as_float(lo_bits(x)))
                                 : "memory");
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&aux->bfull[s]);
#pragma unroll
            for (int k = 0; k < kKP; ++k) e[k] = en[k];
        }
    } else if (warp >= C::CONV_W0 && warp < C::CONV_W0 + 4) {
        // 3xTF32 (TS form): dY^T -> TMEM slot it % NTS as a_hi | a_lo.  The thread owning TMEM lane
        // oc_l = 32 (warp % 4) + lane reads dY[px][oc_l] of the MN-major tile for the 32 pixels
        if (C::TS && p.ts) {
            const int qd = warp & 3;
            const int ocl = 32 * qd + lane;
            const uint32_t lanebase = (uint32_t)(qd * 32) << 16;
            for (int it = 0; it < nkb; ++it) {
                const int s = it % C::STAGES, ts = it % C::NTS;
                mbar_wait(&aux->afull[s], (it / C::STAGES) & 1);
                if (it >= C::NTS) {
                    mbar_wait(&aux->tfree[ts], ((it / C::NTS) - 1) & 1);
                    tc_fence_after();
                }
                if (qd < nblk) {  // rows >= 32 nblk are the m-tile's junk rows (OC < 128): never stored
                    const uint8_t* tile = bptr + s * C::STAGE;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        uint32_t hi[16], lo[16];
#pragma unroll
                        for (int k = 0; k < 16; ++k) {
                            const float e = *reinterpret_cast<const float*>(
                                tile + mnmaj_off((uint32_t)(16 * h + k), (uint32_t)(ocl & ~3)) + (ocl & 3) * 4);
                            const uint32_t hb = __float_as_uint(e) & 0xFFFFE000u;
                            hi[k] = hb;
                            lo[k] = __float_as_uint(e - __uint_as_float(hb));
                        }
                        const uint32_t ta = tmem + lanebase + (uint32_t)(128 + ts * 64);
                        tmem_st_32x32b_x16(ta + h * 16, hi);
                        tmem_st_32x32b_x16(ta + 32 + h * 16, lo);
                    }
                    tmem_st_wait();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&aux->cfull[s]);
            }
        } else if (PLANES == 2) {
            const int ct = tid - C::CONV_W0 * 32;
            for (int it = 0; it < nkb; ++it) {
                const int s = it % C::STAGES;
                mbar_wait(&aux->afull[s], (it / C::STAGES) & 1);
                const float4* src = reinterpret_cast<const float4*>(bptr + s * C::STAGE);
                float4* dst = reinterpret_cast<float4*>(bptr + s * C::STAGE + C::A_BYTES);
                const int n4 = nblk * 256;  // 16-B chunks present
                for (int i = ct; i < n4; i += 128) {
                    const float4 v = src[i];
                    dst[i] = make_float4(__uint_as_float(lo_bits(v.x)), __uint_as_float(lo_bits(v.y)),
                                         __uint_as_float(lo_bits(v.z)), __uint_as_float(lo_bits(v.w)));
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&aux->cfull[s]);
            }
        }
    } else if (warp >= C::PRO_W0 && warp < C::PRO_W0 + 4) {
        // promotion: rows (TMEM lanes) 32q..32q+31 = channels oc0 + 32q + lane
        const int q = warp & 3;
        const uint32_t lanebase = (uint32_t)(q * 32) << 16;
        const int oc = oc0 + 32 * q + lane;
        float acc[kDwN];
#pragma unroll
        for (int k = 0; k < kDwN; ++k) acc[k] = 0.f;
        const int nch = (nkb + C::CHUNK - 1) / C::CHUNK;
        for (int c = 0; c < nch; ++c) {
            const int b = c & 1;
            mbar_wait(&aux->accfull[b], (c >> 1) & 1);
            tc_fence_after();
#pragma unroll
            for (int k0 = 0; k0 < kDwN; k0 += 16) {
                uint32_t r[16];
                tmem_ld_32x32b_x16(tmem + lanebase + (uint32_t)(b * 64 + k0), r);
                tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 16; ++e) acc[k0 + e] += __uint_as_float(r[e]);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&aux->accfree[b]);
        }
        // this CTA's partial [OC][36] (columns 36..47 are the zero padding)
        if (oc < p.OC) {
            float* o = p.out + ((long long)blockIdx.x * p.OC + oc) * kK;
#pragma unroll
            for (int k = 0; k < kK; k += 4)
                *reinterpret_cast<float4*>(o + k) = make_float4(acc[k], acc[k + 1], acc[k + 2], acc[k + 3]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == C::MMA_W) {
        tc_fence_after();
        tmem_dealloc(tmem, C::TCOLS);
    }
}

template <typename K>
int set_smem(K kern, int bytes, char* err, size_t errlen) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) {
        snprintf(err, errlen, "cudaFuncSetAttribute(stem smem=%d): %s", bytes, cudaGetErrorString(cudaGetLastError()));
        return CONV_ECUDA;
    }
    return CONV_OK;
}

}  // namespace

// The STEM variant serves IC == 4 (the padded RGB input), 3x3 filters, any stride / padding;
// fwd with OC in {64, 128, 192}, dW with OC a multiple of 4.
bool stem_supported(int op, int IC, int OC, int FH, int FW) {
    if (IC != 4 || FH != 3 || FW != 3) return false;
    if (op == CONV_OP_FWD) return OC == 64 || OC == 128 || OC == 192;  // B planes + staging fit shared memory
    if (op == CONV_OP_BWD_FILTER) return OC % 4 == 0;
    return false;
}

// dW: CTAs per m-tile and k-blocks per CTA (a CTA's partial covers kb_per_cta k-blocks of 32 pixels)
int stem_dw_split(long long M, int OC, int* kb_per_cta) {
    const long long nkb = (M + 31) / 32;
    const int mt = (OC + 127) / 128;
    long long per = (nkb * mt + kSMs - 1) / kSMs;
    if (per < 8) per = 8;
    *kb_per_cta = (int)per;
    return (int)((nkb + per - 1) / per);
}

int stem_launch(int op, int planes, const GenParams& g, int splits, int kb_per_split, cudaStream_t st, char* err,
                size_t errlen) {
    StemParams p;
    memset(&p, 0, sizeof p);
    p.N = g.N; p.IH = g.IH; p.IW = g.IW; p.OC = g.OC; p.OH = g.OH; p.OW = g.OW;
    p.sh = g.sh; p.sw = g.sw; p.ph = g.ph; p.pw = g.pw;
    p.M = (long long)g.N * g.OH * g.OW;
    if (p.M >= (1LL << 31)) {
        snprintf(err, errlen, "stem: N*OH*OW >= 2^31");
        return CONV_EUNSUPPORTED;
    }
    p.fd_OW = make_fastdiv((uint32_t)g.OW);
    p.fd_OHOW = make_fastdiv((uint32_t)(g.OH * g.OW));
    if (op == CONV_OP_FWD) {
        p.X = g.A;
        p.W = g.B;
        p.out = g.out;
        p.tiles = (int)((p.M + 127) / 128);
        uint64_t dims[2] = {(uint64_t)g.OC, (uint64_t)p.M}, strides[1] = {(uint64_t)g.OC * 4};
        uint32_t box[2] = {32, 32};
        if (!tma_encode_f32(&p.mapY, g.out, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B)) {
            snprintf(err, errlen, "stem: cuTensorMapEncodeTiled(Y) failed");
            return CONV_ECUDA;
        }
        const int grid = p.tiles < kSMs ? p.tiles : kSMs;
        auto go = [&](auto kern, int smem) -> int {
            int rc = set_smem(kern, smem, err, errlen);
            if (rc) return rc;
            const cudaError_t e = launch_k(kern, dim3(grid), dim3(13 * 32), smem, st, 1, p);
            if (e != cudaSuccess) {
                snprintf(err, errlen, "stem fwd launch: %s", cudaGetErrorString(e));
                return CONV_ECUDA;
            }
            return CONV_OK;
        };
        switch (g.OC) {
            case 64: return planes == 2 ? go(stem_fwd_kernel<64, 2>, StemFwdCfg<64, 2>::SMEM)
                                        : go(stem_fwd_kernel<64, 1>, StemFwdCfg<64, 1>::SMEM);
            case 128: return planes == 2 ? go(stem_fwd_kernel<128, 2>, StemFwdCfg<128, 2>::SMEM)
                                         : go(stem_fwd_kernel<128, 1>, StemFwdCfg<128, 1>::SMEM);
            default: return planes == 2 ? go(stem_fwd_kernel<192, 2>, StemFwdCfg<192, 2>::SMEM)
                                        : go(stem_fwd_kernel<192, 1>, StemFwdCfg<192, 1>::SMEM);
        }
    }
    // dW: run() passes A = dY, B = X; partials [splits][OC][36] into g.out (the workspace)
    p.dY = g.A;
    p.X = g.B;
    p.out = g.out;
    p.tiles = (int)((p.M + 31) / 32);
    p.kb_per_cta = kb_per_split;
    static const int ts_knob = getenv("SMCONV_STEM_TS") ? atoi(getenv("SMCONV_STEM_TS")) : 1;
    p.ts = ts_knob;
    CUtensorMap mapA;  // dY viewed [M][OC], box (32 oc, 32 px), MN-major A blocks
    {
        uint64_t dims[2] = {(uint64_t)g.OC, (uint64_t)p.M}, strides[1] = {(uint64_t)g.OC * 4};
        uint32_t box[2] = {32, 32};
        if (!tma_encode_f32(&mapA, g.A, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) {
            snprintf(err, errlen, "stem: cuTensorMapEncodeTiled(dY) failed");
            return CONV_ECUDA;
        }
    }
    const dim3 grid(splits, (g.OC + 127) / 128);
    auto go = [&](auto kern, int smem) -> int {
        int rc = set_smem(kern, smem, err, errlen);
        if (rc) return rc;
        const cudaError_t e = launch_k(kern, grid, dim3(StemDwCfg<1, 4>::NTHREADS), smem, st, 1, p, mapA);
        if (e != cudaSuccess) {
            snprintf(err, errlen, "stem dw launch: %s", cudaGetErrorString(e));
            return CONV_ECUDA;
        }
        return CONV_OK;
    };
    if (g.OC <= 64)
        return planes == 2 ? go(stem_dw_kernel<2, 2>, StemDwCfg<2, 2>::SMEM) : go(stem_dw_kernel<1, 2>, StemDwCfg<1, 2>::SMEM);
    return planes == 2 ? go(stem_dw_kernel<2, 4>, StemDwCfg<2, 4>::SMEM) : go(stem_dw_kernel<1, 4>, StemDwCfg<1, 4>::SMEM);
}

}  // namespace smconv
