// common.cuh — sm_100a device primitives shared by the smconv kernels:
// mbarriers, tcgen05 (TMEM alloc, MMA kind::tf32, commit, ld), UMMA shared-memory
// descriptors for the 128-byte-swizzled canonical layouts, TF32 rounding, fast division.
//
// Compile with -gencode arch=compute_100a,code=sm_100a (tcgen05 needs the "a" target).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define SMCONV_DEV __device__ __forceinline__
#define SMCONV_HD __host__ __device__ __forceinline__

namespace smconv {

// ------------------------------------------------------------------ fast division
// q = floor(n / d) for 0 <= n < 2^31 with one mul.hi (round-up multiplier method).
struct FastDiv {
    uint32_t d, mul, shift;
};

inline FastDiv make_fastdiv(uint32_t d) {
    FastDiv f;
    f.d = d;
    uint32_t s = 0;
    while ((1ull << s) < d) ++s;
    f.shift = s;
    f.mul = (uint32_t)((((1ull << 32) * ((1ull << s) - d)) / d) + 1);
    return f;
}

SMCONV_HD uint32_t umulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
    return __umulhi(a, b);
#else
    return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

SMCONV_HD uint32_t fdiv(uint32_t n, const FastDiv& f) { return (umulhi32(n, f.mul) + n) >> f.shift; }

// ------------------------------------------------------------------ programmatic dependent launch
// (launch.cuh): let the next kernel of the stream be scheduled now / wait until the previous kernels
// have completed and their writes are visible.  Every kernel calls pdl_wait() before its first
// global-memory access; both are no-ops for a kernel launched without the PDL attribute.
SMCONV_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
SMCONV_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ------------------------------------------------------------------ shared-memory helpers
SMCONV_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

SMCONV_DEV void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

SMCONV_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

SMCONV_DEV void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
                 : "memory");
}

SMCONV_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                     smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

SMCONV_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "SMCONV_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra SMCONV_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// One lane of the (converged) warp gets true.  Issue loops for tcgen05.mma / TMA run on the
// whole warp with warp-uniform values and issue under elect_one(): if only `lane == 0` ran the
// loop, ptxas cannot prove the operands uniform and wraps every UTCHMMA / UTMALDG in an
// ELECT + R2UR.BROADCAST + BRA.U.ANY waterfall (measured: ~140 issue instructions per k-block).
SMCONV_DEV bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .b32 r;\n\t.reg .pred p;\n\t"
        "elect.sync r|p, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(pred));
    return pred != 0;
}

// Make this thread's generic-proxy shared-memory writes visible to the async proxy
// (tensor-core operand reads, TMA).  Must precede the release (mbarrier arrive).
SMCONV_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ------------------------------------------------------------------ tcgen05
// TMEM allocation: executed by one full warp; writes the TMEM base address to *dst.
SMCONV_DEV void tmem_alloc(uint32_t* dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

SMCONV_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

SMCONV_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
SMCONV_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T, TF32 inputs, FP32 accumulate, issued by ONE thread.
SMCONV_DEV void mma_tf32_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum)
        : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem]^T (A: 128 lanes = M rows, 8 consecutive 32-bit columns = K).
SMCONV_DEV void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accum)
        : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns <- 16 registers per thread.
SMCONV_DEV void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

// 32 lanes x 32 bit, 8 consecutive columns <- 8 registers per thread.
SMCONV_DEV void tmem_st_32x32b_x8(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

// two fp32 -> packed bf16x2 (round to nearest even); `lo` lands in bits 0-15 (the lower K index)
SMCONV_DEV uint32_t pack_bf16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

// D[tmem] (+)= A[tmem] * B[smem]^T, kind::f16 with bf16 operands and an fp32 accumulator (K = 16)
SMCONV_DEV void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accum)
        : "memory");
}

SMCONV_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Arrive (once) on an mbarrier when all previously issued tcgen05 ops of this thread complete.
SMCONV_DEV void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns -> 16 registers per thread (thread i = lane base + i).
SMCONV_DEV void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

SMCONV_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Instruction descriptor for kind::tf32 (PTX ISA "Instruction descriptor"):
// [4,6) D fmt (1=F32), [7,10) A fmt (2=TF32), [10,13) B fmt (2=TF32), 15 A MN-major,
// 16 B MN-major, [17,23) N>>3, [24,29) M>>4.
SMCONV_HD constexpr uint32_t idesc_tf32(int M, int N, bool a_mn_major, bool b_mn_major) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn_major ? 1u : 0u) << 15) | ((b_mn_major ? 1u : 0u) << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// kind::f16 with bf16 A and B (A/B fmt 1), fp32 D; same field positions as idesc_tf32.
SMCONV_HD constexpr uint32_t idesc_bf16(int M, int N, bool a_mn_major, bool b_mn_major) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn_major ? 1u : 0u) << 15) | ((b_mn_major ? 1u : 0u) << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// Shared-memory matrix descriptor (sm_100 version bit 46).  Layout types used here:
//  2 = SWIZZLE_128B        K-major canonical: 8-row x 128-B atoms, 16-B chunk c of row r stored at
//                          chunk c ^ (r % 8); SBO = byte stride between 8-row groups (LBO unused).
//  1 = SWIZZLE_128B_BASE32B MN-major canonical for 32-bit (TF32) operands: 128 B (32 elements) along
//                          MN per K-row, 32-B chunk j of K-row k stored at chunk j ^ (k % 4);
//                          4-row atoms, SBO = byte stride between 4-row K atoms (512 B when rows are
//                          contiguous), LBO = byte stride between 32-element MN blocks.
//  (tcgen05 requires the BASE32B swizzle for MN-major TF32; plain 128B swizzle is K-major only.)
constexpr uint32_t kLayoutSW128 = 2, kLayoutSW128Base32 = 1;

SMCONV_DEV uint64_t make_sdesc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}

SMCONV_DEV uint64_t make_sdesc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    return make_sdesc(saddr, lbo_bytes, sbo_bytes, kLayoutSW128);
}

// Byte offsets of one 16-byte chunk inside this library's two tile layouts (both 1024-B aligned):
//  K-major tile  [R rows][32 k]  : chunk c (k = 4c..4c+3) of row r                 (SWIZZLE_128B)
//  MN-major tile [32 k][MN cols] : chunk holding mn..mn+3 (mn % 4 == 0) of K-row k (SWIZZLE_128B_BASE32B);
//                                  each 32-wide MN block is a contiguous 4 KB [32 k][128 B].
SMCONV_HD uint32_t kmaj_off(uint32_t r, uint32_t c) { return (r >> 3) * 1024u + (r & 7u) * 128u + ((c ^ (r & 7u)) << 4); }
SMCONV_HD uint32_t mnmaj_off(uint32_t k, uint32_t mn) {
    return (mn >> 5) * 4096u + k * 128u + (((((mn >> 3) & 3u) ^ (k & 3u))) << 5) + (((mn >> 2) & 1u) << 4);
}

// ------------------------------------------------------------------ 3xTF32 operand split
// x = x_hi + x_lo with x_hi = trunc_tf32(x) (what kind::tf32 reads from an fp32 word) and x_lo exact.
// The product a*b = a_hi*b_hi + [a_hi*b_lo + a_lo*b]: the first term runs as a TF32 MMA, the
// bracket (~2^-10 of it) as ONE bf16 MMA pair with K doubled, A' = [bf16(a_hi) | bf16(a_lo)],
// B' = [bf16(b_lo) | bf16(b)] (bf16 keeps 8 bits of a term already 2^-10 small: ~2^-18 relative,
// and a bf16 flop costs half a TF32 flop of tensor-pipe time and energy).

// one A row, 16 consecutive k: hi[] = a_hi bits (TF32 operand columns), xh[] / xl[] = bf16 pairs
SMCONV_DEV void split_a16(const float (&e)[16], uint32_t (&hi)[16], uint32_t (&xh)[8], uint32_t (&xl)[8]) {
#pragma unroll
    for (int k = 0; k < 16; ++k) hi[k] = __float_as_uint(e[k]) & 0xFFFFE000u;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const float h0 = __uint_as_float(hi[2 * i]), h1 = __uint_as_float(hi[2 * i + 1]);
        xh[i] = pack_bf16x2(h0, h1);
        xl[i] = pack_bf16x2(e[2 * i] - h0, e[2 * i + 1] - h1);
    }
}

// ------------------------------------------------------------------ CTA pairs (cta_group::2)
// A 2-CTA cluster runs one M = 256 MMA per instruction: each CTA holds 128 rows of A (here in its
// own TMEM) and N/2 columns of B in its shared memory, each CTA's TMEM receives its 128 rows x N of
// the accumulator.  Measured (tools/pair_bench.cu vs tools/ring_bench.cu, random operands, at the
// power cap): N = 64 tiles 894 vs 507 TFLOP/s TF32, N = 128 tiles 898 vs 759.
SMCONV_DEV uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// 16-byte load from the shared memory of CTA `cta` of this cluster at the offset of local address `la`
// In-switch reduction through an NVLink multicast (NVLS) address: adds v into the element at `mc` of
// EVERY GPU bound to the multicast object (smconv_mcast.h)
SMCONV_DEV void mc_red_add_f4(float* mc, float4 v) {
    asm volatile("multimem.red.relaxed.sys.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}

// 16-B store into the shared memory of CTA `cta` of the cluster at local offset-address `la`
SMCONV_DEV void st_cluster_f4(uint32_t la, uint32_t cta, float4 v) {
    asm volatile(
        "{\n\t.reg .b32 ra;\n\t"
        "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
        "st.shared::cluster.v4.f32 [ra], {%2, %3, %4, %5};\n\t}" ::"r"(la),
        "r"(cta), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
        : "memory");
}

SMCONV_DEV float4 ld_cluster_f4(uint32_t la, uint32_t cta) {
    float4 v;
    asm volatile(
        "{\n\t.reg .b32 ra;\n\t"
        "mapa.shared::cluster.u32 ra, %4, %5;\n\t"
        "ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [ra];\n\t}"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
        : "r"(la), "r"(cta)
        : "memory");
    return v;
}

SMCONV_DEV void cluster_arrive_wait() {  // same as cluster_sync_all, for one role's threads at a time
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// arrival without release semantics: `.release` compiles to MEMBAR.ALL.GPU + ERRBAR, i.e. the
// arriving thread first waits for ALL of its outstanding global stores (3-4 % of the stall samples of
// the small-map csk kernels, ncu r02bg); enough where the barrier only keeps a CTA alive while its
// peers still read its shared memory (the reads completed before the arrival: their values were used)
SMCONV_DEV void cluster_sync_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

SMCONV_DEV void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// arrive on the mbarrier at the same shared-memory offset in CTA `cta`.  Default semantics
// (release at CTA scope, no fence in the SASS): what crosses the CTA boundary here is TMEM state
// (converter tcgen05.st / epilogue tcgen05.ld), ordered by tcgen05.wait::{st,ld} +
// tcgen05.fence::before_thread_sync on this side and fence::after_thread_sync after the wait.
// The explicit `.release.cluster` form compiles to MEMBAR.ALL.GPU + ERRBAR, which waited for
// every outstanding global store of the arriving warp (ncu r01n: 'membar' the second stall
// reason of the pair kernel, pairs 1.7x slower than single-CTA tiles).
SMCONV_DEV void mbar_arrive_remote(uint64_t* bar, uint32_t cta) {
    asm volatile(
        "{\n\t.reg .b32 ra;\n\t"
        "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
        "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
        "r"(cta)
        : "memory");
}

// wait on a barrier the peer CTA (or a multicast commit) arrives on.  CTA-scope acquire (the
// default): no generic-proxy data crosses the CTA boundary here (TMEM state is ordered by the
// tcgen05 fences, smem stages by the TMA / MMA mbarrier protocol).  `.acquire.cluster` compiles to
// a CCTL.IVALL (L1 invalidate) after every successful wait: 22 % of the stall samples of the pair
// l2.0a dX kernel (ncu source view, r01r) sat on it; dropping it bought ~0.5 % of the step (r01t,
// the step is power-capped).
SMCONV_DEV void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "SMCONV_WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra SMCONV_WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// both CTAs' warps with the same warp id execute these
SMCONV_DEV void tmem_alloc2(uint32_t* dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
SMCONV_DEV void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// D[tmem, both CTAs] (+)= A[tmem, both CTAs] * B[smem, N/2 per CTA]^T; issued by one thread of CTA 0
SMCONV_DEV void mma2_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accum)
        : "memory");
}

SMCONV_DEV void mma2_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accum)
        : "memory");
}

// arrive once on the mbarrier at this offset in both CTAs of the pair when the issued MMAs complete
SMCONV_DEV void mma2_commit_both(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}

// ------------------------------------------------------------------ TF32 split
SMCONV_DEV float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

SMCONV_DEV void st_shared_v4(uint32_t addr, float a, float b, float c, float d) {
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

SMCONV_DEV float4 ldg_f4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

}  // namespace smconv
