// pair_bench.cu — does a CTA pair (tcgen05.mma.cta_group::2, M = 256) run N = 64 MMAs faster per SM
// than one CTA (cta_group::1, M = 128)?  Timing only, garbage operands.  (tools only)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude tools/pair_bench.cu -o tools/pair_bench.bin
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2305_08819_b200/csrc/common.cuh"

using namespace smconv;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int BN, bool SS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) pair_kernel(int iters, int nmma, int commits_per_iter) {
    __shared__ uint64_t bar;
    __shared__ uint64_t bar2[4];
    __shared__ uint32_t tbase;
    extern __shared__ __align__(1024) uint8_t dyn[];
    const int warp = threadIdx.x >> 5;
    const uint32_t rank = cluster_rank();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        for (int i = 0; i < 4; ++i) mbar_init(&bar2[i], 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tbase;
    {   // non-zero operands (power depends on data toggling): random smem, random TMEM A columns
        uint32_t x = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x;
        float* f = reinterpret_cast<float*>(dyn);
        for (int i = threadIdx.x; i < 130 * 1024 / 4; i += blockDim.x) {
            x = x * 1664525u + 1013904223u;
            f[i] = __uint_as_float((x >> 9) | 0x3F800000u) - 1.5f;
        }
        uint32_t v[16];
        for (int c = 0; c < 256; c += 16) {
            for (int e = 0; e < 16; ++e) {
                x = x * 1664525u + 1013904223u;
                v[e] = __float_as_uint(__uint_as_float((x >> 9) | 0x3F800000u) - 1.5f);
            }
            tmem_st_32x32b_x16(tmem + ((uint32_t)(warp * 32) << 16) + 256 + c, v);
        }
        tmem_st_wait();
        fence_proxy_async_smem();
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
    }
    if (rank == 0 && warp == 1) {
        const uint32_t base = (smem_u32(dyn) + 1023u) & ~1023u;
        constexpr uint32_t IDESC = idesc_tf32(256, BN, false, true);
        const uint64_t bd = make_sdesc(base, 4096u, 512u, kLayoutSW128Base32);
        const uint64_t ad = make_sdesc(base + 65536, 16u, 1024u, kLayoutSW128);
        for (int q = 0; q < iters; ++q) {
            if (elect_one()) {
                if (commits_per_iter > 0 && q > 0)
                    for (int cc = 0; cc < commits_per_iter; ++cc)
                        asm volatile(
                            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                                smem_u32(&bar2[cc])),
                            "h"((uint16_t)3)
                            : "memory");
                for (int i = 0; i < nmma; ++i) {
                    const uint32_t acc = i > 0 ? 1u : 0u;
                    if (SS)
                        asm volatile(
                            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                            "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                            "l"(ad + (i & 3) * 2), "l"(bd + (i & 3) * 64), "r"(IDESC), "r"(acc)
                            : "memory");
                    else
                        asm volatile(
                            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                            "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                            "r"(tmem + 256 + (i & 3) * 8), "l"(bd + (i & 3) * 64), "r"(IDESC), "r"(acc)
                            : "memory");
                }
            }
            __syncwarp();
        }
        if (elect_one())
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                    smem_u32(&bar)),
                "h"((uint16_t)3)
                : "memory");
        __syncwarp();
    }
    if (threadIdx.x == 0) mbar_wait(&bar, 0);
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    }
}

int main(int argc, char** argv) {
    const int iters = argc > 1 ? atoi(argv[1]) : 2657;
    const int only = argc > 2 ? atoi(argv[2]) : -1;  // run only case #only
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int smem = 140 * 1024;
    struct Case { int bn; bool ss; int nmma; int commits; };
    const Case cases[] = {{64, false, 24, 0}, {128, false, 24, 0}, {64, false, 24, 2}, {128, false, 24, 2},
                          {64, false, 12, 2}, {128, false, 12, 2}, {128, false, 12, 0}};
    int ci = -1;
    for (const Case& c : cases) {
        if (++ci, only >= 0 && ci != only) continue;
        void (*k)(int, int, int) = nullptr;
        if (c.bn == 32) k = c.ss ? pair_kernel<32, true> : pair_kernel<32, false>;
        if (c.bn == 64) k = c.ss ? pair_kernel<64, true> : pair_kernel<64, false>;
        if (c.bn == 128) k = c.ss ? pair_kernel<128, true> : pair_kernel<128, false>;
        if (c.bn == 256) k = c.ss ? pair_kernel<256, true> : pair_kernel<256, false>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k<<<148, 128, smem>>>(iters, c.nmma, c.commits);
        cudaEventRecord(e0);
        for (int rep = 0; rep < 5; ++rep) k<<<148, 128, smem>>>(iters, c.nmma, c.commits);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaError_t err = cudaGetLastError();
        const double flop = 2.0 * 256 * c.bn * 8 * c.nmma * (double)iters * 74;
        printf("cta_group::2 %s M=256 N=%d x%d commits/iter %d: %.1f ns per k-block (per pair), %.0f TFLOP/s tf32  %s\n",
               c.ss ? "ss" : "ts", c.bn, c.nmma, c.commits, ms / 5 * 1e6 / iters, flop / (ms / 5 * 1e-3) / 1e12,
               cudaGetErrorString(err));
    }
    return 0;
}
