// pair_ring_bench.cu — cost of the CTA-pair barrier ring of conv_tma_kernel<..., PAIR>: producer ->
// converters (both CTAs; remote per-warp arrivals on CTA 0) -> MMA warp (CTA 0; M = 256 MMAs) ->
// multicast commits (empty / tfree in both CTAs).  No memory traffic.  (tools only)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude tools/pair_ring_bench.cu -o tools/pair_ring_bench.bin
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../paper_2305_08819_b200/csrc/common.cuh"

using namespace smconv;

constexpr int SS = 6, NT = 4;
struct Aux { uint64_t full[SS], empty[SS], conv[NT], tfree[NT]; uint32_t tmem; };

template <bool PAIR>
__global__ void __launch_bounds__(576, 1) ring_kernel(int iters, int nmma) {
    __shared__ Aux aux;
    extern __shared__ __align__(1024) uint8_t dyn[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = PAIR ? (int)cluster_ctarank() : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < SS; ++s) { mbar_init(&aux.full[s], 1); mbar_init(&aux.empty[s], 1); }
        for (int t = 0; t < NT; ++t) { mbar_init(&aux.conv[t], PAIR ? 16 : 8); mbar_init(&aux.tfree[t], 1); }
        fence_mbar_init();
    }
    if (warp == 9) { if (PAIR) tmem_alloc2(&aux.tmem, 512); else tmem_alloc(&aux.tmem, 512); }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = aux.tmem;
    if (warp == 8) {  // producer
        for (int q = 0; q < iters; ++q) {
            const int s = q % SS, r = q / SS;
            if (r > 0) { if (PAIR) mbar_wait_cluster(&aux.empty[s], (r - 1) & 1); else mbar_wait(&aux.empty[s], (r - 1) & 1); }
            if (elect_one()) mbar_arrive(&aux.full[s]);
            __syncwarp();
        }
    } else if (warp == 9) {
        if (!PAIR || rank == 0) {
            const uint32_t base = (smem_u32(dyn) + 1023u) & ~1023u;
            const uint64_t bd = make_sdesc(base, 4096u, 512u, kLayoutSW128Base32);
            for (int q = 0; q < iters; ++q) {
                const int s = q % SS, t = q % NT, rt = q / NT;
                if (PAIR) mbar_wait_cluster(&aux.conv[t], rt & 1); else mbar_wait(&aux.conv[t], rt & 1);
                tc_fence_after();
                if (elect_one()) {
                    for (int i = 0; i < nmma; ++i) {
                        if (PAIR) mma2_tf32_ts(tmem, tmem + 256 + t * 64 + (i & 3) * 8, bd + (i & 3) * 64, idesc_tf32(256, 128, false, true), i > 0);
                        else mma_tf32_ts(tmem, tmem + 256 + t * 64 + (i & 3) * 8, bd + (i & 3) * 64, idesc_tf32(128, 128, false, true), i > 0);
                    }
                    if (PAIR) { mma2_commit_both(&aux.empty[s]); mma2_commit_both(&aux.tfree[t]); }
                    else { mma_commit(&aux.empty[s]); mma_commit(&aux.tfree[t]); }
                }
                __syncwarp();
            }
        }
    } else if (warp >= 10) {  // converters
        for (int q = 0; q < iters; ++q) {
            const int s = q % SS, t = q % NT, rt = q / NT;
            mbar_wait(&aux.full[s], (q / SS) & 1);
            if (rt > 0) { if (PAIR) mbar_wait_cluster(&aux.tfree[t], (rt - 1) & 1); else mbar_wait(&aux.tfree[t], (rt - 1) & 1); }
            tc_fence_after();
            tmem_st_wait();
            fence_proxy_async_smem();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) { if (PAIR) mbar_arrive_remote(&aux.conv[t], 0); else mbar_arrive(&aux.conv[t]); }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync_all();
    if (warp == 9) { tc_fence_after(); if (PAIR) tmem_dealloc2(tmem, 512); else tmem_dealloc(tmem, 512); }
}

template <bool PAIR>
float run(int iters, int nmma) {
    const int smem = 100 * 1024;
    cudaFuncSetAttribute(ring_kernel<PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148, 1, 1);
    cfg.blockDim = dim3(576, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = PAIR ? 2 : 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaLaunchKernelEx(&cfg, ring_kernel<PAIR>, iters, nmma);
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) cudaLaunchKernelEx(&cfg, ring_kernel<PAIR>, iters, nmma);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%s nmma=%d: %.1f ns per k-block  %s\n", PAIR ? "pair  " : "single", nmma, ms / 3 * 1e6 / iters, cudaGetErrorString(cudaGetLastError()));
    return ms;
}

int main() {
    for (int nmma : {0, 12}) { run<false>(4000, nmma); run<true>(4000, nmma); }
    return 0;
}
