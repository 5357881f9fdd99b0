// ring_bench.cu — microbenchmark of the warp-specialised mbarrier pipeline used by the conv
// kernels, with no memory traffic and no MMAs: how many k-blocks per microsecond can the
// producer -> converters -> MMA-issuer -> producer ring sustain?  (tools only; not part of the library)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../include tools/ring_bench.cu -o /tmp/ring_bench
//   /tmp/ring_bench
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2305_08819_b200/csrc/common.cuh"

using namespace smconv;

struct Aux {
    uint64_t full[8], empty[8], conv[8], tfree[8];
};

// mode bit 1: converters present (else MMA waits full directly)
// mode bit 2: use tcgen05.commit for empty/tfree (else plain arrive)
// mode bit 4: per-thread (256) conv arrivals instead of per-warp (8)
// mode bit 8: converters also issue fence.proxy.async + tcgen05 fences
// mode bit 16: the MMA warp issues nmma tf32 MMAs per k-block (M=128, N=BN, K=8): TS form (A in
//              TMEM) unless bit 32 (SS form, A in smem); operands are garbage (timing only)
template <int SS, int ST, int BN, int BM = 128>
__global__ void __launch_bounds__(576, 1) ring_kernel(int iters, int mode, int nconvw, int nmma) {
    __shared__ Aux aux;
    __shared__ uint32_t tbase;
    extern __shared__ __align__(1024) uint8_t dyn[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool conv = mode & 1, commit = mode & 2, perthread = mode & 4, fences = mode & 8;
    const int conv_count = perthread ? nconvw * 32 : nconvw;
    if (tid == 0) {
        for (int s = 0; s < SS; ++s) {
            mbar_init(&aux.full[s], 1);
            mbar_init(&aux.empty[s], 1);
        }
        for (int t = 0; t < ST; ++t) {
            mbar_init(&aux.conv[t], conv_count);
            mbar_init(&aux.tfree[t], 1);
        }
        fence_mbar_init();
    }
    if (warp == 9) tmem_alloc(&tbase, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp < 4) {  // non-zero operands (power depends on data toggling): random smem, random TMEM A columns
        uint32_t x = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x;
        float* f = reinterpret_cast<float*>(dyn);
        for (int i = threadIdx.x; i < 130 * 1024 / 4; i += 128) {
            x = x * 1664525u + 1013904223u;
            f[i] = __uint_as_float((x >> 9) | 0x3F800000u) - 1.5f;
        }
        uint32_t v[16];
        for (int c = 0; c < 256; c += 16) {
            for (int e = 0; e < 16; ++e) {
                x = x * 1664525u + 1013904223u;
                v[e] = __float_as_uint(__uint_as_float((x >> 9) | 0x3F800000u) - 1.5f);
            }
            tmem_st_32x32b_x16(tbase + ((uint32_t)(warp * 32) << 16) + 256 + c, v);
        }
        tmem_st_wait();
        fence_proxy_async_smem();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 8) {
        for (int q = 0; q < iters; ++q) {
            const int s = q % SS, r = q / SS;
            if (r > 0) mbar_wait(&aux.empty[s], (r - 1) & 1);
            if (elect_one()) mbar_arrive(&aux.full[s]);
            __syncwarp();
        }
    } else if (warp == 9) {
        for (int q = 0; q < iters; ++q) {
            const int s = q % SS, t = q % ST;
            if (conv) mbar_wait(&aux.conv[t], (q / ST) & 1);
            else mbar_wait(&aux.full[s], (q / SS) & 1);
            tc_fence_after();
            if (elect_one()) {
                if (mode & 16) {
                    const uint32_t base = (smem_u32(dyn) + 1023u) & ~1023u;
                    constexpr uint32_t IDESC = idesc_tf32(BM, BN, false, true);
                    const uint64_t bd = make_sdesc(base, 4096u, 512u, kLayoutSW128Base32);
                    const uint64_t ad = make_sdesc(base + 65536, 16u, 1024u, kLayoutSW128);
                    for (int i = 0; i < nmma; ++i) {
                        if (mode & 32) mma_tf32_ss(tbase, ad + (i & 3) * 2, bd + (i & 3) * 64, IDESC, i > 0 ? 1u : 0u);
                        else mma_tf32_ts(tbase, tbase + 256 + (i & 3) * 8, bd + (i & 3) * 64, IDESC, i > 0 ? 1u : 0u);
                    }
                }
                if (commit) {
                    mma_commit(&aux.empty[s]);
                    if (conv) mma_commit(&aux.tfree[t]);
                } else {
                    mbar_arrive(&aux.empty[s]);
                    if (conv) mbar_arrive(&aux.tfree[t]);
                }
            }
            __syncwarp();
        }
    } else if (warp >= 10 && warp < 10 + nconvw && conv) {
        for (int q = 0; q < iters; ++q) {
            const int s = q % SS, t = q % ST, rt = q / ST;
            mbar_wait(&aux.full[s], (q / SS) & 1);
            if (rt > 0) mbar_wait(&aux.tfree[t], (rt - 1) & 1);
            tc_fence_after();
            if (fences) {
                tmem_st_wait();
                fence_proxy_async_smem();
                tc_fence_before();
            }
            if (perthread) {
                mbar_arrive(&aux.conv[t]);
            } else {
                __syncwarp();
                if (lane == 0) mbar_arrive(&aux.conv[t]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 9) {
        tc_fence_after();
        tmem_dealloc(tbase, 512);
    }
}

int main(int argc, char** argv) {
    const int iters = argc > 1 ? atoi(argv[1]) : 2657;
    const int only = argc > 2 ? atoi(argv[2]) : -1;  // run only case #only
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int smem = 140 * 1024;
    struct Case { int mode, nmma, bm, bn; };
    const Case cases[] = {{18, 24, 128, 64}, {18, 24, 128, 128}, {18, 24, 128, 256}, {50, 24, 128, 256},
                          {18, 24, 64, 64},  {18, 24, 64, 128},  {18, 24, 64, 256},  {50, 24, 64, 256},
                          {50, 24, 64, 128}, {18, 48, 128, 32}};
    int ci = -1;
    for (const Case& c : cases) {
        if (++ci, only >= 0 && ci != only) continue;
        void (*k)(int, int, int, int) = nullptr;
        if (c.bm == 128 && c.bn == 32) k = ring_kernel<6, 3, 32, 128>;
        if (c.bm == 128 && c.bn == 64) k = ring_kernel<6, 3, 64, 128>;
        if (c.bm == 128 && c.bn == 128) k = ring_kernel<6, 3, 128, 128>;
        if (c.bm == 128 && c.bn == 256) k = ring_kernel<6, 3, 256, 128>;
        if (c.bm == 64 && c.bn == 64) k = ring_kernel<6, 3, 64, 64>;
        if (c.bm == 64 && c.bn == 128) k = ring_kernel<6, 3, 128, 64>;
        if (c.bm == 64 && c.bn == 256) k = ring_kernel<6, 3, 256, 64>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k<<<148, 576, smem>>>(iters, c.mode, 8, c.nmma);
        cudaEventRecord(e0);
        for (int rep = 0; rep < 5; ++rep) k<<<148, 576, smem>>>(iters, c.mode, 8, c.nmma);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaError_t err = cudaGetLastError();
        const double ns = ms / 5 * 1e6 / iters;
        const double flop = 2.0 * c.bm * c.bn * 8 * c.nmma * iters * 148;
        printf("mma=%s M=%d N=%d x%d: %.1f ns per k-block, %.0f TFLOP/s tf32  %s\n", (c.mode & 32) ? "ss" : "ts", c.bm,
               c.bn, c.nmma, ns, flop / (ms / 5 * 1e-3) / 1e12, cudaGetErrorString(err));
    }
    return 0;
}
