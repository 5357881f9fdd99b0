// probe.cu — TEST-ONLY precision probe for tcgen05.mma.kind::tf32.
//
// Runs 1-2 MMAs of shape M=128, N=32, K=8 on hand-built operands and writes D[i][0] for
// rows i = 0..15 of three experiments to out[mode*16 + i]:
//
//  mode 0  operand conversion: D = a_i * 1 (one MMA, accumulate off)
//          a_0 = 1+2^-11 (tie)          RNE->1        RNA->1+2^-10   trunc->1
//          a_1 = 1+2^-11+2^-20          RN ->1+2^-10                 trunc->1
//          a_2 = 1+3*2^-11 (tie, odd)   RNE->1+2^-9   RNA->1+2^-9    trunc->1+2^-10
//          a_3 = 1+2^-12                RN ->1                       trunc->1
//          a_4 = -(1+2^-11+2^-20)       RN ->-(1+2^-10)              trunc->-1
//  mode 1  accumulator rounding across MMAs: D = 1 (first MMA), then D += d_i (second MMA)
//          d_0 = 0.75 ulp(1)  RN->1+2^-23  RZ->1
//          d_1 = 0.25 ulp(1)  RN->1        RZ->1
//          d_2 = 0.5 ulp(1)   RNE->1       RNA->1+2^-23
//          d_3 = -0.125 ulp(1) RN->1       RZ->1-2^-24
//          d_4 = 1.75 ulp(1)  RN->1+2^-22  RZ->1+2^-23
//  mode 2  the same sums inside ONE MMA: A row i = [1, d_i, 0...], B col 0 = [1, 1, 0...]
#include <cstdio>
#include "common.cuh"
#include "../../include/smconv_ext.h"

namespace smconv {

__global__ void __launch_bounds__(128, 1) probe_tf32_kernel(float* out, int mode) {
    __shared__ __align__(1024) uint8_t sA[128 * 128];  // K-major [128 rows][32 k]
    __shared__ __align__(1024) uint8_t sB[32 * 128];   // K-major [32 rows][32 k]
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    float* a = reinterpret_cast<float*>(sA);
    float* b = reinterpret_cast<float*>(sB);
    for (int i = tid; i < 128 * 32; i += 128) a[i] = 0.f;
    for (int i = tid; i < 32 * 32; i += 128) b[i] = 0.f;
    __syncthreads();
    const float u = 1.1920928955078125e-07f;  // 2^-23 = ulp(1)
    auto A = [&](int r, int k, float v) { a[kmaj_off(r, k >> 2) / 4 + (k & 3)] = v; };
    auto B = [&](int r, int k, float v) { b[kmaj_off(r, k >> 2) / 4 + (k & 3)] = v; };
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
        if (mode == 0) {
            A(0, 0, 1.f + 0x1p-11f);
            A(1, 0, 1.f + 0x1p-11f + 0x1p-20f);
            A(2, 0, 1.f + 3.f * 0x1p-11f);
            A(3, 0, 1.f + 0x1p-12f);
            A(4, 0, -(1.f + 0x1p-11f + 0x1p-20f));
            B(0, 0, 1.f);
        } else if (mode == 1) {
            for (int r = 0; r < 8; ++r) A(r, 0, 1.f);
            B(0, 0, 1.f);
        } else {
            const float d[5] = {0.75f * u, 0.25f * u, 0.5f * u, -0.125f * u, 1.75f * u};
            for (int r = 0; r < 5; ++r) {
                A(r, 0, 1.f);
                A(r, 1, d[r]);
            }
            B(0, 0, 1.f);
            B(0, 1, 1.f);
        }
    }
    fence_proxy_async_smem();
    if (warp == 0) tmem_alloc(&tbase, 32);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tbase;
    constexpr uint32_t IDESC = idesc_tf32(128, 32, false, false);
    if (tid == 0) {
        mma_tf32_ss(tmem, make_sdesc_sw128(smem_u32(sA), 16, 1024), make_sdesc_sw128(smem_u32(sB), 16, 1024), IDESC, 0);
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    if (mode == 1) {
        __syncthreads();
        if (tid == 0) {
            const float d[5] = {0.75f * u, 0.25f * u, 0.5f * u, -0.125f * u, 1.75f * u};
            for (int r = 0; r < 5; ++r) A(r, 0, d[r]);
            fence_proxy_async_smem();
            tc_fence_after();
            mma_tf32_ss(tmem, make_sdesc_sw128(smem_u32(sA), 16, 1024), make_sdesc_sw128(smem_u32(sB), 16, 1024), IDESC, 1);
            mma_commit(&bar);
        }
        mbar_wait(&bar, 1);
    }
    tc_fence_after();
    uint32_t v[16];
    tmem_ld_32x32b_x16(tmem + ((uint32_t)(warp * 32) << 16), v);
    tmem_ld_wait();
    if (warp == 0 && lane < 16) out[mode * 16 + lane] = __uint_as_float(v[0]);
    // also report D[0][1..15] (must be 0) in the slots after the 3 modes
    if (warp == 0 && lane == 0 && mode == 0)
        for (int j = 1; j < 16; ++j) out[48 + j] = __uint_as_float(v[j]);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 32);
    }
}

}  // namespace smconv

extern "C" int smconv_probe_tf32(float* out) {
    for (int mode = 0; mode < 3; ++mode) {
        smconv::probe_tf32_kernel<<<1, 128>>>(out, mode);
        if (cudaGetLastError() != cudaSuccess) return CONV_ECUDA;
    }
    return cudaDeviceSynchronize() == cudaSuccess ? CONV_OK : CONV_ECUDA;
}
