/*
 * smconv_ext.h — introspection and test hooks of libsmconv (not needed by ordinary callers).
 *
 * SPEC.md:48-51 gives the conv descriptor an `algorithm` override
 * {auto, general_im2col, small_feature_direct} and SPEC.md:247,843 require the
 * paths to be equivalent on shapes straddling the small-map threshold
 * ("smaller than a certain threshold").  Here the override selects a
 * kernel family of this library; the equivalence is tested in tests/.
 */
#ifndef SMCONV_EXT_H
#define SMCONV_EXT_H

#include <stddef.h>
#include "smconv.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Kernel families ("variants").  AUTO = the heuristic table's choice. */
enum {
    CONV_VARIANT_AUTO = 0,
    CONV_VARIANT_GENERIC = 1,   /* register-staged implicit GEMM: any IC%4 / OC%4, any geometry */
    CONV_VARIANT_TMA = 2,       /* TMA-staged implicit GEMM: channel extents multiple of 32 */
    CONV_VARIANT_STRIP = 3,     /* TMA strips with input-slab reuse across filter columns:
                                   stride-1 3-wide fwd / dX, BN <= 128 (TF32) / 64 (3xTF32) */
    CONV_VARIANT_DIRECT = 4,    /* CUDA-core fp32 direct conv for few-channel (IC <= 8) stems, fwd / dW */
    CONV_VARIANT_DWS = 5,       /* dW of 3x3 s1 64->64 convs on 8/16/32-wide maps: one activation slab
                                   per k-block shared by 4 taps (shift applied by the TF32 split stage) */
    CONV_VARIANT_STEM = 6       /* the IC = 4 (padded RGB) 3x3 stems on the tensor cores: fwd with the
                                   IM2COL rows written into TMEM and a TMA-store epilogue (OC 64/128/192),
                                   dW with dY by TMA and per-CTA partials (any OC % 4 == 0) */
};

/* Force a variant for all subsequent calls of `op` in this process (thread-safe);
 * CONV_VARIANT_AUTO restores the heuristic.  The environment variable
 * SMCONV_FORCE_VARIANT="<op>:<variant>[,...]" is read once at load time.
 * Returns CONV_EARG for an unknown op/variant. */
int conv2d_force_variant(int op, int variant);

/* CTA pairs (tcgen05 cta_group::2, M = 256 tiles, B split across the pair), 3xTF32 only: the TMA
 * variant's fwd / dX when N % 256 == 0 and dW when OC % 256 == 0, and the STRIP variant at BN 64 when
 * N % 64 == 0.  1 = on (default; SMCONV_PAIR=0 at load time turns it off), 0 = off.  Results are
 * identical in both modes up to summation order (parity-tested in both).  DESIGN.md §6 / §9: pairs
 * won once the peer arrivals stopped emitting MEMBAR.ALL.GPU (ResNet-18 b4096 step 62.4 -> 59.1 ms,
 * dW pairs -> 57.5 ms).  Returns the previous value. */
int smconv_set_pair(int on);

/* 3xTF32 fwd / dX on the TMA variant: calls with less than `gflop` GFLOP of valid-tap work run three
 * TF32 MMAs per product with b_lo split in the kernel ("3mma" in the plan text) instead of the hybrid
 * form (a_hi*b_hi TF32 + the cross terms as one K-doubled bf16 MMA on a W' plane that a separate
 * wx_prep kernel builds per call).  Default 12 (SMCONV_HYB_MIN_GFLOP at load time); 0 = always hybrid.
 * Clears the plan cache.  Returns the previous value. */
double smconv_set_hybrid_min_gflop(double gflop);

/* Plan the call would use, as text: "variant=.. BN=.. splits=.. tiles=.. kernels=..".
 * Returns CONV_OK and writes at most `len` bytes (NUL-terminated) into `buf`. */
int conv2d_plan_describe(int op, int N, int IH, int IW, int IC, int OC, int FH, int FW,
                         int sh, int sw, int ph, int pw, int math, char* buf, size_t len);

/* Number of kernels one call with these arguments enqueues (for bench gpu_launches). */
int conv2d_plan_kernels(int op, int N, int IH, int IW, int IC, int OC, int FH, int FW,
                        int sh, int sw, int ph, int pw, int math);

/* EXPERIMENT hook: when device_buf != NULL (>= 16 * grid u64, device memory), the TMA-variant kernels
 * write per-CTA phase timestamps (clock64; slot 15 = globaltimer at entry) into it: 0 entry, 1 setup
 * done, 2 first TMA issue, 4 first MMA issue, 5 last MMA commit, 6 accumulator ready (epilogue),
 * 7 epilogue done, 8 CTA barrier, 9/10 cluster split-K reduce start/end, 11 exit.  NULL (default) = off. */
int smconv_set_trace(void* device_buf);

/* Host-only self test of the library's index arithmetic (fast division); 0 = pass. */
int smconv_selftest_host(void);

/* TEST-ONLY precision probe: runs tiny tcgen05.mma.kind::tf32
 * problems whose results reveal how the tensor core rounds fp32 operands to TF32 and
 * how it rounds accumulation.  `out` is a device buffer of >= 64 floats; results are
 * documented in csrc/probe.cu.  Synchronous. */
int smconv_probe_tf32(float* out);

#ifdef __cplusplus
}
#endif
#endif
