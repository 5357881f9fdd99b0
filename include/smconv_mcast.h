/*
 * smconv_mcast.h — the weight gradient fused with its data-parallel all-reduce.
 *
 * In batch-sharded data parallelism (north_star item (e)) dW is a sum over images, so
 * every rank needs dW = sum over ranks of its shard's dW (reading L10: SUM).  The plain path computes
 * the shard's dW (conv2d_bwd_filter) and then all-reduces the flat dW buffer with NCCL.  Here the dW
 * kernel itself performs the all-reduce through an NVLink multicast (NVLS) object: where the plan's
 * last kernel would store a dW element it instead issues `multimem.red.relaxed.sys.global.add.f32`
 * (.v4) on the multicast address, and the NVSwitch adds the value into the copy of EVERY rank bound to
 * the object.  That is the TMA dW epilogue itself when the plan has one split (the whole reduction in
 * one pass: no dW store, no NCCL pass), otherwise the deterministic split-K reduce kernel (its fixed-order
 * sum goes to the switch instead of to local memory: no separate NCCL pass).
 *
 *   int conv2d_bwd_filter_mcast(X, dY, dW_mc, N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw, math, ws, ws_bytes,
 *                               stream);
 *     X, dY       this rank's shard, as conv2d_bwd_filter (device pointers, NHWC, 16-B aligned)
 *     dW_mc       the MULTICAST virtual address of a [OC,FH,FW,IC] fp32 buffer bound on every rank of the
 *                 group (cuMulticastCreate + cuMulticastBindMem + cuMemMap, or torch symmetric memory's
 *                 multicast_ptr), 16-B aligned
 *     ws          conv2d_bwd_filter_mcast_workspace_bytes(...) device bytes
 *   Contract (caller): every rank's copy is zero before ANY rank's call starts adding into it, and no rank
 *   reads dW before EVERY rank's call has completed (a device- or host-side barrier across the ranks on
 *   both sides, e.g. the symmetric-memory barrier).  The call only adds: calling it for several
 *   micro-batches accumulates them.
 *   Determinism: each rank's contribution is computed in a fixed order, but the order in which the switch
 *   adds the ranks' contributions (and, for TMA plans with one split, nothing else) is not fixed, so
 *   results are reproducible only up to fp32 rounding of the cross-rank sum — unlike the NCCL path
 *   (contract 6 of smconv.h holds per rank).  Integer-valued inputs (pin P7) stay bit-exact.
 *   Errors: those of conv2d_bwd_filter (CONV_* codes, conv2d_last_error_detail names this entry point).
 */
#ifndef SMCONV_MCAST_H
#define SMCONV_MCAST_H

#include <stddef.h>

#include "smconv.h"

#ifdef __cplusplus
extern "C" {
#endif

size_t conv2d_bwd_filter_mcast_workspace_bytes(int N, int IH, int IW, int IC, int OC, int FH, int FW, int sh, int sw,
                                               int ph, int pw, int math);

int conv2d_bwd_filter_mcast(const float* X, const float* dY, float* dW_mc, int N, int IH, int IW, int IC, int OC,
                            int FH, int FW, int sh, int sw, int ph, int pw, int math, void* workspace,
                            size_t workspace_bytes, conv_stream_t stream);

/* Test hook: "variant=.. BN=.. splits=.. mcast=epilogue|reduce ws=.. kernels=..". */
int conv2d_bwd_filter_mcast_plan_describe(int N, int IH, int IW, int IC, int OC, int FH, int FW, int sh, int sw,
                                          int ph, int pw, int math, char* buf, size_t len);

#ifdef __cplusplus
}
#endif

#endif
