// launch.cuh — every kernel of the library is launched through launch_k(): cudaLaunchKernelEx with
// (optionally) a thread-block-cluster shape and PROGRAMMATIC DEPENDENT LAUNCH (PDL).
//
// Why PDL: the small-map layers (VGG-16 at batch 128: 2x2..8x8 maps, ~40 kernels per step) run
// 10-40 us kernels whose CTAs spend ~4 us before their first TMA load (barrier init, TMEM alloc,
// tensor-map prefetch, work-item bookkeeping; smconv_set_trace) plus ~2 us of launch
// gap.  With programmaticStreamSerializationAllowed the next kernel of the stream may be scheduled
// as soon as every CTA of the current one has executed `griddepcontrol.launch_dependents`
// (pdl_trigger, first thing in every kernel): its CTAs take SMs as the current kernel's CTAs retire
// and run their set-up there.  Correctness does not depend on the trigger's placement: every kernel
// executes `griddepcontrol.wait` (pdl_wait) before its first global-memory access, which blocks
// until all prerequisite grids have COMPLETED and their memory operations are visible.  A kernel
// launched without the attribute (SMCONV_PDL=0, or after a non-PDL predecessor) waits for nothing.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace smconv {

// SMCONV_PDL: 0 = never, 1 = auto (default): calls whose plan runs plain TF32 MMAs, 2 = always.
// Measured on VGG-16 b128 (r02p, 2 runs each): TF32 step 1.080 -> 0.991 ms with PDL, but 3xTF32
// 1.628 -> 1.697 ms and ResNet-18 b4096 3xTF32 57.5 -> 58.7 ms, so "auto" leaves 3xTF32 calls without.
inline int pdl_mode() {
    static const int m = getenv("SMCONV_PDL") ? atoi(getenv("SMCONV_PDL")) : 1;
    return m;
}
// set by the C-ABI entry for the kernels of the current call (thread-local: calls on other host threads
// are independent)
inline bool& pdl_this_call() {
    static thread_local bool on = false;
    return on;
}
inline bool pdl_enabled() { return pdl_this_call(); }

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int cluster,
                     Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int n = 0;
    if (cluster > 1) {
        at[n].id = cudaLaunchAttributeClusterDimension;
        at[n].val.clusterDim.x = cluster;
        at[n].val.clusterDim.y = 1;
        at[n].val.clusterDim.z = 1;
        ++n;
    }
    if (pdl_enabled()) {
        at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    cfg.attrs = at;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace smconv
