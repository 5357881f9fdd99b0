// conv_tma.cuh — TMA variant (placeholder until implemented; never selected).
#pragma once
#include "conv_gen.cuh"

namespace smconv {

struct TmaParams {
    int dummy;
};

inline bool tma_supported(int, int, int, int, int, int, int, int) { return false; }

inline int tma_make_plan(int, const GenParams&, int, int, TmaParams&, dim3&, char*, size_t) { return 5; }

inline int tma_launch(int, int, int, const GenParams&, TmaParams&, dim3, cudaStream_t, char*, size_t) { return 5; }

}  // namespace smconv
