// conv_bi16r2.cu -- k_bi instances, 16 compute warps, 2-row pixel blocks (fused-pool capable).
#include "conv_bi.cuh"

namespace usc_bi {
int launch_16r2(const usc_plan *pl, const BiArgs &a, cudaStream_t st) {
    return launch_rows2<1, 16, 1>(pl, a, st);
}
}  // namespace usc_bi
