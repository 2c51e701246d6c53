// conv_bi16.cu -- k_bi instances, 16 compute warps + 1 producer warp, 1 CTA/SM, 1-row pixel blocks.
#include "conv_bi.cuh"

namespace usc_bi {
int launch_16(const usc_plan *pl, const BiArgs &a, cudaStream_t st) {
    if (pl->PR == 2) return launch_16r2(pl, a, st);
    return pl->g.stride_w == 1 ? launch_rows1<1, 16, 1>(pl, a, st) : launch_rows1<2, 16, 1>(pl, a, st);
}
}  // namespace usc_bi
