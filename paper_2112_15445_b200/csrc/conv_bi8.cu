// conv_bi8.cu -- k_bi instances, 8 compute warps + 1 producer warp, 2 CTAs/SM.
#include "conv_bi.cuh"

namespace usc_bi {
int launch_8(const usc_plan *pl, const BiArgs &a, cudaStream_t st) {
    return pl->g.stride_w == 1 ? launch_rows1<1, 8, 2>(pl, a, st) : launch_rows1<2, 8, 2>(pl, a, st);
}
}  // namespace usc_bi
