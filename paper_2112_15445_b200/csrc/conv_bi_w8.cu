// conv_bi_w8.cu -- k_bi instances with 8 compute warps + 1 producer warp (bi_instances.h).
#include "bi_instances.h"
#include "conv_bi.cuh"

namespace usc_bi {
int launch_w8(const usc_plan *pl, const BiArgs &a, cudaStream_t st) {
    const int spl = pl->in.interleave / 32;
#define X(PC_, PR_, DW_, SW_, SPL_)                                                                 \
    if (pl->PC == PC_ && pl->PR == PR_ && pl->DW == DW_ && pl->g.stride_w == SW_ && spl == SPL_) \
        return launch_inst<USC_F32, PC_, PR_, DW_, SW_, 8, SPL_>(pl, a, st);
    USC_BI_W8(X)
#undef X
    return usc::fail(USC_ERR_UNSUPPORTED, "no k_bi instance for %d warps PC=%d PR=%d DW=%d SW=%d SPL=%d", 8,
                     pl->PC, pl->PR, pl->DW, pl->g.stride_w, spl);
}
}  // namespace usc_bi
