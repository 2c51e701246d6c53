// conv_bi_hi8.cu -- k_bi instances for USC_I8 (binary16-staged activations, BI64; bi_instances.h).
#include "bi_instances.h"
#include "conv_bi.cuh"

namespace usc_bi {
int launch_hi8(const usc_plan *pl, const BiArgs &a, cudaStream_t st) {
    const int nw = pl->threads / 32;
    if (pl->in.interleave != 64) return usc::fail(USC_ERR_UNSUPPORTED, "binary16-staged BI kernels need BI64");
#define X(NW_, PC_, PR_, DW_, SW_)                                                               \
    if (nw == NW_ && pl->PC == PC_ && pl->PR == PR_ && pl->DW == DW_ && pl->g.stride_w == SW_) \
        return launch_inst<USC_I8, PC_, PR_, DW_, SW_, NW_, 2>(pl, a, st);
    USC_BI_H(X)
#undef X
    return usc::fail(USC_ERR_UNSUPPORTED, "no USC_I8 k_bi instance for %d warps PC=%d PR=%d DW=%d SW=%d", nw,
                     pl->PC, pl->PR, pl->DW, pl->g.stride_w);
}
}  // namespace usc_bi
