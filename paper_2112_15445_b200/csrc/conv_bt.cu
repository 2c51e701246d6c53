// conv_bt.cu -- k_bt instances (tensor-memory-fed fp32 BI64, bi_instances.h USC_BT).
#include "bi_instances.h"
#include "conv_bt.cuh"

namespace usc_bi {
int launch_bt(const usc_plan *pl, const BiArgs &a, cudaStream_t st) {
    const int nw = pl->threads / 32;
#define X(NW_, PC_, PR_, DW_)                                                                          \
    if (nw == NW_ && pl->PC == PC_ && pl->PR == PR_ && pl->DW == DW_) return launch_bt_inst<PC_, PR_, DW_, NW_>(pl, a, st);
    USC_BT(X)
#undef X
    return usc::fail(USC_ERR_UNSUPPORTED, "no k_bt instance for %d warps PC=%d PR=%d DW=%d", nw, pl->PC, pl->PR,
                     pl->DW);
}
}  // namespace usc_bi
