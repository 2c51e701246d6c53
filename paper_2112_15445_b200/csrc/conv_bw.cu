// conv_bw.cu -- k_bw instances (register-window batch-interleaved kernel, conv_bw.cuh).
#include "bi_instances.h"
#include "conv_bw.cuh"

namespace usc_bi {
int launch_bw(const usc_plan *pl, const BiArgs &a, cudaStream_t st) {
    const int fam = pl->dtype == USC_F32 ? 0 : (pl->dtype == USC_F16 ? 1 : -1);
    const int nw = pl->threads / 32, kw = pl->g.filter_w;
#define X(F_, NW_, PC_, DW_, KW_)                                                                   \
    if (fam == F_ && nw == NW_ && pl->PC == PC_ && pl->DW == DW_ && kw == KW_)                      \
        return launch_bw_inst < F_ == 0 ? USC_F32 : USC_F16, PC_, DW_, KW_, NW_ > (pl, a, st);
    USC_BW(X)
#undef X
    return usc::fail(USC_ERR_UNSUPPORTED, "no k_bw instance for dtype %d, %d warps PC=%d DW=%d KW=%d", pl->dtype,
                     nw, pl->PC, pl->DW, kw);
}
}  // namespace usc_bi
