// conv_bi.cu -- host-side launcher of the batch-interleaved kernel (conv_bi.cuh):
// builds the TMA tensor map of the input and the kernel arguments.
#include <cudaTypedefs.h>

#include <cmath>

#include "conv_bt.cuh"
#include "conv_bw.cuh"

namespace usc {

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
static PFN_cuTensorMapEncodeTiled_v12000 encode_tiled() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

int launch_bi(const usc_plan *pl, const void *blob, const void *x, void *y, const usc_dev::Epi &ep,
              cudaStream_t st, const usc_act_layout *xv, int step_h, int step_w) {
    // blob = [64 B][int32 blk[G*n_chunks + 1]][int32 perm[G*DT]][int32 rowcls[Yh], colcls[Yw]]
    // [blocks], each part 16-B aligned (usc_pack, kernel 3)
    const char *cb = static_cast<const char *>(blob);
    const long long nb = (long long)pl->groups * pl->n_chunks;
    const long long cp_bytes = (4 * (nb + 1) + 15) / 16 * 16;
    const long long perm_bytes = (4LL * pl->groups * pl->DT + 15) / 16 * 16;
    const int IL = pl->in.interleave;
    if (IL != 32 && IL != 64) return fail(USC_ERR_VALUE, "BI plan needs a 32/64-interleaved input");
    usc_bi::BiArgs a{};
    // x: [Nb][C][Hp][Wp][IL] fp32 or binary16; TMA dims innermost first, box = one chunk's tile
    auto enc = encode_tiled();
    if (!enc) return fail(USC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[5] = {(cuuint64_t)IL, (cuuint64_t)pl->in.ws, (cuuint64_t)pl->in.hp,
                                (cuuint64_t)pl->g.in_channels, (cuuint64_t)((pl->n + IL - 1) / IL)};
    const bool h16 = pl->dtype != USC_F32;  // binary16-staged activations (F16, CB4, I8 codes)
    const cuuint64_t px = (cuuint64_t)IL * (h16 ? 2 : 4);
    // strides of the buffer x lives in: the plan's own layout, or a larger buffer the plan's
    // (hp x ws) input is a window of (usc_conv_forward_view)
    const usc_act_layout &bl = xv ? *xv : pl->in;
    // a strided view (usc_conv_forward_strided) reads every step-th pixel of the buffer
    if (xv && (xv->interleave != IL || (pl->in.hp - 1) * step_h + 1 > xv->hp ||
               (pl->in.ws - 1) * step_w + 1 > xv->ws || xv->channels != pl->g.in_channels))
        return fail(USC_ERR_VALUE, "input view does not fit its buffer layout");
    const cuuint64_t strides[4] = {px * step_w, px * bl.ws * step_h, px * bl.ws * bl.hp,
                                   (cuuint64_t)bl.sample_stride * (px / IL)};
    const cuuint32_t box[5] = {(cuuint32_t)IL, (cuuint32_t)pl->TWs, (cuuint32_t)pl->HS, (cuuint32_t)pl->CC, 1};
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = enc(&a.xmap, h16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<void *>(x), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(USC_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    a.y = y;
    a.blk = reinterpret_cast<const int *>(cb + 64);
    a.perm = reinterpret_cast<const int *>(cb + 64 + cp_bytes);
    const long long ctab_bytes = (4LL * (pl->out_h + pl->out_w) + 15) / 16 * 16;
    a.rowcls = reinterpret_cast<const int *>(cb + 64 + cp_bytes + perm_bytes);
    a.colcls = a.rowcls + pl->out_h;
    a.ncls_c = pl->ncls_c > 0 ? pl->ncls_c : 1;
    a.ncls = (pl->ncls_r > 0 ? pl->ncls_r : 1) * a.ncls_c;
    a.blocks = cb + 64 + cp_bytes + perm_bytes + ctab_bytes;
    a.N = pl->n;
    a.D = pl->g.out_channels;
    a.n_chunks = pl->n_chunks;
    a.CC = pl->CC;
    a.DT = pl->DT;
    a.HS = pl->HS;
    a.TWs = pl->TWs;
    a.Yh = pl->out_h;
    a.Yw = pl->out_w;
    a.s_h = pl->g.stride_h;
    a.WS = pl->WS;
    a.WC = pl->WC;
    a.SPRt = pl->SPRt;
    a.TH = pl->TH;
    a.row_tiles = pl->row_tiles;
    a.col_tiles = pl->col_tiles;
    a.G = pl->groups;
    a.tiles = pl->groups * pl->sample_tiles * pl->row_tiles * pl->col_tiles;
    a.S = pl->stages;
    // tail split chosen by the planner (usc_plan_make): tiles [0, tail_full) whole,
    // the rest as tail_split slot-subset items each
    a.split = pl->tail_split > 1 ? pl->tail_split : 1;
    a.tfull = a.split > 1 ? pl->tail_full : a.tiles;
    a.items = a.tfull + a.split * (a.tiles - a.tfull);
    a.fG = usc_bi::fdiv_make(static_cast<uint32_t>(a.G));
    a.fCT = usc_bi::fdiv_make(static_cast<uint32_t>(a.col_tiles));
    a.fRT = usc_bi::fdiv_make(static_cast<uint32_t>(a.row_tiles));
    a.x_stage_bytes = static_cast<int>(pl->smem_stage_bytes);
    a.stage_bytes = static_cast<int>(pl->smem_stage_bytes + pl->ent_stage_bytes);
    a.ep = ep;
    a.fast = (pl->dtype == USC_F32 || pl->dtype == USC_F16) && !ep.saturate && !ep.saturate2 && !ep.requant &&
             ep.out_padded && ep.oil == pl->in.interleave && (!ep.residual || ep.ril == pl->in.interleave) &&
             (ep.relu || !ep.pool);
    if (pl->dtype == USC_I8 && ep.requant && ep.relu && !ep.saturate && !ep.saturate2 && !ep.residual &&
        ep.out_padded && ep.oil == pl->in.interleave) {
        // the integer requantisation needs both scales to be powers of two (fixed-point sigmas)
        int e1, e2;
        const float m1 = std::frexp(ep.scale, &e1), m2 = std::frexp(ep.rq_scale, &e2);
        if (m1 == 0.5f && m2 == 0.5f) {
            a.fast = 1;
            a.i8shift = -((e1 - 1) + (e2 - 1));
        }
    }
    if (pl->dtype == USC_CB4 && !ep.requant && !ep.residual && ep.out_padded && ep.oil == pl->in.interleave &&
        (ep.relu || !ep.pool))
        a.fast = 1;  // the 4b/16b hook with its saturations (store_tile_fast)
    if (pl->kernel == 4) return usc_bi::launch_bt(pl, a, st);
    if (pl->window) return usc_bi::launch_bw(pl, a, st);
    if (pl->dtype == USC_F16) return usc_bi::launch_h16(pl, a, st);
    if (pl->dtype == USC_CB4) return usc_bi::launch_hcb(pl, a, st);
    if (pl->dtype == USC_I8) return usc_bi::launch_hi8(pl, a, st);
    switch (pl->threads) {
        case 256: return usc_bi::launch_w8(pl, a, st);
        case 384: return usc_bi::launch_w12(pl, a, st);
        default: return usc_bi::launch_w16(pl, a, st);
    }
}

}  // namespace usc
