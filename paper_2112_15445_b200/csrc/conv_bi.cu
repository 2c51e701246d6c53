// conv_bi.cu -- host-side launcher of the batch-interleaved kernel (conv_bi.cuh).
#include "conv_bi.cuh"

namespace usc {

int launch_bi(const usc_plan *pl, const void *blob, const void *x, void *y, const usc_dev::Epi &ep,
              cudaStream_t st) {
    // blob = [64 B][int32 blk[G*n_chunks + 1]][int32 perm[G*DT]][blocks], each part 16-B
    // aligned (usc_pack, kernel 3)
    const char *cb = static_cast<const char *>(blob);
    const long long nb = (long long)pl->groups * pl->n_chunks;
    const long long cp_bytes = (4 * (nb + 1) + 15) / 16 * 16;
    usc_bi::BiArgs a{};
    a.x = static_cast<const float *>(x);
    a.y = static_cast<float *>(y);
    const long long perm_bytes = (4LL * pl->groups * pl->DT + 15) / 16 * 16;
    a.blk = reinterpret_cast<const int *>(cb + 64);
    a.perm = reinterpret_cast<const int *>(cb + 64 + cp_bytes);
    a.blocks = cb + 64 + cp_bytes + perm_bytes;
    a.N = pl->n;
    a.C = pl->g.in_channels;
    a.D = pl->g.out_channels;
    a.n_chunks = pl->n_chunks;
    a.CC = pl->CC;
    a.DT = pl->DT;
    a.HS = pl->HS;
    a.TWs = pl->TWs;
    a.Hp = pl->in.hp;
    a.Wp = pl->in.ws;
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
    a.full_rows = (pl->col_tiles == 1 && pl->TWs == pl->in.ws) ? 1 : 0;
    a.x_blk_stride = pl->in.sample_stride;
    a.x_stage_bytes = static_cast<int>(pl->smem_stage_bytes);
    a.stage_bytes = static_cast<int>(pl->smem_stage_bytes + pl->ent_stage_bytes);
    a.ep = ep;
    switch (pl->threads) {
        case 256: return usc_bi::launch_w8(pl, a, st);
        case 384: return usc_bi::launch_w12(pl, a, st);
        default: return usc_bi::launch_w16(pl, a, st);
    }
}

}  // namespace usc
