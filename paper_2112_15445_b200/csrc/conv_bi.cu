// conv_bi.cu -- the batch-interleaved fp32 direct sparse conv kernel (sm_100a).
//
// Replaces the reference's hot loop kernels.sparse_conv_blocks
// (/root/reference/pkg/src/unsparse/kernels.py:57-100) for BINARY32.
//
// Layout: activations are BI32 ([n/32][C][Hp][Wp][32], zero halo): the 32 lanes
// of a warp are 32 samples, so for a given (pixel, tap) every shared-memory load
// is one conflict-free 128-byte wavefront and every output store is one
// coalesced 128-byte line.
//
// CTA = one 32-sample block x a tile of WS strips (P consecutive output pixels of
// a row) x DT = WC*DW output channels.  Warp w owns strip w % WS for the DW
// channels of subgroup w / WS; it keeps DW*P fp32 accumulators per lane for the
// whole input-channel loop.  Input channels are staged CC at a time into a
// double-buffered [CC][HS][TWs][32] tile by bulk-async copies (UBLKCP, the TMA
// engine) issued by one thread and completed on an mbarrier.
//
// Per output element the arithmetic is the reference's: stored-order entries
// (ascending (c, kh, kw)), IEEE fp32 multiply then add (__fmul_rn/__fadd_rn),
// so results are bit-identical to the reference for every tile configuration.
#include "common.cuh"

namespace {
using namespace usc_dev;

struct BiArgs {
    const float *x;
    float *y;
    const int *cpg;
    const int2 *ents;
    int N, C, D, n_chunks, CC, DT;
    int HS, TWs, Hp, Wp, Yh, Yw, s_h;
    int WS, WC, SPRt, TH, row_tiles, col_tiles, G;
    int full_rows;
    long long x_blk_stride;  // elements per 32-sample block
    int stage_words;
    Epi ep;
};

template <int P, int DW, int SW>
__global__ void __launch_bounds__(256) k_bi(const BiArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
    float *stage0 = reinterpret_cast<float *>(smem + 128);
    float *stage1 = stage0 + a.stage_words;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int cta = blockIdx.x;
    const int g = cta % a.G;  // channel group fastest: CTAs sharing an input tile run together
    cta /= a.G;
    const int ct = cta % a.col_tiles;
    cta /= a.col_tiles;
    const int rt = cta % a.row_tiles;
    const int sb = cta / a.row_tiles;
    const int r0 = rt * a.TH, cs0 = ct * a.SPRt;
    const int y0 = r0 * a.s_h;
    const int x0 = cs0 * P * SW;
    const int rows = min(a.HS, a.Hp - y0);
    const int wsi = warp % a.WS, wc = warp / a.WS;
    const bool active = wc < a.WC;
    const int tr = wsi / a.SPRt, tcs = wsi - tr * a.SPRt;
    const int r = r0 + tr;
    const int col0 = (cs0 + tcs) * P;
    const int base = ((tr * a.s_h) * a.TWs + tcs * P * SW) * 32 + lane;

    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const float *xblk = a.x + (long long)sb * a.x_blk_stride;
    auto issue = [&](int k, int s) {
        const int c0 = k * a.CC;
        const int cc = min(a.CC, a.C - c0);
        float *dst = s ? stage1 : stage0;
        const int plane_words = a.HS * a.TWs * 32;
        if (a.full_rows) {
            if (y0 == 0 && rows == a.Hp && a.HS == a.Hp) {
                const uint32_t bytes = static_cast<uint32_t>(cc) * a.Hp * a.Wp * 128u;
                mbar_expect_tx(&bar[s], bytes);
                bulk_g2s(dst, xblk + (long long)c0 * a.Hp * a.Wp * 32, bytes, &bar[s]);
            } else {
                const uint32_t bytes = static_cast<uint32_t>(rows) * a.Wp * 128u;
                mbar_expect_tx(&bar[s], bytes * cc);
                for (int c = 0; c < cc; ++c)
                    bulk_g2s(dst + c * plane_words,
                             xblk + (((long long)(c0 + c) * a.Hp + y0) * a.Wp) * 32, bytes, &bar[s]);
            }
        } else {
            const int w = min(a.TWs, a.Wp - x0);
            const uint32_t bytes = static_cast<uint32_t>(w) * 128u;
            mbar_expect_tx(&bar[s], bytes * cc * rows);
            for (int c = 0; c < cc; ++c)
                for (int rr = 0; rr < rows; ++rr)
                    bulk_g2s(dst + c * plane_words + rr * a.TWs * 32,
                             xblk + ((((long long)(c0 + c) * a.Hp + y0 + rr) * a.Wp) + x0) * 32, bytes,
                             &bar[s]);
        }
    };
    if (tid == 0) {
        issue(0, 0);
        if (a.n_chunks > 1) issue(1, 1);
    }

    float acc[DW][P];
#pragma unroll
    for (int i = 0; i < DW; ++i)
#pragma unroll
        for (int p = 0; p < P; ++p) acc[i][p] = 0.0f;

    // chunk boundaries of this warp's DW channels: lanes 0..DW hold them
    const int *cp = a.cpg + (long long)g * a.n_chunks * a.DT + wc * DW;
    int bnd = (active && lane <= DW) ? __ldg(cp + lane) : 0;
    for (int k = 0; k < a.n_chunks; ++k) {
        const int s = k & 1;
        const int bnd_cur = bnd;
        if (active && lane <= DW && k + 1 < a.n_chunks) bnd = __ldg(cp + (k + 1) * a.DT + lane);
        mbar_wait(&bar[s], (k >> 1) & 1);
        if (active) {
            const float *xs = (s ? stage1 : stage0) + base;
#pragma unroll
            for (int dw = 0; dw < DW; ++dw) {
                const int e0 = __shfl_sync(0xffffffffu, bnd_cur, dw);
                const int e1 = __shfl_sync(0xffffffffu, bnd_cur, dw + 1);
                if (e0 < e1) {
                    int2 en = __ldg(a.ents + e0);
                    for (int e = e0; e < e1; ++e) {
                        const int2 nx = __ldg(a.ents + min(e + 1, e1 - 1));
                        const float th = __int_as_float(en.y);
                        const float *xp = xs + en.x;
                        float v[P];
#pragma unroll
                        for (int p = 0; p < P; ++p) v[p] = xp[p * SW * 32];
#pragma unroll
                        for (int p = 0; p < P; ++p) acc[dw][p] = __fadd_rn(acc[dw][p], __fmul_rn(th, v[p]));
                        en = nx;
                    }
                }
            }
        }
        __syncthreads();
        if (tid == 0 && k + 2 < a.n_chunks) {
            fence_proxy_async();
            issue(k + 2, s);
        }
    }

    const int b = sb * 32 + lane;
    if (!active || b >= a.N || r >= a.Yh) return;
#pragma unroll
    for (int dw = 0; dw < DW; ++dw) {
        const int d = g * a.DT + wc * DW + dw;
        if (d >= a.D) break;
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const int col = col0 + p;
            if (col >= a.Yw) break;
            float v = acc[dw][p];
            if (a.ep.relu) v = v > 0.0f ? v : 0.0f;
            long long idx;
            if (!a.ep.out_padded)
                idx = (((long long)b * a.D + d) * a.Yh + r) * a.Yw + col;
            else if (a.ep.oil == 32)
                idx = (long long)sb * a.ep.o_sample_stride +
                      ((((long long)d * a.ep.oHp + r + a.ep.oph) * a.ep.oWs + col + a.ep.opw) << 5) + lane;
            else
                idx = (long long)b * a.ep.o_sample_stride +
                      ((long long)d * a.ep.oHp + r + a.ep.oph) * a.ep.oWs + col + a.ep.opw;
            a.y[idx] = v;
        }
    }
}

template <int P, int DW, int SW>
int launch_inst(const usc_plan *pl, const BiArgs &a, cudaStream_t st) {
    auto fn = k_bi<P, DW, SW>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        attr = true;
    }
    fn<<<static_cast<unsigned>(pl->grid_x), 256, pl->smem_bytes, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return usc::fail(USC_ERR_CUDA, "k_bi launch: %s", cudaGetErrorString(e));
    return USC_OK;
}

template <int P, int DW>
int launch_sw(const usc_plan *pl, const BiArgs &a, cudaStream_t st) {
    return pl->g.stride_w == 1 ? launch_inst<P, DW, 1>(pl, a, st) : launch_inst<P, DW, 2>(pl, a, st);
}

template <int P>
int launch_dw(const usc_plan *pl, const BiArgs &a, cudaStream_t st) {
    switch (pl->DW) {
        case 4: return launch_sw<P, 4>(pl, a, st);
        case 8: return launch_sw<P, 8>(pl, a, st);
        default: return launch_sw<P, 16>(pl, a, st);
    }
}

}  // namespace

namespace usc {

int launch_bi(const usc_plan *pl, const void *blob, const void *x, void *y, const usc_dev::Epi &ep,
              cudaStream_t st) {
    const char *cb = static_cast<const char *>(blob);
    const long long cp_bytes = ((4LL * ((long long)pl->groups * pl->n_chunks * pl->DT + 1)) + 15) / 16 * 16;
    BiArgs a{};
    a.x = static_cast<const float *>(x);
    a.y = static_cast<float *>(y);
    a.cpg = reinterpret_cast<const int *>(cb + 64);
    a.ents = reinterpret_cast<const int2 *>(cb + 64 + cp_bytes);
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
    a.full_rows = (pl->col_tiles == 1 && pl->TWs == pl->in.ws) ? 1 : 0;
    a.x_blk_stride = pl->in.sample_stride;
    a.stage_words = static_cast<int>(pl->smem_stage_bytes / 4);
    a.ep = ep;
    switch (pl->P) {
        case 1: return launch_dw<1>(pl, a, st);
        case 2: return launch_dw<2>(pl, a, st);
        default: return launch_dw<4>(pl, a, st);
    }
}

}  // namespace usc
