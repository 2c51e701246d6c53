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
    int stage_words, ent_stage_bytes;
    Epi ep;
};

template <int P, int DW, int SW, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_bi(const BiArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
    float *stage0 = reinterpret_cast<float *>(smem + 128);
    float *stage1 = stage0 + a.stage_words;
    char *ents0 = reinterpret_cast<char *>(stage1 + a.stage_words);
    char *ents1 = ents0 + a.ent_stage_bytes;

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
    const int *cpg_g = a.cpg + (long long)g * a.n_chunks * a.DT;
    auto issue = [&](int k, int s) {
        const int c0 = k * a.CC;
        const int cc = min(a.CC, a.C - c0);
        float *dst = s ? stage1 : stage0;
        // this (group, chunk)'s entry block: 16-byte aligned start (packer), 16-byte
        // rounded size (the pack has 64 bytes of tail slack)
        const int blk_lo = __ldg(cpg_g + k * a.DT), blk_hi = __ldg(cpg_g + k * a.DT + a.DT);
        const uint32_t eb = static_cast<uint32_t>((blk_hi - blk_lo) * 8 + 15) & ~15u;
        const int plane_words = a.HS * a.TWs * 32;
        if (a.full_rows) {
            if (y0 == 0 && rows == a.Hp && a.HS == a.Hp) {
                const uint32_t bytes = static_cast<uint32_t>(cc) * a.Hp * a.Wp * 128u;
                mbar_expect_tx(&bar[s], bytes + eb);
                bulk_g2s(dst, xblk + (long long)c0 * a.Hp * a.Wp * 32, bytes, &bar[s]);
            } else {
                const uint32_t bytes = static_cast<uint32_t>(rows) * a.Wp * 128u;
                mbar_expect_tx(&bar[s], bytes * cc + eb);
#pragma unroll 1
                for (int c = 0; c < cc; ++c)
                    bulk_g2s(dst + c * plane_words,
                             xblk + (((long long)(c0 + c) * a.Hp + y0) * a.Wp) * 32, bytes, &bar[s]);
            }
        } else {
            const int w = min(a.TWs, a.Wp - x0);
            const uint32_t bytes = static_cast<uint32_t>(w) * 128u;
            mbar_expect_tx(&bar[s], bytes * cc * rows + eb);
#pragma unroll 1
            for (int c = 0; c < cc; ++c)
#pragma unroll 1
                for (int rr = 0; rr < rows; ++rr)
                    bulk_g2s(dst + c * plane_words + rr * a.TWs * 32,
                             xblk + ((((long long)(c0 + c) * a.Hp + y0 + rr) * a.Wp) + x0) * 32, bytes,
                             &bar[s]);
        }
        if (eb) bulk_g2s(s ? ents1 : ents0, a.ents + blk_lo, eb, &bar[s]);
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

    // chunk boundaries of this warp's DW channels: lanes 0..DW hold them, lane
    // DW+1 holds the start of the (group, chunk) block staged in shared memory
    const int *cp = cpg_g + wc * DW;
    const int bl = lane <= DW ? lane : -wc * DW;
    int bnd = (active && lane <= DW + 1) ? __ldg(cp + bl) : 0;
    const char *xs_b0 = reinterpret_cast<const char *>(stage0 + base);
    const char *xs_b1 = reinterpret_cast<const char *>(stage1 + base);
    for (int k = 0; k < a.n_chunks; ++k) {
        const int s = k & 1;
        const int bnd_cur = bnd;
        if (active && lane <= DW + 1 && k + 1 < a.n_chunks) bnd = __ldg(cp + (k + 1) * a.DT + bl);
        mbar_wait(&bar[s], (k >> 1) & 1);
        if (active) {
            const char *xs = s ? xs_b1 : xs_b0;
            const int blk0 = __shfl_sync(0xffffffffu, bnd_cur, DW + 1);
            const int2 *eb = reinterpret_cast<const int2 *>(s ? ents1 : ents0) - blk0;
#pragma unroll
            for (int dw = 0; dw < DW; ++dw) {
                const int e0 = __shfl_sync(0xffffffffu, bnd_cur, dw);
                const int e1 = __shfl_sync(0xffffffffu, bnd_cur, dw + 1);
                int e = e0;
                // two entries per step: both entries' P loads are in flight before
                // the mul/adds, which then run in stored order
#pragma unroll 1
                for (; e + 2 <= e1; e += 2) {
                    const int2 n0 = eb[e], n1 = eb[e + 1];
                    const float *x0p = reinterpret_cast<const float *>(xs + n0.x);
                    const float *x1p = reinterpret_cast<const float *>(xs + n1.x);
                    float v0[P], v1[P];
#pragma unroll
                    for (int p = 0; p < P; ++p) v0[p] = x0p[p * SW * 32];
#pragma unroll
                    for (int p = 0; p < P; ++p) v1[p] = x1p[p * SW * 32];
                    const float t0 = __int_as_float(n0.y), t1 = __int_as_float(n1.y);
#pragma unroll
                    for (int p = 0; p < P; ++p) acc[dw][p] = __fadd_rn(acc[dw][p], __fmul_rn(t0, v0[p]));
#pragma unroll
                    for (int p = 0; p < P; ++p) acc[dw][p] = __fadd_rn(acc[dw][p], __fmul_rn(t1, v1[p]));
                }
                if (e < e1) {
                    const int2 n0 = eb[e];
                    const float *x0p = reinterpret_cast<const float *>(xs + n0.x);
                    const float t0 = __int_as_float(n0.y);
#pragma unroll
                    for (int p = 0; p < P; ++p) acc[dw][p] = __fadd_rn(acc[dw][p], __fmul_rn(t0, x0p[p * SW * 32]));
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
    // output addressing: base + dw*dstride + p*cstride for all three layouts
    const int d0 = g * a.DT + wc * DW;
    long long obase, dstride;
    int cstride;
    if (!a.ep.out_padded) {
        obase = (((long long)b * a.D + d0) * a.Yh + r) * a.Yw + col0;
        dstride = (long long)a.Yh * a.Yw;
        cstride = 1;
    } else if (a.ep.oil == 32) {
        obase = (long long)sb * a.ep.o_sample_stride +
                ((((long long)d0 * a.ep.oHp + r + a.ep.oph) * a.ep.oWs + col0 + a.ep.opw) << 5) + lane;
        dstride = (long long)a.ep.oHp * a.ep.oWs * 32;
        cstride = 32;
    } else {
        obase = (long long)b * a.ep.o_sample_stride + ((long long)d0 * a.ep.oHp + r + a.ep.oph) * a.ep.oWs +
                col0 + a.ep.opw;
        dstride = (long long)a.ep.oHp * a.ep.oWs;
        cstride = 1;
    }
    const int ndw = min(DW, a.D - d0);
    const int np = min(P, a.Yw - col0);
    const bool relu = a.ep.relu != 0;
#pragma unroll
    for (int dw = 0; dw < DW; ++dw) {
#pragma unroll
        for (int p = 0; p < P; ++p) {
            if (dw < ndw && p < np) {
                float v = acc[dw][p];
                if (relu) v = v > 0.0f ? v : 0.0f;
                a.y[obase + dw * dstride + p * cstride] = v;
            }
        }
    }
}

template <int P, int DW, int SW, int NT, int MINB>
int launch_inst(const usc_plan *pl, const BiArgs &a, cudaStream_t st) {
    auto fn = k_bi<P, DW, SW, NT, MINB>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        attr = true;
    }
    fn<<<static_cast<unsigned>(pl->grid_x), NT, pl->smem_bytes, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return usc::fail(USC_ERR_CUDA, "k_bi launch: %s", cudaGetErrorString(e));
    return USC_OK;
}

// Instantiated tiles: 256 threads x 4 CTAs/SM (<= 64 registers, DW*P <= 32) and
// 512 threads x 1 CTA/SM (<= 128 registers, DW*P <= 64).
template <int SW>
int launch_tile(const usc_plan *pl, const BiArgs &a, cudaStream_t st) {
    const int P = pl->P, DW = pl->DW;
#define USC_BI(PP, DD, NT, MB) \
    if (P == PP && DW == DD) return launch_inst<PP, DD, SW, NT, MB>(pl, a, st);
    if (pl->threads == 512) {
        // 512 threads x 1 CTA/SM: <= 128 registers, DW*P <= 64
        USC_BI(1, 4, 512, 1) USC_BI(1, 8, 512, 1) USC_BI(1, 16, 512, 1)
        USC_BI(2, 4, 512, 1) USC_BI(2, 8, 512, 1) USC_BI(2, 16, 512, 1)
        USC_BI(4, 4, 512, 1) USC_BI(4, 8, 512, 1) USC_BI(4, 16, 512, 1)
        USC_BI(8, 4, 512, 1) USC_BI(8, 8, 512, 1)
    } else {
        // 256 threads x 4 CTAs/SM: <= 64 registers, DW*P <= 32
        USC_BI(1, 4, 256, 4) USC_BI(1, 8, 256, 4) USC_BI(1, 16, 256, 4)
        USC_BI(2, 4, 256, 4) USC_BI(2, 8, 256, 4) USC_BI(2, 16, 256, 4)
        USC_BI(4, 4, 256, 4) USC_BI(4, 8, 256, 4)
        USC_BI(8, 4, 256, 4)
    }
#undef USC_BI
    return usc::fail(USC_ERR_UNSUPPORTED, "no BI kernel instance for P=%d DW=%d threads=%d", P, DW,
                     pl->threads);
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
    a.ent_stage_bytes = pl->ent_stage_bytes;
    a.ep = ep;
    return pl->g.stride_w == 1 ? launch_tile<1>(pl, a, st) : launch_tile<2>(pl, a, st);
}

}  // namespace usc
