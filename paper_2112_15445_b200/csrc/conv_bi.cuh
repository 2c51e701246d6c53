// conv_bi.cuh -- the batch-interleaved fp32 direct sparse conv kernel (sm_100a).
//
// Replaces the reference's hot loop kernels.sparse_conv_blocks
// (/root/reference/pkg/src/unsparse/kernels.py:57-100) for BINARY32.
//
// Layout: activations are BI32 ([n/32][C][Hp][Wp][32], zero halo): the 32 lanes
// of a warp are 32 samples, so for a given (pixel, tap) every shared-memory load
// is one conflict-free 128-byte wavefront and every output store is one
// coalesced 128-byte line.
//
// Persistent, warp-specialised CTA:
//   * warp NWC (the last) is the producer: one elected lane streams, for every
//     tile this CTA owns and every chunk of CC input channels, the input tile
//     ([CC][HS][TWs][32] floats) plus that (group, chunk)'s CSR entry block into
//     an S-stage shared-memory ring with cp.async.bulk (UBLKCP, the TMA engine),
//     completing on full[s] and waiting on empty[s] before reuse;
//   * warps 0..NWC-1 compute: warp w owns strip w % WS (P consecutive output
//     pixels of a row) for the DW output channels of subgroup w / WS, lane =
//     sample, DW*P fp32 accumulators for the whole input-channel loop; after a
//     stage each warp arrives on empty[s] -- no CTA-wide barrier in the loop.
//   * tiles = (channel group fastest, column tile, row tile, 32-sample block); a
//     CTA takes tiles blockIdx.x, +gridDim.x, ... so the producer runs ahead into
//     the next tile while the compute warps store the previous one.
//
// Per output element the arithmetic is the reference's: stored-order entries
// (ascending (c, kh, kw)), IEEE fp32 multiply then add (__fmul_rn/__fadd_rn),
// so results are bit-identical to the reference for every tile configuration.
#pragma once
#include "common.cuh"

namespace usc_bi {
using namespace usc_dev;

struct BiArgs {
    const float *x;
    float *y;
    const int *cpg;
    const int2 *ents;
    int N, C, D, n_chunks, CC, DT;
    int HS, TWs, Hp, Wp, Yh, Yw, s_h;
    int WS, WC, SPRt, TH, row_tiles, col_tiles, G, tiles, S;
    int full_rows;
    long long x_blk_stride;  // elements per 32-sample block
    int x_stage_bytes, stage_bytes;
    Epi ep;
};

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int PC, int PR, int DW, int SW, int NWC, int MINB>
__global__ void __launch_bounds__((NWC + 1) * 32, MINB) k_bi(const BiArgs a) {
    constexpr int P = PC * PR;                          // a thread's pixel block: PR rows x PC cols
    constexpr int U = P >= 8 ? 2 : (P >= 4 ? 4 : 8);  // U*P = 16-32 loads in flight
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint64_t *empty = full + 8;
    unsigned char *ring = smem + 128;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        for (int s = 0; s < a.S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NWC);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == NWC) {
        // ---------------- producer warp ----------------
        if (lane == 0) {
            int it = 0;
            for (int t = blockIdx.x; t < a.tiles; t += gridDim.x) {
                int q = t;
                const int g = q % a.G;
                q /= a.G;
                const int ct = q % a.col_tiles;
                q /= a.col_tiles;
                const int rt = q % a.row_tiles;
                const int sb = q / a.row_tiles;
                const int y0 = rt * a.TH * a.s_h;
                const int x0 = ct * a.SPRt * PC * SW;
                const int rows = min(a.HS, a.Hp - y0);
                const float *xblk = a.x + (long long)sb * a.x_blk_stride;
                const int *cpg_g = a.cpg + (long long)g * a.n_chunks * a.DT;
                const int plane_words = a.HS * a.TWs * 32;
                for (int k = 0; k < a.n_chunks; ++k, ++it) {
                    const int s = it % a.S;
                    mbar_wait(&empty[s], ((it / a.S) & 1) ^ 1);
                    float *dst = reinterpret_cast<float *>(ring + (long long)s * a.stage_bytes);
                    char *edst = reinterpret_cast<char *>(ring + (long long)s * a.stage_bytes + a.x_stage_bytes);
                    const int c0 = k * a.CC;
                    const int cc = min(a.CC, a.C - c0);
                    // the (group, chunk) entry block: 16-byte aligned start (packer),
                    // 16-byte rounded size (the pack has tail slack)
                    const int blk_lo = __ldg(cpg_g + k * a.DT), blk_hi = __ldg(cpg_g + k * a.DT + a.DT);
                    const uint32_t eb = static_cast<uint32_t>((blk_hi - blk_lo) * 8 + 15) & ~15u;
                    fence_proxy_async();
                    if (a.full_rows) {
                        if (y0 == 0 && rows == a.Hp && a.HS == a.Hp) {
                            const uint32_t bytes = static_cast<uint32_t>(cc) * a.Hp * a.Wp * 128u;
                            mbar_expect_tx(&full[s], bytes + eb);
                            bulk_g2s(dst, xblk + (long long)c0 * a.Hp * a.Wp * 32, bytes, &full[s]);
                        } else {
                            const uint32_t bytes = static_cast<uint32_t>(rows) * a.Wp * 128u;
                            mbar_expect_tx(&full[s], bytes * cc + eb);
#pragma unroll 1
                            for (int c = 0; c < cc; ++c)
                                bulk_g2s(dst + c * plane_words,
                                         xblk + (((long long)(c0 + c) * a.Hp + y0) * a.Wp) * 32, bytes,
                                         &full[s]);
                        }
                    } else {
                        const int w = min(a.TWs, a.Wp - x0);
                        const uint32_t bytes = static_cast<uint32_t>(w) * 128u;
                        mbar_expect_tx(&full[s], bytes * cc * rows + eb);
#pragma unroll 1
                        for (int c = 0; c < cc; ++c)
#pragma unroll 1
                            for (int rr = 0; rr < rows; ++rr)
                                bulk_g2s(dst + c * plane_words + rr * a.TWs * 32,
                                         xblk + ((((long long)(c0 + c) * a.Hp + y0 + rr) * a.Wp) + x0) * 32,
                                         bytes, &full[s]);
                    }
                    if (eb) bulk_g2s(edst, a.ents + blk_lo, eb, &full[s]);
                }
            }
        }
        return;
    }

    // ---------------- compute warps ----------------
    const int wsi = warp % a.WS, wc = warp / a.WS;
    const bool active = wc < a.WC;
    const int tr = wsi / a.SPRt, tcs = wsi - tr * a.SPRt;  // strip-row, strip within the tile
    const int base = ((tr * PR * a.s_h) * a.TWs + tcs * PC * SW) * 32 + lane;
    const int rstep = a.s_h * a.TWs * 32;  // floats between a thread's two pixel rows
    const int bl = lane <= DW ? lane : -wc * DW;  // lane DW+1 reads the block start
    int it = 0;
    for (int t = blockIdx.x; t < a.tiles; t += gridDim.x) {
        int q = t;
        const int g = q % a.G;
        q /= a.G;
        const int ct = q % a.col_tiles;
        q /= a.col_tiles;
        const int rt = q % a.row_tiles;
        const int sb = q / a.row_tiles;
        const int r = rt * a.TH + tr * PR;
        const int col0 = (ct * a.SPRt + tcs) * PC;

        float acc[DW][P];
#pragma unroll
        for (int i = 0; i < DW; ++i)
#pragma unroll
            for (int p = 0; p < P; ++p) acc[i][p] = 0.0f;

        // chunk boundaries of this warp's DW channels (lanes 0..DW) and the block
        // start (lane DW+1), one chunk ahead
        const int *cp = a.cpg + (long long)g * a.n_chunks * a.DT + wc * DW;
        int bnd = (active && lane <= DW + 1) ? __ldg(cp + bl) : 0;
        for (int k = 0; k < a.n_chunks; ++k, ++it) {
            const int s = it % a.S;
            const int bnd_cur = bnd;
            if (active && lane <= DW + 1 && k + 1 < a.n_chunks) bnd = __ldg(cp + (k + 1) * a.DT + bl);
            mbar_wait(&full[s], (it / a.S) & 1);
            if (active) {
                const unsigned char *st = ring + (long long)s * a.stage_bytes;
                const char *xs = reinterpret_cast<const char *>(reinterpret_cast<const float *>(st) + base);
                const int blk0 = __shfl_sync(0xffffffffu, bnd_cur, DW + 1);
                const int2 *eb = reinterpret_cast<const int2 *>(st + a.x_stage_bytes) - blk0;
#pragma unroll
                for (int dw = 0; dw < DW; ++dw) {
                    const int e0 = __shfl_sync(0xffffffffu, bnd_cur, dw);
                    const int e1 = __shfl_sync(0xffffffffu, bnd_cur, dw + 1);
                    int e = e0;
                    // U entries per step: all U*P loads are in flight before the math;
                    // products first, then the adds in stored order (no FMUL->FADD stall)
#pragma unroll 1
                    for (; e + U <= e1; e += U) {
                        int2 n[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) n[u] = eb[e + u];
                        float v[U][P];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const float *xp = reinterpret_cast<const float *>(xs + n[u].x);
#pragma unroll
                            for (int p = 0; p < P; ++p) v[u][p] = xp[(p / PC) * rstep + (p % PC) * SW * 32];
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const float th = __int_as_float(n[u].y);
#pragma unroll
                            for (int p = 0; p < P; ++p) v[u][p] = __fmul_rn(th, v[u][p]);
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u)
#pragma unroll
                            for (int p = 0; p < P; ++p) acc[dw][p] = __fadd_rn(acc[dw][p], v[u][p]);
                    }
#pragma unroll 1
                    for (; e < e1; ++e) {
                        const int2 n0 = eb[e];
                        const float *x0p = reinterpret_cast<const float *>(xs + n0.x);
                        const float t0 = __int_as_float(n0.y);
#pragma unroll
                        for (int p = 0; p < P; ++p)
                            acc[dw][p] = __fadd_rn(acc[dw][p],
                                                   __fmul_rn(t0, x0p[(p / PC) * rstep + (p % PC) * SW * 32]));
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }

        // epilogue: obase + dw*dstride + row*rstride + col*cstride for all three output
        // layouts; ReLU (nn.py:96-98) then, if fused, the 2x2/2 max-pool (nn.py:124-135)
        const int b = sb * 32 + lane;
        if (!active || b >= a.N || r >= a.Yh) continue;
        const int d0 = g * a.DT + wc * DW;
        const bool pool = PR == 2 && a.ep.pool;
        const int orow = pool ? r / 2 : r, ocol = pool ? col0 / 2 : col0;
        long long obase, dstride;
        int rstride, cstride;
        if (!a.ep.out_padded) {
            const int oh = pool ? a.Yh / 2 : a.Yh, ow = pool ? a.Yw / 2 : a.Yw;
            obase = (((long long)b * a.D + d0) * oh + orow) * ow + ocol;
            dstride = (long long)oh * ow;
            rstride = ow;
            cstride = 1;
        } else if (a.ep.oil == 32) {
            obase = (long long)sb * a.ep.o_sample_stride +
                    ((((long long)d0 * a.ep.oHp + orow + a.ep.oph) * a.ep.oWs + ocol + a.ep.opw) << 5) + lane;
            dstride = (long long)a.ep.oHp * a.ep.oWs * 32;
            rstride = a.ep.oWs * 32;
            cstride = 32;
        } else {
            obase = (long long)b * a.ep.o_sample_stride +
                    ((long long)d0 * a.ep.oHp + orow + a.ep.oph) * a.ep.oWs + ocol + a.ep.opw;
            dstride = (long long)a.ep.oHp * a.ep.oWs;
            rstride = a.ep.oWs;
            cstride = 1;
        }
        const int ndw = min(DW, a.D - d0);
        const int ncol = min(PC, a.Yw - col0);
        const int nrow = min(PR, a.Yh - r);
        const bool relu = a.ep.relu != 0;
#pragma unroll
        for (int dw = 0; dw < DW; ++dw) {
            if (dw >= ndw) break;
            float v[P];
#pragma unroll
            for (int p = 0; p < P; ++p) {
                v[p] = acc[dw][p];
                if (relu) v[p] = v[p] > 0.0f ? v[p] : 0.0f;
            }
            if constexpr (PR == 2 && PC % 2 == 0) {
                if (pool) {
#pragma unroll
                    for (int j = 0; j < PC / 2; ++j) {
                        if (2 * j >= ncol) break;
                        const float w4[4] = {v[2 * j], v[2 * j + 1], v[PC + 2 * j], v[PC + 2 * j + 1]};
                        float m = w4[0];
                        if (!isnan(m)) {
#pragma unroll
                            for (int q = 1; q < 4; ++q) {
                                if (isnan(w4[q])) {
                                    m = w4[q];
                                    break;
                                }
                                if (w4[q] > m) m = w4[q];
                            }
                        }
                        a.y[obase + dw * dstride + j * cstride] = m;
                    }
                    continue;
                }
            }
#pragma unroll
            for (int p = 0; p < P; ++p)
                if ((p / PC) < nrow && (p % PC) < ncol)
                    a.y[obase + dw * dstride + (p / PC) * rstride + (p % PC) * cstride] = v[p];
        }
    }
}

template <int PC, int PR, int DW, int SW, int NWC, int MINB>
int launch_inst(const usc_plan *pl, const BiArgs &a, cudaStream_t st) {
    auto fn = k_bi<PC, PR, DW, SW, NWC, MINB>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024);
        attr = true;
    }
    fn<<<static_cast<unsigned>(pl->grid_x), (NWC + 1) * 32, pl->smem_bytes, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return usc::fail(USC_ERR_CUDA, "k_bi launch: %s", cudaGetErrorString(e));
    return USC_OK;
}

// instantiated tiles: DW * PR * PC <= 64 accumulators
#define USC_BI(PCC, PRR, DD) \
    if (PC == PCC && PR == PRR && DW == DD) return launch_inst<PCC, PRR, DD, SW, NWC, MINB>(pl, a, st);

template <int SW, int NWC, int MINB>
int launch_rows1(const usc_plan *pl, const BiArgs &a, cudaStream_t st) {
    const int PC = pl->PC, PR = pl->PR, DW = pl->DW;
    USC_BI(1, 1, 4) USC_BI(1, 1, 8) USC_BI(1, 1, 16)
    USC_BI(2, 1, 4) USC_BI(2, 1, 8) USC_BI(2, 1, 16)
    USC_BI(4, 1, 4) USC_BI(4, 1, 8) USC_BI(4, 1, 16)
    USC_BI(8, 1, 4) USC_BI(8, 1, 8)
    return usc::fail(USC_ERR_UNSUPPORTED, "no BI kernel instance for PC=%d PR=%d DW=%d", PC, PR, DW);
}

template <int SW, int NWC, int MINB>
int launch_rows2(const usc_plan *pl, const BiArgs &a, cudaStream_t st) {
    const int PC = pl->PC, PR = pl->PR, DW = pl->DW;
    USC_BI(1, 2, 4) USC_BI(1, 2, 8) USC_BI(1, 2, 16)
    USC_BI(2, 2, 2) USC_BI(2, 2, 4) USC_BI(2, 2, 8) USC_BI(2, 2, 16)
    USC_BI(4, 2, 4) USC_BI(4, 2, 8)
    USC_BI(8, 2, 4)
    return usc::fail(USC_ERR_UNSUPPORTED, "no BI kernel instance for PC=%d PR=%d DW=%d", PC, PR, DW);
}
#undef USC_BI

int launch_16(const usc_plan *pl, const BiArgs &a, cudaStream_t st);  // 16 compute warps, 1 CTA/SM
int launch_16r2(const usc_plan *pl, const BiArgs &a, cudaStream_t st);  // ... with 2-row pixel blocks
int launch_8(const usc_plan *pl, const BiArgs &a, cudaStream_t st);   // 8 compute warps, 2 CTAs/SM

}  // namespace usc_bi
