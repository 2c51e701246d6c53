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
// Persistent, warp-specialised CTA of NWC compute warps + 1 producer warp:
//   * the producer's elected lane streams, for every tile this CTA owns and
//     every chunk of CC input channels, the input tile ([CC][HS][TWs][32]
//     floats) plus that (group, chunk)'s entry block into an S-stage shared
//     memory ring with cp.async.bulk (UBLKCP, the TMA engine), completing on
//     full[s] and waiting on empty[s] before reuse;
//   * compute warp w owns strip w % WS (a PR x PC output-pixel block) for the DW
//     output channels of subgroup w / WS; lane = sample; DW*P fp32 accumulators
//     live for the whole input-channel loop; after a stage each warp arrives on
//     empty[s] -- no CTA-wide barrier inside the loop.
//   * entry block of one (group, chunk): int2 hdr[DT] = {first, end} entry index
//     of every output channel's run, then the runs, each starting 16-byte aligned
//     so two entries are one LDS.128 broadcast.  Everything the compute warps
//     read in the loop is in shared memory.
//   * the register budget is what sets NWC: warps are spread over 4 SM
//     sub-partitions, so (NWC+1) warps leave 65536 / (4 * ceil((NWC+1)/4) * 32)
//     registers per thread: 168 for NWC = 8, 128 for NWC = 12, 96 for NWC = 16.
//
// Per output element the arithmetic is the reference's: stored-order entries
// (ascending (c, kh, kw)), IEEE fp32 multiply then add (__fmul_rn/__fadd_rn),
// so results are bit-identical to the reference for every tile configuration.
#pragma once
#include <utility>

#include "common.cuh"

namespace usc_bi {
using namespace usc_dev;

struct BiArgs {
    const float *x;
    float *y;
    const int *blk;          // byte offset of every (group, chunk) block, G*n_chunks+1
    const int *perm;         // output channel of every (group, warp, slot); -1 = empty
    const char *blocks;      // block base (16-byte aligned)
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

// shared-memory loads on 32-bit addresses with immediate offsets (LDS [R+imm]);
// not volatile: the address depends on an entry read after the stage's mbarrier
// wait, which keeps them behind it
template <int OFF>
__device__ __forceinline__ float lds_f32(uint32_t a) {
    float v;
    asm("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(a), "n"(OFF));
    return v;
}
__device__ __forceinline__ int4 lds_v4(uint32_t a) {
    int4 v;
    asm("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ int2 lds_v2(uint32_t a) {
    int2 v;
    asm("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}

// the P pixels of a thread for one tap: row 0 at a0, row 1 at a1 (bytes), columns
// SW*128 bytes apart
template <int PC, int PR, int SW, int... I>
__device__ __forceinline__ void load_px_(float *v, uint32_t a0, uint32_t a1, std::integer_sequence<int, I...>) {
    ((v[I] = (I / PC == 0) ? lds_f32<(I % PC) * SW * 128>(a0) : lds_f32<(I % PC) * SW * 128>(a1)), ...);
}
template <int PC, int PR, int SW>
__device__ __forceinline__ void load_px(float (&v)[PC * PR], uint32_t a0, uint32_t a1) {
    load_px_<PC, PR, SW>(v, a0, a1, std::make_integer_sequence<int, PC * PR>{});
}

// acc[p] += t0*v0[p], then += t1*v1[p]: IEEE multiply then add, stored order
template <int P>
__device__ __forceinline__ void mac_pair(float (&acc)[P], float (&v0)[P], float (&v1)[P], const int4 &n) {
    const float t0 = __int_as_float(n.y), t1 = __int_as_float(n.w);
#pragma unroll
    for (int p = 0; p < P; ++p) {
        v0[p] = __fmul_rn(t0, v0[p]);
        v1[p] = __fmul_rn(t1, v1[p]);
    }
#pragma unroll
    for (int p = 0; p < P; ++p) acc[p] = __fadd_rn(acc[p], v0[p]);
#pragma unroll
    for (int p = 0; p < P; ++p) acc[p] = __fadd_rn(acc[p], v1[p]);
}

template <int PC, int PR, int SW>
__device__ __forceinline__ void load_pair(float (&v0)[PC * PR], float (&v1)[PC * PR], uint32_t xs, uint32_t rs,
                                          const int4 &n) {
    const uint32_t p0 = xs + n.x, p1 = xs + n.z;
    load_px<PC, PR, SW>(v0, p0, p0 + rs);
    load_px<PC, PR, SW>(v1, p1, p1 + rs);
}

// One output channel's run of entries [ep, ee) (byte addresses, ep 16-B aligned),
// two entries (one LDS.128) per step.  PIPE: software pipelined -- the next pair's
// 2P pixel loads are issued before this pair's math (ping-pong registers), so the
// shared-memory latency hides inside one warp.  Reads of the entry after a run stay
// inside the stage's 16-byte slack.
template <int PC, int PR, int SW, bool PIPE>
__device__ __forceinline__ void run_pairs(float (&acc)[PC * PR], uint32_t xs, uint32_t rs, uint32_t ep,
                                          uint32_t ee) {
    constexpr int P = PC * PR;
    int4 nn = lds_v4(ep);
    if constexpr (PIPE) {
        if (ep + 16 <= ee) {
            float a0[P], a1[P], b0[P], b1[P];
            int4 n = nn;
            load_pair<PC, PR, SW>(a0, a1, xs, rs, n);
            ep += 16;
            nn = lds_v4(ep);
#pragma unroll 1
            while (true) {  // a* hold pair n; nn is the pair at ep
                if (ep + 16 > ee) {
                    mac_pair<P>(acc, a0, a1, n);
                    break;
                }
                load_pair<PC, PR, SW>(b0, b1, xs, rs, nn);
                int4 m = nn;
                ep += 16;
                nn = lds_v4(ep);
                mac_pair<P>(acc, a0, a1, n);
                n = m;
                if (ep + 16 > ee) {
                    mac_pair<P>(acc, b0, b1, n);
                    break;
                }
                load_pair<PC, PR, SW>(a0, a1, xs, rs, nn);
                m = nn;
                ep += 16;
                nn = lds_v4(ep);
                mac_pair<P>(acc, b0, b1, n);
                n = m;
            }
        }
    } else {
#pragma unroll 1
        for (; ep + 16 <= ee; ep += 16) {
            float v0[P], v1[P];
            load_pair<PC, PR, SW>(v0, v1, xs, rs, nn);
            const int4 n = nn;
            nn = lds_v4(ep + 16);
            mac_pair<P>(acc, v0, v1, n);
        }
    }
    if (ep < ee) {  // odd run: the last entry is nn.x, nn.y
        float v0[P];
        const uint32_t p0 = xs + nn.x;
        load_px<PC, PR, SW>(v0, p0, p0 + rs);
        const float t0 = __int_as_float(nn.y);
#pragma unroll
        for (int p = 0; p < P; ++p) acc[p] = __fadd_rn(acc[p], __fmul_rn(t0, v0[p]));
    }
}

template <int PC, int PR, int DW, int SW, int NWC>
__global__ void __launch_bounds__((NWC + 1) * 32, 1) k_bi(const BiArgs a) {
    constexpr int P = PC * PR;  // a thread's pixel block: PR rows x PC cols
    // software-pipeline the pair loop when the second value set fits the register cap
    constexpr int REGCAP = NWC <= 8 ? 168 : (NWC <= 12 ? 128 : 96);
    constexpr bool PIPE = DW * P + 4 * P + 40 <= REGCAP;
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
            int s = 0;
            uint32_t ph = 1;
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
                const int *blk_g = a.blk + g * a.n_chunks;
                const int plane_words = a.HS * a.TWs * 32;
                for (int k = 0; k < a.n_chunks; ++k) {
                    mbar_wait(&empty[s], ph);
                    unsigned char *st = ring + s * a.stage_bytes;
                    float *dst = reinterpret_cast<float *>(st);
                    const int c0 = k * a.CC;
                    const int cc = min(a.CC, a.C - c0);
                    const int lo = __ldg(blk_g + k), hi = __ldg(blk_g + k + 1);
                    const uint32_t eb = static_cast<uint32_t>(hi - lo);
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
                    bulk_g2s(st + a.x_stage_bytes, a.blocks + lo, eb, &full[s]);
                    if (++s == a.S) {
                        s = 0;
                        ph ^= 1;
                    }
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
    const uint32_t rs = a.s_h * a.TWs * 128;  // bytes between a thread's two pixel rows
    const int hdr_bytes = a.DT * 8;
    int s = 0;
    uint32_t ph = 0;
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

        for (int k = 0; k < a.n_chunks; ++k) {
            const unsigned char *st = ring + s * a.stage_bytes;
            mbar_wait(&full[s], ph);
            if (active) {
                const uint32_t xs = smem_u32(st) + base * 4;  // this thread's first pixel, tap (0,0,0)
                const uint32_t bp = smem_u32(st) + a.x_stage_bytes;
                const uint32_t hdr = bp + wc * DW * 8, E = bp + hdr_bytes;
#pragma unroll
                for (int dw = 0; dw < DW; ++dw) {
                    const int2 h = lds_v2(hdr + dw * 8);  // run [h.x, h.y), h.x even
                    uint32_t ep = E + h.x * 8;
                    const uint32_t ee = E + h.y * 8;
                    run_pairs<PC, PR, SW, PIPE>(acc[dw], xs, rs, ep, ee);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == a.S) {
                s = 0;
                ph ^= 1;
            }
        }

        // epilogue: obase + d*dstride + row*rstride + col*cstride for all three output
        // layouts; ReLU (nn.py:96-98) then, if fused, the 2x2/2 max-pool (nn.py:124-135)
        const int b = sb * 32 + lane;
        if (!active || b >= a.N || r >= a.Yh) continue;
        const int *pm = a.perm + g * a.DT + wc * DW;  // this warp's output channels (balanced)
        const bool pool = PR == 2 && a.ep.pool;
        const int orow = pool ? r / 2 : r, ocol = pool ? col0 / 2 : col0;
        long long obase, dstride;  // element of (b, d, orow, ocol) = obase + d*dstride
        int rstride, cstride;
        if (!a.ep.out_padded) {
            const int oh = pool ? a.Yh / 2 : a.Yh, ow = pool ? a.Yw / 2 : a.Yw;
            obase = ((long long)b * a.D * oh + orow) * ow + ocol;
            dstride = (long long)oh * ow;
            rstride = ow;
            cstride = 1;
        } else if (a.ep.oil == 32) {
            obase = (long long)sb * a.ep.o_sample_stride +
                    ((((long long)orow + a.ep.oph) * a.ep.oWs + ocol + a.ep.opw) << 5) + lane;
            dstride = (long long)a.ep.oHp * a.ep.oWs * 32;
            rstride = a.ep.oWs * 32;
            cstride = 32;
        } else {
            obase = (long long)b * a.ep.o_sample_stride +
                    ((long long)orow + a.ep.oph) * a.ep.oWs + ocol + a.ep.opw;
            dstride = (long long)a.ep.oHp * a.ep.oWs;
            rstride = a.ep.oWs;
            cstride = 1;
        }
        const int ncol = min(PC, a.Yw - col0);
        const int nrow = min(PR, a.Yh - r);
        const bool relu = a.ep.relu != 0;
#pragma unroll
        for (int dw = 0; dw < DW; ++dw) {
            const int d = __ldg(pm + dw);
            if (d < 0) continue;
            const long long od = obase + d * dstride;
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
                            for (int q2 = 1; q2 < 4; ++q2) {
                                if (isnan(w4[q2])) {
                                    m = w4[q2];
                                    break;
                                }
                                if (w4[q2] > m) m = w4[q2];
                            }
                        }
                        a.y[od + j * cstride] = m;
                    }
                    continue;
                }
            }
#pragma unroll
            for (int p = 0; p < P; ++p)
                if ((p / PC) < nrow && (p % PC) < ncol)
                    a.y[od + (p / PC) * rstride + (p % PC) * cstride] = v[p];
        }
    }
}

template <int PC, int PR, int DW, int SW, int NWC>
int launch_inst(const usc_plan *pl, const BiArgs &a, cudaStream_t st) {
    auto fn = k_bi<PC, PR, DW, SW, NWC>;
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

int launch_w8(const usc_plan *pl, const BiArgs &a, cudaStream_t st);   // 8 compute warps (168 regs)
int launch_w12(const usc_plan *pl, const BiArgs &a, cudaStream_t st);  // 12 compute warps (128 regs)
int launch_w16(const usc_plan *pl, const BiArgs &a, cudaStream_t st);  // 16 compute warps (96 regs)

}  // namespace usc_bi
