// conv_bi.cuh -- the batch-interleaved fp32 direct sparse conv kernel (sm_100a).
//
// Replaces the reference's hot loop kernels.sparse_conv_blocks
// (/root/reference/pkg/src/unsparse/kernels.py:57-100) for BINARY32.
//
// Layout: activations are batch-interleaved, IL = 32*SPL samples innermost
// ([n/IL][C][Hp][Wp][IL], zero halo): lane l of a warp holds samples SPL*l ..
// SPL*l+SPL-1, so for a given (pixel, tap) a warp's shared-memory load is SPL
// conflict-free 128-byte wavefronts and an output store is one coalesced line.
//   SPL = 1 (BI32): LDS.32, FMUL, FADD per MAC.
//   SPL = 2 (BI64): one LDS.64 feeds two samples; two FMUL then one packed FADD2
//   (add.rn.f32x2) -- 2 instructions per MAC instead of 3.  (mul.rn.f32x2 followed by
//   add.rn.f32x2 is contracted to FFMA2 by ptxas 12.9 even with --fmad=false, which
//   would break the reference's separately rounded multiply; FMUL + FADD2 is not.)
//
// Persistent, warp-specialised CTA of NWC compute warps + 1 producer warp:
//   * the producer's elected lane streams, for every tile this CTA owns and
//     every chunk of CC input channels, the input box [CC][HS][TWs][IL] with ONE
//     TMA tensor copy (cp.async.bulk.tensor.5d, out-of-range rows/columns/channels
//     zero-filled) plus that (group, chunk)'s entry block with one bulk copy into an
//     S-stage shared-memory ring, completing on full[s] and waiting on empty[s];
//   * compute warp w owns strip w % WS (a PR x PC output-pixel block) for the DW
//     output-channel slots of subgroup w / WS; DW*P accumulators per lane (SPL
//     samples each) live for the whole input-channel loop; after a stage each warp
//     arrives on empty[s] -- no CTA-wide barrier inside the loop;
//   * entry block of one (group, chunk): int2 hdr[NCLS][DT] = {first, end} entry
//     index of every (pixel class, slot) run, then the runs, each starting 16-byte
//     aligned so two entries are one LDS.128 broadcast.  Slots map to output
//     channels through perm[] (the packer balances the warps' per-chunk work).  With
//     pixel classes (1x1 pixel blocks on small maps) a pixel's run omits the taps that
//     land on its zero halo: theta*0 adds +-0, a no-op for the never -0 accumulator;
//   * the register budget sets NWC: warps are spread over 4 SM sub-partitions, so
//     (NWC+1) warps leave 65536 / (4 * ceil((NWC+1)/4) * 32) registers per thread:
//     168 for NWC = 8, 128 for NWC = 12, 96 for NWC = 16.
//
// Per output element the arithmetic is the reference's: stored-order entries
// (ascending (c, kh, kw)), IEEE fp32 multiply then add, each rounded, so results
// are bit-identical to the reference for every tile configuration.
#pragma once
#include <cuda.h>

#include <utility>

#include "common.cuh"

namespace usc_bi {
using namespace usc_dev;

struct BiArgs {
    CUtensorMap xmap;        // x as 5-D [Nb][C][Hp][Wp][IL] fp32 (innermost first in the map)
    float *y;
    const int *blk;          // byte offset of every (group, chunk) block, G*n_chunks+1
    const int *perm;         // output channel of every (group, warp, slot); -1 = empty
    const char *blocks;      // block base (16-byte aligned)
    const int *rowcls, *colcls;  // pixel class of every output row / column
    int ncls, ncls_c;        // classes (runs per slot), column classes
    int N, D, n_chunks, CC, DT;
    int HS, TWs, Yh, Yw, s_h;
    int WS, WC, SPRt, TH, row_tiles, col_tiles, G, tiles, S;
    int items, tfull, split;  // work items: tiles [0, tfull) whole, the rest split in `split` slot subsets
    int x_stage_bytes, stage_bytes;
    Epi ep;
};

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tma_load_5d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                            int c4, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
        : "memory");
}

// ---------------------------------------------------------------------------
// lane value types: SPL samples per lane

template <int SPL> struct LaneT;
template <> struct LaneT<1> {
    using V = float;  // one tap value
    using A = float;  // one accumulator
};
template <> struct LaneT<2> {
    using V = float2;
    using A = unsigned long long;  // packed (sample 2l, sample 2l+1) for FADD2
};

// shared-memory loads on 32-bit addresses with immediate offsets (LDS [R+imm]);
// not volatile: the address depends on an entry read after the stage's mbarrier
// wait, which keeps them behind it
template <int OFF>
__device__ __forceinline__ void lds_val(float &v, uint32_t a) {
    asm("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(a), "n"(OFF));
}
template <int OFF>
__device__ __forceinline__ void lds_val(float2 &v, uint32_t a) {
    asm("ld.shared.v2.f32 {%0, %1}, [%2+%3];" : "=f"(v.x), "=f"(v.y) : "r"(a), "n"(OFF));
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

// product t*v, rounded (IEEE multiply)
__device__ __forceinline__ float mul_v(float t, float v) { return __fmul_rn(t, v); }
__device__ __forceinline__ float2 mul_v(float t, float2 v) { return make_float2(__fmul_rn(t, v.x), __fmul_rn(t, v.y)); }
// acc + product, rounded (IEEE add)
__device__ __forceinline__ void add_v(float &acc, float p) { acc = __fadd_rn(acc, p); }
__device__ __forceinline__ void add_v(unsigned long long &acc, float2 p) {
    unsigned long long q;
    asm("mov.b64 %0, {%1, %2};" : "=l"(q) : "f"(p.x), "f"(p.y));
    asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(q));
}
__device__ __forceinline__ void zero_a(float &a) { a = 0.0f; }
__device__ __forceinline__ void zero_a(unsigned long long &a) { a = 0ull; }  // (+0.0f, +0.0f)
__device__ __forceinline__ void unpack_a(float a, float (&o)[1]) { o[0] = a; }
__device__ __forceinline__ void unpack_a(unsigned long long a, float (&o)[2]) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(o[0]), "=f"(o[1]) : "l"(a));
}

// the P pixels of a thread for one tap: row 0 at a0, row 1 at a1 (bytes), columns
// SW pixels (SW*PXB bytes) apart
template <int PC, int PXB, int SW, typename V, int... I>
__device__ __forceinline__ void load_px_(V *v, uint32_t a0, uint32_t a1, std::integer_sequence<int, I...>) {
    ((I / PC == 0 ? lds_val<(I % PC) * SW * PXB>(v[I], a0) : lds_val<(I % PC) * SW * PXB>(v[I], a1)), ...);
}
template <int PC, int PR, int SW, int SPL>
__device__ __forceinline__ void load_px(typename LaneT<SPL>::V (&v)[PC * PR], uint32_t a0, uint32_t a1) {
    load_px_<PC, 128 * SPL, SW>(v, a0, a1, std::make_integer_sequence<int, PC * PR>{});
}

// acc[p] += t0*v0[p], then += t1*v1[p]: products first, then the adds in stored order
template <int P, int SPL>
__device__ __forceinline__ void mac_pair(typename LaneT<SPL>::A (&acc)[P], typename LaneT<SPL>::V (&v0)[P],
                                         typename LaneT<SPL>::V (&v1)[P], const int4 &n) {
    const float t0 = __int_as_float(n.y), t1 = __int_as_float(n.w);
#pragma unroll
    for (int p = 0; p < P; ++p) {
        v0[p] = mul_v(t0, v0[p]);
        v1[p] = mul_v(t1, v1[p]);
    }
#pragma unroll
    for (int p = 0; p < P; ++p) add_v(acc[p], v0[p]);
#pragma unroll
    for (int p = 0; p < P; ++p) add_v(acc[p], v1[p]);
}

template <int PC, int PR, int SW, int SPL>
__device__ __forceinline__ void load_pair(typename LaneT<SPL>::V (&v0)[PC * PR], typename LaneT<SPL>::V (&v1)[PC * PR],
                                          uint32_t xs, uint32_t rs, const int4 &n) {
    const uint32_t p0 = xs + n.x, p1 = xs + n.z;
    load_px<PC, PR, SW, SPL>(v0, p0, p0 + rs);
    load_px<PC, PR, SW, SPL>(v1, p1, p1 + rs);
}

// One slot's run of entries [ep, ee) (byte addresses, ep 16-B aligned), two entries
// (one LDS.128) per step.  PIPE: software pipelined -- the next pair's pixel loads
// are issued before this pair's math (ping-pong registers), so the shared-memory
// latency hides inside one warp.  Reads of the entry after a run stay inside the
// stage's 16-byte slack.
template <int PC, int PR, int SW, int SPL, bool PIPE>
__device__ __forceinline__ void run_pairs(typename LaneT<SPL>::A (&acc)[PC * PR], uint32_t xs, uint32_t rs,
                                          uint32_t ep, uint32_t ee) {
    constexpr int P = PC * PR;
    using V = typename LaneT<SPL>::V;
    int4 nn = lds_v4(ep);
    if constexpr (PIPE) {
        if (ep + 16 <= ee) {
            V a0[P], a1[P], b0[P], b1[P];
            int4 n = nn;
            load_pair<PC, PR, SW, SPL>(a0, a1, xs, rs, n);
            ep += 16;
            nn = lds_v4(ep);
#pragma unroll 1
            while (true) {  // a* hold pair n; nn is the pair at ep
                if (ep + 16 > ee) {
                    mac_pair<P, SPL>(acc, a0, a1, n);
                    break;
                }
                load_pair<PC, PR, SW, SPL>(b0, b1, xs, rs, nn);
                int4 m = nn;
                ep += 16;
                nn = lds_v4(ep);
                mac_pair<P, SPL>(acc, a0, a1, n);
                n = m;
                if (ep + 16 > ee) {
                    mac_pair<P, SPL>(acc, b0, b1, n);
                    break;
                }
                load_pair<PC, PR, SW, SPL>(a0, a1, xs, rs, nn);
                m = nn;
                ep += 16;
                nn = lds_v4(ep);
                mac_pair<P, SPL>(acc, b0, b1, n);
                n = m;
            }
        }
    } else {
#pragma unroll 1
        for (; ep + 16 <= ee; ep += 16) {
            V v0[P], v1[P];
            load_pair<PC, PR, SW, SPL>(v0, v1, xs, rs, nn);
            const int4 n = nn;
            nn = lds_v4(ep + 16);
            mac_pair<P, SPL>(acc, v0, v1, n);
        }
    }
    if (ep < ee) {  // odd run: the last entry is nn.x, nn.y
        V v0[P];
        const uint32_t p0 = xs + nn.x;
        load_px<PC, PR, SW, SPL>(v0, p0, p0 + rs);
        const float t0 = __int_as_float(nn.y);
#pragma unroll
        for (int p = 0; p < P; ++p) v0[p] = mul_v(t0, v0[p]);
#pragma unroll
        for (int p = 0; p < P; ++p) add_v(acc[p], v0[p]);
    }
}

// max-pool of a 2x2 window in np.argmax order (nn.py:124-135): first NaN, else
// first maximum
__device__ __forceinline__ float pool4(float w0, float w1, float w2, float w3) {
    const float w[4] = {w0, w1, w2, w3};
    float m = w[0];
    if (!isnan(m)) {
#pragma unroll
        for (int q = 1; q < 4; ++q) {
            if (isnan(w[q])) {
                m = w[q];
                break;
            }
            if (w[q] > m) m = w[q];
        }
    }
    return m;
}

// Work item -> (tile, slot part).  The last tiles of the schedule are split into
// `split` interleaved slot subsets (part p runs slots dw % split == p) so the final
// round of the persistent grid is not a partial wave of whole tiles.
__device__ __forceinline__ int item_tile(const BiArgs &a, int it, int &part) {
    if (it < a.tfull) {
        part = -1;
        return it;
    }
    const int j = it - a.tfull;
    part = j % a.split;
    return a.tfull + j / a.split;
}

template <int PC, int PR, int DW, int SW, int NWC, int SPL>
__global__ void __launch_bounds__((NWC + 1) * 32, 1) k_bi(const __grid_constant__ BiArgs a) {
    constexpr int P = PC * PR;      // a thread's pixel block: PR rows x PC cols
    constexpr int IL = 32 * SPL;    // samples per interleave block
    constexpr int PXB = 4 * IL;     // bytes per staged pixel
    using A = typename LaneT<SPL>::A;
    // software-pipeline the pair loop when the second value set fits the register cap
    constexpr int REGCAP = NWC <= 8 ? 168 : (NWC <= 12 ? 128 : 96);
    constexpr bool PIPE = SPL * (DW * P + 4 * P) + 40 <= REGCAP;
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
            const uint32_t xbytes = static_cast<uint32_t>(a.CC) * a.HS * a.TWs * PXB;  // full box
            for (int it = blockIdx.x; it < a.items; it += gridDim.x) {
                int part;
                int q = item_tile(a, it, part);
                const int g = q % a.G;
                q /= a.G;
                const int ct = q % a.col_tiles;
                q /= a.col_tiles;
                const int rt = q % a.row_tiles;
                const int sb = q / a.row_tiles;
                const int y0 = rt * a.TH * a.s_h;
                const int x0 = ct * a.SPRt * PC * SW;
                const int *blk_g = a.blk + g * a.n_chunks;
                for (int k = 0; k < a.n_chunks; ++k) {
                    mbar_wait(&empty[s], ph);
                    unsigned char *st = ring + s * a.stage_bytes;
                    const int lo = __ldg(blk_g + k), hi = __ldg(blk_g + k + 1);
                    const uint32_t eb = static_cast<uint32_t>(hi - lo);
                    mbar_expect_tx(&full[s], xbytes + eb);
                    tma_load_5d(st, &a.xmap, 0, x0, y0, k * a.CC, sb, &full[s]);
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
    const uint32_t base = ((tr * PR * a.s_h) * a.TWs + tcs * PC * SW) * PXB + lane * 4 * SPL;
    const uint32_t rs = a.s_h * a.TWs * PXB;  // bytes between a thread's two pixel rows
    const int hdr_bytes = a.ncls * a.DT * 8;
    int s = 0;
    uint32_t ph = 0;
    for (int it = blockIdx.x; it < a.items; it += gridDim.x) {
        int part;
        int q = item_tile(a, it, part);
        const int g = q % a.G;
        q /= a.G;
        const int ct = q % a.col_tiles;
        q /= a.col_tiles;
        const int rt = q % a.row_tiles;
        const int sb = q / a.row_tiles;
        const int r = rt * a.TH + tr * PR;
        const int col0 = (ct * a.SPRt + tcs) * PC;
        // pixel class (1x1 blocks): selects the runs without this pixel's halo taps
        const int cls = (a.ncls > 1 && r < a.Yh && col0 < a.Yw)
                            ? __ldg(a.rowcls + r) * a.ncls_c + __ldg(a.colcls + col0) : 0;

        A acc[DW][P];
#pragma unroll
        for (int i = 0; i < DW; ++i)
#pragma unroll
            for (int p = 0; p < P; ++p) zero_a(acc[i][p]);

        for (int k = 0; k < a.n_chunks; ++k) {
            const uint32_t st = smem_u32(ring + s * a.stage_bytes);
            mbar_wait(&full[s], ph);
            if (active) {
                const uint32_t xs = st + base;  // this thread's first pixel, tap (0,0,0)
                const uint32_t bp = st + a.x_stage_bytes;
                const uint32_t hdr = bp + (cls * a.DT + wc * DW) * 8, E = bp + hdr_bytes;
#pragma unroll
                for (int dw = 0; dw < DW; ++dw) {
                    const int2 h = lds_v2(hdr + dw * 8);  // run [h.x, h.y), h.x even
                    if (part >= 0 && dw % a.split != part) continue;
                    run_pairs<PC, PR, SW, SPL, PIPE>(acc[dw], xs, rs, E + h.x * 8, E + h.y * 8);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == a.S) {
                s = 0;
                ph ^= 1;
            }
        }

        // epilogue: ReLU (nn.py:96-98) then, if fused, the 2x2/2 max-pool
        // (nn.py:124-135); element (b, d, row, col) of the output layout is
        // obase + d*dstride + row*rstride + col*cstride (+ j*sstride for the lane's
        // j-th sample)
        if (!active || r >= a.Yh) continue;
        const int *pm = a.perm + g * a.DT + wc * DW;  // this warp's output channels (balanced)
        const bool pool = PR == 2 && a.ep.pool;
        const int orow = pool ? r / 2 : r, ocol = pool ? col0 / 2 : col0;
        const int b0 = sb * IL + lane * SPL;  // first sample of this lane
        const int oil = a.ep.out_padded ? a.ep.oil : 0;
        long long obase, dstride, sstride;
        int rstride, cstride;
        if (!a.ep.out_padded) {
            const int oh = pool ? a.Yh / 2 : a.Yh, ow = pool ? a.Yw / 2 : a.Yw;
            obase = ((long long)b0 * a.D * oh + orow) * ow + ocol;
            dstride = (long long)oh * ow;
            sstride = (long long)a.D * oh * ow;
            rstride = ow;
            cstride = 1;
        } else if (oil) {
            obase = (long long)(b0 / oil) * a.ep.o_sample_stride +
                    (((long long)orow + a.ep.oph) * a.ep.oWs + ocol + a.ep.opw) * oil + b0 % oil;
            dstride = (long long)a.ep.oHp * a.ep.oWs * oil;
            sstride = 1;
            rstride = a.ep.oWs * oil;
            cstride = oil;
        } else {
            obase = (long long)b0 * a.ep.o_sample_stride + ((long long)orow + a.ep.oph) * a.ep.oWs + ocol + a.ep.opw;
            dstride = (long long)a.ep.oHp * a.ep.oWs;
            sstride = a.ep.o_sample_stride;
            rstride = a.ep.oWs;
            cstride = 1;
        }
        const bool vec = SPL == 2 && oil == IL;  // the lane's two samples adjacent: one 8-byte store
        const int ncol = min(PC, a.Yw - col0);
        const int nrow = min(PR, a.Yh - r);
        const bool relu = a.ep.relu != 0;
#pragma unroll
        for (int dw = 0; dw < DW; ++dw) {
            if (part >= 0 && dw % a.split != part) continue;
            const int d = __ldg(pm + dw);
            if (d < 0) continue;
            const long long od = obase + d * dstride;
            float v[P][SPL];
#pragma unroll
            for (int p = 0; p < P; ++p) {
                unpack_a(acc[dw][p], v[p]);
#pragma unroll
                for (int j = 0; j < SPL; ++j)
                    if (relu) v[p][j] = v[p][j] > 0.0f ? v[p][j] : 0.0f;
            }
            // the thread's outputs: PC/2 pooled values of one row, or its P pixels
            float o[P][SPL];
            long long off[P];
            bool ok[P];
            int no = 0;
            if constexpr (PR == 2 && PC % 2 == 0) {
                if (pool) {
#pragma unroll
                    for (int c2 = 0; c2 < PC / 2; ++c2) {
#pragma unroll
                        for (int j = 0; j < SPL; ++j)
                            o[c2][j] = pool4(v[2 * c2][j], v[2 * c2 + 1][j], v[PC + 2 * c2][j],
                                             v[PC + 2 * c2 + 1][j]);
                        off[c2] = od + c2 * cstride;
                        ok[c2] = 2 * c2 < ncol;
                    }
                    no = PC / 2;
                }
            }
            if (no == 0) {
#pragma unroll
                for (int p = 0; p < P; ++p) {
#pragma unroll
                    for (int j = 0; j < SPL; ++j) o[p][j] = v[p][j];
                    off[p] = od + (p / PC) * rstride + (p % PC) * cstride;
                    ok[p] = (p / PC) < nrow && (p % PC) < ncol;
                }
                no = P;
            }
#pragma unroll
            for (int i = 0; i < P; ++i) {
                if (i >= no || !ok[i]) continue;
                if (vec) {
                    *reinterpret_cast<float2 *>(a.y + off[i]) = make_float2(o[i][0], o[i][SPL - 1]);
                } else {
#pragma unroll
                    for (int j = 0; j < SPL; ++j)
                        if (b0 + j < a.N) a.y[off[i] + j * sstride] = o[i][j];
                }
            }
        }
    }
}

template <int PC, int PR, int DW, int SW, int NWC, int SPL>
int launch_inst(const usc_plan *pl, const BiArgs &a, cudaStream_t st) {
    auto fn = k_bi<PC, PR, DW, SW, NWC, SPL>;
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
