// conv_bw.cuh -- the register-window variant of the batch-interleaved kernel (sm_100a).
//
// Same hot loop as k_bi (/root/reference/pkg/src/unsparse/kernels.py:87-96: per output
// element, entries in stored (c, kh, kw) order, multiply then add, each rounded) and the
// same producer / ring / epilogue, but a different operand path.  In k_bi every MAC
// reads its staged x value from shared memory (4 B per fp32 MAC, the 128 B/clk/SM LDS
// port is the roof).  Here a warp's DW output-channel slots share ONE merged entry
// stream per chunk, ordered by input row (c, kh): a ROW entry loads the window
// x[c][row + kh][col0 .. col0 + PC + KW - 2] (PC + KW - 1 values, SPL samples each)
// into registers once, and the MAC entries that follow -- every (slot dw, kw) of every
// slot with a nonzero at (c, kh, *) -- each run acc[dw][p] += theta * win[p + kw] from
// registers.  One x load now feeds ~DW*KW*density*PC/(PC+KW-1) MACs instead of one.
//
// The (slot, kw) of a MAC entry is static register indexing only through a dispatch:
// the entry's 6-bit code selects one of DW*KW unrolled case blocks through a PTX
// brx.idx jump table (SASS BRX; bw_asm.h, generated) -- the code is uniform across the
// warp, so no divergence.  The loop is direct-threaded: each case block prefetches the
// next entry and jumps.  Codes:
//   0 .. DW*KW-1   MAC (slot code / KW, tap code % KW), theta in the second word
//   62             ROW: load the window at byte offset (word & 0xffffff) of the stage
//   63             END of the run
// Per slot the MAC entries still come in ascending (c, kh, kw) order, so every
// accumulator sees exactly the reference's sequence of rounded operations.
//
// Thread block: PR = 1 (one output row per thread), column stride 1, BI64 (SPL = 2).
#pragma once
#include "conv_bi.cuh"
#include "bw_asm.h"

namespace usc_bi {

constexpr uint32_t BW_ROW = 62, BW_END = 63;

template <int KIND, int PC, int DW, int KW, int NWC, bool RES>
__global__ void __launch_bounds__((NWC + 1) * 32, 1) k_bw(const __grid_constant__ BiArgs a) {
    using O = Ops<KIND, 2>;
    using A = typename O::A;
    constexpr int P = PC;
    constexpr int PXB = O::EB * 64;
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
        // ---------------- producer warp (as k_bi) ----------------
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 1;
            const uint32_t xbytes = static_cast<uint32_t>(a.CC) * a.HS * a.TWs * PXB;
            for (int it = blockIdx.x; it < a.items; it += gridDim.x) {
                int q = it;
                const int g = q % a.G;
                q /= a.G;
                const int ct = q % a.col_tiles;
                q /= a.col_tiles;
                const int rt = q % a.row_tiles;
                const int sb = q / a.row_tiles;
                const int y0 = rt * a.TH * a.s_h;
                const int x0 = ct * a.SPRt * PC;
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
    const int tr = wsi / a.SPRt, tcs = wsi - tr * a.SPRt;
    const uint32_t base = ((tr * a.s_h) * a.TWs + tcs * PC) * PXB + lane * O::EB * 2;
    const int hdr_bytes = (a.WC * 8 + 15) & ~15;
    int s = 0;
    uint32_t ph = 0;
    for (int it = blockIdx.x; it < a.items; it += gridDim.x) {
        int q = it;
        int q2 = fdiv(q, a.fG);
        const int g = q - q2 * a.G;
        q = fdiv(q2, a.fCT);
        const int ct = q2 - q * a.col_tiles;
        const int sb = fdiv(q, a.fRT);
        const int rt = q - sb * a.row_tiles;
        const int r = rt * a.TH + tr;
        const int col0 = (ct * a.SPRt + tcs) * PC;

        A acc[DW][P];
#pragma unroll
        for (int i = 0; i < DW; ++i)
#pragma unroll
            for (int p = 0; p < P; ++p) O::zero(acc[i][p]);

        for (int k = 0; k < a.n_chunks; ++k) {
            const uint32_t st = smem_u32(ring + s * a.stage_bytes);
            mbar_wait(&full[s], ph);
            if (active) {
                const uint32_t bp = st + a.x_stage_bytes;
                const int2 h = lds_v2(bp + wc * 8);  // this channel subgroup's run, END-terminated
                BwAsm<KIND, PC, DW, KW>::run(acc, st + base, bp + hdr_bytes + h.x * 8);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == a.S) {
                s = 0;
                ph ^= 1;
            }
        }

        if (active && r < a.Yh) {
            if (a.fast) {
                int dch[DW];
                ResV<KIND, 2> rv[DW][P];
                fast_loads<KIND, PC, 1, DW, 2, RES>(a, g, wc, sb, r, col0, -1, lane, dch, rv);
                store_tile_fast<KIND, PC, 1, DW, 2, RES>(a, acc, sb, r, col0, lane, dch, rv);
                continue;
            }
            store_tile<KIND, PC, 1, DW, 2>(a, acc, g, wc, sb, r, col0, -1, lane);
        }
    }
}

template <int KIND, int PC, int DW, int KW, int NWC>
int launch_bw_inst(const usc_plan *pl, const BiArgs &a, cudaStream_t st) {
    constexpr bool HAS_RES = KIND == USC_F32 || KIND == USC_F16;
    const bool res = HAS_RES && a.fast && a.ep.residual;
    auto fn = res ? k_bw<KIND, PC, DW, KW, NWC, HAS_RES> : k_bw<KIND, PC, DW, KW, NWC, false>;
    static std::atomic<uint64_t> attr_res{0}, attr_plain{0};
    std::atomic<uint64_t> &attr = res ? attr_res : attr_plain;
    cudaError_t ae = ensure_smem_attr(fn, attr, 224 * 1024);
    if (ae != cudaSuccess) return usc::fail(USC_ERR_CUDA, "smem attribute: %s", cudaGetErrorString(ae));
    fn<<<static_cast<unsigned>(pl->grid_x), (NWC + 1) * 32, pl->smem_bytes, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return usc::fail(USC_ERR_CUDA, "k_bw launch: %s", cudaGetErrorString(e));
    return USC_OK;
}

int launch_bw(const usc_plan *pl, const BiArgs &a, cudaStream_t st);

}  // namespace usc_bi
