// conv_bt.cuh -- the tensor-memory-fed variant of the BI64 fp32 kernel (kernel 4).
//
// Same math, layouts, entry blocks and epilogue as k_bi (conv_bi.cuh), but the
// compute warps read the staged input from TENSOR MEMORY instead of shared memory:
// the shared-memory port (128 B/clk/SM) bounds k_bi at 32 fp32 MAC/clk/SM, while
// tcgen05.ld streams ~300 B/clk/SM (tools/tmem_bench.cu, tools/tmem_mac_bench.cu).
//
//   * TMA still lands each chunk ([CC][HS][TWs][64] fp32) in a shared-memory ring;
//   * the compute warps of each lane quarter copy the chunk into that quarter's
//     TMEM lanes (LDS.64 -> tcgen05.st.32x32b.x16): lane l of quarter q holds samples
//     2l, 2l+1, position j (= (c*HS + row)*TWs + col) in columns 2j, 2j+1 -- every
//     quarter holds the whole chunk, since a warp can only read its own quarter;
//     two 256-column buffers alternate between chunks (<= 128 positions each);
//   * a named barrier per quarter publishes the fill; then each warp runs its output
//     channels' entry runs, four entries per tcgen05.wait::ld: one
//     tcgen05.ld.32x32b.x(2*PC) per pixel row per entry (PC pixels x 2 samples), two
//     FMUL + one FADD2 per pixel (the reference's multiply-then-add order).
#pragma once
#include "conv_bi.cuh"

namespace usc_bi {

template <int N>
__device__ __forceinline__ void ldtm(uint32_t a, float (&v)[N]) {
    static_assert(N == 4 || N == 8 || N == 16, "x4/x8/x16");
    if constexpr (N == 4)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
                     : "r"(a));
    else if constexpr (N == 8)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                     : "r"(a));
    else
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
            "%14, %15}, [%16];"
            : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
              "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
            : "r"(a));
}
__device__ __forceinline__ void sttm16(uint32_t a, const float (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16};" ::"r"(a),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
        "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]));
}
__device__ __forceinline__ void sttm2(uint32_t a, float v0, float v1) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(a), "f"(v0), "f"(v1));
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// U entries (U <= 4) of a run: PR tcgen05.ld per entry, one wait, then the
// products and the adds in stored order
template <int PC, int PR, int U>
__device__ __forceinline__ void bt_entries(unsigned long long (&acc)[PC * PR], uint32_t col, uint32_t rcol,
                                           const int4 &n01, const int4 &n23) {
    float v[U][PR][2 * PC];
    const int off[4] = {n01.x, n01.z, n23.x, n23.z};
    const int th[4] = {n01.y, n01.w, n23.y, n23.w};
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
        for (int r = 0; r < PR; ++r) ldtm<2 * PC>(col + off[u] + r * rcol, v[u][r]);
    tm_wait_ld();
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const float t = __int_as_float(th[u]);
#pragma unroll
        for (int r = 0; r < PR; ++r)
#pragma unroll
            for (int c = 0; c < PC; ++c)
                fadd2(acc[r * PC + c], __fmul_rn(t, v[u][r][2 * c]), __fmul_rn(t, v[u][r][2 * c + 1]));
    }
}

template <int PC, int PR, int DW, int NWC>
__global__ void __launch_bounds__((NWC + 1) * 32, 1) k_bt(const __grid_constant__ BiArgs a) {
    static_assert(NWC % 4 == 0, "compute warps fill TMEM per lane quarter");
    using A = unsigned long long;
    constexpr int P = PC * PR;
    constexpr int PXB = 256;         // staged bytes per pixel (64 fp32 samples)
    constexpr int MATES = NWC / 4;   // compute warps per lane quarter
    constexpr int UB = P <= 4 ? 4 : 2;  // entries per tcgen05.wait::ld (registers for 2*P*UB values)
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint32_t taddr_s;
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
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tm_fence_before();
    __syncthreads();
    tm_fence_after();

    if (warp == NWC) {
        // ---------------- producer warp (as k_bi) ----------------
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 1;
            const uint32_t xbytes = static_cast<uint32_t>(a.CC) * a.HS * a.TWs * PXB;
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
    const int quarter = warp & 3, mate = warp >> 2;
    const uint32_t tq = taddr_s + (static_cast<uint32_t>(32 * quarter) << 16);
    const int wsi = warp % a.WS, wc = warp / a.WS;
    const bool active = wc < a.WC;
    const int tr = wsi / a.SPRt, tcs = wsi - tr * a.SPRt;
    const uint32_t base_col = static_cast<uint32_t>(((tr * PR * a.s_h) * a.TWs + tcs * PC) * 2);
    const uint32_t rcol = static_cast<uint32_t>(a.s_h * a.TWs * 2);
    const int npos = a.CC * a.HS * a.TWs;  // positions of one chunk (<= 128)
    const int share = ((npos + MATES - 1) / MATES + 7) / 8 * 8;
    const int j0 = min(npos, mate * share), j1 = min(npos, j0 + share);
    const int hdr_bytes = (a.ncls * a.DT * 8 + 15) & ~15;  // entries start 16-B aligned
    int s = 0, kk = 0;
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
        const int cls = (a.ncls > 1 && r < a.Yh && col0 < a.Yw)
                            ? __ldg(a.rowcls + r) * a.ncls_c + __ldg(a.colcls + col0) : 0;

        A acc[DW][P];
#pragma unroll
        for (int i = 0; i < DW; ++i)
#pragma unroll
            for (int p = 0; p < P; ++p) acc[i][p] = 0ull;

        for (int k = 0; k < a.n_chunks; ++k, ++kk) {
            const uint32_t st = smem_u32(ring + s * a.stage_bytes);
            const uint32_t buf = tq + static_cast<uint32_t>((kk & 1) * 256);
            mbar_wait(&full[s], ph);
            // fill this quarter's copy of the chunk: positions [j0, j1) of this warp
            {
                int j = j0;
#pragma unroll 1
                for (; j + 8 <= j1; j += 8) {
                    float v[16];
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];"
                                     : "=f"(v[2 * i]), "=f"(v[2 * i + 1])
                                     : "r"(st + (j + i) * PXB + lane * 8));
                    sttm16(buf + 2 * j, v);
                }
#pragma unroll 1
                for (; j < j1; ++j) {
                    float v0, v1;
                    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v0), "=f"(v1) : "r"(st + j * PXB + lane * 8));
                    sttm2(buf + 2 * j, v0, v1);
                }
            }
            tm_wait_st();
            tm_fence_before();
            named_bar(1 + quarter, 32 * MATES);
            tm_fence_after();
            if (active) {
                const uint32_t bp = st + a.x_stage_bytes;
                const uint32_t hdr = bp + (cls * a.DT + wc * DW) * 8, E = bp + hdr_bytes;
                const uint32_t col = buf + base_col;
#pragma unroll
                for (int dw = 0; dw < DW; ++dw) {
                    const int2 h = lds_v2(hdr + dw * 8);  // run [h.x, h.y), h.x even
                    if (part >= 0 && dw % a.split != part) continue;
                    uint32_t ep = E + h.x * 8;
                    const uint32_t ee = E + h.y * 8;
#pragma unroll 1
                    for (; ep + 8 * UB <= ee; ep += 8 * UB) {
                        const int4 n01 = lds_v4(ep);
                        bt_entries<PC, PR, UB>(acc[dw], col, rcol, n01, UB == 4 ? lds_v4(ep + 16) : n01);
                    }
                    const int rem = static_cast<int>(ee - ep) / 8;  // < UB (reads stay in the slack)
                    if (UB == 4 && rem == 3) bt_entries<PC, PR, 3>(acc[dw], col, rcol, lds_v4(ep), lds_v4(ep + 16));
                    else if (UB == 4 && rem == 2) bt_entries<PC, PR, 2>(acc[dw], col, rcol, lds_v4(ep), lds_v4(ep));
                    else if (rem == 1) bt_entries<PC, PR, 1>(acc[dw], col, rcol, lds_v4(ep), lds_v4(ep));
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == a.S) {
                s = 0;
                ph ^= 1;
            }
        }
        if (active && r < a.Yh) store_tile<USC_F32, PC, PR, DW, 2>(a, acc, g, wc, sb, r, col0, part, lane);
    }
    // every compute warp is done with tensor memory
    tm_fence_before();
    named_bar(5, 32 * NWC);
    tm_fence_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

template <int PC, int PR, int DW, int NWC>
int launch_bt_inst(const usc_plan *pl, const BiArgs &a, cudaStream_t st) {
    auto fn = k_bt<PC, PR, DW, NWC>;
    static std::atomic<uint64_t> attr{0};
    cudaError_t ae = ensure_smem_attr(fn, attr, 224 * 1024);
    if (ae != cudaSuccess) return usc::fail(USC_ERR_CUDA, "smem attribute: %s", cudaGetErrorString(ae));
    fn<<<static_cast<unsigned>(pl->grid_x), (NWC + 1) * 32, pl->smem_bytes, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return usc::fail(USC_ERR_CUDA, "k_bt launch: %s", cudaGetErrorString(e));
    return USC_OK;
}

int launch_bt(const usc_plan *pl, const BiArgs &a, cudaStream_t st);

}  // namespace usc_bi
