// dense_tc.cu -- the dense backend of the per-layer dispatcher on the 5th-generation
// tensor cores: an implicit-GEMM binary16 convolution that reads and writes the network's
// resident BI64 layout directly (no NHWC transposes), tcgen05.mma with the accumulator in
// tensor memory.  For binary16 networks only (the north star's 1e-2 tolerance path):
// tensor-core sums are not the reference's sequential fp32 order.
//
// GEMM view of one CTA tile (one output row y, TWP output pixels x0.., one 64-sample
// block, 128 output channels d0..):
//   D[d][(x, s)] = sum_{t = (kh, kw), c} W[d][t][c] * X[c][s*y + kh][s*x + kw][sample s]
//   M = 128 (d), N = TWP * 64 (pixels x samples), K = taps * C.
// Operands (TMA, 128-byte swizzle, 1024-B aligned stages):
//   A = weights [D][taps*C] binary16, K-major: box [64 k][128 d] (16 KB per stage);
//   B = activations: per tile pixel one box [64 samples][1][1][64 channels] of the BI64
//       tensor -> [64 c][64 s] (8 KB), i.e. MN-major (samples contiguous), one 128-B
//       swizzle row per channel; the TWP boxes of a stage are the MN atoms of B.
// MMAs of K = 16 (tcgen05.mma.cta_group::1.kind::f16, M128 x N, fp32 acc), see k_dtc for
// the stage shapes.  Warp roles: warps 0-7 epilogue (TMEM lane quarter = warp % 4), warp 8
// TMA producer and TMEM owner, warp 9 MMA issuer.  Epilogue (each warp on its own 32
// channels and every other pixel): tcgen05.ld, binary16 rounding with saturation (cvt.satfinite), optional
// residual add (binary16) + saturation, ReLU (NaN -> 0), TMA stores of [32 c][64 s] boxes
// into the output layout (halo untouched).
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "usc_internal.h"

using namespace usc_dev;

namespace {

#ifdef DTC_TRACE  // timeline probe (tools/dtc_trace.cu): %globaltimer stamps per CTA, never in the product build
__device__ unsigned long long g_dtc_trace[1024][8];
__device__ __forceinline__ void dtc_stamp(int k) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_dtc_trace[blockIdx.x][k] = t;
}
#define DTC_STAMP(k) dtc_stamp(k)
#else
#define DTC_STAMP(k)
#endif

constexpr int kKC = 64;               // channels (K) per stage and tap
constexpr int kABytes = 128 * kKC * 2;  // 16 KB
constexpr int kBPix = kKC * 64 * 2;     // 8 KB per pixel box

struct DtcArgs {
    CUtensorMap xmap, wmap, ymap, rmap;  // activations, weights, output, shortcut (TMA)
    void *y;
    const void *res;
    LayoutD Lo, Lr;
    int C, D, Kh, Kw, stride, offh, offw;  // input coord = stride*o + k + off
    int Yh, Yw, NB, relu;
    int m_blocks, x_tiles;
    int k_iters, cb;  // k_iters = taps * cb, cb = C / 64
    int splits, kper;  // split-K: work item = (tile, split), split s runs k-iterations [s*kper, (s+1)*kper)
    float *part;       // split-K partial sums [tile][split][N columns][128 rows] fp32
    int *cnt;          // split-K arrival counter per tile (zero between launches)
    int xrow;          // window kernels: xmap is (s, c, x, y, nb) and one box covers the row window
    int pool;          // fused 2x2 max-pool (window kernel, 4-pixel tiles): a CTA runs the two
                       // output rows of a pool window back to back; y is the pooled layout
};

__device__ __forceinline__ void mbar_wait_bounded(uint64_t *bar, uint32_t parity) {
    // a descriptor or transaction-count bug must fail the launch, not hang the GPU
    uint32_t ok = 0;
    for (long long it = 0; it < (1LL << 27) && !ok; ++it)
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    if (!ok) __trap();
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tma_store_5d(const CUtensorMap *map, const void *src, int c0, int c1, int c2, int c3,
                                             int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
        : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, %0;" ::"n"(8 * 32) : "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_5d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, int c3, int c4,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
        : "memory");
}

// UMMA shared-memory descriptors (sm_100 format, version 1), 128-byte swizzle:
//   K-major A tile [rows][64 k]: rows 128 B apart, 8-row groups SBO = 1024 B;
//   MN-major B tile: 128-B rows = 64 MN elements, K rows 128 B apart (8-row groups
//   SBO = 1024 B), MN atoms (tile pixels) LBO = 8 KB apart.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;  // version 1 (Blackwell)
    d |= 2ull << 61;  // SWIZZLE_128B
    return d;
}

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// Epilogue: kEW warps, two per TMEM lane quarter (warp w: channels 32 (w % 4) .. +31 of
// the tile, the tile's even (w < 4) or odd pixels).  Staging per warp: kOS output slots
// and, with a shortcut, kRS shortcut slots of one pixel box [32 channels][64 samples]
// binary16 = 4 KB each (128-byte swizzle, 1024-B aligned).
constexpr int kWarpBox = 32 * 128;
constexpr int kEW = 8, kOS = 1, kRS = 2;
constexpr int kThreads = (kEW + 2) * 32;  // + TMA producer warp + MMA warp

// ring depth: the ring and the staging slots share the 227 KB of dynamic shared memory
template <int TWP, bool WIN, bool RES>
constexpr int dtc_stages() {
    return WIN ? 2 : (TWP == 4 ? (RES ? 2 : 3) : 4);
}

__device__ __forceinline__ uint32_t cvt_f16x2_sat(float lo, float hi) {  // +-inf/overflow -> +-65504, NaN kept
    uint32_t r;
    asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ uint32_t add_f16x2_sat(uint32_t x, uint32_t y) {  // binary16 sum, saturated, NaN kept
    uint32_t r;
    asm("{\n.reg .b32 t;\nadd.rn.f16x2 t, %1, %2;\nmin.NaN.f16x2 t, t, %3;\nmax.NaN.f16x2 %0, t, %4;\n}\n"
        : "=r"(r)
        : "r"(x), "r"(y), "r"(0x7bff7bffu), "r"(0xfbfffbffu));
    return r;
}
__device__ __forceinline__ uint32_t hmax_f16x2(uint32_t x, uint32_t y) {  // NaN-free operands (post-ReLU)
    uint32_t r;
    asm("max.f16x2 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(y));
    return r;
}
__device__ __forceinline__ uint32_t relu_f16x2(uint32_t x) {  // max(x, 0): negatives and NaN -> 0
    uint32_t r;
    asm("max.f16x2 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(0u));
    return r;
}

// Persistent CTA (one per SM), tiles round-robin.  WIN (3x3, stride 1): a stage is one
// (kh, 64-channel chunk): the TWP+2 input pixels of the row (one 8-KB box each) and the A
// tiles of the 3 taps kw = 0..2 -- each pixel box is read once for 3 taps (tap kw's B
// operand is the MN atoms kw .. kw+TWP-1 of the window); 12 MMAs per stage.  Otherwise a
// stage is one (tap, chunk): TWP boxes + one A tile, 4 MMAs.  Two TMEM accumulators
// (2 x N fp32 columns): the epilogue of tile i overlaps the main loop of tile i+1.
template <int TWP, bool WIN, bool RES>
__global__ void __launch_bounds__(kThreads, 1) k_dtc(const __grid_constant__ DtcArgs a) {
    constexpr int N = TWP * 64;
    constexpr int NA = WIN ? 3 : 1;                 // A tiles (taps) per stage
    constexpr int NBX = WIN ? TWP + 2 : TWP;        // pixel boxes per stage
    constexpr int kStage = NA * kABytes + NBX * kBPix;
    constexpr int S = dtc_stages<TWP, WIN, RES>();  // ring depth
    constexpr uint32_t kCols = 2 * N;               // two accumulators
    static_assert(kEW == 8, "epi_sync counts 8 epilogue warps");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char *ostage = smem + S * kStage;           // [kEW warps][kOS] output boxes
    unsigned char *rstage = ostage + kEW * kOS * kWarpBox;  // [kEW warps][kRS] shortcut boxes (RES)
    uint64_t *full = reinterpret_cast<uint64_t *>(rstage + (RES ? kEW * kRS * kWarpBox : 0));
    uint64_t *empty = full + S;
    uint64_t *tfull = empty + S;   // [2]
    uint64_t *tempty = tfull + 2;  // [2]
    uint64_t *rfull = tempty + 2;  // [kEW warps][kRS] shortcut box landed
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(rfull + kEW * kRS);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles = a.m_blocks * a.x_tiles * a.Yh * a.NB;
    const int kiters = WIN ? a.Kh * a.cb : a.k_iters;
    const int items = tiles * a.splits;
    auto krange = [&](int t, int &tile, int &sp, int &k0, int &k1) {  // work item -> tile, k-iteration range
        tile = t / a.splits;
        sp = t - tile * a.splits;
        k0 = sp * a.kper;
        k1 = min(kiters, k0 + a.kper);
    };

    if (threadIdx.x == 0) {
        DTC_STAMP(0);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], kEW);  // one arrive per epilogue warp
        }
        for (int b = 0; b < kEW * kRS; ++b) mbar_init(&rfull[b], 1);
        fence_mbar_init();
    }
    if (warp == kEW) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(kCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) DTC_STAMP(1);
    if (threadIdx.x == 0) {  // descriptors into the TMA unit while the previous kernel drains
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.xmap)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.wmap)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.ymap)) : "memory");
        if (RES) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.rmap)) : "memory");
    }
    pdl_release();
    // every global access below waits for the previous kernel's output, except the producer's
    // weight tiles for the first S stages (constant data, loaded while the previous kernel drains)
    if (warp != kEW) pdl_wait();

    auto decode = [&](int t, int &mb, int &xt, int &yo, int &nb) {
        const int r = a.pool ? (t & 1) : 0;  // pool: consecutive tiles = rows 2y, 2y+1
        if (a.pool) t >>= 1;
        mb = t % a.m_blocks;
        t /= a.m_blocks;
        xt = t % a.x_tiles;
        t /= a.x_tiles;
        const int rows = a.pool ? a.Yh >> 1 : a.Yh;
        yo = t % rows;
        nb = t / rows;
        if (a.pool) yo = 2 * yo + r;
    };
    auto item_at = [&](int j) -> int {  // this CTA's j-th work item, -1 past the end
        if (a.pool) {
            const int p = blockIdx.x + (j >> 1) * gridDim.x;
            return p < (items >> 1) ? 2 * p + (j & 1) : -1;
        }
        const int t = blockIdx.x + j * gridDim.x;
        return t < items ? t : -1;
    };

    if (warp == kEW) {
        // ---------------- TMA producer ----------------
        // The stage's boxes are issued by parallel lanes, one box per lane: successive TMA
        // instructions of one thread issue ~370 clocks apart (tools/tma_rate_bench.cu), so a
        // single issuing lane caps the stream at ~20-35 B/clk per SM.
        auto load_a = [&](unsigned char *st, uint64_t *bar, int i, int mb) {  // weight tiles of k-iteration i
            if constexpr (WIN) {
                const int kh = i / a.cb, cb = i - kh * a.cb;
                if (lane < 3) tma_load_2d(st + lane * kABytes, &a.wmap, (kh * 3 + lane) * a.C + cb * kKC, mb * 128, bar);
            } else {
                const int tap = i / a.cb, cb = i - tap * a.cb;
                if (lane == 0) tma_load_2d(st, &a.wmap, tap * a.C + cb * kKC, mb * 128, bar);
            }
        };
        auto load_b = [&](unsigned char *st, uint64_t *bar, int i, int xt, int yo, int nb) {  // activation boxes
            if constexpr (WIN) {
                const int kh = i / a.cb, cb = i - kh * a.cb;
                if (a.xrow) {
                    if (lane == 3)
                        tma_load_5d(st + NA * kABytes, &a.xmap, 0, cb * kKC, xt * TWP + a.offw, yo + kh + a.offh, nb, bar);
                } else if (lane >= 3 && lane < 3 + NBX) {
                    tma_load_5d(st + NA * kABytes + (lane - 3) * kBPix, &a.xmap, 0, xt * TWP + (lane - 3) + a.offw,
                                yo + kh + a.offh, cb * kKC, nb, bar);
                }
            } else {
                const int tap = i / a.cb, cb = i - tap * a.cb;
                const int kh = tap / a.Kw, kw = tap - kh * a.Kw;
                if (lane >= 1 && lane <= TWP)
                    tma_load_5d(st + kABytes + (lane - 1) * kBPix, &a.xmap, 0, a.stride * (xt * TWP + lane - 1) + kw + a.offw,
                                a.stride * yo + kh + a.offh, cb * kKC, nb, bar);
            }
        };
        {  // the first S stages' weight tiles go out before the wait on the previous kernel
            int it = 0;
            for (int j = 0, t; it < S && (t = item_at(j)) >= 0; ++j) {
                int tile, sp, k0, k1, mb, xt, yo, nb;
                krange(t, tile, sp, k0, k1);
                decode(tile, mb, xt, yo, nb);
                for (int i = k0; i < k1 && it < S; ++i, ++it) {
                    if (lane == 0) mbar_expect_tx(&full[it], kStage);
                    __syncwarp();
                    load_a(smem + it * kStage, &full[it], i, mb);
                }
            }
        }
        pdl_wait();
        int it = 0;  // running stage counter
        for (int j = 0, t; (t = item_at(j)) >= 0; ++j) {
            int tile, sp, k0, k1, mb, xt, yo, nb;
            krange(t, tile, sp, k0, k1);
            decode(tile, mb, xt, yo, nb);
            for (int i = k0; i < k1; ++i, ++it) {
                const int s = it % S;
                unsigned char *st = smem + s * kStage;
                if (it >= S) {
                    mbar_wait_bounded(&empty[s], ((it / S) - 1) & 1);
                    if (lane == 0) mbar_expect_tx(&full[s], kStage);
                    __syncwarp();
                    load_a(st, &full[s], i, mb);
                }
                load_b(st, &full[s], i, xt, yo, nb);
            }
        }
    } else if (warp == kEW + 1) {
        // ---------------- MMA issuer ----------------
        const uint32_t idesc = (1u << 4) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        int it = 0, lt = 0;
        for (int t; (t = item_at(lt)) >= 0; ++lt) {
            int tile, sp, k0, k1;
            krange(t, tile, sp, k0, k1);
            const int ab = lt & 1;
            if (lt >= 2) mbar_wait_bounded(&tempty[ab], ((lt >> 1) - 1) & 1);  // epilogue drained it
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t acc = tmem + ab * N;
            for (int i = k0; i < k1; ++i, ++it) {
                const int s = it % S;
                mbar_wait_bounded(&full[s], (it / S) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (lane == 0 && it == 0) DTC_STAMP(2);
                if (lane == 0) {
                    const uint32_t abase = smem_u32(smem + s * kStage), bbase = abase + NA * kABytes;
#pragma unroll
                    for (int q = 0; q < NA; ++q)
#pragma unroll
                        for (int k = 0; k < kKC / 16; ++k) {
                            const uint64_t ad = desc_sw128(abase + q * kABytes + k * 32, 16, 1024);
                            const uint64_t bd = desc_sw128(bbase + q * kBPix + k * 16 * 128, kBPix, 1024);
                            umma_f16(acc, ad, bd, idesc, (i > k0 || q > 0 || k > 0) ? 1u : 0u);
                        }
                    umma_commit(&empty[s]);
                    if (i == k1 - 1) umma_commit(&tfull[ab]);
                    if (i == k1 - 1 && lt < 2) DTC_STAMP(3 + lt);
                }
                __syncwarp();
            }
        }
    } else {
        // ---------------- epilogue (warp w: TMEM lanes 32 (w % 4) .. +31) ----------------
        // Each warp owns output channels mb*128 + 32 (w % 4) .. +31 and every other pixel of
        // every tile, and runs on its own: per output pixel, TMEM -> registers (64 samples
        // of its channel row), binary16 with saturation, + shortcut, ReLU, 128-B rows into a
        // swizzled 4-KB staging box, one TMA store of [32 channels][64 samples].  The
        // shortcut boxes stream in through a kRS-deep per-warp ring issued ahead (HBM
        // latency off the critical path).  j counts this warp's pixels (CTA pixel 2j + half).
        const int ch0 = (warp & 3) * 32, half = warp >> 2;
        unsigned char *ost = ostage + warp * kOS * kWarpBox;
        unsigned char *rst = rstage + warp * kRS * kWarpBox;
        uint64_t *rbar = rfull + warp * kRS;
        auto pixel_coords = [&](int q, int &mb, int &xo, int &yo, int &nb) {  // q-th pixel of this CTA
            const int t = item_at(q / TWP);
            int xt;
            decode(t, mb, xt, yo, nb);
            xo = xt * TWP + q % TWP;
        };
        const int my_pixels = ((tiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x) * (TWP / 2);
        const bool res = RES && a.res != nullptr;
        auto issue_res = [&](int jj) {  // lane 0: shortcut box of this warp's channels at its pixel jj
            int mb, xo, yo, nb;
            pixel_coords(2 * jj + half, mb, xo, yo, nb);
            const int slot = jj % kRS;
            mbar_expect_tx(&rbar[slot], kWarpBox);
            tma_load_5d(rst + slot * kWarpBox, &a.rmap, 0, xo + a.Lr.pw, yo + a.Lr.ph, mb * 128 + ch0, nb, &rbar[slot]);
        };
        if (res && lane == 0)
            for (int jj = 0; jj < kRS && jj < my_pixels; ++jj) issue_res(jj);
        auto tmem_ld64 = [&](uint32_t addr, uint32_t(&v)[64]) {  // 64 fp32 columns of this warp's lanes
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, "
                "[%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                  "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                  "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                  "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(addr));
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, "
                "[%32];"
                : "=r"(v[32]), "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]), "=r"(v[38]),
                  "=r"(v[39]), "=r"(v[40]), "=r"(v[41]), "=r"(v[42]), "=r"(v[43]), "=r"(v[44]), "=r"(v[45]),
                  "=r"(v[46]), "=r"(v[47]), "=r"(v[48]), "=r"(v[49]), "=r"(v[50]), "=r"(v[51]), "=r"(v[52]),
                  "=r"(v[53]), "=r"(v[54]), "=r"(v[55]), "=r"(v[56]), "=r"(v[57]), "=r"(v[58]), "=r"(v[59]),
                  "=r"(v[60]), "=r"(v[61]), "=r"(v[62]), "=r"(v[63])
                : "r"(addr + 32));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        };
        // one output pixel of this warp's 32 channels: fp32 sums -> binary16 (+ shortcut,
        // ReLU) -> staging box -> TMA store; q counts this warp's pixels
        // one output box of this warp's 32 channels: 32 packed binary16 words per lane ->
        // staging box -> TMA store; q counts this warp's stores
        auto store_box = [&](const uint32_t(&h)[32], int q, int mb, int xo, int yo, int nb, bool live) {
            // staging slot q % kOS is free once the store issued kOS boxes ago has read it
            unsigned char *obox = ost + (q % kOS) * kWarpBox;
            if (lane == 0) bulk_wait_read<kOS - 1>();
            __syncwarp();
            unsigned char *orow = obox + lane * 128;
#pragma unroll
            for (int c = 0; c < 8; ++c)
                *reinterpret_cast<uint4 *>(orow + ((c ^ (lane & 7)) << 4)) =
                    make_uint4(h[4 * c], h[4 * c + 1], h[4 * c + 2], h[4 * c + 3]);
            fence_proxy_async();  // the staged rows -> visible to the TMA engine
            __syncwarp();
            if (lane == 0 && live && xo < (a.pool ? a.Yw >> 1 : a.Yw))
                tma_store_5d(&a.ymap, obox, 0, xo + a.Lo.pw, yo + a.Lo.ph, mb * 128 + ch0, nb);
        };
        // one output pixel: fp32 sums -> binary16 (+ shortcut, ReLU) -> store_box
        auto emit = [&](const uint32_t(&v)[64], int q, int mb, int xo, int yo, int nb, bool live) {
            uint32_t h[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) h[k] = cvt_f16x2_sat(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1]));
            if (res) {
                const int slot = q % kRS;
                mbar_wait_bounded(&rbar[slot], (q / kRS) & 1);
                const unsigned char *rrow = rst + slot * kWarpBox + lane * 128;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const uint4 r = *reinterpret_cast<const uint4 *>(rrow + ((c ^ (lane & 7)) << 4));
                    h[4 * c] = add_f16x2_sat(h[4 * c], r.x);
                    h[4 * c + 1] = add_f16x2_sat(h[4 * c + 1], r.y);
                    h[4 * c + 2] = add_f16x2_sat(h[4 * c + 2], r.z);
                    h[4 * c + 3] = add_f16x2_sat(h[4 * c + 3], r.w);
                }
                __syncwarp();  // every lane has read the slot: refill it kRS pixels ahead
                if (lane == 0 && q + kRS < my_pixels) {
                    fence_proxy_async();
                    issue_res(q + kRS);
                }
            }
            if (a.relu) {
#pragma unroll
                for (int k = 0; k < 32; ++k) h[k] = relu_f16x2(h[k]);
            }
            store_box(h, q, mb, xo, yo, nb, live);
        };
        __shared__ int s_last;  // split-K: this CTA completed the tile's last split
        uint32_t keep[32];      // pool: the horizontal maxima of the window's first row
        int lt = 0, q = 0;
        for (int t; (t = item_at(lt)) >= 0; ++lt) {
            int tile, sp, k0, k1, mb, xt, yo, nb;
            krange(t, tile, sp, k0, k1);
            decode(tile, mb, xt, yo, nb);
            const int ab = lt & 1;
            const bool live = mb * 128 + ch0 < a.D;  // rows past D (64-channel layers) are not stored
            mbar_wait_bounded(&tfull[ab], (lt >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (warp == 0 && lane == 0 && lt < 2) DTC_STAMP(5 + lt);
            const uint32_t taddr = tmem + ab * N + ((uint32_t)(ch0) << 16);
            if constexpr (WIN && TWP == 4 && !RES) {
                if (a.pool) {  // warp half h: pixels 2h, 2h+1 = one pool window's columns
                    uint32_t v[64], hm[32];
                    tmem_ld64(taddr + (2 * half) * 64, v);
#pragma unroll
                    for (int k = 0; k < 32; ++k)
                        hm[k] = relu_f16x2(cvt_f16x2_sat(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1])));
                    tmem_ld64(taddr + (2 * half + 1) * 64, v);
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[ab]);
#pragma unroll
                    for (int k = 0; k < 32; ++k)
                        hm[k] = hmax_f16x2(hm[k], relu_f16x2(cvt_f16x2_sat(__uint_as_float(v[2 * k]),
                                                                            __uint_as_float(v[2 * k + 1]))));
                    if ((lt & 1) == 0) {  // the window's first row: hold it
#pragma unroll
                        for (int k = 0; k < 32; ++k) keep[k] = hm[k];
                        continue;
                    }
#pragma unroll
                    for (int k = 0; k < 32; ++k) hm[k] = hmax_f16x2(keep[k], hm[k]);
                    store_box(hm, q++, mb, xt * 2 + half, yo >> 1, nb, live);
                    continue;
                }
            }
            if (a.splits == 1) {
#pragma unroll 1
                for (int px = half; px < TWP; px += 2, ++q) {
                    uint32_t v[64];
                    tmem_ld64(taddr + px * 64, v);
                    if (px + 2 >= TWP) {  // this warp's columns of the accumulator are in registers: release
                        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[ab]);
                    }
                    emit(v, q, mb, xt * TWP + px, yo, nb, live);
                }
                continue;
            }
            // split-K: the partial sums go to the workspace (column-major, 128 B per column
            // and warp); the CTA that completes a tile's last split sums the splits in split
            // order (deterministic) and runs the epilogue
            float *mine = a.part + ((size_t)tile * a.splits + sp) * (N * 128) + ch0 + lane;
#pragma unroll 1
            for (int px = half; px < TWP; px += 2) {
                uint32_t v[64];
                tmem_ld64(taddr + px * 64, v);
                if (px + 2 >= TWP) {
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[ab]);
                }
#pragma unroll
                for (int c = 0; c < 64; ++c) mine[(px * 64 + c) * 128] = __uint_as_float(v[c]);
            }
            __threadfence();
            epi_sync();
            if (threadIdx.x == 0) s_last = atomicAdd(&a.cnt[tile], 1) == a.splits - 1;
            epi_sync();
            if (!s_last) continue;
            __threadfence();
            const float *base = a.part + (size_t)tile * a.splits * (N * 128) + ch0 + lane;
#pragma unroll 1
            for (int px = half; px < TWP; px += 2, ++q) {
                float acc[64];  // split 0, then + split 1, 2, ... (64 independent loads per split)
#pragma unroll
                for (int c = 0; c < 64; ++c) acc[c] = __ldcg(base + (px * 64 + c) * 128);
#pragma unroll 1
                for (int sp2 = 1; sp2 < a.splits; ++sp2) {
                    const float *ps = base + (size_t)sp2 * (N * 128) + px * 64 * 128;
                    float t[64];
#pragma unroll
                    for (int c = 0; c < 64; ++c) t[c] = __ldcg(ps + c * 128);
#pragma unroll
                    for (int c = 0; c < 64; ++c) acc[c] += t[c];
                }
                uint32_t v[64];
#pragma unroll
                for (int c = 0; c < 64; ++c) v[c] = __float_as_uint(acc[c]);
                emit(v, q, mb, xt * TWP + px, yo, nb, live);
            }
            if (threadIdx.x == 0) a.cnt[tile] = 0;  // ready for the next launch
        }
        if (lane == 0) bulk_wait_all();
        if (warp == 0 && lane == 0) DTC_STAMP(7);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == kEW) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols));
    }
}

template <int TWP, bool WIN, bool RES>
constexpr int dtc_smem() {
    constexpr int NA = WIN ? 3 : 1, NBX = WIN ? TWP + 2 : TWP, S = dtc_stages<TWP, WIN, RES>();
    return S * (NA * kABytes + NBX * kBPix) + kEW * (kOS + (RES ? kRS : 0)) * kWarpBox + 1024 + 256;
}

template <int TWP, bool WIN, bool RES>
cudaError_t launch_dtc(const DtcArgs &a, int tiles, cudaStream_t st) {
    static std::atomic<uint64_t> attr{0};
    constexpr int smem = dtc_smem<TWP, WIN, RES>();
    static_assert(smem <= 227 * 1024, "k_dtc shared memory");
    cudaError_t e = ensure_smem_attr(k_dtc<TWP, WIN, RES>, attr, smem);
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    int sms = usc_device_sm_count(dev);
    if (sms <= 0) sms = 148;
    return launch_pdl(k_dtc<TWP, WIN, RES>, dim3((unsigned)(tiles < sms ? tiles : sms)), dim3(kThreads), smem, st, a);
}

// ---------------------------------------------------------------------------------------
// k_dts: 64-output-channel layers with the operands swapped.  M = 128 for cta_group::1
// costs the same MMA time at M = 64, so a 64-channel layer on k_dtc wastes half of every
// MMA on zero weight rows.  Here the activations are the A operand (MN-major: M = 128 =
// 2 output pixels x 64 samples, the two pixel boxes its M atoms, LBO 8 KB) and the weights
// the B operand (K-major, N = 64 output channels): D[(pixel, sample)][channel] in TMEM,
// lane = (pixel, sample), column = channel.  A tile is TWP pixels = TWP/2 MMA groups
// (accumulator columns 64 g ..).  WIN (3x3 stride 1): a stage is (kh, 64-channel chunk):
// the TWP+2 pixel boxes of the input row and the 3 taps' [64 d][64 k] weight tiles; tap
// kw's A operand for group g starts at box kw + 2g.  Epilogue: warp w reads TMEM lane
// quarter w % 4 (pixel (w % 4) / 2 of group w / 4, samples 32 (w % 2) ..), converts its
// 64 channels and writes them transposed into the pixel's [64 c][64 s] swizzled staging
// box (16-bit stores, conflict-free); the two warps of a pixel meet at a named barrier and
// one TMA store writes the box.
// KC = 16: the first-layer form (a few input channels, zero-filled to 16 by the TMA): pixel
// boxes [16 c][64 s] (2 KB), the weights MN-major [16 k][64 d] per tap (packed
// [taps][16][64], one 2-KB tile per tap), one K = 16 MMA per tap.
template <int KC>
constexpr int dts_wbox() {
    return 64 * KC * 2;  // [64 d][KC k] binary16 weight tile
}
template <int KC>
constexpr int dts_xbox() {
    return KC * 64 * 2;  // [KC c][64 s] binary16 pixel box
}
template <int TWP, bool WIN, int KC>
constexpr int dts_stages() {
    return KC == 16 ? 6 : (WIN ? 2 : 4);
}
template <int TWP, bool WIN, int KC>
constexpr int dts_smem() {
    constexpr int NW = WIN ? 3 : 1, NBX = WIN ? TWP + 2 : TWP;
    return dts_stages<TWP, WIN, KC>() * (NW * dts_wbox<KC>() + NBX * dts_xbox<KC>()) + TWP * 2 * kBPix + 1024 + 256;
}

__device__ __forceinline__ void pair_sync(int id) {  // the two warps of one output pixel
    asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}

template <int TWP, bool WIN, int KC>
__global__ void __launch_bounds__(kThreads, 1) k_dts(const __grid_constant__ DtcArgs a) {
    constexpr int G = TWP / 2;                   // MMA groups (pixel pairs) per tile
    constexpr int NW = WIN ? 3 : 1;              // weight tiles (taps) per stage
    constexpr int NBX = WIN ? TWP + 2 : TWP;     // pixel boxes per stage
    constexpr int kW = dts_wbox<KC>(), kX = dts_xbox<KC>();
    constexpr int kStage = NW * kW + NBX * kX;
    constexpr int S = dts_stages<TWP, WIN, KC>();
    static_assert(KC == 64 || (KC == 16 && WIN), "the 16-channel form is the 3x3 stride-1 window");
    constexpr uint32_t kCols = 2 * G * 64 < 32 ? 32 : 2 * G * 64;  // two accumulators
    static_assert(kEW == 8, "two epilogue warps per pixel of a 4-pixel tile");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char *ostage = smem + S * kStage;  // [TWP pixels][2 slots] [64 c][64 s] boxes
    uint64_t *full = reinterpret_cast<uint64_t *>(ostage + TWP * 2 * kBPix);
    uint64_t *empty = full + S;
    uint64_t *tfull = empty + S;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles = a.x_tiles * a.Yh * a.NB;
    const int kiters = WIN ? a.Kh * a.cb : a.k_iters;
    if (threadIdx.x == 0) {
        DTC_STAMP(0);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], kEW);
        }
        fence_mbar_init();
    }
    if (warp == kEW) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(kCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) DTC_STAMP(1);
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.xmap)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.wmap)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.ymap)) : "memory");
    }
    pdl_release();
    if (warp != kEW) pdl_wait();  // the producer waits after issuing the first stages' weight tiles

    auto decode = [&](int t, int &xt, int &yo, int &nb) {
        xt = t % a.x_tiles;
        t /= a.x_tiles;
        yo = t % a.Yh;
        nb = t / a.Yh;
    };

    if (warp == kEW) {
        // ---------------- TMA producer: one box per lane ----------------
        auto load_w = [&](unsigned char *st, uint64_t *bar, int i) {  // weight tiles of k-iteration i
            if constexpr (KC == 16) {  // [taps][16 k][64 d]: rows (tap * 16 ..), 64 channels
                if (lane < 3) tma_load_2d(st + lane * kW, &a.wmap, 0, (i * 3 + lane) * 16, bar);
            } else if constexpr (WIN) {
                const int kh = i / a.cb, cb = i - kh * a.cb;
                if (lane < 3) tma_load_2d(st + lane * kW, &a.wmap, (kh * 3 + lane) * a.C + cb * kKC, 0, bar);
            } else {
                const int tap = i / a.cb, cb = i - tap * a.cb;
                if (lane == 0) tma_load_2d(st, &a.wmap, tap * a.C + cb * kKC, 0, bar);
            }
        };
        auto load_x = [&](unsigned char *st, uint64_t *bar, int i, int xt, int yo, int nb) {
            if constexpr (WIN) {
                const int kh = i / a.cb, cb = i - kh * a.cb;
                if (a.xrow) {
                    if (lane == 3)
                        tma_load_5d(st + NW * kW, &a.xmap, 0, cb * KC, xt * TWP + a.offw, yo + kh + a.offh, nb, bar);
                } else if (lane >= 3 && lane < 3 + NBX) {
                    tma_load_5d(st + NW * kW + (lane - 3) * kX, &a.xmap, 0, xt * TWP + (lane - 3) + a.offw,
                                yo + kh + a.offh, cb * KC, nb, bar);
                }
            } else {
                const int tap = i / a.cb, cb = i - tap * a.cb;
                const int kh = tap / a.Kw, kw = tap - kh * a.Kw;
                if (lane >= 1 && lane <= TWP)
                    tma_load_5d(st + kW + (lane - 1) * kX, &a.xmap, 0, a.stride * (xt * TWP + lane - 1) + kw + a.offw,
                                a.stride * yo + kh + a.offh, cb * KC, nb, bar);
            }
        };
        {  // weights of the first S stages before the wait on the previous kernel
            int it = 0;
            for (int t = blockIdx.x; it < S && t < tiles; t += gridDim.x)
                for (int i = 0; i < kiters && it < S; ++i, ++it) {
                    if (lane == 0) mbar_expect_tx(&full[it], kStage);
                    __syncwarp();
                    load_w(smem + it * kStage, &full[it], i);
                }
        }
        pdl_wait();
        int it = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
            int xt, yo, nb;
            decode(t, xt, yo, nb);
            for (int i = 0; i < kiters; ++i, ++it) {
                const int s = it % S;
                unsigned char *st = smem + s * kStage;
                if (it >= S) {
                    mbar_wait_bounded(&empty[s], ((it / S) - 1) & 1);
                    if (lane == 0) mbar_expect_tx(&full[s], kStage);
                    __syncwarp();
                    load_w(st, &full[s], i);
                }
                load_x(st, &full[s], i, xt, yo, nb);
            }
        }
    } else if (warp == kEW + 1) {
        // ---------------- MMA issuer: A = activations (MN-major), B = weights (K-major) ----------------
        // A MN-major (bit 15); B K-major, or MN-major (bit 16) in the 16-channel form
        const uint32_t idesc = (1u << 4) | (1u << 15) | (KC == 16 ? (1u << 16) : 0u) | ((uint32_t)(64 >> 3) << 17) |
                               ((uint32_t)(128 >> 4) << 24);
        int it = 0, lt = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++lt) {
            const int ab = lt & 1;
            if (lt >= 2) mbar_wait_bounded(&tempty[ab], ((lt >> 1) - 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            for (int i = 0; i < kiters; ++i, ++it) {
                const int s = it % S;
                mbar_wait_bounded(&full[s], (it / S) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (lane == 0 && it == 0) DTC_STAMP(2);
                if (lane == 0) {
                    const uint32_t wbase = smem_u32(smem + s * kStage), xbase = wbase + NW * kW;
#pragma unroll
                    for (int q = 0; q < NW; ++q)
#pragma unroll
                        for (int g = 0; g < G; ++g)
#pragma unroll
                            for (int k = 0; k < KC / 16; ++k) {
                                const uint64_t ad = desc_sw128(xbase + (q + 2 * g) * kX + k * 16 * 128, kX, 1024);
                                const uint64_t bd = KC == 16 ? desc_sw128(wbase + q * kW, kW, 1024)
                                                             : desc_sw128(wbase + q * kW + k * 32, 16, 1024);
                                umma_f16(tmem + ab * (G * 64) + g * 64, ad, bd, idesc, (i > 0 || q > 0 || k > 0) ? 1u : 0u);
                            }
                    umma_commit(&empty[s]);
                    if (i == kiters - 1) umma_commit(&tfull[ab]);
                    if (i == kiters - 1 && (lt == 0 || lt == 6)) DTC_STAMP(3 + (lt != 0));
                }
                __syncwarp();
            }
        }
    } else {
        // ---------------- epilogue ----------------
        const int qd = warp & 3, g = warp >> 2;       // TMEM lane quarter, MMA group
        const int pxg = qd >> 1, shalf = qd & 1;      // pixel within the group, sample half
        const int px = 2 * g + pxg;                   // pixel within the tile
        const int s = shalf * 32 + lane;              // this lane's sample
        const bool active = g < G;
        int lt = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++lt) {
            int xt, yo, nb;
            decode(t, xt, yo, nb);
            const int ab = lt & 1;
            mbar_wait_bounded(&tfull[ab], (lt >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (warp == 0 && lane == 0 && (lt == 0 || lt == 6)) DTC_STAMP(5 + (lt != 0));
            uint32_t v[64];
            if (active) {
                const uint32_t taddr = tmem + ab * (G * 64) + g * 64 + ((uint32_t)(qd * 32) << 16);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                    "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, "
                    "[%32];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                      "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                      "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                      "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                      "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                    : "r"(taddr));
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                    "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, "
                    "[%32];"
                    : "=r"(v[32]), "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]), "=r"(v[38]),
                      "=r"(v[39]), "=r"(v[40]), "=r"(v[41]), "=r"(v[42]), "=r"(v[43]), "=r"(v[44]), "=r"(v[45]),
                      "=r"(v[46]), "=r"(v[47]), "=r"(v[48]), "=r"(v[49]), "=r"(v[50]), "=r"(v[51]), "=r"(v[52]),
                      "=r"(v[53]), "=r"(v[54]), "=r"(v[55]), "=r"(v[56]), "=r"(v[57]), "=r"(v[58]), "=r"(v[59]),
                      "=r"(v[60]), "=r"(v[61]), "=r"(v[62]), "=r"(v[63])
                    : "r"(taddr + 32));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[ab]);
            if (!active) continue;
            // pixel px's staging slot lt & 1: free once the store issued two tiles ago read it
            const int bar_id = 1 + px;  // named barriers 1..TWP: the two warps of pixel px
            const bool issuer = shalf == 0 && lane == 0;
            unsigned char *box = ostage + (px * 2 + (lt & 1)) * kBPix;
            if (issuer) bulk_wait_read<1>();
            pair_sync(bar_id);
            const uint32_t sb = smem_u32(box);
#pragma unroll
            for (int c2 = 0; c2 < 32; ++c2) {
                uint32_t h = cvt_f16x2_sat(__uint_as_float(v[2 * c2]), __uint_as_float(v[2 * c2 + 1]));
                if (a.relu) h = relu_f16x2(h);
#pragma unroll
                for (int e = 0; e < 2; ++e) {  // channel c = 2 c2 + e: row c, column s of the swizzled box
                    const int c = 2 * c2 + e;
                    const uint32_t off = c * 128 + ((((s >> 3) ^ (c & 7)) << 4) | ((s & 7) << 1));
                    asm volatile("st.shared.u16 [%0], %1;" ::"r"(sb + off), "h"((unsigned short)(h >> (16 * e))) : "memory");
                }
            }
            fence_proxy_async();
            pair_sync(bar_id);
            const int xo = xt * TWP + px;
            if (issuer) {  // one bulk group per tile and pixel (empty past the map) keeps the slot accounting
                if (xo < a.Yw)
                    tma_store_5d(&a.ymap, box, 0, xo + a.Lo.pw, yo + a.Lo.ph, 0, nb);
                else
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        }
        if (lane == 0) bulk_wait_all();
        if (warp == 0 && lane == 0) DTC_STAMP(7);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == kEW) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols));
    }
}

template <int TWP, bool WIN, int KC = 64>
cudaError_t launch_dts(const DtcArgs &a, int tiles, cudaStream_t st) {
    static std::atomic<uint64_t> attr{0};
    constexpr int smem = dts_smem<TWP, WIN, KC>();
    static_assert(smem <= 227 * 1024 - 1024, "k_dts shared memory");
    cudaError_t e = ensure_smem_attr(k_dts<TWP, WIN, KC>, attr, smem);
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    int sms = usc_device_sm_count(dev);
    if (sms <= 0) sms = 148;
    return launch_pdl(k_dts<TWP, WIN, KC>, dim3((unsigned)(tiles < sms ? tiles : sms)), dim3(kThreads), smem, st, a);
}

// ---------------------------------------------------------------------------------------
// k_dtc2: the 3x3 stride-1 window tile on a CTA pair (cta_group::2, cluster of 2 on one TPC).
// The pair computes M = 256 output channels x N = 4 pixels x 64 samples: each CTA stages
// its 128 weight rows (A) and the row window of ITS two pixels (+ the 2-pixel halo, 4 boxes:
// half of B); the leader's single thread issues tcgen05.mma.cta_group::2, which reads A and
// B from both CTAs' shared memory at the same offsets.  Each SM thus reads half of B per MMA
// (the shared-memory port bound of k_dtc's window tiles).  Every TMA of
// both CTAs completes on the LEADER's full barrier (.cta_group::2, peer bit cleared); the
// leader's commits multicast to both CTAs' empty / tfull barriers; both CTAs' epilogue warps
// release the accumulator on the leader's tempty barrier.  Each CTA's TMEM holds its 128
// channels for all 4 pixels; the epilogue is k_dtc's.
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // shared::cluster address of the leader's copy

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma2_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar) & kPeerMask)
        : "memory");
}
__device__ __forceinline__ void tma2_load_5d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, int c3, int c4,
                                             uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar) & kPeerMask)
        : "memory");
}
__device__ __forceinline__ void umma2_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma2_commit_both(uint64_t *bar) {  // arrive on the barrier in both CTAs
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t *bar) {  // arrive on the leader CTA's copy
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(bar)));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

constexpr int kCg2Stage = 3 * kABytes + 4 * kBPix;  // 3 taps of own A rows + own half window (80 KB)
constexpr int kCg2S = 2;
constexpr int cg2_smem() { return kCg2S * kCg2Stage + kEW * kOS * kWarpBox + 1024 + 256; }

__global__ void __launch_bounds__(kThreads, 1) k_dtc2(const __grid_constant__ DtcArgs a) {
    constexpr int TWP = 4, N = 256, S = kCg2S, kStage = kCg2Stage;
    constexpr uint32_t kCols = 2 * N;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char *ostage = smem + S * kStage;
    uint64_t *full = reinterpret_cast<uint64_t *>(ostage + kEW * kOS * kWarpBox);
    uint64_t *empty = full + S;
    uint64_t *tfull = empty + S;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int tiles = a.m_blocks * a.x_tiles * a.Yh * a.NB;  // m_blocks: 256-channel blocks
    const int kiters = a.Kh * a.cb;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 2 * kEW);  // both CTAs' epilogue warps (the leader's copy counts)
        }
        fence_mbar_init();
    }
    if (warp == kEW) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(kCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync_all();  // barriers of both CTAs initialised before any cross-CTA signal
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.xmap)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.wmap)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.ymap)) : "memory");
    }
    pdl_release();
    pdl_wait();

    auto decode = [&](int t, int &mb, int &xt, int &yo, int &nb) {
        mb = t % a.m_blocks;
        t /= a.m_blocks;
        xt = t % a.x_tiles;
        t /= a.x_tiles;
        yo = t % a.Yh;
        nb = t / a.Yh;
    };

    if (warp == kEW) {
        // ---------------- TMA producer (both CTAs): own A rows + own half window ----------------
        int it = 0;
        for (int t = pair; t < tiles; t += npairs) {
            int mb, xt, yo, nb;
            decode(t, mb, xt, yo, nb);
            for (int i = 0; i < kiters; ++i, ++it) {
                const int s = it % S;
                if (it >= S) mbar_wait_bounded(&empty[s], ((it / S) - 1) & 1);
                unsigned char *st = smem + s * kStage;
                if (leader && lane == 0) mbar_expect_tx(&full[s], 2 * kStage);  // both CTAs' bytes
                __syncwarp();
                const int kh = i / a.cb, cb = i - kh * a.cb;
                if (lane < 3)
                    tma2_load_2d(st + lane * kABytes, &a.wmap, (kh * 3 + lane) * a.C + cb * kKC, mb * 256 + rank * 128,
                                 &full[s]);
                else if (lane == 3)  // own half window: pixels 2 rank .. 2 rank + 3 of the tile's 6 (map (s, c, x, y, nb))
                    tma2_load_5d(st + 3 * kABytes, &a.xmap, 0, cb * kKC, xt * TWP + rank * 2 + a.offw, yo + kh + a.offh,
                                 nb, &full[s]);
            }
        }
    } else if (warp == kEW + 1) {
        // ---------------- MMA issuer (leader only) ----------------
        if (leader) {
            const uint32_t idesc = (1u << 4) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
            int it = 0, lt = 0;
            for (int t = pair; t < tiles; t += npairs, ++lt) {
                const int ab = lt & 1;
                if (lt >= 2) mbar_wait_bounded(&tempty[ab], ((lt >> 1) - 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t acc = tmem + ab * N;
                for (int i = 0; i < kiters; ++i, ++it) {
                    const int s = it % S;
                    mbar_wait_bounded(&full[s], (it / S) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    if (lane == 0) {
                        const uint32_t abase = smem_u32(smem + s * kStage), bbase = abase + 3 * kABytes;
#pragma unroll
                        for (int q = 0; q < 3; ++q)
#pragma unroll
                            for (int k = 0; k < kKC / 16; ++k) {
                                const uint64_t ad = desc_sw128(abase + q * kABytes + k * 32, 16, 1024);
                                const uint64_t bd = desc_sw128(bbase + q * kBPix + k * 16 * 128, kBPix, 1024);
                                umma2_f16(acc, ad, bd, idesc, (i > 0 || q > 0 || k > 0) ? 1u : 0u);
                            }
                        umma2_commit_both(&empty[s]);
                        if (i == kiters - 1) umma2_commit_both(&tfull[ab]);
                    }
                    __syncwarp();
                }
            }
        }
    } else {
        // ---------------- epilogue (both CTAs): own 128 channels, 4 pixels ----------------
        const int ch0 = (warp & 3) * 32, half = warp >> 2;
        unsigned char *ost = ostage + warp * kOS * kWarpBox;
        int lt = 0, q = 0;
        for (int t = pair; t < tiles; t += npairs, ++lt) {
            int mb, xt, yo, nb;
            decode(t, mb, xt, yo, nb);
            const int ab = lt & 1;
            mbar_wait_bounded(&tfull[ab], (lt >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t taddr = tmem + ab * N + ((uint32_t)(ch0) << 16);
            const int cbase = mb * 256 + (int)rank * 128 + ch0;
#pragma unroll 1
            for (int px = half; px < TWP; px += 2, ++q) {
                uint32_t v[64];
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                    "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, "
                    "[%32];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                      "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                      "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                      "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                      "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                    : "r"(taddr + px * 64));
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                    "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, "
                    "[%32];"
                    : "=r"(v[32]), "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]), "=r"(v[38]),
                      "=r"(v[39]), "=r"(v[40]), "=r"(v[41]), "=r"(v[42]), "=r"(v[43]), "=r"(v[44]), "=r"(v[45]),
                      "=r"(v[46]), "=r"(v[47]), "=r"(v[48]), "=r"(v[49]), "=r"(v[50]), "=r"(v[51]), "=r"(v[52]),
                      "=r"(v[53]), "=r"(v[54]), "=r"(v[55]), "=r"(v[56]), "=r"(v[57]), "=r"(v[58]), "=r"(v[59]),
                      "=r"(v[60]), "=r"(v[61]), "=r"(v[62]), "=r"(v[63])
                    : "r"(taddr + px * 64 + 32));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (px + 2 >= TWP) {
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) mbar_arrive_leader(&tempty[ab]);
                }
                uint32_t h[32];
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    h[k] = cvt_f16x2_sat(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1]));
                    if (a.relu) h[k] = relu_f16x2(h[k]);
                }
                unsigned char *obox = ost + (q % kOS) * kWarpBox;
                if (lane == 0) bulk_wait_read<kOS - 1>();
                __syncwarp();
                unsigned char *orow = obox + lane * 128;
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    *reinterpret_cast<uint4 *>(orow + ((c ^ (lane & 7)) << 4)) =
                        make_uint4(h[4 * c], h[4 * c + 1], h[4 * c + 2], h[4 * c + 3]);
                fence_proxy_async();
                __syncwarp();
                const int xo = xt * TWP + px;
                if (lane == 0 && cbase < a.D && xo < a.Yw)
                    tma_store_5d(&a.ymap, obox, 0, xo + a.Lo.pw, yo + a.Lo.ph, cbase, nb);
            }
        }
        if (lane == 0) bulk_wait_all();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync_all();  // both CTAs done with the pair's tensor memory and barriers
    if (warp == kEW) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols));
    }
}

cudaError_t launch_dtc2(const DtcArgs &a, int pair_tiles, cudaStream_t st) {
    static std::atomic<uint64_t> attr{0};
    constexpr int smem = cg2_smem();
    static_assert(smem <= 227 * 1024 - 1024, "k_dtc2 shared memory");
    cudaError_t e = ensure_smem_attr(k_dtc2, attr, smem);
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    int sms = usc_device_sm_count(dev);
    if (sms <= 0) sms = 148;
    const int pairs = pair_tiles < sms / 2 ? pair_tiles : sms / 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * pairs));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, k_dtc2, a);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_tiled() {
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

}  // namespace

#ifdef DTC_TRACE
extern "C" int usc_dtc_trace_read(unsigned long long *out, int ctas) {
    return cudaMemcpyFromSymbol(out, g_dtc_trace, (size_t)ctas * 8 * sizeof(unsigned long long)) == cudaSuccess ? 0 : -1;
}
#endif

namespace {

bool xrow_enabled() {  // USC_NO_XROW=1: one TMA box per pixel in the window kernels (A/B measurements)
    static const bool on = [] {
        const char *v = std::getenv("USC_NO_XROW");
        return !(v && *v && *v != '0');
    }();
    return on;
}

bool cg2_enabled() {  // USC_CG2=1: 3x3 window tiles of >= 256-channel layers on CTA pairs (opt-in while measured)
    static const bool on = [] {
        const char *v = std::getenv("USC_CG2");
        return v && *v && *v != '0';
    }();
    return on;
}

bool dts_enabled() {  // USC_NO_DTS=1: 64-channel layers on k_dtc (A/B measurements)
    static const bool on = [] {
        const char *v = std::getenv("USC_NO_DTS");
        return !(v && *v && *v != '0');
    }();
    return on;
}

// Tile shape and split-K factor of one launch (shared by the launch and the workspace query)
struct DtcShape {
    int twp, x_tiles, m_blocks, NB, Yh, Yw, kiters, splits, kper;
    long long tiles;
};

// req_twp (2 or 4) / req_splits (>= 1) override the automatic choice (0 = automatic)
DtcShape dtc_shape(const usc_geometry *g, int n, const usc_act_layout *xl, bool res, bool win, int sms,
                   int req_twp = 0, int req_splits = 0) {
    DtcShape d{};
    const int s = g->stride_h, K = g->filter_h, pad = K / 2;
    d.Yh = (xl->height + 2 * pad - K) / s + 1;
    d.Yw = (xl->width + 2 * pad - K) / s + 1;
    d.NB = (n + 63) / 64;
    d.m_blocks = (g->out_channels + 127) / 128;
    // N = 256 (4 pixels) unless that leaves SMs idle: then 2-pixel tiles (twice the tiles)
    d.twp = d.Yw % 4 == 0 ? 4 : 2;
    if (d.twp == 4 && (long long)d.m_blocks * (d.Yw / 4) * d.Yh * d.NB < sms) d.twp = 2;
    if (req_twp == 2 || req_twp == 4) d.twp = req_twp;
    d.x_tiles = (d.Yw + d.twp - 1) / d.twp;
    d.tiles = (long long)d.m_blocks * d.x_tiles * d.Yh * d.NB;
    // (a first layer with < 64 input channels runs one 16-channel chunk)
    d.kiters = (win ? K : K * K) * std::max(1, g->in_channels / kKC);
    // split-K when the tiles fill at most half the SMs (small maps): each split >= 4 k-iterations
    d.splits = 1;
    if (!res && d.tiles > 0 && d.tiles * 2 <= sms) {
        const int want = (int)std::min<long long>(sms / d.tiles, d.kiters / 4);
        if (want >= 2) d.splits = want;
    }
    if (req_splits >= 1) d.splits = res ? 1 : std::min(req_splits, d.kiters);
    d.kper = (d.kiters + d.splits - 1) / d.splits;
    d.splits = (d.kiters + d.kper - 1) / d.kper;
    return d;
}

// Fused 2x2 pool: 4-pixel window tiles run in row pairs by one CTA.  Cost model (us): a
// 4-pixel tile takes kiters stages of 12 MMAs of 128 clocks; the separate pool kernel
// streams the full-resolution output once (+ its quarter) at ~5 TB/s plus ~2 us.  Fuse
// when the pair schedule's makespan is no longer than conv makespan + pool.
bool dtc_pool_ok(const usc_geometry *g, int n, const usc_act_layout *xl, int sms) {
    if (g->filter_h != 3 || g->filter_w != 3 || g->stride_h != 1 || g->stride_w != 1 || g->in_channels % kKC)
        return false;
    const DtcShape d = dtc_shape(g, n, xl, false, true, sms);
    if (d.Yh % 2 || d.Yw % 4 || d.splits > 1) return false;
    const long long tiles4 = (long long)d.m_blocks * (d.Yw / 4) * d.Yh * d.NB, pairs = tiles4 / 2;
    const double t_tile = d.kiters * 12.0 * 128.0 / 1900.0;
    const double pool_bytes = 2.0 * d.NB * 64.0 * g->out_channels * d.Yh * d.Yw * 1.25;
    const double waves = (double)((d.tiles + sms - 1) / sms) * (d.twp == 4 ? 1.0 : 0.5);
    const double unfused = waves * t_tile + pool_bytes / 5e6 + 2.0;
    const double fused = 2.0 * (double)((pairs + sms - 1) / sms) * t_tile;
    return fused <= unfused;
}

size_t dtc_ws_bytes(const DtcShape &d) {
    if (d.splits <= 1) return 0;
    const size_t part = (size_t)d.tiles * d.splits * (d.twp * 64) * 128 * sizeof(float);
    return part + (size_t)d.tiles * sizeof(int) + 256;
}

int dense_conv_impl(const usc_geometry *g, int32_t n, const void *w_dev, const usc_act_layout *xl, const void *x,
                    const usc_act_layout *yl, void *y, const usc_act_layout *rl, const void *res, int32_t relu,
                    void *workspace, size_t ws_bytes, int pool, int req_twp, int req_splits, void *stream) {
    if (!g || !w_dev || !xl || !x || !yl || !y || n < 1) return usc::fail(USC_ERR_VALUE, "dense conv: null argument");
    if (req_twp != 0 && req_twp != 2 && req_twp != 4)
        return usc::fail(USC_ERR_VALUE, "dense conv: pixels per tile must be 0 (auto), 2 or 4");
    if (req_splits < 0) return usc::fail(USC_ERR_VALUE, "dense conv: negative split count");
    if (g->filter_h != g->filter_w || (g->filter_h != 1 && g->filter_h != 3) || g->stride_h != g->stride_w ||
        (g->stride_h != 1 && g->stride_h != 2))
        return usc::fail(USC_ERR_UNSUPPORTED, "dense conv: 1x1 / 3x3 filters, stride 1 or 2");
    // first-layer form: <= 16 input channels (zero-filled to 16), 3x3 stride 1, 64 outputs
    const bool first = g->in_channels < kKC && g->in_channels <= 16 && g->filter_h == 3 && g->stride_h == 1 &&
                       g->out_channels == 64 && !res && !pool;
    if ((g->in_channels % kKC && !first) || g->out_channels % 64)
        return usc::fail(USC_ERR_UNSUPPORTED,
                         "dense conv: channels in %% 64 (or <= 16 for a 3x3 stride-1 64-channel first layer) and out %% 64");
    if (xl->interleave != 64 || yl->interleave != 64 || (res && (!rl || rl->interleave != 64)))
        return usc::fail(USC_ERR_UNSUPPORTED, "dense conv: BI64 layouts only");
    const int s = g->stride_h, K = g->filter_h, pad = K / 2;
    const int Yh = (xl->height + 2 * pad - K) / s + 1, Yw = (xl->width + 2 * pad - K) / s + 1;
    if (yl->height != (pool ? Yh / 2 : Yh) || yl->width != (pool ? Yw / 2 : Yw) || yl->channels != g->out_channels ||
        xl->channels != g->in_channels)
        return usc::fail(USC_ERR_VALUE, "dense conv: layouts do not match the convolution");
    if (xl->pad_h < pad || xl->pad_w < pad)
        return usc::fail(USC_ERR_VALUE, "dense conv: input halo smaller than the padding");
    if (res && (rl->height != Yh || rl->width != Yw || rl->channels != g->out_channels))
        return usc::fail(USC_ERR_VALUE, "dense conv: shortcut layout does not match the output");
    auto enc = encode_tiled();
    if (!enc) return usc::fail(USC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    DtcArgs a{};
    const int NB = (n + 63) / 64;
    {   // activations: [NB][C][Hp][Wp][64] binary16, box = one pixel x 64 channels x 64 samples
        const cuuint64_t dims[5] = {64, (cuuint64_t)xl->ws, (cuuint64_t)xl->hp, (cuuint64_t)xl->channels, (cuuint64_t)NB};
        const cuuint64_t strides[4] = {128, (cuuint64_t)xl->ws * 128, (cuuint64_t)xl->ws * xl->hp * 128,
                                       (cuuint64_t)xl->sample_stride * 2};
        const cuuint32_t box[5] = {64, 1, 1, (cuuint32_t)(first ? 16 : kKC), 1};  // first layer: OOB channels read 0
        const cuuint32_t es[5] = {1, 1, 1, 1, 1};
        CUresult r = enc(&a.xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, const_cast<void *>(x), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return usc::fail(USC_ERR_CUDA, "dense conv: activation tensor map (%d)", (int)r);
    }
    const int taps = K * K, Kd = taps * g->in_channels;
    const int Dpad = (g->out_channels + 127) / 128 * 128;  // the packed weights carry zero rows up to 128k
    if (!first) {  // weights: [Dpad][taps*C] binary16 K-major, box [64 k][128 d]
        const cuuint64_t dims[2] = {(cuuint64_t)Kd, (cuuint64_t)Dpad};
        const cuuint64_t strides[1] = {(cuuint64_t)Kd * 2};
        const cuuint32_t box[2] = {(cuuint32_t)kKC, 128};
        const cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&a.wmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void *>(w_dev), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return usc::fail(USC_ERR_CUDA, "dense conv: weight tensor map (%d)", (int)r);
    }
    // output and shortcut: the same BI64 box shape, [32 channels][64 samples] of one pixel
    auto bi_map = [&](CUtensorMap *m, const usc_act_layout *l, const void *p) -> CUresult {
        const cuuint64_t dims[5] = {64, (cuuint64_t)l->ws, (cuuint64_t)l->hp, (cuuint64_t)l->channels, (cuuint64_t)NB};
        const cuuint64_t strides[4] = {128, (cuuint64_t)l->ws * 128, (cuuint64_t)l->ws * l->hp * 128,
                                       (cuuint64_t)l->sample_stride * 2};
        const cuuint32_t box[5] = {64, 1, 1, 32, 1};  // one epilogue warp's 32 channels
        const cuuint32_t es[5] = {1, 1, 1, 1, 1};
        return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, const_cast<void *>(p), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    if (bi_map(&a.ymap, yl, y) != CUDA_SUCCESS) return usc::fail(USC_ERR_CUDA, "dense conv: output tensor map");
    if (res && bi_map(&a.rmap, rl, res) != CUDA_SUCCESS)
        return usc::fail(USC_ERR_CUDA, "dense conv: shortcut tensor map");
    a.y = y;
    a.res = res;
    a.Lo = to_dev(*yl);
    a.Lr = res ? to_dev(*rl) : a.Lo;
    a.C = g->in_channels;
    a.D = g->out_channels;
    a.Kh = K;
    a.Kw = K;
    a.stride = s;
    a.offh = xl->pad_h - pad;
    a.offw = xl->pad_w - pad;
    a.Yh = Yh;
    a.Yw = Yw;
    a.NB = NB;
    a.relu = relu;
    a.m_blocks = Dpad / 128;  // a 64-channel layer runs M = 128 with zero rows; the TMA store clips them
    a.cb = g->in_channels / kKC;
    a.k_iters = taps * a.cb;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess && usc_device_sm_count(dev) > 0) sms = usc_device_sm_count(dev);
    const bool win = K == 3 && s == 1 && !res;  // the 3-tap row window (stride 1; no shortcut staging room)
    DtcShape d = dtc_shape(g, n, xl, res != nullptr, win, sms, req_twp, req_splits);
    if (first) d.splits = 1, d.kper = d.kiters;  // the first-layer form has no split-K
    if (pool) {  // 4-pixel window tiles in row pairs, no split
        if (res || !relu || !dtc_pool_ok(g, n, xl, sms))
            return usc::fail(USC_ERR_UNSUPPORTED, "dense conv: fused pool not available for this shape");
        d.twp = 4;
        d.x_tiles = Yw / 4;
        d.tiles = (long long)d.m_blocks * d.x_tiles * Yh * d.NB;
        d.splits = 1;
        d.kper = d.kiters;
        a.pool = 1;
    }
    const int twp = d.twp;
    a.x_tiles = d.x_tiles;
    if (win && xrow_enabled()) {  // one TMA box per row window: the map re-ordered as (s, c, x, y, nb)
        const cuuint64_t dims[5] = {64, (cuuint64_t)xl->channels, (cuuint64_t)xl->ws, (cuuint64_t)xl->hp, (cuuint64_t)NB};
        const cuuint64_t strides[4] = {(cuuint64_t)xl->ws * xl->hp * 128, 128, (cuuint64_t)xl->ws * 128,
                                       (cuuint64_t)xl->sample_stride * 2};
        const cuuint32_t box[5] = {64, (cuuint32_t)(first ? 16 : kKC), (cuuint32_t)(twp + 2), 1, 1};
        const cuuint32_t es[5] = {1, 1, 1, 1, 1};
        if (enc(&a.xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, const_cast<void *>(x), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return usc::fail(USC_ERR_CUDA, "dense conv: row-window activation tensor map");
        a.xrow = 1;
    }
    if (d.tiles * d.splits > 0x7fffffffLL) return usc::fail(USC_ERR_UNSUPPORTED, "dense conv: grid too large");
    const size_t need = dtc_ws_bytes(d);
    if (need == 0 || !workspace || ws_bytes < need) d.splits = 1, d.kper = d.kiters;  // no workspace: no split
    a.splits = d.splits;
    a.kper = d.kper;
    if (d.splits > 1) {
        a.part = static_cast<float *>(workspace);
        a.cnt = reinterpret_cast<int *>(static_cast<char *>(workspace) +
                                        (size_t)d.tiles * d.splits * (twp * 64) * 128 * sizeof(float));
    }
    const long long tiles = d.tiles * d.splits;  // work items
    cudaError_t e;
    if (win && !first && !pool && d.splits == 1 && twp == 4 && g->out_channels % 256 == 0 && cg2_enabled()) {
        // CTA pairs: M = 256 (weights packed to 128 rows suffice: D % 256 == 0), 4-pixel tiles
        a.m_blocks = g->out_channels / 256;
        a.x_tiles = Yw / 4 + (Yw % 4 != 0);
        {  // activations as (s, c, x, y, nb), one box = a CTA's 4-pixel half window
            const cuuint64_t dims[5] = {64, (cuuint64_t)xl->channels, (cuuint64_t)xl->ws, (cuuint64_t)xl->hp,
                                        (cuuint64_t)NB};
            const cuuint64_t strides[4] = {(cuuint64_t)xl->ws * xl->hp * 128, 128, (cuuint64_t)xl->ws * 128,
                                           (cuuint64_t)xl->sample_stride * 2};
            const cuuint32_t box[5] = {64, (cuuint32_t)kKC, 4, 1, 1};
            const cuuint32_t es[5] = {1, 1, 1, 1, 1};
            if (enc(&a.xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, const_cast<void *>(x), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
                return usc::fail(USC_ERR_CUDA, "dense conv: pair-window activation tensor map");
        }
        const long long pair_tiles = (long long)a.m_blocks * a.x_tiles * Yh * NB;
        e = launch_dtc2(a, (int)pair_tiles, st);
        if (e == cudaSuccess) e = cudaGetLastError();
        return e == cudaSuccess ? USC_OK : usc::fail(USC_ERR_CUDA, "k_dtc2: %s", cudaGetErrorString(e));
    }
    if (first) {  // [taps][16 k][64 d] MN-major weights, one 2-KB tile per tap; one 16-channel chunk
        a.cb = 1;
        const cuuint64_t wdims[2] = {64, (cuuint64_t)(taps * 16)};
        const cuuint64_t wstrides[1] = {128};
        const cuuint32_t wbox[2] = {64, 16};
        const cuuint32_t es2[2] = {1, 1};
        if (enc(&a.wmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void *>(w_dev), wdims, wstrides, wbox, es2,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return usc::fail(USC_ERR_CUDA, "dense conv: first-layer weight tensor map");
    }
    if (g->out_channels == 64 && !res && !pool && d.splits == 1 && (dts_enabled() || first)) {
        // 64 output channels: swapped operands (k_dts), N = 64 channels, no zero weight rows
        const cuuint64_t wdims[2] = {(cuuint64_t)(taps * g->in_channels), (cuuint64_t)64};
        const cuuint64_t wstrides[1] = {(cuuint64_t)(taps * g->in_channels) * 2};
        const cuuint32_t wbox[2] = {(cuuint32_t)kKC, 64};
        const cuuint32_t es2[2] = {1, 1};
        if (!first && enc(&a.wmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void *>(w_dev), wdims, wstrides, wbox, es2,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return usc::fail(USC_ERR_CUDA, "dense conv: weight tensor map (64 rows)");
        const cuuint64_t ydims[5] = {64, (cuuint64_t)yl->ws, (cuuint64_t)yl->hp, (cuuint64_t)yl->channels, (cuuint64_t)NB};
        const cuuint64_t ystrides[4] = {128, (cuuint64_t)yl->ws * 128, (cuuint64_t)yl->ws * yl->hp * 128,
                                        (cuuint64_t)yl->sample_stride * 2};
        const cuuint32_t ybox[5] = {64, 1, 1, 64, 1};
        const cuuint32_t es5[5] = {1, 1, 1, 1, 1};
        if (enc(&a.ymap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, y, ydims, ystrides, ybox, es5, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return usc::fail(USC_ERR_CUDA, "dense conv: output tensor map (64 channels)");
        const long long ntiles = (long long)a.x_tiles * Yh * NB;
        if (first)
            e = twp == 4 ? launch_dts<4, true, 16>(a, (int)ntiles, st) : launch_dts<2, true, 16>(a, (int)ntiles, st);
        else if (twp == 4)
            e = win ? launch_dts<4, true>(a, (int)ntiles, st) : launch_dts<4, false>(a, (int)ntiles, st);
        else
            e = win ? launch_dts<2, true>(a, (int)ntiles, st) : launch_dts<2, false>(a, (int)ntiles, st);
        if (e == cudaSuccess) e = cudaGetLastError();
        return e == cudaSuccess ? USC_OK : usc::fail(USC_ERR_CUDA, "k_dts: %s", cudaGetErrorString(e));
    }
    if (twp == 4)
        e = win ? launch_dtc<4, true, false>(a, (int)tiles, st)
                : (res ? launch_dtc<4, false, true>(a, (int)tiles, st) : launch_dtc<4, false, false>(a, (int)tiles, st));
    else
        e = win ? launch_dtc<2, true, false>(a, (int)tiles, st)
                : (res ? launch_dtc<2, false, true>(a, (int)tiles, st) : launch_dtc<2, false, false>(a, (int)tiles, st));
    if (e == cudaSuccess) e = cudaGetLastError();
    return e == cudaSuccess ? USC_OK : usc::fail(USC_ERR_CUDA, "k_dtc: %s", cudaGetErrorString(e));
}

}  // namespace

int usc_dense_conv_f16(const usc_geometry *g, int32_t n, const void *w_dev, const usc_act_layout *xl, const void *x,
                       const usc_act_layout *yl, void *y, const usc_act_layout *rl, const void *res, int32_t relu,
                       void *stream) {
    return dense_conv_impl(g, n, w_dev, xl, x, yl, y, rl, res, relu, nullptr, 0, 0, 0, 0, stream);
}

int usc_dense_conv_f16_pool(const usc_geometry *g, int32_t n, const void *w_dev, const usc_act_layout *xl,
                            const void *x, const usc_act_layout *yl, void *y, void *stream) {
    return dense_conv_impl(g, n, w_dev, xl, x, yl, y, nullptr, nullptr, 1, nullptr, 0, 1, 0, 0, stream);
}

int32_t usc_dense_conv_f16_pool_ok(const usc_geometry *g, int32_t n, const usc_act_layout *xl) {
    if (!g || !xl || n < 1) return 0;
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess && usc_device_sm_count(dev) > 0) sms = usc_device_sm_count(dev);
    return dtc_pool_ok(g, n, xl, sms) ? 1 : 0;
}

int usc_dense_conv_f16_ws(const usc_geometry *g, int32_t n, const void *w_dev, const usc_act_layout *xl, const void *x,
                          const usc_act_layout *yl, void *y, const usc_act_layout *rl, const void *res, int32_t relu,
                          void *workspace, int64_t ws_bytes, int32_t twp, int32_t splits, void *stream) {
    if (ws_bytes < 0) return usc::fail(USC_ERR_VALUE, "dense conv: negative workspace size");
    return dense_conv_impl(g, n, w_dev, xl, x, yl, y, rl, res, relu, workspace, (size_t)ws_bytes, 0, twp, splits,
                           stream);
}

int64_t usc_dense_conv_f16_ws_bytes(const usc_geometry *g, int32_t n, const usc_act_layout *xl, int32_t has_res,
                                    int32_t twp, int32_t splits) {
    if (!g || !xl || n < 1 || g->filter_h != g->filter_w || (g->filter_h != 1 && g->filter_h != 3) ||
        g->in_channels % kKC)
        return 0;
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess && usc_device_sm_count(dev) > 0) sms = usc_device_sm_count(dev);
    const bool win = g->filter_h == 3 && g->stride_h == 1 && !has_res;
    return (int64_t)dtc_ws_bytes(dtc_shape(g, n, xl, has_res != 0, win, sms, twp, splits));
}
