// conv.cu -- sm_100a kernels of the direct sparse convolution engine.
//
// The hot kernel (k_tiled) replaces the reference's numba inner loop
// kernels.sparse_conv_blocks (/root/reference/pkg/src/unsparse/kernels.py:57-100)
// and its driver sparse_conv_forward (engine.py:64-111):
//
//   * activations live in HBM in the zero-haloed, 16-byte-row-aligned "padded
//     NCHW" layout (the reference's materialised zero_pad, tensor.py:225-235), so
//     one CTA's input tile for a chunk of CC input channels is a handful of
//     contiguous byte ranges; a single elected thread moves them into shared
//     memory with bulk-async copies (cp.async.bulk -> UBLKCP, the TMA engine),
//     double-buffered on mbarriers;
//   * a CTA owns NS samples x TH output rows x DT output channels; each thread
//     owns a strip of P consecutive output pixels for all DT channels and keeps
//     DT*P accumulators in registers for the whole input-channel loop;
//   * the CSR entries of a channel group are warp-uniform: every lane reads the
//     same (offset, weight) pair (a broadcast L1 hit) and applies it to its P
//     pixels;
//   * per output element the accumulation is the reference's: entries in stored
//     (ascending offset == ascending (c,kh,kw)) order, IEEE fp32 multiply then
//     add (__fmul_rn/__fadd_rn: ptxas must not contract them into FFMA), so the
//     fp32 result is bit-identical to the reference.  Zero-weight entries are
//     deduplicated by the packer (no-ops for finite inputs; one copy per offset
//     preserves NaN propagation).
#include <cstdlib>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include <type_traits>

#include "common.cuh"
#include "usc_internal.h"

using usc::fail;

namespace usc_dev {
bool pdl_enabled() {
    static const bool on = [] {
        const char *v = std::getenv("USC_NO_PDL");
        return !(v && *v && *v != '0');
    }();
    return on;
}
}  // namespace usc_dev

namespace {
using namespace usc_dev;

struct TiledArgs {
    const void *x;
    void *y;
    const int *cpg;
    const void *ents;
    const float *tbl;
    int N, C, D, n_chunks, CC;
    int NS, TH, HS, Ws, Hp, Yh, Yw, s_h, SPR, row_tiles;
    long long x_sample_stride;  // elements
    int stage_elems;            // elements per stage buffer (incl. slack)
    Epi ep;
};

// The hot kernel.  grid = (sample_tiles*row_tiles, groups), block = NT threads.
template <int KIND, int P, int DT, int SW, int NT>
__global__ void __launch_bounds__(NT) k_tiled(const TiledArgs a) {
    using TX = typename Kind<KIND>::TX;
    using ACC = typename Kind<KIND>::ACC;
    using TY = typename Kind<KIND>::TY;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
    float *tbl = reinterpret_cast<float *>(smem + 16);
    TX *stage0 = reinterpret_cast<TX *>(smem + 128);
    TX *stage1 = stage0 + a.stage_elems;

    const int tid = threadIdx.x;
    const int g = blockIdx.y;
    const int st = blockIdx.x / a.row_tiles, rt = blockIdx.x - st * a.row_tiles;
    const int b0 = st * a.NS;
    const int nvalid = min(a.NS, a.N - b0);
    const int r0 = rt * a.TH;
    const int y0 = r0 * a.s_h;                      // first staged padded row
    const int rows = min(a.HS, a.Hp - y0);          // rows actually copied
    const bool full_planes = (y0 == 0 && rows == a.Hp);

    // thread -> (sample, output row, strip)
    const int strips_per_sample = a.TH * a.SPR;
    int ns = tid / strips_per_sample;
    const int rem = tid - ns * strips_per_sample;
    const int rr = rem / a.SPR;
    const int col0 = (rem - rr * a.SPR) * P;
    const int r = r0 + rr;
    const bool in_tile = ns < a.NS;
    if (!in_tile) ns = 0;
    const bool valid = in_tile && ns < nvalid && r < a.Yh;
    const int stage_sample = a.CC * a.HS * a.Ws;
    const int base = in_tile ? ns * stage_sample + rr * a.s_h * a.Ws + col0 * SW : 0;

    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    if constexpr (KIND == USC_CB4) {
        if (tid < 16) tbl[tid] = a.tbl[tid];
    }
    __syncthreads();

    const TX *xg = static_cast<const TX *>(a.x);
    auto issue = [&](int k, int s) {
        const int c0 = k * a.CC;
        const int cc = min(a.CC, a.C - c0);
        TX *dst = s ? stage1 : stage0;
        const uint32_t row_bytes = static_cast<uint32_t>(a.Ws * sizeof(TX));
        if (full_planes) {
            const uint32_t bytes = cc * a.Hp * row_bytes;
            mbar_expect_tx(&bar[s], bytes * nvalid);
            for (int q = 0; q < nvalid; ++q)
                bulk_g2s(dst + q * stage_sample,
                         xg + (long long)(b0 + q) * a.x_sample_stride + (long long)c0 * a.Hp * a.Ws,
                         bytes, &bar[s]);
        } else {
            const uint32_t bytes = rows * row_bytes;
            mbar_expect_tx(&bar[s], bytes * nvalid * cc);
            for (int q = 0; q < nvalid; ++q)
                for (int c = 0; c < cc; ++c)
                    bulk_g2s(dst + q * stage_sample + c * a.HS * a.Ws,
                             xg + (long long)(b0 + q) * a.x_sample_stride +
                                 ((long long)(c0 + c) * a.Hp + y0) * a.Ws,
                             bytes, &bar[s]);
        }
    };
    if (tid == 0) {
        issue(0, 0);
        if (a.n_chunks > 1) issue(1, 1);
    }

    ACC acc[DT][P];
#pragma unroll
    for (int i = 0; i < DT; ++i)
#pragma unroll
        for (int p = 0; p < P; ++p) acc[i][p] = 0;

    const int *cpg = a.cpg + (long long)g * a.n_chunks * DT;
    for (int k = 0; k < a.n_chunks; ++k) {
        const int s = k & 1;
        mbar_wait(&bar[s], (k >> 1) & 1);
        const TX *xs = (s ? stage1 : stage0) + base;
        const int *cp = cpg + k * DT;
#pragma unroll
        for (int dl = 0; dl < DT; ++dl)
            apply_entries<KIND, P, SW>(acc[dl], a.ents, __ldg(cp + dl), __ldg(cp + dl + 1), xs, tbl);
        __syncthreads();
        if (tid == 0 && k + 2 < a.n_chunks) {
            fence_proxy_async();
            issue(k + 2, s);
        }
    }

    if (!valid) return;
    TY *y = static_cast<TY *>(a.y);
    const int b = b0 + ns;
#pragma unroll
    for (int dl = 0; dl < DT; ++dl) {
        const int d = g * DT + dl;
        if (d >= a.D) break;
        long long row;
        if (a.ep.out_padded)
            row = (long long)b * a.ep.o_sample_stride +
                  ((long long)d * a.ep.oHp + r + a.ep.oph) * a.ep.oWs + a.ep.opw;
        else
            row = (((long long)b * a.D + d) * a.Yh + r) * a.Yw;
#pragma unroll
        for (int p = 0; p < P; ++p)
            if (col0 + p < a.Yw) store_one<KIND>(y, row + col0 + p, acc[dl][p], a.ep);
    }
}

// Generic fallback: one thread per output element, entries from global, any stride.
struct GenArgs {
    const void *x;
    void *y;
    const int *cpg;
    const void *ents;
    const float *tbl;
    int N, D, Yh, Yw, s_h, s_w, Ws;
    long long x_sample_stride;
    Epi ep;
};

template <int KIND>
__global__ void __launch_bounds__(256) k_generic(const GenArgs a) {
    using TX = typename Kind<KIND>::TX;
    using ACC = typename Kind<KIND>::ACC;
    using TY = typename Kind<KIND>::TY;
    const long long total = (long long)a.N * a.D * a.Yh * a.Yw;
    for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < total;
         o += (long long)gridDim.x * blockDim.x) {
        const int col = static_cast<int>(o % a.Yw);
        long long t = o / a.Yw;
        const int r = static_cast<int>(t % a.Yh);
        t /= a.Yh;
        const int d = static_cast<int>(t % a.D);
        const int b = static_cast<int>(t / a.D);
        const TX *xb = static_cast<const TX *>(a.x) + (long long)b * a.x_sample_stride +
                       (long long)r * a.s_h * a.Ws + (long long)col * a.s_w;
        ACC acc[1] = {0};
        apply_entries<KIND, 1, 1>(acc, a.ents, __ldg(a.cpg + d), __ldg(a.cpg + d + 1), xb, a.tbl);
        long long idx;
        if (a.ep.out_padded)
            idx = (long long)b * a.ep.o_sample_stride +
                  ((long long)d * a.ep.oHp + r + a.ep.oph) * a.ep.oWs + a.ep.opw + col;
        else
            idx = o;
        store_one<KIND>(static_cast<TY *>(a.y), idx, acc[0], a.ep);
    }
}

// Reference-shaped FFI kernel: kernels.sparse_conv_blocks (kernels.py:57-100) on a
// materialised padded xflat, every stored entry (padding included), stored order.
__global__ void __launch_bounds__(256)
    k_blocks(const float *__restrict__ xflat, const int64_t *__restrict__ rp,
             const int64_t *__restrict__ col, const float *__restrict__ th, float *__restrict__ out,
             const int64_t *__restrict__ blocks, long long nb, int sb, long long x_size, int s_h,
             int s_w, int Wp, int D, int Yh, int Yw) {
    const long long total = nb * sb * Yh * Yw;
    for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < total;
         o += (long long)gridDim.x * blockDim.x) {
        const int cc = static_cast<int>(o % Yw);
        long long t = o / Yw;
        const int r = static_cast<int>(t % Yh);
        t /= Yh;
        const int tt = static_cast<int>(t % sb);
        const long long bi = t / sb;
        const long long d = blocks[2 * bi], g0 = blocks[2 * bi + 1];
        const long long n_nz = rp[1] - rp[0], base = rp[d];
        const long long x0 = (g0 + tt) * x_size + (long long)r * s_h * Wp + (long long)cc * s_w;
        float acc = 0.0f;
        for (long long j = 0; j < n_nz; ++j)
            acc = __fadd_rn(acc, __fmul_rn(__ldg(th + base + j), __ldg(xflat + x0 + col[base + j])));
        out[(((g0 + tt) * D + d) * Yh + r) * Yw + cc] = acc;
    }
}

// --------------------------------------------------------------------------
// elementwise utility kernels

// plain NCHW -> any layout; writes every destination element (halo and padding
// samples become zeros).  Destination-ordered so stores are coalesced.
template <typename T, typename TD = T>
__global__ void k_pad_any(const T *__restrict__ src, TD *__restrict__ dst, int n, int H, int W,
                          const LayoutD L, long long total) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        long long t = i;
        int lane = 0;
        if (L.il) {
            lane = static_cast<int>(t % L.il);
            t /= L.il;
        }
        const int x = static_cast<int>(t % L.Ws);
        t /= L.Ws;
        const int y = static_cast<int>(t % L.Hp);
        t /= L.Hp;
        const int c = static_cast<int>(t % L.C);
        const long long b = L.il ? (t / L.C) * L.il + lane : t / L.C;
        const int iy = y - L.ph, ix = x - L.pw;
        T v{};
        if (b < n && iy >= 0 && iy < H && ix >= 0 && ix < W) v = src[((b * L.C + c) * H + iy) * W + ix];
        if constexpr (std::is_same<T, TD>::value)
            dst[i] = v;
        else  // int8 code -> binary16 (exact)
            dst[i] = __short2half_rn(static_cast<short>(v));
    }
}

// plain NCHW -> a batch-interleaved layout, one CTA per (sample block, channel, padded
// row): the IL samples x 32 pixels of a row segment go through a [IL][33] shared tile so
// the NCHW reads (pixels contiguous per sample) and the BI writes (samples contiguous per
// pixel) are both coalesced; halo rows / columns and samples past n are written as zeros.
template <typename T, typename TD = T>
__global__ void k_pad_bi(const T *__restrict__ src, TD *__restrict__ dst, int n, int H, int W, const LayoutD L) {
    __shared__ T tile[64][33];
    const int IL = L.il;
    const int yp = blockIdx.x % L.Hp;
    const int c = (blockIdx.x / L.Hp) % L.C;
    const long long nb = blockIdx.x / ((long long)L.Hp * L.C);
    TD *drow = dst + nb * L.ss + ((long long)c * L.Hp + yp) * L.Ws * IL;
    const int iy = yp - L.ph;
    const bool rowin = iy >= 0 && iy < H;
    {  // one 32-column chunk of the row per block (blockIdx.y): many short blocks keep HBM busy
        const int x0 = blockIdx.y * 32;
        for (int i = threadIdx.x; i < IL * 32; i += blockDim.x) {
            const int sm = i >> 5, xx = i & 31, ix = x0 + xx - L.pw;
            const long long b = nb * IL + sm;
            T v{};
            if (rowin && b < n && ix >= 0 && ix < W) v = src[((b * L.C + c) * H + iy) * W + ix];
            tile[sm][xx] = v;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < IL * 32; i += blockDim.x) {
            const int xx = i / IL, sm = i - xx * IL, xp = x0 + xx;
            if (xp < L.Ws) {
                if constexpr (std::is_same<T, TD>::value)
                    drow[(long long)xp * IL + sm] = tile[sm][xx];
                else  // int8 code -> binary16 (exact)
                    drow[(long long)xp * IL + sm] = __short2half_rn(static_cast<short>(tile[sm][xx]));
            }
        }
    }
}

// any layout -> plain NCHW (n x C x H x W); index arithmetic in 32 bits when the
// element count allows (64-bit division is a long emulated sequence)
template <typename T, typename I>
__global__ void k_unpad_any(const T *__restrict__ src, T *__restrict__ dst, int H, int W, const LayoutD L,
                            long long total) {
    for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < total;
         i0 += (long long)gridDim.x * blockDim.x) {
        const I i = static_cast<I>(i0);
        const int x = static_cast<int>(i % W);
        I t = i / W;
        const int y = static_cast<int>(t % H);
        t /= H;
        const int c = static_cast<int>(t % L.C);
        const long long b = t / L.C;
        dst[i0] = src[lay_index(L, b, c, y, x)];
    }
}

__global__ void k_round16(const float *__restrict__ src, void *dst, long long n, int to_half) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        __half h = sat_half(src[i]);
        if (to_half)
            static_cast<__half *>(dst)[i] = h;
        else
            static_cast<float *>(dst)[i] = __half2float(h);
    }
}

__global__ void k_h2f(const __half *__restrict__ src, float *__restrict__ dst, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        dst[i] = __half2float(src[i]);
}

// nn.MaxPool2.forward (nn.py:124-135): value at np.argmax of the 2x2 window in
// order (0,0),(0,1),(1,0),(1,1) -- first NaN if any, else first maximum.
// Works between any two layouts; output-ordered (sample fastest for BI layouts).
template <typename T, typename I>
__global__ void k_maxpool2(const T *__restrict__ src, T *__restrict__ dst, int n_total, int C, int OH,
                           int OW, const LayoutD Li, const LayoutD Lo) {
    const long long total = (long long)n_total * C * OH * OW;
    for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < total;
         i0 += (long long)gridDim.x * blockDim.x) {
        I t = static_cast<I>(i0);  // 32-bit index arithmetic when the count allows
        int lane = 0;
        if (Lo.il) {
            lane = static_cast<int>(t % Lo.il);
            t /= Lo.il;
        }
        const int x = static_cast<int>(t % OW);
        t /= OW;
        const int y = static_cast<int>(t % OH);
        t /= OH;
        const int c = static_cast<int>(t % C);
        const long long b = Lo.il ? (t / C) * Lo.il + lane : t / C;
        const long long p00 = lay_index(Li, b, c, 2 * y, 2 * x);
        const long long p01 = lay_index(Li, b, c, 2 * y, 2 * x + 1);
        const long long p10 = lay_index(Li, b, c, 2 * y + 1, 2 * x);
        const long long p11 = lay_index(Li, b, c, 2 * y + 1, 2 * x + 1);
        const T w[4] = {src[p00], src[p01], src[p10], src[p11]};
        int m = 0;
        float vm = static_cast<float>(w[0]);
        if (!isnan(vm))
            for (int k = 1; k < 4; ++k) {
                const float v = static_cast<float>(w[k]);
                if (isnan(v)) {
                    m = k;
                    break;
                }
                if (v > vm) {
                    vm = v;
                    m = k;
                }
            }
        dst[lay_index(Lo, b, c, y, x)] = w[m];
    }
}

// The same pooling between two batch-interleaved layouts (BI32 / BI64): one 16-byte
// vector of consecutive samples per thread, four vector loads (the 2x2 window), one
// vector store -- every access a coalesced 16-B transaction.
template <typename T, typename I>
__global__ void k_maxpool2_bi(const T *__restrict__ src, T *__restrict__ dst, int NB, int C, int OH, int OW,
                              const LayoutD Li, const LayoutD Lo) {
    constexpr int V = 16 / sizeof(T);
    pdl_release();
    pdl_wait();
    const int lanes = Lo.il / V;
    const long long total = (long long)NB * C * OH * OW * lanes;
    const long long rs = (long long)Li.Ws * Li.il;  // one input row
    for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < total;
         i0 += (long long)gridDim.x * blockDim.x) {
        I t = static_cast<I>(i0);
        const int l = static_cast<int>(t % lanes);
        t /= lanes;
        const int x = static_cast<int>(t % OW);
        t /= OW;
        const int y = static_cast<int>(t % OH);
        t /= OH;
        const int c = static_cast<int>(t % C);
        const long long nb = static_cast<long long>(t / C);
        const long long pi = nb * Li.ss + (((long long)c * Li.Hp + 2 * y + Li.ph) * Li.Ws + 2 * x + Li.pw) * Li.il + l * V;
        const long long po = nb * Lo.ss + (((long long)c * Lo.Hp + y + Lo.ph) * Lo.Ws + x + Lo.pw) * Lo.il + l * V;
        uint4 raw[4];
        raw[0] = *reinterpret_cast<const uint4 *>(src + pi);
        raw[1] = *reinterpret_cast<const uint4 *>(src + pi + Li.il);
        raw[2] = *reinterpret_cast<const uint4 *>(src + pi + rs);
        raw[3] = *reinterpret_cast<const uint4 *>(src + pi + rs + Li.il);
        const T *w0 = reinterpret_cast<const T *>(&raw[0]);
        uint4 out;
        T *o = reinterpret_cast<T *>(&out);
#pragma unroll
        for (int e = 0; e < V; ++e) {
            T best = w0[e];
            float vm = static_cast<float>(best);
            if (!isnan(vm)) {
#pragma unroll
                for (int k = 1; k < 4; ++k) {
                    const T wk = reinterpret_cast<const T *>(&raw[k])[e];
                    const float v = static_cast<float>(wk);
                    if (isnan(v)) {
                        best = wk;
                        break;
                    }
                    if (v > vm) {
                        vm = v;
                        best = wk;
                    }
                }
            }
            o[e] = best;
        }
        *reinterpret_cast<uint4 *>(dst + po) = out;
    }
}

__global__ void k_quant_i8(const float *__restrict__ src, int8_t *__restrict__ dst, long long n,
                           double sigma, double limit) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double s = static_cast<double>(src[i]) / sigma;
        double c = copysign(floor(fabs(s) + 0.5), s);
        c = c < -limit ? -limit : (c > limit ? limit : c);
        dst[i] = static_cast<int8_t>(c);
    }
}

// FMUL+FADD throughput probe (8 independent chains per thread).
__global__ void k_peak_muladd(float *out, float a, float b, int iters) {
    float acc[8], x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        acc[i] = threadIdx.x * 0.001f + i;
        x[i] = b + i;
    }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = __fadd_rn(x[i], __fmul_rn(a, acc[i]));
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 1.2345f) out[0] = s;
}

// The BI64 fp32 inner-loop mix: per lane two samples, FMUL x2 then one packed FADD2
// (add.rn.f32x2) per MAC pair (8 independent chains per thread).
__global__ void k_peak_fadd2(float *out, float a, float b, int iters) {
    unsigned long long acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float lo = threadIdx.x * 0.001f + i, hi = lo + 0.5f;
        asm("mov.b64 %0, {%1, %2};" : "=l"(acc[i]) : "f"(lo), "f"(hi));
    }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float lo, hi, p0, p1;
            asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[i]));
            asm volatile("mul.rn.f32 %0, %1, %2;" : "=f"(p0) : "f"(lo), "f"(a));
            asm volatile("mul.rn.f32 %0, %1, %2;" : "=f"(p1) : "f"(hi), "f"(b));
            unsigned long long q;
            asm("mov.b64 %0, {%1, %2};" : "=l"(q) : "f"(p0), "f"(p1));
            asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(acc[i]) : "l"(q));
        }
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[i]));
        s += lo + hi;
    }
    if (s == 1.2345f) out[0] = s;
}

// The binary16 path's FHFMA (fma.rn.f32.f16: fp32 += f16 * f16), 8 chains per thread.
__global__ void k_peak_fhfma(float *out, float a, float b, int iters) {
    float acc[8];
    const unsigned short th = __half_as_ushort(__float2half(a));
    const unsigned short xv = (unsigned short)(0x3800 + (threadIdx.x & 255));
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = b + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc[i]) : "h"(th), "h"(xv));
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 1.2345f) out[0] = s;
}

int grid_for(long long total, int threads = 256) {
    long long g = (total + threads - 1) / threads;
    return static_cast<int>(std::max<long long>(1, std::min<long long>(g, 148LL * 32)));
}

int cuda_check(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(USC_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return USC_OK;
}

// --------------------------------------------------------------------------
// tiled-kernel dispatch table

template <int KIND, int P, int DT, int SW>
int launch_tiled_inst(const usc_plan *pl, const TiledArgs &a, cudaStream_t st) {
    auto fn = k_tiled<KIND, P, DT, SW, 256>;
    static std::atomic<uint64_t> attr{0};  // per instantiation and device
    cudaError_t ae = usc_dev::ensure_smem_attr(fn, attr, 220 * 1024);
    if (ae != cudaSuccess) return fail(USC_ERR_CUDA, "smem attribute: %s", cudaGetErrorString(ae));
    dim3 grid(static_cast<unsigned>(pl->grid_x), static_cast<unsigned>(pl->grid_y));
    fn<<<grid, 256, pl->smem_bytes, st>>>(a);
    return cuda_check("k_tiled launch");
}

template <int KIND, int P, int DT>
int launch_tiled_sw(const usc_plan *pl, const TiledArgs &a, cudaStream_t st) {
    if (pl->g.stride_w == 1) return launch_tiled_inst<KIND, P, DT, 1>(pl, a, st);
    return launch_tiled_inst<KIND, P, DT, 2>(pl, a, st);
}

template <int KIND, int P>
int launch_tiled_dt(const usc_plan *pl, const TiledArgs &a, cudaStream_t st) {
    if (pl->DT == 8) return launch_tiled_sw<KIND, P, 8>(pl, a, st);
    return launch_tiled_sw<KIND, P, 16>(pl, a, st);
}

template <int KIND>
int launch_tiled_p(const usc_plan *pl, const TiledArgs &a, cudaStream_t st) {
    switch (pl->P) {
        case 1: return launch_tiled_dt<KIND, 1>(pl, a, st);
        case 2: return launch_tiled_dt<KIND, 2>(pl, a, st);
        case 4: return launch_tiled_dt<KIND, 4>(pl, a, st);
        default: return launch_tiled_dt<KIND, 8>(pl, a, st);
    }
}

Epi make_epi(const usc_epilogue *e) {
    Epi ep{};
    if (!e) {
        ep.scale = 1.0f;
        return ep;
    }
    ep.relu = e->relu;
    ep.pool = e->pool;
    ep.saturate = e->saturate;
    ep.saturate2 = e->saturate2;
    ep.cap = e->cap;
    ep.cap2 = e->cap2;
    ep.scale = e->scale;
    ep.out_padded = e->out_padded;
    ep.requant = e->requant;
    ep.rq_scale = e->rq_scale;
    ep.rq_limit = e->rq_limit;
    ep.residual = e->residual;
    if (e->residual) {
        ep.res = reinterpret_cast<const void *>(e->res);
        ep.rC = e->res_layout.channels;
        ep.rHp = e->res_layout.hp;
        ep.rWs = e->res_layout.ws;
        ep.rph = e->res_layout.pad_h;
        ep.rpw = e->res_layout.pad_w;
        ep.ril = e->res_layout.interleave;
        ep.r_sample_stride = e->res_layout.sample_stride;
    }
    if (e->out_padded) {
        ep.oHp = e->out.hp;
        ep.oWs = e->out.ws;
        ep.oph = e->out.pad_h;
        ep.opw = e->out.pad_w;
        ep.o_sample_stride = e->out.sample_stride;
        ep.oil = e->out.interleave;
    }
    return ep;
}

}  // namespace

extern "C" {

int usc_device_sm_count(int device) {
    int v = -1;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    return v;
}

int usc_peak_fp32_muladd(int32_t device, double *tflops) { return usc_peak_mix(device, 0, tflops); }

int usc_peak_mix(int32_t device, int32_t mix, double *tflops) {
    if (mix < 0 || mix > 2) return fail(USC_ERR_VALUE, "unknown instruction mix %d", mix);
    int sms = usc_device_sm_count(device);
    if (sms <= 0) return fail(USC_ERR_CUDA, "no CUDA device %d", device);
    cudaSetDevice(device);
    float *out = nullptr;
    cudaEvent_t e0, e1;
    if (cudaMalloc(&out, 4) != cudaSuccess) return cuda_check("peak malloc");
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 8, threads = 256, iters = 8192;
    auto fn = mix == 0 ? k_peak_muladd : (mix == 1 ? k_peak_fadd2 : k_peak_fhfma);
    const double macs_per_iter = mix == 1 ? 16.0 : 8.0;  // per thread: 8 chains (x2 samples for FADD2)
    fn<<<blocks, threads>>>(out, 1.0001f, 0.5f, iters);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        fn<<<blocks, threads>>>(out, 1.0001f, 0.5f, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    *tflops = (double)blocks * threads * iters * macs_per_iter * 2 / (best * 1e-3) / 1e12;
    return cuda_check("peak probe");
}

static int conv_forward_impl(const usc_plan *pl, const void *blob, const void *x, const usc_act_layout *xv, void *y,
                             const usc_epilogue *epi, void *stream, int step_h = 1, int step_w = 1);

int usc_conv_forward(const usc_plan *pl, const void *blob, const void *x, void *y,
                     const usc_epilogue *epi, void *stream) {
    return conv_forward_impl(pl, blob, x, nullptr, y, epi, stream);
}

int usc_conv_forward_view(const usc_plan *pl, const void *blob, const void *x, const usc_act_layout *x_layout,
                          void *y, const usc_epilogue *epi, void *stream) {
    if (!x_layout) return fail(USC_ERR_VALUE, "null input layout");
    if (pl && pl->kernel < 3) return fail(USC_ERR_UNSUPPORTED, "input views need a batch-interleaved plan");
    return conv_forward_impl(pl, blob, x, x_layout, y, epi, stream);
}

int usc_conv_forward_strided(const usc_plan *pl, const void *blob, const void *x, const usc_act_layout *x_layout,
                             int32_t step_h, int32_t step_w, void *y, const usc_epilogue *epi, void *stream) {
    if (!x_layout) return fail(USC_ERR_VALUE, "null input layout");
    if (step_h < 1 || step_w < 1 || step_h > 8 || step_w > 8) return fail(USC_ERR_VALUE, "steps must be 1..8");
    if (pl && pl->kernel < 3) return fail(USC_ERR_UNSUPPORTED, "input views need a batch-interleaved plan");
    if (pl && (pl->g.filter_h != 1 || pl->g.filter_w != 1 || pl->g.stride_h != 1 || pl->g.stride_w != 1 ||
               pl->g.pad_h || pl->g.pad_w))
        return fail(USC_ERR_VALUE, "a strided view runs a 1x1, stride-1, unpadded plan");
    return conv_forward_impl(pl, blob, x, x_layout, y, epi, stream, step_h, step_w);
}

static int conv_forward_impl(const usc_plan *pl, const void *blob, const void *x, const usc_act_layout *xv, void *y,
                             const usc_epilogue *epi, void *stream, int step_h, int step_w) {
    if (!pl || !blob || !x || !y) return fail(USC_ERR_VALUE, "null argument");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const usc_geometry &g = pl->g;
    Epi ep = make_epi(epi);
    if (ep.out_padded && pl->transposed)
        return fail(USC_ERR_UNSUPPORTED, "padded output of a transposed 1-D plan");
    if (ep.out_padded && !epi->pool &&
        (epi->out.channels != g.out_channels || epi->out.height != pl->out_h || epi->out.width != pl->out_w))
        return fail(USC_ERR_VALUE, "output layout does not match the plan");
    if (epi && epi->pool) {
        if (pl->kernel < 3 || pl->PR != 2 || pl->PC % 2 || pl->out_h % 2 || pl->out_w % 2)
            return fail(USC_ERR_VALUE, "fused max-pool needs a BI plan with 2-row, even-width pixel blocks");
        if (!ep.out_padded || epi->out.height != pl->out_h / 2 || epi->out.width != pl->out_w / 2)
            return fail(USC_ERR_VALUE, "fused max-pool needs the pooled output layout");
    }
    if (ep.residual && (pl->kernel < 3 || (pl->dtype != USC_F32 && pl->dtype != USC_F16) || !epi->res ||
                        epi->res_layout.interleave == 0 || epi->res_layout.channels != g.out_channels ||
                        epi->res_layout.height != pl->out_h || epi->res_layout.width != pl->out_w ||
                        epi->pool))
        return fail(USC_ERR_VALUE, "residual epilogue needs an F32/F16 BI plan, an interleaved shortcut of the "
                                   "output's shape and no fused pool");
    if (ep.requant && (pl->kernel < 3 || pl->dtype != USC_I8))
        return fail(USC_ERR_UNSUPPORTED, "requantising epilogue needs an int8 BI plan");
    if (pl->kernel == 3 || pl->kernel == 4) return usc::launch_bi(pl, blob, x, y, ep, st, xv, step_h, step_w);
    if (ep.out_padded && ep.oil != 0)
        return fail(USC_ERR_UNSUPPORTED, "kernels 1/2 write interleave-0 layouts only");
    // blob = [16 x f32 centroid table][int32 cpg, 16-B aligned][entries]
    const char *cb = static_cast<const char *>(blob);
    const long long cp_bytes = ((4LL * ((long long)pl->groups * pl->n_chunks * pl->DT + 1)) + 15) / 16 * 16;
    const float *tbl = reinterpret_cast<const float *>(cb);
    const int *cpg = reinterpret_cast<const int *>(cb + 64);
    const void *ents = cb + 64 + cp_bytes;
    if (pl->kernel == 1) {
        TiledArgs a{};
        a.x = x;
        a.y = y;
        a.cpg = cpg;
        a.ents = ents;
        a.tbl = tbl;
        a.N = pl->n;
        a.C = g.in_channels;
        a.D = g.out_channels;
        a.n_chunks = pl->n_chunks;
        a.CC = pl->CC;
        a.NS = pl->NS;
        a.TH = pl->TH;
        a.HS = pl->HS;
        a.Ws = pl->in.ws;
        a.Hp = pl->in.hp;
        a.Yh = pl->out_h;
        a.Yw = pl->out_w;
        a.s_h = g.stride_h;
        a.SPR = pl->strips_per_row;
        a.row_tiles = pl->row_tiles;
        a.x_sample_stride = pl->in.sample_stride;
        a.stage_elems = static_cast<int>(pl->smem_stage_bytes / usc::elem_bytes(pl->dtype));
        a.ep = ep;
        switch (pl->dtype) {
            case USC_F32: return launch_tiled_p<USC_F32>(pl, a, st);
            case USC_F16: return launch_tiled_p<USC_F16>(pl, a, st);
            case USC_I8: return launch_tiled_p<USC_I8>(pl, a, st);
            default: return launch_tiled_p<USC_CB4>(pl, a, st);
        }
    }
    GenArgs a{};
    a.x = x;
    a.y = y;
    a.cpg = cpg;
    a.ents = ents;
    a.tbl = tbl;
    a.N = pl->n;
    a.D = g.out_channels;
    a.Yh = pl->out_h;
    a.Yw = pl->out_w;
    a.s_h = g.stride_h;
    a.s_w = g.stride_w;
    a.Ws = pl->in.ws;
    a.x_sample_stride = pl->in.sample_stride;
    a.ep = ep;
    const int grid = static_cast<int>(pl->grid_x);
    switch (pl->dtype) {
        case USC_F32: k_generic<USC_F32><<<grid, 256, 0, st>>>(a); break;
        case USC_F16: k_generic<USC_F16><<<grid, 256, 0, st>>>(a); break;
        case USC_I8: k_generic<USC_I8><<<grid, 256, 0, st>>>(a); break;
        default: k_generic<USC_CB4><<<grid, 256, 0, st>>>(a); break;
    }
    return cuda_check("k_generic launch");
}

int usc_sparse_conv_blocks(const float *xflat, const int64_t *row_ptr, const int64_t *col_offsets,
                           const float *theta, float *out, const int64_t *blocks, int64_t n_blocks,
                           int32_t sb, int64_t x_size, int32_t s_h, int32_t s_w, int32_t padded_w,
                           int32_t D, int32_t out_h, int32_t out_w, void *stream) {
    if (n_blocks <= 0) return USC_OK;
    if (sb < 1 || s_h < 1 || s_w < 1) return fail(USC_ERR_VALUE, "bad block arguments");
    const long long total = (long long)n_blocks * sb * out_h * out_w;
    k_blocks<<<grid_for(total), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        xflat, row_ptr, col_offsets, theta, out, blocks, n_blocks, sb, x_size, s_h, s_w, padded_w, D,
        out_h, out_w);
    return cuda_check("k_blocks launch");
}

int usc_pad_input(const usc_act_layout *l, int32_t dtype, int32_t n, const void *src, void *dst,
                  void *stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long long total = usc_act_layout_elems(l, n);
    const int grid = grid_for(total);
    const LayoutD L = to_dev(*l);
    if (l->interleave) {  // batch-interleaved: the tiled transpose
        const long long rows = (long long)((n + l->interleave - 1) / l->interleave) * l->channels * l->hp;
        if (rows > 0x7fffffffLL) return fail(USC_ERR_UNSUPPORTED, "pad: too many rows");
        const dim3 blocks((unsigned)rows, (unsigned)((l->ws + 31) / 32));
        switch (usc::elem_bytes(dtype)) {
            case 4:
                k_pad_bi<float><<<blocks, 256, 0, st>>>(static_cast<const float *>(src),
                                                                   static_cast<float *>(dst), n, l->height, l->width, L);
                break;
            case 2:
                k_pad_bi<uint16_t><<<blocks, 256, 0, st>>>(static_cast<const uint16_t *>(src),
                                                                      static_cast<uint16_t *>(dst), n, l->height,
                                                                      l->width, L);
                break;
            case 1:  // the BI kernel stages int8 codes as binary16
                k_pad_bi<int8_t, __half><<<blocks, 256, 0, st>>>(static_cast<const int8_t *>(src),
                                                                            static_cast<__half *>(dst), n, l->height,
                                                                            l->width, L);
                break;
            default: return fail(USC_ERR_VALUE, "unknown dtype %d", dtype);
        }
        return cuda_check("k_pad_bi launch");
    }
    switch (usc::elem_bytes(dtype)) {
        case 4:
            k_pad_any<float><<<grid, 256, 0, st>>>(static_cast<const float *>(src), static_cast<float *>(dst),
                                                   n, l->height, l->width, L, total);
            break;
        case 2:
            k_pad_any<uint16_t><<<grid, 256, 0, st>>>(static_cast<const uint16_t *>(src),
                                                      static_cast<uint16_t *>(dst), n, l->height, l->width, L,
                                                      total);
            break;
        case 1:
            if (l->interleave)  // the BI kernel stages int8 codes as binary16
                k_pad_any<int8_t, __half><<<grid, 256, 0, st>>>(static_cast<const int8_t *>(src),
                                                                static_cast<__half *>(dst), n, l->height,
                                                                l->width, L, total);
            else
                k_pad_any<int8_t><<<grid, 256, 0, st>>>(static_cast<const int8_t *>(src),
                                                        static_cast<int8_t *>(dst), n, l->height, l->width, L,
                                                        total);
            break;
        default: return fail(USC_ERR_VALUE, "unknown dtype %d", dtype);
    }
    return cuda_check("k_pad launch");
}

int usc_unpad_output(const usc_act_layout *l, int32_t dtype, int32_t n, const void *src, void *dst,
                     void *stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long long total = (long long)n * l->channels * l->height * l->width;
    const int grid = grid_for(total);
    const LayoutD L = to_dev(*l);
    const bool small = total < 0x7fffffffLL;
    switch (usc::elem_bytes(dtype)) {
        case 4:
            (small ? k_unpad_any<float, unsigned> : k_unpad_any<float, long long>)<<<grid, 256, 0, st>>>(
                static_cast<const float *>(src), static_cast<float *>(dst), l->height, l->width, L, total);
            break;
        case 2:
            (small ? k_unpad_any<uint16_t, unsigned> : k_unpad_any<uint16_t, long long>)<<<grid, 256, 0, st>>>(
                static_cast<const uint16_t *>(src), static_cast<uint16_t *>(dst), l->height, l->width, L, total);
            break;
        case 1:
            (small ? k_unpad_any<int8_t, unsigned> : k_unpad_any<int8_t, long long>)<<<grid, 256, 0, st>>>(
                static_cast<const int8_t *>(src), static_cast<int8_t *>(dst), l->height, l->width, L, total);
            break;
        default: return fail(USC_ERR_VALUE, "unknown dtype %d", dtype);
    }
    return cuda_check("k_unpad launch");
}

int usc_round_binary16(const float *src, void *dst, int64_t count, int32_t to_half, void *stream) {
    if (count <= 0) return USC_OK;
    k_round16<<<grid_for(count), 256, 0, static_cast<cudaStream_t>(stream)>>>(src, dst, count, to_half);
    return cuda_check("k_round16 launch");
}

int usc_convert(const void *src, int32_t sd, void *dst, int32_t dd, int64_t count, void *stream) {
    if (count <= 0) return USC_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (sd == USC_F32 && (dd == USC_F16 || dd == USC_CB4)) {
        k_round16<<<grid_for(count), 256, 0, st>>>(static_cast<const float *>(src), dst, count, 1);
    } else if ((sd == USC_F16 || sd == USC_CB4) && dd == USC_F32) {
        k_h2f<<<grid_for(count), 256, 0, st>>>(static_cast<const __half *>(src), static_cast<float *>(dst),
                                                count);
    } else {
        return fail(USC_ERR_VALUE, "unsupported conversion %d -> %d", sd, dd);
    }
    return cuda_check("convert launch");
}

int usc_maxpool2(const usc_act_layout *in_l, const usc_act_layout *out_l, int32_t dtype, int32_t n,
                 const void *src, void *dst, void *stream) {
    if (in_l->height % 2 || in_l->width % 2)
        return fail(USC_ERR_VALUE, "maxpool needs even spatial dims, got %dx%d", in_l->height, in_l->width);
    const int OH = in_l->height / 2, OW = in_l->width / 2;
    if (out_l->height != OH || out_l->width != OW || out_l->channels != in_l->channels)
        return fail(USC_ERR_VALUE, "maxpool output layout mismatch");
    if (in_l->interleave != out_l->interleave)
        return fail(USC_ERR_VALUE, "maxpool layouts must share the interleave");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int il = out_l->interleave;
    const int n_total = il ? (n + il - 1) / il * il : n;
    const long long total = (long long)n_total * in_l->channels * OH * OW;
    const LayoutD Li = to_dev(*in_l), Lo = to_dev(*out_l);
    if (il && (dtype == USC_F32 || dtype == USC_F16 || dtype == USC_CB4)) {  // vectorised BI path
        const int NB = n_total / il, V = dtype == USC_F32 ? 4 : 8;
        const long long vecs = total / V;
        const dim3 grid(grid_for(vecs)), block(256);
        cudaError_t e;
        if (dtype == USC_F32)
            e = launch_pdl(vecs < 0x7fffffffLL ? k_maxpool2_bi<float, unsigned> : k_maxpool2_bi<float, long long>, grid,
                           block, 0, st, static_cast<const float *>(src), static_cast<float *>(dst), NB,
                           (int)in_l->channels, OH, OW, Li, Lo);
        else
            e = launch_pdl(vecs < 0x7fffffffLL ? k_maxpool2_bi<__half, unsigned> : k_maxpool2_bi<__half, long long>,
                           grid, block, 0, st, static_cast<const __half *>(src), static_cast<__half *>(dst), NB,
                           (int)in_l->channels, OH, OW, Li, Lo);
        if (e != cudaSuccess) return fail(USC_ERR_CUDA, "k_maxpool2_bi launch: %s", cudaGetErrorString(e));
        return cuda_check("k_maxpool2_bi launch");
    }
    if (dtype == USC_F32) {
        (total < 0x7fffffffLL ? k_maxpool2<float, unsigned> : k_maxpool2<float, long long>)<<<grid_for(total), 256, 0, st>>>(static_cast<const float *>(src),
                                                           static_cast<float *>(dst), n_total,
                                                           in_l->channels, OH, OW, Li, Lo);
    } else if (dtype == USC_F16 || dtype == USC_CB4) {
        (total < 0x7fffffffLL ? k_maxpool2<__half, unsigned> : k_maxpool2<__half, long long>)<<<grid_for(total), 256, 0, st>>>(static_cast<const __half *>(src),
                                                            static_cast<__half *>(dst), n_total,
                                                            in_l->channels, OH, OW, Li, Lo);
    } else {
        return fail(USC_ERR_VALUE, "maxpool dtype %d unsupported", dtype);
    }
    return cuda_check("k_maxpool2 launch");
}

int usc_quantize_i8(const float *src, int8_t *dst, int64_t count, double sigma, int32_t bits, void *stream) {
    if (bits < 2 || bits > 8) return fail(USC_ERR_VALUE, "bits must be in [2, 8]");
    if (count <= 0) return USC_OK;
    const double limit = static_cast<double>((1 << (bits - 1)) - 1);
    k_quant_i8<<<grid_for(count), 256, 0, static_cast<cudaStream_t>(stream)>>>(src, dst, count, sigma, limit);
    return cuda_check("k_quant_i8 launch");
}

}  // extern "C"
