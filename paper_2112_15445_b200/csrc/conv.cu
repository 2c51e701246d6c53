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
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "usc_internal.h"

using usc::fail;

namespace {

// --------------------------------------------------------------------------
// PTX helpers: mbarrier + bulk async copy (TMA engine, non-tensor form)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// --------------------------------------------------------------------------
// operand kinds

template <int KIND> struct Kind;
template <> struct Kind<USC_F32> { using TX = float;  using ACC = float; using TY = float;  };
template <> struct Kind<USC_F16> { using TX = __half; using ACC = float; using TY = __half; };
template <> struct Kind<USC_I8>  { using TX = int8_t; using ACC = int;   using TY = float;  };
template <> struct Kind<USC_CB4> { using TX = __half; using ACC = float; using TY = __half; };

// round_to_binary16 (tensor.py:48-63): RNE, finite overflow saturates to +-65504
__device__ __forceinline__ __half sat_half(float v) {
    __half h = __float2half_rn(v);
    if (__hisinf(h) && isfinite(v)) h = __float2half_rn(copysignf(65504.0f, v));
    return h;
}
__device__ __forceinline__ float round16f(float v) { return __half2float(sat_half(v)); }

struct Epi {
    int relu, saturate, saturate2, out_padded;
    float cap, cap2, scale;
    int oHp, oWs, oph, opw;
    long long o_sample_stride;  // elements per sample of the padded output
};

// Apply the stored entries [e0, e1) of one output channel to P pixels.
// xs points at the thread's first pixel's top-left tap in the staged tile.
template <int KIND, int P, int SW>
__device__ __forceinline__ void apply_entries(typename Kind<KIND>::ACC (&acc)[P], const void *ents,
                                              int e0, int e1, const typename Kind<KIND>::TX *xs,
                                              const float *tbl) {
    if constexpr (KIND == USC_F32 || KIND == USC_F16) {
        const int2 *E = static_cast<const int2 *>(ents);
#pragma unroll 2
        for (int e = e0; e < e1; ++e) {
            const int2 en = __ldg(E + e);
            const float th = __int_as_float(en.y);
            const typename Kind<KIND>::TX *xp = xs + en.x;
#pragma unroll
            for (int p = 0; p < P; ++p) {
                if constexpr (KIND == USC_F32)
                    acc[p] = __fadd_rn(acc[p], __fmul_rn(th, xp[p * SW]));
                else  // binary16 x binary16 is exact in fp32: FFMA == FMUL+FADD
                    acc[p] = __fmaf_rn(th, __half2float(xp[p * SW]), acc[p]);
            }
        }
    } else {
        const int *E = static_cast<const int *>(ents);
#pragma unroll 2
        for (int e = e0; e < e1; ++e) {
            const int en = __ldg(E + e);
            if constexpr (KIND == USC_I8) {
                const int th = en >> 24;  // signed code
                const int8_t *xp = xs + (en & 0xFFFFFF);
#pragma unroll
                for (int p = 0; p < P; ++p) acc[p] += th * static_cast<int>(xp[p * SW]);
            } else {
                const float th = tbl[static_cast<unsigned>(en) >> 28];
                const __half *xp = xs + (en & 0x0FFFFFFF);
#pragma unroll
                for (int p = 0; p < P; ++p)
                    acc[p] = __fadd_rn(acc[p], __fmul_rn(th, __half2float(xp[p * SW])));
            }
        }
    }
}

template <int KIND>
__device__ __forceinline__ void store_one(typename Kind<KIND>::TY *y, long long idx,
                                          typename Kind<KIND>::ACC acc, const Epi &ep) {
    if constexpr (KIND == USC_F32) {
        float v = acc;
        if (ep.relu) v = v > 0.0f ? v : 0.0f;
        y[idx] = v;
    } else if constexpr (KIND == USC_I8) {
        float v = __fmul_rn(static_cast<float>(acc), ep.scale);
        if (ep.relu) v = v > 0.0f ? v : 0.0f;
        y[idx] = v;
    } else {
        float v = acc;
        if (ep.saturate) v = v > ep.cap ? ep.cap : v;  // np.minimum keeps NaN
        v = round16f(v);
        if (ep.relu) v = v > 0.0f ? v : 0.0f;
        if (ep.saturate2) {
            v = v > ep.cap2 ? ep.cap2 : v;
            v = round16f(v);
        }
        y[idx] = __float2half_rn(v);  // exact: v is on the binary16 grid
    }
}

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

template <typename T>
__global__ void k_pad(const T *__restrict__ src, T *__restrict__ dst, int n, int C, int H, int W,
                      int ph, int pw, int Hp, int Ws) {
    const long long total = (long long)n * C * Hp * Ws;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int x = static_cast<int>(i % Ws);
        long long t = i / Ws;
        const int y = static_cast<int>(t % Hp);
        const long long pc = t / Hp;  // b*C + c
        const int iy = y - ph, ix = x - pw;
        T v{};
        if (iy >= 0 && iy < H && ix >= 0 && ix < W) v = src[(pc * H + iy) * W + ix];
        dst[i] = v;
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
template <typename T>
__global__ void k_maxpool2(const T *__restrict__ src, T *__restrict__ dst, int n, int C, int OH,
                           int OW, int iHp, int iWs, int iph, int ipw, long long iss, int oHp, int oWs,
                           int oph, int opw, long long oss) {
    const long long total = (long long)n * C * OH * OW;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int x = static_cast<int>(i % OW);
        long long t = i / OW;
        const int y = static_cast<int>(t % OH);
        t /= OH;
        const int c = static_cast<int>(t % C);
        const long long b = t / C;
        const T *p = src + b * iss + ((long long)c * iHp + 2 * y + iph) * iWs + 2 * x + ipw;
        float v[4];
        v[0] = static_cast<float>(p[0]);
        v[1] = static_cast<float>(p[1]);
        v[2] = static_cast<float>(p[iWs]);
        v[3] = static_cast<float>(p[iWs + 1]);
        int m = 0;
        if (!isnan(v[0]))
            for (int k = 1; k < 4; ++k) {
                if (isnan(v[k])) {
                    m = k;
                    break;
                }
                if (v[k] > v[m]) m = k;
            }
        const T *q = (m < 2) ? p + m : p + iWs + (m - 2);
        dst[b * oss + ((long long)c * oHp + y + oph) * oWs + x + opw] = *q;
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
    static bool attr_set = false;  // per instantiation
    if (!attr_set || pl->smem_bytes > 48 * 1024) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        attr_set = true;
    }
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
    ep.saturate = e->saturate;
    ep.saturate2 = e->saturate2;
    ep.cap = e->cap;
    ep.cap2 = e->cap2;
    ep.scale = e->scale;
    ep.out_padded = e->out_padded;
    if (e->out_padded) {
        ep.oHp = e->out.hp;
        ep.oWs = e->out.ws;
        ep.oph = e->out.pad_h;
        ep.opw = e->out.pad_w;
        ep.o_sample_stride = e->out.sample_stride;
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

int usc_conv_forward(const usc_plan *pl, const void *blob, const void *x, void *y,
                     const usc_epilogue *epi, void *stream) {
    if (!pl || !blob || !x || !y) return fail(USC_ERR_VALUE, "null argument");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const usc_geometry &g = pl->g;
    Epi ep = make_epi(epi);
    if (ep.out_padded && pl->transposed)
        return fail(USC_ERR_UNSUPPORTED, "padded output of a transposed 1-D plan");
    if (ep.out_padded && (epi->out.channels != g.out_channels || epi->out.height != pl->out_h ||
                          epi->out.width != pl->out_w))
        return fail(USC_ERR_VALUE, "output layout does not match the plan");
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
    const long long total = (long long)n * l->sample_stride;
    const int grid = grid_for(total);
    switch (usc::elem_bytes(dtype)) {
        case 4:
            k_pad<float><<<grid, 256, 0, st>>>(static_cast<const float *>(src), static_cast<float *>(dst), n,
                                               l->channels, l->height, l->width, l->pad_h, l->pad_w, l->hp, l->ws);
            break;
        case 2:
            k_pad<uint16_t><<<grid, 256, 0, st>>>(static_cast<const uint16_t *>(src), static_cast<uint16_t *>(dst),
                                                  n, l->channels, l->height, l->width, l->pad_h, l->pad_w,
                                                  l->hp, l->ws);
            break;
        case 1:
            k_pad<int8_t><<<grid, 256, 0, st>>>(static_cast<const int8_t *>(src), static_cast<int8_t *>(dst), n,
                                                l->channels, l->height, l->width, l->pad_h, l->pad_w, l->hp, l->ws);
            break;
        default: return fail(USC_ERR_VALUE, "unknown dtype %d", dtype);
    }
    return cuda_check("k_pad launch");
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
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long long total = (long long)n * in_l->channels * OH * OW;
    if (dtype == USC_F32) {
        k_maxpool2<float><<<grid_for(total), 256, 0, st>>>(
            static_cast<const float *>(src), static_cast<float *>(dst), n, in_l->channels, OH, OW, in_l->hp,
            in_l->ws, in_l->pad_h, in_l->pad_w, in_l->sample_stride, out_l->hp, out_l->ws, out_l->pad_h,
            out_l->pad_w, out_l->sample_stride);
    } else if (dtype == USC_F16 || dtype == USC_CB4) {
        k_maxpool2<__half><<<grid_for(total), 256, 0, st>>>(
            static_cast<const __half *>(src), static_cast<__half *>(dst), n, in_l->channels, OH, OW, in_l->hp,
            in_l->ws, in_l->pad_h, in_l->pad_w, in_l->sample_stride, out_l->hp, out_l->ws, out_l->pad_h,
            out_l->pad_w, out_l->sample_stride);
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
