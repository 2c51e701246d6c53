// layout.cu -- batch-interleaved (BI64) <-> NHWC transposes for the per-layer backend
// dispatcher (the reference's backend_config, bench.py:212-227 /
// pipeline.py:381-389): a layer the dispatcher hands to cuDNN reads its input as NHWC
// (channels_last, what cuDNN's fp16 tensor-core convolutions consume) and its NHWC
// output is written back into the network's resident BI64 layout with the layer's
// epilogue (binary16 saturation, residual add, ReLU) fused.
//
// Register transposes, no shared memory: a warp owns one (64-sample block, pixel,
// 16-channel group) unit; lane l owns the sample pair (2l, 2l+1).  In BI64 a 32-bit
// word is one channel's sample pair, so the warp's 16 word loads/stores per side are
// 128-byte lines; two PRMTs turn the words of channels (c, c+1) into the NHWC words
// of samples 2l and 2l+1, written as two full 32-byte sectors per sample row.
#include "common.cuh"
#include "usc_internal.h"

using namespace usc_dev;

namespace {

constexpr int kGroup = 16;  // channels per warp unit

__device__ __forceinline__ uint32_t sat16x2(uint32_t w) {  // +-inf from a finite overflow -> +-65504 per half
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const uint32_t h = (w >> (16 * k)) & 0xffffu;
        if ((h & 0x7fffu) == 0x7c00u) w = (w & ~(0xffffu << (16 * k))) | (((h & 0x8000u) | 0x7bffu) << (16 * k));
    }
    return w;
}

// where(v > 0, v, 0) per binary16 half (nn.py:96-98): -0, NaN and negatives -> +0
__device__ __forceinline__ uint32_t relu16x2(uint32_t w) {
    uint32_t out = 0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const uint32_t h = (w >> (16 * k)) & 0xffffu, m = h & 0x7fffu;
        if (!(h & 0x8000u) && m != 0 && m <= 0x7c00u) out |= h << (16 * k);
    }
    return out;
}

// BI64 (binary16) -> NHWC [n][H][W][C]
__global__ void k_bi_to_nhwc(const uint32_t *__restrict__ src, __half *__restrict__ dst, int n, int H, int W,
                             const LayoutD L, long long units) {
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    const int G = L.C / kGroup;
    const long long cword = (long long)L.Hp * L.Ws * 32;  // words between channels
    for (long long u = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); u < units; u += warps) {
        const int cg = static_cast<int>(u % G);
        const long long pu = u / G;
        const int pix = static_cast<int>(pu % (H * W));
        const long long nb = pu / (H * W);
        const int y = pix / W, x = pix % W;
        const long long base = lay_index(L, nb * 64, cg * kGroup, y, x) / 2 + lane;  // in words
        uint32_t w[kGroup];
#pragma unroll
        for (int k = 0; k < kGroup; ++k) w[k] = __ldg(src + base + k * cword);
        uint32_t r0[kGroup / 2], r1[kGroup / 2];
#pragma unroll
        for (int k = 0; k < kGroup / 2; ++k) {
            r0[k] = __byte_perm(w[2 * k], w[2 * k + 1], 0x5410);  // sample 2l: channels (c, c+1)
            r1[k] = __byte_perm(w[2 * k], w[2 * k + 1], 0x7632);  // sample 2l+1
        }
        const long long b0 = nb * 64 + 2 * lane;
        const long long o = ((b0 * H + y) * W + x) * L.C + cg * kGroup;
        if (b0 < n) {
            uint4 *p = reinterpret_cast<uint4 *>(dst + o);
            p[0] = make_uint4(r0[0], r0[1], r0[2], r0[3]);
            p[1] = make_uint4(r0[4], r0[5], r0[6], r0[7]);
        }
        if (b0 + 1 < n) {
            uint4 *p = reinterpret_cast<uint4 *>(dst + o + (long long)H * W * L.C);
            p[0] = make_uint4(r1[0], r1[1], r1[2], r1[3]);
            p[1] = make_uint4(r1[4], r1[5], r1[6], r1[7]);
        }
    }
}

// NHWC [n][H][W][C] -> BI64 interior, with the layer epilogue:
// v = sat16(y); residual: v = sat16(v + r) (binary16 add = round16 of the exact sum);
// ReLU: where(v > 0, v, 0) (NaN -> 0)
__global__ void k_nhwc_to_bi(const __half *__restrict__ src, uint32_t *__restrict__ dst, int n, int H, int W,
                             const LayoutD L, const uint32_t *__restrict__ res, const LayoutD R, int relu,
                             long long units) {
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    const int G = L.C / kGroup;
    const long long cword = (long long)L.Hp * L.Ws * 32, rcword = (long long)R.Hp * R.Ws * 32;
    for (long long u = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); u < units; u += warps) {
        const int cg = static_cast<int>(u % G);
        const long long pu = u / G;
        const int pix = static_cast<int>(pu % (H * W));
        const long long nb = pu / (H * W);
        const int y = pix / W, x = pix % W;
        const long long b0 = nb * 64 + 2 * lane;
        const long long o = ((b0 * H + y) * W + x) * L.C + cg * kGroup;
        uint4 a[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)}, b[2] = {a[0], a[1]};
        if (b0 < n) {
            const uint4 *p = reinterpret_cast<const uint4 *>(src + o);
            a[0] = __ldg(p);
            a[1] = __ldg(p + 1);
        }
        if (b0 + 1 < n) {
            const uint4 *p = reinterpret_cast<const uint4 *>(src + o + (long long)H * W * L.C);
            b[0] = __ldg(p);
            b[1] = __ldg(p + 1);
        }
        const uint32_t r0[8] = {a[0].x, a[0].y, a[0].z, a[0].w, a[1].x, a[1].y, a[1].z, a[1].w};
        const uint32_t r1[8] = {b[0].x, b[0].y, b[0].z, b[0].w, b[1].x, b[1].y, b[1].z, b[1].w};
        const long long base = lay_index(L, nb * 64, cg * kGroup, y, x) / 2 + lane;
        const long long rbase = res ? lay_index(R, nb * 64, cg * kGroup, y, x) / 2 + lane : 0;
#pragma unroll
        for (int k = 0; k < kGroup; ++k) {
            // channel c+k, samples (2l, 2l+1)
            const uint32_t lo = r0[k / 2], hi = r1[k / 2];
            uint32_t w = sat16x2((k & 1) ? __byte_perm(lo, hi, 0x7632) : __byte_perm(lo, hi, 0x5410));
            if (res) {
                const uint32_t rw = __ldg(res + rbase + k * rcword);
                __half2 s = __hadd2(*reinterpret_cast<const __half2 *>(&w), *reinterpret_cast<const __half2 *>(&rw));
                w = sat16x2(*reinterpret_cast<uint32_t *>(&s));
            }
            if (relu) w = relu16x2(w);
            dst[base + k * cword] = w;
        }
    }
}

// in place, any layout (elementwise): v = sat16(y); residual: v = sat16(v + r); ReLU
__global__ void k_f16_epilogue(uint32_t *__restrict__ y, const uint32_t *__restrict__ res, long long words,
                               int relu) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < words;
         i += (long long)gridDim.x * blockDim.x) {
        uint32_t w = sat16x2(y[i]);
        if (res) {
            const uint32_t rw = __ldg(res + i);
            __half2 s = __hadd2(*reinterpret_cast<const __half2 *>(&w), *reinterpret_cast<const __half2 *>(&rw));
            w = sat16x2(*reinterpret_cast<uint32_t *>(&s));
        }
        if (relu) w = relu16x2(w);
        y[i] = w;
    }
}

int check_bi(const usc_act_layout *l, int32_t n) {
    if (!l || n < 1) return usc::fail(USC_ERR_VALUE, "layout conversion: bad arguments");
    if (l->interleave != 64) return usc::fail(USC_ERR_UNSUPPORTED, "layout conversion needs the BI64 layout");
    if (l->channels % kGroup) return usc::fail(USC_ERR_UNSUPPORTED, "layout conversion needs channels %% 16 == 0");
    return USC_OK;
}

int grid_of(long long units) {
    const long long blocks = (units + 3) / 4;  // 4 warps per CTA
    return static_cast<int>(blocks < 148LL * 16 ? blocks : 148LL * 16);
}

}  // namespace

int usc_bi_to_nhwc(const usc_act_layout *l, int32_t n, const void *src, void *dst, void *stream) {
    if (int rc = check_bi(l, n)) return rc;
    const LayoutD L = to_dev(*l);
    const long long units = (long long)((n + 63) / 64) * l->height * l->width * (l->channels / kGroup);
    k_bi_to_nhwc<<<grid_of(units), 128, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint32_t *>(src), static_cast<__half *>(dst), n, l->height, l->width, L, units);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? USC_OK : usc::fail(USC_ERR_CUDA, "k_bi_to_nhwc: %s", cudaGetErrorString(e));
}

int usc_nhwc_to_bi(const usc_act_layout *l, int32_t n, const void *src, void *dst, const usc_act_layout *res_layout,
                   const void *res, int32_t relu, void *stream) {
    if (int rc = check_bi(l, n)) return rc;
    if (res && (!res_layout || res_layout->interleave != 64 || res_layout->channels != l->channels ||
                res_layout->height != l->height || res_layout->width != l->width))
        return usc::fail(USC_ERR_VALUE, "residual layout does not match the output");
    const LayoutD L = to_dev(*l);
    const LayoutD R = res ? to_dev(*res_layout) : L;
    const long long units = (long long)((n + 63) / 64) * l->height * l->width * (l->channels / kGroup);
    k_nhwc_to_bi<<<grid_of(units), 128, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const __half *>(src), static_cast<uint32_t *>(dst), n, l->height, l->width, L,
        static_cast<const uint32_t *>(res), R, relu, units);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? USC_OK : usc::fail(USC_ERR_CUDA, "k_nhwc_to_bi: %s", cudaGetErrorString(e));
}

int usc_f16_epilogue(void *y, const void *res, int64_t count, int32_t relu, void *stream) {
    if (!y || count < 0 || (count & 1)) return usc::fail(USC_ERR_VALUE, "f16 epilogue: even element count needed");
    const long long words = count / 2;
    if (!words) return USC_OK;
    const long long blocks = (words + 255) / 256;
    k_f16_epilogue<<<static_cast<int>(blocks < 148LL * 32 ? blocks : 148LL * 32), 256, 0,
                     static_cast<cudaStream_t>(stream)>>>(static_cast<uint32_t *>(y),
                                                          static_cast<const uint32_t *>(res), words, relu);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? USC_OK : usc::fail(USC_ERR_CUDA, "k_f16_epilogue: %s", cudaGetErrorString(e));
}
