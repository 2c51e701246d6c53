// common.cuh -- device helpers shared by the conv kernels: mbarrier + bulk async
// copy (TMA engine) PTX wrappers, operand kinds, binary16 rounding, epilogue.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <utility>

#include "usc_internal.h"

namespace usc_dev {


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
    // try_wait with a suspend-time hint: the warp sleeps in hardware until the phase
    // completes (or ~1 ms passes) instead of spinning on issue slots other warps need
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000)
        : "memory");
}

// Opt a kernel into the large dynamic shared-memory carve-out once per (kernel,
// device): the attribute is per device, and launches may come from several threads.
template <typename F>
inline cudaError_t ensure_smem_attr(F fn, std::atomic<uint64_t> &done, int bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

// --------------------------------------------------------------------------
// Programmatic dependent launch (PDL): a kernel launched with launch_pdl may start its
// prologue (barriers, TMEM, descriptor prefetch) while the previous kernel on the
// stream drains; it must call pdl_wait() before its first global-memory access
// (griddepcontrol.wait returns once the previous grid has completed and its writes
// are visible -- a no-op for a plain launch).  pdl_release() lets the next PDL kernel
// be scheduled onto SMs this grid frees.  USC_NO_PDL=1 turns the attribute off.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_release() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();  // host.cpp: false when USC_NO_PDL is set

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
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
    int oHp, oWs, oph, opw, oil, pool;
    int requant, rq_limit;
    float rq_scale;
    long long o_sample_stride;  // elements per sample (il 0) / interleave block (il 32, 64)
    int residual;               // add the shortcut tensor before the ReLU
    const void *res;
    int rC, rHp, rWs, rph, rpw, ril;
    long long r_sample_stride;
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


// element offset of logical (b, c, y, x) in an activation layout
struct LayoutD {
    int C, Hp, Ws, ph, pw, il;
    long long ss;  // sample (il 0) / block (il 32, 64) stride
};
__device__ __forceinline__ long long lay_index(const LayoutD &L, long long b, int c, int y, int x) {
    if (L.il)
        return (b / L.il) * L.ss + (((long long)c * L.Hp + y + L.ph) * L.Ws + x + L.pw) * L.il + b % L.il;
    return b * L.ss + ((long long)c * L.Hp + y + L.ph) * L.Ws + x + L.pw;
}
inline LayoutD to_dev(const usc_act_layout &l) {
    return LayoutD{l.channels, l.hp, l.ws, l.pad_h, l.pad_w, l.interleave, (long long)l.sample_stride};
}

}  // namespace usc_dev
