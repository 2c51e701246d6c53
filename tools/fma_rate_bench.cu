// FMA-pipe rates on sm_100a: FFMA vs FHFMA (fma.rn.f32.f16: fp32 += f16*f16) vs FMUL+FADD2.
// Prints warp instructions per clock per SM for each (8 independent chains per thread).
// Also the FMUL+FADD and FMUL+FADD2 mixes the bit-exact fp32 kernels issue.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fma_rate_bench tools/fma_rate_bench.cu
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__global__ void k_ffma(float *out, int iters, long long *cyc) {
    float acc[8];
    float a = threadIdx.x * 1e-3f, b = 1.0001f;
    for (int i = 0; i < 8; ++i) acc[i] = i;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = __fmaf_rn(acc[i], b, a);
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 1.2345f) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_fhfma(float *out, int iters, long long *cyc) {
    float acc[8];
    const unsigned short th = 0x3c01, xv = (unsigned short)(0x3800 + threadIdx.x);
    for (int i = 0; i < 8; ++i) acc[i] = i;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc[i]) : "h"(th), "h"(xv));
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 1.2345f) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// The fp32 BI64 inner-loop mix: per lane two samples, two FMUL then one packed FADD2
// (add.rn.f32x2) per MAC pair -- 3 warp instructions per 64 MACs.
__global__ void k_fmul_fadd2(float *out, int iters, long long *cyc) {
    unsigned long long acc[8];
    float a = threadIdx.x * 1e-3f, b = 1.0001f;
    for (int i = 0; i < 8; ++i) {
        float lo = i, hi = i + 0.5f;
        asm("mov.b64 %0, {%1, %2};" : "=l"(acc[i]) : "f"(lo), "f"(hi));
    }
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float p0, p1, lo, hi;  // products depend on the chain so they are not hoisted
            asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[i]));
            asm volatile("mul.rn.f32 %0, %1, %2;" : "=f"(p0) : "f"(lo), "f"(b));
            asm volatile("mul.rn.f32 %0, %1, %2;" : "=f"(p1) : "f"(hi), "f"(a));
            unsigned long long q;
            asm("mov.b64 %0, {%1, %2};" : "=l"(q) : "f"(p0), "f"(p1));
            asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(acc[i]) : "l"(q));
        }
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[i]));
        s += lo + hi;
    }
    if (s == 1.2345f) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
// Scalar reference mix: FMUL then FADD per MAC.
__global__ void k_fmul_fadd(float *out, int iters, long long *cyc) {
    float acc[8];
    float a = threadIdx.x * 1e-3f, b = 1.0001f;
    for (int i = 0; i < 8; ++i) acc[i] = i;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float p;
            asm volatile("mul.rn.f32 %0, %1, %2;" : "=f"(p) : "f"(acc[i]), "f"(b));
            asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(acc[i]) : "f"(p));
        }
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 1.2345f) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <typename F>
void run(const char *name, F kern, int iters, double instr_per_thread_iter) {
    float *out;
    long long *cyc;
    cudaMalloc(&out, 4);
    cudaMalloc(&cyc, 148 * 8);
    kern<<<148, 512>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    kern<<<148, 512>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("{\"test\": \"%s\", \"warp_instr_per_clk_per_sm\": %.3f}\n", name, instr_per_thread_iter * iters * 16 / mx);
}
int main() {
    run("ffma", k_ffma, 4096, 8);
    run("fhfma", k_fhfma, 4096, 8);
    // MAC rates: ffma/fhfma 32 MAC per warp instr; fmul_fadd 16; fmul_fadd2 64 per 3 instrs
    run("fmul_fadd (instr = 2 per 32 MAC)", k_fmul_fadd, 4096, 16);
    run("fmul_fadd2 (instr = 3 per 64 MAC)", k_fmul_fadd2, 4096, 24);
    return 0;
}
