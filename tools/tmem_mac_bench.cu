// MAC-loop microbenchmark: the sparse conv inner loop (entry pair -> 2x(2 rows x 4 px)
// values -> FMUL+FADD in order) fed from shared memory (LDS, BI32 / BI64) vs from tensor
// memory (tcgen05.ld.32x32b, dynamic column per entry, one wait::ld per pair).
// Prints fp32 MACs per clock per SM (128 B/clk of LDS = 32 fp32 MAC/clk/SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_mac_bench tools/tmem_mac_bench.cu
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int NE = 256;  // entries in the table (pairs = NE/2)

// x4 load of 4 consecutive columns
__device__ __forceinline__ void ldtm4(uint32_t a, float &v0, float &v1, float &v2, float &v3) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v0), "=f"(v1), "=f"(v2), "=f"(v3) : "r"(a));
}
__device__ __forceinline__ void ldtm8(uint32_t a, float (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "r"(a));
}

// TMEM-fed, one sample per lane (BI32-like): per entry 2 x4 loads (2 rows x 4 px)
template <int DW>
__global__ void k_tmem1(const int2 *ents_g, float *out, int iters, long long *cyc) {
    __shared__ uint32_t taddr_s;
    __shared__ int2 ents[NE];
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < NE; i += blockDim.x) ents[i] = ents_g[i];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16);
    float acc[DW][8];
    for (int d = 0; d < DW; ++d)
        for (int p = 0; p < 8; ++p) acc[d][p] = 0.f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int d = 0; d < DW; ++d) {
#pragma unroll 1
            for (int e = 0; e < NE / DW; e += 2) {
                const int2 n0 = ents[(d * (NE / DW) + e + warp) & (NE - 1)];
                const int2 n1 = ents[(d * (NE / DW) + e + 1 + warp) & (NE - 1)];
                float a[8], b[8];
                ldtm4(base + n0.x, a[0], a[1], a[2], a[3]);
                ldtm4(base + n0.x + 40, a[4], a[5], a[6], a[7]);
                ldtm4(base + n1.x, b[0], b[1], b[2], b[3]);
                ldtm4(base + n1.x + 40, b[4], b[5], b[6], b[7]);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                const float t0v = __int_as_float(n0.y), t1v = __int_as_float(n1.y);
#pragma unroll
                for (int p = 0; p < 8; ++p) acc[d][p] = __fadd_rn(acc[d][p], __fmul_rn(t0v, a[p]));
#pragma unroll
                for (int p = 0; p < 8; ++p) acc[d][p] = __fadd_rn(acc[d][p], __fmul_rn(t1v, b[p]));
            }
        }
    }
    long long t1 = clock64();
    float s = 0;
    for (int d = 0; d < DW; ++d)
        for (int p = 0; p < 8; ++p) s += acc[d][p];
    if (s == 1.2345f) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

// TMEM-fed, two samples per lane (column pairs): per entry 2 x8 loads, FMUL x2 + FADD2
__device__ __forceinline__ void fadd2(unsigned long long &acc, float lo, float hi) {
    unsigned long long q;
    asm("mov.b64 %0, {%1, %2};" : "=l"(q) : "f"(lo), "f"(hi));
    asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(q));
}
template <int DW>
__global__ void k_tmem2(const int2 *ents_g, float *out, int iters, long long *cyc) {
    __shared__ uint32_t taddr_s;
    __shared__ int2 ents[NE];
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < NE; i += blockDim.x) ents[i] = ents_g[i];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16);
    unsigned long long acc[DW][4];
    for (int d = 0; d < DW; ++d)
        for (int p = 0; p < 4; ++p) acc[d][p] = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int d = 0; d < DW; ++d) {
#pragma unroll 1
            for (int e = 0; e < NE / DW; e += 2) {
                const int2 n0 = ents[(d * (NE / DW) + e + warp) & (NE - 1)];
                const int2 n1 = ents[(d * (NE / DW) + e + 1 + warp) & (NE - 1)];
                float a[8], b[8];  // 4 px x 2 samples, one row (P = 4 per entry)
                ldtm8(base + n0.x, a);
                ldtm8(base + n1.x, b);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                const float t0v = __int_as_float(n0.y), t1v = __int_as_float(n1.y);
#pragma unroll
                for (int p = 0; p < 4; ++p) fadd2(acc[d][p], __fmul_rn(t0v, a[2 * p]), __fmul_rn(t0v, a[2 * p + 1]));
#pragma unroll
                for (int p = 0; p < 4; ++p) fadd2(acc[d][p], __fmul_rn(t1v, b[2 * p]), __fmul_rn(t1v, b[2 * p + 1]));
            }
        }
    }
    long long t1 = clock64();
    float s = 0;
    for (int d = 0; d < DW; ++d)
        for (int p = 0; p < 4; ++p) s += __uint_as_float((unsigned)acc[d][p]);
    if (s == 1.2345f) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

// LDS-fed BI32 (one sample per lane): per entry 8 LDS.32 (2 rows x 4 px)
template <int DW>
__global__ void k_lds1(const int2 *ents_g, float *out, int iters, long long *cyc) {
    __shared__ float xs[40 * 8 * 32];
    __shared__ int2 ents[NE];
    for (int i = threadIdx.x; i < NE; i += blockDim.x) ents[i] = ents_g[i];
    for (int i = threadIdx.x; i < 40 * 8 * 32; i += blockDim.x) xs[i] = i * 1e-3f;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float acc[DW][8];
    for (int d = 0; d < DW; ++d)
        for (int p = 0; p < 8; ++p) acc[d][p] = 0.f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int d = 0; d < DW; ++d) {
#pragma unroll 1
            for (int e = 0; e < NE / DW; e += 2) {
                const int2 n0 = ents[(d * (NE / DW) + e + warp) & (NE - 1)];
                const int2 n1 = ents[(d * (NE / DW) + e + 1 + warp) & (NE - 1)];
                float a[8], b[8];
#pragma unroll
                for (int p = 0; p < 8; ++p) {
                    a[p] = xs[((n0.x & 255) + (p >> 2) * 40 + (p & 3)) * 32 + lane];
                    b[p] = xs[((n1.x & 255) + (p >> 2) * 40 + (p & 3)) * 32 + lane];
                }
                const float t0v = __int_as_float(n0.y), t1v = __int_as_float(n1.y);
#pragma unroll
                for (int p = 0; p < 8; ++p) acc[d][p] = __fadd_rn(acc[d][p], __fmul_rn(t0v, a[p]));
#pragma unroll
                for (int p = 0; p < 8; ++p) acc[d][p] = __fadd_rn(acc[d][p], __fmul_rn(t1v, b[p]));
            }
        }
    }
    long long t1 = clock64();
    float s = 0;
    for (int d = 0; d < DW; ++d)
        for (int p = 0; p < 8; ++p) s += acc[d][p];
    if (s == 1.2345f) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}


template <int DW>
__global__ void k_tmem2q(const int2 *ents_g, float *out, int iters, long long *cyc) {
    __shared__ uint32_t taddr_s;
    __shared__ int2 ents[NE];
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < NE; i += blockDim.x) ents[i] = ents_g[i];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16);
    unsigned long long acc[DW][4];
    for (int d = 0; d < DW; ++d)
        for (int p = 0; p < 4; ++p) acc[d][p] = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int d = 0; d < DW; ++d) {
#pragma unroll 1
            for (int e = 0; e < NE / DW; e += 4) {
                int2 n[4];
                float a[4][8];
#pragma unroll
                for (int u = 0; u < 4; ++u) n[u] = ents[(d * (NE / DW) + e + u + warp) & (NE - 1)];
#pragma unroll
                for (int u = 0; u < 4; ++u) ldtm8(base + n[u].x, a[u]);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float t = __int_as_float(n[u].y);
#pragma unroll
                    for (int p = 0; p < 4; ++p) fadd2(acc[d][p], __fmul_rn(t, a[u][2 * p]), __fmul_rn(t, a[u][2 * p + 1]));
                }
            }
        }
    }
    long long t1 = clock64();
    float s = 0;
    for (int d = 0; d < DW; ++d)
        for (int p = 0; p < 4; ++p) s += __uint_as_float((unsigned)acc[d][p]);
    if (s == 1.2345f) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

// LDS-fed BI64 (two samples per lane): per entry 4 LDS.64 (4 px x 2 samples)
template <int DW>
__global__ void k_lds2(const int2 *ents_g, float *out, int iters, long long *cyc) {
    __shared__ float2 xs[20 * 8 * 32];
    __shared__ int2 ents[NE];
    for (int i = threadIdx.x; i < NE; i += blockDim.x) ents[i] = ents_g[i];
    for (int i = threadIdx.x; i < 20 * 8 * 32; i += blockDim.x) xs[i] = make_float2(i * 1e-3f, i);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long acc[DW][4];
    for (int d = 0; d < DW; ++d)
        for (int p = 0; p < 4; ++p) acc[d][p] = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int d = 0; d < DW; ++d) {
#pragma unroll 1
            for (int e = 0; e < NE / DW; e += 2) {
                const int2 n0 = ents[(d * (NE / DW) + e + warp) & (NE - 1)];
                const int2 n1 = ents[(d * (NE / DW) + e + 1 + warp) & (NE - 1)];
                float2 a[4], b[4];
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    a[p] = xs[((n0.x & 127) + p) * 32 + lane];
                    b[p] = xs[((n1.x & 127) + p) * 32 + lane];
                }
                const float t0v = __int_as_float(n0.y), t1v = __int_as_float(n1.y);
#pragma unroll
                for (int p = 0; p < 4; ++p) fadd2(acc[d][p], __fmul_rn(t0v, a[p].x), __fmul_rn(t0v, a[p].y));
#pragma unroll
                for (int p = 0; p < 4; ++p) fadd2(acc[d][p], __fmul_rn(t1v, b[p].x), __fmul_rn(t1v, b[p].y));
            }
        }
    }
    long long t1 = clock64();
    float s = 0;
    for (int d = 0; d < DW; ++d)
        for (int p = 0; p < 4; ++p) s += __uint_as_float((unsigned)acc[d][p]);
    if (s == 1.2345f) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename F>
void run(const char *name, F kern, int threads, int iters, double macs_per_warp_iter) {
    float *out;
    long long *cyc;
    int2 *ents;
    int2 h[NE];
    for (int i = 0; i < NE; ++i) {
        float t = 0.5f + i * 1e-3f;
        int ti;
        memcpy(&ti, &t, 4);
        h[i] = make_int2((i * 37) % 200, ti);
    }
    cudaMalloc(&out, 4);
    cudaMalloc(&cyc, 148 * 8);
    cudaMalloc(&ents, sizeof h);
    cudaMemcpy(ents, h, sizeof h, cudaMemcpyHostToDevice);
    kern<<<148, threads>>>(ents, out, iters, cyc);
    cudaDeviceSynchronize();
    kern<<<148, threads>>>(ents, out, iters, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    long long hc[148];
    cudaMemcpy(hc, cyc, sizeof hc, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = hc[i] > mx ? hc[i] : mx;
    printf("{\"test\": \"%s\", \"warps\": %d, \"mac_per_clk_per_sm\": %.1f, \"err\": \"%s\"}\n", name, threads / 32,
           macs_per_warp_iter * (threads / 32) * iters / mx, cudaGetErrorString(e));
    cudaFree(out);
    cudaFree(cyc);
    cudaFree(ents);
}

int main() {
    const int it = 64;
    for (int w : {8, 12, 16}) {
        // per warp-iteration: NE entries x 8 pixel-MACs x 32 lanes (x2 samples for tmem2 with 4 px)
        run("lds_bi32_dw4", k_lds1<4>, 32 * w, it, NE * 8.0 * 32);
        run("tmem_spl1_dw4", k_tmem1<4>, 32 * w, it, NE * 8.0 * 32);
        run("tmem_spl2_dw4", k_tmem2<4>, 32 * w, it, NE * 8.0 * 32);
        run("tmem_spl2_dw8", k_tmem2<8>, 32 * w, it, NE * 8.0 * 32);
        run("tmem_spl2q_dw4", k_tmem2q<4>, 32 * w, it, NE * 8.0 * 32);
        run("lds_bi64_dw4", k_lds2<4>, 32 * w, it, NE * 8.0 * 32);
    }
    return 0;
}
