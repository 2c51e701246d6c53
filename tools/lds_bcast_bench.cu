// Shared-memory broadcast load cost on sm_100a: warp-uniform LDS.32 / LDS.64 / LDS.128
// (every lane reads the same address) vs a conflict-free per-lane LDS.64.  Prints loads
// per clock per SM (1.0 = one wavefront per clock).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lds_bcast_bench tools/lds_bcast_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int BYTES, bool BCAST>
__global__ void k(float *out, int iters, long long *cyc) {
    __shared__ __align__(16) uint32_t buf[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = i;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t acc = 0;
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint32_t idx = ((it * 16 + j) * 4 + warp * 64) & 4095;
            const uint32_t a = base + (BCAST ? idx * 4 : (idx * 4 + lane * BYTES) & 32767) & ~(BYTES - 1);
            if constexpr (BYTES == 4) {
                uint32_t v;
                asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
                acc += v;
            } else if constexpr (BYTES == 8) {
                uint32_t v0, v1;
                asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(v0), "=r"(v1) : "r"(a));
                acc += v0 ^ v1;
            } else {
                uint32_t v0, v1, v2, v3;
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3) : "r"(a));
                acc += v0 ^ v1 ^ v2 ^ v3;
            }
        }
    }
    long long t1 = clock64();
    if (acc == 12345u) out[0] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename F>
void run(const char *name, F kern, int iters) {
    float *out;
    long long *cyc;
    cudaMalloc(&out, 4);
    cudaMalloc(&cyc, 148 * 8);
    const int threads = 512;
    kern<<<148, threads>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    kern<<<148, threads>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("{\"test\": \"%s\", \"warp_loads_per_clk_per_sm\": %.3f}\n", name, 16.0 * iters * (threads / 32) / mx);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    run("bcast_lds32", k<4, true>, 2048);
    run("bcast_lds64", k<8, true>, 2048);
    run("bcast_lds128", k<16, true>, 2048);
    run("lane_lds32", k<4, false>, 2048);
    run("lane_lds64", k<8, false>, 2048);
    run("lane_lds128", k<16, false>, 2048);
    return 0;
}
