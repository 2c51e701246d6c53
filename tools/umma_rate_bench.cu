// tcgen05.mma issue rate on sm_100a with operands resident in shared memory (no TMA, no
// epilogue): one thread per CTA issues R x 12 MMAs (kind::f16, M = 128, K = 16) on a fixed
// smem A tile (K-major, SW128) and B tile (K-major or MN-major, SW128), commits to an
// mbarrier every 12 MMAs and keeps INFL such batches in flight.  Prints the dense fp16 rate per SM and for
// 148 SMs, per (N, B major) -- the tensor-core ceiling of k_dtc's stage shapes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_rate_bench tools/umma_rate_bench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;
    d |= 2ull << 61;
    return d;
}

template <int N, bool BMN, int INFL>
__global__ void __launch_bounds__(128, 1) k(int reps, long long *cyc) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char *sm = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar[INFL];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (48 + 96) * 1024 / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(sm)[i] = make_uint4(0x3c003c00u, 0, 0, 0);
    if (threadIdx.x == 0) {
        for (int i = 0; i < INFL; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[i])), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "n"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = (1u << 4) | (BMN ? (1u << 16) : 0u) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint32_t abase = su32(sm), bbase = abase + 48 * 1024;
        const long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int q = 0; q < 3; ++q)
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint64_t ad = desc_sw128(abase + q * 16384 + kk * 32, 16, 1024);
                    const uint64_t bd = BMN ? desc_sw128(bbase + q * 8192 + kk * 16 * 128, 8192, 1024)
                                            : desc_sw128(bbase + q * (N * 128) + kk * 32, 16, 1024);
                    const uint32_t acc = (r > 0 || q > 0 || kk > 0) ? 1u : 0u;
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                                 "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[r % INFL]))
                         : "memory");
            if (r >= INFL - 1) {  // keep INFL batches in flight
                uint32_t ok = 0;
                const int rr = r - (INFL - 1);
                while (!ok)
                    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                                 : "=r"(ok)
                                 : "r"(su32(&bar[rr % INFL])), "r"((rr / INFL) & 1)
                                 : "memory");
            }
        }
        cyc[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256));
    }
}

template <int N, bool BMN, int INFL>
void run(const char *name, long long *cyc) {
    const int smem = (48 + 96) * 1024 + 1024, reps = 20000;
    cudaFuncSetAttribute(k<N, BMN, INFL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<N, BMN, INFL><<<148, 128, smem>>>(reps, cyc);
    k<N, BMN, INFL><<<148, 128, smem>>>(reps, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("%s: %s\n", name, cudaGetErrorString(e));
        return;
    }
    long long h[148], mx = 0;
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    for (long long v : h) mx = v > mx ? v : mx;
    const double macs = (double)reps * 12 * 128 * N * 16;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-22s %7.0f MAC/clk/SM  (%5.0f clk per 12 MMAs; %6.1f TF/s at %d MHz x 148)\n", name, macs / mx,
           (double)mx / reps, 2.0 * macs / mx * 148 * clk * 1e3 / 1e12, clk / 1000);
}

int main() {
    long long *cyc = nullptr;
    cudaMalloc(&cyc, 148 * sizeof(long long));
    run<256, true, 1>("N=256 MN 1 in flight", cyc);
    run<256, true, 2>("N=256 MN 2 in flight", cyc);
    run<256, true, 4>("N=256 MN 4 in flight", cyc);
    run<128, true, 1>("N=128 MN 1 in flight", cyc);
    run<128, true, 4>("N=128 MN 4 in flight", cyc);
    run<64, false, 1>("N=64 K 1 in flight", cyc);
    run<64, false, 4>("N=64 K 4 in flight", cyc);
    return 0;
}
