// TMA delivery per SM for the tensor-core backend's activation reads, by layout: a row window
// of 6 pixels x 64 channels x 64 samples (binary16, 48 KB) from
//  (a) BI64  [block][C][Hp][Wp][64]: 64 channel planes, 768-B runs 148 KB apart;
//  (b) pixel-major [block][Hp][Wp][C][64]: one contiguous 48-KB run;
// plus the 3 weight tiles [64 d][64 k] of a stage (24 KB), one stage = one TMA per lane.
// Ring of S stages per CTA, 148 CTAs, 1 producer warp / 1 consumer thread (no compute).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_layout_bench tools/tma_layout_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_parity(uint64_t *bar, uint32_t ph) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(ok)
                     : "r"(su32(bar)), "r"(ph)
                     : "memory");
}

__global__ void k(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap wmap, int layout, int S,
                  int iters, int Hp, int Wp, int NB, long long *cyc) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char *sm = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    const int stage = 48 * 1024 + 24 * 1024;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + S * stage), *empty = full + S;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(1));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        for (int it = 0; it < iters; ++it) {
            const int s = it % S;
            if (it >= S) wait_parity(&empty[s], ((it / S) - 1) & 1);
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(stage)
                             : "memory");
            __syncwarp();
            const unsigned long long t = (unsigned long long)blockIdx.x * 977 + it * 13;
            const int x0 = (int)(t % (Wp - 6)), y = (int)((t / 7) % Hp), nb = (int)((t / 97) % NB);
            const uint32_t dst = su32(sm + s * stage);
            if (lane < 3)
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                                 dst + 48 * 1024 + lane * 8192),
                             "l"(reinterpret_cast<uint64_t>(&wmap)), "r"((lane * 3 + (it % 3)) * 64), "r"(0),
                             "r"(su32(&full[s]))
                             : "memory");
            else if (lane == 3) {
                // (a) dims (s, x, y, c, nb) box (64, 6, 1, 64, 1) -- re-ordered as (s, c, x, y, nb) for the
                // same bytes; (b) dims (s, c, x, y, nb) box (64, 64, 6, 1, 1), contiguous
                asm volatile(
                    "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
                        dst),
                    "l"(reinterpret_cast<uint64_t>(&xmap)), "r"(0), "r"(0), "r"(x0), "r"(y), "r"(nb), "r"(su32(&full[s]))
                    : "memory");
            }
        }
    } else if (threadIdx.x == 32) {
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const int s = it % S;
            wait_parity(&full[s], (it / S) & 1);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
        }
        cyc[blockIdx.x] = clock64() - t0;
    }
    __syncthreads();
}

int main() {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    const int NB = 4, C = 64, Hp = 34, Wp = 34;  // the 64->64 @32 layer's padded input, batch 256
    const size_t elems = (size_t)NB * C * Hp * Wp * 64;
    void *x = nullptr, *w = nullptr;
    cudaMalloc(&x, elems * 2);
    cudaMemset(x, 0, elems * 2);
    cudaMalloc(&w, 64 * 9 * 64 * 2 * 8);
    cudaMemset(w, 0, 64 * 9 * 64 * 2 * 8);
    long long *cyc = nullptr;
    cudaMalloc(&cyc, 148 * sizeof(long long));
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    CUtensorMap wmap;
    {
        const cuuint64_t dims[2] = {9 * 64 * 8, 64}, strides[1] = {9 * 64 * 8 * 2};
        const cuuint32_t box[2] = {64, 64}, es[2] = {1, 1};
        enc(&wmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, w, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    printf("layout S | B/clk/SM delivered\n");
    for (int layout = 0; layout < 2; ++layout)
        for (int S : {2, 3}) {
            CUtensorMap xmap;
            const cuuint64_t dims[5] = {64, (cuuint64_t)C, (cuuint64_t)Wp, (cuuint64_t)Hp, (cuuint64_t)NB};
            cuuint64_t strides[4];
            if (layout == 0) {  // BI64 [nb][c][y][x][s] viewed as (s, c, x, y, nb)
                strides[0] = (cuuint64_t)Hp * Wp * 128;
                strides[1] = 128;
                strides[2] = (cuuint64_t)Wp * 128;
            } else {  // pixel-major [nb][y][x][c][s]
                strides[0] = 128;
                strides[1] = (cuuint64_t)C * 128;
                strides[2] = (cuuint64_t)Wp * C * 128;
            }
            strides[3] = (cuuint64_t)C * Hp * Wp * 128;
            const cuuint32_t box[5] = {64, 64, 6, 1, 1}, es[5] = {1, 1, 1, 1, 1};
            if (enc(&xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
                CUDA_SUCCESS) {
                printf("encode failed\n");
                return 1;
            }
            const int stage = 72 * 1024, smem = S * stage + 1024 + 64;
            if (smem > 227 * 1024) continue;
            const int iters = 2000;
            for (int rep = 0; rep < 2; ++rep) k<<<148, 64, smem>>>(xmap, wmap, layout, S, iters, Hp, Wp, NB, cyc);
            cudaDeviceSynchronize();
            std::vector<long long> h(148);
            cudaMemcpy(h.data(), cyc, 148 * sizeof(long long), cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (long long v : h) mx = v > mx ? v : mx;
            printf("%s %d | %.1f\n", layout ? "pixel-major" : "BI64       ", S, (double)iters * stage / mx);
        }
    return 0;
}
