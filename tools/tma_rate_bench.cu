// Per-SM TMA load throughput on sm_100a (L2-resident source): one producer thread per CTA
// streams 2D boxes of 128-byte rows into a ring of S stages, a consumer thread releases
// each stage as soon as it lands (no compute).  Prints bytes delivered per clock per SM
// for box sizes, stage sizes, ring depths and cluster multicast (each CTA of a cluster
// issues 1/csz of a stage's boxes with .multicast::cluster to every CTA).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_rate_bench tools/tma_rate_bench.cu -lcuda
#include <cuda.h>
#include <cuda_fp16.h>
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

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void k_tma(const __grid_constant__ CUtensorMap map, int box_bytes, int boxes, int S, int iters,
                      int rows_total, int box_rows, int csz, int lanes, int prefetch, long long *cyc) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char *sm = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    const int stage = box_bytes * boxes;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + S * stage);
    uint64_t *empty = full + S;
    const uint32_t rank = csz > 1 ? cluster_rank() : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(csz));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (csz > 1)
        cluster_sync();
    else
        __syncthreads();
    const int cluster_id = blockIdx.x / csz;
    if (prefetch && threadIdx.x == 0)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map)) : "memory");
    if (threadIdx.x < lanes) {  // producer: lane l issues boxes l, l + lanes, ...
        const int l = threadIdx.x;
        for (int it = 0; it < iters; ++it) {
            const int s = it % S;
            if (it >= S) wait_parity(&empty[s], ((it / S) - 1) & 1);
            if (l == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(stage)
                             : "memory");
            for (int b = l; b < boxes; b += lanes) {
                if (csz > 1 && (b % csz) != (int)rank) continue;
                const int row = (int)(((long long)(cluster_id * 7919 + it * boxes + b) * box_rows) % rows_total);
                const uint32_t dst = su32(sm + s * stage + b * box_bytes);
                if (csz == 1)
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                        "%3}], [%4];" ::"r"(dst),
                        "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(row), "r"(su32(&full[s]))
                        : "memory");
                else
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::"
                        "cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
                        "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(row), "r"(su32(&full[s])),
                        "h"((uint16_t)((1u << csz) - 1))
                        : "memory");
            }
        }
    } else if (threadIdx.x == 32) {  // consumer
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const int s = it % S;
            wait_parity(&full[s], (it / S) & 1);
            for (int c = 0; c < csz; ++c) {  // release the slot to every producer that writes it
                if (csz == 1) {
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
                } else {
                    uint32_t remote;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(su32(&empty[s])), "r"(c));
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
                }
            }
        }
        cyc[blockIdx.x] = clock64() - t0;
    }
    if (csz > 1)
        cluster_sync();
    else
        __syncthreads();
}

int main() {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int rows_total = 1 << 17;  // 16 MB of 128-byte rows: L2-resident
    void *src = nullptr;
    cudaMalloc(&src, (size_t)rows_total * 128);
    cudaMemset(src, 0, (size_t)rows_total * 128);
    long long *cyc = nullptr;
    cudaMalloc(&cyc, 4096 * sizeof(long long));
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    struct Cfg {
        int box_rows, boxes, S, csz, lanes, prefetch, grid;
    };
    std::vector<Cfg> cfgs = {
        {128, 1, 4, 1, 1, 0, 0},  {128, 1, 4, 1, 1, 1, 0},  {128, 1, 4, 1, 1, 0, 1},  {128, 1, 12, 1, 1, 0, 1},
        {128, 6, 2, 1, 1, 0, 1},  {128, 6, 2, 1, 6, 0, 0},  {128, 6, 2, 1, 6, 1, 0},  {64, 12, 2, 1, 12, 0, 0},
        {128, 2, 6, 1, 2, 0, 0},  {64, 4, 6, 1, 4, 0, 0},   {128, 1, 12, 1, 1, 1, 16}, {128, 6, 2, 1, 1, 0, 16},
        {128, 6, 2, 1, 6, 0, 74}, {128, 6, 2, 2, 3, 0, 0},  {64, 12, 2, 2, 6, 0, 0},  {128, 4, 3, 4, 1, 0, 0}};
    printf("box_rows box_KB boxes_per_stage stage_KB depth cluster lanes prefetch grid | delivered_B_per_clk_per_SM issued_B_per_clk_per_SM\n");
    for (const Cfg &c : cfgs) {
        CUtensorMap map;
        const cuuint64_t dims[2] = {64, (cuuint64_t)rows_total};
        const cuuint64_t strides[1] = {128};
        const cuuint32_t box[2] = {64, (cuuint32_t)c.box_rows};
        const cuuint32_t es[2] = {1, 1};
        if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS) {
            printf("encode failed for box_rows %d\n", c.box_rows);
            continue;
        }
        const int box_bytes = c.box_rows * 128, stage = box_bytes * c.boxes;
        const int smem = c.S * stage + 1024 + 2 * c.S * 8;
        if (smem > 227 * 1024) continue;
        const int iters = (int)(64LL * 1024 * 1024 / stage);  // 64 MB per CTA
        const int grid = c.grid ? c.grid : sms / c.csz * c.csz;
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(grid);
        lc.blockDim = dim3(64);  // warp 0: producer lanes, warp 1 lane 0: consumer
        lc.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = c.csz;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        for (int rep = 0; rep < 2; ++rep)
            cudaLaunchKernelEx(&lc, k_tma, map, box_bytes, c.boxes, c.S, iters, rows_total, c.box_rows, c.csz, c.lanes,
                               c.prefetch, cyc);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return 1;
        }
        std::vector<long long> h(grid);
        cudaMemcpy(h.data(), cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (long long v : h) mx = v > mx ? v : mx;
        const double delivered = (double)iters * stage / mx;
        printf("%8d %6d %15d %8d %5d %7d %5d %8d %4d | %8.1f %8.1f\n", c.box_rows, box_bytes / 1024, c.boxes, stage / 1024,
               c.S, c.csz, c.lanes, c.prefetch, grid, delivered, delivered / c.csz);
    }
    return 0;
}
