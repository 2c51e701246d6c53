// encode.cu -- device-side CSR encoder: build_csr (/root/reference/pkg/src/unsparse/
// csr.py:86-112) on the GPU, bit-identical to the host encoder (host.cpp
// usc_build_csr), for pruning loops whose masks change every iteration.
//
//   pass 1 (k_csr_count): one CTA per output channel counts the genuine nonzeros
//     (value != 0, csr.py:97-99) of its C*Kh*Kw weights;
//   n_nz = max(1, max_d count) (csr.py:103) is reduced on the device;
//   pass 2 (k_csr_build): one CTA per output channel writes its n_nz - count
//     padding entries (offset 0, weight 0) first, then the genuine entries in
//     ascending (c, kh, kw) order -- the stable order np.nonzero + argsort gives --
//     using a block-wide exclusive scan of the nonzero flags, tile by tile.
#include <cub/block/block_scan.cuh>

#include "common.cuh"

namespace {

constexpr int ENC_THREADS = 256;

__global__ void k_csr_count(const float *__restrict__ w, long long per, int *__restrict__ counts,
                            int *__restrict__ max_count) {
    const float *wd = w + (long long)blockIdx.x * per;
    int c = 0;
    for (long long k = threadIdx.x; k < per; k += blockDim.x) c += (wd[k] != 0.0f);
    __shared__ int red[ENC_THREADS / 32];
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int i = 0; i < ENC_THREADS / 32; ++i) t += red[i];
        counts[blockIdx.x] = t;
        atomicMax(max_count, t);
    }
}

__global__ void k_csr_build(const float *__restrict__ w, usc_geometry g, long long per, const int *__restrict__ counts,
                            const int *__restrict__ n_nz_dev, long long *__restrict__ row_ptr,
                            long long *__restrict__ col, float *__restrict__ theta) {
    using Scan = cub::BlockScan<int, ENC_THREADS>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int carry;
    const int d = blockIdx.x;
    const long long n_nz = max(1, *n_nz_dev);
    const int cnt = counts[d];
    const long long base = (long long)d * n_nz;
    const long long pad = n_nz - cnt;
    const float *wd = w + (long long)d * per;
    const long long Hp = g.input_h + 2 * g.pad_h, Wp = g.input_w + 2 * g.pad_w;
    const int KK = g.filter_h * g.filter_w;
    for (long long i = threadIdx.x; i < pad; i += blockDim.x) {  // padding first (csr.py:107-108)
        col[base + i] = 0;
        theta[base + i] = 0.0f;
    }
    if (threadIdx.x == 0) carry = 0;
    if (d == 0 && threadIdx.x == 0) row_ptr[0] = 0;
    if (threadIdx.x == 0) row_ptr[d + 1] = (long long)(d + 1) * n_nz;
    __syncthreads();
    for (long long t0 = 0; t0 < per; t0 += ENC_THREADS) {
        const long long k = t0 + threadIdx.x;
        const float v = k < per ? wd[k] : 0.0f;
        const int flag = v != 0.0f;
        int pos, total;
        Scan(tmp).ExclusiveSum(flag, pos, total);
        if (flag) {
            const long long c = k / KK, r = k % KK, kh = r / g.filter_w, kw = r % g.filter_w;
            const long long j = base + pad + carry + pos;
            col[j] = (c * Hp + kh) * Wp + kw;  // tap_to_offset (csr.py:25-27)
            theta[j] = v;
        }
        __syncthreads();
        if (threadIdx.x == 0) carry += total;
        __syncthreads();
    }
}

}  // namespace

extern "C" {

int usc_csr_count_device(const float *w, const usc_geometry *g, int32_t *counts, int32_t *n_nz, void *stream) {
    int rc = usc_geometry_check(g);
    if (rc) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long long per = (long long)g->in_channels * g->filter_h * g->filter_w;
    cudaMemsetAsync(n_nz, 0, sizeof(int32_t), st);
    k_csr_count<<<g->out_channels, ENC_THREADS, 0, st>>>(w, per, counts, n_nz);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return usc::fail(USC_ERR_CUDA, "k_csr_count: %s", cudaGetErrorString(e));
    return USC_OK;
}

int usc_build_csr_device(const float *w, const usc_geometry *g, const int32_t *counts, const int32_t *n_nz,
                         int64_t *row_ptr, int64_t *col, float *theta, void *stream) {
    int rc = usc_geometry_check(g);
    if (rc) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long long per = (long long)g->in_channels * g->filter_h * g->filter_w;
    k_csr_build<<<g->out_channels, ENC_THREADS, 0, st>>>(w, *g, per, counts, n_nz, reinterpret_cast<long long *>(row_ptr),
                                                       reinterpret_cast<long long *>(col), theta);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return usc::fail(USC_ERR_CUDA, "k_csr_build: %s", cudaGetErrorString(e));
    return USC_OK;
}

}  // extern "C"
