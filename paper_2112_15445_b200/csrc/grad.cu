// grad.cu -- the training kernels of the reference's dense Conv2D layer (SURVEY.md
// §8f.4: pruning with retraining), on the GPU and bit-identical to
// /root/reference/pkg/src/unsparse/kernels.py:103-162 (called by nn.Conv2D.backward,
// nn.py:62-72).
//
//   k_grad_weights: dw[d,c,kh,kw] = sum over b, r, cc of the fp32 product
//     dout[b,d,r,cc] * xpad[b,c,r*s_h+kh,cc*s_w+kw], accumulated in DOUBLE in that
//     order (the reference's accumulator `s = 0.0` is a numba float64) and stored as
//     fp32.  One thread per weight; a warp's lanes are consecutive (c, kh, kw) of one
//     d, so every dout load is a broadcast.
//   k_grad_input: the reference scatters dxpad[b,c,r*s_h+kh,cc*s_w+kw] +=
//     dout[b,d,r,cc] * w[d,c,kh,kw] (fp32 multiply, fp32 add) in loop order b, d, r,
//     c, kh, kw, cc -- so one element receives its terms in (d, r ascending, kw
//     ascending) order (Yw == 1: loops b, d, c, kh, kw, r -> (d, kh ascending)).  The
//     GPU gathers: one thread per dxpad element sums exactly those terms in exactly
//     that order, starting from the zero the reference initialises (nn.py:67), so no
//     atomics and the same bits.  A warp's lanes are consecutive x of one row: dout
//     loads coalesce along cc.
#include "common.cuh"

namespace {

__global__ void k_grad_weights(const float *__restrict__ xpad, const float *__restrict__ dout,
                               float *__restrict__ dw, int n, int C, int Hp, int Wp, int D, int Kh, int Kw,
                               int Yh, int Yw, int s_h, int s_w) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long total = (long long)D * C * Kh * Kw;
    if (i >= total) return;
    const int kw = static_cast<int>(i % Kw), kh = static_cast<int>((i / Kw) % Kh);
    const int c = static_cast<int>((i / ((long long)Kw * Kh)) % C), d = static_cast<int>(i / ((long long)Kw * Kh * C));
    double s = 0.0;
    for (int b = 0; b < n; ++b) {
        const float *xb = xpad + ((long long)b * C + c) * Hp * Wp + kh * (long long)Wp + kw;
        const float *gb = dout + ((long long)b * D + d) * Yh * Yw;
        for (int r = 0; r < Yh; ++r) {
            const float *row = xb + (long long)r * s_h * Wp;
            const float *go = gb + (long long)r * Yw;
            for (int cc = 0; cc < Yw; ++cc) s = __dadd_rn(s, static_cast<double>(__fmul_rn(__ldg(go + cc), __ldg(row + cc * s_w))));
        }
    }
    dw[i] = static_cast<float>(s);  // round to nearest, as numba's float64 -> float32 store
}

__global__ void k_grad_input(const float *__restrict__ w, const float *__restrict__ dout, float *__restrict__ dxpad,
                             int n, int C, int Hp, int Wp, int D, int Kh, int Kw, int Yh, int Yw, int s_h, int s_w) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long total = (long long)n * C * Hp * Wp;
    if (i >= total) return;
    const int x = static_cast<int>(i % Wp), y = static_cast<int>((i / Wp) % Hp);
    const int c = static_cast<int>((i / ((long long)Wp * Hp)) % C), b = static_cast<int>(i / ((long long)Wp * Hp * C));
    float acc = 0.0f;
    if (Yw == 1) {  // kernels.py:143-153: only column kw == x receives terms
        if (x < Kw) {
            for (int d = 0; d < D; ++d) {
                const float *wd = w + (((long long)d * C + c) * Kh) * Kw + x;
                const float *gd = dout + ((long long)b * D + d) * Yh;
                for (int kh = 0; kh < Kh; ++kh) {
                    const int t = y - kh;
                    if (t < 0 || t % s_h) continue;
                    const int r = t / s_h;
                    if (r >= Yh) continue;
                    acc = __fadd_rn(acc, __fmul_rn(__ldg(gd + r), __ldg(wd + kh * Kw)));
                }
            }
        }
    } else {  // kernels.py:154-162
        const int r_lo = y - Kh + 1 > 0 ? (y - Kh + 1 + s_h - 1) / s_h : 0;
        const int r_hi = min(y / s_h, Yh - 1);
        for (int d = 0; d < D; ++d) {
            const float *wd = w + ((long long)d * C + c) * Kh * Kw;
            const float *gd = dout + ((long long)b * D + d) * Yh * Yw;
            for (int r = r_lo; r <= r_hi; ++r) {
                const int kh = y - r * s_h;
                const float *go = gd + (long long)r * Yw;
                for (int kw = 0; kw < Kw; ++kw) {
                    const int t = x - kw;
                    if (t < 0 || t % s_w) continue;
                    const int cc = t / s_w;
                    if (cc >= Yw) continue;
                    acc = __fadd_rn(acc, __fmul_rn(__ldg(go + cc), __ldg(wd + kh * Kw + kw)));
                }
            }
        }
    }
    dxpad[i] = acc;
}

int grad_dims(const usc_geometry *g, int *Hp, int *Wp, int *Yh, int *Yw) {
    int rc = usc_geometry_check(g);
    if (rc) return rc;
    *Hp = g->input_h + 2 * g->pad_h;
    *Wp = g->input_w + 2 * g->pad_w;
    return usc_geometry_out(g, Yh, Yw);
}

}  // namespace

extern "C" {

int usc_conv_grad_weights(const usc_geometry *g, int32_t n, const float *xpad, const float *dout, float *dw,
                          void *stream) {
    int Hp, Wp, Yh, Yw;
    int rc = grad_dims(g, &Hp, &Wp, &Yh, &Yw);
    if (rc) return rc;
    if (n < 1) return usc::fail(USC_ERR_VALUE, "batch must be >= 1");
    const long long total = (long long)g->out_channels * g->in_channels * g->filter_h * g->filter_w;
    const int threads = 128;
    k_grad_weights<<<static_cast<unsigned>((total + threads - 1) / threads), threads, 0,
                     static_cast<cudaStream_t>(stream)>>>(xpad, dout, dw, n, g->in_channels, Hp, Wp, g->out_channels,
                                                          g->filter_h, g->filter_w, Yh, Yw, g->stride_h, g->stride_w);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return usc::fail(USC_ERR_CUDA, "k_grad_weights: %s", cudaGetErrorString(e));
    return USC_OK;
}

int usc_conv_grad_input(const usc_geometry *g, int32_t n, const float *w, const float *dout, float *dxpad,
                        void *stream) {
    int Hp, Wp, Yh, Yw;
    int rc = grad_dims(g, &Hp, &Wp, &Yh, &Yw);
    if (rc) return rc;
    if (n < 1) return usc::fail(USC_ERR_VALUE, "batch must be >= 1");
    const long long total = (long long)n * g->in_channels * Hp * Wp;
    const int threads = 256;
    k_grad_input<<<static_cast<unsigned>((total + threads - 1) / threads), threads, 0,
                   static_cast<cudaStream_t>(stream)>>>(w, dout, dxpad, n, g->in_channels, Hp, Wp, g->out_channels,
                                                        g->filter_h, g->filter_w, Yh, Yw, g->stride_h, g->stride_w);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return usc::fail(USC_ERR_CUDA, "k_grad_input: %s", cudaGetErrorString(e));
    return USC_OK;
}

}  // extern "C"
