// Timeline of one k_dtc launch per CTA (%globaltimer, ns from the first CTA's entry):
// entry, setup done (barriers + TMEM), first stage landed, last MMA of tile 0/1 issued,
// tile 0/1 accumulator ready at the epilogue, epilogue drained.  Built against a
// DTC_TRACE compile of dense_tc.cu (tools/gpu_r02s.sh), never the product library.
//   tools/dtc_trace C D K stride HW
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../include/unsparse_b200.h"

extern "C" int usc_dtc_trace_read(unsigned long long *out, int ctas);

int main(int argc, char **argv) {
    const int C = argc > 1 ? atoi(argv[1]) : 256, D = argc > 2 ? atoi(argv[2]) : 256, K = argc > 3 ? atoi(argv[3]) : 3,
              s = argc > 4 ? atoi(argv[4]) : 1, hw = argc > 5 ? atoi(argv[5]) : 8, n = 256;
    usc_geometry g = {C, D, K, K, hw, hw, s, s, K / 2, K / 2};
    usc_act_layout xl, yl;
    usc_act_layout_make(C, hw, hw, K / 2, K / 2, 2, 64, &xl);
    const int ho = (hw + 2 * (K / 2) - K) / s + 1;
    usc_act_layout_make(D, ho, ho, 1, 1, 2, 64, &yl);
    void *x, *y, *w;
    const size_t xe = (size_t)(n / 64) * xl.sample_stride, ye = (size_t)(n / 64) * yl.sample_stride;
    cudaMalloc(&x, xe * 2);
    cudaMalloc(&y, ye * 2);
    const int Dp = (D + 127) / 128 * 128;
    const size_t wbytes = std::max((size_t)Dp * K * K * C * 2, (size_t)9 * 16 * 64 * 2);  // (first-layer packing)
    cudaMalloc(&w, wbytes);
    cudaMemset(x, 0, xe * 2);
    cudaMemset(w, 0, wbytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int r = 0; r < 5; ++r) usc_dense_conv_f16(&g, n, w, &xl, x, &yl, y, nullptr, nullptr, 1, nullptr);
    cudaEventRecord(a);
    int rc = usc_dense_conv_f16(&g, n, w, &xl, x, &yl, y, nullptr, nullptr, 1, nullptr);
    cudaEventRecord(b);
    cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<unsigned long long> t(148 * 8);
    usc_dtc_trace_read(t.data(), 148);
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < 148; ++c) t0 = std::min(t0, t[c * 8]);
    printf("C %d D %d K %d s %d hw %d rc %d event_us %.1f\n", C, D, K, s, hw, rc, ms * 1e3);
    printf("cta   entry  setup  land0  mma0  mma1  acc0  acc1  drained (us from first entry; k_dtc: tiles 0/1, k_dts: tiles 0/6)\n");
    double sum[8] = {0};
    int cnt[8] = {0};
    for (int c = 0; c < 148; ++c) {
        if (c < 6 || c > 141) printf("%3d", c);
        for (int k = 0; k < 8; ++k) {
            const unsigned long long v = t[c * 8 + k];
            const double us = v >= t0 && v - t0 < 100000000ull ? (v - t0) * 1e-3 : -1;
            if (us >= 0) sum[k] += us, cnt[k]++;
            if (c < 6 || c > 141) printf(" %6.2f", us);
        }
        if (c < 6 || c > 141) printf("\n");
    }
    printf("avg");
    for (int k = 0; k < 8; ++k) printf(" %6.2f", cnt[k] ? sum[k] / cnt[k] : -1.0);
    printf("\nmax drained %.2f\n", [&] {
        double m = 0;
        for (int c = 0; c < 148; ++c) m = std::max(m, (t[c * 8 + 7] - t0) * 1e-3);
        return m;
    }());
    return 0;
}
