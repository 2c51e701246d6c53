/*
 * unsparse_b200.h -- C ABI of the B200-native direct sparse convolution engine.
 *
 * This is the drop-in boundary for the reference `unsparse` conv-layer path
 * (/root/reference/pkg/src/unsparse).  Plain pointers and sizes only; no torch
 * or CUDA C++ types.  Device pointers are CUDA device addresses; `stream` is a
 * cudaStream_t passed as void*.  All device work is stream-ordered and
 * asynchronous; no entry point allocates device memory or synchronises.
 *
 * Each entry point names the reference interface it replaces (file:line,
 * relative to /root/reference/pkg/src/unsparse/).
 *
 * Error convention: every function returns USC_OK (0) or a status code;
 * usc_last_error() returns a thread-local message for the last failure.
 * USC_ERR_VALUE maps to Python ValueError, USC_ERR_CORRUPT to
 * CsrCorruptionError(ValueError) (csr.py:21), USC_ERR_CUDA to RuntimeError.
 */
#ifndef UNSPARSE_B200_H
#define UNSPARSE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define USC_ABI_VERSION 1

enum usc_status {
    USC_OK = 0,
    USC_ERR_VALUE = 1,       /* geometry / precision / divisibility / shape (ValueError) */
    USC_ERR_CORRUPT = 2,     /* CSR offset does not decode to a filter tap (CsrCorruptionError) */
    USC_ERR_CUDA = 3,        /* CUDA runtime error (launch, copy) */
    USC_ERR_UNSUPPORTED = 4  /* configuration this build cannot run */
};

/* Operand kinds of the conv kernels. */
enum usc_dtype {
    USC_F32 = 0,  /* binary32 in/out, bitwise = reference BINARY32 (mul then add, stored order) */
    USC_F16 = 1,  /* binary16 storage, fp32 accumulate, saturating RNE output (engine.py:109-110) */
    USC_I8 = 2,   /* int8 fixed-point codes, int32 accumulate, fp32 out = acc*sigma_w*sigma_x */
    USC_CB4 = 3   /* 4-bit codebook index -> fp32 centroid, binary16 input, binary16 output */
};

/* ConvGeometry (tensor.py:156-222).  Output dims must divide exactly
 * (tensor.py:182-190); usc_geometry_check enforces it. */
typedef struct usc_geometry {
    int32_t in_channels, out_channels;
    int32_t filter_h, filter_w;
    int32_t input_h, input_w;
    int32_t stride_h, stride_w;
    int32_t pad_h, pad_w;
} usc_geometry;

/* Resident activation layouts -- the reference's materialised zero_pad layout
 * (tensor.py:225-235) made bulk-copy-legal:
 *  interleave == 0  "padded NCHW": [n][C][Hp][Ws], zero halo (pad_h, pad_w), row
 *                   stride Ws rounded up to a multiple of 16 bytes;
 *                   element (b,c,y,x) at ((b*C + c)*Hp + y+pad_h)*Ws + x+pad_w.
 *  interleave == IL "batch-interleaved" (BI32 / BI64, IL = 32 or 64):
 *                   [ceil(n/IL)][C][Hp][Wp][IL], zero halo, IL samples innermost so
 *                   a warp reads one (BI32) or two (BI64, two samples per lane)
 *                   128-byte lines per pixel; element (b,c,y,x) at
 *                   (((b/IL*C + c)*Hp + y+pad_h)*Wp + x+pad_w)*IL + b%IL.
 * sample_stride is the stride of one sample (il 0) or one IL-sample block. */
typedef struct usc_act_layout {
    int32_t channels, height, width;   /* logical (unpadded) plane */
    int32_t pad_h, pad_w;              /* halo */
    int32_t hp, ws;                    /* padded height, padded (+aligned for il 0) row stride */
    int32_t interleave;                /* 0, 32 or 64 */
    int64_t sample_stride;             /* elements per sample (il 0) / per 32-sample block (il 32) */
} usc_act_layout;

/* Execution / tile configuration.  sub_batch and worker_count keep the meaning of
 * ExecConfig (engine.py:25-41); the remaining fields are the B200 tile knobs the
 * autotuner searches (0 = choose automatically). */
typedef struct usc_exec_cfg {
    int32_t sub_batch;        /* samples per virtual block; must divide n (engine.py:81-82) */
    int32_t worker_count;     /* accepted for API parity; the GPU ignores it */
    int32_t pix_per_thread;   /* P: consecutive output pixels per thread (1,2,4,8) */
    int32_t ch_per_cta;       /* DT: output channels per CTA (4,8,16,32) */
    int32_t samples_per_cta;  /* NS: samples per CTA (kernel 1: full-map tiles; kernel 3: the
                               * interleave, 32 = BI32 or 64 = BI64) */
    int32_t chunk_channels;   /* CC: input channels per shared-memory stage */
    int32_t threads;          /* kernel 1: threads per CTA (128/256); kernel 3: compute threads
                               * (256/384/512 = 8/12/16 compute warps, + 1 producer warp) */
    int32_t kernel;           /* 0 auto, 1 tiled (padded NCHW), 2 generic, 3 batch-interleaved */
    int32_t pixel_warps;      /* kernel 3: warps over output strips (must divide the warps; the
                               * rest split the CTA's ch_per_cta output channels) */
    int32_t stages;           /* kernel 3: shared-memory ring depth (2..4) */
    int32_t rows_per_thread;  /* kernel 3: output rows per thread (1 or 2); pixels = rows x pix_per_thread */
    int32_t ent_reserve;      /* kernel 3: shared-memory bytes reserved per stage for CSR entries (0 auto) */
    int32_t pixel_classes;    /* kernel 3, 1x1 pixel blocks: 1 = per-pixel-class entry runs that drop
                               * the taps landing on the zero halo (exact for finite weights) */
    int32_t window;           /* kernel 3: 1 = register-window variant (k_bw): one output row of
                               * pix_per_thread pixels per thread, the warp's ch_per_cta/warps slots
                               * share one entry stream ordered by input row, each x window loaded
                               * into registers once per (c, kh); stride 1, F32/F16, filter_w 1 or 3 */
} usc_exec_cfg;

/* Resolved plan for one (geometry, batch, dtype, cfg): tile shape, packing
 * parameters and launch dimensions.  Produced by usc_plan, consumed by usc_pack
 * and usc_conv_forward. */
typedef struct usc_plan {
    usc_geometry g;
    int32_t dtype;
    int32_t n;
    int32_t out_h, out_w;
    usc_act_layout in;           /* input layout the kernel reads */
    int32_t kernel;              /* 1 tiled, 2 generic, 3 batch-interleaved */
    int32_t P, DT, NS, CC, threads;
    int32_t TH, HS;              /* output rows per CTA tile, staged rows per channel */
    int32_t strips_per_row, row_tiles, sample_tiles, groups, n_chunks;
    int32_t WS, WC, DW;          /* BI kernel: warps over strips, warps over channels, channels/warp */
    int32_t SPRt, col_tiles, TWs;/* BI kernel: strips per tile row, column tiles, staged row width */
    int32_t ent_stage_bytes;     /* BI kernel: shared-memory reserve for one chunk's entries */
    int32_t stages;              /* BI kernel: shared-memory ring depth */
    int32_t PR, PC;              /* BI kernel: a thread's pixel block = PR rows x PC columns (P = PR*PC) */
    int32_t transposed;          /* 1D layer (W==1) run as its H/W transpose */
    int32_t ncls_r, ncls_c;      /* BI kernel: pixel classes (rows x columns with the same valid taps);
                                  * 1 x 1 = no classes */
    int32_t tail_full, tail_split;  /* BI kernel: tiles [0, tail_full) run whole, each later tile as
                                     * tail_split slot-subset items (balances the last wave) */
    int32_t window;              /* BI kernel: register-window variant (usc_exec_cfg.window) */
    int64_t smem_stage_bytes, smem_bytes;
    int64_t grid_x, grid_y;
} usc_plan;

/* Epilogue of one conv launch (fused): ReLU (nn.py:96-98), saturation cap
 * (quantization.py:79-93 with the _half_hook order, 238-244), output layout. */
typedef struct usc_epilogue {
    int32_t relu;                /* 1: where(v > 0, v, 0) */
    int32_t saturate;            /* 1: v = min(v, cap) before the binary16 rounding */
    float cap;                   /* float32(threshold * calibrated_max) */
    int32_t saturate2;           /* 1: after ReLU, v = min(v, cap2) then binary16 rounding again */
    float cap2;                  /* (the _half_hook of the ReLU layer in a 4b/16b model) */
    float scale;                 /* USC_I8: sigma_w * sigma_x (exact power of two) */
    int32_t out_padded;          /* 0: plain NCHW output; 1: padded layout `out` */
    usc_act_layout out;          /* used when out_padded */
    int32_t pool;                /* 1: fused 2x2/2 max-pool after ReLU (nn.py:124-135); `out` is the
                                  * pooled layout; needs a BI plan with PR == 2 and even PC */
    int32_t requant;             /* USC_I8, BI kernel: 1 = requantise the ReLU output to the next
                                  * layer's fixed-point codes (linear_quantize, quantization.py:61-76):
                                  * clip(copysign(floor(|v*rq_scale| + 0.5)), +-rq_limit), written as
                                  * binary16 codes (the BI kernel's int8 staging) */
    float rq_scale;              /* 1/sigma of the next layer's input (a power of two) */
    int32_t rq_limit;            /* 2^(bits-1) - 1 */
    int32_t residual;            /* BI kernel, F32/F16: 1 = add the shortcut tensor `res` (same logical
                                  * shape as the output, layout `res_layout`) before the ReLU:
                                  * F32 v = acc + r; F16 v = round16(round16(acc) + r) */
    usc_act_layout res_layout;
    uint64_t res;                /* device address of the shortcut tensor */
} usc_epilogue;

/* ---- library ---------------------------------------------------------- */
int usc_abi_version(void);
const char *usc_last_error(void);
/* Device properties the planner uses (SM count etc.); -1 when no device. */
int usc_device_sm_count(int device);

/* ---- geometry (tensor.py:174-210) ------------------------------------ */
int usc_geometry_check(const usc_geometry *g);
int usc_geometry_out(const usc_geometry *g, int32_t *out_h, int32_t *out_w);
/* Padded activation layout for `channels x h x w` planes with halo (ph, pw) and
 * element size `elem_bytes` (4 f32, 2 f16, 1 i8). */
int usc_act_layout_make(int32_t channels, int32_t h, int32_t w, int32_t ph, int32_t pw,
                        int32_t elem_bytes, int32_t interleave, usc_act_layout *out);
/* Elements a buffer of `n` samples in `layout` needs. */
int64_t usc_act_layout_elems(const usc_act_layout *layout, int32_t n);

/* ---- encoder (host) -- replaces csr.py:86-112 build_csr ----------------
 * Pass 1: n_nz = max(1, max_d count_nonzero(w[d])) (csr.py:103).
 * Pass 2: RP/Lambda/theta bit-identical to the reference: padding entries
 * (offset 0, weight 0) first, genuine entries in ascending offset order. */
int usc_csr_count(const float *w, const usc_geometry *g, int64_t *n_nz);
int usc_build_csr(const float *w, const usc_geometry *g, int64_t n_nz, int64_t *row_ptr,
                  int64_t *col_offsets, float *theta);
/* Device-side encoder (csr.py:86-112 on the GPU, bit-identical to usc_build_csr), for
 * pruning loops that re-encode every iteration.  w: device f32 D x C x Kh x Kw.
 * Pass 1 writes the per-channel genuine-nonzero counts (int32[D]) and their maximum
 * (int32[1]); the caller reads n_nz = max(1, max) to size col/theta (D*n_nz), then
 * pass 2 writes row_ptr (int64[D+1]), col_offsets (int64) and theta (f32) on the device. */
int usc_csr_count_device(const float *w_dev, const usc_geometry *g, int32_t *counts_dev, int32_t *max_count_dev,
                         void *stream);
int usc_build_csr_device(const float *w_dev, const usc_geometry *g, const int32_t *counts_dev,
                         const int32_t *max_count_dev, int64_t *row_ptr_dev, int64_t *col_offsets_dev,
                         float *theta_dev, void *stream);
/* CsrFilter.validate (csr.py:66-83).  On USC_ERR_CORRUPT, *bad_index receives
 * the first entry whose offset does not decode to a tap (or -1 for a
 * row_ptr / length violation). */
int usc_csr_validate(const usc_geometry *g, const int64_t *row_ptr, int64_t row_ptr_len,
                     const int64_t *col_offsets, int64_t n_col, int64_t n_theta, int64_t n_nz,
                     int64_t *bad_index);
/* csr_to_dense (csr.py:115-128). */
int usc_csr_to_dense(const usc_geometry *g, const int64_t *row_ptr, const int64_t *col_offsets,
                     const float *theta, int64_t n_nz, float *w_out);

/* ---- planner / packer (host) -------------------------------------------
 * usc_plan resolves tile/launch parameters (the B200 analogue of plan_blocks,
 * engine.py:53-61).  usc_pack writes the kernel-private entry stream for one
 * plan into a HOST buffer of plan->pack_bytes bytes, which the caller copies to
 * the device.  Zero-weight entries are deduplicated per (channel, offset):
 * for finite inputs they are no-ops, and one copy per distinct offset keeps the
 * reference's NaN propagation exact.
 * host_blob == NULL is a dry run: *n_entries receives the largest (group, chunk)
 * entry block in bytes (kernel 3 plans; pass it back as usc_exec_cfg.ent_reserve).
 * payload: USC_F32/USC_F16 -> the CSR theta (fp32, binary16 values for F16);
 *          USC_I8 -> int8 codes (one per CSR entry, theta = code*sigma_w);
 *          USC_CB4 -> uint8 centroid indices (one per CSR entry) + 16-entry
 *                     fp32 centroid table `table`. */
int usc_plan_make(const usc_geometry *g, int32_t n, int32_t dtype, const usc_exec_cfg *cfg,
                  usc_plan *out);
/* The batch-interleaved kernel's compiled tile instances: writes up to max_count
 * records of 6 int32 (compute warps, PC, PR, DW, stride_w, samples per lane) and
 * returns the total count.  The autotuner's kernel-3 search space (threads =
 * warps*32, samples_per_cta = 32*samples per lane). */
int usc_bi_instances(int32_t *out, int32_t max_count);
/* The register-window variant's compiled tiles (usc_exec_cfg.window = 1): up to
 * max_count records of 5 int32 (family 0 fp32 / 1 binary16, compute warps, PC, DW,
 * filter width); returns the total count. */
int usc_bw_instances(int32_t *out, int32_t max_count);
int usc_pack_size(const usc_plan *plan, int64_t n_nz, int64_t *bytes);
/* autotune_sb (engine.py:139-170) behind the C ABI: plans, packs and times every
 * tile candidate of the layer (the batch-interleaved kernel's compiled instances x
 * warp splits x ring depths x pixel classes, and kernel 1's sub-batch x pixels x
 * channels -- engine.tile_candidates) on `x_dev` (plain NCHW, n x C x H x W in the
 * dtype's storage: f32, binary16, int8 codes, binary16) with CUDA events on
 * `stream` (median of `repeats` after `warmup` launches) and writes the fastest
 * config to *best (candidates within noise_floor of it resolve to the earliest, in
 * ascending sub-batch order, as the reference's rule).  Allocates and frees its
 * own scratch buffers; synchronises `stream`.  row_ptr/col_offsets/payload/table
 * as usc_pack.  *best_ms (may be NULL) receives the winner's median time. */
int usc_autotune(const usc_geometry *g, int32_t n, int32_t dtype, const int64_t *row_ptr,
                 const int64_t *col_offsets, const void *payload, int64_t n_nz, const float *table,
                 const void *x_dev, int32_t repeats, int32_t warmup, float noise_floor, usc_exec_cfg *best,
                 float *best_ms, void *stream);
int usc_pack(const usc_plan *plan, const int64_t *row_ptr, const int64_t *col_offsets,
             const void *payload, int64_t n_nz, const float *table, void *host_blob,
             int64_t blob_bytes, int64_t *n_entries);

/* ---- device kernels ------------------------------------------------------
 * usc_pad_input: plain NCHW (n x C x H x W, dtype elements) -> `layout`
 * (zero_pad, tensor.py:225-235; halo and padding samples written as zeros).
 * `dst` must hold usc_act_layout_elems(layout, n) elements. */
int usc_pad_input(const usc_act_layout *layout, int32_t dtype, int32_t n, const void *src,
                  void *dst, void *stream);
/* Inverse: `layout` -> plain NCHW (extract_interior, tensor.py:238-244). */
int usc_unpad_output(const usc_act_layout *layout, int32_t dtype, int32_t n, const void *src,
                     void *dst, void *stream);
/* Direct sparse convolution -- replaces engine.py:64-111 sparse_conv_forward with
 * kernels.py:57-100 as its hot loop.  x_dev is in plan->in layout, blob_dev is
 * the device copy of usc_pack's output, y_dev receives n x D x Yh x Yw (plain)
 * or the epilogue's padded layout. */
int usc_conv_forward(const usc_plan *plan, const void *blob_dev, const void *x_dev, void *y_dev,
                     const usc_epilogue *epi, void *stream);
/* usc_conv_forward on a window of a larger resident buffer: the plan's (hp x ws) input
 * is read from x_dev with the strides of `x_layout` (same channels and interleave, at
 * least as large).  Exact-geometry views of ResNet's stride-2 layers (ConvGeometry
 * rejects 32 -> 16 with pad 1, tensor.py:186-190): a 3x3 stride-2 conv reads the
 * top/left 33x33 of the 34x34 halo buffer with pad 0; a 1x1 stride-2 projection reads
 * the 31x31 interior window (x_dev advanced to element (1,1)).  BI plans only. */
int usc_conv_forward_view(const usc_plan *plan, const void *blob_dev, const void *x_dev,
                          const usc_act_layout *x_layout, void *y_dev, const usc_epilogue *epi, void *stream);
/* A 1x1 stride-s convolution (ResNet's stride-2 projections) run as a stride-1,
 * unpadded 1x1 plan over every (step_h, step_w)-th pixel of the buffer `x_layout`
 * describes: the TMA map strides over the skipped pixels, so only the pixels the
 * convolution uses are read.  Same result as the stride-s plan (a 1x1 conv is
 * pointwise); the filter must be encoded for the plan's stride-1 geometry. */
int usc_conv_forward_strided(const usc_plan *plan, const void *blob_dev, const void *x_dev,
                             const usc_act_layout *x_layout, int32_t step_h, int32_t step_w, void *y_dev,
                             const usc_epilogue *epi, void *stream);
/* Reference-shaped kernel entry, the exact analogue of the numba FFI
 * kernels.sparse_conv_blocks(xflat, row_ptr, col_offsets, theta, out, blocks, sb,
 * x_size, s_h, s_w, padded_w) (kernels.py:57-58), all arrays on the device:
 * xflat f32[n*x_size] (materialised padded input), row_ptr i64[D+1],
 * col_offsets i64, theta f32, out f32[n][D][Yh][Yw], blocks i64[nb][2]. */
int usc_sparse_conv_blocks(const float *xflat, const int64_t *row_ptr, const int64_t *col_offsets,
                           const float *theta, float *out, const int64_t *blocks, int64_t n_blocks,
                           int32_t sb, int64_t x_size, int32_t s_h, int32_t s_w, int32_t padded_w,
                           int32_t D, int32_t out_h, int32_t out_w, void *stream);
/* Layout transposes for the per-layer sparse/dense backend dispatcher (bench.py:212-227,
 * pipeline.py:381-389): a layer run on cuDNN reads the network's resident BI64 binary16
 * layout `l` as NHWC [n][H][W][C] (usc_bi_to_nhwc) and its NHWC binary16 output is
 * written back into `l`'s interior (usc_nhwc_to_bi) with the epilogue fused:
 * v = sat16(y); with a shortcut (`res` in `res_layout`, same logical shape)
 * v = sat16(v + r) (binary16 add); ReLU where(v > 0, v, 0) when relu != 0.
 * BI64 layouts with channels % 16 == 0 only. */
int usc_bi_to_nhwc(const usc_act_layout *l, int32_t n, const void *src, void *dst, void *stream);
int usc_nhwc_to_bi(const usc_act_layout *l, int32_t n, const void *src, void *dst, const usc_act_layout *res_layout,
                   const void *res, int32_t relu, void *stream);
/* The same epilogue in place on `count` binary16 values of any layout (a cuDNN layer's
 * NHWC output inside a dense chain): v = sat16(y); res: v = sat16(v + r); ReLU when relu. */
int usc_f16_epilogue(void *y, const void *res, int64_t count, int32_t relu, void *stream);
/* The dense backend on the 5th-generation tensor cores (binary16 networks, fp16 tolerance
 * path): an implicit-GEMM convolution (tcgen05.mma, fp32 accumulation in tensor memory,
 * TMA-staged 128-byte-swizzled operands) reading the BI64 binary16 input `x` in
 * `x_layout` and writing the BI64 output `y` in `y_layout` (interior only) with the
 * epilogue fused: round to binary16 with saturation, + shortcut `res` (binary16, sat16),
 * ReLU when relu != 0.  torch conv2d semantics: padding = filter/2 (read from the input
 * halo, which must be at least that wide), stride g->stride_h (= stride_w, 1 or 2),
 * filters 1x1 or 3x3; in_channels % 64 == 0, out_channels % 64 == 0.  `w_dev`: the dense
 * weights as [out_channels][filter_h*filter_w][in_channels] binary16 (K-major), padded with
 * zero rows to a multiple of 128 output channels.  First-layer form: in_channels <= 16,
 * 3x3 stride 1, out_channels == 64, no shortcut, `w_dev` = [9][16][64] binary16 (input
 * channels zero-padded to 16, output channel fastest). */
int usc_dense_conv_f16(const usc_geometry *g, int32_t n, const void *w_dev, const usc_act_layout *x_layout,
                       const void *x, const usc_act_layout *y_layout, void *y, const usc_act_layout *res_layout,
                       const void *res, int32_t relu, void *stream);
/* The same with a tile configuration and a device workspace for split-K: `twp` output
 * pixels per tile (2 or 4; 0 = automatic), `splits` K splits (>= 1; 0 = automatic: split
 * only small maps whose tiles fill at most half the SMs; never with a shortcut).  The CTA
 * completing a tile's last K split sums the splits' fp32 partials in split order and runs
 * the epilogue.  `workspace` must hold usc_dense_conv_f16_ws_bytes() bytes for the same
 * (twp, splits) and be zero-filled once before its first use (the kernel leaves its
 * counters at zero); a null or short workspace runs without split. */
int usc_dense_conv_f16_ws(const usc_geometry *g, int32_t n, const void *w_dev, const usc_act_layout *x_layout,
                          const void *x, const usc_act_layout *y_layout, void *y, const usc_act_layout *res_layout,
                          const void *res, int32_t relu, void *workspace, int64_t ws_bytes, int32_t twp,
                          int32_t splits, void *stream);
/* The 3x3 stride-1 conv + ReLU + 2x2 max-pool (nn.py:124-135 on the ReLU output, which has
 * no NaN) in one launch: `y_layout` is the pooled output (height/2 x width/2).  Returns
 * USC_ERR_UNSUPPORTED when usc_dense_conv_f16_pool_ok() is 0 for the shape (then run the
 * conv and usc_maxpool2). */
int usc_dense_conv_f16_pool(const usc_geometry *g, int32_t n, const void *w_dev, const usc_act_layout *x_layout,
                            const void *x, const usc_act_layout *y_layout, void *y, void *stream);
/* 1 when the fused pool runs this shape at least as fast as conv + pool would (even output
 * dims, width % 4 == 0, enough row pairs to fill the SMs), else 0. */
int32_t usc_dense_conv_f16_pool_ok(const usc_geometry *g, int32_t n, const usc_act_layout *x_layout);
/* Workspace bytes usc_dense_conv_f16_ws needs for this shape and configuration on the current
 * device (0: no split). */
int64_t usc_dense_conv_f16_ws_bytes(const usc_geometry *g, int32_t n, const usc_act_layout *x_layout,
                                    int32_t has_res, int32_t twp, int32_t splits);
/* round_to_binary16 (tensor.py:48-63) on device: f32 in -> f32 on the binary16 grid
 * (to_half == 0) or binary16 storage (to_half == 1). */
int usc_round_binary16(const float *src, void *dst, int64_t count, int32_t to_half, void *stream);
/* Elementwise conversions between storage kinds (f32 <-> binary16). */
int usc_convert(const void *src, int32_t src_dtype, void *dst, int32_t dst_dtype, int64_t count,
                void *stream);
/* 2x2 stride-2 max pooling (nn.py:109-135): NaN-first argmax semantics.
 * Input in `in_l` (padded or plain when in_l->pad_* == 0 and ws == width),
 * output written to `out_l` layout. dtype USC_F32 or USC_F16. */
int usc_maxpool2(const usc_act_layout *in_l, const usc_act_layout *out_l, int32_t dtype,
                 int32_t n, const void *src, void *dst, void *stream);
/* Quantise a device f32 tensor to int8 fixed-point codes (quantization.py:61-76):
 * code = clip(copysign(floor(|x/sigma| + 0.5)), -(2^(bits-1)-1), 2^(bits-1)-1). */
int usc_quantize_i8(const float *src, int8_t *dst, int64_t count, double sigma, int32_t bits,
                    void *stream);

/* ---- diagnostics ----------------------------------------------------------
 * Live CUDA-core peak of the exact fp32 path's instruction mix (IEEE multiply
 * then add, never contracted) on `device`, in TFLOP/s (2 flops per pair); the
 * roofline denominator bench.py reports the sparse conv kernel against. */
int usc_peak_fp32_muladd(int32_t device, double *tflops);
/* Same probe for a chosen mix, in nonzero TFLOP/s (2 flops per MAC):
 *   0 = FMUL + FADD (one sample per lane, kernels 1/2 and BI32),
 *   1 = FMUL, FMUL + one packed FADD2 per two samples (the fp32 BI64 inner loop),
 *   2 = FHFMA (fma.rn.f32.f16, the binary16 BI64 inner loop). */
int usc_peak_mix(int32_t device, int32_t mix, double *tflops);

/* ---- quantisation primitives (host) -- quantization.py ------------------ */
/* fit_fixed_point (quantization.py:41-58): from max|x| */
int usc_fit_fixed_point(double amax, int32_t total_bits, int32_t *int_bits, int32_t *frac_bits,
                        double *sigma);
/* linear_quantize codes (quantization.py:61-76), fp64 arithmetic. */
int usc_linear_codes(const double *x, int64_t count, double sigma, int32_t total_bits,
                     double *codes);
/* kmeans_codebook (quantization.py:112-180): zero-pinned 1-D Lloyd with
 * deterministic quantile seeding; bit-identical to the numpy reference.
 * centroids/quantized have room for omega values; *k_out receives the codebook
 * size; assignments has `count` entries. */
int usc_kmeans_codebook(const double *w, int64_t count, int32_t omega, int32_t psi,
                        double *centroids, double *quantized, int64_t *assignments,
                        int32_t *k_out, int32_t *zero_pinned);

/* Training kernels of the dense Conv2D layer (nn.py:62-72), bit-identical to the
 * reference (pruning with retraining).  All fp32, device pointers:
 *   usc_conv_grad_weights -- kernels.conv_grad_weights (kernels.py:103-130):
 *     xpad [n][C][Hp][Wp] (the zero-padded forward input), dout [n][D][Yh][Yw] ->
 *     dw [D][C][Kh][Kw] (overwritten); fp64 accumulation in (b, r, cc) order.
 *   usc_conv_grad_input -- kernels.conv_grad_input (kernels.py:133-162) into a zeroed
 *     dxpad (nn.py:67): w [D][C][Kh][Kw], dout -> dxpad [n][C][Hp][Wp] (overwritten,
 *     every element; crop the halo for dx, nn.py:69-71). */
int usc_conv_grad_weights(const usc_geometry *g, int32_t n, const float *xpad_dev, const float *dout_dev,
                          float *dw_dev, void *stream);
int usc_conv_grad_input(const usc_geometry *g, int32_t n, const float *w_dev, const float *dout_dev,
                        float *dxpad_dev, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* UNSPARSE_B200_H */
