// host.cpp -- host side of the C ABI: geometry, activation layouts, the CSR
// encoder (bit-exact build_csr), validation, the tile planner and the packer
// that turns a CsrFilter into the kernel-private entry stream, and the
// quantisation primitives (fixed point, codebook k-means).
//
// References are to /root/reference/pkg/src/unsparse/<file>:<line>.
#include "usc_internal.h"
#include "bi_instances.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <unordered_set>
#include <vector>

namespace usc {

thread_local std::string g_last_error;

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

int elem_bytes(int dtype) {
    switch (dtype) {
        case USC_F32: return 4;
        case USC_F16: return 2;
        case USC_I8: return 1;
        case USC_CB4: return 2;  // binary16 activations
    }
    return 0;
}

int entry_bytes(int dtype) { return (dtype == USC_F32 || dtype == USC_F16) ? 8 : 4; }

}  // namespace usc

using namespace usc;

extern "C" {

int usc_abi_version(void) { return USC_ABI_VERSION; }

const char *usc_last_error(void) { return g_last_error.c_str(); }

// tensor.py:174-190 -- stride >= 1, pad >= 0, filter fits, exact division.
int usc_geometry_check(const usc_geometry *g) {
    if (!g) return fail(USC_ERR_VALUE, "null geometry");
    if (g->stride_h < 1) return fail(USC_ERR_VALUE, "stride_h must be >= 1, got %d", g->stride_h);
    if (g->stride_w < 1) return fail(USC_ERR_VALUE, "stride_w must be >= 1, got %d", g->stride_w);
    if (g->pad_h < 0 || g->pad_w < 0) return fail(USC_ERR_VALUE, "padding must be non-negative");
    if (g->in_channels < 1 || g->out_channels < 1 || g->filter_h < 1 || g->filter_w < 1 ||
        g->input_h < 1 || g->input_w < 1)
        return fail(USC_ERR_VALUE, "geometry dims must be positive");
    int num_h = g->input_h + 2 * g->pad_h - g->filter_h;
    int num_w = g->input_w + 2 * g->pad_w - g->filter_w;
    if (num_h < 0 || num_w < 0) return fail(USC_ERR_VALUE, "filter larger than padded input");
    if (num_h % g->stride_h || num_w % g->stride_w)
        return fail(USC_ERR_VALUE, "output dims not integral for geometry: (%d %% %d, %d %% %d)",
                    num_h, g->stride_h, num_w, g->stride_w);
    return USC_OK;
}

int usc_geometry_out(const usc_geometry *g, int32_t *out_h, int32_t *out_w) {
    int rc = usc_geometry_check(g);
    if (rc) return rc;
    *out_h = (g->input_h + 2 * g->pad_h - g->filter_h) / g->stride_h + 1;
    *out_w = (g->input_w + 2 * g->pad_w - g->filter_w) / g->stride_w + 1;
    return USC_OK;
}

int usc_act_layout_make(int32_t channels, int32_t h, int32_t w, int32_t ph, int32_t pw,
                        int32_t eb, int32_t il, usc_act_layout *out) {
    if (channels < 1 || h < 1 || w < 1 || ph < 0 || pw < 0 || (eb != 1 && eb != 2 && eb != 4) ||
        (il != 0 && il != 32 && il != 64))
        return fail(USC_ERR_VALUE, "bad activation layout");
    out->channels = channels;
    out->height = h;
    out->width = w;
    out->pad_h = ph;
    out->pad_w = pw;
    out->hp = h + 2 * ph;
    out->interleave = il;
    if (il == 0) {
        int per16 = 16 / eb;
        out->ws = (w + 2 * pw + per16 - 1) / per16 * per16;
        out->sample_stride = (int64_t)channels * out->hp * out->ws;
    } else {
        out->ws = w + 2 * pw;  // a pixel is il*eb >= 32 bytes: always 16-B aligned
        out->sample_stride = (int64_t)channels * out->hp * out->ws * il;
    }
    return USC_OK;
}

int64_t usc_act_layout_elems(const usc_act_layout *l, int32_t n) {
    if (l->interleave) return (int64_t)((n + l->interleave - 1) / l->interleave) * l->sample_stride;
    return (int64_t)n * l->sample_stride;
}

// ---------------------------------------------------------------------------
// encoder

// csr.py:97-103
int usc_csr_count(const float *w, const usc_geometry *g, int64_t *n_nz) {
    int rc = usc_geometry_check(g);
    if (rc) return rc;
    int64_t per = (int64_t)g->in_channels * g->filter_h * g->filter_w, best = 0;
    for (int64_t d = 0; d < g->out_channels; ++d) {
        int64_t cnt = 0;
        const float *wd = w + d * per;
        for (int64_t k = 0; k < per; ++k) cnt += (wd[k] != 0.0f);
        best = std::max(best, cnt);
    }
    *n_nz = std::max<int64_t>(1, best);
    return USC_OK;
}

// csr.py:94-112.  np.nonzero walks (c, kh, kw) in C order, which is already
// ascending in offset = (c*Hp + kh)*Wp + kw, so the stable argsort is the
// identity; padding (offset 0, weight 0) goes first in each slice.
int usc_build_csr(const float *w, const usc_geometry *g, int64_t n_nz, int64_t *row_ptr,
                  int64_t *col, float *theta) {
    int rc = usc_geometry_check(g);
    if (rc) return rc;
    const int64_t C = g->in_channels, D = g->out_channels, Kh = g->filter_h, Kw = g->filter_w;
    const int64_t Hp = g->input_h + 2 * g->pad_h, Wp = g->input_w + 2 * g->pad_w;
    const int64_t per = C * Kh * Kw;
    for (int64_t d = 0; d <= D; ++d) row_ptr[d] = d * n_nz;
    for (int64_t d = 0; d < D; ++d) {
        const float *wd = w + d * per;
        int64_t cnt = 0;
        for (int64_t k = 0; k < per; ++k) cnt += (wd[k] != 0.0f);
        if (cnt > n_nz) return fail(USC_ERR_VALUE, "n_nz %lld smaller than channel count %lld",
                                    (long long)n_nz, (long long)cnt);
        int64_t pos = d * n_nz;
        for (int64_t i = 0; i < n_nz - cnt; ++i, ++pos) {
            col[pos] = 0;
            theta[pos] = 0.0f;
        }
        for (int64_t c = 0; c < C; ++c)
            for (int64_t kh = 0; kh < Kh; ++kh)
                for (int64_t kw = 0; kw < Kw; ++kw) {
                    float v = wd[(c * Kh + kh) * Kw + kw];
                    if (v != 0.0f) {
                        col[pos] = (c * Hp + kh) * Wp + kw;
                        theta[pos] = v;
                        ++pos;
                    }
                }
    }
    return USC_OK;
}

// csr.py:66-83 (with offset_to_tap, csr.py:30-42)
int usc_csr_validate(const usc_geometry *g, const int64_t *row_ptr, int64_t rp_len,
                     const int64_t *col, int64_t n_col, int64_t n_theta, int64_t n_nz,
                     int64_t *bad) {
    *bad = -1;
    int rc = usc_geometry_check(g);
    if (rc) return rc;
    const int64_t D = g->out_channels;
    if (rp_len != D + 1 || row_ptr[0] != 0)
        return fail(USC_ERR_CORRUPT, "row_ptr must have length D+1 and start at 0");
    for (int64_t d = 0; d < D; ++d)
        if (row_ptr[d + 1] - row_ptr[d] != n_nz)
            return fail(USC_ERR_CORRUPT, "row_ptr slices are not uniform");
    if (n_col != D * n_nz || n_theta != D * n_nz)
        return fail(USC_ERR_CORRUPT, "col_offsets/weights length must be D*n_nz");
    const int64_t Hp = g->input_h + 2 * g->pad_h, Wp = g->input_w + 2 * g->pad_w;
    const int64_t plane = Hp * Wp, x_size = (int64_t)g->in_channels * plane;
    for (int64_t i = 0; i < n_col; ++i) {
        int64_t lam = col[i];
        if (lam < 0 || lam >= x_size) {
            *bad = i;
            return fail(USC_ERR_CORRUPT, "offset %lld outside padded sample", (long long)lam);
        }
        int64_t c = lam / plane, rem = lam % plane, kh = rem / Wp, kw = rem % Wp;
        if (kh >= g->filter_h || kw >= g->filter_w) {
            *bad = i;
            return fail(USC_ERR_CORRUPT, "offset %lld decodes to (%lld,%lld,%lld), not a %dx%d tap",
                        (long long)lam, (long long)c, (long long)kh, (long long)kw, g->filter_h,
                        g->filter_w);
        }
    }
    return USC_OK;
}

// csr.py:115-128
int usc_csr_to_dense(const usc_geometry *g, const int64_t *row_ptr, const int64_t *col,
                     const float *theta, int64_t n_nz, float *w_out) {
    int rc = usc_geometry_check(g);
    if (rc) return rc;
    const int64_t C = g->in_channels, D = g->out_channels, Kh = g->filter_h, Kw = g->filter_w;
    const int64_t Hp = g->input_h + 2 * g->pad_h, Wp = g->input_w + 2 * g->pad_w;
    const int64_t plane = Hp * Wp;
    std::memset(w_out, 0, sizeof(float) * D * C * Kh * Kw);
    for (int64_t d = 0; d < D; ++d)
        for (int64_t i = row_ptr[d]; i < row_ptr[d + 1]; ++i) {
            float v = theta[i];
            if (v == 0.0f) continue;
            int64_t lam = col[i], c = lam / plane, rem = lam % plane;
            int64_t kh = rem / Wp, kw = rem % Wp;
            if (lam < 0 || c >= C || kh >= Kh || kw >= Kw)
                return fail(USC_ERR_CORRUPT, "offset %lld does not decode to a tap", (long long)lam);
            w_out[((d * C + c) * Kh + kh) * Kw + kw] = v;
        }
    (void)n_nz;
    return USC_OK;
}

// ---------------------------------------------------------------------------
// planner (the GPU analogue of plan_blocks, engine.py:53-61)

static int pow2_floor(int v) {
    int p = 1;
    while (p * 2 <= v) p *= 2;
    return p;
}

// Pixel classes of one output axis: output index y reads padded input indices
// y*stride + k (k < K); bit k of its mask is set when that index is inside the
// image (not the zero halo).  Indices with equal masks form one class.
static void tap_classes(int Y, int stride, int pad, int K, int X, std::vector<int> &cls,
                        std::vector<uint32_t> &masks) {
    cls.assign(Y, 0);
    masks.clear();
    for (int y = 0; y < Y; ++y) {
        uint32_t m = 0;
        for (int k = 0; k < K && k < 32; ++k) {
            const int i = y * stride + k - pad;
            if (i >= 0 && i < X) m |= 1u << k;
        }
        size_t id = std::find(masks.begin(), masks.end(), m) - masks.begin();
        if (id == masks.size()) masks.push_back(m);
        cls[y] = (int)id;
    }
}

// The k_bi instances compiled into the library (bi_instances.h).
static bool bi_instance(int PC, int PR, int DW, int NW, int SW, int SPL, int dtype) {
    if (dtype == USC_F16 || dtype == USC_CB4 || dtype == USC_I8) {
        if (SPL != 2) return false;
#define XH(NW_, PC_, PR_, DW_, SW_) \
    if (NW == NW_ && PC == PC_ && PR == PR_ && DW == DW_ && SW == SW_) return true;
        USC_BI_H(XH)
#undef XH
        return false;
    }
    if (dtype != USC_F32) return false;
#define X(PC_, PR_, DW_, SW_, SPL_) \
    if (PC == PC_ && PR == PR_ && DW == DW_ && SW == SW_ && SPL == SPL_) return true;
    if (NW == 8) {
        USC_BI_W8(X)
    } else if (NW == 12) {
        USC_BI_W12(X)
    } else if (NW == 16) {
        USC_BI_W16(X)
    }
#undef X
    return false;
}

// the k_bw (register-window) instances compiled into the library (bi_instances.h)
static bool bw_instance(int PC, int DW, int NW, int KW, int dtype) {
    const int fam = dtype == USC_F32 ? 0 : (dtype == USC_F16 ? 1 : -1);
#define XW(F_, NW_, PC_, DW_, KW_) \
    if (fam == F_ && NW == NW_ && PC == PC_ && DW == DW_ && KW == KW_) return true;
    USC_BW(XW)
#undef XW
    return false;
}

int usc_bw_instances(int32_t *out, int32_t max_count) {
    int n = 0;
#define XW(F_, NW_, PC_, DW_, KW_)        \
    if (n < max_count && out) {           \
        int32_t *o = out + 5 * n;         \
        o[0] = F_;                        \
        o[1] = NW_;                       \
        o[2] = PC_;                       \
        o[3] = DW_;                       \
        o[4] = KW_;                       \
    }                                     \
    ++n;
    USC_BW(XW)
#undef XW
    return n;
}

static bool bt_instance(int PC, int PR, int DW, int NW) {
#define XT(NW_, PC_, PR_, DW_) \
    if (NW == NW_ && PC == PC_ && PR == PR_ && DW == DW_) return true;
    USC_BT(XT)
#undef XT
    return false;
}

int usc_bi_instances(int32_t *out, int32_t max_count) {
    int n = 0;
#define X7(NW_, PC_, PR_, DW_, SW_, SPL_, K_)                   \
    if (n < max_count && out) {                                \
        int32_t *o = out + 7 * n;                              \
        o[0] = NW_;                                            \
        o[1] = PC_;                                            \
        o[2] = PR_;                                            \
        o[3] = DW_;                                            \
        o[4] = SW_;                                            \
        o[5] = SPL_;                                           \
        o[6] = K_;                                             \
    }                                                          \
    ++n;
#define X(PC_, PR_, DW_, SW_, SPL_) X7(NW_, PC_, PR_, DW_, SW_, SPL_, 0)
#define XH(NWH_, PC_, PR_, DW_, SW_) X7(NWH_, PC_, PR_, DW_, SW_, 2, 1)
    {
        const int NW_ = 8;
        USC_BI_W8(X)
    }
    {
        const int NW_ = 12;
        USC_BI_W12(X)
    }
    {
        const int NW_ = 16;
        USC_BI_W16(X)
    }
    USC_BI_H(XH)
#define XT(NWT_, PC_, PR_, DW_) X7(NWT_, PC_, PR_, DW_, 1, 2, 2)
    USC_BT(XT)
#undef XT
#undef X
#undef XH
#undef X7
    return n;
}

int usc_plan_make(const usc_geometry *g0, int32_t n, int32_t dtype, const usc_exec_cfg *cfg,
                  usc_plan *pl) {
    int rc = usc_geometry_check(g0);
    if (rc) return rc;
    if (n < 1) return fail(USC_ERR_VALUE, "batch must be >= 1");
    if (dtype < USC_F32 || dtype > USC_CB4) return fail(USC_ERR_VALUE, "unknown dtype %d", dtype);
    usc_exec_cfg c = cfg ? *cfg : usc_exec_cfg{};
    if (c.sub_batch < 1) c.sub_batch = 1;
    if (n % c.sub_batch)
        return fail(USC_ERR_VALUE, "sub_batch %d does not divide batch %d", c.sub_batch, n);
    if (c.kernel == 0) {
        // auto: the batch-interleaved kernel when a compiled tile fits this layer, else
        // the padded-NCHW kernel
        usc_exec_cfg k3 = c;
        k3.kernel = 3;
        if (usc_plan_make(g0, n, dtype, &k3, pl) == USC_OK) return USC_OK;
        c.kernel = 1;
    }
    std::memset(pl, 0, sizeof *pl);
    pl->dtype = dtype;
    pl->n = n;
    usc_geometry g = *g0;
    // A 1-D layer along H (input_w == filter_w == 1) is the same memory as its
    // H/W transpose; run it along W so pixels of a thread are contiguous.
    if (g.input_w == 1 && g.filter_w == 1 && g.pad_w == 0 && g.input_h > 1) {
        std::swap(g.filter_h, g.filter_w);
        std::swap(g.input_h, g.input_w);
        std::swap(g.stride_h, g.stride_w);
        std::swap(g.pad_h, g.pad_w);
        pl->transposed = 1;
    }
    pl->g = g;
    usc_geometry_out(&g, &pl->out_h, &pl->out_w);
    // staged element size: the BI kernel holds int8 codes as binary16 (exact, |code| <= 127)
    int kernel = c.kernel ? c.kernel : 3;
    if (g.stride_w > 2) kernel = 2;
    if (kernel == 4 && (dtype != USC_F32 || g.stride_w != 1 || g.stride_h != 1))
        return fail(USC_ERR_UNSUPPORTED, "the tensor-memory kernel is fp32, stride 1 only");
    const bool bi = kernel == 3 || kernel == 4;  // batch-interleaved families
    const bool win = bi && c.window != 0;        // register-window variant (k_bw)
    if (win && (kernel != 3 || (dtype != USC_F32 && dtype != USC_F16) || g.stride_w != 1 ||
                (g.filter_w != 1 && g.filter_w != 3)))
        return fail(USC_ERR_UNSUPPORTED, "the register-window kernel is F32/F16, stride_w 1, filter_w 1 or 3");
    const int eb = (kernel == 3 && dtype == USC_I8) ? 2 : elem_bytes(dtype);

    // kernel 3 sample interleave: samples_per_cta 32 (BI32) or 64 (BI64, two samples per
    // lane); default BI64 once the batch fills two 32-sample blocks
    int IL = 0;
    if (bi) {
        IL = (c.samples_per_cta == 32 || c.samples_per_cta == 64) ? c.samples_per_cta : (n > 32 ? 64 : 32);
        if (dtype != USC_F32 || kernel == 4 || win) IL = 64;  // binary16-staged kinds, TMEM, k_bw: BI64 only
    }
    rc = usc_act_layout_make(g.in_channels, g.input_h, g.input_w, g.pad_h, g.pad_w, eb, IL, &pl->in);
    if (rc) return rc;
    const int Yh = pl->out_h, Yw = pl->out_w, Ws = pl->in.ws;
    const int threads = (c.threads == 128 || c.threads == 256) ? c.threads : 256;
    if (bi) {
        // batch-interleaved: a CTA = 32 samples x (WS strips of PR x PC pixels) x (WC*DW
        // channels), NW compute warps (threads = NW*32) + 1 producer warp; warp w owns
        // strip w % WS for channel subgroup w / WS; lane = sample.
        const bool even = Yh % 2 == 0 && Yw % 2 == 0 && g.stride_w == 1;
        int PR = c.rows_per_thread ? c.rows_per_thread : (even && Yh >= 2 ? 2 : 1);
        if (PR != 1 && PR != 2) return fail(USC_ERR_VALUE, "BI rows_per_thread must be 1 or 2");
        if (PR > Yh || win) PR = 1;
        int PC = c.pix_per_thread;
        if (win && !PC) PC = 4;
        if (!PC) {  // widest block that divides the row, else 4 with a partial last strip
            PC = Yw >= 4 ? 4 : (Yw >= 2 ? 2 : 1);
            for (int q : {8, 4, 2})
                if (Yw % q == 0 && q * PR <= 8) {
                    PC = q;
                    break;
                }
        }
        if (!win && (!c.pix_per_thread || !c.rows_per_thread)) {
            // no compiled instance for the preferred block: the first (PR, PC) that has one
            auto any_inst = [&](int pr, int pc) {
                for (int nw : {8, 12, 16})
                    for (int dw : {2, 4, 8, 16})
                        if (kernel == 4 ? bt_instance(pc, pr, dw, nw)
                                        : bi_instance(pc, pr, dw, nw, g.stride_w, IL / 32, dtype))
                            return true;
                return false;
            };
            if (!any_inst(PR, PC)) {
                bool found = false;
                for (int pr : {PR, 1})
                    for (int pc : {8, 4, 2, 1}) {
                        if (found || (c.rows_per_thread && pr != c.rows_per_thread) ||
                            (c.pix_per_thread && pc != c.pix_per_thread) || pr > Yh)
                            continue;
                        if (any_inst(pr, pc)) {
                            PR = pr;
                            PC = pc;
                            found = true;
                        }
                    }
            }
        }
        if (PC != 1 && PC != 2 && PC != 4 && PC != 8)
            return fail(USC_ERR_VALUE, "BI pix_per_thread must be 1,2,4,8");
        const int P = PR * PC;
        const int SPR = (Yw + PC - 1) / PC;  // strips per strip-row
        const int SR = (Yh + PR - 1) / PR;   // strip-rows
        // warps: the requested count, else the first of 8/12/16 with a compiled
        // instance for this pixel block (channels per warp 8, 16 or 4 unless given)
        int NW = 0, WS = 0, WC = 0, DW = 0;
        for (int nw : {8, 12, 16}) {
            if (c.threads && c.threads != nw * 32) continue;
            // pixel warps: as given, else the largest divisor of the warps (<= warps/4)
            // whose strips tile the map's strip grid
            auto tileable = [&](int w) {
                for (int t = 1; t <= w; ++t)
                    if (w % t == 0 && t <= SR && w / t <= SPR) return true;
                return false;
            };
            int ws = c.pixel_warps;
            if (ws && (ws > nw || nw % ws))
                return fail(USC_ERR_VALUE, "pixel_warps %d must divide %d warps", ws, nw);
            if (!ws)
                for (ws = std::max(1, nw / 4); ws > 1; --ws)
                    if (nw % ws == 0 && tileable(ws)) break;
            const int wc = nw / ws;
            if (c.ch_per_cta && c.ch_per_cta % wc)
                return fail(USC_ERR_VALUE, "ch_per_cta %d not a multiple of %d channel warps", c.ch_per_cta, wc);
            for (int dw : {8, 16, 4, 2, 12}) {
                if (c.ch_per_cta) dw = c.ch_per_cta / wc;
                const bool inst = win ? bw_instance(PC, dw, nw, g.filter_w, dtype)
                                      : (kernel == 4 ? bt_instance(PC, PR, dw, nw)
                                                     : bi_instance(PC, PR, dw, nw, g.stride_w, IL / 32, dtype));
                if (inst) {
                    NW = nw, WS = ws, WC = wc, DW = dw;
                    break;
                }
                if (c.ch_per_cta) break;
            }
            if (NW) break;
        }
        if (!NW)
            return fail(USC_ERR_VALUE, "no BI kernel instance for PC=%d PR=%d threads=%d ch_per_cta=%d stride=%d",
                        PC, PR, c.threads, c.ch_per_cta, g.stride_w);
        // tile = TSR strip-rows x SPRt strips (TSR*SPRt == WS): fewest tiles (strip work),
        // then the smallest staged footprint
        int TSR = 1, SPRt = WS;
        int64_t best_tiles = INT64_MAX, best_foot = INT64_MAX;
        for (int tsr = 1; tsr <= WS; ++tsr) {
            if (WS % tsr) continue;
            const int sprt = WS / tsr;
            // strips of a tile stay inside the map (a full-row stage is exactly Yw wide)
            if (sprt > SPR || (tsr > SR && tsr > 1)) continue;
            const int64_t tiles = (int64_t)((SR + tsr - 1) / tsr) * ((SPR + sprt - 1) / sprt);
            const int ct = (SPR + sprt - 1) / sprt;
            const int tws = (ct == 1 && SPR * PC == Yw && pl->in.ws <= 256) ? pl->in.ws
                                                                             : (sprt * PC - 1) * g.stride_w + g.filter_w;
            if (tws > 256 || (int64_t)(tsr * PR - 1) * g.stride_h + g.filter_h > 256) continue;  // TMA box
            const int64_t foot = tiles * ((int64_t)(tsr * PR - 1) * g.stride_h + g.filter_h) * tws;
            if (tiles < best_tiles || (tiles == best_tiles && foot < best_foot)) {
                best_tiles = tiles;
                best_foot = foot;
                TSR = tsr;
                SPRt = sprt;
            }
        }
        if (best_tiles == INT64_MAX)
            return fail(USC_ERR_VALUE, "%d pixel warps do not tile a %dx%d strip grid", WS, SR, SPR);
        const int TH = TSR * PR;  // output rows per tile
        const int col_tiles = (SPR + SPRt - 1) / SPRt;
        const bool full_rows = (col_tiles == 1 && SPR * PC == Yw && pl->in.ws <= 256);
        const int TWs = full_rows ? pl->in.ws : (SPRt * PC - 1) * g.stride_w + g.filter_w;
        const int HS = (TH - 1) * g.stride_h + g.filter_h;
        const int64_t per_ch = (int64_t)HS * TWs * IL * eb;  // one channel of the TMA box
        const int DT = WC * DW;
        // per-pixel-class runs (1x1 pixel blocks): one entry run per (class, slot) without
        // the taps that land on the zero halo
        int ncr = 1, ncc = 1;
        // (row classes need 1-row blocks, column classes 1-column blocks: every pixel of a
        // thread's block must share the valid-tap set along a classed axis)
        if (c.pixel_classes && !win && (PC == 1 || PR == 1) && g.filter_h <= 32 && g.filter_w <= 32) {
            std::vector<int> cl;
            std::vector<uint32_t> mk;
            if (PR == 1) {
                tap_classes(Yh, g.stride_h, g.pad_h, g.filter_h, g.input_h, cl, mk);
                ncr = (int)mk.size();
            }
            if (PC == 1) {
                tap_classes(Yw, g.stride_w, g.pad_w, g.filter_w, g.input_w, cl, mk);
                ncc = (int)mk.size();
            }
        }
        const int NCLS = ncr * ncc;
        int CC = c.chunk_channels ? c.chunk_channels : 64;
        CC = std::min(std::min(CC, g.in_channels), 256);
        if (kernel == 4) {  // a chunk's positions fill one 256-column TMEM buffer (2 columns each)
            if (HS * TWs > 128) return fail(USC_ERR_VALUE, "tile of %d positions exceeds tensor memory", HS * TWs);
            CC = std::min(CC, 128 / (HS * TWs));
        }
        const int S = c.stages ? std::max(2, std::min(4, c.stages)) : 2;
        const int64_t budget = 200 * 1024;
        // per-stage entry block: hdr DT*8 + runs padded to even (16-B aligned starts) +
        // 16 B read slack.  The exact worst case is DT*CC*Kh*Kw entries; reserve at most
        // R bytes -- usc_pack rejects a filter whose densest (group, chunk) block
        // exceeds it (the caller re-plans with the measured size).
        const int64_t R = c.ent_reserve ? c.ent_reserve : 24 * 1024;
        auto ent_bytes = [&](int cc) {
            // k_bw: hdr int2[WC], per channel subgroup its MAC entries + one ROW entry per (c, kh)
            // + an even-count pad
            const int64_t worst =
                win ? (int64_t)WC * 8 + 16 + ((int64_t)DT * cc * g.filter_h * g.filter_w +
                                             (int64_t)WC * (cc * g.filter_h + 2)) * 8 + 16
                    : (int64_t)NCLS * DT * 8 + 8 + NCLS * ((int64_t)DT * cc * g.filter_h * g.filter_w + DT) * 8 + 16;
            return (std::min(worst, R) + 127) / 128 * 128;
        };
        while (CC > 1 && S * ((CC * per_ch + 127) / 128 * 128 + ent_bytes(CC)) > budget) --CC;
        const int64_t stage = (CC * per_ch + 127) / 128 * 128;
        const int64_t ent_stage = ent_bytes(CC);
        if (S * (stage + ent_stage) + 128 > 224 * 1024)
            return fail(USC_ERR_VALUE, "BI tile does not fit shared memory");
        pl->kernel = kernel;
        pl->window = win ? 1 : 0;
        pl->ncls_r = ncr;
        pl->ncls_c = ncc;
        pl->P = P;
        pl->PR = PR;
        pl->PC = PC;
        pl->WS = WS;
        pl->WC = WC;
        pl->DW = DW;
        pl->DT = DT;
        pl->NS = IL;
        pl->CC = CC;
        pl->TH = TH;
        pl->HS = HS;
        pl->SPRt = SPRt;
        pl->col_tiles = col_tiles;
        pl->TWs = TWs;
        pl->threads = NW * 32;
        pl->strips_per_row = SPR;
        pl->row_tiles = (Yh + TH - 1) / TH;
        pl->sample_tiles = (n + IL - 1) / IL;
        pl->groups = (g.out_channels + DT - 1) / DT;
        pl->n_chunks = (g.in_channels + CC - 1) / CC;
        pl->smem_stage_bytes = stage;
        pl->ent_stage_bytes = static_cast<int32_t>(ent_stage);
        pl->stages = S;
        pl->smem_bytes = S * (stage + ent_stage) + 128;
        // persistent grid: one CTA per SM, each walks its tiles
        const int64_t tiles = (int64_t)pl->groups * pl->sample_tiles * pl->row_tiles * pl->col_tiles;
        int sms = usc_device_sm_count(0);
        if (sms <= 0) sms = 148;
        pl->grid_x = std::min<int64_t>(tiles, sms);
        pl->grid_y = 1;
        // last-wave balance: split the last R tiles into F interleaved slot subsets
        // (F | DW) when that shortens the round-robin makespan (whole tile = 1 unit)
        pl->tail_full = (int32_t)tiles;
        pl->tail_split = 1;
        if (!win) {  // (k_bw runs whole tiles: its merged run covers every slot of the warp)
            const int64_t C = sms;
            auto makespan = [&](int64_t R, int F) {
                const int64_t full = tiles - R, nsplit = F * R;
                double worst = 0;
                for (int64_t c = 0; c < C; ++c) {
                    const int64_t nf = full / C + (c < full % C);
                    const int64_t cs = ((c - full) % C + C) % C;
                    const int64_t ns = nsplit / C + (cs < nsplit % C);
                    worst = std::max(worst, nf + ns / (double)F);
                }
                return worst;
            };
            double best = makespan(0, 1);
            for (int F : {2, 4}) {
                if (DW % F) continue;
                for (int64_t R = 1; R <= std::min<int64_t>(tiles, C); ++R) {
                    const double m = makespan(R, F);
                    if (m < best - 1e-9) {
                        best = m;
                        pl->tail_full = (int32_t)(tiles - R);
                        pl->tail_split = F;
                    }
                }
            }
            const int64_t items = pl->tail_full + (int64_t)pl->tail_split * (tiles - pl->tail_full);
            pl->grid_x = std::min<int64_t>(items, sms);
        }
        return USC_OK;
    }
    if (kernel == 1) {
        int P = c.pix_per_thread ? c.pix_per_thread : std::min(4, pow2_floor(Yw));
        if (P != 1 && P != 2 && P != 4 && P != 8) return fail(USC_ERR_VALUE, "pix_per_thread must be 1,2,4,8");
        int SPR = (Yw + P - 1) / P;
        while (SPR > threads && P < 8) {
            P *= 2;
            SPR = (Yw + P - 1) / P;
        }
        if (SPR > threads) kernel = 2;
        if (kernel == 1) {
            int DT = c.ch_per_cta ? c.ch_per_cta : 16;
            if (DT != 8 && DT != 16) return fail(USC_ERR_VALUE, "ch_per_cta must be 8 or 16");
            int per_sample = Yh * SPR;
            int NS, TH;
            if (per_sample <= threads) {
                TH = Yh;
                int maxNS = threads / per_sample;
                NS = c.samples_per_cta ? std::min(c.samples_per_cta, maxNS) : maxNS;
                NS = std::max(1, std::min(NS, n));
            } else {
                NS = 1;
                TH = threads / SPR;
            }
            int HS = (TH - 1) * g.stride_h + g.filter_h;
            if (TH == Yh) HS = pl->in.hp;
            // stage = NS samples x CC channels x HS rows x Ws, plus read slack for
            // partial strips (row wrap of the last row)
            const int64_t per_ch = (int64_t)HS * Ws * eb;
            const int64_t slack = 64 * eb;
            const int64_t budget = c.chunk_channels ? INT64_MAX : 48 * 1024;  // per stage
            int CC = c.chunk_channels ? c.chunk_channels : 32;
            CC = std::min(CC, g.in_channels);
            while (CC > 1 && NS * CC * per_ch + slack > budget) --CC;
            int64_t stage = ((int64_t)NS * CC * per_ch + slack + 127) / 128 * 128;
            if (2 * stage + 256 > 220 * 1024) kernel = 2;
            if (kernel == 1) {
                pl->P = P;
                pl->DT = DT;
                pl->NS = NS;
                pl->CC = CC;
                pl->TH = TH;
                pl->HS = HS;
                pl->threads = threads;
                pl->strips_per_row = SPR;
                pl->row_tiles = (Yh + TH - 1) / TH;
                pl->sample_tiles = (n + NS - 1) / NS;
                pl->groups = (g.out_channels + DT - 1) / DT;
                pl->n_chunks = (g.in_channels + CC - 1) / CC;
                pl->smem_stage_bytes = stage;
                pl->smem_bytes = 2 * stage + 128;
                pl->grid_x = (int64_t)pl->sample_tiles * pl->row_tiles;
                pl->grid_y = pl->groups;
            }
        }
    }
    pl->kernel = kernel;
    if (kernel == 2) {
        pl->P = 1;
        pl->DT = 1;
        pl->NS = 1;
        pl->CC = g.in_channels;
        pl->TH = Yh;
        pl->HS = pl->in.hp;
        pl->threads = 256;
        pl->groups = g.out_channels;
        pl->n_chunks = 1;
        int64_t total = (int64_t)n * g.out_channels * Yh * Yw;
        pl->grid_x = std::min<int64_t>((total + 255) / 256, 148 * 64);
        pl->grid_y = 1;
    }
    return USC_OK;
}

// ---------------------------------------------------------------------------
// packer: CsrFilter -> kernel-private entry stream
//
// blob = 16-float centroid table (CB4; zeros otherwise), int32 cpg[G][n_chunks*DT + 1]
// (padded to 16 B), entries (int2 for F32/F16 = {offset, theta bits}; int32 for
// I8 = code<<24 | offset and for CB4 = index<<28 | offset).
// Entries are laid out (group, chunk, d_local, stored order) so one chunk of one
// group is contiguous and its DT+1 boundaries are consecutive in cpg.

static int64_t align16(int64_t v) { return (v + 15) / 16 * 16; }

// binary16 bits of an fp32 value (round to nearest even; exact for the binary16-grid
// weights of a BINARY16 filter)
static uint16_t f32_to_f16_bits(float f) {
    uint32_t x;
    std::memcpy(&x, &f, 4);
    const uint32_t sign = (x >> 16) & 0x8000u;
    const uint32_t ax = x & 0x7fffffffu;
    if (ax >= 0x7f800000u) return (uint16_t)(sign | 0x7c00u | (ax > 0x7f800000u ? 0x200u : 0u));  // inf/nan
    if (ax >= 0x477ff000u) return (uint16_t)(sign | 0x7c00u);  // rounds past 65504 -> inf
    if (ax < 0x33000001u) return (uint16_t)sign;               // < half the smallest subnormal
    const int e = (int)(ax >> 23);
    uint32_t m = (ax & 0x7fffffu) | 0x800000u;
    int shift = 126 - e;  // normal half exponent field = e - 112; subnormal below
    uint32_t hb;
    if (e >= 113) {  // normal
        hb = ((uint32_t)(e - 112) << 10) | ((m >> 13) & 0x3ffu);
        const uint32_t rem = m & 0x1fffu;
        if (rem > 0x1000u || (rem == 0x1000u && (hb & 1u))) ++hb;
    } else {         // subnormal: value = m * 2^(e-150), unit 2^-24
        shift = 126 - e;  // 14 + (113 - e)
        const uint32_t q = m >> shift, rem = m & ((1u << shift) - 1u), half = 1u << (shift - 1);
        hb = q;
        if (rem > half || (rem == half && (hb & 1u))) ++hb;
    }
    return (uint16_t)(sign | hb);
}

// the 32-bit theta word of stored entry j in a kernel-3 entry: fp32 bits (F32), the
// binary16 bits in the low half (F16; I8 codes, exact), the decoded fp32 centroid (CB4)
static int32_t theta_word(int dtype, const void *payload, const float *table, int64_t j) {
    int32_t w = 0;
    if (dtype == USC_F16) return (int32_t)f32_to_f16_bits(((const float *)payload)[j]);
    if (dtype == USC_I8) return (int32_t)f32_to_f16_bits((float)((const int8_t *)payload)[j]);
    if (dtype == USC_CB4) {
        std::memcpy(&w, &table[((const uint8_t *)payload)[j] & 15], 4);
        return w;
    }
    std::memcpy(&w, &((const float *)payload)[j], 4);
    return w;
}

int usc_pack_size(const usc_plan *pl, int64_t n_nz, int64_t *bytes) {
    const int64_t nb = (int64_t)pl->groups * pl->n_chunks;
    if (pl->kernel == 3 || pl->kernel == 4) {
        // [64 B][int32 blk[nb+1]][int32 perm[G*DT]][blocks: hdr int2[DT], runs padded to
        // even, 16-B rounded]
        const int64_t ncls = std::max(1, pl->ncls_r * pl->ncls_c);
        if (pl->window) {  // k_bw: per (block, channel subgroup) up to CC*Kh ROW entries + END
            *bytes = 64 + align16(4 * (nb + 1)) + align16(4 * (int64_t)pl->groups * pl->DT) +
                     align16(4 * ((int64_t)pl->out_h + pl->out_w)) + nb * ((int64_t)pl->WC * 8 + 32) +
                     ((int64_t)pl->g.out_channels * n_nz + nb * pl->WC * ((int64_t)pl->CC * pl->g.filter_h + 1)) * 8 +
                     64;
            return USC_OK;
        }
        *bytes = 64 + align16(4 * (nb + 1)) + align16(4 * (int64_t)pl->groups * pl->DT) +
                 align16(4 * ((int64_t)pl->out_h + pl->out_w)) + nb * (ncls * pl->DT * 8 + 16) +
                 ncls * ((int64_t)pl->g.out_channels * n_nz + nb * pl->DT) * 8 + 64;
        return USC_OK;
    }
    int64_t cp = align16(4 * (nb * pl->DT + 1));
    int64_t ent = align16((int64_t)pl->g.out_channels * n_nz * entry_bytes(pl->dtype)) + 64;
    *bytes = 64 + cp + ent;  // [16-float centroid table][cpg][entries]
    return USC_OK;
}

int usc_pack(const usc_plan *pl, const int64_t *row_ptr, const int64_t *col, const void *payload,
             int64_t n_nz, const float *table, void *blob, int64_t blob_bytes, int64_t *n_entries) {
    int64_t need;
    usc_pack_size(pl, n_nz, &need);
    const bool dry = blob == nullptr;  // dry run: *n_entries <- largest (group, chunk) block in bytes
    std::vector<char> scratch;
    if (dry) {
        scratch.resize(need);
        blob = scratch.data();
        blob_bytes = need;
    }
    if (blob_bytes < need) return fail(USC_ERR_VALUE, "pack buffer too small");
    const usc_geometry &g = pl->g;
    const int D = g.out_channels, DT = pl->DT, G = pl->groups, NC = pl->n_chunks, CC = pl->CC;
    // decode offsets against the ORIGINAL (untransposed) geometry
    int Hp0, Wp0, Kh0, Kw0;
    if (pl->transposed) {
        Hp0 = g.input_w + 2 * g.pad_w;  // original H
        Wp0 = 1;
        Kh0 = g.filter_w;
        Kw0 = 1;
    } else {
        Hp0 = g.input_h + 2 * g.pad_h;
        Wp0 = g.input_w + 2 * g.pad_w;
        Kh0 = g.filter_h;
        Kw0 = g.filter_w;
    }
    const int64_t plane0 = (int64_t)Hp0 * Wp0;
    const int Ws = pl->in.ws, Hp = pl->in.hp;
    const int64_t cs_tiled = (int64_t)pl->HS * Ws;  // channel stride inside a stage
    std::memset(blob, 0, 64);
    if (pl->dtype == USC_CB4) std::memcpy(blob, table, 16 * sizeof(float));
    // one stored entry j of channel d -> (input channel, offset in the kernel's staged
    // tile), or off = -1 to drop it (a repeated zero-weight offset)
    const int64_t max_off = pl->dtype == USC_I8 ? (1 << 24) : (1 << 28);
    std::unordered_set<int64_t> zero_seen;  // distinct zero-weight offsets of the channel
    int64_t dec_kh = 0, dec_kw = 0;  // tap of the last decoded entry (plan orientation)
    auto decode = [&](int64_t j, int64_t *cpos, int64_t *off) -> int {
        const int64_t lam = col[j];
        int64_t c = lam / plane0, rem = lam % plane0, kh = rem / Wp0, kw = rem % Wp0;
        if (lam < 0 || c >= g.in_channels || kh >= Kh0 || kw >= Kw0)
            return fail(USC_ERR_CORRUPT, "offset %lld does not decode to a tap", (long long)lam);
        *cpos = c;
        bool zero;
        switch (pl->dtype) {
            case USC_F32:
            case USC_F16: zero = ((const float *)payload)[j] == 0.0f; break;
            case USC_I8: zero = ((const int8_t *)payload)[j] == 0; break;
            default: zero = table[((const uint8_t *)payload)[j] & 15] == 0.0f; break;
        }
        if (zero) {
            // a zero-weight entry only matters when x is non-finite, where one copy
            // per distinct offset already yields the NaN
            if (!zero_seen.insert(lam).second) {
                *off = -1;
                return USC_OK;
            }
        }
        if (pl->transposed) std::swap(kh, kw);  // (c, kh, 0) -> (c, 0, kh)
        dec_kh = kh;
        dec_kw = kw;
        const int64_t cl = c - (c / CC) * CC;
        if (pl->kernel == 1)
            *off = cl * cs_tiled + kh * Ws + kw;
        else if (pl->kernel == 4)  // TMEM column of the position (two samples per lane)
            *off = ((cl * pl->HS + kh) * pl->TWs + kw) * 2;
        else if (pl->kernel == 3)  // byte offset in the [CC][HS][TWs][IL] f32 stage
            *off = ((cl * pl->HS + kh) * pl->TWs + kw) * (pl->dtype == USC_F32 ? 4 : 2) * pl->in.interleave;
        else
            *off = (c * Hp + kh) * Ws + kw;
        if (*off >= max_off || *off > INT32_MAX)
            return fail(USC_ERR_UNSUPPORTED, "packed offset %lld too large", (long long)*off);
        return USC_OK;
    };
    if (pl->kernel == 3 || pl->kernel == 4) {
        // blob = [64 B][int32 blk[nb+1]][int32 perm[G*DT]][blocks].  Block (group, chunk):
        // int2 hdr[DT] = {first, end} entry index of each slot's run (relative to the
        // entries after hdr), runs start at even indices (16-B aligned pairs).
        // perm: output channel of every (group, warp, slot), -1 for an empty slot.  The
        // assignment balances the warps: channels in decreasing entry count go to the
        // warp whose worst per-chunk load grows least (the ring lets a warp run at most
        // stages-1 chunks ahead of the slowest, so per-chunk balance is what counts).
        const int64_t nb = (int64_t)G * NC;
        const int WC = pl->WC, DW = pl->DW;
        const int NCLS = std::max(1, pl->ncls_r * pl->ncls_c);
        int32_t *blk = (int32_t *)((char *)blob + 64);
        int32_t *perm = (int32_t *)((char *)blob + 64 + align16(4 * (nb + 1)));
        int32_t *ctab = (int32_t *)((char *)perm + align16(4 * (int64_t)G * DT));  // rowcls[Yh], colcls[Yw]
        char *base = (char *)ctab + align16(4 * ((int64_t)pl->out_h + pl->out_w));
        const int64_t cap = blob_bytes - (base - (char *)blob);
        std::vector<int> rowcls(pl->out_h, 0), colcls(pl->out_w, 0);
        std::vector<uint32_t> rmask(NCLS, ~0u), cmask(NCLS, ~0u);
        // halo taps are dropped only when every weight is finite (theta*0 must be +-0)
        bool finite = true;
        for (int64_t j = 0; j < (int64_t)D * n_nz && finite; ++j) {
            float t;
            const int32_t w = theta_word(pl->dtype, payload, table, j);
            if (pl->dtype == USC_F16 || pl->dtype == USC_I8) {
                finite = (w & 0x7c00) != 0x7c00;
                continue;
            }
            std::memcpy(&t, &w, 4);
            finite = std::isfinite(t);
        }
        if (NCLS > 1 && finite) {
            if (pl->ncls_r > 1) tap_classes(pl->out_h, g.stride_h, g.pad_h, g.filter_h, g.input_h, rowcls, rmask);
            if (pl->ncls_c > 1) tap_classes(pl->out_w, g.stride_w, g.pad_w, g.filter_w, g.input_w, colcls, cmask);
        }
        std::vector<std::vector<std::pair<int64_t, int64_t>>> per(D);  // (chunk, off) per d
        std::vector<std::vector<int64_t>> src(D);
        std::vector<std::vector<uint16_t>> tap(D);  // kh << 8 | kw per entry
        std::vector<std::vector<int32_t>> chan(D);  // input channel per entry
        std::vector<int64_t> cnt((size_t)D * NC, 0);
        for (int d = 0; d < D; ++d) {
            zero_seen.clear();
            for (int64_t j = row_ptr[d]; j < row_ptr[d] + n_nz; ++j) {
                int64_t cpos, off;
                int rc = decode(j, &cpos, &off);
                if (rc) return rc;
                if (off < 0) continue;
                per[d].push_back({cpos / CC, off});
                src[d].push_back(j);
                tap[d].push_back((uint16_t)(dec_kh << 8 | dec_kw));
                chan[d].push_back((int32_t)cpos);
                ++cnt[(size_t)d * NC + cpos / CC];
            }
        }
        std::vector<int> order(D);
        for (int d = 0; d < D; ++d) order[d] = d;
        std::stable_sort(order.begin(), order.end(),
                         [&](int x, int y) { return per[x].size() > per[y].size(); });
        const int bins = G * WC;
        std::vector<int64_t> load((size_t)bins * NC, 0), tot(bins, 0);
        std::vector<int> used(bins, 0);
        std::vector<int32_t> slot((size_t)G * DT, -1);
        for (int d : order) {
            int best = -1;
            int64_t bmax = INT64_MAX, btot = INT64_MAX;
            for (int bi = 0; bi < bins; ++bi) {
                if (used[bi] == DW) continue;
                int64_t m = 0;
                for (int k = 0; k < NC; ++k)
                    m = std::max(m, load[(size_t)bi * NC + k] + cnt[(size_t)d * NC + k]);
                if (m < bmax || (m == bmax && tot[bi] < btot)) {
                    best = bi;
                    bmax = m;
                    btot = tot[bi];
                }
            }
            for (int k = 0; k < NC; ++k) load[(size_t)best * NC + k] += cnt[(size_t)d * NC + k];
            tot[best] += (int64_t)per[d].size();
            slot[(size_t)(best / WC) * DT + (best % WC) * DW + used[best]++] = d;
        }
        int64_t pos = 0, worst = 0, total = 0;
        if (pl->window) {
            // k_bw block (group, chunk): int2 hdr[WC] = {first, end} of every channel subgroup's
            // merged run; a run lists, per input row (c, kh) in ascending order, one ROW entry
            // (window offset) then the MAC entries (code = slot * KW + kw, theta) of the
            // subgroup's slots -- per slot still in stored (c, kh, kw) order -- and ends with an
            // END entry (the kernel prefetches one entry ahead: 16 B of slack follow the block)
            const int KW = g.filter_w;
            const int64_t pxb = (pl->dtype == USC_F32 ? 4 : 2) * (int64_t)pl->in.interleave;
            const uint32_t ROW = 62u << 24, END = 63u << 24;
            for (int gi = 0; gi < G; ++gi)
                for (int k = 0; k < NC; ++k) {
                    blk[(int64_t)gi * NC + k] = (int32_t)pos;
                    char *b = base + pos;
                    std::vector<int32_t> runs(2 * (size_t)WC);
                    std::vector<std::pair<uint32_t, int64_t>> out;  // (word0, stored entry j or -1)
                    for (int wc = 0; wc < WC; ++wc) {
                        runs[2 * wc] = (int32_t)out.size();
                        struct E {
                            int cl, kh, dw, kw;
                            int64_t j;
                        };
                        std::vector<E> ents;
                        for (int dw = 0; dw < DW; ++dw) {
                            const int d = slot[(size_t)gi * DT + wc * DW + dw];
                            if (d < 0) continue;
                            for (size_t i = 0; i < per[d].size(); ++i)
                                if (per[d][i].first == k)
                                    ents.push_back({chan[d][i] - k * CC, tap[d][i] >> 8, dw, tap[d][i] & 255, src[d][i]});
                        }
                        std::stable_sort(ents.begin(), ents.end(), [](const E &x, const E &y) {
                            if (x.cl != y.cl) return x.cl < y.cl;
                            if (x.kh != y.kh) return x.kh < y.kh;
                            if (x.dw != y.dw) return x.dw < y.dw;
                            return x.kw < y.kw;
                        });
                        int lc = -1, lk = -1;
                        for (const E &en : ents) {
                            if (en.cl != lc || en.kh != lk) {
                                const int64_t off = ((int64_t)en.cl * pl->HS + en.kh) * pl->TWs * pxb;
                                if (off >= (1 << 24)) return fail(USC_ERR_UNSUPPORTED, "window offset too large");
                                out.push_back({ROW | (uint32_t)off, -1});
                                lc = en.cl;
                                lk = en.kh;
                            }
                            out.push_back({(uint32_t)(en.dw * KW + en.kw) << 24, en.j});
                        }
                        out.push_back({END, -1});
                        runs[2 * wc + 1] = (int32_t)out.size();
                    }
                    const int64_t hdr_raw = (int64_t)WC * 8, hdr = align16(hdr_raw);
                    const int64_t bytes = align16(hdr + (int64_t)out.size() * 8);
                    if (!dry && pos + bytes + 16 > cap) return fail(USC_ERR_VALUE, "pack buffer too small");
                    if (!dry) {
                        std::memset(b, 0, (size_t)bytes);
                        std::memcpy(b, runs.data(), (size_t)hdr_raw);
                        char *ents = b + hdr;
                        for (size_t i = 0; i < out.size(); ++i) {
                            int32_t v[2] = {(int32_t)out[i].first,
                                            out[i].second < 0 ? 0 : theta_word(pl->dtype, payload, table, out[i].second)};
                            std::memcpy(ents + i * 8, v, 8);
                        }
                    }
                    total += (int64_t)out.size();
                    worst = std::max(worst, bytes + 16);
                    pos += bytes;
                }
        }
        for (int gi = 0; gi < (pl->window ? 0 : G); ++gi)
            for (int k = 0; k < NC; ++k) {
                blk[(int64_t)gi * NC + k] = (int32_t)pos;
                char *b = base + pos;
                int64_t e = 0;  // entry index after the header
                std::vector<int32_t> runs(2 * (size_t)NCLS * DT);
                std::vector<std::pair<int64_t, int64_t>> out;  // (off, j)
                for (int cls = 0; cls < NCLS; ++cls) {
                    const int ncc = std::max(1, pl->ncls_c);  // class = row class * ncc + column class
                    const uint32_t rm = rmask[cls / ncc], cm = cmask[cls % ncc];
                    for (int dl = 0; dl < DT; ++dl) {
                        if (e & 1) {
                            out.push_back({-1, -1});  // alignment pad, never referenced
                            ++e;
                        }
                        const size_t h = (size_t)cls * DT + dl;
                        runs[2 * h] = (int32_t)e;
                        const int d = slot[(size_t)gi * DT + dl];
                        if (d >= 0)
                            for (size_t i = 0; i < per[d].size(); ++i) {  // stored order within the chunk
                                if (per[d][i].first != k) continue;
                                // a tap on this class's zero halo adds theta*0 = +-0: skipped
                                // (exact: acc is never -0 and theta is finite)
                                if (NCLS > 1 && !((rm >> (tap[d][i] >> 8)) & 1 && (cm >> (tap[d][i] & 255)) & 1))
                                    continue;
                                out.push_back({per[d][i].second, src[d][i]});
                                ++e;
                            }
                        runs[2 * h + 1] = (int32_t)e;
                    }
                }
                const int64_t hdr_raw = (int64_t)NCLS * DT * 8, hdr = align16(hdr_raw);  // entries 16-B aligned
                const int64_t bytes = align16(hdr + e * 8);
                if (!dry && pos + bytes + 16 > cap) return fail(USC_ERR_VALUE, "pack buffer too small");
                if (!dry) {
                    std::memset(b, 0, (size_t)bytes);
                    std::memcpy(b, runs.data(), (size_t)hdr_raw);
                    char *ents = b + hdr;
                    for (int64_t i = 0; i < (int64_t)out.size(); ++i) {
                        if (out[i].first < 0) continue;
                        int32_t v[2];
                        v[0] = (int32_t)out[i].first;
                        v[1] = theta_word(pl->dtype, payload, table, out[i].second);
                        std::memcpy(ents + i * 8, v, 8);
                    }
                }
                total += (int64_t)out.size();
                worst = std::max(worst, bytes + 16);
                pos += bytes;
            }
        if (!dry) {
            blk[nb] = (int32_t)pos;
            std::memcpy(perm, slot.data(), slot.size() * 4);
            std::memcpy(ctab, rowcls.data(), rowcls.size() * 4);
            std::memcpy(ctab + pl->out_h, colcls.data(), colcls.size() * 4);
        }
        *n_entries = dry ? worst : total;
        if (!dry && worst > pl->ent_stage_bytes)
            return fail(USC_ERR_VALUE, "entry block of %lld bytes exceeds the %d-byte stage reserve",
                        (long long)worst, pl->ent_stage_bytes);
        return USC_OK;
    }
    int32_t *cpg = (int32_t *)((char *)blob + 64);
    const int64_t cp_bytes = align16(4 * ((int64_t)G * NC * DT + 1));
    char *ent = (char *)blob + 64 + cp_bytes;
    const int eb = entry_bytes(pl->dtype);
    int64_t pos = 0;
    for (int gi = 0; gi < G; ++gi)
        for (int k = 0; k < NC; ++k)
            for (int dl = 0; dl < DT; ++dl) {
                cpg[((int64_t)gi * NC + k) * DT + dl] = (int32_t)pos;
                int d = gi * DT + dl;
                if (d >= D) continue;
                zero_seen.clear();
                for (int64_t j = row_ptr[d]; j < row_ptr[d] + n_nz; ++j) {
                    int64_t c, off;
                    int rc = decode(j, &c, &off);
                    if (rc) return rc;
                    if (off < 0 || c / CC != k) continue;
                    char *e = ent + pos * eb;
                    switch (pl->dtype) {
                        case USC_F32:
                        case USC_F16: {
                            int32_t v[2];
                            v[0] = (int32_t)off;
                            std::memcpy(&v[1], &((const float *)payload)[j], 4);
                            std::memcpy(e, v, 8);
                            break;
                        }
                        case USC_I8: {
                            int32_t v = (int32_t)((uint32_t)(uint8_t)((const int8_t *)payload)[j] << 24 |
                                                  (uint32_t)off);
                            std::memcpy(e, &v, 4);
                            break;
                        }
                        default: {
                            uint32_t idx = ((const uint8_t *)payload)[j] & 15;
                            uint32_t v = idx << 28 | (uint32_t)off;
                            std::memcpy(e, &v, 4);
                            break;
                        }
                    }
                    ++pos;
                }
            }
    cpg[(int64_t)G * NC * DT] = (int32_t)pos;
    *n_entries = pos;
    return USC_OK;
}

// ---------------------------------------------------------------------------
// quantisation primitives (quantization.py)

// quantization.py:41-58
int usc_fit_fixed_point(double amax, int32_t total_bits, int32_t *int_bits, int32_t *frac_bits,
                        double *sigma) {
    if (total_bits < 2) return fail(USC_ERR_VALUE, "total_bits must be >= 2");
    // the reference's math.ceil(log2(inf or nan)) raises (OverflowError / ValueError)
    if (!std::isfinite(amax)) return fail(USC_ERR_VALUE, "cannot fit a fixed-point format to a non-finite maximum");
    int ib = amax == 0.0 ? 0 : (int)std::ceil(std::log2(amax));
    *int_bits = ib;
    *frac_bits = total_bits - ib - 1;
    *sigma = std::pow(2.0, (double)(-(*frac_bits)));
    return USC_OK;
}

// quantization.py:61-76: copysign(floor(|x/sigma| + 0.5)) clipped to +-(2^(b-1)-1)
int usc_linear_codes(const double *x, int64_t count, double sigma, int32_t bits, double *codes) {
    const double limit = std::ldexp(1.0, bits - 1) - 1.0;
    for (int64_t i = 0; i < count; ++i) {
        double s = x[i] / sigma;
        double c = std::copysign(std::floor(std::fabs(s) + 0.5), s);
        codes[i] = c < -limit ? -limit : (c > limit ? limit : c);  // np.clip (NaN stays NaN)
    }
    return USC_OK;
}

// numpy's pairwise summation (the add.reduce behind ndarray.mean), so the
// k-means centroids are bit-identical to the reference's `sel.mean()`.
static double pairwise_sum(const double *a, int64_t n) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; ++i) r += a[i];
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
}

// quantization.py:112-131
static void kmeans_1d(const std::vector<double> &values, int k_req, std::vector<double> &cent,
                      std::vector<int64_t> &assign) {
    std::vector<double> uniq(values);
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    const int64_t U = (int64_t)uniq.size();
    const int k = (int)std::min<int64_t>(k_req, U);
    cent.assign(k, 0.0);
    for (int i = 0; i < k; ++i) {
        double t = ((double)i + 0.5) / (double)k * (double)U;
        double m = std::min(t, (double)(U - 1));
        cent[i] = uniq[(int64_t)m];
    }
    const int64_t n = (int64_t)values.size();
    std::vector<int64_t> na(n);
    std::vector<double> sel;
    assign.clear();
    for (int it = 0; it < 100; ++it) {
        for (int64_t i = 0; i < n; ++i) {
            int best = 0;
            double bd = std::fabs(values[i] - cent[0]);
            for (int j = 1; j < k; ++j) {
                double dd = std::fabs(values[i] - cent[j]);
                if (dd < bd) {
                    bd = dd;
                    best = j;
                }
            }
            na[i] = best;
        }
        if (!assign.empty() && na == assign) break;
        assign = na;
        for (int j = 0; j < k; ++j) {
            sel.clear();
            for (int64_t i = 0; i < n; ++i)
                if (assign[i] == j) sel.push_back(values[i]);
            if (!sel.empty()) cent[j] = pairwise_sum(sel.data(), (int64_t)sel.size()) / (double)sel.size();
        }
    }
}

// quantization.py:134-180
int usc_kmeans_codebook(const double *w, int64_t count, int32_t omega, int32_t psi, double *centroids,
                        double *quantized, int64_t *assignments, int32_t *k_out, int32_t *zp_out) {
    if (omega < 1) return fail(USC_ERR_VALUE, "omega must be >= 1");
    if (psi != 8 && psi != 16) return fail(USC_ERR_VALUE, "psi must be 8 or 16");
    std::vector<double> nz;
    for (int64_t i = 0; i < count; ++i)
        if (w[i] != 0.0) nz.push_back(w[i]);
    const bool zp = (int64_t)nz.size() < count;
    const int budget = zp ? omega - 1 : omega;
    if (budget < 1) return fail(USC_ERR_VALUE, "omega too small to pin zero and keep a cluster");
    std::vector<double> cent;
    if (nz.empty()) {
        cent = {0.0};
        for (int64_t i = 0; i < count; ++i) assignments[i] = 0;
    } else {
        std::vector<double> nc;
        std::vector<int64_t> na;
        kmeans_1d(nz, budget, nc, na);
        if (zp) {
            cent.push_back(0.0);
            cent.insert(cent.end(), nc.begin(), nc.end());
            int64_t j = 0;
            for (int64_t i = 0; i < count; ++i) assignments[i] = (w[i] != 0.0) ? na[j++] + 1 : 0;
        } else {
            cent = nc;
            for (int64_t i = 0; i < count; ++i) assignments[i] = na[i];
        }
    }
    const int K = (int)cent.size();
    double amax = 0.0;
    for (double v : cent) amax = std::max(amax, std::fabs(v));
    int32_t ib, fb;
    double sigma;
    usc_fit_fixed_point(amax, psi, &ib, &fb, &sigma);
    for (int i = 0; i < K; ++i) {
        centroids[i] = cent[i];
        double code;
        usc_linear_codes(&cent[i], 1, sigma, psi, &code);
        quantized[i] = 0.0 + sigma * code;  // mu + sigma*codes (quantization.py:73)
    }
    if (zp) quantized[0] = 0.0;
    *k_out = K;
    *zp_out = zp ? 1 : 0;
    return USC_OK;
}

}  // extern "C"
