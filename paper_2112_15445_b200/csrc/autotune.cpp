// usc_autotune: the per-layer tile search behind the C ABI, so a non-Python caller
// (the reference's FFI) can tune a layer without the Python engine.
//
// Mirrors autotune_sb (/root/reference/pkg/src/unsparse/engine.py:139-170): every
// candidate is timed (median of `repeats` after `warmup`) and the fastest wins, with
// candidates within `noise_floor` of the best resolved toward the earlier one -- the
// reference's "smallest sub-batch within the noise floor" rule, since candidates are
// enumerated in ascending sub-batch order.  The reference's candidates are the
// sub-batch sizes (2, 4, 8); on the B200 a candidate is a tile: the batch-interleaved
// kernel's compiled instances x warp splits x ring depths x pixel classes (kernel 3),
// and the padded-NCHW kernel's sub-batch x pixels x channels (kernel 1) -- the same
// space engine.tile_candidates enumerates in Python.
#include "usc_internal.h"
#include "bi_instances.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstring>
#include <set>
#include <vector>

using usc::fail;

namespace {

struct DevBuf {
    void *p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    bool alloc(size_t bytes) {
        if (p) cudaFree(p);
        p = nullptr;
        return cudaMalloc(&p, bytes < 16 ? 16 : bytes) == cudaSuccess;
    }
};

int storage_bytes(int dtype, bool bi) {
    switch (dtype) {
        case USC_F32: return 4;
        case USC_I8: return bi ? 2 : 1;  // the BI kernel stages int8 codes as binary16
        default: return 2;
    }
}

int out_bytes(int dtype) { return (dtype == USC_F32 || dtype == USC_I8) ? 4 : 2; }

// engine.tile_candidates, restated
std::vector<usc_exec_cfg> candidates(const usc_geometry &g, int n, int dtype) {
    std::vector<usc_exec_cfg> out;
    const bool one_d = g.input_w == 1;
    int oh, ow;
    usc_geometry_out(&g, &oh, &ow);
    const int yw = one_d ? oh : ow, yh = one_d ? ow : oh;
    const int sw = one_d ? g.stride_h : g.stride_w;
    const bool h16 = dtype != USC_F32;
    int cnt = usc_bi_instances(nullptr, 0);
    std::vector<int32_t> inst(7 * (size_t)cnt);
    usc_bi_instances(inst.data(), cnt);
    for (int i = 0; i < cnt; ++i) {
        const int32_t *r = &inst[7 * (size_t)i];
        const int nw = r[0], pc = r[1], pr = r[2], dw = r[3], isw = r[4], spl = r[5], kind = r[6];
        if (kind != (h16 ? 1 : 0)) continue;
        if (isw != sw || (pc > std::max(1, yw) && pc > 1) || pr > yh || (spl == 2 && n <= 32 && !h16)) continue;
        const int strips = ((yh + pr - 1) / pr) * ((yw + pc - 1) / pc);
        for (int ws = 1; ws <= nw; ++ws) {
            if (nw % ws) continue;
            if (ws > strips) break;
            const bool classes = (pc == 1 || pr == 1) && yh * yw <= 64;
            for (int st = 2; st <= 3; ++st)
                for (int pcl = 0; pcl <= (classes ? 1 : 0); ++pcl) {
                    usc_exec_cfg c{};
                    c.sub_batch = 1;
                    c.worker_count = 1;
                    c.pix_per_thread = pc;
                    c.rows_per_thread = pr;
                    c.ch_per_cta = dw * (nw / ws);
                    c.kernel = 3;
                    c.threads = nw * 32;
                    c.pixel_warps = ws;
                    c.stages = st;
                    c.samples_per_cta = 32 * spl;
                    c.pixel_classes = pcl;
                    out.push_back(c);
                }
        }
    }
    for (int sb : {1, 2, 4, 8}) {
        if (n % sb) continue;
        for (int p : {2, 4, 8}) {
            if (p > std::max(2, yw)) continue;
            for (int dt : {8, 16}) {
                usc_exec_cfg c{};
                c.sub_batch = sb;
                c.worker_count = 1;
                c.samples_per_cta = sb > 1 ? sb : 0;
                c.pix_per_thread = p;
                c.ch_per_cta = dt;
                c.kernel = 1;
                out.push_back(c);
            }
        }
    }
    return out;
}

}  // namespace

int usc_autotune(const usc_geometry *g, int32_t n, int32_t dtype, const int64_t *row_ptr,
                 const int64_t *col_offsets, const void *payload, int64_t n_nz, const float *table,
                 const void *x_dev, int32_t repeats, int32_t warmup, float noise_floor, usc_exec_cfg *best,
                 float *best_ms, void *stream) {
    if (!g || !row_ptr || !col_offsets || !payload || !x_dev || !best) return fail(USC_ERR_VALUE, "null argument");
    if (n < 1 || repeats < 1 || warmup < 0 || noise_floor < 0.0f) return fail(USC_ERR_VALUE, "bad search settings");
    if (dtype == USC_CB4 && !table) return fail(USC_ERR_VALUE, "USC_CB4 needs the centroid table");
    int rc = usc_geometry_check(g);
    if (rc) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int oh, ow;
    usc_geometry_out(g, &oh, &ow);
    DevBuf y;
    if (!y.alloc((size_t)n * g->out_channels * oh * ow * out_bytes(dtype)))
        return fail(USC_ERR_CUDA, "autotune: output allocation failed");
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct Tried {
        float ms;
        usc_exec_cfg cfg;
    };
    std::vector<Tried> tried;
    std::set<std::array<int, 13>> seen;
    // padded inputs per resolved input layout (reused across candidates)
    std::vector<std::pair<std::array<int, 8>, DevBuf *>> pads;
    std::vector<DevBuf> pad_store(64);
    std::vector<char> blob;
    for (usc_exec_cfg cfg : candidates(*g, n, dtype)) {
        usc_plan pl;
        if (usc_plan_make(g, n, dtype, &cfg, &pl)) continue;
        if (pl.kernel == 3 || pl.kernel == 4) {  // size the entry reserve from the filter (engine.fit_plan)
            usc_exec_cfg probe_cfg = cfg;
            probe_cfg.chunk_channels = pl.CC;
            probe_cfg.ent_reserve = 256;
            usc_plan probe;
            if (usc_plan_make(g, n, dtype, &probe_cfg, &probe)) continue;
            int64_t worst = 0;
            if (usc_pack(&probe, row_ptr, col_offsets, payload, n_nz, table, nullptr, 0, &worst)) continue;
            probe_cfg.ent_reserve = (int32_t)std::max<int64_t>(256, worst);
            if (usc_plan_make(g, n, dtype, &probe_cfg, &pl)) continue;
            cfg = probe_cfg;
        }
        std::array<int, 13> key{pl.kernel, pl.P, pl.PR, pl.PC, pl.DT, pl.DW, pl.WS, pl.NS, pl.CC,
                                pl.threads, pl.stages, pl.ncls_r, pl.ncls_c};
        if (!seen.insert(key).second) continue;
        int64_t bytes = 0, n_ent = 0;
        if (usc_pack_size(&pl, n_nz, &bytes)) continue;
        blob.assign((size_t)bytes, 0);
        if (usc_pack(&pl, row_ptr, col_offsets, payload, n_nz, table, blob.data(), bytes, &n_ent)) continue;
        DevBuf dblob;
        if (!dblob.alloc((size_t)bytes)) continue;
        cudaMemcpyAsync(dblob.p, blob.data(), (size_t)bytes, cudaMemcpyHostToDevice, st);
        std::array<int, 8> lk{pl.in.channels, pl.in.height, pl.in.width, pl.in.pad_h, pl.in.pad_w, pl.in.hp,
                              pl.in.ws, pl.in.interleave};
        DevBuf *xp = nullptr;
        for (auto &e : pads)
            if (e.first == lk) xp = e.second;
        if (!xp) {
            if (pads.size() == pad_store.size()) continue;
            xp = &pad_store[pads.size()];
            const int64_t elems = usc_act_layout_elems(&pl.in, n);
            if (!xp->alloc((size_t)elems * storage_bytes(dtype, pl.in.interleave != 0))) continue;
            if (usc_pad_input(&pl.in, dtype, n, x_dev, xp->p, stream)) continue;
            pads.push_back({lk, xp});
        }
        bool ok = true;
        for (int w = 0; w < warmup && ok; ++w) ok = usc_conv_forward(&pl, dblob.p, xp->p, y.p, nullptr, stream) == 0;
        std::vector<float> ts;
        for (int r = 0; r < repeats && ok; ++r) {
            cudaEventRecord(e0, st);
            ok = usc_conv_forward(&pl, dblob.p, xp->p, y.p, nullptr, stream) == 0;
            cudaEventRecord(e1, st);
            cudaEventSynchronize(e1);
            float ms = 0.0f;
            cudaEventElapsedTime(&ms, e0, e1);
            ts.push_back(ms);
        }
        if (!ok || cudaStreamSynchronize(st) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        std::nth_element(ts.begin(), ts.begin() + ts.size() / 2, ts.end());
        tried.push_back({ts[ts.size() / 2], cfg});
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (tried.empty()) return fail(USC_ERR_UNSUPPORTED, "autotune: no candidate tile runs this layer");
    float fastest = tried[0].ms;
    for (auto &t : tried) fastest = std::min(fastest, t.ms);
    for (auto &t : tried)
        if (t.ms <= fastest * (1.0f + noise_floor)) {
            *best = t.cfg;
            if (best_ms) *best_ms = t.ms;
            return USC_OK;
        }
    return USC_OK;
}
