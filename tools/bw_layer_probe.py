"""Per-layer timing of the register-window kernel (k_bw) against the batch-interleaved
tiles (k_bi) on the VGG-16 layers (batch 256, resident BI64 output as the network
writes it).  One JSON line per layer: best k_bi and best k_bw tile and their times,
plus every k_bw candidate's time.

    python tools/bw_layer_probe.py [fp32|fp16] [layers, e.g. 1,5,9]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "fp32"
    from paper_2112_15445_b200 import PrecisionMode, _lib
    from paper_2112_15445_b200.engine import launch, padded_input, plan_for, tile_candidates, time_median_cuda
    from paper_2112_15445_b200.models import vgg16_geometries, vgg16_rng, vgg16_weights
    from paper_2112_15445_b200.csr import build_csr
    prec = PrecisionMode.BINARY16 if mode == "fp16" else PrecisionMode.BINARY32
    dtype = _lib.USC_F16 if mode == "fp16" else _lib.USC_F32
    tdt = torch.float16 if mode == "fp16" else torch.float32
    eb = 2 if mode == "fp16" else 4
    ws = vgg16_weights(vgg16_rng(0.93, 0), 0.93, precision=prec)
    geoms = vgg16_geometries()
    layers = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else range(1, 10)
    n = 256
    for li in layers:
        g = geoms[li]
        f = build_csr(ws[li], g)
        x = torch.randn(n, g.in_channels, g.input_h, g.input_w, device="cuda").to(tdt)
        lay = _lib.act_layout(g.out_channels, g.out_h, g.out_w, 1, 1, eb, 64)
        y = torch.zeros(lay.elems(n), dtype=tdt, device="cuda")
        epi = _lib.Epilogue()
        epi.relu, epi.scale, epi.out_padded, epi.out = 1, 1.0, 1, lay
        res, pads = [], {}
        for cfg in tile_candidates(g, n, [1], prec, (3,)):
            if cfg.samples_per_cta != 64:
                continue
            try:
                plan, blob = plan_for(f, n, dtype, cfg, f.weights)
            except (ValueError, RuntimeError):
                continue
            k = (plan.in_.hp, plan.in_.ws)
            if k not in pads:
                pads[k] = padded_input(x, plan)
            try:
                ms = time_median_cuda(lambda: launch(plan, blob, pads[k], y, epi), 5, 2)
            except RuntimeError as e:
                print(json.dumps({"layer": li, "error": str(e), "plan": plan.describe()}), flush=True)
                continue
            res.append((ms, plan.describe(), bool(cfg.window)))
            f._packs.clear()
        bi = min((r for r in res if not r[2]), key=lambda r: r[0])
        bw = sorted((r for r in res if r[2]), key=lambda r: r[0])
        print(json.dumps({"layer": li, "mode": mode, "bi_us": round(bi[0] * 1e3, 1), "bi_plan": bi[1],
                          "bw_us": round(bw[0][0] * 1e3, 1) if bw else None, "bw_plan": bw[0][1] if bw else None,
                          "bw_all_us": [round(r[0] * 1e3, 1) for r in bw]}), flush=True)


if __name__ == "__main__":
    main()
