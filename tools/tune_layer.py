"""Time every autotuner candidate of the given VGG-16 layers (the model's real
buffers and epilogues) and print the fastest ones with their plans.

    python tools/tune_layer.py 10 7 1 [--top 12]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import BATCH, build_model  # noqa: E402
from paper_2112_15445_b200.engine import launch, plan_for, tile_candidates, time_median_cuda  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("layers", type=int, nargs="+")
    ap.add_argument("--top", type=int, default=12)
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--fp16", action="store_true", help="the BINARY16 network")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    if args.fp16:
        from paper_2112_15445_b200 import PrecisionMode
        from paper_2112_15445_b200.models import SparseVGG16, vgg16_rng, vgg16_weights
        F16 = PrecisionMode.BINARY16
        model = SparseVGG16(vgg16_weights(vgg16_rng(0.93, 0), 0.93, precision=F16), args.batch, precision=F16)
    else:
        model, _ = build_model(args.batch, dev)
    for st in [s for s in model.steps if s[0] == "conv" and s[1] in args.layers]:
        _, li, plan0, _, xin, yout, epi = st
        g = model.geoms[li]
        cands = [c for c in tile_candidates(g, args.batch, [1], model.precision, (3, 4))
                 if c.samples_per_cta == model.interleave]
        if epi.pool:
            cands = [c for c in cands if c.rows_per_thread == 2 and c.pix_per_thread % 2 == 0]
        res = []
        for cfg in cands:
            try:
                plan, blob = model._plan_for(li, cfg)
            except ValueError:
                continue
            ms = time_median_cuda(lambda: launch(plan, blob, xin, yout, epi), 7, 2)
            res.append((ms, plan.describe()))
        res.sort(key=lambda r: r[0])
        print(f"layer {li} ({g.in_channels}->{g.out_channels}, {g.input_h}x{g.input_w}): {len(res)} candidates")
        best_by_kernel = {}
        for ms, d in res:
            best_by_kernel.setdefault(d["kernel"], (ms, d))
        shown = res[:args.top] + [v for v in best_by_kernel.values() if v not in res[:args.top]]
        for ms, d in shown:
            keep = {k: d[k] for k in ("kernel", "P", "PR", "PC", "DT", "DW", "WS", "threads", "CC", "stages", "grid",
                                      "pixel_classes")}
            print(f"  {ms * 1e3:8.1f} us  {keep}")


if __name__ == "__main__":
    main()
