"""Run every autotuner candidate of every VGG-16 layer (with the model's real
epilogue and buffers) once, synchronising after each launch, and compare the
layer output bitwise with the layer's default plan.  Prints the first failing
candidate.  Run under compute-sanitizer to locate an illegal access:

    compute-sanitizer --print-limit 3 python tools/check_tiles.py [batch]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import build_model  # noqa: E402
from paper_2112_15445_b200.engine import launch, plan_for, tile_candidates  # noqa: E402


def main():
    batch = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    fp16 = "--fp16" in sys.argv
    only = [int(a) for a in sys.argv[2:] if a.isdigit()]
    dev = torch.device("cuda", 0)
    if fp16:
        from paper_2112_15445_b200 import PrecisionMode
        from paper_2112_15445_b200.models import SparseVGG16, vgg16_rng, vgg16_weights
        F16 = PrecisionMode.BINARY16
        model = SparseVGG16(vgg16_weights(vgg16_rng(0.93, 0), 0.93, precision=F16), batch, precision=F16)
        x = torch.randn(batch, 3, 32, 32, device=dev).half()
    else:
        model, _ = build_model(batch, dev)
        x = torch.randn(batch, 3, 32, 32, device=dev)
    model.load_input(x)
    model.run()
    torch.cuda.synchronize()
    bad = 0
    for st in [s for s in model.steps if s[0] == "conv" and (not only or s[1] in only)]:
        _, li, plan0, blob0, xin, yout, epi = st
        keep = yout.clone()
        yout.fill_(float("nan"))  # the halo stays NaN in every run; only the interior is written
        launch(plan0, blob0, xin, yout, epi)
        torch.cuda.synchronize()
        ref = yout.clone()
        g = model.geoms[li]
        cands = [c for c in tile_candidates(g, batch, [1], model.precision, (3, 4))
                 if c.samples_per_cta == model.interleave]
        if epi.pool:
            cands = [c for c in cands if c.rows_per_thread == 2 and c.pix_per_thread % 2 == 0]
        n = 0
        for cfg in cands:
            try:
                plan, blob = model._plan_for(li, cfg)
            except ValueError:
                continue
            yout.fill_(float("nan"))
            print(f"layer {li} P{cfg.rows_per_thread}x{cfg.pix_per_thread} DT{cfg.ch_per_cta} "
                  f"T{cfg.threads} WS{cfg.pixel_warps}", flush=True)
            launch(plan, blob, xin, yout, epi)
            torch.cuda.synchronize()
            n += 1
            if not torch.equal(yout.view(torch.int32), ref.view(torch.int32)):
                bad += 1
                print(f"MISMATCH layer {li}: {cfg} plan={plan.describe()}", flush=True)
        yout.copy_(keep)
        print(f"layer {li}: {n} candidates checked", flush=True)
    print("bad", bad)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
