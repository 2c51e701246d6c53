"""Per-conv breakdown of the autotuned ResNet-50 CIFAR network (configs[2]): each
step's device time (its own buffers and epilogue), the chosen plan, achieved
nonzero TF/s and HBM GB/s (algorithmic bytes: unpadded input + output (+ shortcut)
+ entries), sorted by time.

    python tools/resnet_layers.py [fp16|fp32] [--batch 256]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2112_15445_b200 import PrecisionMode  # noqa: E402
from paper_2112_15445_b200.engine import time_median_cuda  # noqa: E402
from paper_2112_15445_b200.resnet import SparseResNet50, resnet50_weights  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("prec", nargs="?", default="fp16")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--no-tune", action="store_true")
    args = ap.parse_args()
    prec = PrecisionMode.BINARY16 if args.prec == "fp16" else PrecisionMode.BINARY32
    m = SparseResNet50(resnet50_weights(0.9, 0, prec), args.batch, precision=prec)
    if not args.no_tune:
        m.autotune()
    m.load_input(torch.randn(args.batch, 3, 32, 32, device="cuda").to(m.tdtype))
    m.run()
    torch.cuda.synchronize()
    rows, total = [], 0.0
    for st in m.steps:
        li, plan, blob, x, view, y, e = st
        name, g, role, s = m.layers[li]
        ms = time_median_cuda(lambda: m._launch(st), 9, 2)
        total += ms
        f = m.filters[li]
        nnz = int((f.weights != 0).sum())
        flops = 2.0 * nnz * g.out_h * g.out_w * args.batch
        byt = args.batch * (g.in_channels * g.input_h * g.input_w + g.out_channels * g.out_h * g.out_w
                            * (2 if e.residual else 1)) * m.eb + f.weights.size * 8
        d = plan.describe()
        rows.append((ms, name, f"{g.in_channels}->{g.out_channels} k{g.filter_h} {g.input_h}x{g.input_w} s{s}",
                     d["kernel"], f"P{d['PR']}x{d['PC']} DT{d['DT']} DW{d['DW']} T{d['threads']} CC{d['CC']}",
                     flops / ms / 1e9, byt / ms / 1e6))
    print(f"total {total:.3f} ms over {len(rows)} convs ({args.prec}, batch {args.batch})")
    for ms, name, geo, k, tile, tf, gbs in sorted(rows, reverse=True):
        print(f"{ms * 1e3:8.1f} us {ms / total * 100:5.1f}%  {name:10s} {geo:26s} {k:5s} {tile:34s} "
              f"{tf:6.2f} TF/s {gbs:7.0f} GB/s")


if __name__ == "__main__":
    main()
