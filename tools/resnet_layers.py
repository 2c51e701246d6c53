"""Per-conv device time of the ResNet-50 CIFAR network (batch 256, committed tuned state) on
the sparse kernel: each step timed alone on the network's own buffers, with its nonzero
TF/s and algorithmic HBM GB/s (input + output (+ shortcut) once, packed entries).

    python tools/resnet_layers.py [fp32|fp16]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    from paper_2112_15445_b200 import PrecisionMode
    from paper_2112_15445_b200.engine import time_median_cuda
    from paper_2112_15445_b200.resnet import SparseResNet50, resnet50_weights
    pn = sys.argv[1] if len(sys.argv) > 1 else "fp32"
    prec = PrecisionMode.BINARY16 if pn == "fp16" else PrecisionMode.BINARY32
    eb = 2 if pn == "fp16" else 4
    ws = resnet50_weights(0.9, 0, prec)
    n = 256
    m = SparseResNet50(ws, n, precision=prec)
    m.load_tuned_state(json.load(open(os.path.join(ROOT, "profiles", f"r02_tuned_resnet50_{pn}.json"))))
    m.run()
    torch.cuda.synchronize()
    tot = 0.0
    for st in m.steps:
        li = st[0]
        if st[1] is None:
            continue
        name, g, role, s = m.layers[li]
        ms = time_median_cuda(lambda: m._launch(st), 7, 2, 2)
        tot += ms
        nnz = int(np.count_nonzero(np.asarray(ws[li].data)))
        macs = nnz * g.out_h * g.out_w * n
        res = role == "c3"
        byts = eb * n * (g.in_channels * g.input_h * g.input_w + g.out_channels * g.out_h * g.out_w * (2 if res else 1))
        print(json.dumps({"conv": name, "shape": f"{g.in_channels}->{g.out_channels} {g.filter_h}x{g.filter_w}"
                          f" s{g.stride[0]} @{g.input_h}", "us": round(ms * 1e3, 1),
                          "nonzero_tflops": round(2 * macs / ms / 1e9, 2), "hbm_gbs": round(byts / ms / 1e6, 1),
                          "plan": {k: v for k, v in st[1].describe().items() if k in ("P", "DT", "NS", "CC", "threads")}}),
              flush=True)
    print(json.dumps({"sum_ms": round(tot, 3)}))


if __name__ == "__main__":
    main()
