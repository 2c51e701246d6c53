"""Per-layer device time of the tensor-core dense backend (usc_dense_conv_f16 on the BI64
layout) next to cuDNN fp16 (channels_last, tensor cores) and the sparse binary16 kernel,
on the VGG-16 CIFAR and ResNet-50 CIFAR layer shapes at batch 256.

    python tools/tc_probe.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    from paper_2112_15445_b200 import _lib
    from paper_2112_15445_b200.dense import dense_conv, dense_workspace, pack_weights, tc_eligible
    from paper_2112_15445_b200.engine import time_median_cuda
    torch.backends.cudnn.benchmark = True
    n = 256
    shapes = [("vgg-128x128-16", 128, 128, 3, 1, 16), ("vgg-256x256-8", 256, 256, 3, 1, 8),
              ("vgg-128x256-8", 128, 256, 3, 1, 8), ("vgg-256x512-4", 256, 512, 3, 1, 4),
              ("vgg-512x512-4", 512, 512, 3, 1, 4), ("vgg-512x512-2", 512, 512, 3, 1, 2),
              ("vgg-64x128-16", 64, 128, 3, 1, 16),
              ("r50-1x1-64x256-32", 64, 256, 1, 1, 32), ("r50-1x1-256x128-32", 256, 128, 1, 1, 32),
              ("r50-3x3-128x128-16", 128, 128, 3, 1, 16), ("r50-1x1-512x256-16", 512, 256, 1, 1, 16),
              ("r50-3x3-256x256-8", 256, 256, 3, 1, 8), ("r50-1x1-1024x256-8", 1024, 256, 1, 1, 8),
              ("r50-3x3-128x128-32-s2", 128, 128, 3, 2, 32), ("r50-1x1-256x512-32-s2", 256, 512, 1, 2, 32),
              ("vgg-3x64-32-first", 3, 64, 3, 1, 32), ("vgg-64x64-32", 64, 64, 3, 1, 32), ("r50-1x1-256x64-32", 256, 64, 1, 1, 32),
              ("r50-1x1-64x64-32", 64, 64, 1, 1, 32),
              ("r50-1x1-64x256-32-res", 64, 256, 1, 1, 32), ("r50-1x1-128x512-16-res", 128, 512, 1, 1, 16),
              ("r50-1x1-256x1024-8-res", 256, 1024, 1, 1, 8), ("r50-1x1-512x2048-4-res", 512, 2048, 1, 1, 4)]
    for name, C, D, k, s, hw in shapes:
        use_res = name.endswith("-res")
        if not tc_eligible(C, D, k, s):
            continue
        x = torch.randn(n, C, hw, hw, device="cuda").half()
        w = (torch.randn(D, C, k, k, device="cuda") / (C * k * k) ** 0.5).half()
        halo = k // 2
        xl = _lib.act_layout(C, hw, hw, halo, halo, 2, 64)
        xb = torch.zeros(xl.elems(n), dtype=torch.float16, device="cuda")
        _lib.check(_lib.lib().usc_pad_input(_lib.ref(xl), _lib.USC_F16, n, _lib.t_ptr(x), _lib.t_ptr(xb),
                                            _lib.stream_ptr()))
        ho = (hw + 2 * halo - k) // s + 1
        yl = _lib.act_layout(D, ho, ho, 1, 1, 2, 64)
        yb = torch.zeros(yl.elems(n), dtype=torch.float16, device="cuda")
        wp = pack_weights(w)
        rb = rl = rc = None
        if use_res:
            rl = _lib.act_layout(D, ho, ho, 0, 0, 2, 64)
            rb = torch.randn(rl.elems(n), device="cuda").half()
            rc = torch.randn(n, D, ho, ho, device="cuda").half().contiguous(memory_format=torch.channels_last)
        ws = dense_workspace(C, D, k, s, n, xl, use_res)
        tc = time_median_cuda(lambda: dense_conv(wp, C, D, k, s, n, xb, xl, yb, yl, rb, rl, True, None, ws), 9, 3)
        xc = x.contiguous(memory_format=torch.channels_last)
        wc = w.contiguous(memory_format=torch.channels_last)
        if use_res:
            cd = time_median_cuda(lambda: torch.relu_(torch.nn.functional.conv2d(xc, wc, stride=s, padding=halo) + rc),
                                  9, 3)
        else:
            cd = time_median_cuda(lambda: torch.relu(torch.nn.functional.conv2d(xc, wc, stride=s, padding=halo)), 9, 3)
        flops = 2.0 * n * D * ho * ho * C * k * k
        hbm = 2.0 * (n * C * hw * hw + n * D * ho * ho * (2 if use_res else 1) + D * C * k * k)
        print(json.dumps({"layer": name, "tc_us": round(tc * 1e3, 1), "cudnn_us": round(cd * 1e3, 1),
                          "speedup_vs_cudnn": round(cd / tc, 2), "tc_dense_tflops": round(flops / tc / 1e9, 1),
                          "tc_algorithmic_gbs": round(hbm / tc / 1e6, 1), "split_k": ws is not None}),
              flush=True)


if __name__ == "__main__":
    main()
