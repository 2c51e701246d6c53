"""Tile configurations of the tensor-core backend per layer shape (b256, binary16, BI64):
every (pixels per tile, K splits) pair timed as a captured CUDA graph of 10 launches (no
host-side cost), next to the automatic choice.  One JSON line per shape.

    python tools/tc_cfg_probe.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

CONFIGS = [(0, 0), (2, 1), (4, 1), (2, 2), (4, 2), (2, 4), (4, 4)]
SHAPES = [  # name, C, D, k, stride, hw, shortcut
    ("vgg-128x128-16", 128, 128, 3, 1, 16, False), ("vgg-256x256-8", 256, 256, 3, 1, 8, False),
    ("vgg-256x512-4", 256, 512, 3, 1, 4, False), ("vgg-512x512-4", 512, 512, 3, 1, 4, False),
    ("vgg-512x512-2", 512, 512, 3, 1, 2, False),
    ("r50-1x1-256x64-32", 256, 64, 1, 1, 32, False), ("r50-3x3-64x64-32", 64, 64, 3, 1, 32, False),
    ("r50-1x1-64x256-32-res", 64, 256, 1, 1, 32, True), ("r50-1x1-512x128-16", 512, 128, 1, 1, 16, False),
    ("r50-3x3-128x128-16", 128, 128, 3, 1, 16, False), ("r50-1x1-128x512-16-res", 128, 512, 1, 1, 16, True),
    ("r50-1x1-1024x256-8", 1024, 256, 1, 1, 8, False), ("r50-3x3-256x256-8", 256, 256, 3, 1, 8, False),
    ("r50-1x1-256x1024-8-res", 256, 1024, 1, 1, 8, True), ("r50-1x1-2048x512-4", 2048, 512, 1, 1, 4, False),
    ("r50-3x3-512x512-4", 512, 512, 3, 1, 4, False), ("r50-1x1-512x2048-4-res", 512, 2048, 1, 1, 4, True),
    ("r50-3x3-256x256-16-s2", 256, 256, 3, 2, 16, False), ("r50-3x3-512x512-8-s2", 512, 512, 3, 2, 8, False),
    ("r50-1x1-512x1024-16-s2", 512, 1024, 1, 2, 16, False)]


def graph_us(fn, reps=10, iters=5):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / reps)
    return sorted(ts)[len(ts) // 2]


def main():
    from paper_2112_15445_b200 import _lib
    from paper_2112_15445_b200.dense import dense_conv, dense_workspace, pack_weights
    n = 256
    for name, C, D, k, s, hw, res in SHAPES:
        halo = k // 2
        xl = _lib.act_layout(C, hw, hw, halo, halo, 2, 64)
        xb = torch.randn(xl.elems(n), device="cuda").half()
        ho = (hw + 2 * halo - k) // s + 1
        yl = _lib.act_layout(D, ho, ho, 1, 1, 2, 64)
        yb = torch.zeros(yl.elems(n), dtype=torch.float16, device="cuda")
        rl = rb = None
        if res:
            rl = _lib.act_layout(D, ho, ho, 0, 0, 2, 64)
            rb = torch.randn(rl.elems(n), device="cuda").half()
        wp = pack_weights((torch.randn(D, C, k, k, device="cuda") / (C * k * k) ** 0.5).half())
        out = {"layer": name}
        for twp, sp in CONFIGS:
            if res and sp > 1:
                continue
            ws = dense_workspace(C, D, k, s, n, xl, res, twp=twp, splits=sp)
            try:
                us = graph_us(lambda: dense_conv(wp, C, D, k, s, n, xb, xl, yb, yl, rb, rl, True, None, ws, twp, sp))
            except RuntimeError as e:
                out[f"{twp}/{sp}"] = str(e)[:60]
                continue
            out[f"{twp}/{sp}"] = round(us, 2)
        cands = {k2: v for k2, v in out.items() if k2 != "layer" and isinstance(v, float)}
        out["best"] = min(cands, key=cands.get)
        out["gain_vs_auto"] = round(cands["0/0"] / cands[out["best"]], 3)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
