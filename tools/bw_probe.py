"""Register-window kernel (k_bw) vs the committed k_bi tiles on the VGG-16 network.

For fp32 (bench.py's workload) and binary16: the network with the committed tuned
state, then re-autotuned with the window candidates in the search; per-conv device
time of both, graph step time of both, and a bitwise comparison of the two outputs
(both must equal the reference, so they must equal each other).

    python tools/bw_probe.py [--modes fp32,fp16] [--dump DIR]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def step_ms(m, steps=30):
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for _ in range(3):
        m.graph.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        m.graph.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def per_conv(m):
    from paper_2112_15445_b200.engine import time_median_cuda
    out = {}
    for st in m.steps:
        out.setdefault(st[1], 0.0)
        out[st[1]] += time_median_cuda(lambda: m._run_step(st), 9, 2)
    return {k: round(v * 1e3, 1) for k, v in out.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--modes", default="fp32,fp16")
    ap.add_argument("--dump", default="gpurun_out")
    args = ap.parse_args()
    from paper_2112_15445_b200 import PrecisionMode
    from paper_2112_15445_b200.models import SparseVGG16, vgg16_rng, vgg16_weights
    for mode in args.modes.split(","):
        prec = PrecisionMode.BINARY16 if mode == "fp16" else PrecisionMode.BINARY32
        ws = vgg16_weights(vgg16_rng(0.93, 0), 0.93, precision=prec)
        x = torch.from_numpy(np.random.default_rng([1, 0]).standard_normal((256, 3, 32, 32)).astype(np.float32)).cuda()
        if mode == "fp16":
            x = x.half()
        tuned = os.path.join(ROOT, "profiles", "r01_tuned.json" if mode == "fp32" else "r02_tuned_vgg16_fp16.json")
        m0 = SparseVGG16(ws, 256, precision=prec)
        m0.load_tuned_state(json.load(open(tuned)))
        m0.capture()
        out0 = m0.forward(x).float().cpu().numpy()
        t0, l0 = step_ms(m0), per_conv(m0)
        m1 = SparseVGG16(ws, 256, precision=prec)
        m1.autotune(repeats=3, warmup=1)
        m1.capture()
        out1 = m1.forward(x).float().cpu().numpy()
        t1, l1 = step_ms(m1), per_conv(m1)
        picks = {li: m1.steps[[s[1] for s in m1.steps].index(li)][2].describe()["kernel"]
                 for li in range(13) if m1.steps[[s[1] for s in m1.steps].index(li)][0] == "conv"}
        os.makedirs(args.dump, exist_ok=True)
        with open(os.path.join(args.dump, f"bw_tuned_vgg16_{mode}.json"), "w") as fh:
            json.dump(m1.tuned_state(), fh)
        print(json.dumps({"mode": mode, "bitwise_equal": bool(np.array_equal(out0, out1)),
                          "committed_ms": round(t0, 4), "retuned_ms": round(t1, 4),
                          "images_per_s": {"committed": round(256 / t0 * 1e3), "retuned": round(256 / t1 * 1e3)},
                          "per_conv_us": {"committed": l0, "retuned": l1}, "kernels": picks}), flush=True)


if __name__ == "__main__":
    main()
