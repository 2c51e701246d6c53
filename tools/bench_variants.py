"""Secondary configurations of BASELINE.json next to cuDNN on the same B200
(the headline fp32 VGG-16 line is bench.py's):

  * vgg16-fp16  -- pruned VGG-16 CIFAR-10, 93% sparsity, BINARY16 (binary16 storage,
    fp32 accumulate, binary16 hook), batch 256, vs cuDNN fp16 (channels_last, tensor
    cores) on the same masked weights;
  * sweep       -- one 3x3 layer shape at batch 1024 across sparsities 50-98%
    (configs[4]), fp32, vs cuDNN fp32 (TF32 off).

One JSON line per measurement.  Device time with CUDA events, L2 flushed between
timed network steps.

    python tools/bench_variants.py [--only vgg16-fp16|sweep] [--steps 50]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def timed(fn, steps, flush=None):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        if flush is not None:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def cudnn_vgg(ws, batch, dtype, tf32=False, channels_last=False):
    from paper_2112_15445_b200.models import VGG16_CIFAR
    torch.backends.cudnn.benchmark = True
    torch.backends.cudnn.allow_tf32 = tf32
    mf = torch.channels_last if channels_last else torch.contiguous_format
    wd = [torch.from_numpy(np.array(w.data)).cuda().to(dtype).contiguous(memory_format=mf) for w in ws]
    x = torch.randn(batch, 3, 32, 32, device="cuda", dtype=dtype).contiguous(memory_format=mf)

    def fwd():
        a, li = x, 0
        for v in VGG16_CIFAR:
            if v == "M":
                a = torch.nn.functional.max_pool2d(a, 2)
            else:
                a = torch.relu(torch.nn.functional.conv2d(a, wd[li], padding=1))
                li += 1
        return a
    return fwd


def vgg16_fp16(steps):
    from paper_2112_15445_b200 import PrecisionMode
    from paper_2112_15445_b200.models import SparseVGG16, vgg16_rng, vgg16_weights
    batch = 256
    ws = vgg16_weights(vgg16_rng(0.93, 0), 0.93, precision=PrecisionMode.BINARY16)
    m = SparseVGG16(ws, batch, precision=PrecisionMode.BINARY16)
    m.autotune(repeats=3, warmup=1)
    m.capture()
    m.load_input(torch.randn(batch, 3, 32, 32, device="cuda").half())
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    ms = timed(lambda: m.graph.replay(), steps, flush)
    cd = timed(cudnn_vgg(ws, batch, torch.float16, channels_last=True), steps, flush)
    return {"config": "pruned VGG-16 CIFAR-10 93% BINARY16, batch 256", "dtype": "f16 storage, f32 accumulate",
            "images_per_s": round(batch / (ms / 1e3), 1), "ms_per_step": round(ms, 4),
            "cudnn_fp16_tensor_core": {"images_per_s": round(batch / (cd / 1e3), 1), "ms_per_step": round(cd, 4)},
            "speedup_vs_cudnn": round(cd / ms, 3)}


def vgg16_quantised(mode, steps):
    """int8 / cb4 VGG-16 at batch 256 (cfg4): calibrated on the timed batch itself."""
    from paper_2112_15445_b200.models import SparseVGG16, vgg16_rng, vgg16_weights
    from paper_2112_15445_b200.tensor import round_to_binary16
    batch = 256
    ws = vgg16_weights(vgg16_rng(0.93, 0), 0.93)
    x = torch.randn(batch, 3, 32, 32, device="cuda")
    if mode == "cb4":
        x = round_to_binary16(x)
    m = SparseVGG16(ws, batch, mode=mode, calibration=x)
    m.autotune(repeats=3, warmup=1)
    m.capture()
    m.load_input(x if mode == "int8" else x.half())
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    ms = timed(lambda: m.graph.replay(), steps, flush)
    return {"config": f"pruned VGG-16 CIFAR-10 93% {mode}, batch 256",
            "dtype": {"int8": "int8 codes (staged binary16), exact fp32 accumulate",
                      "cb4": "4-bit codebook weights, binary16 activations"}[mode],
            "images_per_s": round(batch / (ms / 1e3), 1), "ms_per_step": round(ms, 4)}


def sweep(steps):
    from paper_2112_15445_b200 import DenseTensor4, autotune_sb, build_csr, sparse_conv_forward
    from paper_2112_15445_b200.engine import launch, padded_input, plan_for, time_median_cuda
    from paper_2112_15445_b200.pruning import synthesize_masked_weights
    from paper_2112_15445_b200.tensor import ConvGeometry
    out = []
    batch = 1024
    for name, (c, d, hw) in {"r50-3x3-64x32": (64, 64, 32), "r50-3x3-256x8": (256, 256, 8)}.items():
        g = ConvGeometry(c, d, 3, 3, hw, hw, padding=(1, 1))
        x = torch.randn(batch, c, hw, hw, device="cuda")
        for s in (0.5, 0.7, 0.9, 0.95, 0.98):
            rng = np.random.default_rng([0, int(s * 1000)])
            w = synthesize_masked_weights(g, s, rng)
            f = build_csr(w, g)
            xd = DenseTensor4(x)
            cfg = autotune_sb(xd, f, repeats=3, warmup=1)
            plan, blob = plan_for(f, batch, 0, cfg, f.weights)
            xp = padded_input(x, plan)
            y = torch.empty(batch, d, hw, hw, device="cuda")
            ms = time_median_cuda(lambda: launch(plan, blob, xp, y), 9, 2)
            torch.backends.cudnn.benchmark = True
            torch.backends.cudnn.allow_tf32 = False
            wd = torch.from_numpy(np.array(w.data)).cuda()
            cd = time_median_cuda(lambda: torch.nn.functional.conv2d(x, wd, padding=1), 9, 2)
            genuine = int(np.count_nonzero(f.weights))
            flops = 2.0 * genuine * hw * hw * batch
            out.append({"layer": name, "sparsity": s, "batch": batch, "us": round(ms * 1e3, 1),
                        "nonzero_tflops": round(flops / (ms / 1e3) / 1e12, 2),
                        "cudnn_fp32_us": round(cd * 1e3, 1), "speedup_vs_cudnn": round(cd / ms, 3),
                        "plan": plan.describe()})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    ap.add_argument("--steps", type=int, default=50)
    args = ap.parse_args()
    if args.only in (None, "vgg16-fp16"):
        print(json.dumps({"variant": "vgg16-fp16", **vgg16_fp16(args.steps)}), flush=True)
    for mode in ("int8", "cb4"):
        if args.only in (None, f"vgg16-{mode}"):
            print(json.dumps({"variant": f"vgg16-{mode}", **vgg16_quantised(mode, args.steps)}), flush=True)
    if args.only in (None, "sweep"):
        for row in sweep(args.steps):
            print(json.dumps({"variant": "sweep", **row}), flush=True)


if __name__ == "__main__":
    main()
