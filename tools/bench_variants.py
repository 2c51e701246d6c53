"""Secondary configurations of BASELINE.json next to cuDNN on the same B200
(the headline fp32 VGG-16 line is bench.py's):

  * vgg16-fp16  -- pruned VGG-16 CIFAR-10, 93% sparsity, BINARY16 (binary16 storage,
    fp32 accumulate, binary16 hook), batch 256, vs cuDNN fp16 (channels_last, tensor
    cores) on the same masked weights;
  * vgg16-int8 / vgg16-cb4 -- the quantised networks of configs[3];
  * resnet50-fp16 -- configs[2]: the 53 convs of ResNet-50 CIFAR at 90%, BINARY16, vs
    cuDNN fp16 on tensor cores (layer sum);
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


def measured_hbm_peak() -> float:
    """HBM GB/s from the driver-written MEASURED_PEAKS.json, else the profiling
    guide's B200 fallback."""
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p)).get("hbm_gbs", 6650.0))
    return 6650.0


OUT_DIR = os.environ.get("TUNED_OUT", "gpurun_out")


def dump_state(name, state):
    """Tuned tiles of a variant -> <TUNED_OUT>/r02_tuned_<name>.json (committed under
    profiles/ so the -m gpu parity tests run exactly the benchmarked plans)."""
    os.makedirs(OUT_DIR, exist_ok=True)
    with open(os.path.join(OUT_DIR, f"r02_tuned_{name}.json"), "w") as fh:
        json.dump(state, fh)


def load_state(name):
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                     f"r02_tuned_{name}.json")
    if os.environ.get("RETUNE") or not os.path.exists(p):
        return None
    if name.endswith("_dispatch") and os.environ.get("RETUNE_DISPATCH"):
        return None
    with open(p) as fh:
        return json.load(fh)


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
    st = load_state("vgg16_fp16")
    if st:
        m.load_tuned_state(st)
    else:
        m.autotune(repeats=3, warmup=1)
        dump_state("vgg16_fp16", m.tuned_state())
    m.capture()
    m.load_input(torch.randn(batch, 3, 32, 32, device="cuda").half())
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    ms = timed(lambda: m.graph.replay(), steps, flush)
    cd = timed(cudnn_vgg(ws, batch, torch.float16, channels_last=True), steps, flush)
    disp = dispatched(m, "vgg16_fp16", steps, flush, cd)
    return {"config": "pruned VGG-16 CIFAR-10 93% BINARY16, batch 256", "dtype": "f16 storage, f32 accumulate",
            "images_per_s": round(batch / (ms / 1e3), 1), "ms_per_step": round(ms, 4),
            "cudnn_fp16_tensor_core": {"images_per_s": round(batch / (cd / 1e3), 1), "ms_per_step": round(cd, 4)},
            "speedup_vs_cudnn": round(cd / ms, 3), "dispatch": disp}


def dispatched(m, name, steps, flush, cudnn_ms):
    """The per-layer sparse/cuDNN dispatcher (backend_config, ref bench.py:212-227) on a
    binary16 network: argmin per conv on the network's buffers, then the mixed network
    timed as one CUDA graph (fp16 tolerance path, tests/test_gpu_dispatch.py)."""
    st = load_state(f"{name}_dispatch")
    if st:
        m.load_tuned_state(st)
    else:
        m.autotune_backends(repeats=5, warmup=2)
        dump_state(f"{name}_dispatch", m.tuned_state())
    m.capture()
    ms = timed(lambda: m.graph.replay(), steps, flush)
    backends = list(m.backends)
    out = {"images_per_s": round(m.batch / (ms / 1e3), 1), "ms_per_step": round(ms, 4),
           "speedup_vs_cudnn": round(cudnn_ms / ms, 3), "sparse_layers": backends.count("sparse"),
           "dense_layers": backends.count("dense"), "backends": backends,
           "tc_layers": backends.count("tc"),
           "rule": "network-level search over per-conv argmins of sparse / tensor-core / cuDNN and block splits; "
                   "then the tensor-core tile search (pixels per tile, K splits) per conv"}
    if hasattr(m, "backend_search"):
        out["pick"], out["search"] = m.backend_pick, m.backend_search
    if hasattr(m, "backend_times"):
        out["per_conv_ms"] = {str(k): {a: (round(b, 4) if b is not None else None) for a, b in v.items()}
                              for k, v in m.backend_times.items()}
    out["tc_tiles"] = {str(k): list(v) for k, v in getattr(m, "tc_cfg", {}).items() if tuple(v) != (0, 0)}
    if hasattr(m, "tc_search"):
        out["tc_search"] = m.tc_search
    return out


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
    st = load_state(f"vgg16_{mode}")
    if st:
        m.load_tuned_state(st)
    else:
        m.autotune(repeats=3, warmup=1)
        dump_state(f"vgg16_{mode}", m.tuned_state())
    m.capture()
    m.load_input(x if mode == "int8" else x.half())
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    ms = timed(lambda: m.graph.replay(), steps, flush)
    return {"config": f"pruned VGG-16 CIFAR-10 93% {mode}, batch 256",
            "dtype": {"int8": "int8 codes (staged binary16), exact fp32 accumulate",
                      "cb4": "4-bit codebook weights, binary16 activations"}[mode],
            "images_per_s": round(batch / (ms / 1e3), 1), "ms_per_step": round(ms, 4)}


def _resident_launch(plan, blob, xp, d, g, batch, dtype):
    """One layer launch writing the engine's resident layout (the plan's interleave,
    zero halo of 1 as the next 3x3 layer reads) -- what a network layer does; the
    plain-NCHW output of sparse_conv_forward is a host-facing convenience."""
    from paper_2112_15445_b200 import _lib
    from paper_2112_15445_b200.engine import launch
    il = plan.in_.interleave
    lay = _lib.act_layout(d, g.out_h, g.out_w, 1, 1, 4 if dtype == torch.float32 else 2, il)
    y = torch.zeros(lay.elems(batch), dtype=dtype, device="cuda")
    epi = _lib.Epilogue()
    epi.scale, epi.out_padded, epi.out = 1.0, 1, lay
    return lambda: launch(plan, blob, xp, y, epi)


def resnet50_cifar_convs():
    """(name, geometry kwargs, torch stride/padding, count) for the 53 convs of ResNet-50
    on 32x32 inputs (3x3 stem, no max-pool, bottleneck stages at 32/16/8/4, stride on the
    3x3 and the projection).  Stride-2 layers use the reference's exact geometries
    (ConvGeometry rejects 32 -> 16 with pad 1, tensor.py:186-190): the 3x3 reads a
    top/left pre-padded 33x33 input with pad 0, the 1x1 projection a 31x31 crop."""
    out = [("stem-3x3-3x64-32", dict(c=3, d=64, k=3, hw=32, s=1, p=1), 1)]
    c_in, hw = 64, 32
    for width, blocks, stride in ((64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2)):
        for b in range(blocks):
            s = stride if b == 0 else 1
            out.append((f"1x1-{c_in}x{width}-{hw}", dict(c=c_in, d=width, k=1, hw=hw, s=1, p=0), 1))
            out.append((f"3x3-{width}x{width}-{hw}-s{s}", dict(c=width, d=width, k=3, hw=hw, s=s, p=1), 1))
            hw_out = hw // s
            out.append((f"1x1-{width}x{4 * width}-{hw_out}", dict(c=width, d=4 * width, k=1, hw=hw_out, s=1, p=0), 1))
            if b == 0:
                out.append((f"proj-1x1-{c_in}x{4 * width}-{hw}-s{s}", dict(c=c_in, d=4 * width, k=1, hw=hw, s=s, p=0), 1))
            c_in, hw = 4 * width, hw_out
    merged = {}
    for name, kw, n in out:
        merged.setdefault(name, [kw, 0])[1] += n
    return [(k, v[0], v[1]) for k, v in merged.items()]


def resnet50_fp16(batch=256, sparsity=0.9):
    """cfg3: per-layer binary16 sparse conv vs cuDNN fp16 (tensor cores), summed over the
    53 convs of ResNet-50 CIFAR (layer-sum; residual adds and the classifier excluded)."""
    from paper_2112_15445_b200 import DenseTensor4, PrecisionMode, autotune_sb, build_csr
    from paper_2112_15445_b200 import PrecisionMode
    from paper_2112_15445_b200.engine import launch, padded_input, plan_for, tile_candidates, time_median_cuda
    from paper_2112_15445_b200.pruning import synthesize_masked_weights
    from paper_2112_15445_b200.tensor import ConvGeometry
    F16 = PrecisionMode.BINARY16
    rows, tot_s, tot_c, tot_d, n_convs = [], 0.0, 0.0, 0.0, 0
    torch.backends.cudnn.benchmark = True
    for name, kw, count in resnet50_cifar_convs():
        c, d, k, hw, s, p = kw["c"], kw["d"], kw["k"], kw["hw"], kw["s"], kw["p"]
        if s == 2 and k == 3:
            g = ConvGeometry(c, d, 3, 3, hw + 1, hw + 1, stride=(2, 2))
        elif s == 2:
            g = ConvGeometry(c, d, 1, 1, hw - 1, hw - 1, stride=(2, 2))
        else:
            g = ConvGeometry(c, d, k, k, hw, hw, padding=(p, p))
        rng = np.random.default_rng([0, len(name), c, d, hw])
        w = synthesize_masked_weights(g, sparsity, rng, F16)
        f = build_csr(w, g)
        x = torch.randn(batch, c, g.input_h, g.input_w, device="cuda").half()
        cfg = autotune_sb(DenseTensor4(x, F16), f, repeats=3, warmup=1)
        plan, blob = plan_for(f, batch, 1, cfg, f.weights)
        xp = padded_input(x, plan)
        ms = time_median_cuda(_resident_launch(plan, blob, xp, d, g, batch, torch.float16), 9, 2)
        xt = torch.randn(batch, c, hw, hw, device="cuda").half().contiguous(memory_format=torch.channels_last)
        wt = torch.from_numpy(np.array(w.data)).cuda().half().contiguous(memory_format=torch.channels_last)
        cd = time_median_cuda(lambda: torch.nn.functional.conv2d(xt, wt, stride=s, padding=p), 9, 2)
        backend = "sparse" if ms < cd else "dense"  # layer_bench.backend_config: ties -> dense
        rows.append({"layer": name, "count": count, "us": round(ms * 1e3, 1), "cudnn_fp16_us": round(cd * 1e3, 1),
                     "kernel": plan.describe()["kernel"], "backend": backend})
        tot_s += ms * count
        tot_c += cd * count
        tot_d += min(ms, cd) * count
        n_convs += count
    return {"config": f"pruned ResNet-50 CIFAR {int(sparsity * 100)}% BINARY16, batch {batch}, 53-conv layer sum",
            "convs": n_convs, "sparse_ms": round(tot_s, 4), "cudnn_fp16_ms": round(tot_c, 4),
            "images_per_s_conv_only": round(batch / (tot_s / 1e3), 1),
            "cudnn_images_per_s_conv_only": round(batch / (tot_c / 1e3), 1),
            "speedup_vs_cudnn": round(tot_c / tot_s, 3),
            "dispatch": {"ms": round(tot_d, 4), "images_per_s_conv_only": round(batch / (tot_d / 1e3), 1),
                         "rule": "per-layer argmin of sparse vs cuDNN, ties to dense (backend_config, "
                                 "ref bench.py:212-227)",
                         "sparse_layers": sum(r["count"] for r in rows if r["backend"] == "sparse")},
            "layers": rows}


SWEEP_SHAPES = {"r50-3x3-64x32": (64, 64, 3, 32), "r50-3x3-256x8": (256, 256, 3, 8),
                "r50-1x1-64x256-32": (64, 256, 1, 32), "r50-1x1-256x64-32": (256, 64, 1, 32)}


def resnet50_network(prec_name, steps, batch=256, sparsity=0.9):
    """configs[2] as a network: the 53-conv ResNet-50 CIFAR trunk (residual adds and ReLU
    fused) on the engine, autotuned + CUDA graph, vs the same network on cuDNN (torch,
    channels_last; fp16 on tensor cores, fp32 with TF32 off)."""
    from paper_2112_15445_b200 import PrecisionMode
    from paper_2112_15445_b200.resnet import STAGES, SparseResNet50, resnet50_layers, resnet50_weights
    prec = PrecisionMode.BINARY16 if prec_name == "fp16" else PrecisionMode.BINARY32
    tdt = torch.float16 if prec_name == "fp16" else torch.float32
    ws = resnet50_weights(sparsity, 0, prec)
    m = SparseResNet50(ws, batch, precision=prec)
    st = load_state(f"resnet50_{prec_name}")
    if st:
        m.load_tuned_state(st)
    else:
        m.autotune()
        dump_state(f"resnet50_{prec_name}", m.tuned_state())
    m.capture()
    m.load_input(torch.randn(batch, 3, 32, 32, device="cuda").to(tdt))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    ms = timed(lambda: m.graph.replay(), steps, flush)
    # cuDNN: torch semantics (stride-2 3x3 pad 1, stride-2 1x1) on the same masked weights
    torch.backends.cudnn.benchmark = True
    torch.backends.cudnn.allow_tf32 = False
    cl = torch.channels_last
    wt = [torch.from_numpy(np.array(w.data)).cuda().to(tdt).contiguous(memory_format=cl) for w in ws]
    layers = resnet50_layers()
    xt = torch.randn(batch, 3, 32, 32, device="cuda", dtype=tdt).contiguous(memory_format=cl)
    F = torch.nn.functional

    def fwd():
        a = F.relu(F.conv2d(xt, wt[0], padding=1))
        li = 1
        for width, blocks, stride in STAGES:
            for b in range(blocks):
                s = stride if b == 0 else 1
                h = F.relu(F.conv2d(a, wt[li]))
                h = F.relu(F.conv2d(h, wt[li + 1], stride=s, padding=1))
                li += 2
                if b == 0:
                    sc = F.conv2d(a, wt[li], stride=s)
                    li += 1
                else:
                    sc = a
                a = F.relu(F.conv2d(h, wt[li]) + sc)
                li += 1
        return a
    cd = timed(fwd, steps, flush)
    out = {"config": f"pruned ResNet-50 CIFAR {int(sparsity * 100)}% {prec_name}, batch {batch}, full network "
                     f"(53 sparse convs, residual adds)",
           "images_per_s": round(batch / (ms / 1e3), 1), "ms_per_step": round(ms, 4),
           "cudnn": {"images_per_s": round(batch / (cd / 1e3), 1), "ms_per_step": round(cd, 4),
                     "kind": "fp16 tensor cores" if prec_name == "fp16" else "fp32, TF32 off"},
           "speedup_vs_cudnn": round(cd / ms, 3)}
    if prec_name == "fp16":
        out["dispatch"] = dispatched(m, "resnet50_fp16", steps, flush, cd)
    return out


def sweep(steps, shapes=None, sparsities=(0.5, 0.7, 0.9, 0.95, 0.98)):
    from paper_2112_15445_b200 import DenseTensor4, autotune_sb, build_csr, sparse_conv_forward
    from paper_2112_15445_b200 import PrecisionMode
    from paper_2112_15445_b200.engine import launch, padded_input, plan_for, tile_candidates, time_median_cuda
    from paper_2112_15445_b200.pruning import synthesize_masked_weights
    from paper_2112_15445_b200.tensor import ConvGeometry
    import dataclasses
    out, tiles = [], {}
    batch = 1024
    for name, (c, d, k, hw) in SWEEP_SHAPES.items():
        if shapes and name not in shapes:
            continue
        g = ConvGeometry(c, d, k, k, hw, hw, padding=(k // 2, k // 2))
        x = torch.randn(batch, c, hw, hw, device="cuda")
        for s in sparsities:
            rng = np.random.default_rng([0, int(s * 1000)])
            w = synthesize_masked_weights(g, s, rng)
            f = build_csr(w, g)
            xd = DenseTensor4(x)
            cfg = autotune_sb(xd, f, repeats=3, warmup=1)
            # the resident (BI output) launch is what a network runs: search its tile too
            pads, best = {}, None
            for cand in [cfg] + tile_candidates(g, batch, [1], PrecisionMode.BINARY32, (3,)):
                try:
                    p_, b_ = plan_for(f, batch, 0, cand, f.weights)
                except ValueError:
                    continue
                if p_.kernel not in (3, 4):
                    continue
                key = (p_.in_.interleave, p_.in_.hp, p_.in_.ws)
                if key not in pads:
                    pads[key] = padded_input(x, p_)
                t = time_median_cuda(_resident_launch(p_, b_, pads[key], d, g, batch, torch.float32), 3, 1)
                if best is None or t < best[0]:
                    best = (t, cand)
                f._packs.clear()
            pick = best[1] if best else cfg
            tiles[f"{name}@{s}"] = dataclasses.asdict(pick)
            plan, blob = plan_for(f, batch, 0, pick, f.weights)
            xp = pads.get((plan.in_.interleave, plan.in_.hp, plan.in_.ws)) if plan.kernel in (3, 4) else None
            xp = xp if xp is not None else padded_input(x, plan)
            ms = time_median_cuda(_resident_launch(plan, blob, xp, d, g, batch, torch.float32), 9, 2)
            y = torch.empty(batch, d, hw, hw, device="cuda")
            ms_plain = time_median_cuda(lambda: launch(plan, blob, xp, y), 9, 2)
            torch.backends.cudnn.benchmark = True
            torch.backends.cudnn.allow_tf32 = False
            wd = torch.from_numpy(np.array(w.data)).cuda()
            cd = time_median_cuda(lambda: torch.nn.functional.conv2d(x, wd, padding=k // 2), 9, 2)
            genuine = int(np.count_nonzero(f.weights))
            flops = 2.0 * genuine * hw * hw * batch
            # algorithmic bytes: input + output once + 8 B per entry
            nbytes = 4.0 * batch * (c + d) * hw * hw + 8.0 * genuine
            out.append({"layer": name, "sparsity": s, "batch": batch, "us": round(ms * 1e3, 1),
                        "us_plain_nchw_out": round(ms_plain * 1e3, 1),
                        "nonzero_tflops": round(flops / (ms / 1e3) / 1e12, 2),
                        "hbm_gbs": round(nbytes / (ms / 1e3) / 1e9, 1),
                        "hbm_frac": round(nbytes / (ms / 1e3) / 1e9 / measured_hbm_peak(), 3),
                        "cudnn_fp32_us": round(cd * 1e3, 1), "speedup_vs_cudnn": round(cd / ms, 3),
                        "plan": plan.describe()})
    if not shapes:
        dump_state("sweep", tiles)
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
    for pn in ("fp16", "fp32"):
        if args.only in (None, f"resnet50-net-{pn}"):
            print(json.dumps({"variant": f"resnet50-net-{pn}", **resnet50_network(pn, args.steps)}), flush=True)
    if args.only in (None, "resnet50-fp16"):
        print(json.dumps({"variant": "resnet50-fp16", **resnet50_fp16()}), flush=True)
    if args.only in (None, "sweep") or (args.only or "").startswith("sweep:"):
        shapes = args.only.split(":", 1)[1].split(",") if args.only and ":" in args.only else None
        for row in sweep(args.steps, shapes):
            print(json.dumps({"variant": "sweep", **row}), flush=True)


if __name__ == "__main__":
    main()
