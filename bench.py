"""Benchmark: pruned VGG-16 CIFAR-10 inference (13 sparse 3x3 convs + ReLU + 5
max-pools, ~93% layer-global sparsity, fp32 bit-exact, batch 256 per GPU) --
BASELINE.json configs[1] -- on N B200s, batch-sharded (weak scaling, no
collective on the hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--global-batch B]

Prints ONE JSON line (rank 0).  ``--gpus N`` without a torchrun environment
re-launches itself under torch.distributed.run with N ranks (one per GPU);
under torchrun the world size must equal N.  Default: weak scaling, 256 images
per rank; ``--global-batch B`` splits B images over the ranks instead (strong
scaling, sharding.ShardedRun).  The e2e leg ends every step with the final
gather of the features (the one collective of the batch-sharded job).
``--impl reference`` times the reference's CPU algorithm (the oracle port in
oracle/, all host threads) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sparse conv layer µs & images/sec vs cuDNN dense at 90–95% sparsity, HBM GB/s"
SPARSITY = 0.93
BATCH = 256
WORKLOAD = ("pruned VGG-16 CIFAR-10 inference: 13 sparse 3x3 conv (ReLU fused) + 5 maxpool, "
            "93% layer-global sparsity, fp32 bit-exact to the reference")


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


# ---------------------------------------------------------------------------
# clocks sampler (NVML) -- runs during the timed region

class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int, period: float = 0.02):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def loop():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for bit, name in self.REASONS.items():
                            if r & bit and bit != 0x1:
                                self.reasons.add(name)
                    except Exception:
                        pass
                    time.sleep(self.period)

            self._t = threading.Thread(target=loop, daemon=True)
            self._t.start()
        except Exception as exc:  # no NVML: report it instead of guessing
            self.reasons.add(f"nvml-unavailable:{type(exc).__name__}")
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# measured peaks

def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


MIX_NAMES = {0: "FMUL+FADD", 1: "FMUL,FMUL+FADD2 (two samples per lane)", 2: "FHFMA"}


def mix_peak(device_index: int, mix: int) -> float:
    """Live CUDA-core peak (nonzero TFLOP/s) of an exact instruction mix on this GPU,
    from the library's probe (usc_peak_mix): 0 = FMUL+FADD, 1 = the fp32 BI64 inner
    loop's FMUL,FMUL+FADD2, 2 = binary16 FHFMA."""
    import ctypes
    from paper_2112_15445_b200 import _lib
    v = ctypes.c_double(0.0)
    _lib.check(_lib.lib().usc_peak_mix(device_index, mix, ctypes.byref(v)), "peak")
    return float(v.value)


TUNED_REL = os.path.join("profiles", "r01_tuned.json")


def ncu_traffic(plan_desc) -> float | None:
    """DRAM bytes per launch of the dominant kernel from the committed ncu captures
    (profiles/traffic.json, written by tools/ncu_summary.py: one entry per captured
    conv plan), if one is for the same tile."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        d = json.load(fh)
    want = json.loads(json.dumps(plan_desc))
    for e in d.get("entries", [d]):
        if e.get("plan") == want:
            return e.get("dram_bytes")
    return None


# ---------------------------------------------------------------------------
# workload

def build_model(batch, device, seed=0):
    import torch
    from paper_2112_15445_b200.models import SparseVGG16, vgg16_rng, vgg16_weights
    rng = vgg16_rng(SPARSITY, seed)
    ws = vgg16_weights(rng, SPARSITY)
    model = SparseVGG16(ws, batch, device=device)
    return model, ws


def layer_stats(model):
    """Algorithmic bytes and nonzero FLOPs per conv launch."""
    out = []
    n = model.batch
    for st in model.steps:
        if st[0] != "conv":
            continue
        li = st[1]
        g = model.geoms[li]
        f = model.filters[li]
        genuine = int(np.count_nonzero(f.weights))
        flops = 2.0 * genuine * g.out_h * g.out_w * n
        byts = (n * g.in_channels * g.input_h * g.input_w * 4 + n * g.out_channels * g.out_h * g.out_w * 4
                + g.out_channels * f.n_nz * 8 + 4 * (g.out_channels + 1))
        out.append(dict(layer=li, flops=flops, bytes=byts))
    return out


def time_per_launch(model, steps=20):
    """Per-launch device time (CUDA events on the launching stream)."""
    import torch
    from paper_2112_15445_b200 import _lib
    L = _lib.lib()
    times = {}
    sp = _lib.stream_ptr()
    for st in model.steps:
        evs = []
        for _ in range(steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(200_000)  # device busy while the launch is enqueued (no host gap)
            a.record()
            if st[0] == "conv":
                _, li, plan, blob, xin, yout, epi = st
                L.usc_conv_forward(_lib.ref(plan), _lib.t_ptr(blob), _lib.t_ptr(xin), _lib.t_ptr(yout),
                                   _lib.ref(epi), sp)
            else:
                _, li, lin, lout, xin, yout = st
                L.usc_maxpool2(_lib.ref(lin), _lib.ref(lout), model.dtype, model.batch, _lib.t_ptr(xin),
                               _lib.t_ptr(yout), sp)
            b.record()
            evs.append((a, b))
        torch.cuda.synchronize()
        times[(st[0], st[1])] = float(np.median([a.elapsed_time(b) for a, b in evs]))
    return times


def cudnn_reference(ws, batch, device, steps=10, tf32=False):
    """The same network on cuDNN dense conv (torch), equal precision (TF32 off) unless tf32."""
    import torch
    from paper_2112_15445_b200.models import VGG16_CIFAR
    torch.backends.cudnn.benchmark = True
    torch.backends.cudnn.allow_tf32 = tf32
    torch.backends.cuda.matmul.allow_tf32 = tf32
    wd = [torch.from_numpy(np.array(w.data)).to(device) for w in ws]
    x = torch.randn(batch, 3, 32, 32, device=device)

    def fwd():
        a, li = x, 0
        for v in VGG16_CIFAR:
            if v == "M":
                a = torch.nn.functional.max_pool2d(a, 2)
            else:
                a = torch.relu(torch.nn.functional.conv2d(a, wd[li], padding=1))
                li += 1
        return a

    for _ in range(3):
        fwd()
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fwd()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    torch.backends.cudnn.allow_tf32 = True
    ms = float(np.median(ts))
    return {"ms_per_step": ms, "images_per_s": batch / ms * 1e3}


def cpu_reference_run(batch_sample, threads, ws_data, seed=1, x=None):
    """The reference's algorithm (oracle port, C) for the same network on a sample
    (seeded N(0,1) images, or the given `x`)."""
    import oracle
    from paper_2112_15445_b200.models import VGG16_CIFAR, vgg16_geometries
    geoms = vgg16_geometries()
    csrs = []
    for w, g in zip(ws_data, geoms):
        gt = (g.in_channels, g.out_channels, 3, 3, g.input_h, g.input_w, (1, 1), (1, 1))
        csrs.append((gt, oracle.build_csr(w, gt)))
    if x is None:
        x = np.random.default_rng(seed).standard_normal((batch_sample, 3, 32, 32)).astype(np.float32)

    def fwd():
        a, li = x, 0
        for v in VGG16_CIFAR:
            if v == "M":
                a = oracle.maxpool2(a)
            else:
                gt, csr = csrs[li]
                a = oracle.relu(oracle.sparse_conv_forward(a, csr, gt, sb=1, threads=threads))
                li += 1
        return a

    return fwd


def run_reference(args, rank, world):
    """--impl reference: the reference CPU implementation (oracle port) on the host cores."""
    if rank != 0:
        return
    import oracle
    from paper_2112_15445_b200.models import vgg16_geometries, vgg16_rng
    from paper_2112_15445_b200.pruning import synthesize_masked_weights
    oracle.build()
    rng = vgg16_rng(SPARSITY)
    ws = [synthesize_masked_weights(g, SPARSITY, rng).data for g in vgg16_geometries()]
    threads = oracle.max_threads()
    sample = int(os.environ.get("REF_SAMPLE", 8))
    fwd = cpu_reference_run(sample, threads, ws)
    for _ in range(args.warmup):
        fwd()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fwd()
    dt = time.perf_counter() - t0
    v = sample * args.steps / dt
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "images/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "per_step_sample": sample, "global_batch": sample},
            "cpu_baseline": {"value": round(v, 3), "unit": "images/s", "cores": threads, "kind": "port",
                             "sample": f"{sample} images per step through the 13-layer trunk "
                                       f"(oracle/oracle.c, C restatement of kernels.py:57-100)"},
            "e2e": {"value": round(v, 3), "unit": "images/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch_ranks(args, script=None):
    """`--gpus N` outside torchrun: re-exec this script (or `script`) under
    torch.distributed.run with N local ranks (127.0.0.1 rendezvous); rank 0 prints."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}",
           os.path.abspath(script or __file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def self_check(model, x_np, ws, samples=8):
    """The first `samples` images of the timed batch through the oracle (the
    reference's algorithm restated in C, the checker only) vs the timed graph's
    output: bitwise equality required (fp32 path)."""
    import oracle
    oracle.build()
    ref = cpu_reference_run(samples, oracle.max_threads(), [w.data for w in ws], x=x_np[:samples])()
    got = model.output().cpu().numpy()[:samples]
    return {"samples": samples, "bitwise": bool(np.array_equal(got, ref)),
            "checker": "oracle/oracle.c (C restatement of kernels.py:57-100, pinned to the reference's golden vectors)"}


def binary16_leg(steps=20):
    """BASELINE configs[2] (and the binary16 VGG-16) in the same run: the networks with the
    committed per-layer dispatch states (profiles/r02_tuned_*_fp16_dispatch.json: sparse /
    tcgen05 backend per conv, tile configurations) next to all-sparse and cuDNN fp16, batch
    256, L2 flushed between steps (tools/bench_variants.py, the fp16 tolerance path)."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import bench_variants as bv
    out = {"note": "binary16 storage, fp32 accumulate; committed dispatch states; timed in this run"}
    v = bv.vgg16_fp16(steps)
    out["vgg16"] = {"all_sparse_images_per_s": v["images_per_s"],
                    "dispatch_images_per_s": v["dispatch"]["images_per_s"],
                    "cudnn_fp16_images_per_s": v["cudnn_fp16_tensor_core"]["images_per_s"],
                    "dispatch_vs_cudnn": v["dispatch"]["speedup_vs_cudnn"],
                    "backends": sorted(set(v["dispatch"]["backends"]))}
    r = bv.resnet50_network("fp16", steps)
    out["resnet50"] = {"all_sparse_images_per_s": r["images_per_s"],
                       "dispatch_images_per_s": r["dispatch"]["images_per_s"],
                       "cudnn_fp16_images_per_s": r["cudnn"]["images_per_s"],
                       "dispatch_vs_cudnn": r["dispatch"]["speedup_vs_cudnn"],
                       "backends": sorted(set(r["dispatch"]["backends"]))}
    return out


def exact_variants_leg(steps=20):
    """BASELINE configs[3] (int8 and 4b/16b codebook VGG-16, bit-exact) and the fp32 ResNet-50
    network vs cuDNN fp32 (TF32 off), committed tiles, in the same run."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import bench_variants as bv
    out = {"note": "bit-exact sparse kernels; committed tiles; timed in this run"}
    for mode in ("int8", "cb4"):
        q = bv.vgg16_quantised(mode, steps)
        out[f"vgg16_{mode}_images_per_s"] = q["images_per_s"]
    r = bv.resnet50_network("fp32", steps)
    out["resnet50_fp32"] = {"images_per_s": r["images_per_s"], "cudnn_fp32_images_per_s": r["cudnn"]["images_per_s"],
                            "speedup_vs_cudnn": r["speedup_vs_cudnn"]}
    return out


def sweep_leg(sparsities=(0.9, 0.95, 0.98)):
    """BASELINE configs[4] at its >= 90% points in the same run: the ResNet-50 layer shapes at
    batch 1024, fp32, each point's committed tile (profiles/r02_tuned_sweep.json), the launch
    that writes the resident BI layout, vs cuDNN fp32 (TF32 off); algorithmic HBM GB/s."""
    import numpy as np
    import torch
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import bench_variants as bv
    from paper_2112_15445_b200 import build_csr
    from paper_2112_15445_b200.engine import ExecConfig, padded_input, plan_for, time_median_cuda
    from paper_2112_15445_b200.pruning import synthesize_masked_weights
    from paper_2112_15445_b200.tensor import ConvGeometry
    tiles = json.load(open(os.path.join(ROOT, "profiles", "r02_tuned_sweep.json")))
    batch, out = 1024, []
    torch.backends.cudnn.benchmark = True
    torch.backends.cudnn.allow_tf32 = False
    for name, (c, d, k, hw) in bv.SWEEP_SHAPES.items():
        g = ConvGeometry(c, d, k, k, hw, hw, padding=(k // 2, k // 2))
        x = torch.randn(batch, c, hw, hw, device="cuda")
        for sp in sparsities:
            key = f"{name}@{sp}"
            if key not in tiles:
                continue
            w = synthesize_masked_weights(g, sp, np.random.default_rng([0, int(sp * 1000)]))
            f = build_csr(w, g)
            plan, blob = plan_for(f, batch, 0, ExecConfig(**tiles[key]), f.weights)
            ms = time_median_cuda(bv._resident_launch(plan, blob, padded_input(x, plan), d, g, batch, torch.float32), 9, 2)
            wd = torch.from_numpy(np.array(w.data)).cuda()
            cd = time_median_cuda(lambda: torch.nn.functional.conv2d(x, wd, padding=k // 2), 9, 2)
            nnz = int(np.count_nonzero(f.weights))
            nbytes = 4.0 * batch * (c + d) * hw * hw + 8.0 * nnz
            out.append({"point": key, "us": round(ms * 1e3, 1), "cudnn_fp32_us": round(cd * 1e3, 1),
                        "speedup_vs_cudnn": round(cd / ms, 3),
                        "nonzero_tflops": round(2.0 * nnz * hw * hw * batch / (ms / 1e3) / 1e12, 2),
                        "hbm_frac": round(nbytes / (ms / 1e3) / 1e9 / bv.measured_hbm_peak(), 3)})
            f._packs.clear()
    return out


def cfg1_leg(device, steps=50, cpu=True):
    """BASELINE configs[0]: one pruned VGG-16 256->256 3x3 layer, 8x8 map, batch 32,
    90% sparsity, fp32 -- the reference's bench_layer comparison (bench.py:98-130):
    device us of the kernel (L2 flushed), the drop-in API with host numpy buffers
    (H2D + pad + kernel + D2H inside the timing), cuDNN dense at equal precision,
    and the reference's CPU algorithm on the host cores."""
    import zlib

    import torch
    import paper_2112_15445_b200 as U
    from paper_2112_15445_b200.engine import _storage_dtype, dtype_of, launch, padded_input, plan_for
    from paper_2112_15445_b200.pruning import synthesize_masked_weights
    g = U.ConvGeometry(256, 256, 3, 3, 8, 8, padding=(1, 1))
    n, sparsity = 32, 0.9
    rng = np.random.default_rng([0, zlib.crc32(b"cfg1-vgg16-256x8"), int(round(sparsity * 1000))])
    w = synthesize_masked_weights(g, sparsity, rng)
    x_np = rng.standard_normal((n, 256, 8, 8)).astype(np.float32)
    filt = U.build_csr(w, g)
    xd = U.DenseTensor4(torch.from_numpy(x_np).to(device))
    cfg = U.autotune_sb(xd, filt, repeats=5, warmup=2)
    plan, blob = plan_for(filt, n, dtype_of(xd.precision), cfg, filt.weights)
    x_pad = padded_input(xd.device(), plan)
    y = torch.empty((n, 256, 8, 8), dtype=_storage_dtype(plan.dtype), device=device)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)

    def dev_time(fn, flush_l2):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(steps):
            if flush_l2:
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(100_000)
            a.record()
            fn()
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        return float(np.median([a.elapsed_time(b) for a, b in ts])) * 1e3

    kern_us = dev_time(lambda: launch(plan, blob, x_pad, y), True)
    kern_warm_us = dev_time(lambda: launch(plan, blob, x_pad, y), False)
    api_dev_us = dev_time(lambda: U.sparse_conv_forward(xd, filt, cfg), True)
    # host cost of one drop-in call (plans cached on the filter): enqueue time per call
    for _ in range(5):
        U.sparse_conv_forward(xd, filt, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        U.sparse_conv_forward(xd, filt, cfg)
    host_us = (time.perf_counter() - t0) / steps * 1e6
    torch.cuda.synchronize()
    # e2e through the reference-facing API: host numpy in, host numpy out
    e2e = []
    for i in range(steps + 3):
        t0 = time.perf_counter()
        out = U.sparse_conv_forward(U.DenseTensor4(x_np), filt, cfg).data
        if i >= 3:
            e2e.append(time.perf_counter() - t0)
    e2e_us = float(np.median(e2e)) * 1e6
    # cuDNN dense on the same masked weights, equal precision (TF32 off) and TF32
    wt = torch.from_numpy(np.array(w.data)).to(device)
    xt = xd.device()
    torch.backends.cudnn.benchmark = True
    cud = {}
    for name, tf32 in (("fp32_tf32_off", False), ("tf32", True)):
        torch.backends.cudnn.allow_tf32 = tf32
        cud[name] = round(dev_time(lambda: torch.nn.functional.conv2d(xt, wt, padding=1), True), 2)
    torch.backends.cudnn.allow_tf32 = True
    genuine = int(np.count_nonzero(filt.weights))
    flops = 2.0 * genuine * 64 * n
    byts = n * 256 * 64 * 4 * 2 + filt.n_nz * 256 * 8 + 4 * 257
    res = {"workload": "VGG-16 256->256 3x3, 8x8 map, pad 1, batch 32, 90% layer-global sparsity, fp32 "
                       "(BASELINE configs[0])",
           "tile": {k: v for k, v in plan.describe().items()},
           "kernel_us": round(kern_us, 2), "kernel_us_l2_warm": round(kern_warm_us, 2),
           "api_device_us": round(api_dev_us, 2), "api_host_us_per_call": round(host_us, 1),
           "e2e_us": round(e2e_us, 1),
           "e2e_path": "sparse_conv_forward(DenseTensor4(host numpy), build_csr(...)).data: pageable H2D, "
                       "pad, kernel, D2H to numpy (wall clock, median)",
           "images_per_s": {"kernel": round(n / kern_us * 1e6, 1), "e2e": round(n / e2e_us * 1e6, 1)},
           "nonzero_tflops": round(flops / kern_us / 1e6, 2), "hbm_gbs": round(byts / kern_us / 1e3, 1),
           "cudnn_us": cud, "speedup_vs_cudnn_fp32": round(cud["fp32_tf32_off"] / kern_us, 2)}
    import oracle
    oracle.build()
    csr = (filt.row_ptr, filt.col_offsets, filt.weights, filt.n_nz)
    gt = (256, 256, 3, 3, 8, 8, (1, 1), (1, 1))
    ref = oracle.sparse_conv_forward(x_np, csr, gt, threads=oracle.max_threads())
    res["parity"] = {"samples": n, "bitwise": bool(np.array_equal(out, ref))}
    if cpu:
        th = oracle.max_threads()
        t0, reps = time.perf_counter(), 0
        while time.perf_counter() - t0 < 5.0 or reps < 2:
            oracle.sparse_conv_forward(x_np, csr, gt, threads=th)
            reps += 1
        cpu_us = (time.perf_counter() - t0) / reps * 1e6
        res["cpu_reference"] = {"us": round(cpu_us, 1), "cores": th, "kind": "port",
                                "sample": f"{reps} full cfg1 calls (32 images), ~5 s"}
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None,
                    help="ranks (one per GPU); without torchrun env, re-launches under torchrun")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--global-batch", type=int, default=None,
                    help="strong scaling: split this many images over the ranks (default: 256 per rank)")
    ap.add_argument("--no-autotune", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cudnn", action="store_true")
    ap.add_argument("--no-cfg1", action="store_true")
    ap.add_argument("--no-binary16", action="store_true",
                    help="skip the variant legs (binary16 dispatcher networks, int8 / cb4 VGG-16, fp32 ResNet-50, "
                         "the >= 90%% sweep points)")
    ap.add_argument("--dump-configs", default=None, help="write the autotuned per-layer tiles (JSON)")
    ap.add_argument("--configs", default=None, help="per-layer tiles (JSON from --dump-configs); no autotune")
    ap.add_argument("--retune", action="store_true",
                    help="autotune the tiles this run instead of loading the committed " + TUNED_REL)
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and (args.gpus or 1) > 1:
        launch_ranks(args)
    rank, local_rank, world = env_rank()
    if args.gpus is not None and args.gpus != world:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started {world} rank(s)")
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_2112_15445_b200.sharding import ShardedRun
    # BENCH_SHARE_GPU=1 + BENCH_DIST_BACKEND=gloo: every rank on cuda:0 -- a test hook that
    # exercises the multi-rank path (launch, barriers, max over ranks, final gather) on a
    # one-GPU box; the numbers of such a run are not a scaling measurement
    gpu = 0 if os.environ.get("BENCH_SHARE_GPU") == "1" else local_rank
    torch.cuda.set_device(gpu)
    device = torch.device("cuda", gpu)
    if world > 1:
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(backend)
    if args.global_batch:
        job = ShardedRun(args.global_batch, rank, world, align=64)
        scaling = "strong"
    else:
        job = ShardedRun.weak(BATCH, rank, world)
        scaling = "weak"
    batch = job.local_batch
    if batch < 1:
        raise SystemExit(f"bench.py: rank {rank} has no images (global batch {job.global_batch})")
    if (not args.configs and not args.retune and not args.no_autotune and batch == BATCH
            and os.path.exists(os.path.join(ROOT, TUNED_REL))):
        args.configs = os.path.join(ROOT, TUNED_REL)  # the committed autotuner result (matches profiles/)

    model, ws = build_model(batch, device)
    if args.configs:
        model.load_tuned_state(json.load(open(args.configs)))
    elif not args.no_autotune:
        model.autotune(repeats=3, warmup=1)
    if args.dump_configs and rank == 0:
        with open(args.dump_configs, "w") as fh:
            json.dump(model.tuned_state(), fh)
    model.capture()
    x_np = np.random.default_rng([1, rank]).standard_normal((batch, 3, 32, 32)).astype(np.float32)
    x_host = torch.from_numpy(x_np).pin_memory()
    x_dev = x_host.to(device)
    model.load_input(x_dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)  # 2x L2

    io_graph = model.capture(io_src=x_dev)  # pad of the resident input + 18 launches + unpack

    def step():  # one pass: pad the resident input into the BI layout, the 18 launches, unpack
        io_graph.replay()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, inputs resident, L2 flushed between steps -----
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(gpu) as clk:
        for a, b in evs:
            flush.zero_()
            a.record()
            step()
            b.record()
        torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = float(np.sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    ms_per_step = total_ms / args.steps
    value = job.global_batch * args.steps / (total_ms / 1e3)
    # the timed graph's own output checked against the oracle on its first images
    parity = self_check(model, x_np, ws) if rank == 0 else None

    # ---- e2e through the public API with host buffers ---------------------------
    e2e_steps = max(10, args.steps // 2)
    gathered = job.world > 1
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    out_rows = job.global_batch if gathered else batch
    # (a) one batch at a time: H2D, forward, final gather, D2H serialised on one stream
    out_host = torch.empty((out_rows, 512, 1, 1), dtype=torch.float32).pin_memory()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(e2e_steps):
        x_dev.copy_(x_host, non_blocking=True)
        out = job.gather(model.forward(x_dev)) if gathered else model.forward(x_dev)
        if rank == 0:
            out_host.copy_(out, non_blocking=True)
    b.record()
    b.synchronize()
    e2e_serial_ms = a.elapsed_time(b)
    # (b) the streaming API: every step still moves its input H2D and its features D2H,
    # overlapped with the neighbouring steps' compute (SparseVGG16.stream_forward); at N>1
    # each step's features are gathered to rank 0 before the D2H
    x_hosts = [torch.from_numpy(np.random.default_rng([2, rank, i]).standard_normal(
        (batch, 3, 32, 32)).astype(np.float32)).pin_memory() for i in range(4)]
    x_seq = [x_hosts[i % 4] for i in range(e2e_steps)]
    out_seq = [torch.empty((out_rows, 512, 1, 1), dtype=torch.float32).pin_memory()
               for _ in range(e2e_steps)]
    collect = None
    if gathered:
        def collect(t):
            full = job.gather(t)
            return full if rank == 0 else None
    model.stream_forward(x_seq[:2], out_seq[:2], collect=collect).synchronize()  # warm streams / buffers
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    model.stream_forward(x_seq, out_seq, collect=collect)
    b.record()
    b.synchronize()
    e2e_ms = a.elapsed_time(b)
    if world > 1:
        t = torch.tensor([e2e_ms, e2e_serial_ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms, e2e_serial_ms = float(t[0].item()), float(t[1].item())
    e2e = {"value": round(job.global_batch * e2e_steps / (e2e_ms / 1e3), 1), "unit": "images/s",
           "h2d_bytes_per_step": int(job.global_batch * 3 * 32 * 32 * 4),
           "d2h_bytes_per_step": int(out_rows * 512 * 4),
           "path": "SparseVGG16.stream_forward: per step pinned H2D of the input, pad + CUDA graph, "
                   + ("all_gather of the features to rank 0 (sharding.ShardedRun.gather), " if gathered else "")
                   + "D2H of the features, transfers overlapped with neighbouring steps on two copy streams",
           "serial": {"value": round(job.global_batch * e2e_steps / (e2e_serial_ms / 1e3), 1),
                      "path": "SparseVGG16.forward with H2D" + (", gather" if gathered else "")
                              + " and D2H serialised on one stream"}}

    # ---- per-launch breakdown, roofline of the dominant kernel --------------------
    per = time_per_launch(model)
    stats = {s["layer"]: s for s in layer_stats(model)}
    conv_ms = {li: ms for (k, li), ms in per.items() if k == "conv"}
    dom = max(conv_ms, key=conv_ms.get)
    dom_ms = conv_ms[dom]
    hbm_peak, peak_kind = measured_peaks()
    plan = next(st[2] for st in model.steps if st[0] == "conv" and st[1] == dom)
    mix = 1 if plan.kernel in (3, 4) and plan.NS == 64 else 0
    core_peak = mix_peak(gpu, mix)
    s = stats[dom]
    achieved_gbs = s["bytes"] / (dom_ms / 1e3) / 1e9
    achieved_tf = s["flops"] / (dom_ms / 1e3) / 1e12
    g = model.geoms[dom]
    ai = s["flops"] / s["bytes"]
    # attainable roof = min(core peak, AI * HBM): every 3x3 layer here is far right of the
    # ridge, so the bound is the CUDA-core issue rate of the kernel's own exact mix (no
    # tensor cores: the contraction is unstructured-sparse and must round like the reference)
    roofline = {"bound": "fp32-cuda-core" if ai * hbm_peak / 1e3 > core_peak else "hbm",
                "achieved": round(achieved_tf, 3), "peak": round(core_peak, 2), "unit": "TFLOP/s",
                "frac": round(achieved_tf / core_peak, 4),
                "traffic": ncu_traffic(plan.describe()),
                "peak_source": f"live {MIX_NAMES[mix]} probe on this GPU (usc_peak_mix {mix}: the dominant "
                               f"kernel's own multiply/add instruction mix)",
                "kernel": f"k_bi conv layer {dom} ({g.in_channels}->{g.out_channels}, {g.input_h}x{g.input_w})",
                "kernel_share_of_step": round(dom_ms / sum(per.values()), 3),
                "launch_us": round(dom_ms * 1e3, 2),
                "algorithmic_flops_per_launch": s["flops"], "algorithmic_bytes_per_launch": s["bytes"],
                "arith_intensity_flop_per_byte": round(ai, 1),
                "hbm": {"achieved": round(achieved_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                        "frac": round(achieved_gbs / hbm_peak, 4), "peak_source": peak_kind},
                "plan": plan.describe()}
    # the roof this kernel actually meets: every MAC reads one staged fp32 x
    # value through the 128 B/clk/SM shared-memory port -> 32 MAC/clk/SM
    clk_mhz = clk.summary().get("sm_mhz") or 1965.0
    n_sm = torch.cuda.get_device_properties(device).multi_processor_count
    smem_peak_tf = 32 * 2 * n_sm * clk_mhz * 1e6 / 1e12
    roofline["smem"] = {"achieved": round(achieved_tf, 3), "peak": round(smem_peak_tf, 2), "unit": "TFLOP/s",
                        "frac": round(achieved_tf / smem_peak_tf, 4),
                        "peak_source": f"128 B/clk/SM shared-memory loads = 32 fp32 MAC/clk/SM x {n_sm} SMs x "
                                       f"{clk_mhz:.0f} MHz (median SM clock under load)",
                        "achieved_smem_gbs": round(s["flops"] / 2 * 4 / (dom_ms / 1e3) / 1e9, 1)}
    layers = [{"layer": li, "us": round(conv_ms[li] * 1e3, 1),
               "nonzero_tflops": round(stats[li]["flops"] / (conv_ms[li] / 1e3) / 1e12, 2),
               "gbs": round(stats[li]["bytes"] / (conv_ms[li] / 1e3) / 1e9, 1)} for li in sorted(conv_ms)]

    line = None
    if rank == 0:
        cudnn = None
        if not args.no_cudnn:
            cudnn = {"fp32_tf32_off": cudnn_reference(ws, batch, device),
                     "tf32": cudnn_reference(ws, batch, device, tf32=True)}
        cfg1 = None if args.no_cfg1 else cfg1_leg(device, cpu=not args.no_cpu_baseline and world == 1)
        def aux(leg):  # an auxiliary leg never costs the headline line
            if args.no_binary16 or world > 1:
                return None
            try:
                return leg()
            except Exception as exc:  # noqa: BLE001 -- reported in the line, not raised
                return {"error": f"{type(exc).__name__}: {exc}"[:300]}
        b16, exact, sweep = aux(binary16_leg), aux(exact_variants_leg), aux(sweep_leg)
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            import oracle
            oracle.build()
            threads = oracle.max_threads()
            sample = 8
            fwd = cpu_reference_run(sample, threads, [w.data for w in ws])
            fwd()
            t0 = time.perf_counter()
            reps = 0
            while time.perf_counter() - t0 < 10.0:
                fwd()
                reps += 1
            dt = time.perf_counter() - t0
            cpu = {"value": round(sample * reps / dt, 3), "unit": "images/s", "cores": threads,
                   "kind": "port", "sample": f"{reps}x{sample} images through the same 13-conv trunk "
                                             f"(oracle/oracle.c), ~10 s of host work"}
        line = {"impl": "ours", "metric": METRIC, "value": round(value, 1), "unit": "images/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
                "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded N(0,1) inputs, random-init pruned weights)",
                "config": {"workload": WORKLOAD, "model": "vgg16-cifar10", "global_batch": job.global_batch,
                           "per_gpu_batch": batch, "seq_len": None, "sparsity": SPARSITY,
                           "parallelism": f"dp{world} (batch-sharded, no collective in the timed step; "
                                          f"final all_gather in the e2e leg)",
                           "l2": "flushed (256 MiB write) between timed steps",
                           "timed_step": "one CUDA graph: input pad into the BI64 layout + 13 conv + pools + "
                                         "output unpack, device-resident input",
                           "cuda_graph": True,
                           "tiles": (os.path.relpath(args.configs, ROOT) + " (committed autotuner result)")
                           if args.configs else "autotuned this run"},
                "e2e": e2e, "gpu_launches": args.steps * (model.launches_per_forward + 2),
                "parity": parity,
                "roofline": roofline, "layers": layers, "cudnn": cudnn, "cpu_baseline": cpu,
                "cfg1": cfg1, "binary16": b16, "exact_variants": exact, "sweep": sweep, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
