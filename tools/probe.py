"""Per-layer timing probe: VGG-16 CIFAR b256 93% fp32 -- sparse kernel (default
and autotuned tiles) vs cuDNN dense fp32 (TF32 off) on the same GPU."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2112_15445_b200 as U
from paper_2112_15445_b200.models import SparseVGG16, vgg16_rng, vgg16_weights
from paper_2112_15445_b200.engine import time_median_cuda, launch

torch.backends.cudnn.benchmark = True
torch.backends.cudnn.allow_tf32 = False
torch.backends.cuda.matmul.allow_tf32 = False
B = int(os.environ.get("B", 256))
S = float(os.environ.get("S", 0.93))
prec = U.PrecisionMode.BINARY16 if os.environ.get("F16") else U.PrecisionMode.BINARY32
rng = vgg16_rng(S)
ws = vgg16_weights(rng, S, prec)
x = torch.randn(B, 3, 32, 32, device="cuda")
if prec is U.PrecisionMode.BINARY16:
    x = x.half()
m = SparseVGG16(ws, B, prec)
m.forward(x); torch.cuda.synchronize()
res = []
def layer_times(m):
    out = []
    for st in m.steps:
        if st[0] == "conv":
            _, li, plan, blob, xin, yout, epi = st
            ms = time_median_cuda(lambda: launch(plan, blob, xin, yout, epi), 9, 3)
            g = m.geoms[li]
            nnz = int(np.count_nonzero(m.filters[li].weights))
            fl = 2.0 * nnz * g.out_h * g.out_w * B
            out.append(dict(layer=li, C=g.in_channels, D=g.out_channels, hw=g.input_h, n_nz=m.filters[li].n_nz,
                            us=ms * 1e3, tflops=fl / ms / 1e9, plan=plan.describe()))
    return out
t0 = layer_times(m)
tot = time_median_cuda(lambda: m.run(), 9, 3)
print("default total ms", tot, "img/s", B / tot * 1e3)
for r in t0: print(json.dumps(r))
t = time.time(); cfgs = m.autotune(repeats=3, warmup=1); print("autotune s", time.time() - t)
t1 = layer_times(m)
tot1 = time_median_cuda(lambda: m.run(), 9, 3)
print("tuned total ms", tot1, "img/s", B / tot1 * 1e3)
for r in t1: print(json.dumps(r))
m.capture()
tg = time_median_cuda(lambda: m.graph.replay(), 9, 3)
print("graph total ms", tg, "img/s", B / tg * 1e3)
# cuDNN dense
dt = torch.float16 if prec is U.PrecisionMode.BINARY16 else torch.float32
tot_c = 0
for li, g in enumerate(m.geoms):
    xi = torch.randn(B, g.in_channels, g.input_h, g.input_w, device="cuda", dtype=dt)
    wi = torch.from_numpy(ws[li].data).cuda().to(dt)
    if dt == torch.float16:
        xi = xi.to(memory_format=torch.channels_last); wi = wi.to(memory_format=torch.channels_last)
    f = lambda: torch.nn.functional.conv2d(xi, wi, padding=1)
    ms = time_median_cuda(f, 9, 3)
    tot_c += ms
    print("cudnn layer", li, ms * 1e3, "us")
print("cudnn conv total ms", tot_c, "img/s", B / tot_c * 1e3)
