"""One tensor-core dense conv launch (usc_dense_conv_f16, batch 256, binary16, BI64)
between cudaProfilerStart/Stop, for an ncu capture:
    ncu --set full --profile-from-start off -c 1 -o gpurun_out/tc python tools/ncu_tc.py [C,D,k,s,hw[,res|pool]]
Default: the VGG conv3_x shape 256->256 3x3 8x8.  `pool`: conv + ReLU + 2x2 pool in one
launch; otherwise the automatic tile with its split-K workspace when the shape splits.  Writes gpurun_out/tc.json (the MAC and
algorithmic-byte counts ncu_summary.py derives rates from)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2112_15445_b200 import _lib  # noqa: E402
from paper_2112_15445_b200.dense import dense_conv, dense_conv_pool, dense_workspace, pack_weights  # noqa: E402

spec = (sys.argv[1] if len(sys.argv) > 1 else "256,256,3,1,8").split(",")
C, D, k, s, hw = (int(v) for v in spec[:5])
use_res = len(spec) > 5 and spec[5] == "res"
use_pool = len(spec) > 5 and spec[5] == "pool"
n = 256
halo = k // 2
ho = (hw + 2 * halo - k) // s + 1
x = torch.randn(n, C, hw, hw, device="cuda").half()
w = (torch.randn(D, C, k, k, device="cuda") / (k * k * C) ** 0.5).half()
xl = _lib.act_layout(C, hw, hw, halo, halo, 2, 64)
xb = torch.zeros(xl.elems(n), dtype=torch.float16, device="cuda")
_lib.check(_lib.lib().usc_pad_input(_lib.ref(xl), _lib.USC_F16, n, _lib.t_ptr(x), _lib.t_ptr(xb), _lib.stream_ptr()))
yl = _lib.act_layout(D, ho // 2, ho // 2, 1, 1, 2, 64) if use_pool else _lib.act_layout(D, ho, ho, 1, 1, 2, 64)
yb = torch.zeros(yl.elems(n), dtype=torch.float16, device="cuda")
rl = rb = None
if use_res:
    rl = _lib.act_layout(D, ho, ho, 0, 0, 2, 64)
    rb = torch.randn(rl.elems(n), device="cuda").half()
wp = pack_weights(w)
ws = dense_workspace(C, D, k, s, n, xl, use_res)


def run():
    if use_pool:
        dense_conv_pool(wp, C, D, n, xb, xl, yb, yl)
    else:
        dense_conv(wp, C, D, k, s, n, xb, xl, yb, yl, rb, rl, True, None, ws)


run()
torch.cuda.synchronize()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
macs = n * D * ho * ho * C * k * k
json.dump({"spec": f"tc:{C}x{D}x{k}x{k}/s{s}@{hw}x{hw},b{n}" + (",shortcut" if use_res else "") +
                   (",pool" if use_pool else "") + (",split-K" if ws is not None else ""),
           "plan": {"kernel": "k_dtc (TWP and window mode chosen by the host)"},
           "nonzero_macs": macs,
           "algorithmic_bytes": 2 * n * (C * hw * hw + D * ho * ho * (2 if use_res else (0.25 if use_pool else 1))) +
           2 * D * C * k * k},
          open(os.path.join(ROOT, "gpurun_out", "tc.json"), "w"))
torch.cuda.profiler.start()
run()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
