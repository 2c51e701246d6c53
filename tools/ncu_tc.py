"""One tensor-core dense conv launch (VGG conv3_x shape: 256->256 3x3, 8x8, batch 256,
binary16, BI64) between cudaProfilerStart/Stop, for an ncu capture:
    ncu --set full --profile-from-start off -c 1 -o gpurun_out/tc python tools/ncu_tc.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2112_15445_b200 import _lib  # noqa: E402
from paper_2112_15445_b200.dense import dense_conv, pack_weights  # noqa: E402

n, C, D, hw = 256, 256, 256, 8
x = torch.randn(n, C, hw, hw, device="cuda").half()
w = (torch.randn(D, C, 3, 3, device="cuda") / (9 * C) ** 0.5).half()
xl = _lib.act_layout(C, hw, hw, 1, 1, 2, 64)
xb = torch.zeros(xl.elems(n), dtype=torch.float16, device="cuda")
_lib.check(_lib.lib().usc_pad_input(_lib.ref(xl), _lib.USC_F16, n, _lib.t_ptr(x), _lib.t_ptr(xb), _lib.stream_ptr()))
yl = _lib.act_layout(D, hw, hw, 1, 1, 2, 64)
yb = torch.zeros(yl.elems(n), dtype=torch.float16, device="cuda")
wp = pack_weights(w)
dense_conv(wp, C, D, 3, 1, n, xb, xl, yb, yl)
torch.cuda.synchronize()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
macs = n * D * hw * hw * C * 9
json.dump({"spec": "tc:256x256x3x3@8x8,b256", "plan": {"kernel": "k_dtc (TWP and window mode chosen by the host)"},
           "nonzero_macs": macs,
           "algorithmic_bytes": 2 * n * (C + D) * hw * hw + 2 * D * C * 9},
          open(os.path.join(ROOT, "gpurun_out", "tc.json"), "w"))
torch.cuda.profiler.start()
dense_conv(wp, C, D, 3, 1, n, xb, xl, yb, yl)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
