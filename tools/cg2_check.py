import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2112_15445_b200 import _lib
from paper_2112_15445_b200.dense import dense_conv, pack_weights
from paper_2112_15445_b200.engine import time_median_cuda
import os
shapes = [(256, 256, 8, 256), (512, 512, 4, 256), (256, 512, 8, 64), (512, 256, 4, 70), (256, 256, 8, 128)]
if os.environ.get('CG2_BIG'):
    shapes = [(256, 256, 8, 1024), (256, 256, 16, 256), (512, 512, 8, 256), (256, 256, 32, 64)]
for (C, D, hw, n) in shapes:
    rng = np.random.default_rng([C, D, hw, n])
    x = torch.from_numpy(rng.standard_normal((n, C, hw, hw)).astype(np.float32)).cuda().half()
    w = torch.from_numpy((rng.standard_normal((D, C, 3, 3)) / np.sqrt(C * 9)).astype(np.float32)).cuda().half()
    xl = _lib.act_layout(C, hw, hw, 1, 1, 2, 64)
    xb = torch.zeros(xl.elems(n), dtype=torch.float16, device="cuda")
    _lib.check(_lib.lib().usc_pad_input(_lib.ref(xl), _lib.USC_F16, n, _lib.t_ptr(x), _lib.t_ptr(xb), _lib.stream_ptr()))
    yl = _lib.act_layout(D, hw, hw, 1, 1, 2, 64)
    yb = torch.zeros(yl.elems(n), dtype=torch.float16, device="cuda")
    wp = pack_weights(w)
    dense_conv(wp, C, D, 3, 1, n, xb, xl, yb, yl, twp=4, splits=1)
    out = torch.empty((n, D, hw, hw), dtype=torch.float16, device="cuda")
    _lib.check(_lib.lib().usc_unpad_output(_lib.ref(yl), _lib.USC_F16, n, _lib.t_ptr(yb), _lib.t_ptr(out), _lib.stream_ptr()))
    torch.cuda.synchronize()
    ref = torch.relu(torch.nn.functional.conv2d(x.float(), w.float(), padding=1))
    err = float((out.float() - ref).abs().max()); tol = 1e-2 * float(ref.abs().max())
    us = time_median_cuda(lambda: dense_conv(wp, C, D, 3, 1, n, xb, xl, yb, yl, twp=4, splits=1), 9, 3) * 1e3
    print(C, D, hw, n, "err", round(err, 4), "tol", round(tol, 4), "ok" if err <= tol else "FAIL", "us", round(us, 1), flush=True)
