"""The A/B switches of the native library (read once per process, so each run is a
subprocess): USC_NO_PDL (plain launches instead of programmatic dependent launch),
USC_NO_DTS (64-channel layers on the zero-padded M = 128 kernel) and USC_NO_XROW (one TMA
box per pixel in the window kernels) change scheduling only: the fp32 sparse network is
bitwise the same and the binary16 tensor-core network stays within the fp16 tolerance."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys, numpy as np, torch
sys.path.insert(0, %r)
from paper_2112_15445_b200 import PrecisionMode
from paper_2112_15445_b200.models import SparseVGG16, vgg16_rng, vgg16_weights
x = np.random.default_rng(5).standard_normal((64, 3, 32, 32)).astype(np.float32)
m32 = SparseVGG16(vgg16_weights(vgg16_rng(0.93, 0), 0.93), 64)
m32.capture()
y32 = m32.forward(torch.from_numpy(x).cuda()).cpu().numpy()
import paper_2112_15445_b200 as U
F16 = PrecisionMode.BINARY16
ws = [U.DenseTensor4.from_array(np.array(w.data) * np.float32(np.sqrt(2.0 / (np.array(w.data)[0].size * 0.07))), F16)
      for w in vgg16_weights(vgg16_rng(0.93, 0), 0.93, precision=F16)]  # He-scaled: no binary16 saturation
m16 = SparseVGG16(ws, 64, precision=PrecisionMode.BINARY16, backends=["tc"] * 13)
m16.capture()
y16 = m16.forward(torch.from_numpy(x).cuda().half()).float().cpu().numpy()
np.save(sys.argv[1] + "_32.npy", y32)
np.save(sys.argv[1] + "_16.npy", y16)
""" % ROOT


def _run(tag, env_extra, tmp_path):
    env = dict(os.environ)
    env.update(env_extra)
    out = str(tmp_path / tag)
    subprocess.run([sys.executable, "-c", SCRIPT, out], check=True, env=env, timeout=600)
    return np.load(out + "_32.npy"), np.load(out + "_16.npy")


def test_scheduling_switches_do_not_change_results(tmp_path):
    a32, a16 = _run("default", {}, tmp_path)
    b32, b16 = _run("switched", {"USC_NO_PDL": "1", "USC_NO_DTS": "1", "USC_NO_XROW": "1"}, tmp_path)
    assert np.array_equal(a32.view(np.uint32), b32.view(np.uint32))
    assert np.isfinite(a16).all() and float(np.abs(a16).max()) > 0
    assert float(np.abs(a16 - b16).max()) <= 1e-2 * float(np.abs(a16).max())


CG2_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
from paper_2112_15445_b200 import _lib
from paper_2112_15445_b200.dense import dense_conv, pack_weights
out = []
for (C, D, hw, n) in [(256, 256, 8, 256), (512, 256, 4, 70), (256, 512, 8, 64), (256, 256, 7, 64)]:
    rng = np.random.default_rng([C, D, hw, n])
    x = torch.from_numpy(rng.standard_normal((n, C, hw, hw)).astype(np.float32)).cuda().half()
    w = torch.from_numpy((rng.standard_normal((D, C, 3, 3)) / np.sqrt(C * 9)).astype(np.float32)).cuda().half()
    xl = _lib.act_layout(C, hw, hw, 1, 1, 2, 64)
    xb = torch.zeros(xl.elems(n), dtype=torch.float16, device="cuda")
    _lib.check(_lib.lib().usc_pad_input(_lib.ref(xl), _lib.USC_F16, n, _lib.t_ptr(x), _lib.t_ptr(xb), _lib.stream_ptr()))
    yl = _lib.act_layout(D, hw, hw, 1, 1, 2, 64)
    yb = torch.zeros(yl.elems(n), dtype=torch.float16, device="cuda")
    dense_conv(pack_weights(w), C, D, 3, 1, n, xb, xl, yb, yl, twp=4, splits=1)
    o = torch.empty((n, D, hw, hw), dtype=torch.float16, device="cuda")
    _lib.check(_lib.lib().usc_unpad_output(_lib.ref(yl), _lib.USC_F16, n, _lib.t_ptr(yb), _lib.t_ptr(o), _lib.stream_ptr()))
    ref = torch.relu(torch.nn.functional.conv2d(x.float(), w.float(), padding=1))
    out.append(float((o.float() - ref).abs().max()) / float(ref.abs().max()))
    assert torch.isfinite(yb.float()).all()
print(max(out))
""" % ROOT


def test_cta_pair_tiles_match_torch():
    """USC_CG2=1: >= 256-channel 3x3 window tiles on CTA pairs (tcgen05.mma.cta_group::2,
    2CTA TMA completing on the leader's barrier, multicast commits) -- same results within
    the fp16 tolerance, including a ragged batch and a partial last x tile."""
    env = dict(os.environ)
    env["USC_CG2"] = "1"
    r = subprocess.run([sys.executable, "-c", CG2_SCRIPT], check=True, env=env, timeout=600, capture_output=True,
                       text=True)
    assert float(r.stdout.strip().splitlines()[-1]) <= 1e-2
