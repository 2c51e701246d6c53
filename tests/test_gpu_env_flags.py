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
