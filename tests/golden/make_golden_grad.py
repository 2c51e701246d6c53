"""Golden vectors for the training-kernel row: the reference's
conv_grad_weights / conv_grad_input (kernels.py:103-162) and Conv2D.backward
(nn.py:62-72) on seeded inputs.

Run ONLY in the build container, where the read-only reference exists:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_grad.py

Writes grad_cases.npz (inputs and the reference's outputs, small shapes).  Nothing
on the GPU box reads /root/reference; the tests read this file.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF)

import unsparse as U  # noqa: E402  (the reference)
from unsparse import kernels as RK  # noqa: E402
from unsparse import nn as RN  # noqa: E402

# (C, D, Kh, Kw, H, W, stride, pad, batch): 3x3 same, stride-2 exact geometry, 1x1,
# 1-D (W = 1: the Yw == 1 loops), a non-square filter, a wide batch
CASES = [
    (3, 4, 3, 3, 6, 6, (1, 1), (1, 1), 2),
    (4, 5, 3, 3, 7, 7, (2, 2), (0, 0), 3),
    (6, 3, 1, 1, 5, 5, (1, 1), (0, 0), 2),
    (5, 4, 3, 1, 9, 1, (1, 1), (1, 0), 3),
    (2, 3, 3, 1, 9, 1, (2, 1), (0, 0), 2),
    (3, 2, 2, 3, 6, 7, (2, 1), (0, 1), 2),
    (8, 8, 3, 3, 8, 8, (1, 1), (1, 1), 16),
]


def main():
    rng = np.random.default_rng([2112, 15445])
    arrays = {}
    for k, (c, d, kh, kw, h, w, s, p, n) in enumerate(CASES):
        g = U.ConvGeometry(c, d, kh, kw, h, w, stride=s, padding=p)
        layer = RN.Conv2D(g, rng)
        layer.w.reshape(-1)[rng.choice(layer.w.size, layer.w.size // 2, replace=False)] = 0.0  # pruned
        x = rng.standard_normal((n, c, h, w)).astype(np.float32)
        y = layer.forward(x)
        dout = rng.standard_normal(y.shape).astype(np.float32)
        dx = layer.backward(dout)
        # the raw kernels as well (dxpad before the crop)
        dxpad = np.zeros_like(layer._xpad)
        RK.conv_grad_input(layer.w, dout, dxpad, s[0], s[1])
        arrays.update({f"g{k}_x": x, f"g{k}_w": layer.w, f"g{k}_dout": dout, f"g{k}_dw": layer.grad_w,
                       f"g{k}_dx": dx, f"g{k}_dxpad": dxpad,
                       f"g{k}_geom": np.array([c, d, kh, kw, h, w, s[0], s[1], p[0], p[1]], np.int64)})
    np.savez_compressed(os.path.join(HERE, "grad_cases.npz"), **arrays)
    print("wrote", len(CASES), "gradient cases")


if __name__ == "__main__":
    main()
