"""The dispatcher's dense backend on the B200's tensor cores.

The reference picks, per layer, its sparse engine or a dense comparator
(backend_config, /root/reference/pkg/src/unsparse/bench.py:212-227;
pipeline.py:381-389).  For binary16 networks (the north star's 1e-2 tolerance path)
the dense choice here is usc_dense_conv_f16: an implicit-GEMM convolution on tcgen05
(fp32 accumulation in tensor memory) that reads and writes the networks' resident BI64
layout, so a dense layer needs no layout transposes.  fp32 / int8 / 4b-16b networks stay
on the bit-exact sparse kernels.
"""

from __future__ import annotations

import numpy as np

from . import _lib


def tc_eligible(in_channels: int, out_channels: int, k: int, stride: int) -> bool:
    """Shapes the tensor-core kernel takes."""
    return in_channels % 64 == 0 and out_channels % 64 == 0 and k in (1, 3) and stride in (1, 2)


def pack_weights(w, device=None):
    """Dense (D, C, K, K) weights -> the kernel's binary16 [D][K*K][C] (K-major) tensor, zero
    rows appended up to a multiple of 128 output channels (the MMA's M)."""
    import torch
    t = w if type(w).__module__.startswith("torch") else torch.from_numpy(
        np.array(w.data if hasattr(w, "data") else w, dtype=np.float32))
    t = t.to(device or "cuda", torch.float16)
    D, C, kh, kw = t.shape
    packed = t.permute(0, 2, 3, 1).reshape(D, kh * kw * C)
    dpad = -(-D // 128) * 128
    if dpad != D:
        packed = torch.cat([packed, packed.new_zeros((dpad - D, kh * kw * C))])
    return packed.contiguous()


def dense_conv(w_packed, in_channels: int, out_channels: int, k: int, stride: int, n: int, x, x_lay, y, y_lay,
               res=None, res_lay=None, relu: bool = True, stream=None):
    """One tensor-core convolution on BI64 buffers (usc_dense_conv_f16)."""
    g = _lib.Geometry(in_channels, out_channels, k, k, x_lay.height, x_lay.width, stride, stride, k // 2, k // 2)
    _lib.check(_lib.lib().usc_dense_conv_f16(
        _lib.ref(g), n, _lib.t_ptr(w_packed), _lib.ref(x_lay), _lib.t_ptr(x), _lib.ref(y_lay), _lib.t_ptr(y),
        None if res is None else _lib.ref(res_lay), None if res is None else _lib.t_ptr(res), int(relu),
        _lib.stream_ptr(stream)), "dense_conv_f16")
