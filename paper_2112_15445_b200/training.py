"""Training path of the dense Conv2D layer on the GPU (pruning with
retraining), bit-identical to the reference.

  conv_grad_weights / conv_grad_input -- the numba FFI kernels of
      /root/reference/pkg/src/unsparse/kernels.py:103-162 with device tensors
      (csrc/grad.cu through usc_conv_grad_weights / usc_conv_grad_input);
  Conv2D -- nn.Conv2D (nn.py:28-78): glorot-uniform init from the caller's rng
      (nn.py:23-25, same draws), forward through the sparse engine on build_csr of the
      current weights (bitwise equal to the reference's dense_conv_channels for finite
      inputs), backward through the two gradient kernels.
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib
from .csr import build_csr
from .engine import sparse_conv_forward
from .tensor import ConvGeometry, DenseTensor4


def _geom(C, D, Kh, Kw, Hp, Wp, s_h, s_w) -> _lib.Geometry:
    """Geometry of the padded problem (pad already materialised in xpad)."""
    return _lib.Geometry(C, D, Kh, Kw, Hp, Wp, s_h, s_w, 0, 0)


def conv_grad_weights(xpad, dout, dw, s_h: int, s_w: int, stream=None) -> None:
    """kernels.conv_grad_weights(xpad, dout, dw, s_h, s_w) (kernels.py:103-130) on CUDA
    fp32 tensors: dw[d,c,kh,kw] = sum_b sum_(r,cc) dout[b,d,r,cc] *
    xpad[b,c,r*s_h+kh,cc*s_w+kw], fp64 accumulation in the reference's order."""
    n, C, Hp, Wp = xpad.shape
    D, C2, Kh, Kw = dw.shape
    if C2 != C or dout.shape[0] != n or dout.shape[1] != D:
        raise ValueError(f"shapes xpad {tuple(xpad.shape)}, dout {tuple(dout.shape)}, dw {tuple(dw.shape)} differ")
    g = _geom(C, D, Kh, Kw, Hp, Wp, s_h, s_w)
    _check_out(g, dout)
    _lib.check(_lib.lib().usc_conv_grad_weights(_lib.ref(g), n, _lib.t_ptr(_f32(xpad)), _lib.t_ptr(_f32(dout)),
                                                 _lib.t_ptr(_f32(dw)), _lib.stream_ptr(stream)), "conv_grad_weights")


def conv_grad_input(w, dout, dxpad, s_h: int, s_w: int, stream=None) -> None:
    """kernels.conv_grad_input(w, dout, dxpad, s_h, s_w) (kernels.py:133-162) on CUDA
    fp32 tensors.  The reference accumulates into a zeroed dxpad (nn.py:67); here
    every element of dxpad is overwritten with that accumulation."""
    n, C, Hp, Wp = dxpad.shape
    D, C2, Kh, Kw = w.shape
    if C2 != C or dout.shape[0] != n or dout.shape[1] != D:
        raise ValueError(f"shapes w {tuple(w.shape)}, dout {tuple(dout.shape)}, dxpad {tuple(dxpad.shape)} differ")
    g = _geom(C, D, Kh, Kw, Hp, Wp, s_h, s_w)
    _check_out(g, dout)
    _lib.check(_lib.lib().usc_conv_grad_input(_lib.ref(g), n, _lib.t_ptr(_f32(w)), _lib.t_ptr(_f32(dout)),
                                               _lib.t_ptr(_f32(dxpad)), _lib.stream_ptr(stream)), "conv_grad_input")


def _f32(t):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise ValueError("expected a contiguous float32 CUDA tensor")
    return t


def _check_out(g, dout):
    yh, yw = ctypes_out(g)
    if tuple(dout.shape[2:]) != (yh, yw):
        raise ValueError(f"dout spatial {tuple(dout.shape[2:])} != geometry output {(yh, yw)}")


def ctypes_out(g):
    import ctypes
    yh, yw = ctypes.c_int32(), ctypes.c_int32()
    _lib.check(_lib.lib().usc_geometry_out(_lib.ref(g), ctypes.byref(yh), ctypes.byref(yw)), "geometry")
    return yh.value, yw.value


def glorot_uniform(rng, shape, fan_in, fan_out, dtype=np.float32):
    """nn.py:23-25 (same draws from the caller's generator)."""
    bound = math.sqrt(6.0 / (fan_in + fan_out))
    return rng.uniform(-bound, bound, size=shape).astype(dtype)


class Conv2D:
    """nn.Conv2D (nn.py:28-78) on the GPU: convolution without bias, weights (D, C, Kh, Kw)
    as a host fp32 array (prunable in place, like the reference), activations and
    gradients as CUDA tensors."""

    kind = "conv2d"
    prunable = True

    def __init__(self, geometry: ConvGeometry, rng, dtype=np.float32):
        self.geometry = g = geometry
        fan_in = g.in_channels * g.filter_h * g.filter_w
        fan_out = g.out_channels * g.filter_h * g.filter_w
        self.w = glorot_uniform(rng, (g.out_channels, g.in_channels, g.filter_h, g.filter_w), fan_in, fan_out, dtype)
        self.grad_w = None
        self._xpad = None

    def forward(self, x):
        """x: (n, C, H, W) fp32 CUDA tensor (or array) -> (n, D, Yh, Yw) CUDA tensor."""
        import torch
        g = self.geometry
        x = torch.as_tensor(x, dtype=torch.float32, device="cuda").contiguous()
        ph, pw = g.padding
        self._xpad = torch.nn.functional.pad(x, (pw, pw, ph, ph)) if (ph or pw) else x
        filt = build_csr(DenseTensor4.from_array(self.w), g)
        return sparse_conv_forward(DenseTensor4(x), filt).device()

    def backward(self, dout):
        """nn.py:62-72: grad_w and dx (the padded-input gradient cropped to the input)."""
        import torch
        g = self.geometry
        dout = torch.as_tensor(dout, dtype=torch.float32, device="cuda").contiguous()
        w = torch.from_numpy(np.ascontiguousarray(self.w, np.float32)).cuda()
        dw = torch.empty_like(w)
        conv_grad_weights(self._xpad, dout, dw, g.stride[0], g.stride[1])
        dxpad = torch.empty_like(self._xpad)
        conv_grad_input(w, dout, dxpad, g.stride[0], g.stride[1])
        self.grad_w = dw.cpu().numpy()
        ph, pw = g.padding
        if ph or pw:
            return dxpad[:, :, ph:ph + g.input_h, pw:pw + g.input_w].contiguous()
        return dxpad

    def params(self):
        return {"w": self.w}

    def grads(self):
        return {"w": self.grad_w}
