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
    """Shapes the tensor-core kernel takes: channels in % 64 (1x1 / 3x3, stride 1 / 2), or the
    first-layer form (<= 16 input channels, 3x3 stride 1, 64 outputs)."""
    if in_channels <= 16 and in_channels % 64:
        return out_channels == 64 and k == 3 and stride == 1
    return in_channels % 64 == 0 and out_channels % 64 == 0 and k in (1, 3) and stride in (1, 2)


def pack_weights(w, device=None):
    """Dense (D, C, K, K) weights -> the kernel's binary16 [D][K*K][C] (K-major) tensor, zero
    rows appended up to a multiple of 128 output channels (the MMA's M); a first layer with
    <= 16 input channels packs as [K*K][16][D] (channels zero-padded, D contiguous)."""
    import torch
    t = w if type(w).__module__.startswith("torch") else torch.from_numpy(
        np.array(w.data if hasattr(w, "data") else w, dtype=np.float32))
    t = t.to(device or "cuda", torch.float16)
    D, C, kh, kw = t.shape
    if C <= 16 and C % 64:  # first-layer form: [taps][16 channels (zero-padded)][D], D contiguous
        packed = t.new_zeros((kh * kw, 16, D))
        packed[:, :C, :] = t.permute(2, 3, 1, 0).reshape(kh * kw, C, D)
        return packed.reshape(kh * kw * 16, D).contiguous()
    packed = t.permute(0, 2, 3, 1).reshape(D, kh * kw * C)
    dpad = -(-D // 128) * 128
    if dpad != D:
        packed = torch.cat([packed, packed.new_zeros((dpad - D, kh * kw * C))])
    return packed.contiguous()


def dense_workspace(in_channels: int, out_channels: int, k: int, stride: int, n: int, x_lay, res: bool = False,
                    device=None, twp: int = 0, splits: int = 0):
    """Zero-filled split-K workspace for dense_conv on this shape and tile configuration
    (None when it does not split: automatic configurations split only small maps; a fused
    shortcut never splits).  Reusable across launches of the same shape (the kernel leaves
    its counters at zero); not shareable between launches that may run concurrently."""
    import torch
    g = _lib.Geometry(in_channels, out_channels, k, k, x_lay.height, x_lay.width, stride, stride, k // 2, k // 2)
    nbytes = int(_lib.lib().usc_dense_conv_f16_ws_bytes(_lib.ref(g), n, _lib.ref(x_lay), int(res), int(twp),
                                                        int(splits)))
    if nbytes <= 0:
        return None
    return torch.zeros(nbytes, dtype=torch.uint8, device=device or "cuda")


def dense_conv(w_packed, in_channels: int, out_channels: int, k: int, stride: int, n: int, x, x_lay, y, y_lay,
               res=None, res_lay=None, relu: bool = True, stream=None, workspace=None, twp: int = 0,
               splits: int = 0):
    """One tensor-core convolution on BI64 buffers (usc_dense_conv_f16[_ws]).  `twp` /
    `splits` pick the tile (pixels per tile 2 or 4, K splits; 0 = automatic); `workspace`
    from dense_workspace(..., twp, splits) enables split-K."""
    g = _lib.Geometry(in_channels, out_channels, k, k, x_lay.height, x_lay.width, stride, stride, k // 2, k // 2)
    args = (_lib.ref(g), n, _lib.t_ptr(w_packed), _lib.ref(x_lay), _lib.t_ptr(x), _lib.ref(y_lay), _lib.t_ptr(y),
            None if res is None else _lib.ref(res_lay), None if res is None else _lib.t_ptr(res), int(relu))
    if workspace is None and not twp and not splits:
        _lib.check(_lib.lib().usc_dense_conv_f16(*args, _lib.stream_ptr(stream)), "dense_conv_f16")
    else:
        _lib.check(_lib.lib().usc_dense_conv_f16_ws(
            *args, None if workspace is None else _lib.t_ptr(workspace), 0 if workspace is None else workspace.numel(),
            int(twp), int(splits), _lib.stream_ptr(stream)), "dense_conv_f16_ws")


def pool_fusable(in_channels: int, out_channels: int, n: int, x_lay) -> bool:
    """True when the 3x3 conv + ReLU + 2x2 pool runs as one tensor-core launch
    (usc_dense_conv_f16_pool_ok) at least as fast as conv + pool."""
    g = _lib.Geometry(in_channels, out_channels, 3, 3, x_lay.height, x_lay.width, 1, 1, 1, 1)
    return bool(_lib.lib().usc_dense_conv_f16_pool_ok(_lib.ref(g), n, _lib.ref(x_lay)))


def dense_conv_pool(w_packed, in_channels: int, out_channels: int, n: int, x, x_lay, y, y_lay, stream=None):
    """3x3 stride-1 conv + ReLU + 2x2 max-pool in one launch; `y_lay` is the pooled layout."""
    g = _lib.Geometry(in_channels, out_channels, 3, 3, x_lay.height, x_lay.width, 1, 1, 1, 1)
    _lib.check(_lib.lib().usc_dense_conv_f16_pool(_lib.ref(g), n, _lib.t_ptr(w_packed), _lib.ref(x_lay),
                                                  _lib.t_ptr(x), _lib.ref(y_lay), _lib.t_ptr(y),
                                                  _lib.stream_ptr(stream)), "dense_conv_f16_pool")


# (pixels per tile, K splits) candidates of the per-layer tile search; 0 = automatic
TILE_CANDIDATES = ((0, 0), (2, 1), (4, 1), (2, 2), (4, 2), (2, 4), (4, 4))


def tune_tile(launch, in_channels: int, out_channels: int, k: int, stride: int, n: int, x_lay, res: bool = False,
              device=None, repeats: int = 5) -> tuple:
    """Per-layer tile search of the tensor-core backend (the dense-side analogue of the
    sparse autotune_sb, ref/engine.py:139-170): `launch(twp, splits, workspace)` runs the
    layer on its real buffers; every candidate is timed with CUDA events (host cost hidden)
    and the fastest (twp, splits) returned.  Splits never combine with a fused shortcut."""
    from .engine import time_median_cuda
    best, best_ms = (0, 0), None
    for twp, sp in TILE_CANDIDATES:
        if res and sp > 1:
            continue
        ws = dense_workspace(in_channels, out_channels, k, stride, n, x_lay, res, device, twp, sp)
        ms = time_median_cuda(lambda: launch(twp, sp, ws), repeats, 2, 4)
        if best_ms is None or ms < best_ms:
            best, best_ms = (twp, sp), ms
    return best
