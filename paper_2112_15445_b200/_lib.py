"""ctypes binding of the C ABI (include/unsparse_b200.h) -> libunsparse_b200.so.

The product path has no CPU fallback: if the shared library is missing or was
built without a usable device, calls fail loudly.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libunsparse_b200.so")

USC_OK, USC_ERR_VALUE, USC_ERR_CORRUPT, USC_ERR_CUDA, USC_ERR_UNSUPPORTED = range(5)
USC_F32, USC_F16, USC_I8, USC_CB4 = range(4)

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_ptr = ctypes.c_void_p


class Geometry(ctypes.Structure):
    _fields_ = [(n, c_i32) for n in ("in_channels", "out_channels", "filter_h", "filter_w",
                                     "input_h", "input_w", "stride_h", "stride_w", "pad_h", "pad_w")]


class ActLayout(ctypes.Structure):
    _fields_ = [("channels", c_i32), ("height", c_i32), ("width", c_i32), ("pad_h", c_i32),
                ("pad_w", c_i32), ("hp", c_i32), ("ws", c_i32), ("interleave", c_i32),
                ("sample_stride", c_i64)]

    def key(self):
        return (self.channels, self.height, self.width, self.pad_h, self.pad_w, self.hp, self.ws,
                self.interleave)

    def elems(self, n: int) -> int:
        """Elements a buffer of n samples needs (usc_act_layout_elems)."""
        return int(lib().usc_act_layout_elems(ctypes.byref(self), n))


class ExecCfg(ctypes.Structure):
    _fields_ = [(n, c_i32) for n in ("sub_batch", "worker_count", "pix_per_thread", "ch_per_cta",
                                     "samples_per_cta", "chunk_channels", "threads", "kernel",
                                     "pixel_warps", "stages", "rows_per_thread", "ent_reserve",
                                     "pixel_classes", "window")]


class Plan(ctypes.Structure):
    _fields_ = [("g", Geometry), ("dtype", c_i32), ("n", c_i32), ("out_h", c_i32), ("out_w", c_i32),
                ("in_", ActLayout), ("kernel", c_i32), ("P", c_i32), ("DT", c_i32), ("NS", c_i32),
                ("CC", c_i32), ("threads", c_i32), ("TH", c_i32), ("HS", c_i32),
                ("strips_per_row", c_i32), ("row_tiles", c_i32), ("sample_tiles", c_i32),
                ("groups", c_i32), ("n_chunks", c_i32), ("WS", c_i32), ("WC", c_i32), ("DW", c_i32),
                ("SPRt", c_i32), ("col_tiles", c_i32), ("TWs", c_i32), ("ent_stage_bytes", c_i32), ("stages", c_i32), ("PR", c_i32), ("PC", c_i32),
                ("transposed", c_i32), ("ncls_r", c_i32), ("ncls_c", c_i32), ("tail_full", c_i32),
                ("tail_split", c_i32), ("window", c_i32),
                ("smem_stage_bytes", c_i64), ("smem_bytes", c_i64), ("grid_x", c_i64),
                ("grid_y", c_i64)]

    def describe(self) -> dict:
        kern = {1: "tiled", 2: "generic", 3: f"bw{self.NS}" if self.window else f"bi{self.NS}", 4: "bt64"}[self.kernel]
        return dict(kernel=kern, P=self.P, DT=self.DT,
                    NS=self.NS, CC=self.CC, TH=self.TH, threads=self.threads, WS=self.WS,
                    WC=self.WC, DW=self.DW, PR=self.PR, PC=self.PC, stages=self.stages,
                    grid=(self.grid_x, self.grid_y), smem_bytes=self.smem_bytes,
                    n_chunks=self.n_chunks, transposed=bool(self.transposed),
                    pixel_classes=self.ncls_r * self.ncls_c, tail_split=self.tail_split)


class Epilogue(ctypes.Structure):
    _fields_ = [("relu", c_i32), ("saturate", c_i32), ("cap", ctypes.c_float), ("saturate2", c_i32),
                ("cap2", ctypes.c_float), ("scale", ctypes.c_float), ("out_padded", c_i32),
                ("out", ActLayout), ("pool", c_i32), ("requant", c_i32), ("rq_scale", ctypes.c_float),
                ("rq_limit", c_i32), ("residual", c_i32), ("res_layout", ActLayout), ("res", ctypes.c_uint64)]


class CsrCorruptionError(ValueError):
    """A stored offset does not decode to a valid filter tap (csr.py:21)."""


_lib = None

_SIGS = {
    "usc_abi_version": (c_i32, []),
    "usc_last_error": (ctypes.c_char_p, []),
    "usc_device_sm_count": (c_i32, [c_i32]),
    "usc_geometry_check": (c_i32, [c_ptr]),
    "usc_geometry_out": (c_i32, [c_ptr, c_ptr, c_ptr]),
    "usc_act_layout_make": (c_i32, [c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_ptr]),
    "usc_act_layout_elems": (c_i64, [c_ptr, c_i32]),
    "usc_csr_count": (c_i32, [c_ptr, c_ptr, c_ptr]),
    "usc_build_csr": (c_i32, [c_ptr, c_ptr, c_i64, c_ptr, c_ptr, c_ptr]),
    "usc_csr_count_device": (c_i32, [c_ptr, c_ptr, c_ptr, c_ptr, c_ptr]),
    "usc_build_csr_device": (c_i32, [c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr]),
    "usc_csr_validate": (c_i32, [c_ptr, c_ptr, c_i64, c_ptr, c_i64, c_i64, c_i64, c_ptr]),
    "usc_conv_grad_weights": (c_i32, [c_ptr, c_i32, c_ptr, c_ptr, c_ptr, c_ptr]),
    "usc_conv_grad_input": (c_i32, [c_ptr, c_i32, c_ptr, c_ptr, c_ptr, c_ptr]),
    "usc_csr_to_dense": (c_i32, [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_ptr]),
    "usc_plan_make": (c_i32, [c_ptr, c_i32, c_i32, c_ptr, c_ptr]),
    "usc_bi_instances": (c_i32, [c_ptr, c_i32]),
    "usc_bw_instances": (c_i32, [c_ptr, c_i32]),
    "usc_pack_size": (c_i32, [c_ptr, c_i64, c_ptr]),
    "usc_autotune": (c_i32, [c_ptr, c_i32, c_i32, c_ptr, c_ptr, c_ptr, c_i64, c_ptr, c_ptr, c_i32, c_i32,
                             ctypes.c_float, c_ptr, c_ptr, c_ptr]),
    "usc_pack": (c_i32, [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_ptr, c_ptr, c_i64, c_ptr]),
    "usc_pad_input": (c_i32, [c_ptr, c_i32, c_i32, c_ptr, c_ptr, c_ptr]),
    "usc_unpad_output": (c_i32, [c_ptr, c_i32, c_i32, c_ptr, c_ptr, c_ptr]),
    "usc_bi_to_nhwc": (c_i32, [c_ptr, c_i32, c_ptr, c_ptr, c_ptr]),
    "usc_nhwc_to_bi": (c_i32, [c_ptr, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_i32, c_ptr]),
    "usc_f16_epilogue": (c_i32, [c_ptr, c_ptr, c_i64, c_i32, c_ptr]),
    "usc_dense_conv_f16": (c_i32, [c_ptr, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_i32, c_ptr]),
    "usc_dense_conv_f16_ws": (c_i32, [c_ptr, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_i32, c_ptr,
                                      c_i64, c_i32, c_i32, c_ptr]),
    "usc_dense_conv_f16_ws_bytes": (c_i64, [c_ptr, c_i32, c_ptr, c_i32, c_i32, c_i32]),
    "usc_dense_conv_f16_pool": (c_i32, [c_ptr, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr]),
    "usc_dense_conv_f16_pool_ok": (c_i32, [c_ptr, c_i32, c_ptr]),
    "usc_conv_forward": (c_i32, [c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr]),
    "usc_conv_forward_view": (c_i32, [c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr]),
    "usc_conv_forward_strided": (c_i32, [c_ptr, c_ptr, c_ptr, c_ptr, c_i32, c_i32, c_ptr, c_ptr, c_ptr]),
    "usc_sparse_conv_blocks": (c_i32, [c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i32, c_i64,
                                       c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_ptr]),
    "usc_round_binary16": (c_i32, [c_ptr, c_ptr, c_i64, c_i32, c_ptr]),
    "usc_convert": (c_i32, [c_ptr, c_i32, c_ptr, c_i32, c_i64, c_ptr]),
    "usc_maxpool2": (c_i32, [c_ptr, c_ptr, c_i32, c_i32, c_ptr, c_ptr, c_ptr]),
    "usc_quantize_i8": (c_i32, [c_ptr, c_ptr, c_i64, ctypes.c_double, c_i32, c_ptr]),
    "usc_peak_fp32_muladd": (c_i32, [c_i32, c_ptr]),
    "usc_peak_mix": (c_i32, [c_i32, c_i32, c_ptr]),
    "usc_fit_fixed_point": (c_i32, [ctypes.c_double, c_i32, c_ptr, c_ptr, c_ptr]),
    "usc_linear_codes": (c_i32, [c_ptr, c_i64, ctypes.c_double, c_i32, c_ptr]),
    "usc_kmeans_codebook": (c_i32, [c_ptr, c_i64, c_i32, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr]),
}

EXPORTED = tuple(_SIGS)


def lib():
    """Load the native library (fail loudly when it is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (make -C paper_2112_15445_b200/csrc)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.usc_abi_version() != 1:
            raise ImportError("libunsparse_b200.so ABI version mismatch")
        _lib = L
    return _lib


def bi_instances(binary16: bool = False, tmem: bool = False) -> list[tuple[int, int, int, int, int, int]]:
    """The batch-interleaved kernels' compiled tiles: (compute warps, PC, PR, DW,
    stride_w, samples per lane) of the fp32 (kernel 3), binary16-input (F16/CB4/I8,
    kernel 3) or tensor-memory fp32 (kernel 4) family."""
    L = lib()
    n = L.usc_bi_instances(None, 0)
    buf = (c_i32 * (7 * n))()
    L.usc_bi_instances(buf, n)
    kind = 2 if tmem else int(binary16)
    return [tuple(buf[7 * i:7 * i + 6]) for i in range(n) if buf[7 * i + 6] == kind]


def bw_instances() -> list[tuple[int, int, int, int, int]]:
    """The register-window kernel's compiled tiles: (family 0 fp32 / 1 binary16, compute
    warps, PC, DW, KW)."""
    L = lib()
    n = L.usc_bw_instances(None, 0)
    buf = (c_i32 * (5 * n))()
    L.usc_bw_instances(buf, n)
    return [tuple(buf[5 * i:5 * i + 5]) for i in range(n)]


def check(rc: int, what: str = ""):
    if rc == USC_OK:
        return
    msg = lib().usc_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc == USC_ERR_CORRUPT:
        raise CsrCorruptionError(msg)
    if rc == USC_ERR_VALUE:
        raise ValueError(msg)
    raise RuntimeError(msg)


def ref(obj):
    return ctypes.byref(obj)


def np_ptr(a):
    return ctypes.c_void_p(a.ctypes.data)


def t_ptr(t):
    """Device pointer of a CUDA tensor (kernel arguments; a host tensor here would
    fault inside the kernel and poison the context, so it is rejected)."""
    if not t.is_cuda:
        raise ValueError(f"expected a CUDA tensor, got one on {t.device}")
    return ctypes.c_void_p(t.data_ptr())


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def make_geometry(g) -> Geometry:
    return Geometry(g.in_channels, g.out_channels, g.filter_h, g.filter_w, g.input_h, g.input_w,
                    g.stride[0], g.stride[1], g.padding[0], g.padding[1])


def act_layout(channels, h, w, ph, pw, elem_bytes, interleave: int = 0) -> ActLayout:
    lay = ActLayout()
    check(lib().usc_act_layout_make(channels, h, w, ph, pw, elem_bytes, interleave, ref(lay)), "layout")
    return lay
