"""Linear (fixed-point) and non-linear (codebook) quantisation
(/root/reference/pkg/src/unsparse/quantization.py) and the quantised conv paths.

The primitives keep the reference's signatures and are computed natively
(usc_fit_fixed_point, usc_linear_codes, usc_kmeans_codebook -- bit-identical to
the numpy reference, including numpy's pairwise summation in the k-means means).

The quantised sparse conv variants the reference only defines by composition
 run as dedicated sm_100a kernels:

* int8: ``build_csr_int8`` + ``quantize_input_int8`` + ``sparse_conv_forward_int8``
  equal the reference composition ``sparse_conv_forward(linear_quantize(x),
  build_csr(linear_quantize(w)))`` bitwise: the batch-interleaved kernel (the
  default) accumulates the code products in fp32 in the reference's order and
  rescales once by a power of two; kernel 1 accumulates in int32, which equals
  the composition whenever max_d sum|k_w| * max|k_x| < 2**24;
* 4b/16b: ``build_csr_codebook`` + ``sparse_conv_forward_codebook`` store a
  4-bit centroid index per entry, decode through a 16-entry fp32 table in shared
  memory, accumulate fp32 in reference order and apply the 4b/16b activation hook
  (saturate at threshold*calibrated max, round to binary16, _half_hook 238-244).
"""

from __future__ import annotations

import ctypes
import json
import math
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .csr import CsrFilter, build_csr
from .engine import ExecConfig, launch, padded_input, plan_for, sparse_conv_forward
from .tensor import ConvGeometry, DenseTensor4, PrecisionMode, round_to_binary16

MODES = ("passthrough", "16b/16b", "4b/16b")


@dataclass(frozen=True)
class FixedPointParams:
    """quantization.py:24-38."""

    total_bits: int
    int_bits: int
    frac_bits: int
    sigma: float
    mu: float = 0.0
    degenerate: bool = False


def _amax(tensor) -> float:
    if type(tensor).__module__.startswith("torch"):
        return float(tensor.detach().abs().max().item())
    if isinstance(tensor, DenseTensor4):
        return _amax(tensor.device() if tensor.on_device else tensor.data)
    arr = np.asarray(tensor)
    if arr.size == 0:
        raise ValueError("cannot fit an empty tensor")
    return float(np.max(np.abs(arr)))


def fit_fixed_point(tensor, total_bits: int) -> FixedPointParams:
    """quantization.py:41-58: int_bits = ceil(log2 max|x|), frac = bits - int - 1."""
    if total_bits < 2:
        raise ValueError("total_bits must be >= 2")
    amax = _amax(tensor)
    ib, fb, sg = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_double()
    _lib.check(_lib.lib().usc_fit_fixed_point(amax, total_bits, _lib.ref(ib), _lib.ref(fb),
                                              _lib.ref(sg)), "fit_fixed_point")
    return FixedPointParams(total_bits, ib.value, fb.value, sg.value, 0.0, amax == 0.0)


def linear_codes(x, params: FixedPointParams) -> np.ndarray:
    """The integer codes of linear_quantize (round half away from zero, clipped)."""
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64) - params.mu)
    out = np.empty_like(arr)
    _lib.check(_lib.lib().usc_linear_codes(_lib.np_ptr(arr), arr.size, params.sigma,
                                           params.total_bits, _lib.np_ptr(out)), "linear_codes")
    return out


def linear_quantize(x, params: FixedPointParams):
    """quantization.py:61-76: q = mu + sigma*round((x - mu)/sigma), half away from zero."""
    q = params.mu + params.sigma * linear_codes(x, params)
    if np.isscalar(x) or np.ndim(x) == 0:
        return float(q.reshape(-1)[0])
    q = q.reshape(np.shape(x))
    return q.astype(np.asarray(x).dtype) if np.asarray(x).dtype.kind == "f" else q


def saturate_activations(activations, quantile_threshold: float, calibrated_max: float | None = None):
    """quantization.py:79-93: min(A, threshold * max) (NaN propagates)."""
    if not 0.0 < quantile_threshold <= 1.0:
        raise ValueError("threshold must be in (0, 1]")
    if type(activations).__module__.startswith("torch"):
        import torch
        m = float(activations.max().item()) if calibrated_max is None else float(calibrated_max)
        cap = torch.tensor(np.float32(quantile_threshold * m), device=activations.device)
        return torch.where(activations > cap, cap, activations)
    arr = np.asarray(activations)
    if arr.size == 0:
        raise ValueError("empty activation tensor")
    m = float(np.max(arr)) if calibrated_max is None else float(calibrated_max)
    return np.minimum(arr, quantile_threshold * m)


@dataclass
class Codebook:
    """quantization.py:96-109."""

    centroids: np.ndarray
    quantized_centroids: np.ndarray
    assignments: np.ndarray
    omega: int
    psi: int
    zero_pinned: bool

    def reconstruct(self, shape):
        return self.quantized_centroids[self.assignments].reshape(shape).astype(np.float32)


def kmeans_codebook(weights, omega: int, psi: int = 16) -> Codebook:
    """quantization.py:134-180 (zero-pinned 1-D Lloyd, psi-bit centroids), natively."""
    if omega < 1:
        raise ValueError("omega must be >= 1")
    if psi not in (8, 16):
        raise ValueError("psi must be 8 or 16")
    flat = np.ascontiguousarray(np.asarray(weights, dtype=np.float64).ravel())
    cent = np.zeros(max(omega, 1), np.float64)
    quant = np.zeros_like(cent)
    assign = np.zeros(flat.size, np.int64)
    k, zp = ctypes.c_int32(), ctypes.c_int32()
    _lib.check(_lib.lib().usc_kmeans_codebook(_lib.np_ptr(flat), flat.size, omega, psi,
                                              _lib.np_ptr(cent), _lib.np_ptr(quant),
                                              _lib.np_ptr(assign), _lib.ref(k), _lib.ref(zp)),
               "kmeans_codebook")
    return Codebook(cent[:k.value].copy(), quant[:k.value].copy(), assign, omega, psi, bool(zp.value))


def kmeans_cost(values, centroids, assignments) -> float:
    """quantization.py:183-185."""
    d = values - centroids[assignments]
    return float(np.sum(d * d))


def save_codebook(cb: Codebook, path) -> None:
    """quantization.py:188-202."""
    if len(cb.centroids) > 256:
        raise ValueError("assignment export supports at most 256 centroids")
    meta = {"omega": cb.omega, "psi": cb.psi, "zero_pinned": cb.zero_pinned,
            "centroids": [float(c) for c in cb.centroids],
            "quantized_centroids": [float(c) for c in cb.quantized_centroids],
            "weight_count": int(cb.assignments.size)}
    with open(path, "w") as fh:
        json.dump(meta, fh, indent=2, sort_keys=True)
    cb.assignments.astype(np.uint8).tofile(str(path) + ".bin")


def load_codebook(path) -> Codebook:
    """quantization.py:205-218."""
    with open(path) as fh:
        meta = json.load(fh)
    assignments = np.fromfile(str(path) + ".bin", dtype=np.uint8).astype(np.int64)
    if assignments.size != meta["weight_count"]:
        raise ValueError("assignment array length mismatch")
    return Codebook(np.asarray(meta["centroids"]), np.asarray(meta["quantized_centroids"]),
                    assignments, meta["omega"], meta["psi"], meta["zero_pinned"])


# ---------------------------------------------------------------------------
# int8 fixed-point sparse conv

@dataclass
class Int8CsrFilter:
    """A CsrFilter of the fixed-point weights plus their int8 codes.

    ``filt`` is exactly the reference's build_csr(linear_quantize(w)) (weights
    that quantise to zero drop out of the CSR, csr.py:99); ``codes`` holds the
    code of every stored entry (0 for padding)."""

    filt: CsrFilter
    codes: np.ndarray
    params: FixedPointParams
    weight_bound: int = field(default=-1, repr=False)  # max_d sum|k_w| (cached)

    @property
    def geometry(self) -> ConvGeometry:
        return self.filt.geometry


@dataclass
class Int8Tensor:
    """int8 fixed-point activations on the device (plain NCHW codes)."""

    codes: object  # torch.int8 CUDA tensor
    params: FixedPointParams

    @property
    def shape(self):
        return tuple(self.codes.shape)

    @property
    def n(self) -> int:
        return int(self.codes.shape[0])


def build_csr_int8(dense_weights: DenseTensor4, geometry: ConvGeometry, total_bits: int = 8,
                   params: FixedPointParams | None = None) -> Int8CsrFilter:
    w = dense_weights.data
    params = params or fit_fixed_point(w, total_bits)
    if params.total_bits > 8:  # codes above 127 would wrap in the int8 payload
        raise ValueError(f"int8 path needs total_bits <= 8, got params with {params.total_bits}")
    wq = linear_quantize(w, params)
    filt = build_csr(DenseTensor4.from_array(wq), geometry)
    codes = np.rint(filt.weights.astype(np.float64) / params.sigma)
    if not np.array_equal(codes * params.sigma, filt.weights.astype(np.float64)):
        raise ValueError("weights are not on the fixed-point grid")
    return Int8CsrFilter(filt, codes.astype(np.int8), params)


def quantize_input_int8(x: DenseTensor4, total_bits: int = 8,
                        params: FixedPointParams | None = None) -> Int8Tensor:
    """Fixed-point codes of the activations (fit_fixed_point + linear_quantize,
    quantization.py:41-76), quantised on the device."""
    import torch
    src = x.device() if isinstance(x, DenseTensor4) else x
    src = src.to(torch.float32).contiguous()
    params = params or fit_fixed_point(src, total_bits)
    if params.total_bits > 8:
        raise ValueError(f"int8 path needs total_bits <= 8, got params with {params.total_bits}")
    codes = torch.empty(src.shape, dtype=torch.int8, device=src.device)
    # clip to the params' own code range, exactly as linear_quantize(x, params)
    _lib.check(_lib.lib().usc_quantize_i8(_lib.t_ptr(src), _lib.t_ptr(codes), src.numel(),
                                          params.sigma, params.total_bits, _lib.stream_ptr()), "quantize")
    return Int8Tensor(codes, params)


def int8_exact_bound(fq: Int8CsrFilter, xq: Int8Tensor, exact: bool = False) -> int:
    """max_d sum_j |k_w| * max|k_x|: below 2**24 every partial sum of the fp32
    reference composition is an exact integer.  Without ``exact`` the activation
    factor is the code limit 2**(bits-1)-1 (no device read); with it, the
    measured max|k_x| (one device->host sync)."""
    if fq.weight_bound < 0:
        fq.weight_bound = int(np.abs(fq.codes.astype(np.int64)).reshape(fq.geometry.out_channels, -1)
                              .sum(axis=1).max())
    per = fq.weight_bound
    if exact:
        return per * int(xq.codes.abs().max().item())
    return per * (2 ** (xq.params.total_bits - 1) - 1)


def sparse_conv_forward_int8(xq: Int8Tensor, fq: Int8CsrFilter, config: ExecConfig | None = None,
                             relu: bool = False) -> DenseTensor4:
    """int32-accumulating sparse conv of int8 codes; fp32 out = acc * sigma_w * sigma_x."""
    import torch
    g = fq.geometry
    if tuple(xq.codes.shape[1:]) != (g.in_channels, g.input_h, g.input_w):
        raise ValueError(f"input shape {tuple(xq.codes.shape[1:])} does not match geometry")
    config = config or ExecConfig()
    n = xq.n
    if n % config.sub_batch:
        raise ValueError(f"sub_batch {config.sub_batch} does not divide batch {n}")
    plan, blob = plan_for(fq.filt, n, _lib.USC_I8, config, fq.codes)
    if plan.kernel == 1 and int8_exact_bound(fq, xq) >= 2 ** 24 and int8_exact_bound(fq, xq, True) >= 2 ** 24:
        # kernel 3 accumulates the code products in fp32 in the reference's order (equal to
        # the composition at any magnitude); kernel 1 accumulates in exact int32
        warnings.warn("int8 partial sums exceed 2**24: the fp32 reference composition rounds, "
                      "kernel 1 accumulates exactly in int32 and may differ from it", RuntimeWarning)
    x_pad = padded_input(xq.codes, plan)
    y = torch.empty((n, g.out_channels, g.out_h, g.out_w), dtype=torch.float32, device=x_pad.device)
    epi = _lib.Epilogue()
    epi.relu = 1 if relu else 0
    epi.scale = float(np.float32(fq.params.sigma * xq.params.sigma))
    launch(plan, blob, x_pad, y, epi)
    return DenseTensor4._adopt(y, PrecisionMode.BINARY32)


# ---------------------------------------------------------------------------
# 4-bit codebook (4b/16b) sparse conv

@dataclass
class CodebookCsrFilter:
    """CsrFilter of the reconstructed codebook weights + a 4-bit index per entry."""

    filt: CsrFilter
    indices: np.ndarray       # uint8, one per stored entry
    table: np.ndarray         # float32[16]: quantized centroids (zero-padded)
    codebook: Codebook

    @property
    def geometry(self) -> ConvGeometry:
        return self.filt.geometry


def build_csr_codebook(dense_weights: DenseTensor4, geometry: ConvGeometry, omega: int = 16,
                       psi: int = 16, codebook: Codebook | None = None) -> CodebookCsrFilter:
    if omega > 16:
        raise ValueError("4-bit codebook needs omega <= 16")
    w = dense_weights.data
    cb = codebook or kmeans_codebook(w, omega, psi)
    wc = cb.reconstruct(w.shape)
    filt = build_csr(DenseTensor4.from_array(wc), geometry)
    table = np.zeros(16, np.float32)
    table[:len(cb.quantized_centroids)] = cb.quantized_centroids.astype(np.float32)
    # entry -> index: look the stored weight up in the table (exact fp32 match)
    idx = np.zeros(filt.weights.size, np.uint8)
    for i, v in enumerate(table[:len(cb.quantized_centroids)]):
        if v != 0.0:
            idx[filt.weights == v] = i
    if not np.array_equal(table[idx], filt.weights):
        raise ValueError("codebook weights do not decode from the table")
    return CodebookCsrFilter(filt, idx, table, cb)


def sparse_conv_forward_codebook(x: DenseTensor4, fc: CodebookCsrFilter,
                                 saturation: float | None = None,
                                 calibrated_max: float | None = None,
                                 config: ExecConfig | None = None) -> DenseTensor4:
    """4b/16b sparse conv: binary16 activations, 4-bit weights decoded to fp32
    centroids, fp32 accumulation in reference order, then the layer's activation
    hook (saturate at `saturation` * calibrated max, round to binary16)."""
    import torch
    g = fc.geometry
    g.check_input(x)
    config = config or ExecConfig()
    if x.n % config.sub_batch:
        raise ValueError(f"sub_batch {config.sub_batch} does not divide batch {x.n}")
    xh = x.device()
    if xh.dtype != torch.float16:
        xh = round_to_binary16(xh).to(torch.float16)
    plan, blob = plan_for(fc.filt, x.n, _lib.USC_CB4, config, fc.indices, fc.table)
    x_pad = padded_input(xh, plan)
    y = torch.empty((x.n, g.out_channels, g.out_h, g.out_w), dtype=torch.float16, device=xh.device)
    epi = _lib.Epilogue()
    if saturation is not None and calibrated_max is not None:
        epi.saturate = 1
        epi.cap = float(np.float32(saturation * float(calibrated_max)))
    launch(plan, blob, x_pad, y, epi)
    return DenseTensor4._adopt(y, PrecisionMode.BINARY16)


# ---------------------------------------------------------------------------
# whole-model quantisation (quantization.py:221-301) for the VGG-16 trunk

def calibrate_activation_maxima(model, X_val, batch_size: int = 64) -> dict:
    """quantization.py:223-235: per-layer activation maxima over one validation pass,
    keyed by the reference's layer index (Conv2D, ReLU, MaxPool2 each count,
    models.vgg16_layer_sequence).  ``model``: a QuantizedModel, a SparseVGG16 or the
    list of pruned conv weights; the pass runs the layers eagerly on the GPU through
    sparse_conv_forward in binary32 without hooks (the reference records, it does not
    modify)."""
    import torch
    from .models import VGG16_CIFAR, vgg16_geometries, vgg16_layer_sequence
    if isinstance(model, QuantizedModel):
        weights = model.weights
    elif hasattr(model, "filters") and hasattr(model, "geoms"):
        weights = None
        filters = [getattr(q, "filt", q) for q in getattr(model, "qfilters", model.filters)]
    else:
        weights = model
    if weights is not None:
        filters = [build_csr(w if isinstance(w, DenseTensor4) else DenseTensor4.from_array(w), g)
                   for w, g in zip(weights, vgg16_geometries())]
    filters = [f if f.precision is PrecisionMode.BINARY32 else
               CsrFilter(f.row_ptr, f.col_offsets, f.weights, f.n_nz, f.geometry) for f in filters]
    seq = vgg16_layer_sequence(VGG16_CIFAR)
    xs = X_val if type(X_val).__module__.startswith("torch") else torch.from_numpy(np.asarray(X_val, np.float32))
    maxima = {}
    for start in range(0, xs.shape[0], batch_size):
        a = xs[start:start + batch_size].to("cuda", torch.float32)
        li = 0
        for i, (kind,) in enumerate(seq):
            if kind == "conv":
                a = sparse_conv_forward(DenseTensor4._adopt(a.contiguous()), filters[li]).device()
                li += 1
            elif kind == "relu":
                a = torch.where(a > 0, a, torch.zeros_like(a))
            else:
                a = torch.nn.functional.max_pool2d(a, 2)
            m = float(a.max().item()) if a.numel() else 0.0
            maxima[i] = max(maxima.get(i, -np.inf), m)
    return maxima


@dataclass
class QuantizedModel:
    """quantization.py:247-254: the quantised pruned weights plus what the activation
    hook needs (calibrated maxima, saturation), and the codebooks of 4b/16b."""

    weights: list
    mode: str
    maxima: dict | None = None
    codebooks: list | None = None
    saturation: float = 0.99

    def network(self, batch: int, device=None, configs=None, calibration=None):
        """The fused sparse VGG-16 trunk for this model (passthrough -> fp32,
        16b/16b -> binary16, 4b/16b -> codebook weights + _half_hook epilogues)."""
        from .models import SparseVGG16
        net_mode = {"passthrough": "fp32", "16b/16b": "fp16", "4b/16b": "cb4"}[self.mode]
        prec = PrecisionMode.BINARY16 if net_mode == "fp16" else PrecisionMode.BINARY32
        return SparseVGG16(self.weights, batch, precision=prec, configs=configs, device=device, mode=net_mode,
                           calibration=calibration, saturation=self.saturation, maxima=self.maxima,
                           codebooks=self.codebooks)


def quantize_model(pruned, mode: str, calibration=None, omega: int = 16, psi: int = 16,
                   saturation: float = 0.99) -> QuantizedModel:
    """quantization.py:257-301 for the pruned VGG-16 trunk (``pruned``: its conv
    weights, DenseTensor4 or arrays, in network order).

    passthrough: binary32 copy.  16b/16b: weights rounded to binary16 (every
    activation is then rounded after each layer by the network's epilogue).
    4b/16b: each prunable weight tensor shared across ``omega`` zero-pinned
    centroids (psi-bit fixed point, kept in binary32), activations binary16 with
    saturation at ``saturation`` x the calibrated per-layer maximum; ``calibration``
    supplies the inputs of the calibration pass.  Masked positions stay zero."""
    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r}; expected one of {MODES}")
    ws = [np.array(w.data if isinstance(w, DenseTensor4) else w, dtype=np.float32) for w in pruned]
    masks = [w != 0 for w in ws]
    if mode == "passthrough":
        return QuantizedModel([DenseTensor4.from_array(w) for w in ws], mode, saturation=saturation)
    if mode == "16b/16b":
        return QuantizedModel([DenseTensor4.from_array(w * m, PrecisionMode.BINARY16) for w, m in zip(ws, masks)],
                              mode, saturation=saturation)
    if calibration is None:
        raise ValueError("4b/16b needs calibration inputs")
    codebooks, qws = [], []
    for w, m in zip(ws, masks):
        cb = kmeans_codebook(w, omega, psi)
        codebooks.append(cb)
        qws.append(DenseTensor4.from_array(cb.reconstruct(w.shape) * m))
    qm = QuantizedModel(qws, mode, codebooks=codebooks, saturation=saturation)
    qm.maxima = calibrate_activation_maxima(qm, calibration)
    return qm
