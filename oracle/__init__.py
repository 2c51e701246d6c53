"""CPU oracle for the direct sparse convolution hot path.

TEST INFRASTRUCTURE ONLY -- this package is the parity checker and the CPU
baseline.  Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg
and ``--impl reference``) may import it; the product package
``paper_2112_15445_b200`` never does.

It restates the reference ``unsparse`` package (/root/reference/pkg/src/unsparse):
  * the numeric hot loop in C (oracle.c, built to liboracle.so by oracle/Makefile),
  * the host-side quantisation primitives and fixture generators in numpy (below).

Parity of this restatement is pinned against the reference itself by the golden
vectors in tests/golden/ (tests/golden/make_golden.py imports the reference in
the build container and records its outputs; tests/test_oracle_golden.py checks
this oracle against them).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import zlib

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_i64 = ctypes.c_int64
_ptr = ctypes.c_void_p


def build() -> str:
    """Compile liboracle.so (gcc) if it is missing or stale."""
    src = os.path.join(_HERE, "oracle.c")
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_csr_nnz.restype = _i64
        L.orc_csr_validate.restype = _i64
        L.orc_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def max_threads() -> int:
    return int(lib().orc_max_threads())


# --------------------------------------------------------------------------
# geometry (tensor.py:156-210)

def geometry_dims(geom):
    """geom = (C, D, Kh, Kw, H, W, (s_h, s_w), (p_h, p_w)) -> derived dims."""
    C, D, Kh, Kw, H, W, (sh, sw), (ph, pw) = geom
    Hp, Wp = H + 2 * ph, W + 2 * pw
    if (Hp - Kh) % sh or (Wp - Kw) % sw or Hp < Kh or Wp < Kw:
        raise ValueError("output dims not integral")  # tensor.py:182-190
    return dict(C=C, D=D, Kh=Kh, Kw=Kw, H=H, W=W, sh=sh, sw=sw, ph=ph, pw=pw, Hp=Hp, Wp=Wp,
                Yh=(Hp - Kh) // sh + 1, Yw=(Wp - Kw) // sw + 1, x_size=C * Hp * Wp)


# --------------------------------------------------------------------------
# numeric hot path (C)

def round_to_binary16(x):
    """tensor.py:48-63."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty_like(a)
    lib().orc_round_to_binary16(_p(a), _p(out), _i64(a.size))
    return out


def build_csr(w: np.ndarray, geom):
    """csr.py:86-112 -> (row_ptr int64[D+1], col_offsets int64[D*n_nz], theta f32, n_nz)."""
    g = geometry_dims(geom)
    w = np.ascontiguousarray(w, dtype=np.float32)
    assert w.shape == (g["D"], g["C"], g["Kh"], g["Kw"])
    L = lib()
    n_nz = int(L.orc_csr_nnz(_p(w), _i64(g["D"]), _i64(g["C"] * g["Kh"] * g["Kw"])))
    rp = np.empty(g["D"] + 1, np.int64)
    col = np.empty(g["D"] * n_nz, np.int64)
    th = np.empty(g["D"] * n_nz, np.float32)
    L.orc_build_csr(_p(w), _i64(g["D"]), _i64(g["C"]), _i64(g["Kh"]), _i64(g["Kw"]),
                    _i64(g["Hp"]), _i64(g["Wp"]), _i64(n_nz), _p(rp), _p(col), _p(th))
    return rp, col, th, n_nz


def csr_validate(rp, col, th, n_nz, geom) -> int:
    """csr.py:66-83; -1 valid, -2 row_ptr, -3 lengths, >=0 first bad offset index."""
    g = geometry_dims(geom)
    rp = np.ascontiguousarray(rp, np.int64)
    col = np.ascontiguousarray(col, np.int64)
    return int(lib().orc_csr_validate(_p(rp), _i64(rp.size), _i64(col.size), _i64(np.size(th)),
                                      _p(col), _i64(n_nz), _i64(g["D"]), _i64(g["Kh"]),
                                      _i64(g["Kw"]), _i64(g["Hp"]), _i64(g["Wp"]),
                                      _i64(g["x_size"])))


def sparse_conv_forward(x: np.ndarray, csr, geom, sb: int = 1, binary16: bool = False,
                        threads: int = 1) -> np.ndarray:
    """engine.py:64-111 with kernels.py:57-100 as the inner loop."""
    g = geometry_dims(geom)
    x = np.ascontiguousarray(x, dtype=np.float32)
    n = x.shape[0]
    assert x.shape[1:] == (g["C"], g["H"], g["W"])
    if n % sb:
        raise ValueError(f"sub_batch {sb} does not divide batch {n}")  # engine.py:81-82
    rp, col, th, n_nz = csr
    rp = np.ascontiguousarray(rp, np.int64)
    col = np.ascontiguousarray(col, np.int64)
    th = np.ascontiguousarray(th, np.float32)
    out = np.empty((n, g["D"], g["Yh"], g["Yw"]), np.float32)
    lib().orc_sparse_conv_forward(
        _p(x), _i64(n), _i64(g["C"]), _i64(g["H"]), _i64(g["W"]), _p(rp), _p(col), _p(th),
        _i64(g["D"]), _i64(g["Kh"]), _i64(g["Kw"]), _i64(g["sh"]), _i64(g["sw"]),
        _i64(g["ph"]), _i64(g["pw"]), _i64(sb), ctypes.c_int(1 if binary16 else 0), _p(out),
        ctypes.c_int(threads))
    return out


def sparse_conv_blocks(xflat, rp, col, th, out_shape, blocks, sb, x_size, s_h, s_w, padded_w,
                       threads: int = 1, out=None):
    """kernels.py:57-100 FFI-shaped; writes only the blocks' output slices."""
    n, D, Yh, Yw = out_shape
    xflat = np.ascontiguousarray(xflat, np.float32)
    rp = np.ascontiguousarray(rp, np.int64)
    col = np.ascontiguousarray(col, np.int64)
    th = np.ascontiguousarray(th, np.float32)
    blocks = np.ascontiguousarray(blocks, np.int64).reshape(-1, 2)
    if out is None:
        out = np.zeros(out_shape, np.float32)
    lib().orc_sparse_conv_blocks(_p(xflat), _p(rp), _p(col), _p(th), _p(out), _i64(D), _i64(Yh),
                                 _i64(Yw), _p(blocks), _i64(blocks.shape[0]), _i64(sb),
                                 _i64(x_size), _i64(s_h), _i64(s_w), _i64(padded_w),
                                 ctypes.c_int(threads))
    return out


def zero_pad(x, geom):
    g = geometry_dims(geom)
    x = np.ascontiguousarray(x, np.float32)
    n = x.shape[0]
    xp = np.empty((n, g["C"], g["Hp"], g["Wp"]), np.float32)
    lib().orc_zero_pad(_p(x), _i64(n), _i64(g["C"]), _i64(g["H"]), _i64(g["W"]), _i64(g["ph"]),
                       _i64(g["pw"]), _p(xp))
    return xp


def dense_conv(x, w, geom, binary16=False, threads: int = 1):
    """tensor.py:247-292 / kernels.py:16-54."""
    g = geometry_dims(geom)
    xp = zero_pad(x, geom)
    w = np.ascontiguousarray(w, np.float32)
    n = xp.shape[0]
    out = np.empty((n, g["D"], g["Yh"], g["Yw"]), np.float32)
    lib().orc_dense_conv(_p(xp), _i64(n), _i64(g["C"]), _i64(g["Hp"]), _i64(g["Wp"]), _p(w),
                         _i64(g["D"]), _i64(g["Kh"]), _i64(g["Kw"]), _i64(g["sh"]), _i64(g["sw"]),
                         _p(out), _i64(g["Yh"]), _i64(g["Yw"]), ctypes.c_int(threads))
    return round_to_binary16(out) if binary16 else out


def conv_grad_weights(xpad, dout, s_h: int, s_w: int, kh: int, kw: int, threads: int = 1):
    """kernels.py:103-130: dw (D, C, Kh, Kw) from the padded input and the output gradient."""
    xpad = np.ascontiguousarray(xpad, np.float32)
    dout = np.ascontiguousarray(dout, np.float32)
    n, C, Hp, Wp = xpad.shape
    D, Yh, Yw = dout.shape[1:]
    dw = np.zeros((D, C, kh, kw), np.float32)
    lib().orc_conv_grad_weights(_p(xpad), _p(dout), _p(dw), _i64(n), _i64(C), _i64(Hp), _i64(Wp), _i64(D),
                                _i64(kh), _i64(kw), _i64(Yh), _i64(Yw), _i64(s_h), _i64(s_w), ctypes.c_int(threads))
    return dw


def conv_grad_input(w, dout, xpad_shape, s_h: int, s_w: int, threads: int = 1):
    """kernels.py:133-162: dxpad (zero-initialised, nn.py:67) from the weights and the
    output gradient."""
    w = np.ascontiguousarray(w, np.float32)
    dout = np.ascontiguousarray(dout, np.float32)
    n, C, Hp, Wp = xpad_shape
    D, _, Kh, Kw = w.shape
    Yh, Yw = dout.shape[2:]
    dxpad = np.zeros(xpad_shape, np.float32)
    lib().orc_conv_grad_input(_p(w), _p(dout), _p(dxpad), _i64(n), _i64(C), _i64(Hp), _i64(Wp), _i64(D),
                              _i64(Kh), _i64(Kw), _i64(Yh), _i64(Yw), _i64(s_h), _i64(s_w), ctypes.c_int(threads))
    return dxpad


def relu(x):
    """nn.py:96-98."""
    x = np.ascontiguousarray(x, np.float32)
    out = np.empty_like(x)
    lib().orc_relu(_p(x), _p(out), _i64(x.size))
    return out


def maxpool2(x):
    """nn.py:124-135."""
    x = np.ascontiguousarray(x, np.float32)
    n, c, h, w = x.shape
    out = np.empty((n, c, h // 2, w // 2), np.float32)
    lib().orc_maxpool2(_p(x), _p(out), _i64(n * c), _i64(h), _i64(w))
    return out


# --------------------------------------------------------------------------
# quantisation primitives (numpy restatement of quantization.py)

def fit_fixed_point(tensor, total_bits: int):
    """quantization.py:41-58 -> dict(total_bits, int_bits, frac_bits, sigma, degenerate)."""
    if total_bits < 2:
        raise ValueError("total_bits must be >= 2")
    arr = np.asarray(tensor)
    amax = float(np.max(np.abs(arr)))
    degenerate = amax == 0.0
    int_bits = 0 if degenerate else int(math.ceil(math.log2(amax)))
    frac = total_bits - int_bits - 1
    return dict(total_bits=total_bits, int_bits=int_bits, frac_bits=frac, sigma=2.0 ** (-frac),
                mu=0.0, degenerate=degenerate)


def linear_quantize(x, p):
    """quantization.py:61-76 (round half away from zero, symmetric clip)."""
    arr = np.asarray(x, dtype=np.float64)
    scaled = (arr - p["mu"]) / p["sigma"]
    codes = np.copysign(np.floor(np.abs(scaled) + 0.5), scaled)
    limit = float(2 ** (p["total_bits"] - 1) - 1)
    codes = np.clip(codes, -limit, limit)
    q = p["mu"] + p["sigma"] * codes
    if np.isscalar(x) or np.ndim(x) == 0:
        return float(q)
    return q.astype(np.asarray(x).dtype) if np.asarray(x).dtype.kind == "f" else q


def linear_codes(x, p):
    """The integer codes behind linear_quantize (same rounding and clip)."""
    arr = np.asarray(x, dtype=np.float64)
    scaled = (arr - p["mu"]) / p["sigma"]
    codes = np.copysign(np.floor(np.abs(scaled) + 0.5), scaled)
    limit = float(2 ** (p["total_bits"] - 1) - 1)
    return np.clip(codes, -limit, limit)


def saturate_activations(a, thr, calibrated_max=None):
    """quantization.py:79-93."""
    arr = np.asarray(a)
    m = float(np.max(arr)) if calibrated_max is None else float(calibrated_max)
    return np.minimum(arr, thr * m)


def _kmeans_1d(values, k, max_iter=100):
    """quantization.py:112-131."""
    uniq = np.unique(values)
    k = min(k, uniq.size)
    seeds = uniq[np.minimum((np.arange(k) + 0.5) / k * uniq.size, uniq.size - 1).astype(int)]
    centroids = seeds.astype(np.float64)
    assign = None
    for _ in range(max_iter):
        dist = np.abs(values[:, None] - centroids[None, :])
        new_assign = dist.argmin(axis=1)
        if assign is not None and np.array_equal(new_assign, assign):
            break
        assign = new_assign
        for j in range(k):
            sel = values[assign == j]
            if sel.size:
                centroids[j] = sel.mean()
    return centroids, assign


def kmeans_codebook(weights, omega: int, psi: int = 16):
    """quantization.py:134-180 -> dict(centroids, quantized_centroids, assignments, zero_pinned)."""
    flat = np.asarray(weights, dtype=np.float64).ravel()
    nz = flat[flat != 0]
    zero_pinned = nz.size < flat.size
    budget = omega - 1 if zero_pinned else omega
    if nz.size == 0:
        centroids = np.array([0.0])
        assignments = np.zeros(flat.size, dtype=np.int64)
    else:
        nz_c, nz_a = _kmeans_1d(nz, budget)
        if zero_pinned:
            centroids = np.concatenate([[0.0], nz_c])
            assignments = np.zeros(flat.size, dtype=np.int64)
            assignments[flat != 0] = nz_a + 1
        else:
            centroids = nz_c
            assignments = nz_a.astype(np.int64)
    params = fit_fixed_point(centroids, psi)
    quantized = np.asarray([linear_quantize(float(c), params) for c in centroids], np.float64)
    if zero_pinned:
        quantized[0] = 0.0
    return dict(centroids=centroids, quantized_centroids=quantized, assignments=assignments,
                zero_pinned=zero_pinned, omega=omega, psi=psi)


def codebook_reconstruct(cb, shape):
    """Codebook.reconstruct, quantization.py:108-109."""
    return cb["quantized_centroids"][cb["assignments"]].reshape(shape).astype(np.float32)


# --------------------------------------------------------------------------
# fixture generators (restated so they run where the reference is absent)

KERNELS = [(1, 1), (3, 3), (3, 1), (2, 1)]  # verify.py:20


def random_case(rng, binary16=False):
    """verify.py:23-52 -> (x, w, geom, sb); same RNG draw sequence as the reference."""
    kh, kw = KERNELS[rng.integers(len(KERNELS))]
    c = int(rng.integers(1, 17))
    d = int(rng.integers(1, 17))
    s_h = int(rng.integers(1, 3))
    s_w = int(rng.integers(1, 3))
    h_pad = int(rng.integers(0, 2))
    w_pad = int(rng.integers(0, 2)) if kw > 1 else 0
    y_h = int(rng.integers(1, 7))
    y_w = int(rng.integers(1, 7)) if kw > 1 else 1
    x_h = (y_h - 1) * s_h + kh - 2 * h_pad
    x_w = (y_w - 1) * s_w + kw - 2 * w_pad
    if x_h < 1 or x_w < 1:
        h_pad = w_pad = 0
        x_h = (y_h - 1) * s_h + kh
        x_w = (y_w - 1) * s_w + kw
    geom = (c, d, kh, kw, x_h, x_w, (s_h, s_w), (h_pad, w_pad))
    batch = int(2 ** rng.integers(0, 4))
    sparsity = float(rng.uniform(0.0, 0.99))
    w = rng.standard_normal((d, c, kh, kw)).astype(np.float32)
    kz = int(np.floor(sparsity * w.size))
    if kz:
        w.reshape(-1)[rng.choice(w.size, kz, replace=False)] = 0.0
    x = rng.standard_normal((batch, c, x_h, x_w)).astype(np.float32)
    if binary16:
        w = round_to_binary16(w)
        x = round_to_binary16(x)
    sbs = [s for s in (1, 2, 4, 8) if batch % s == 0]
    sb = int(sbs[rng.integers(len(sbs))])
    return x, w, geom, sb


def synthesize_masked_weights(shape, sparsity, rng, binary16=False):
    """bench.py:84-95: N(0,1) weights with exactly floor(s*size) zeros."""
    w = rng.standard_normal(shape).astype(np.float32)
    size = w.size
    k = int(np.floor(sparsity * size))
    if k:
        w.reshape(-1)[rng.choice(size, size=k, replace=False)] = 0.0
    return round_to_binary16(w) if binary16 else w


def bench_rng(name: str, sparsity: float, seed: int = 0):
    """bench.py:160-161 seeding."""
    return np.random.default_rng([seed, zlib.crc32(name.encode()), int(round(sparsity * 1000))])
