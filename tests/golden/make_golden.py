"""Generate the golden vectors that pin the oracle (and the CUDA path) to the reference.

Run ONLY in the build container, where the read-only reference exists:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports the UNMODIFIED reference package from /root/reference/pkg/src, runs
its public API on seeded synthetic inputs and records
  * golden.json  -- SPEC known-answer tests, sha256 digests of every output,
                    CSR arrays and generated input (so the numpy restatement
                    of the fixture generators is pinned too);
  * small_cases.npz -- full arrays for the small random cases and the
                    non-finite edge cases.
Nothing on the GPU box reads /root/reference; the tests read these files.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import zlib

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF)

import unsparse as U  # noqa: E402  (the reference)
from unsparse import bench as RB  # noqa: E402
from unsparse import csr as RC  # noqa: E402
from unsparse import nn as RN  # noqa: E402
from unsparse import verify as RV  # noqa: E402
from unsparse.tensor import PrecisionMode  # noqa: E402

F32, F16 = PrecisionMode.BINARY32, PrecisionMode.BINARY16


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def geom_tuple(g):
    return [g.in_channels, g.out_channels, g.filter_h, g.filter_w, g.input_h, g.input_w,
            list(g.stride), list(g.padding)]


def csr_record(f):
    return dict(n_nz=int(f.n_nz), row_ptr=sha(f.row_ptr), col_offsets=sha(f.col_offsets),
                weights=sha(f.weights))


def kats():
    out = {}
    out["round16_0.1"] = U.round_to_binary16(0.1)
    out["round16_70000"] = U.round_to_binary16(70000.0)
    out["round16_-70000"] = U.round_to_binary16(-70000.0)
    out["round16_65519"] = U.round_to_binary16(65519.0)
    out["round16_65520"] = U.round_to_binary16(65520.0)
    g = U.ConvGeometry(1, 1, 2, 2, 2, 2)
    x = U.DenseTensor4.from_array(np.array([[[[1, 2], [3, 4]]]], np.float32))
    w = U.DenseTensor4.from_array(np.ones((1, 1, 2, 2), np.float32))
    out["dense_2x2_ones"] = float(U.dense_conv_reference(x, w, g).data.ravel()[0])
    out["tap_offset_0_1_2_in_4x4"] = RC.tap_to_offset(0, 1, 2, U.ConvGeometry(1, 1, 3, 3, 4, 4))
    # SPEC:117 D=2 example: channel 0 one nonzero, channel 1 three
    g2 = U.ConvGeometry(1, 2, 3, 3, 3, 3)
    w2 = np.zeros((2, 1, 3, 3), np.float32)
    w2[0, 0, 1, 1] = 5.0
    w2[1, 0, 0, 0], w2[1, 0, 1, 2], w2[1, 0, 2, 2] = 1.0, 2.0, 3.0
    f2 = U.build_csr(U.DenseTensor4.from_array(w2), g2)
    out["encoder_D2"] = dict(weights=w2.tolist(), geometry=geom_tuple(g2), n_nz=int(f2.n_nz),
                             row_ptr=f2.row_ptr.tolist(), col_offsets=f2.col_offsets.tolist(),
                             theta=f2.weights.tolist())
    fz = U.build_csr(U.DenseTensor4.from_array(np.zeros((3, 2, 3, 3), np.float32)),
                     U.ConvGeometry(2, 3, 3, 3, 5, 5, padding=(1, 1)))
    out["encoder_all_zero"] = dict(n_nz=int(fz.n_nz), row_ptr=fz.row_ptr.tolist(),
                                   col_offsets=fz.col_offsets.tolist(), theta=fz.weights.tolist())
    out["plan_blocks_128_64_4"] = len(U.plan_blocks(U.ConvGeometry(3, 64, 3, 3, 8, 8, padding=(1, 1)), 128, 4))
    fps = {}
    for amax in (1.0, 3.2, 0.4):
        p = U.fit_fixed_point(np.array([amax, -0.1]), 8)
        fps[str(amax)] = [p.int_bits, p.frac_bits, p.sigma]
    out["fit_fixed_point"] = fps
    p = U.fit_fixed_point(np.array([1.0]), 8)
    out["linear_quantize_0.7"] = U.linear_quantize(0.7, p)
    p = U.fit_fixed_point(np.array([3.2]), 8)
    out["linear_quantize_3.2"] = U.linear_quantize(3.2, p)
    cb = U.kmeans_codebook(np.array([1.0, 1.1, -2.0, -2.1]), 2)
    out["kmeans_4pts"] = dict(centroids=cb.centroids.tolist(),
                              assignments=cb.assignments.tolist(),
                              quantized=cb.quantized_centroids.tolist())
    # 1D example: length 300, 64 channels, kernel 2x1 -> 299
    g1 = U.ConvGeometry(64, 64, 2, 1, 300, 1)
    out["conv1d_300_k2_out_h"] = g1.out_h
    return out


def random_corpus(seed=0, cases=400, keep_full=80):
    """check_oracle_equivalence's exact case sequence (verify.py:55-69)."""
    rng = np.random.default_rng([seed, 1])
    recs, arrays = [], {}
    for i in range(cases):
        precision = F16 if i % 4 == 3 else F32
        inp, weights, geometry, cfg = RV.random_case(rng, precision)
        filt = U.build_csr(weights, geometry)
        got = U.sparse_conv_forward(inp, filt, cfg).data
        ref = U.dense_conv_reference(inp, weights, geometry).data
        recs.append(dict(i=i, binary16=precision is F16, geometry=geom_tuple(geometry),
                         sb=cfg.sub_batch, x=sha(inp.data), w=sha(weights.data),
                         csr=csr_record(filt), sparse_out=sha(got), dense_out=sha(ref),
                         bitwise_sparse_eq_dense=bool(np.array_equal(got, ref))))
        if i < keep_full:
            arrays[f"case{i}_out"] = got
    return recs, arrays


def nonfinite_cases():
    """Inputs with inf/nan: padding entries (weight 0 at offset 0) turn them into NaN."""
    rng = np.random.default_rng([7, 7])
    arrays, recs = {}, []
    for k, (c, d, kh, kw, h, w, pad) in enumerate([(3, 5, 3, 3, 6, 6, 1), (4, 6, 1, 1, 5, 5, 0),
                                                    (2, 4, 3, 1, 7, 1, 1)]):
        g = U.ConvGeometry(c, d, kh, kw, h, w, padding=(pad, pad if kw > 1 else 0))
        wt = rng.standard_normal((d, c, kh, kw)).astype(np.float32)
        wt.reshape(-1)[rng.choice(wt.size, wt.size * 2 // 3, replace=False)] = 0.0
        x = rng.standard_normal((2, c, h, w)).astype(np.float32)
        x.reshape(-1)[rng.choice(x.size, 3, replace=False)] = [np.inf, -np.inf, np.nan]
        filt = U.build_csr(U.DenseTensor4.from_array(wt), g)
        out = U.sparse_conv_forward(U.DenseTensor4.from_array(x), filt, U.ExecConfig(1)).data
        arrays[f"nf{k}_x"], arrays[f"nf{k}_w"], arrays[f"nf{k}_out"] = x, wt, out
        recs.append(dict(k=k, geometry=geom_tuple(g)))
    return recs, arrays


def layer_case(name, geometry, sparsity, batch, precision=F32, seed=0):
    """bench_layer's input generation (bench.py:98-108, seeding bench.py:160-161)."""
    rng = np.random.default_rng([seed, zlib.crc32(name.encode()), int(round(sparsity * 1000))])
    weights = RB.synthesize_masked_weights(geometry, sparsity, rng, precision)
    x = U.DenseTensor4.from_array(
        rng.standard_normal((batch, geometry.in_channels, geometry.input_h,
                             geometry.input_w)).astype(np.float32), precision)
    return x, weights


def csr_file_digests(filt):
    """sha256 of the bytes the reference's save_csr writes (binary + JSON sidecar)."""
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "filt.csr")
        RC.save_csr(filt, path)
        with open(path, "rb") as fh:
            binary = hashlib.sha256(fh.read()).hexdigest()
        with open(path + ".json", "rb") as fh:
            sidecar = hashlib.sha256(fh.read()).hexdigest()
    return dict(binary=binary, sidecar=sidecar)


def layer_records():
    recs = {}
    specs = [
        ("cfg1-vgg16-256x8", U.ConvGeometry(256, 256, 3, 3, 8, 8, padding=(1, 1)), 0.9, 32, F32),
        ("cfg1-vgg16-256x8-f16", U.ConvGeometry(256, 256, 3, 3, 8, 8, padding=(1, 1)), 0.9, 8, F16),
        ("vgg16-512x14", U.ConvGeometry(**RB.PRESETS["vgg16-512x14"]), 0.92, 2, F32),
        ("resnet50-1x1-64x256", U.ConvGeometry(**RB.PRESETS["resnet50-1x1-64x256"]), 0.9, 8, F32),
        ("resnet50-1x1-256x64", U.ConvGeometry(**RB.PRESETS["resnet50-1x1-256x64"]), 0.9, 8, F16),
        ("cnn1d-300x64-k2", U.ConvGeometry(**RB.PRESETS["cnn1d-300x64-k2"]), 0.83, 8, F32),
        ("cnn1d-300x64-k3", U.ConvGeometry(**RB.PRESETS["cnn1d-300x64-k3"]), 0.875, 8, F16),
        ("resnet-3x3-s2-prepad", U.ConvGeometry(64, 128, 3, 3, 33, 33, stride=(2, 2)), 0.9, 4, F32),
        ("resnet-1x1-s2-crop", U.ConvGeometry(64, 128, 1, 1, 31, 31, stride=(2, 2)), 0.9, 4, F32),
        ("sweep-3x3-256x8-98", U.ConvGeometry(256, 256, 3, 3, 8, 8, padding=(1, 1)), 0.98, 16, F32),
        ("sweep-3x3-64x32-50", U.ConvGeometry(64, 64, 3, 3, 32, 32, padding=(1, 1)), 0.5, 2, F32),
    ]
    for name, g, s, n, prec in specs:
        x, w = layer_case(name, g, s, n, prec)
        filt = U.build_csr(w, g)
        out = U.sparse_conv_forward(x, filt, U.ExecConfig(1)).data
        recs[name] = dict(geometry=geom_tuple(g), sparsity=s, batch=n, binary16=prec is F16,
                          x=sha(x.data), w=sha(w.data), csr=csr_record(filt), out=sha(out),
                          csr_file=csr_file_digests(filt))
    return recs


def int8_records():
    """int8 = the reference's primitives composed: fixed-point codes for
    weights and inputs, build_csr AFTER quantisation, fp32 sparse conv."""
    recs = {}
    for name, g, s, n in [("int8-vgg16-256x8", U.ConvGeometry(256, 256, 3, 3, 8, 8, padding=(1, 1)), 0.93, 8),
                          ("int8-vgg16-64x32", U.ConvGeometry(64, 64, 3, 3, 32, 32, padding=(1, 1)), 0.93, 2),
                          ("int8-1x1-256x64", U.ConvGeometry(256, 64, 1, 1, 14, 14), 0.9, 4)]:
        x, w = layer_case(name, g, s, n)
        pw, px = U.fit_fixed_point(w.data, 8), U.fit_fixed_point(x.data, 8)
        wq = U.linear_quantize(w.data, pw)
        xq = U.linear_quantize(x.data, px)
        filt = U.build_csr(U.DenseTensor4.from_array(wq), g)
        out = U.sparse_conv_forward(U.DenseTensor4.from_array(xq), filt, U.ExecConfig(1)).data
        recs[name] = dict(geometry=geom_tuple(g), sparsity=s, batch=n,
                          sigma_w=pw.sigma, sigma_x=px.sigma, frac_w=pw.frac_bits,
                          frac_x=px.frac_bits, wq=sha(wq), xq=sha(xq), csr=csr_record(filt),
                          out=sha(out))
    return recs


def cb4_records():
    """4b/16b: codebook weights (fp32 fixed-point centroids), binary16 inputs, fp32
    conv, then the _half_hook epilogue (quantization.py:238-244): saturate at
    0.99*calibrated max, round to binary16."""
    recs = {}
    for name, g, s, n in [("cb4-vgg16-256x8", U.ConvGeometry(256, 256, 3, 3, 8, 8, padding=(1, 1)), 0.93, 8),
                          ("cb4-vgg16-128x16", U.ConvGeometry(128, 128, 3, 3, 16, 16, padding=(1, 1)), 0.93, 2)]:
        x, w = layer_case(name, g, s, n)
        cb = U.kmeans_codebook(w.data, 16, 16)
        wc = cb.reconstruct(w.data.shape)
        x16 = U.round_to_binary16(x.data)
        filt = U.build_csr(U.DenseTensor4.from_array(wc), g)
        conv = U.sparse_conv_forward(U.DenseTensor4.from_array(x16), filt, U.ExecConfig(1)).data
        cal = float(conv.max()) * 0.9  # a calibrated max below the batch max -> saturation bites
        hook = __import__("unsparse.quantization", fromlist=["_half_hook"])._half_hook(0.99, {0: cal})
        out = hook(0, conv)
        recs[name] = dict(geometry=geom_tuple(g), sparsity=s, batch=n,
                          centroids=cb.centroids.tolist(),
                          quantized_centroids=cb.quantized_centroids.tolist(),
                          assignments=sha(cb.assignments), wc=sha(wc), x16=sha(x16),
                          calibrated_max=cal, conv=sha(conv), out=sha(out))
    return recs


VGG16_CIFAR = [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M"]


def vgg_record(batch=2, sparsity=0.93, seed=0):
    """Full VGG-16 CIFAR-10 conv trunk composed from the reference's public pieces:
    sparse_conv_forward + nn.ReLU + nn.MaxPool2."""
    rng = np.random.default_rng([seed, zlib.crc32(b"vgg16-cifar10"), int(round(sparsity * 1000))])
    x = rng.standard_normal((batch, 3, 32, 32)).astype(np.float32)
    c, hw = 3, 32
    layers = []
    a = x
    for v in VGG16_CIFAR:
        if v == "M":
            a = RN.MaxPool2().forward(a)
            hw //= 2
            layers.append(dict(kind="pool", out=sha(a)))
            continue
        g = U.ConvGeometry(c, v, 3, 3, hw, hw, padding=(1, 1))
        w = RB.synthesize_masked_weights(g, sparsity, rng)
        filt = U.build_csr(w, g)
        a = U.sparse_conv_forward(U.DenseTensor4.from_array(a), filt, U.ExecConfig(1)).data
        a = RN.ReLU().forward(a)
        layers.append(dict(kind="conv", cin=c, cout=v, hw=hw, w=sha(w.data), n_nz=int(filt.n_nz),
                           out=sha(a)))
        c = v
    return dict(batch=batch, sparsity=sparsity, x=sha(x), layers=layers, out=sha(a))


def main():
    golden = {"reference": "/root/reference/pkg/src/unsparse", "numpy": np.__version__}
    golden["kats"] = kats()
    recs, arrays = random_corpus()
    golden["random_cases"] = recs
    nrec, narr = nonfinite_cases()
    golden["nonfinite_cases"] = nrec
    arrays.update(narr)
    golden["layers"] = layer_records()
    golden["int8"] = int8_records()
    golden["cb4"] = cb4_records()
    golden["vgg16"] = vgg_record()
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(golden, fh, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **arrays)
    print("wrote", len(recs), "random cases,", len(golden["layers"]), "layers")


if __name__ == "__main__":
    main()
