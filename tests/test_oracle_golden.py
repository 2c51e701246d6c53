"""Pin the CPU oracle (oracle/) to the reference's own outputs (tests/golden/).

CPU-only: these tests run everywhere and make the oracle trustworthy as the
parity checker for the CUDA path.
"""
import numpy as np
import pytest

import oracle
from golden_util import arrays, geom, golden, layer_inputs, sha

VGG16_CIFAR = [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M"]


def test_round_to_binary16_kats():
    k = golden()["kats"]
    vals = oracle.round_to_binary16(np.array([0.1, 70000.0, -70000.0, 65519.0, 65520.0], np.float32))
    assert vals.tolist() == [k["round16_0.1"], k["round16_70000"], k["round16_-70000"],
                             k["round16_65519"], k["round16_65520"]]
    assert k["round16_0.1"] == 0.0999755859375 and k["round16_70000"] == 65504.0


def test_round_to_binary16_matches_numpy_grid():
    rng = np.random.default_rng(3)
    x = (rng.standard_normal(100000) * np.exp(rng.uniform(-20, 12, 100000))).astype(np.float32)
    ref = x.astype(np.float16).astype(np.float32)
    ref = np.where(np.isinf(ref) & np.isfinite(x), np.copysign(np.float32(65504.0), x), ref)
    assert np.array_equal(oracle.round_to_binary16(x), ref)


def test_encoder_spec_examples():
    k = golden()["kats"]
    e = k["encoder_D2"]
    rp, col, th, n_nz = oracle.build_csr(np.array(e["weights"], np.float32), geom(e["geometry"]))
    assert n_nz == e["n_nz"] == 3
    assert rp.tolist() == e["row_ptr"] == [0, 3, 6]
    assert col.tolist() == e["col_offsets"] == [0, 0, 4, 0, 5, 8]
    assert th.tolist() == e["theta"] == [0, 0, 5, 1, 2, 3]
    z = k["encoder_all_zero"]
    rp, col, th, n_nz = oracle.build_csr(np.zeros((3, 2, 3, 3), np.float32),
                                         (2, 3, 3, 3, 5, 5, (1, 1), (1, 1)))
    assert n_nz == z["n_nz"] == 1 and rp.tolist() == z["row_ptr"]
    assert col.tolist() == z["col_offsets"] and th.tolist() == z["theta"]


def test_dense_kat():
    x = np.array([[[[1, 2], [3, 4]]]], np.float32)
    out = oracle.dense_conv(x, np.ones((1, 1, 2, 2), np.float32), (1, 1, 2, 2, 2, 2, (1, 1), (0, 0)))
    assert out.ravel()[0] == golden()["kats"]["dense_2x2_ones"] == 10.0


def test_quantisation_kats():
    k = golden()["kats"]
    for amax, (ib, fb, sg) in k["fit_fixed_point"].items():
        p = oracle.fit_fixed_point(np.array([float(amax), -0.1]), 8)
        assert (p["int_bits"], p["frac_bits"], p["sigma"]) == (ib, fb, sg)
    assert oracle.linear_quantize(0.7, oracle.fit_fixed_point(np.array([1.0]), 8)) == k["linear_quantize_0.7"] == 0.703125
    assert oracle.linear_quantize(3.2, oracle.fit_fixed_point(np.array([3.2]), 8)) == k["linear_quantize_3.2"] == 3.1875
    cb = oracle.kmeans_codebook(np.array([1.0, 1.1, -2.0, -2.1]), 2)
    assert cb["centroids"].tolist() == k["kmeans_4pts"]["centroids"]
    assert cb["assignments"].tolist() == k["kmeans_4pts"]["assignments"]
    assert cb["quantized_centroids"].tolist() == k["kmeans_4pts"]["quantized"]


def test_random_corpus_bitwise():
    """400 random_case()s (verify.py:23-52): generator, encoder, sparse conv and
    dense conv all bit-identical to the reference."""
    rng = np.random.default_rng([0, 1])
    arr = arrays()
    for rec in golden()["random_cases"]:
        x, w, g, sb = oracle.random_case(rng, binary16=rec["binary16"])
        assert list(g[:6]) == rec["geometry"][:6] and sb == rec["sb"]
        assert sha(x) == rec["x"] and sha(w) == rec["w"], rec["i"]
        csr = oracle.build_csr(w, g)
        assert csr[3] == rec["csr"]["n_nz"]
        assert sha(csr[0]) == rec["csr"]["row_ptr"] and sha(csr[1]) == rec["csr"]["col_offsets"]
        assert sha(csr[2]) == rec["csr"]["weights"]
        out = oracle.sparse_conv_forward(x, csr, g, sb=sb, binary16=rec["binary16"], threads=2)
        assert sha(out) == rec["sparse_out"], rec["i"]
        dense = oracle.dense_conv(x, w, g, binary16=rec["binary16"])
        assert sha(dense) == rec["dense_out"], rec["i"]
        key = f"case{rec['i']}_out"
        if key in arr:
            assert np.array_equal(arr[key], out)


def test_nonfinite_cases():
    arr = arrays()
    for rec in golden()["nonfinite_cases"]:
        k = rec["k"]
        g = geom(rec["geometry"])
        out = oracle.sparse_conv_forward(arr[f"nf{k}_x"], oracle.build_csr(arr[f"nf{k}_w"], g), g)
        ref = arr[f"nf{k}_out"]
        assert np.array_equal(np.isnan(out), np.isnan(ref))
        assert np.isnan(ref).any()
        m = ~np.isnan(ref)
        assert np.array_equal(out[m], ref[m])


@pytest.mark.parametrize("name", ["cfg1-vgg16-256x8", "cfg1-vgg16-256x8-f16", "vgg16-512x14",
                                  "resnet50-1x1-64x256", "resnet50-1x1-256x64", "cnn1d-300x64-k2",
                                  "cnn1d-300x64-k3", "resnet-3x3-s2-prepad", "resnet-1x1-s2-crop",
                                  "sweep-3x3-256x8-98", "sweep-3x3-64x32-50"])
def test_layer_configs_bitwise(name):
    rec = golden()["layers"][name]
    g = geom(rec["geometry"])
    x, w = layer_inputs(name, g, rec["sparsity"], rec["batch"], rec["binary16"])
    assert sha(x) == rec["x"] and sha(w) == rec["w"]
    csr = oracle.build_csr(w, g)
    assert csr[3] == rec["csr"]["n_nz"] and sha(csr[1]) == rec["csr"]["col_offsets"]
    out = oracle.sparse_conv_forward(x, csr, g, binary16=rec["binary16"], threads=oracle.max_threads())
    assert sha(out) == rec["out"]


@pytest.mark.parametrize("name", ["int8-vgg16-256x8", "int8-vgg16-64x32", "int8-1x1-256x64"])
def test_int8_composition(name):
    rec = golden()["int8"][name]
    g = geom(rec["geometry"])
    x, w = layer_inputs(name, g, rec["sparsity"], rec["batch"])
    pw, px = oracle.fit_fixed_point(w, 8), oracle.fit_fixed_point(x, 8)
    assert pw["sigma"] == rec["sigma_w"] and px["sigma"] == rec["sigma_x"]
    wq, xq = oracle.linear_quantize(w, pw), oracle.linear_quantize(x, px)
    assert sha(wq) == rec["wq"] and sha(xq) == rec["xq"]
    csr = oracle.build_csr(wq, g)
    out = oracle.sparse_conv_forward(xq, csr, g, threads=oracle.max_threads())
    assert sha(out) == rec["out"]
    # integer-code identity: fp32 result == int32 acc * sigma_w * sigma_x
    kw_ = oracle.linear_codes(w, pw).astype(np.int64)
    kx_ = oracle.linear_codes(x, px).astype(np.int64)
    ref_int = oracle.dense_conv(kx_.astype(np.float64).astype(np.float32), kw_.astype(np.float32), g)
    assert np.array_equal(ref_int * np.float32(pw["sigma"] * px["sigma"]), out)


@pytest.mark.parametrize("name", ["cb4-vgg16-256x8", "cb4-vgg16-128x16"])
def test_codebook_composition(name):
    rec = golden()["cb4"][name]
    g = geom(rec["geometry"])
    x, w = layer_inputs(name, g, rec["sparsity"], rec["batch"])
    cb = oracle.kmeans_codebook(w, 16, 16)
    assert cb["centroids"].tolist() == rec["centroids"]
    assert cb["quantized_centroids"].tolist() == rec["quantized_centroids"]
    assert sha(cb["assignments"]) == rec["assignments"]
    wc = oracle.codebook_reconstruct(cb, w.shape)
    x16 = oracle.round_to_binary16(x)
    conv = oracle.sparse_conv_forward(x16, oracle.build_csr(wc, g), g, threads=oracle.max_threads())
    assert sha(conv) == rec["conv"]
    out = oracle.round_to_binary16(oracle.saturate_activations(conv, 0.99, rec["calibrated_max"]))
    assert sha(out) == rec["out"]


def test_vgg16_trunk_composition():
    import zlib
    rec = golden()["vgg16"]
    rng = np.random.default_rng([0, zlib.crc32(b"vgg16-cifar10"), int(round(rec["sparsity"] * 1000))])
    x = rng.standard_normal((rec["batch"], 3, 32, 32)).astype(np.float32)
    assert sha(x) == rec["x"]
    a, c, hw = x, 3, 32
    for v, lr in zip(VGG16_CIFAR, rec["layers"]):
        if v == "M":
            a = oracle.maxpool2(a)
            hw //= 2
        else:
            g = (c, v, 3, 3, hw, hw, (1, 1), (1, 1))
            w = oracle.synthesize_masked_weights((v, c, 3, 3), rec["sparsity"], rng)
            assert sha(w) == lr["w"]
            a = oracle.relu(oracle.sparse_conv_forward(a, oracle.build_csr(w, g), g, threads=4))
            c = v
        assert sha(a) == lr["out"]
    assert sha(a) == rec["out"]


def test_conv_gradients_match_reference():
    """kernels.py:103-162: the oracle's conv_grad_weights (fp64
    accumulator, b/r/cc order) and conv_grad_input (fp32 scatter order) equal the
    reference's outputs bit for bit, including the Yw == 1 loops and stride 2."""
    from golden_util import grad_cases
    for g, a in grad_cases():
        xpad = np.pad(a["x"], ((0, 0), (0, 0), (g["ph"], g["ph"]), (g["pw"], g["pw"])))
        dw = oracle.conv_grad_weights(xpad, a["dout"], g["sh"], g["sw"], g["Kh"], g["Kw"], threads=4)
        dxpad = oracle.conv_grad_input(a["w"], a["dout"], xpad.shape, g["sh"], g["sw"], threads=4)
        assert np.array_equal(dw, a["dw"]), g
        assert np.array_equal(dxpad, a["dxpad"]), g
        dx = dxpad[:, :, g["ph"]:g["ph"] + g["H"], g["pw"]:g["pw"] + g["W"]]
        assert np.array_equal(dx, a["dx"]), g
