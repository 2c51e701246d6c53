"""Parity of the sm_100a kernels with the reference, through the product API and
the C ABI.  Bitwise for fp32 (the reference's per-element mul-then-add order),
fp16, int8 and the 4-bit codebook path; checked against the golden digests the
reference produced (tests/golden) and against the oracle at larger sizes."""
import numpy as np
import pytest

import oracle
import paper_2112_15445_b200 as U
from golden_util import arrays, geom, golden, layer_inputs, sha

pytestmark = pytest.mark.gpu

F32, F16 = U.PrecisionMode.BINARY32, U.PrecisionMode.BINARY16


def G(t):
    c, d, kh, kw, h, w, s, p = t
    return U.ConvGeometry(c, d, kh, kw, h, w, tuple(s), tuple(p))


def _dev(x, prec=F32):
    import torch
    return U.DenseTensor4.from_array(torch.from_numpy(np.ascontiguousarray(x)).cuda(), prec)


@pytest.mark.parametrize("kernel", [0, 1, 2, 3])
def test_random_corpus_bitwise(kernel):
    """The reference's own oracle corpus (verify.py:55-69), 400 cases: every GPU
    output is bit-identical to the reference's sparse_conv_forward."""
    rng = np.random.default_rng([0, 1])
    for rec in golden()["random_cases"]:
        x, w, g, sb = oracle.random_case(rng, binary16=rec["binary16"])
        prec = F16 if rec["binary16"] else F32
        filt = U.build_csr(U.DenseTensor4.from_array(w, prec), G(rec["geometry"]))
        out = U.sparse_conv_forward(U.DenseTensor4.from_array(x, prec), filt,
                                    U.ExecConfig(sb, kernel=kernel))
        assert sha(out.data) == rec["sparse_out"], (rec["i"], rec["geometry"])


def test_random_corpus_dense_reference():
    rng = np.random.default_rng([0, 1])
    for rec in golden()["random_cases"][:120]:
        x, w, g, sb = oracle.random_case(rng, binary16=rec["binary16"])
        prec = F16 if rec["binary16"] else F32
        out = U.dense_conv_reference(U.DenseTensor4.from_array(x, prec),
                                     U.DenseTensor4.from_array(w, prec), G(rec["geometry"]))
        assert sha(out.data) == rec["dense_out"], rec["i"]


def test_reference_shaped_blocks_kernel():
    """usc_sparse_conv_blocks: the numba FFI kernels.sparse_conv_blocks on device arrays."""
    import torch
    rng = np.random.default_rng([0, 1])
    for rec in golden()["random_cases"][:100]:
        x, w, g, sb = oracle.random_case(rng, binary16=rec["binary16"])
        if rec["binary16"]:
            continue
        gg = G(rec["geometry"])
        f = U.build_csr(U.DenseTensor4.from_array(w), gg)
        xflat = torch.from_numpy(oracle.zero_pad(x, g).reshape(-1)).cuda()
        blocks = np.array([(b.out_channel, b.sample_start) for b in U.plan_blocks(gg, x.shape[0], sb)],
                          np.int64)
        out = torch.zeros((x.shape[0], gg.out_channels, gg.out_h, gg.out_w), device="cuda")
        cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        U.engine.sparse_conv_blocks(xflat, cu(f.row_ptr), cu(f.col_offsets), cu(f.weights), out,
                                    cu(blocks), sb, gg.x_size, gg.stride[0], gg.stride[1], gg.padded_w)
        assert sha(out.cpu().numpy()) == rec["sparse_out"], rec["i"]


def test_nonfinite_inputs_propagate_like_reference():
    arr = arrays()
    for rec in golden()["nonfinite_cases"]:
        k = rec["k"]
        gg = G(rec["geometry"])
        f = U.build_csr(U.DenseTensor4.from_array(arr[f"nf{k}_w"]), gg)
        for kernel in (0, 1, 2, 3):
            got = U.sparse_conv_forward(_dev(arr[f"nf{k}_x"]), f, U.ExecConfig(kernel=kernel)).data
            ref = arr[f"nf{k}_out"]
            assert np.array_equal(np.isnan(got), np.isnan(ref))
            m = ~np.isnan(ref)
            assert np.array_equal(got[m], ref[m])


LAYERS = ["cfg1-vgg16-256x8", "cfg1-vgg16-256x8-f16", "vgg16-512x14", "resnet50-1x1-64x256",
          "resnet50-1x1-256x64", "cnn1d-300x64-k2", "cnn1d-300x64-k3", "resnet-3x3-s2-prepad",
          "resnet-1x1-s2-crop", "sweep-3x3-256x8-98", "sweep-3x3-64x32-50"]


@pytest.mark.parametrize("name", LAYERS)
def test_layer_configs_bitwise_all_tiles(name):
    """Every tile configuration the autotuner may pick gives the same bits
    (schedule determinism, verify.py:139-150) and they equal the reference."""
    rec = golden()["layers"][name]
    g = geom(rec["geometry"])
    prec = F16 if rec["binary16"] else F32
    x, w = layer_inputs(name, g, rec["sparsity"], rec["batch"], rec["binary16"])
    gg = G(rec["geometry"])
    f = U.build_csr(U.DenseTensor4.from_array(w, prec), gg)
    xd = _dev(x, prec)
    cfgs = [U.ExecConfig(), U.ExecConfig(kernel=2), U.ExecConfig(kernel=1)] + \
        U.engine.tile_candidates(gg, rec["batch"], [1, 2], prec)
    # the opt-in tensor-memory kernel (kernel 4): a spread of its tiles
    cfgs += U.engine.tile_candidates(gg, rec["batch"], [1, 2], prec, kernels=(4,))[::7]
    # the opt-in register-window variant (k_bw): every tile
    cfgs += U.engine.tile_candidates(gg, rec["batch"], [1, 2], prec, kernels=(5,))
    for cfg in cfgs:
        out = U.sparse_conv_forward(xd, f, cfg)
        assert sha(out.data) == rec["out"], cfg


@pytest.mark.parametrize("name", ["int8-vgg16-256x8", "int8-vgg16-64x32", "int8-1x1-256x64"])
def test_int8_kernel_equals_reference_composition(name):
    rec = golden()["int8"][name]
    g = geom(rec["geometry"])
    x, w = layer_inputs(name, g, rec["sparsity"], rec["batch"])
    gg = G(rec["geometry"])
    fq = U.build_csr_int8(U.DenseTensor4.from_array(w), gg)
    xq = U.quantize_input_int8(_dev(x))
    assert xq.params.sigma == rec["sigma_x"]
    for cfg in (U.ExecConfig(), U.ExecConfig(kernel=1), U.ExecConfig(kernel=2)):
        out = U.sparse_conv_forward_int8(xq, fq, cfg)
        assert sha(out.data) == rec["out"], cfg


@pytest.mark.parametrize("name", ["cb4-vgg16-256x8", "cb4-vgg16-128x16"])
def test_codebook_kernel_equals_reference_composition(name):
    rec = golden()["cb4"][name]
    g = geom(rec["geometry"])
    x, w = layer_inputs(name, g, rec["sparsity"], rec["batch"])
    gg = G(rec["geometry"])
    fc = U.build_csr_codebook(U.DenseTensor4.from_array(w), gg)
    x16 = _dev(oracle.round_to_binary16(x), F16)
    for cfg in (U.ExecConfig(), U.ExecConfig(kernel=1), U.ExecConfig(kernel=2)):
        plain = U.sparse_conv_forward_codebook(x16, fc, config=cfg)
        assert sha(plain.data) == sha(oracle.round_to_binary16(_conv_ref(x16.data, fc, g)))
        out = U.sparse_conv_forward_codebook(x16, fc, 0.99, rec["calibrated_max"], config=cfg)
        assert sha(out.data) == rec["out"], cfg


def _conv_ref(x, fc, g):
    csr = (fc.filt.row_ptr, fc.filt.col_offsets, fc.filt.weights, fc.filt.n_nz)
    return oracle.sparse_conv_forward(x, csr, g, threads=4)


def test_vgg16_network_matches_reference_composition():
    """The fused VGG-16 pipeline (conv+ReLU epilogue, pools, padded buffers) equals
    the reference's sparse_conv_forward + nn.ReLU + nn.MaxPool2 composition."""
    import zlib

    import torch
    from paper_2112_15445_b200.models import SparseVGG16, vgg16_weights
    rec = golden()["vgg16"]
    rng = np.random.default_rng([0, zlib.crc32(b"vgg16-cifar10"), int(round(rec["sparsity"] * 1000))])
    x = rng.standard_normal((rec["batch"], 3, 32, 32)).astype(np.float32)
    ws = vgg16_weights(rng, rec["sparsity"])
    m = SparseVGG16(ws, rec["batch"])
    out = m.forward(torch.from_numpy(x).cuda())
    assert sha(out.cpu().numpy()) == rec["out"]
    m.capture()
    out2 = m.forward(torch.from_numpy(x).cuda())
    assert sha(out2.cpu().numpy()) == rec["out"]


@pytest.mark.parametrize("special", [False, True])
def test_vgg16_batch64_vs_oracle(special):
    """Larger batch against the oracle (the reference's algorithm restated in C);
    `special` adds NaN / +-inf input pixels (ReLU maps NaN to 0, nn.py:96-98)."""
    import torch
    from paper_2112_15445_b200.models import VGG16_CIFAR, SparseVGG16, vgg16_rng, vgg16_weights
    rng = vgg16_rng(0.93, seed=5)
    ws = vgg16_weights(rng, 0.93)
    x = rng.standard_normal((64, 3, 32, 32)).astype(np.float32)
    if special:
        x[0, 0, 5, 5], x[1, 1, 7, 7], x[2, 2, 9, 9] = np.nan, np.inf, -np.inf
    m = SparseVGG16(ws, 64)
    got = m.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    a, li = x, 0
    for v in VGG16_CIFAR:
        if v == "M":
            a = oracle.maxpool2(a)
            continue
        g = m.geoms[li]
        gt = (g.in_channels, g.out_channels, 3, 3, g.input_h, g.input_w, (1, 1), (1, 1))
        a = oracle.relu(oracle.sparse_conv_forward(a, oracle.build_csr(ws[li].data, gt), gt,
                                                   threads=oracle.max_threads()))
        li += 1
    assert np.array_equal(got, a)


def test_cfg1_full_batch_vs_oracle_and_autotune():
    rec = golden()["layers"]["cfg1-vgg16-256x8"]
    g = geom(rec["geometry"])
    x, w = layer_inputs("cfg1-vgg16-256x8", g, 0.9, 32)
    gg = G(rec["geometry"])
    f = U.build_csr(U.DenseTensor4.from_array(w), gg)
    xd = _dev(x)
    cfg = U.autotune_sb(xd, f, repeats=3, warmup=1)
    assert cfg.sub_batch in (1, 2, 4, 8)
    out = U.sparse_conv_forward(xd, f, cfg)
    assert sha(out.data) == rec["out"]


def test_round_to_binary16_device():
    import torch
    rng = np.random.default_rng(3)
    x = (rng.standard_normal(100000) * np.exp(rng.uniform(-20, 12, 100000))).astype(np.float32)
    got = U.round_to_binary16(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(got, oracle.round_to_binary16(x))


@pytest.mark.parametrize("special", [False, True])
def test_vgg16_binary16_network_vs_oracle(special):
    """BINARY16 VGG-16 on the BI64 kernel (FHFMA, binary16 epilogue + fused pool)
    against the reference composition: binary16 conv (fp32 accumulate, saturating
    RNE output, engine.py:109-110), ReLU, max-pool.  `special`: inputs scaled so
    layer outputs overflow binary16 (saturation to 65504) plus NaN / +-inf pixels."""
    import torch
    from paper_2112_15445_b200.models import VGG16_CIFAR, SparseVGG16, vgg16_rng, vgg16_weights
    rng = vgg16_rng(0.93, seed=7)
    ws = vgg16_weights(rng, 0.93, precision=F16)
    x = rng.standard_normal((64, 3, 32, 32)).astype(np.float32)
    if special:
        x *= 4096.0
        x[0, 0, 5, 5], x[1, 1, 7, 7], x[2, 2, 9, 9] = np.nan, np.inf, -np.inf
    x = oracle.round_to_binary16(x)
    m = SparseVGG16(ws, 64, precision=F16)
    assert m.interleave == 64
    got = m.forward(torch.from_numpy(x).cuda().half()).float().cpu().numpy()
    a, li = x, 0
    for v in VGG16_CIFAR:
        if v == "M":
            a = oracle.maxpool2(a)
            continue
        g = m.geoms[li]
        gt = (g.in_channels, g.out_channels, 3, 3, g.input_h, g.input_w, (1, 1), (1, 1))
        a = oracle.relu(oracle.sparse_conv_forward(a, oracle.build_csr(ws[li].data, gt), gt, binary16=True,
                                                   threads=oracle.max_threads()))
        li += 1
    assert np.array_equal(got, a)


def _vgg_oracle(m, x, conv_fn):
    """Reference composition of the VGG-16 trunk with a per-layer conv function."""
    from paper_2112_15445_b200.models import VGG16_CIFAR
    a, li = x, 0
    for v in VGG16_CIFAR:
        if v == "M":
            a = oracle.maxpool2(a)
            continue
        g = m.geoms[li]
        gt = (g.in_channels, g.out_channels, 3, 3, g.input_h, g.input_w, (1, 1), (1, 1))
        a = conv_fn(li, a, gt)
        li += 1
    return a


def test_vgg16_int8_network_vs_oracle():
    """8-bit fixed-point VGG-16 (calibrated per-layer input scales, requantising
    epilogue) equals the reference composition layer by layer: linear_quantize the
    input with the layer's sigma, sparse_conv_forward with build_csr(linear_quantize(w)),
    ReLU, max-pool (quantization.py:41-76, csr.py:86-112, engine.py:64-111)."""
    import torch
    from paper_2112_15445_b200.models import SparseVGG16, vgg16_rng, vgg16_weights
    rng = vgg16_rng(0.93, seed=11)
    ws = vgg16_weights(rng, 0.93)
    x = rng.standard_normal((64, 3, 32, 32)).astype(np.float32)
    m = SparseVGG16(ws, 64, mode="int8", calibration=torch.from_numpy(x).cuda())
    got = m.forward(torch.from_numpy(x).cuda()).cpu().numpy()

    def conv(li, a, gt):
        s = m.sigmas[li]
        p = dict(total_bits=s.total_bits, sigma=s.sigma, mu=0.0)
        xq = oracle.linear_quantize(a.astype(np.float32), p)
        f = m.filters[li]
        return oracle.relu(oracle.sparse_conv_forward(xq, (f.row_ptr, f.col_offsets, f.weights, f.n_nz), gt,
                                                      threads=oracle.max_threads()))
    assert np.array_equal(got, _vgg_oracle(m, x, conv))


def test_vgg16_int8_requant_shift_range_vs_oracle():
    """The integer requantisation (round-half-away by shift, clamp to +-127) across its
    shift range: every later layer's input sigma is made 2^6 finer than calibrated, so
    every epilogue shift is 6 smaller (many codes clamp at +-127) while the reference
    composition requantises with the same sigmas in fp64."""
    import dataclasses
    import torch
    from paper_2112_15445_b200.models import SparseVGG16, vgg16_rng, vgg16_weights
    rng = vgg16_rng(0.93, seed=12)
    ws = vgg16_weights(rng, 0.93)
    x = rng.standard_normal((64, 3, 32, 32)).astype(np.float32)
    m = SparseVGG16(ws, 64, mode="int8", calibration=torch.from_numpy(x).cuda())
    for li in range(1, len(m.geoms)):
        s = m.sigmas[li]
        m.sigmas[li] = dataclasses.replace(s, int_bits=s.int_bits - 6, frac_bits=s.frac_bits + 6, sigma=s.sigma / 64)
    for li in range(len(m.geoms)):
        p = m.layer_params[li]
        p["scale"] = float(np.float32(m.qfilters[li].params.sigma * m.sigmas[li].sigma))
        if li + 1 < len(m.geoms):
            p["rq_scale"] = float(np.float32(1.0 / m.sigmas[li + 1].sigma))
    m._build()
    got = m.forward(torch.from_numpy(x).cuda()).cpu().numpy()

    def conv(li, a, gt):
        s = m.sigmas[li]
        xq = oracle.linear_quantize(a.astype(np.float32), dict(total_bits=s.total_bits, sigma=s.sigma, mu=0.0))
        f = m.filters[li]
        return oracle.relu(oracle.sparse_conv_forward(xq, (f.row_ptr, f.col_offsets, f.weights, f.n_nz), gt,
                                                      threads=oracle.max_threads()))
    assert np.array_equal(got, _vgg_oracle(m, x, conv))


def test_vgg16_codebook_network_vs_oracle():
    """4b/16b VGG-16: codebook weights, binary16 activations with the _half_hook
    saturation at 0.99 x the calibrated conv / ReLU maxima (quantization.py:223-301)."""
    import torch
    from paper_2112_15445_b200.models import SparseVGG16, vgg16_rng, vgg16_weights
    rng = vgg16_rng(0.93, seed=13)
    ws = vgg16_weights(rng, 0.93)
    x = oracle.round_to_binary16(rng.standard_normal((64, 3, 32, 32)).astype(np.float32))
    m = SparseVGG16(ws, 64, mode="cb4", calibration=torch.from_numpy(x).cuda())
    got = m.forward(torch.from_numpy(x).cuda().half()).float().cpu().numpy()

    def conv(li, a, gt):
        f, lp = m.filters[li], m.layer_params[li]
        y = oracle.sparse_conv_forward(a, (f.row_ptr, f.col_offsets, f.weights, f.n_nz), gt,
                                       threads=oracle.max_threads())
        y = oracle.round_to_binary16(np.minimum(y, np.float32(lp["cap"])))
        y = oracle.relu(y)
        return oracle.round_to_binary16(np.minimum(y, np.float32(lp["cap2"])))
    assert np.array_equal(got, _vgg_oracle(m, x, conv))


@pytest.mark.parametrize("name", ["cfg1-vgg16-256x8", "vgg16-512x14", "resnet50-1x1-64x256", "sweep-3x3-256x8-98",
                                  "cnn1d-300x64-k3"])
def test_device_encoder_bitwise(name):
    """usc_build_csr_device == build_csr (csr.py:86-112): RP, Lambda, theta, n_nz."""
    import torch
    rec = golden()["layers"][name]
    g = geom(rec["geometry"])
    _, w = layer_inputs(name, g, rec["sparsity"], rec["batch"], rec["binary16"])
    gg = G(rec["geometry"])
    host = U.build_csr(U.DenseTensor4.from_array(w), gg)
    dev = U.build_csr_device(torch.from_numpy(np.ascontiguousarray(w)).cuda(), gg)
    assert dev.n_nz == host.n_nz == rec["csr"]["n_nz"]
    assert np.array_equal(dev.row_ptr, host.row_ptr) and np.array_equal(dev.col_offsets, host.col_offsets)
    assert np.array_equal(dev.weights.view(np.uint32), host.weights.view(np.uint32))
    for k in ("row_ptr", "col_offsets", "weights"):  # and the reference's own digests
        assert sha(getattr(dev, k)) == rec["csr"][k]
    zero = np.zeros_like(w)
    assert U.build_csr_device(torch.from_numpy(zero).cuda(), gg).n_nz == 1  # max(1, 0)


def test_stream_forward_matches_forward():
    """The overlapped streaming API returns exactly forward()'s features, in order."""
    import torch
    from paper_2112_15445_b200.models import SparseVGG16, vgg16_rng, vgg16_weights
    rng = vgg16_rng(0.93, seed=3)
    m = SparseVGG16(vgg16_weights(rng, 0.93), 64)
    xs = [torch.from_numpy(rng.standard_normal((64, 3, 32, 32)).astype(np.float32)).pin_memory() for _ in range(5)]
    outs = [torch.empty((64, 512, 1, 1)).pin_memory() for _ in range(5)]
    m.capture()
    m.stream_forward(xs, outs).synchronize()
    for x, o in zip(xs, outs):
        assert torch.equal(m.forward(x.cuda()).cpu(), o)


@pytest.mark.parametrize("prec,scale", [(F32, 1.0), (F16, 1.0), (F16, 256.0)])
def test_resnet50_network_vs_oracle(prec, scale):
    """ResNet-50 CIFAR (53 sparse convs, stride-2 exact-geometry views, residual add +
    ReLU fused into conv3) against the composition of the reference's pieces: per conv
    sparse_conv_forward (binary16 hook for fp16), ReLU, and the block output
    relu(conv3 + shortcut) (fp16: relu(round16(round16(conv3) + shortcut)))."""
    import torch
    from paper_2112_15445_b200.resnet import SparseResNet50, resnet50_layers, resnet50_weights
    ws = resnet50_weights(0.9, seed=2, precision=prec)
    rng = np.random.default_rng(9)
    x = rng.standard_normal((64, 3, 32, 32)).astype(np.float32) * np.float32(scale)
    if prec is F16:
        x = oracle.round_to_binary16(x)
    m = SparseResNet50(ws, 64, precision=prec)
    xd = torch.from_numpy(x).cuda()
    got = m.forward(xd.half() if prec is F16 else xd).float().cpu().numpy()

    layers = resnet50_layers()
    hook = oracle.round_to_binary16 if prec is F16 else (lambda a: a)

    def conv(li, a):
        name, g, role, s = layers[li]
        if role == "c2" and s == 2:
            a = np.pad(a, ((0, 0), (0, 0), (1, 0), (1, 0)))
        if role == "proj" and s == 2:
            a = np.ascontiguousarray(a[:, :, :g.input_h, :g.input_w])
        gt = (g.in_channels, g.out_channels, g.filter_h, g.filter_w, g.input_h, g.input_w, g.stride, g.padding)
        csr = oracle.build_csr(np.ascontiguousarray(ws[li].data), gt)
        return hook(oracle.sparse_conv_forward(a, csr, gt, threads=oracle.max_threads()))

    a = oracle.relu(conv(0, x))
    li = 1
    from paper_2112_15445_b200.resnet import STAGES
    for width, blocks, stride in STAGES:
        for b in range(blocks):
            h1 = oracle.relu(conv(li, a))
            h2 = oracle.relu(conv(li + 1, h1))
            li += 2
            if b == 0:
                sc = conv(li, a)
                li += 1
            else:
                sc = a
            y = conv(li, h2)
            li += 1
            a = oracle.relu(hook((y + sc).astype(np.float32)))
    assert np.array_equal(got, a)


def test_conv_gradients_bitwise_vs_reference():
    """Training kernels: usc_conv_grad_weights / usc_conv_grad_input
    and Conv2D.backward equal the reference's kernels.py:103-162 / nn.py:62-72 outputs
    (golden vectors) bit for bit; the forward equals the oracle's dense conv."""
    import torch
    from golden_util import grad_cases
    from paper_2112_15445_b200 import training as T
    for g, a in grad_cases():
        geom = U.ConvGeometry(g["C"], g["D"], g["Kh"], g["Kw"], g["H"], g["W"], stride=(g["sh"], g["sw"]),
                              padding=(g["ph"], g["pw"]))
        layer = T.Conv2D(geom, np.random.default_rng(0))
        layer.w = a["w"].copy()
        y = layer.forward(torch.from_numpy(a["x"]).cuda())
        gt = (g["C"], g["D"], g["Kh"], g["Kw"], g["H"], g["W"], (g["sh"], g["sw"]), (g["ph"], g["pw"]))
        assert np.array_equal(y.cpu().numpy(), oracle.dense_conv(a["x"], a["w"], gt)), g
        dx = layer.backward(torch.from_numpy(a["dout"]).cuda())
        assert np.array_equal(layer.grad_w, a["dw"]), g
        assert np.array_equal(dx.cpu().numpy(), a["dx"]), g
        dxpad = torch.full(a["dxpad"].shape, float("nan"), device="cuda")  # every element is written
        T.conv_grad_input(torch.from_numpy(a["w"]).cuda(), torch.from_numpy(a["dout"]).cuda(), dxpad,
                          g["sh"], g["sw"])
        assert np.array_equal(dxpad.cpu().numpy(), a["dxpad"]), g


def test_conv_gradients_vgg_layer_vs_oracle():
    """A VGG-sized pruned layer (64->64 3x3 at 16x16, batch 8) against the oracle's
    restatement (pinned to the reference by the golden cases above)."""
    import torch
    from paper_2112_15445_b200 import training as T
    rng = np.random.default_rng(5)
    n, C, D, H = 8, 64, 64, 16
    xpad = np.pad(rng.standard_normal((n, C, H, H)).astype(np.float32), ((0, 0), (0, 0), (1, 1), (1, 1)))
    w = rng.standard_normal((D, C, 3, 3)).astype(np.float32)
    w.reshape(-1)[rng.choice(w.size, int(w.size * 0.9), replace=False)] = 0.0
    dout = rng.standard_normal((n, D, H, H)).astype(np.float32)
    dw = torch.empty((D, C, 3, 3), device="cuda")
    T.conv_grad_weights(torch.from_numpy(xpad).cuda(), torch.from_numpy(dout).cuda(), dw, 1, 1)
    assert np.array_equal(dw.cpu().numpy(), oracle.conv_grad_weights(xpad, dout, 1, 1, 3, 3, threads=4))
    dxpad = torch.empty(xpad.shape, device="cuda")
    T.conv_grad_input(torch.from_numpy(w).cuda(), torch.from_numpy(dout).cuda(), dxpad, 1, 1)
    assert np.array_equal(dxpad.cpu().numpy(), oracle.conv_grad_input(w, dout, xpad.shape, 1, 1, threads=4))


@pytest.mark.parametrize("name", ["cfg1-vgg16-256x8", "cfg1-vgg16-256x8-f16", "resnet50-1x1-64x256"])
def test_native_autotune_c_abi(name):
    """usc_autotune (the C-ABI tile search, engine.py:139-170): its pick runs and is
    bitwise equal to the reference's output."""
    from paper_2112_15445_b200.engine import autotune_native
    rec = golden()["layers"][name]
    g = geom(rec["geometry"])
    prec = F16 if rec["binary16"] else F32
    x, w = layer_inputs(name, g, rec["sparsity"], rec["batch"], binary16=rec["binary16"])
    f = U.build_csr(U.DenseTensor4.from_array(w, prec), G(rec["geometry"]))
    xd = _dev(x, prec)
    cfg = autotune_native(xd, f, repeats=3, warmup=1)
    assert cfg.kernel in (1, 3)
    assert sha(U.sparse_conv_forward(xd, f, cfg).data) == rec["out"]


def test_run_bench_harness_on_gpu():
    """layer_bench.run_bench (bench.py:143-166) end to end on the GPU: presets x
    precisions x sparsities with the reference's seeding, CSV round trip and the
    per-layer backend choice (bench.py:212-227); the timed sparse layer equals the
    reference's output on the same seeded inputs."""
    import zlib
    from paper_2112_15445_b200 import layer_bench as LB
    rep = LB.run_bench({"layers": ["cnn1d-300x64-k2", "resnet50-1x1-256x64"], "sparsities": [0.9],
                        "precisions": ["binary32", "binary16"], "batch": 8, "repeats": 3, "warmup": 1})
    assert len(rep.rows) == 4 and rep.environment["gpu"]
    for r in rep.rows:
        assert r.sparse_ms > 0 and r.dense_ms > 0 and r.dense_backend == "cudnn"
    rows = LB.rows_from_csv(LB.rows_to_csv(rep.rows))
    cfg = LB.backend_config(rows, expected_layers=[r.layer_id for r in rep.rows])
    assert set(v["backend"] for v in cfg.values()) <= {"sparse", "dense"}
    # the seeded layer the harness timed, recomputed, against the oracle
    g = LB.preset_geometry("resnet50-1x1-256x64")
    rng = np.random.default_rng([0, zlib.crc32(b"resnet50-1x1-256x64"), 900])
    w = U.pruning.synthesize_masked_weights(g, 0.9, rng)
    x = rng.standard_normal((8, g.in_channels, g.input_h, g.input_w)).astype(np.float32)
    f = U.build_csr(w, g)
    out = U.sparse_conv_forward(_dev(x), f).data
    gt = (g.in_channels, g.out_channels, 1, 1, g.input_h, g.input_w, (1, 1), (0, 0))
    ref = oracle.sparse_conv_forward(x, (f.row_ptr, f.col_offsets, f.weights, f.n_nz), gt)
    assert np.array_equal(out, ref)

