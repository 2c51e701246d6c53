"""The benchmarked plans themselves, parity-pinned against the oracle.

bench.py and tools/bench_variants.py time networks with committed autotuner
results (profiles/r01_tuned.json, profiles/r02_tuned_*.json).  These tests load
exactly those tiles at the benchmarked batch sizes and compare the outputs with
the reference's algorithm (the oracle composition, layer by layer):

  * VGG-16 CIFAR at batch 256 in all four modes (fp32 / 16b/16b / int8 / 4b/16b);
  * ResNet-50 CIFAR at batch 256 (fp32, 16b/16b);
  * every sparsity-sweep point at batch 1024 (its resident-layout launch), on
    samples from the first, a middle and the last sample block.

Bitwise throughout (the path's parity bar for fp32 and for the quantised modes;
binary16 is bit-exact too).  Reference loops: engine.py:64-111, nn.py:96-135,
quantization.py:41-301; schedule invariance verify.py:139-150.
"""
import json
import os

import numpy as np
import pytest

import oracle
import paper_2112_15445_b200 as U

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
F32, F16 = U.PrecisionMode.BINARY32, U.PrecisionMode.BINARY16


def tuned(name):
    p = os.path.join(ROOT, "profiles", "r01_tuned.json" if name == "vgg16_fp32" else f"r02_tuned_{name}.json")
    if not os.path.exists(p):
        pytest.fail(f"committed tuned state {p} is missing")
    with open(p) as fh:
        return json.load(fh)


def vgg_oracle(m, x, conv_fn):
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


def _csr(f):
    return (f.row_ptr, f.col_offsets, f.weights, f.n_nz)


@pytest.mark.parametrize("mode", ["fp32", "fp16", "int8", "cb4"])
def test_vgg16_benchmarked_tiles_b256_vs_oracle(mode):
    """bench.py's workload (fp32: its weights, batch, tiles and CUDA graph) and the
    bench_variants quantised networks, 256 images, against the oracle composition."""
    import torch
    from paper_2112_15445_b200.models import SparseVGG16, vgg16_rng, vgg16_weights
    batch, th = 256, oracle.max_threads()
    prec = F16 if mode == "fp16" else F32
    ws = vgg16_weights(vgg16_rng(0.93, 0), 0.93, precision=prec)
    x = np.random.default_rng([1, 0]).standard_normal((batch, 3, 32, 32)).astype(np.float32)
    if mode in ("fp16", "cb4"):
        x = oracle.round_to_binary16(x)
    xd = torch.from_numpy(x).cuda()
    kw = dict(mode=mode, calibration=xd) if mode in ("int8", "cb4") else dict(precision=prec)
    m = SparseVGG16(ws, batch, **kw)
    m.load_tuned_state(tuned(f"vgg16_{mode}"))
    m.capture()
    got = m.forward(xd.half() if mode in ("fp16", "cb4") else xd).float().cpu().numpy()

    def conv(li, a, gt):
        f = m.filters[li]
        if mode == "int8":
            s = m.sigmas[li]
            a = oracle.linear_quantize(a.astype(np.float32), dict(total_bits=s.total_bits, sigma=s.sigma, mu=0.0))
        y = oracle.sparse_conv_forward(a, _csr(f), gt, binary16=mode == "fp16", threads=th)
        if mode == "cb4":
            lp = m.layer_params[li]
            y = oracle.round_to_binary16(np.minimum(y, np.float32(lp["cap"])))
            return oracle.round_to_binary16(np.minimum(oracle.relu(y), np.float32(lp["cap2"])))
        return oracle.relu(y)
    assert np.array_equal(got, vgg_oracle(m, x, conv))


@pytest.mark.parametrize("prec_name", ["fp32", "fp16"])
def test_resnet50_benchmarked_tiles_b256_vs_oracle(prec_name):
    """ResNet-50 CIFAR with the committed tiles at batch 256 (bench_variants'
    resnet50-net-<prec>), the whole batch against the oracle composition."""
    import torch
    from paper_2112_15445_b200.resnet import STAGES, SparseResNet50, resnet50_layers, resnet50_weights
    prec = F16 if prec_name == "fp16" else F32
    ws = resnet50_weights(0.9, 0, prec)
    x = np.random.default_rng(21).standard_normal((256, 3, 32, 32)).astype(np.float32)
    if prec is F16:
        x = oracle.round_to_binary16(x)
    m = SparseResNet50(ws, 256, precision=prec)
    m.load_tuned_state(tuned(f"resnet50_{prec_name}"))
    m.capture()
    xd = torch.from_numpy(x).cuda()
    got = m.forward(xd.half() if prec is F16 else xd).float().cpu().numpy()
    layers = resnet50_layers()
    hook = oracle.round_to_binary16 if prec is F16 else (lambda a: a)
    th = oracle.max_threads()

    def conv(li, a):
        _, g, role, s = layers[li]
        if role == "c2" and s == 2:
            a = np.pad(a, ((0, 0), (0, 0), (1, 0), (1, 0)))
        if role == "proj" and s == 2:
            a = np.ascontiguousarray(a[:, :, :g.input_h, :g.input_w])
        gt = (g.in_channels, g.out_channels, g.filter_h, g.filter_w, g.input_h, g.input_w, g.stride, g.padding)
        return hook(oracle.sparse_conv_forward(a, oracle.build_csr(np.ascontiguousarray(ws[li].data), gt), gt,
                                               threads=th))

    a = oracle.relu(conv(0, x))
    li = 1
    for width, blocks, stride in STAGES:
        for b in range(blocks):
            h2 = oracle.relu(conv(li + 1, oracle.relu(conv(li, a))))
            li += 2
            if b == 0:
                sc = conv(li, a)
                li += 1
            else:
                sc = a
            a = oracle.relu(hook((conv(li, h2) + sc).astype(np.float32)))
            li += 1
    assert np.array_equal(got, a)


SWEEP_SHAPES = {"r50-3x3-64x32": (64, 64, 3, 32), "r50-3x3-256x8": (256, 256, 3, 8),
                "r50-1x1-64x256-32": (64, 256, 1, 32), "r50-1x1-256x64-32": (256, 64, 1, 32)}


def test_sweep_benchmarked_tiles_b1024_vs_oracle():
    """Every configs[4] sweep point with its committed tile at batch 1024, launched as
    bench_variants times it (resident BI layout, zero halo), then unpacked; samples of
    the first, a middle and the last sample block against the oracle."""
    import torch
    from paper_2112_15445_b200 import _lib
    from paper_2112_15445_b200.engine import ExecConfig, launch, padded_input, plan_for
    from paper_2112_15445_b200.pruning import synthesize_masked_weights
    tiles = tuned("sweep")
    batch = 1024
    pick = np.r_[0:4, 509:515, 1020:1024]
    th = oracle.max_threads()
    assert len(tiles) == 20
    for key, cfgd in tiles.items():
        name, s = key.split("@")
        s = float(s)
        c, d, k, hw = SWEEP_SHAPES[name]
        g = U.ConvGeometry(c, d, k, k, hw, hw, padding=(k // 2, k // 2))
        w = synthesize_masked_weights(g, s, np.random.default_rng([0, int(s * 1000)]))
        f = U.build_csr(w, g)
        x = np.random.default_rng([3, c, d, hw]).standard_normal((batch, c, hw, hw)).astype(np.float32)
        xd = torch.from_numpy(x).cuda()
        plan, blob = plan_for(f, batch, _lib.USC_F32, ExecConfig(**cfgd), f.weights)
        xp = padded_input(xd, plan)
        lay = _lib.act_layout(d, g.out_h, g.out_w, 1, 1, 4, plan.in_.interleave)
        y = torch.zeros(lay.elems(batch), dtype=torch.float32, device="cuda")
        epi = _lib.Epilogue()
        epi.scale, epi.out_padded, epi.out = 1.0, 1, lay
        launch(plan, blob, xp, y, epi)
        out = torch.empty((batch, d, g.out_h, g.out_w), dtype=torch.float32, device="cuda")
        _lib.check(_lib.lib().usc_unpad_output(_lib.ref(lay), _lib.USC_F32, batch, _lib.t_ptr(y),
                                               _lib.t_ptr(out), _lib.stream_ptr()), "unpad")
        got = out.cpu().numpy()[pick]
        gt = (c, d, k, k, hw, hw, (1, 1), (k // 2, k // 2))
        ref = oracle.sparse_conv_forward(np.ascontiguousarray(x[pick]), _csr(f), gt, threads=th)
        assert np.array_equal(got, ref), key
        f._packs.clear()


@pytest.mark.parametrize("mode", ["passthrough", "16b/16b", "4b/16b"])
def test_quantize_model_network_vs_oracle(mode):
    """quantize_model + calibrate_activation_maxima (quantization.py:223-301): the
    calibrated maxima equal the oracle's unhooked fp32 pass layer by layer, and the
    quantised network equals the composition with the _half_hook epilogues."""
    import torch
    from paper_2112_15445_b200.models import vgg16_rng, vgg16_weights
    ws = vgg16_weights(vgg16_rng(0.93, seed=17), 0.93)
    rng = np.random.default_rng(18)
    calib = rng.standard_normal((96, 3, 32, 32)).astype(np.float32)
    x = rng.standard_normal((64, 3, 32, 32)).astype(np.float32)
    qm = U.quantize_model(ws, mode, calibration=calib if mode == "4b/16b" else None)
    th = oracle.max_threads()
    if mode == "4b/16b":
        # the calibration pass restated: fp32 conv / ReLU / pool maxima in the reference's numbering
        maxima, li, a = {}, 0, calib
        from paper_2112_15445_b200.models import VGG16_CIFAR, vgg16_geometries
        geoms, i = vgg16_geometries(), 0
        for v in VGG16_CIFAR:
            if v == "M":
                a = oracle.maxpool2(a)
                maxima[i] = float(a.max())
                i += 1
                continue
            g = geoms[li]
            gt = (g.in_channels, g.out_channels, 3, 3, g.input_h, g.input_w, (1, 1), (1, 1))
            a = oracle.sparse_conv_forward(a, oracle.build_csr(np.ascontiguousarray(qm.weights[li].data), gt), gt,
                                           threads=th)
            maxima[i] = float(a.max())
            a = oracle.relu(a)
            maxima[i + 1] = float(a.max())
            i += 2
            li += 1
        assert maxima == qm.maxima
        x = oracle.round_to_binary16(x)
    elif mode == "16b/16b":
        x = oracle.round_to_binary16(x)
    m = qm.network(64)
    xd = torch.from_numpy(x).cuda()
    got = m.forward(xd if mode == "passthrough" else xd.half()).float().cpu().numpy()

    def conv(li, a, gt):
        f = m.filters[li]
        y = oracle.sparse_conv_forward(a, _csr(f), gt, binary16=mode == "16b/16b", threads=th)
        if mode == "4b/16b":
            lp = m.layer_params[li]
            y = oracle.round_to_binary16(np.minimum(y, np.float32(lp["cap"])))
            return oracle.round_to_binary16(np.minimum(oracle.relu(y), np.float32(lp["cap2"])))
        return oracle.relu(y)
    assert np.array_equal(got, vgg_oracle(m, x, conv))
