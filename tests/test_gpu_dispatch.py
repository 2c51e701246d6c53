"""The per-layer sparse/dense backend dispatcher (the reference's
backend_config, /root/reference/pkg/src/unsparse/bench.py:212-227, applied per layer
as pipeline.py:381-389 does).

Binary16 networks may hand a layer to cuDNN (tensor cores); the result is then held
to the north star's fp16 tolerance, written here as
    max |got - ref| <= 1e-2 * max |ref|
against the oracle composition (binary16 hooks, fp32 accumulation).  fp32 networks
stay all-sparse and bitwise (a dense backend is refused).  The BI64 <-> NHWC
transposes the dense steps use are checked exactly."""
import numpy as np
import pytest

import oracle
import paper_2112_15445_b200 as U

pytestmark = pytest.mark.gpu

F32, F16 = U.PrecisionMode.BINARY32, U.PrecisionMode.BINARY16
TOL = 1e-2


def _tame(ws, density):
    """He-scaled copies of the pruned weights (binary16 grid): with the generator's raw
    N(0,1) values activations grow ~sqrt(fan_in * density) per layer and the binary16
    networks saturate at 65504 within a few layers, where the test would only compare
    two ways of overflowing."""
    out = []
    for w in ws:
        d = np.array(w.data)
        fan_in = d.shape[1] * d.shape[2] * d.shape[3]
        out.append(U.DenseTensor4.from_array(d * np.float32(np.sqrt(2.0 / (fan_in * density))), F16))
    return out


def _close(got, ref):
    err = float(np.max(np.abs(got.astype(np.float64) - ref.astype(np.float64))))
    return err <= TOL * float(np.max(np.abs(ref))), err


def test_bi64_nhwc_transposes_exact():
    import torch
    from paper_2112_15445_b200 import _lib
    n, C, H, W = 100, 32, 5, 7  # a partial last sample block
    rng = np.random.default_rng(0)
    x = oracle.round_to_binary16(rng.standard_normal((n, C, H, W)).astype(np.float32) * 100)
    x[0, 0, 0, 0], x[1, 1, 1, 1] = np.nan, -np.inf
    lay = _lib.act_layout(C, H, W, 1, 1, 2, 64)
    buf = torch.zeros(lay.elems(n), dtype=torch.float16, device="cuda")
    xd = torch.from_numpy(x).cuda().half()
    _lib.check(_lib.lib().usc_pad_input(_lib.ref(lay), _lib.USC_F16, n, _lib.t_ptr(xd), _lib.t_ptr(buf),
                                        _lib.stream_ptr()))
    nhwc = torch.empty((n, H, W, C), dtype=torch.float16, device="cuda")
    _lib.check(_lib.lib().usc_bi_to_nhwc(_lib.ref(lay), n, _lib.t_ptr(buf), _lib.t_ptr(nhwc), _lib.stream_ptr()))
    assert np.array_equal(nhwc.float().cpu().numpy(), x.transpose(0, 2, 3, 1), equal_nan=True)
    # back, with residual + ReLU: relu(sat16(sat16(y) + r))
    y = oracle.round_to_binary16(rng.standard_normal((n, C, H, W)).astype(np.float32) * 30000)
    r = oracle.round_to_binary16(rng.standard_normal((n, C, H, W)).astype(np.float32) * 30000)
    rlay = _lib.act_layout(C, H, W, 0, 0, 2, 64)
    rbuf = torch.zeros(rlay.elems(n), dtype=torch.float16, device="cuda")
    rd = torch.from_numpy(r).cuda().half()
    _lib.check(_lib.lib().usc_pad_input(_lib.ref(rlay), _lib.USC_F16, n, _lib.t_ptr(rd), _lib.t_ptr(rbuf),
                                        _lib.stream_ptr()))
    yd = torch.from_numpy(np.ascontiguousarray(y.transpose(0, 2, 3, 1))).cuda().half()
    out = torch.zeros(lay.elems(n), dtype=torch.float16, device="cuda")
    _lib.check(_lib.lib().usc_nhwc_to_bi(_lib.ref(lay), n, _lib.t_ptr(yd), _lib.t_ptr(out), _lib.ref(rlay),
                                         _lib.t_ptr(rbuf), 1, _lib.stream_ptr()))
    plain = torch.empty((n, C, H, W), dtype=torch.float16, device="cuda")
    _lib.check(_lib.lib().usc_unpad_output(_lib.ref(lay), _lib.USC_F16, n, _lib.t_ptr(out), _lib.t_ptr(plain),
                                           _lib.stream_ptr()))
    ref = oracle.relu(oracle.round_to_binary16((y + r).astype(np.float32)))
    assert np.array_equal(plain.float().cpu().numpy(), ref)


@pytest.mark.parametrize("mix", ["cudnn", "tc"])
def test_resnet50_fp16_mixed_backends_within_tolerance(mix):
    """Every dense step kind (3x3 stride 1 and 2, projections, residual c3) on cuDNN (or on
    the tensor-core backend where it applies, mixed with cuDNN), the rest sparse, against
    the oracle composition."""
    import torch
    from paper_2112_15445_b200.resnet import STAGES, SparseResNet50, resnet50_layers, resnet50_weights
    ws = _tame(resnet50_weights(0.9, seed=4, precision=F16), 0.1)
    layers = resnet50_layers()
    backends = ["dense" if (role in ("c2", "proj") or (role == "c3" and li % 2 == 0)) else "sparse"
                for li, (_, _, role, _) in enumerate(layers)]
    if mix == "tc":
        probe = SparseResNet50.__new__(SparseResNet50)
        probe.layers, probe.dtype = layers, __import__("paper_2112_15445_b200")._lib.USC_F16
        backends = ["tc" if probe.tc_eligible(li) and li % 3 != 1 else b for li, b in enumerate(backends)]
        assert "tc" in backends
    x = oracle.round_to_binary16(np.random.default_rng(5).standard_normal((64, 3, 32, 32)).astype(np.float32))
    m = SparseResNet50(ws, 64, precision=F16, backends=backends)
    m.capture()
    got = m.forward(torch.from_numpy(x).cuda().half()).float().cpu().numpy()
    th = oracle.max_threads()

    def conv(li, a):
        _, g, role, s = layers[li]
        if role == "c2" and s == 2:
            a = np.pad(a, ((0, 0), (0, 0), (1, 0), (1, 0)))
        if role == "proj" and s == 2:
            a = np.ascontiguousarray(a[:, :, :g.input_h, :g.input_w])
        gt = (g.in_channels, g.out_channels, g.filter_h, g.filter_w, g.input_h, g.input_w, g.stride, g.padding)
        return oracle.round_to_binary16(oracle.sparse_conv_forward(
            a, oracle.build_csr(np.ascontiguousarray(ws[li].data), gt), gt, threads=th))

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
            a = oracle.relu(oracle.round_to_binary16((conv(li, h2) + sc).astype(np.float32)))
            li += 1
    assert float(np.max(np.abs(a))) < 1e4  # a tame network: no saturation to compare
    ok, err = _close(got, a)
    assert ok, err
    with pytest.raises(ValueError):
        SparseResNet50(resnet50_weights(0.9, seed=4), 64, backends=backends)  # fp32: bitwise only


@pytest.mark.parametrize("mix", ["cudnn", "tc"])
def test_vgg16_fp16_mixed_backends_within_tolerance(mix):
    """cudnn: every other conv on cuDNN (NHWC chains, transposes at the borders); tc: the
    tensor-core backend on the BI64 buffers mixed with sparse and cuDNN convs."""
    import torch
    from paper_2112_15445_b200.models import VGG16_CIFAR, SparseVGG16, vgg16_rng, vgg16_weights
    ws = _tame(vgg16_weights(vgg16_rng(0.93, seed=8), 0.93, precision=F16), 0.07)
    if mix == "cudnn":
        backends = ["dense" if li % 2 == 1 else "sparse" for li in range(13)]
    else:
        backends = ["sparse", "sparse", "tc", "dense", "tc", "tc", "sparse", "tc", "dense", "dense", "tc", "sparse",
                    "tc"]
    x = oracle.round_to_binary16(np.random.default_rng(9).standard_normal((64, 3, 32, 32)).astype(np.float32))
    m = SparseVGG16(ws, 64, precision=F16, backends=backends)
    m.capture()
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
    ok, err = _close(got, a)
    assert ok, err


def test_autotune_backends_picks_and_runs():
    """The dispatcher's argmin on the network's buffers; the chosen mix stays within
    tolerance of the all-sparse (bitwise) network."""
    import torch
    from paper_2112_15445_b200.resnet import SparseResNet50, resnet50_weights
    ws = _tame(resnet50_weights(0.9, seed=6, precision=F16), 0.1)
    x = torch.from_numpy(oracle.round_to_binary16(
        np.random.default_rng(7).standard_normal((64, 3, 32, 32)).astype(np.float32))).cuda().half()
    m = SparseResNet50(ws, 64, precision=F16)
    ref = m.forward(x).float().cpu().numpy()
    picks = m.autotune_backends(repeats=3, warmup=1)
    assert set(picks) <= {"sparse", "dense", "tc"} and picks[0] in ("sparse", "tc")  # the 3-channel stem: no cuDNN form
    assert set(m.backend_times) and m.tuned_state()["backends"] == picks
    ok, err = _close(m.forward(x).float().cpu().numpy(), ref)
    assert ok, err
    with pytest.raises(ValueError):
        SparseResNet50(resnet50_weights(0.9, seed=6), 64).autotune_backends()


@pytest.mark.parametrize("net", ["vgg16", "resnet50"])
def test_benchmarked_dispatch_states_within_tolerance(net):
    """The committed dispatcher picks (profiles/r02_tuned_<net>_fp16_dispatch.json: tiles and
    per-conv backends, as bench_variants times them) at batch 256 against the oracle
    composition, on He-scaled weights (the fp16 tolerance is meaningless once the
    raw-N(0,1) networks saturate)."""
    import json
    import os

    import torch
    state = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                                        f"r02_tuned_{net}_fp16_dispatch.json")))
    # the dispatcher routes convs off the sparse path (every ResNet-50 conv runs on tensor
    # cores once the 3-channel stem has its first-layer form)
    assert set(state["backends"]) <= {"sparse", "dense", "tc"} and set(state["backends"]) - {"sparse"}
    x = oracle.round_to_binary16(np.random.default_rng(31).standard_normal((256, 3, 32, 32)).astype(np.float32))
    th = oracle.max_threads()
    if net == "vgg16":
        from paper_2112_15445_b200.models import VGG16_CIFAR, SparseVGG16, vgg16_rng, vgg16_weights
        ws = _tame(vgg16_weights(vgg16_rng(0.93, 0), 0.93, precision=F16), 0.07)
        m = SparseVGG16(ws, 256, precision=F16)
        m.load_tuned_state(state)
        m.capture()
        got = m.forward(torch.from_numpy(x).cuda().half()).float().cpu().numpy()
        a, li = x, 0
        for v in VGG16_CIFAR:
            if v == "M":
                a = oracle.maxpool2(a)
                continue
            g = m.geoms[li]
            gt = (g.in_channels, g.out_channels, 3, 3, g.input_h, g.input_w, (1, 1), (1, 1))
            a = oracle.relu(oracle.sparse_conv_forward(a, oracle.build_csr(ws[li].data, gt), gt, binary16=True,
                                                       threads=th))
            li += 1
    else:
        from paper_2112_15445_b200.resnet import STAGES, SparseResNet50, resnet50_layers, resnet50_weights
        ws = _tame(resnet50_weights(0.9, 0, F16), 0.1)
        layers = resnet50_layers()
        m = SparseResNet50(ws, 256, precision=F16)
        m.load_tuned_state(state)
        m.capture()
        got = m.forward(torch.from_numpy(x).cuda().half()).float().cpu().numpy()

        def conv(li, a):
            _, g, role, s = layers[li]
            if role == "c2" and s == 2:
                a = np.pad(a, ((0, 0), (0, 0), (1, 0), (1, 0)))
            if role == "proj" and s == 2:
                a = np.ascontiguousarray(a[:, :, :g.input_h, :g.input_w])
            gt = (g.in_channels, g.out_channels, g.filter_h, g.filter_w, g.input_h, g.input_w, g.stride, g.padding)
            return oracle.round_to_binary16(oracle.sparse_conv_forward(
                a, oracle.build_csr(np.ascontiguousarray(ws[li].data), gt), gt, threads=th))

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
                a = oracle.relu(oracle.round_to_binary16((conv(li, h2) + sc).astype(np.float32)))
                li += 1
    ok, err = _close(got, a)
    assert ok, err
