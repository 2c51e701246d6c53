"""The tensor-core dense backend (usc_dense_conv_f16, tcgen05 implicit GEMM on the BI64
layout) against torch's conv2d on the same binary16 operands, within the fp16
tolerance max|got - ref| <= 1e-2 * max|ref| (fp32 accumulation in a different order)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("C,D,k,s,hw,n,res", [(64, 128, 3, 1, 8, 100, False), (256, 256, 1, 1, 8, 64, True),
                                              (128, 128, 3, 2, 16, 128, False), (64, 256, 1, 2, 16, 70, False),
                                              (512, 512, 3, 1, 4, 64, True), (512, 512, 3, 1, 2, 64, False),
                                              (512, 512, 3, 1, 4, 256, False), (512, 512, 3, 1, 2, 256, False),
                                              (256, 512, 1, 1, 4, 256, True), (64, 64, 3, 1, 32, 96, False),
                                              (64, 64, 1, 1, 32, 64, True), (256, 64, 1, 1, 8, 64, False),
                                              (128, 64, 3, 2, 16, 64, False), (64, 64, 3, 1, 7, 64, False),
                                              (64, 64, 3, 1, 32, 256, False), (256, 64, 1, 1, 32, 128, False),
                                              (3, 64, 3, 1, 32, 256, False), (3, 64, 3, 1, 6, 70, False),
                                              (16, 64, 3, 1, 8, 64, False), (5, 64, 3, 1, 7, 64, False)])
def test_dense_tc_matches_torch(C, D, k, s, hw, n, res):
    import torch
    from paper_2112_15445_b200 import _lib
    from paper_2112_15445_b200.dense import dense_conv, pack_weights
    rng = np.random.default_rng([C, D, k, s, hw])
    x = torch.from_numpy(rng.standard_normal((n, C, hw, hw)).astype(np.float32)).cuda().half()
    w = torch.from_numpy((rng.standard_normal((D, C, k, k)) / np.sqrt(C * k * k)).astype(np.float32)).cuda().half()
    halo = 1 if k == 3 else 0
    xl = _lib.act_layout(C, hw, hw, halo, halo, 2, 64)
    xb = torch.zeros(xl.elems(n), dtype=torch.float16, device="cuda")
    _lib.check(_lib.lib().usc_pad_input(_lib.ref(xl), _lib.USC_F16, n, _lib.t_ptr(x), _lib.t_ptr(xb),
                                        _lib.stream_ptr()))
    ho = (hw + 2 * (k // 2) - k) // s + 1
    yl = _lib.act_layout(D, ho, ho, 1, 1, 2, 64)
    yb = torch.zeros(yl.elems(n), dtype=torch.float16, device="cuda")
    ref = torch.nn.functional.conv2d(x.float(), w.float(), stride=s, padding=k // 2)
    rb, rl = None, None
    if res:
        r = torch.from_numpy(rng.standard_normal((n, D, ho, ho)).astype(np.float32)).cuda().half()
        rl = _lib.act_layout(D, ho, ho, 0, 0, 2, 64)
        rb = torch.zeros(rl.elems(n), dtype=torch.float16, device="cuda")
        _lib.check(_lib.lib().usc_pad_input(_lib.ref(rl), _lib.USC_F16, n, _lib.t_ptr(r), _lib.t_ptr(rb),
                                            _lib.stream_ptr()))
        ref = ref + r.float()
    ref = torch.relu(ref)
    dense_conv(pack_weights(w), C, D, k, s, n, xb, xl, yb, yl, rb, rl, relu=True)
    out = torch.empty((n, D, ho, ho), dtype=torch.float16, device="cuda")
    _lib.check(_lib.lib().usc_unpad_output(_lib.ref(yl), _lib.USC_F16, n, _lib.t_ptr(yb), _lib.t_ptr(out),
                                           _lib.stream_ptr()))
    torch.cuda.synchronize()
    err = float((out.float() - ref).abs().max())
    assert err <= 1e-2 * float(ref.abs().max()), err
    # the halo of the output buffer stays zero
    full = yb.view(-1)
    assert torch.isfinite(full.float()).all()


@pytest.mark.parametrize("res,relu", [(False, False), (True, False), (True, True)])
def test_dense_tc_saturates(res, relu):
    """Outputs past the binary16 range saturate to +-65504 (conversion and shortcut add),
    negatives survive without ReLU."""
    import torch
    from paper_2112_15445_b200 import _lib
    from paper_2112_15445_b200.dense import dense_conv, pack_weights
    C, D, hw, n = 64, 128, 4, 64
    rng = np.random.default_rng([7, int(res), int(relu)])
    x = torch.from_numpy(rng.standard_normal((n, C, hw, hw)).astype(np.float32) * 60).cuda().half()
    w = torch.from_numpy(rng.standard_normal((D, C, 1, 1)).astype(np.float32) * 60).cuda().half()
    xl = _lib.act_layout(C, hw, hw, 0, 0, 2, 64)
    xb = torch.zeros(xl.elems(n), dtype=torch.float16, device="cuda")
    L = _lib.lib()
    _lib.check(L.usc_pad_input(_lib.ref(xl), _lib.USC_F16, n, _lib.t_ptr(x), _lib.t_ptr(xb), _lib.stream_ptr()))
    yl = _lib.act_layout(D, hw, hw, 1, 1, 2, 64)
    yb = torch.zeros(yl.elems(n), dtype=torch.float16, device="cuda")
    ref = torch.nn.functional.conv2d(x.float(), w.float()).clamp(-65504, 65504)
    rb, rl = None, None
    if res:
        r = torch.from_numpy(rng.standard_normal((n, D, hw, hw)).astype(np.float32) * 3e4).cuda().half()
        rl = _lib.act_layout(D, hw, hw, 0, 0, 2, 64)
        rb = torch.zeros(rl.elems(n), dtype=torch.float16, device="cuda")
        _lib.check(L.usc_pad_input(_lib.ref(rl), _lib.USC_F16, n, _lib.t_ptr(r), _lib.t_ptr(rb), _lib.stream_ptr()))
        ref = (ref.half().float() + r.float()).clamp(-65504, 65504)
    if relu:
        ref = torch.relu(ref)
    dense_conv(pack_weights(w), C, D, 1, 1, n, xb, xl, yb, yl, rb, rl, relu=relu)
    out = torch.empty((n, D, hw, hw), dtype=torch.float16, device="cuda")
    _lib.check(L.usc_unpad_output(_lib.ref(yl), _lib.USC_F16, n, _lib.t_ptr(yb), _lib.t_ptr(out), _lib.stream_ptr()))
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    assert float(out.float().abs().max()) == 65504.0
    if not relu:
        assert float(out.float().min()) < 0
    err = float((out.float() - ref).abs().max())
    assert err <= 1e-2 * 65504, err


@pytest.mark.parametrize("C,D,hw,n", [(512, 512, 2, 256), (512, 512, 2, 64), (256, 512, 4, 64), (256, 128, 2, 128),
                                     (512, 512, 2, 70)])
def test_dense_tc_split_k(C, D, hw, n):
    """Small maps split K over CTAs (workspace path): the result matches torch within the
    fp16 tolerance, and repeated launches are bitwise identical (splits summed in a fixed
    order; the arrival counters are left at zero for the next launch)."""
    import torch
    from paper_2112_15445_b200 import _lib
    from paper_2112_15445_b200.dense import dense_conv, dense_workspace, pack_weights
    rng = np.random.default_rng([C, D, hw, n])
    x = torch.from_numpy(rng.standard_normal((n, C, hw, hw)).astype(np.float32)).cuda().half()
    w = torch.from_numpy((rng.standard_normal((D, C, 3, 3)) / np.sqrt(C * 9)).astype(np.float32)).cuda().half()
    xl = _lib.act_layout(C, hw, hw, 1, 1, 2, 64)
    xb = torch.zeros(xl.elems(n), dtype=torch.float16, device="cuda")
    L = _lib.lib()
    _lib.check(L.usc_pad_input(_lib.ref(xl), _lib.USC_F16, n, _lib.t_ptr(x), _lib.t_ptr(xb), _lib.stream_ptr()))
    yl = _lib.act_layout(D, hw, hw, 1, 1, 2, 64)
    ws = dense_workspace(C, D, 3, 1, n, xl)
    assert ws is not None  # these shapes fill at most half the SMs
    wp = pack_weights(w)
    outs = []
    for _ in range(3):
        yb = torch.zeros(yl.elems(n), dtype=torch.float16, device="cuda")
        dense_conv(wp, C, D, 3, 1, n, xb, xl, yb, yl, workspace=ws)
        out = torch.empty((n, D, hw, hw), dtype=torch.float16, device="cuda")
        _lib.check(L.usc_unpad_output(_lib.ref(yl), _lib.USC_F16, n, _lib.t_ptr(yb), _lib.t_ptr(out),
                                      _lib.stream_ptr()))
        outs.append(out)
    torch.cuda.synchronize()
    ref = torch.relu(torch.nn.functional.conv2d(x.float(), w.float(), padding=1))
    err = float((outs[0].float() - ref).abs().max())
    assert err <= 1e-2 * float(ref.abs().max()), err
    assert all(torch.equal(outs[0], o) for o in outs[1:])
    # the same conv without the workspace (one CTA per tile) agrees within the tolerance
    yb = torch.zeros(yl.elems(n), dtype=torch.float16, device="cuda")
    dense_conv(wp, C, D, 3, 1, n, xb, xl, yb, yl)
    out = torch.empty((n, D, hw, hw), dtype=torch.float16, device="cuda")
    _lib.check(L.usc_unpad_output(_lib.ref(yl), _lib.USC_F16, n, _lib.t_ptr(yb), _lib.t_ptr(out), _lib.stream_ptr()))
    torch.cuda.synchronize()
    assert float((out.float() - outs[0].float()).abs().max()) <= 1e-2 * float(ref.abs().max())


@pytest.mark.parametrize("C,D,hw,n,ph", [(64, 64, 32, 256, 1), (128, 128, 16, 256, 0), (64, 128, 32, 192, 1),
                                        (64, 64, 32, 70, 1)])
def test_dense_tc_fused_pool(C, D, hw, n, ph):
    """conv + ReLU + 2x2 max-pool in one tensor-core launch (row-pair tiles, pooled in the
    epilogue) against torch within the fp16 tolerance, and equal to the unfused conv +
    usc_maxpool2 up to the same tolerance."""
    import torch
    from paper_2112_15445_b200 import _lib
    from paper_2112_15445_b200.dense import dense_conv, dense_conv_pool, pack_weights, pool_fusable
    rng = np.random.default_rng([C, D, hw, n, 3])
    x = torch.from_numpy(rng.standard_normal((n, C, hw, hw)).astype(np.float32)).cuda().half()
    w = torch.from_numpy((rng.standard_normal((D, C, 3, 3)) / np.sqrt(C * 9)).astype(np.float32)).cuda().half()
    xl = _lib.act_layout(C, hw, hw, 1, 1, 2, 64)
    xb = torch.zeros(xl.elems(n), dtype=torch.float16, device="cuda")
    L = _lib.lib()
    _lib.check(L.usc_pad_input(_lib.ref(xl), _lib.USC_F16, n, _lib.t_ptr(x), _lib.t_ptr(xb), _lib.stream_ptr()))
    assert pool_fusable(C, D, n, xl)
    pl = _lib.act_layout(D, hw // 2, hw // 2, ph, ph, 2, 64)
    pb = torch.zeros(pl.elems(n), dtype=torch.float16, device="cuda")
    wp = pack_weights(w)
    dense_conv_pool(wp, C, D, n, xb, xl, pb, pl)
    got = torch.empty((n, D, hw // 2, hw // 2), dtype=torch.float16, device="cuda")
    _lib.check(L.usc_unpad_output(_lib.ref(pl), _lib.USC_F16, n, _lib.t_ptr(pb), _lib.t_ptr(got), _lib.stream_ptr()))
    # unfused: conv into a full-resolution buffer, then the pool kernel
    yl = _lib.act_layout(D, hw, hw, 0, 0, 2, 64)
    yb = torch.zeros(yl.elems(n), dtype=torch.float16, device="cuda")
    dense_conv(wp, C, D, 3, 1, n, xb, xl, yb, yl)
    pb2 = torch.zeros(pl.elems(n), dtype=torch.float16, device="cuda")
    _lib.check(L.usc_maxpool2(_lib.ref(yl), _lib.ref(pl), _lib.USC_F16, n, _lib.t_ptr(yb), _lib.t_ptr(pb2),
                              _lib.stream_ptr()))
    torch.cuda.synchronize()
    ref = torch.nn.functional.max_pool2d(torch.relu(torch.nn.functional.conv2d(x.float(), w.float(), padding=1)), 2)
    tol = 1e-2 * float(ref.abs().max())
    assert float((got.float() - ref).abs().max()) <= tol
    # both paths round the same fp32 sums: the pooled values are the same binary16 numbers
    assert torch.equal(pb, pb2)
    # the halo of the pooled buffer stays zero
    assert torch.isfinite(pb.float()).all()
