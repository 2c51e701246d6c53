"""usc_maxpool2 between batch-interleaved layouts (the vectorised BI32/BI64 path) against
the oracle's nn.MaxPool2 (nn.py:124-135): first NaN of the window if any, else the first
maximum in window order -- bit for bit, including signed zeros, infinities and ragged
batches (padding samples of the last interleave block)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", ["f32", "f16"])
@pytest.mark.parametrize("il,n,c,hw,halo_in,halo_out", [(64, 70, 5, 6, 1, 1), (32, 33, 3, 8, 1, 0),
                                                        (64, 128, 16, 32, 0, 1), (32, 64, 7, 2, 1, 0)])
def test_maxpool_bi_matches_oracle(dtype, il, n, c, hw, halo_in, halo_out):
    import torch
    import oracle
    from paper_2112_15445_b200 import _lib
    rng = np.random.default_rng([il, n, c, hw])
    x = rng.standard_normal((n, c, hw, hw)).astype(np.float32)
    # ties between signed zeros, NaNs and infinities at random window positions
    special = np.array([0.0, -0.0, np.nan, np.inf, -np.inf, 1.0, 1.0], np.float32)
    mask = rng.random(x.shape) < 0.2
    x[mask] = special[rng.integers(0, len(special), int(mask.sum()))]
    tdt, dt, eb = (torch.float32, _lib.USC_F32, 4) if dtype == "f32" else (torch.float16, _lib.USC_F16, 2)
    xt = torch.from_numpy(x).cuda().to(tdt)
    li = _lib.act_layout(c, hw, hw, halo_in, halo_in, eb, il)
    lo = _lib.act_layout(c, hw // 2, hw // 2, halo_out, halo_out, eb, il)
    xb = torch.zeros(li.elems(n), dtype=tdt, device="cuda")
    yb = torch.zeros(lo.elems(n), dtype=tdt, device="cuda")
    L = _lib.lib()
    _lib.check(L.usc_pad_input(_lib.ref(li), dt, n, _lib.t_ptr(xt), _lib.t_ptr(xb), _lib.stream_ptr()))
    _lib.check(L.usc_maxpool2(_lib.ref(li), _lib.ref(lo), dt, n, _lib.t_ptr(xb), _lib.t_ptr(yb), _lib.stream_ptr()))
    out = torch.empty((n, c, hw // 2, hw // 2), dtype=tdt, device="cuda")
    _lib.check(L.usc_unpad_output(_lib.ref(lo), dt, n, _lib.t_ptr(yb), _lib.t_ptr(out), _lib.stream_ptr()))
    torch.cuda.synchronize()
    ref = oracle.maxpool2(xt.float().cpu().numpy())
    got = out.float().cpu().numpy()
    nan = np.isnan(ref)
    assert np.array_equal(nan, np.isnan(got))
    # bitwise on everything else (the sign of a zero included)
    assert np.array_equal(ref[~nan].view(np.uint32), got[~nan].view(np.uint32))
