"""Shared access to the committed golden vectors (tests/golden/)."""
import hashlib
import json
import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
_cache = {}


def golden():
    if "json" not in _cache:
        with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
            _cache["json"] = json.load(fh)
    return _cache["json"]


def arrays():
    if "npz" not in _cache:
        _cache["npz"] = dict(np.load(os.path.join(GOLDEN_DIR, "small_cases.npz")))
    return _cache["npz"]


def sha(a) -> str:
    """Same digest as make_golden.sha: dtype, shape and raw bytes."""
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def geom(t):
    c, d, kh, kw, h, w, s, p = t
    return (c, d, kh, kw, h, w, tuple(s), tuple(p))


def layer_inputs(name, g, sparsity, batch, binary16=False, seed=0):
    """bench_layer's input generation (bench.py:98-108) via the oracle restatement."""
    import oracle
    rng = oracle.bench_rng(name, sparsity, seed)
    C, D, Kh, Kw, H, W = g[:6]
    w = oracle.synthesize_masked_weights((D, C, Kh, Kw), sparsity, rng, binary16)
    x = rng.standard_normal((batch, C, H, W)).astype(np.float32)
    if binary16:
        x = oracle.round_to_binary16(x)
    return x, w


def grad_cases():
    """tests/golden/grad_cases.npz (make_golden_grad.py): [(geometry dims, arrays)] of the
    reference's conv_grad_weights / conv_grad_input / Conv2D.backward."""
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "grad_cases.npz"))
    out, k = [], 0
    while f"g{k}_x" in z:
        c, d, kh, kw, h, w, sh, sw, ph, pw = [int(v) for v in z[f"g{k}_geom"]]
        out.append((dict(C=c, D=d, Kh=kh, Kw=kw, H=h, W=w, sh=sh, sw=sw, ph=ph, pw=pw),
                    {n: z[f"g{k}_{n}"] for n in ("x", "w", "dout", "dw", "dx", "dxpad")}))
        k += 1
    return out
