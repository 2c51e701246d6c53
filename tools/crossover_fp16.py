"""Binary16 sparse/dense crossover on B200 (BASELINE configs[4] layer shapes and sparsities,
batch 1024): per point the sparse binary16 kernel (best batch-interleaved tile, resident BI64
output -- what a network layer runs), the tcgen05 dense backend on the same BI64 buffers
(best of its tile search) and cuDNN fp16 (channels_last, tensor cores).  The sparse kernel's
time falls with sparsity, the dense ones do not: the table shows where the per-layer
dispatcher (`autotune_backends`, the reference's backend_config rule) switches.

    python tools/crossover_fp16.py [--sparsities 0.5,0.7,0.9,0.95,0.98,0.99]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sparsities", default="0.5,0.7,0.9,0.95,0.98,0.99")
    ap.add_argument("--batch", type=int, default=1024)
    args = ap.parse_args()
    from bench_variants import SWEEP_SHAPES, _resident_launch
    from paper_2112_15445_b200 import PrecisionMode, _lib, build_csr
    from paper_2112_15445_b200.dense import dense_conv, dense_workspace, pack_weights, tune_tile
    from paper_2112_15445_b200.engine import padded_input, plan_for, tile_candidates, time_median_cuda
    from paper_2112_15445_b200.pruning import synthesize_masked_weights
    from paper_2112_15445_b200.tensor import ConvGeometry
    torch.backends.cudnn.benchmark = True
    n = args.batch
    F16 = PrecisionMode.BINARY16
    for name, (c, d, k, hw) in SWEEP_SHAPES.items():
        g = ConvGeometry(c, d, k, k, hw, hw, padding=(k // 2, k // 2))
        x = torch.randn(n, c, hw, hw, device="cuda").half()
        xc = x.contiguous(memory_format=torch.channels_last)
        halo = k // 2
        xl = _lib.act_layout(c, hw, hw, halo, halo, 2, 64)
        xb = torch.zeros(xl.elems(n), dtype=torch.float16, device="cuda")
        _lib.check(_lib.lib().usc_pad_input(_lib.ref(xl), _lib.USC_F16, n, _lib.t_ptr(x), _lib.t_ptr(xb),
                                            _lib.stream_ptr()))
        yl = _lib.act_layout(d, hw, hw, 1, 1, 2, 64)
        yb = torch.zeros(yl.elems(n), dtype=torch.float16, device="cuda")
        dense_us = None
        for s in (float(v) for v in args.sparsities.split(",")):
            w = synthesize_masked_weights(g, s, np.random.default_rng([0, int(s * 1000)]), precision=F16)
            f = build_csr(w, g)
            best, pads = None, {}
            for cand in tile_candidates(g, n, [1], F16, (3,)):
                try:
                    p_, b_ = plan_for(f, n, _lib.USC_F16, cand, f.weights)
                except (ValueError, RuntimeError):
                    continue
                key = (p_.in_.interleave, p_.in_.hp, p_.in_.ws)
                if key not in pads:
                    pads[key] = padded_input(x, p_)
                t = time_median_cuda(_resident_launch(p_, b_, pads[key], d, g, n, torch.float16), 3, 1)
                if best is None or t < best[0]:
                    best = (t, p_.describe())
                f._packs.clear()
            wt = torch.from_numpy(np.array(w.data, dtype=np.float32)).cuda().half()
            if dense_us is None:  # dense time does not depend on the sparsity: measure once per shape
                wp = pack_weights(wt)

                def launch(twp, sp, ws):
                    dense_conv(wp, c, d, k, 1, n, xb, xl, yb, yl, None, None, True, None, ws, twp, sp)
                twp, sp = tune_tile(launch, c, d, k, 1, n, xl)
                ws = dense_workspace(c, d, k, 1, n, xl, False, None, twp, sp)
                tc = time_median_cuda(lambda: launch(twp, sp, ws), 9, 2)
                wc = wt.contiguous(memory_format=torch.channels_last)
                cd = time_median_cuda(lambda: torch.relu(torch.nn.functional.conv2d(xc, wc, padding=halo)), 9, 2)
                dense_us = (tc * 1e3, cd * 1e3, [twp, sp])
            sparse_us = best[0] * 1e3
            tc_us, cudnn_us, tile = dense_us
            winner = min((("sparse", sparse_us), ("tc", tc_us), ("cudnn", cudnn_us)), key=lambda kv: kv[1])[0]
            nnz = int(np.count_nonzero(f.weights))
            print(json.dumps({"layer": name, "sparsity": s, "batch": n, "sparse_us": round(sparse_us, 1),
                              "sparse_nonzero_tflops": round(2.0 * nnz * hw * hw * n / sparse_us / 1e6, 2),
                              "tc_us": round(tc_us, 1), "tc_tile": tile, "cudnn_fp16_us": round(cudnn_us, 1),
                              "sparse_vs_tc": round(tc_us / sparse_us, 3), "winner": winner,
                              "sparse_plan": {kk: best[1][kk] for kk in ("P", "DT", "NS", "CC", "threads")}}),
                  flush=True)


if __name__ == "__main__":
    main()
