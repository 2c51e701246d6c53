"""Launch ONE conv of a benchmarked network, with its committed tuned tiles, between
cudaProfilerStart/Stop -- the target of an `ncu --profile-from-start off -c 1` capture:

    ncu --set full --import-source on --clock-control none --profile-from-start off -c 1 \
        -o gpurun_out/<tag> python tools/ncu_target.py vgg16:fp32:9 <tag>
    ncu ... python tools/ncu_target.py resnet50:fp16:s0b0.c3 <tag>

Specs: vgg16:<fp32|fp16|int8|cb4>:<conv index> (profiles/r01_tuned.json for fp32,
r02_tuned_vgg16_<mode>.json otherwise), resnet50:<fp32|fp16>:<conv name>
(r02_tuned_resnet50_<prec>.json).  Writes gpurun_out/<tag>.json: the plan, the
nonzero MACs and the algorithmic bytes of the launch (tools/ncu_summary.py divides the
ncu counters by them).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def tuned(name):
    p = os.path.join(ROOT, "profiles", "r01_tuned.json" if name == "vgg16_fp32" else f"r02_tuned_{name}.json")
    return json.load(open(p))


def main():
    spec, tag = sys.argv[1], sys.argv[2]
    net, mode, which = spec.split(":")
    from paper_2112_15445_b200 import PrecisionMode
    if net == "vgg16":
        from paper_2112_15445_b200.models import SparseVGG16, vgg16_rng, vgg16_weights
        prec = PrecisionMode.BINARY16 if mode == "fp16" else PrecisionMode.BINARY32
        ws = vgg16_weights(vgg16_rng(0.93, 0), 0.93, precision=prec)
        x = torch.randn(256, 3, 32, 32, device="cuda")
        kw = dict(mode=mode, calibration=x) if mode in ("int8", "cb4") else dict(precision=prec)
        m = SparseVGG16(ws, 256, **kw)
        m.load_tuned_state(tuned(f"vgg16_{mode}"))
        m.forward(x if mode in ("fp32", "int8") else x.half())
        li = int(which)
        st = next(s for s in m.steps if s[0] == "conv" and s[1] == li)
        plan, g, f = st[2], m.geoms[li], m.filters[li]
        run = lambda: m._run_step(st)  # noqa: E731
        eb = 4 if mode == "fp32" else 2
    else:
        from paper_2112_15445_b200.resnet import SparseResNet50, resnet50_weights
        prec = PrecisionMode.BINARY16 if mode == "fp16" else PrecisionMode.BINARY32
        m = SparseResNet50(resnet50_weights(0.9, 0, prec), 256, precision=prec)
        m.load_tuned_state(tuned(f"resnet50_{mode}"))
        m.forward(torch.randn(256, 3, 32, 32, device="cuda").to(m.tdtype))
        st = next(s for s in m.steps if m.layers[s[0]][0] == which)
        li = st[0]
        plan, g, f = st[1], m.layers[li][1], m.filters[li]
        run = lambda: m._launch(st)  # noqa: E731
        eb = 4 if mode == "fp32" else 2
    genuine = int(np.count_nonzero(f.weights))
    macs = genuine * g.out_h * g.out_w * 256
    byts = 256 * (g.in_channels * g.input_h * g.input_w + g.out_channels * g.out_h * g.out_w) * eb + \
        g.out_channels * f.n_nz * 8
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump({"spec": spec, "plan": plan.describe(), "nonzero_macs": macs, "algorithmic_bytes": byts},
              open(os.path.join(ROOT, "gpurun_out", f"{tag}.json"), "w"))
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    run()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main()
