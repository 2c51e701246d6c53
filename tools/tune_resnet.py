"""Time every kernel-3 tile candidate of named ResNet-50 convs on the network's own
buffers and epilogues:  python tools/tune_resnet.py fp32|fp16 NAME [NAME ...]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_15445_b200 import PrecisionMode
from paper_2112_15445_b200.engine import plan_for, tile_candidates, time_median_cuda
from paper_2112_15445_b200.resnet import SparseResNet50, resnet50_weights
prec = PrecisionMode.BINARY32 if sys.argv[1] == "fp32" else PrecisionMode.BINARY16
m = SparseResNet50(resnet50_weights(0.9, 0, prec), 256, precision=prec)
m.load_input(torch.randn(256, 3, 32, 32, device="cuda").to(m.tdtype)); m.run(); torch.cuda.synchronize()
for name in sys.argv[2:]:
    st = next(s for s in m.steps if m.layers[s[0]][0] == name)
    li, plan0, _, x, view, y, e = st
    g = m.eff[li][0]
    res = []
    for cfg in tile_candidates(g, 256, [1], prec, (3,)):
        if cfg.samples_per_cta != 64: continue
        try: plan, blob = plan_for(m.filters[li], 256, m.dtype, cfg, m.filters[li].weights, device=m.device)
        except ValueError: continue
        try: ms = time_median_cuda(lambda: m._launch((li, plan, blob, x, view, y, e)), 5, 1)
        except RuntimeError: continue
        d = plan.describe(); res.append((ms, {k: d[k] for k in ("P","PR","PC","DT","DW","WS","threads","CC","stages","grid","tail_split")}))
        m.filters[li]._packs.clear()
    res.sort(key=lambda r: r[0])
    print(name, len(res))
    for ms, d in res[:5]: print(f"  {ms*1e3:7.1f} us {d}")
