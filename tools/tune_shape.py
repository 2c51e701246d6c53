import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2112_15445_b200 import DenseTensor4, build_csr
from paper_2112_15445_b200.engine import launch, padded_input, plan_for, time_median_cuda, tile_candidates
from paper_2112_15445_b200.pruning import synthesize_masked_weights
from paper_2112_15445_b200.tensor import ConvGeometry
c, d, hw, s, batch = 64, 64, 32, float(sys.argv[1]), int(sys.argv[2])
g = ConvGeometry(c, d, 3, 3, hw, hw, padding=(1, 1))
x = torch.randn(batch, c, hw, hw, device="cuda")
w = synthesize_masked_weights(g, s, np.random.default_rng([0, int(s * 1000)]))
f = build_csr(w, g)
res = []
pads = {}
for cfg in tile_candidates(g, batch, [1], kernels=(3,)):
    try:
        plan, blob = plan_for(f, batch, 0, cfg, f.weights)
    except ValueError:
        continue
    k = plan.in_.interleave
    if k not in pads: pads[k] = padded_input(x, plan)
    y = torch.empty(batch, d, hw, hw, device="cuda")
    ms = time_median_cuda(lambda: launch(plan, blob, pads[k], y), 7, 2)
    res.append((ms, plan.describe()))
res.sort(key=lambda r: r[0])
flops = 2.0 * np.count_nonzero(f.weights) * hw * hw * batch
for ms, dsc in res[:8]:
    print(round(ms*1e3,1), "us", round(flops/ms/1e9,2), "TF", {k: dsc[k] for k in ("kernel","P","PR","PC","DT","DW","WS","threads","CC","stages","tail_split")})
