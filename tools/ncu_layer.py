"""Launch one VGG-16 conv layer for an ncu capture:
   ncu --set full -k regex:k_bi -s 13 -c 1 python tools/ncu_layer.py LAYER
(one full forward = 13 conv launches first, then LAYER 3x)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2112_15445_b200.engine import launch
from paper_2112_15445_b200.models import SparseVGG16, vgg16_rng, vgg16_weights
L = int(sys.argv[1]) if len(sys.argv) > 1 else 5
B = int(os.environ.get("B", 256))
rng = vgg16_rng(0.93)
m = SparseVGG16(vgg16_weights(rng, 0.93), B)
if len(sys.argv) > 2:  # per-layer tiles dumped by bench.py --dump-configs
    import json
    m.load_tuned_state(json.load(open(sys.argv[2])))
m.forward(torch.randn(B, 3, 32, 32, device="cuda"))
st = [s for s in m.steps if s[0] == "conv"][L]
_, li, plan, blob, xin, yout, epi = st
print("plan", plan.describe())
import json
os.makedirs("gpurun_out", exist_ok=True)
json.dump(plan.describe(), open("gpurun_out/plan.json", "w"))
for _ in range(3):
    launch(plan, blob, xin, yout, epi)
torch.cuda.synchronize()
