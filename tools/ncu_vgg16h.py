"""Launch one layer of the BINARY16 VGG-16 (autotuned) for an ncu capture:
   ncu --set full -k regex:k_bi -s S -c 1 python tools/ncu_vgg16h.py LAYER [mode]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_15445_b200 import PrecisionMode
from paper_2112_15445_b200.engine import launch
from paper_2112_15445_b200.models import SparseVGG16, vgg16_rng, vgg16_weights
L = int(sys.argv[1])
ws = vgg16_weights(vgg16_rng(0.93, 0), 0.93, precision=PrecisionMode.BINARY16)
m = SparseVGG16(ws, 256, precision=PrecisionMode.BINARY16)
m.autotune(repeats=3, warmup=1)
st = [s for s in m.steps if s[0] == "conv"][L]
_, li, plan, blob, xin, yout, epi = st
os.makedirs("gpurun_out", exist_ok=True)
json.dump(plan.describe(), open("gpurun_out/plan.json", "w"))
print(plan.describe(), flush=True)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(3):
    launch(plan, blob, xin, yout, epi)
torch.cuda.synchronize()
