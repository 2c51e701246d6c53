"""Launch one VGG-16 layer with an explicit ExecConfig (for an ncu capture):
   ncu --set full -k regex:k_b -s 3 -c 1 python tools/ncu_cfg.py LAYER key=value ..."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_15445_b200 import ExecConfig
from paper_2112_15445_b200.engine import launch
from bench import build_model
L = int(sys.argv[1])
kw = {k: int(v) for k, v in (a.split("=") for a in sys.argv[2:])}
model, _ = build_model(256, torch.device("cuda", 0))
st = [s for s in model.steps if s[0] == "conv"][L]
_, li, plan0, _, xin, yout, epi = st
plan, blob = model._plan_for(li, ExecConfig(**kw))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(plan.describe(), open("gpurun_out/plan.json", "w"))
print(plan.describe())
for _ in range(5):
    launch(plan, blob, xin, yout, epi)
torch.cuda.synchronize()
