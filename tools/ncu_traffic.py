"""Launch every conv of the VGG-16 bench model once (committed tuned tiles) for one
ncu --set full capture of all of them; writes gpurun_out/plans.json (launch order).

    ncu --set full --clock-control none --profile-from-start off -k regex:k_bi -o gpurun_out/traffic \\
        python tools/ncu_traffic.py [profiles/r01_tuned.json]
    python tools/ncu_summary.py traffic gpurun_out/traffic.ncu-rep gpurun_out/plans.json profiles/traffic.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import BATCH, build_model  # noqa: E402
from paper_2112_15445_b200.engine import launch  # noqa: E402

tuned = sys.argv[1] if len(sys.argv) > 1 else os.path.join("profiles", "r01_tuned.json")
model, _ = build_model(BATCH, torch.device("cuda", 0))
model.load_tuned_state(json.load(open(tuned)))
model.forward(torch.randn(BATCH, 3, 32, 32, device="cuda"))
convs = [s for s in model.steps if s[0] == "conv"]
os.makedirs("gpurun_out", exist_ok=True)
json.dump([dict(layer=s[1], plan=s[2].describe()) for s in convs], open("gpurun_out/plans.json", "w"))
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _, li, plan, blob, xin, yout, epi in convs:
    launch(plan, blob, xin, yout, epi)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
