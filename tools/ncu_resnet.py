"""Launch one conv of the autotuned ResNet-50 CIFAR network for an ncu capture:
   ncu --set full --profile-from-start off -k regex:k_bi -c 1 python tools/ncu_resnet.py NAME [fp16|fp32]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2112_15445_b200 import PrecisionMode  # noqa: E402
from paper_2112_15445_b200.resnet import SparseResNet50, resnet50_weights  # noqa: E402

name = sys.argv[1]
prec = PrecisionMode.BINARY32 if len(sys.argv) > 2 and sys.argv[2] == "fp32" else PrecisionMode.BINARY16
m = SparseResNet50(resnet50_weights(0.9, 0, prec), 256, precision=prec)
m.autotune()
m.load_input(torch.randn(256, 3, 32, 32, device="cuda").to(m.tdtype))
m.run()
st = next(s for s in m.steps if m.layers[s[0]][0] == name)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(st[1].describe(), open("gpurun_out/plan.json", "w"))
print(st[1].describe(), flush=True)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(2):
    m._launch(st)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
