"""Run a committed binary16 dispatch network (VGG-16 or ResNet-50, batch 256) for a few
captured steps -- the target of an ncu launch list (which kernels a dispatched network runs).

    ncu --metrics gpu__time_duration.sum -c 400 --csv --log-file L python tools/run_dispatch_net.py vgg16
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    from paper_2112_15445_b200 import PrecisionMode
    net = sys.argv[1] if len(sys.argv) > 1 else "vgg16"
    F16 = PrecisionMode.BINARY16
    state = json.load(open(os.path.join(ROOT, "profiles", f"r02_tuned_{net}_fp16_dispatch.json")))
    if net == "vgg16":
        from paper_2112_15445_b200.models import SparseVGG16, vgg16_rng, vgg16_weights
        m = SparseVGG16(vgg16_weights(vgg16_rng(0.93, 0), 0.93, precision=F16), 256, precision=F16)
    else:
        from paper_2112_15445_b200.resnet import SparseResNet50, resnet50_weights
        m = SparseResNet50(resnet50_weights(0.9, 0, F16), 256, precision=F16)
    m.load_tuned_state(state)
    m.capture()
    m.load_input(torch.randn(256, 3, 32, 32, device="cuda").half())
    for _ in range(2):
        m.graph.replay()
    torch.cuda.synchronize()
    print(net, "backends", sorted(set(m.backends)))


if __name__ == "__main__":
    main()
