"""Experiment: the VGG-16 batch as K concurrent sub-batches on K streams in one CUDA
graph (tail waves of one stream's persistent kernels filled by the other's)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2112_15445_b200.models import SparseVGG16, vgg16_rng, vgg16_weights

B = 256
ws = vgg16_weights(vgg16_rng(0.93, 0), 0.93)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")

def timeit(fn, n=30):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        flush.zero_()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts))

for K in (1, 2, 4):
    ms = [SparseVGG16(ws, B // K) for _ in range(K)]
    for m in ms:
        m.autotune(repeats=3, warmup=1)
        m.load_input(torch.randn(B // K, 3, 32, 32, device="cuda"))
    streams = [torch.cuda.Stream() for _ in range(K)]
    for m, s in zip(ms, streams):
        with torch.cuda.stream(s): m.run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cur = torch.cuda.current_stream()
    with torch.cuda.graph(g):
        main = torch.cuda.current_stream()
        for m, s in zip(ms, streams):
            s.wait_stream(main)
            with torch.cuda.stream(s):
                m.run()
        for s in streams:
            main.wait_stream(s)
    t = timeit(lambda: g.replay())
    print(f"K={K}: {t:.4f} ms/step, {B / t * 1e3:.0f} img/s", flush=True)
