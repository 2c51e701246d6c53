#!/bin/bash
# late shortcut prefetch: full GPU suite; re-tune the fp32 ResNet-50 tiles; network timing
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
RETUNE=1 TUNED_OUT=gpurun_out timeout 2400 python tools/bench_variants.py --only resnet50-net-fp32 --steps 30 > gpurun_out/rn32.jsonl 2> gpurun_out/rn.err
timeout 900 python tools/bench_variants.py --only resnet50-net-fp32 --steps 30 > gpurun_out/rn32_old.jsonl 2>> gpurun_out/rn.err
cut -c1-300 gpurun_out/rn32.jsonl gpurun_out/rn32_old.jsonl; tail -2 gpurun_out/rn.err
