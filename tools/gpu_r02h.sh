#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export TUNED_OUT=gpurun_out
timeout 900 python tools/bench_variants.py --only resnet50-net-fp32 --steps 30 > gpurun_out/rn32.jsonl 2> gpurun_out/rn.err
timeout 900 python tools/bench_variants.py --only resnet50-net-fp16 --steps 30 > gpurun_out/rn16.jsonl 2>> gpurun_out/rn.err
timeout 900 python -m pytest tests -m gpu -q -k "resnet" 2>&1 | tail -3 > gpurun_out/pytest_rn.txt
timeout 600 python bench.py --no-cpu-baseline --no-cfg1 > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/pytest_rn.txt; cut -c1-400 gpurun_out/rn32.jsonl gpurun_out/rn16.jsonl; cut -c1-300 gpurun_out/bench.json; tail -3 gpurun_out/rn.err
