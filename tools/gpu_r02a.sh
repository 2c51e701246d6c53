#!/bin/bash
# Round-2 GPU session A: variants (dump tuned tiles), tests (incl. the tuned-plan parity
# tests), bench.py.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export TUNED_OUT=gpurun_out RETUNE=1
timeout 1500 python tools/bench_variants.py --steps 30 > gpurun_out/variants.jsonl 2> gpurun_out/variants.err
cp gpurun_out/r02_tuned_*.json profiles/ 2>/dev/null
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ls gpurun_out; cat gpurun_out/pytest_gpu.txt; tail -3 gpurun_out/variants.err; cut -c1-600 gpurun_out/variants.jsonl; cut -c1-800 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
