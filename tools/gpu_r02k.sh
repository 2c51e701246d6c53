#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python tools/tc_probe.py > gpurun_out/tc_probe.jsonl 2> gpurun_out/tc_probe.err
timeout 900 python -m pytest tests/test_gpu_dispatch.py -q -x 2>&1 | tail -20 > gpurun_out/pytest_disp.txt
cat gpurun_out/tc_probe.jsonl; tail -3 gpurun_out/tc_probe.err; cat gpurun_out/pytest_disp.txt
