#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_dense_tc.py -q -x 2>&1 | tail -30 > gpurun_out/pytest_tc.txt
cat gpurun_out/pytest_tc.txt
grep -q "passed" gpurun_out/pytest_tc.txt && ! grep -q "failed" gpurun_out/pytest_tc.txt && timeout 600 python tools/tc_probe.py > gpurun_out/tc_probe.jsonl 2> gpurun_out/tc_probe.err
cat gpurun_out/tc_probe.jsonl; tail -3 gpurun_out/tc_probe.err
