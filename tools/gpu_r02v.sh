#!/bin/bash
# swapped-operand 64-channel kernel (k_dts): tests, probe with and without it
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense_tc.py -q -x 2>&1 | tail -8 > gpurun_out/pytest_tc.txt
cat gpurun_out/pytest_tc.txt
grep -q "passed" gpurun_out/pytest_tc.txt && ! grep -q "failed\|error" gpurun_out/pytest_tc.txt || exit 1
timeout 600 python tools/tc_probe.py 2>&1 | grep "x64-\|64x64" > gpurun_out/tc_probe_dts.jsonl
USC_NO_DTS=1 timeout 600 python tools/tc_probe.py 2>&1 | grep "x64-\|64x64" > gpurun_out/tc_probe_nodts.jsonl
cat gpurun_out/tc_probe_dts.jsonl gpurun_out/tc_probe_nodts.jsonl
