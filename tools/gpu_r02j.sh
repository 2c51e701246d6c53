#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_dense_tc.py -q -x 2>&1 | tail -30 > gpurun_out/pytest_tc.txt
cat gpurun_out/pytest_tc.txt
