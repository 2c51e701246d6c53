#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_dense_tc.py tests/test_gpu_dispatch.py -q -x 2>&1 | tail -5 > gpurun_out/pytest_tcd.txt
cat gpurun_out/pytest_tcd.txt
bash tools/gpu_r02l.sh
