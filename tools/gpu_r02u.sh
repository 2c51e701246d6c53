#!/bin/bash
# split-K tensor-core path: tests, probe, dispatch re-search
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense_tc.py tests/test_gpu_pool.py tests/test_gpu_dispatch.py -q -x 2>&1 | tail -8 > gpurun_out/pytest_tc.txt
cat gpurun_out/pytest_tc.txt
grep -q "passed" gpurun_out/pytest_tc.txt && ! grep -q "failed\|error" gpurun_out/pytest_tc.txt || exit 1
timeout 600 python tools/tc_probe.py > gpurun_out/tc_probe.jsonl 2> gpurun_out/tc_probe.err
cat gpurun_out/tc_probe.jsonl; tail -3 gpurun_out/tc_probe.err
export RETUNE_DISPATCH=1
timeout 900 python tools/bench_variants.py --only vgg16-fp16 --steps 30 > gpurun_out/disp_vgg.jsonl 2> gpurun_out/disp.err
timeout 1500 python tools/bench_variants.py --only resnet50-net-fp16 --steps 30 > gpurun_out/disp_resnet.jsonl 2>> gpurun_out/disp.err
for f in gpurun_out/disp_resnet.jsonl gpurun_out/disp_vgg.jsonl; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['images_per_s'], d['dispatch']['images_per_s'], d['dispatch']['ms_per_step'], d['dispatch']['speedup_vs_cudnn'], d['dispatch']['backends'])"; done
tail -2 gpurun_out/disp.err
