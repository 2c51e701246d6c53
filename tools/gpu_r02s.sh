#!/bin/bash
# PDL on the tensor-core kernel and the BI pool: tests, dispatch networks with and without PDL
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense_tc.py tests/test_gpu_pool.py tests/test_gpu_dispatch.py -q -x 2>&1 | tail -8 > gpurun_out/pytest_tc.txt
cat gpurun_out/pytest_tc.txt
cp gpurun_out/r02_tuned_resnet50_fp16_dispatch.json profiles/ 2>/dev/null; cp gpurun_out/r02_tuned_vgg16_fp16_dispatch.json profiles/ 2>/dev/null
for pdl in 0 1; do
  if [ $pdl = 0 ]; then export USC_NO_PDL=1; else unset USC_NO_PDL; fi
  timeout 900 python tools/bench_variants.py --only resnet50-net-fp16 --steps 30 > gpurun_out/disp_resnet_pdl$pdl.jsonl 2> gpurun_out/disp.err
  timeout 900 python tools/bench_variants.py --only vgg16-fp16 --steps 30 > gpurun_out/disp_vgg_pdl$pdl.jsonl 2>> gpurun_out/disp.err
done
for f in gpurun_out/disp_*_pdl*.jsonl; do echo $f; python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['dispatch']['images_per_s'], d['dispatch']['ms_per_step'])"; done
tail -3 gpurun_out/disp.err
