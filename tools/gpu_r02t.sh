#!/bin/bash
# PDL on k_bi + k_dtc + BI pool: full GPU suite, headline bench with/without PDL, dispatch networks
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -8 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
USC_NO_PDL=1 timeout 900 python bench.py --no-cfg1 > gpurun_out/bench_nopdl.json 2> gpurun_out/bench.err
timeout 900 python bench.py > gpurun_out/bench.json 2>> gpurun_out/bench.err
for f in gpurun_out/bench_nopdl.json gpurun_out/bench.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['e2e']['value'], d.get('parity'))"; done
timeout 900 python tools/bench_variants.py --only resnet50-net-fp16 --steps 30 > gpurun_out/disp_resnet.jsonl 2> gpurun_out/disp.err
timeout 900 python tools/bench_variants.py --only vgg16-fp16 --steps 30 > gpurun_out/disp_vgg.jsonl 2>> gpurun_out/disp.err
for f in gpurun_out/disp_resnet.jsonl gpurun_out/disp_vgg.jsonl; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['images_per_s'], d['dispatch']['images_per_s'], d['dispatch']['ms_per_step'], d['dispatch']['speedup_vs_cudnn'])"; done
tail -3 gpurun_out/bench.err gpurun_out/disp.err
