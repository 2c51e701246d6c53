#!/bin/bash
# weight / entry prefetch before the PDL wait: full GPU suite, bench, dispatch networks
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --no-cfg1 > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step'], d['e2e']['value'], d['parity']['bitwise'])"
timeout 900 python tools/bench_variants.py --only resnet50-net-fp16 --steps 30 > gpurun_out/disp_resnet.jsonl 2> gpurun_out/disp.err
timeout 900 python tools/bench_variants.py --only vgg16-fp16 --steps 30 > gpurun_out/disp_vgg.jsonl 2>> gpurun_out/disp.err
for f in gpurun_out/disp_resnet.jsonl gpurun_out/disp_vgg.jsonl; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['images_per_s'], d['dispatch']['images_per_s'], d['dispatch']['ms_per_step'], d['dispatch']['speedup_vs_cudnn'])"; done
